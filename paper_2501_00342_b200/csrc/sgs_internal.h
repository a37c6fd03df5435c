// sgs_internal.h -- device data layout shared by the sm_100a kernels.
//
// See DESIGN.md for the roofline of each stage. Reference anchors:
//   K1 preprocess   proj/src/raster.cpp:17-80 (+ color.cpp:99-235, scene.cpp:81-85)
//   K2 depth sort   proj/src/raster.cpp:93-105
//   K3/K4 binning   proj/src/raster.cpp:108-130
//   K5/K6 tile sort + ranges  TileGrid::lists, raster.hpp:86-90
//   K7 composite    proj/src/raster.cpp:155-186
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "sgs.h"

namespace sgs {

// Blending constants, raster.hpp:27-30.
constexpr double kCovarianceDilation = 0.3;
constexpr double kSupportMahalanobisSq = 9.0;
constexpr double kAlphaClamp = 0.999;
constexpr double kAlphaMin = 1.0 / 255.0;

// Data-dependent error codes raised by K1 (the reference's throw sites).
enum DeviceError : uint32_t {
    kErrNone = 0,
    kErrZeroQuaternion = 1,   // common.hpp:126        -> NumericError
    kErrThresholds = 2,       // raster.cpp:9          -> InvalidArgument
    kErrOverrideNonMixed = 3, // raster.cpp:75-76      -> InvalidArgument
    kErrDegreeTooHigh = 4,    // color.cpp:184-189     -> InvalidArgument
    kErrDirection = 5,        // color.cpp:10-16       -> InvalidArgument
};

// Camera constants in FP64, precomputed on the host in the reference's
// operation order (camera.hpp:19-20, raster.cpp:29-30).
struct CamParams {
    double R[9];
    double t[3];
    double C[3];  // -R^T t
    double fx, fy, cx, cy;
    double width, height;
    double near_plane;
    double lim_x, lim_y;  // 1.3 * (0.5 * W / fx)
    int32_t W, H;
};

struct CfgParams {
    int32_t tile_size;
    int32_t tiles_x, tiles_y;
    int32_t has_override, override_degree;
    double lo, hi;
    float early_stop;
};

// Scene planes inside one device blob.
struct ScenePlanes {
    uint64_t n;
    int32_t kind;
    int32_t sh_degree;  // stored
    int32_t geometry_f64;
    int32_t color_planes;  // float4 planes
    // geometry: f32 -> g4[0..2] (pos+opl, quat, logscale); f64 -> g8[0..10]
    const float4* g4[3];
    const double* g8[11];
    const float4* color;  // color_planes consecutive planes of n float4
    float axes[9];        // row-major lobe axes
    float bg[3];
};

// Compositing record written by K1 for visible splats (48 B, 16-B aligned).
struct __align__(16) SplatRec {
    double mx, my;      // mean2d in pixels (FP64 so the compositor can localise exactly)
    float ca, cb2, cc;  // conic (a, 2b, c)
    float op;           // activated opacity
    float r, g, b;      // colour
    float guard;        // FP32 m2 error bound -> FP64 guard band width
};

// FP64 side record read only inside the guard band (32 B).
struct __align__(16) SplatRec64 {
    double ca, cb, cc, op;
};

// Debug record for sgs_project (same field order as sgs_splat).
struct DebugSplat {
    double mean2d[2];
    double conic[3];
    double depth;
    double color[3];
    double opacity;
    double radius;
    int32_t degree;
    int32_t visible;
};

struct Counters {
    unsigned long long err;  // (gaussian << 8) | code, atomicMin; ~0 = none
    unsigned long long visible;
    unsigned long long block_entries;
    unsigned long long guard_hits;
    unsigned long long tile_entries;
};

// Number of float4 colour planes for (kind, stored degree).
inline int color_plane_count(int kind, int degree) {
    int ncoef = (degree + 1) * (degree + 1);
    switch (kind) {
        case SGS_SH: return (3 * ncoef + 3) / 4;
        case SGS_SG1: return 3;
        case SGS_SG3: return 4;
        case SGS_MIXED: return (3 * ncoef + 3) / 4 + 3;
    }
    return 0;
}

// Launchers (defined in the .cu files).
void launch_preprocess(const ScenePlanes& sp, const CamParams& cam, const CfgParams& cfg,
                       unsigned long long* depth_keys, uint32_t* iota, SplatRec* rec,
                       SplatRec64* rec64, int4* rects, uint32_t* ntiles, Counters* counters,
                       DebugSplat* debug, cudaStream_t stream);
void launch_gather_counts(uint64_t n, const uint32_t* order, const uint32_t* ntiles,
                          unsigned long long* counts, cudaStream_t stream);
void launch_emit_tile_keys(uint64_t n_visible, const uint32_t* order, const uint32_t* ntiles,
                           const int4* rects, const unsigned long long* offsets, int tiles_x,
                           unsigned long long* keys, cudaStream_t stream);
void launch_tile_ranges(uint64_t p, const unsigned long long* keys, uint2* ranges,
                        cudaStream_t stream);
void launch_composite(const CamParams& cam, const CfgParams& cfg, const uint2* ranges,
                      const unsigned long long* keys, const SplatRec* rec,
                      const SplatRec64* rec64, float3 bg, float* rgb, float* T,
                      Counters* counters, bool want_stats, cudaStream_t stream);

}  // namespace sgs
