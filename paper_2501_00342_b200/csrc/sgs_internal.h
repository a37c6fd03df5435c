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
#include <string>

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
    int32_t tight_rect;  // K1: tile rectangles of the cut ellipse's box, not the 3-sigma circle's
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
    const double2* cov[3];  // cached 3D covariance (projection.cuh covariance3d)
    const double* color64;  // FP64 colour parameters [k * n + i] when not f32-exact, else null
    const float4* color;  // color_planes consecutive planes of n float4
    float axes[9];        // row-major lobe axes
    float bg[3];
};

// Per-frame constants in device memory, read by K7's cold FP64 guard-band path
// (kept out of kernel parameters so the hot loop does not carry them).
struct FrameConsts {
    ScenePlanes sp;
    CamParams cam;
    float* out_rgb;  // the frame's outputs (K7 reads them here, so a captured frame graph
    float* out_T;    // replays with new output buffers); either may be null
};

// Compositing record written by K1 for visible splats (48 B, 16-B aligned); the
// colour (16 B) goes to a separate float4 array.
// The reference's two skip tests (m2 > 9, alpha < 1/255) are one cutoff on m2:
// alpha < 1/255 <=> m2 > 2 ln(255 op), so cut = min(9, 2 ln(255 op)) (FP64 in K1).
struct __align__(16) SplatRec {
    double mx, my;      // mean2d in pixels (FP64 so the compositor can localise exactly)
    float ca, cb2, cc;  // conic (a, 2b, c)
    float lop;          // log2(opacity)
    float cut;          // min(9, 2 ln(255 op))
    float guard;        // FP32 m2 error bound -> FP64 guard band half-width
    float ext_x, ext_y; // half extents of {m2 <= cut + guard} (warp culling box)
};
static_assert(sizeof(SplatRec) == 48, "splat record");

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
    unsigned long long kmin;  // min / max orderable depth key of the visible splats
    unsigned long long kmax;
    unsigned long long reserved0[2];
    unsigned long long key_overflow;  // a chunk needed more tile keys than allocated
    unsigned long long max_chunk_entries;  // largest chunk P (sizes the retry)
    unsigned long long chunk_entries;  // P of the chunk in flight (clamped to capacity)
    unsigned long long reserved1[4];
};
static_assert(sizeof(Counters) == 128, "counters block");

// Tiles of an inclusive tile rectangle (x0, x1, y0, y1); empty when x1 < x0 or y1 < y0.
__host__ __device__ inline uint32_t rect_area(int4 rc) {
    return rc.y >= rc.x && rc.w >= rc.z ? static_cast<uint32_t>(rc.y - rc.x + 1) * static_cast<uint32_t>(rc.w - rc.z + 1)
                                        : 0u;
}

// Per-pixel compositing state carried between depth chunks (K7).
struct __align__(16) PixelState {
    float r, g, b, T;
};

// Number of float4 colour planes for (kind, stored degree).
inline int color_plane_count(int kind, int degree) {
    int ncoef = (degree + 1) * (degree + 1);
    switch (kind) {
        case SGS_SH: return (3 * ncoef + 3) / 4;
        case SGS_SG1: return 4;  // + raw lobe axis (plane 3) for the backward
        case SGS_SG3: return 4;
        case SGS_MIXED: return (3 * ncoef + 3) / 4 + 3;
    }
    return 0;
}

// Launchers (defined in the .cu files).
void launch_preprocess(const ScenePlanes& sp, const CamParams& cam, const CfgParams& cfg,
                       unsigned long long* depth_keys, SplatRec* rec, int4* rects,
                       float4* colour, Counters* counters, DebugSplat* debug,
                       cudaStream_t stream);
// K1's outputs for its view. (A multi-view K1 -- every Gaussian read once, projected
// into up to 4 views' arenas, SURVEY.md §8f row 1 -- was built and measured: 152 us
// per view at NV=1, 154 at NV=2, 167 at NV=4, batch throughput 0.719 vs 0.724 ms per
// frame, because with the covariance cached K1 is bound by its per-view FP64 work and
// writes, not by the shared scene read. It is not kept.)
struct K1Out {
    unsigned long long* keys;
    SplatRec* rec;
    int4* rects;
    float4* colour;
    Counters* ctr;
    CamParams cam;
};
// The last K1 launch of this thread (function, configuration, arguments), so a frame
// graph can patch the camera of its captured K1 node (capi.cu launch_frame_graph).
struct K1Record;
K1Record* k1_last_launch_clone();
void k1_record_free(K1Record* r);
const void* k1_record_func(const K1Record* r);
cudaError_t k1_record_patch(cudaGraphExec_t exec, cudaGraphNode_t node, K1Record* r, const CamParams& cam);
// per-scene 3D covariance cache: 3 planes of n double2 (projection.cuh)
void launch_cov3d(const ScenePlanes& sp, double2* cov, cudaStream_t stream);
// The digit split of a tile-id sort: passes of <= 8 bits, LSD first.
struct TileDigits {
    int passes;
    int shift[4];
    int bits[4];
};
// Per-slice digit histograms of one pass (radix_hist_words() u32).
size_t radix_hist_words();
// One stable pass on bits [shift, shift + bits) of *dcount (key, value) pairs.
cudaError_t launch_radix_pass(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                              const unsigned long long* dcount, int shift, int bits, uint32_t* hist,
                              cudaStream_t stream);
// K2 (depth_sort.cu): the depth order of n splats -- order[r], and the rank-ordered
// binning inputs brect[r] / bmeta[r] = (index, tiles of its rectangle) -- by a
// two-level bucket sort. Scratch: ghist / cur depth_two_level_scratch bytes each,
// part 16 n bytes, tmp_idx n u32; key (K1's, dead once partitioned) doubles as the
// big buckets' merge scratch.
int depth_coarse_log2(uint64_t n);
size_t depth_two_level_scratch(int log2c);
cudaError_t launch_depth_two_level(uint64_t n, unsigned long long* key, Counters* ctr, int log2c,
                                   uint32_t* ghist, uint32_t* cur, void* part, uint32_t* order,
                                   uint32_t* tmp_idx, const int4* rects, int4* brect, uint2* bmeta,
                                   cudaStream_t stream, uint64_t* launches);
// K3 + K4 (binning.cu): for the ranks [rb, re) of a depth chunk, count each rank's
// live tiles, then emit the (tile id, Gaussian index) pairs into tk / tv in rank order
// at offsets each CTA scans itself; the chunk's P goes to ctr (chunk_entries).
// scratch: bin_scratch_bytes(ranks) bytes.
size_t bin_scratch_bytes(uint64_t ranks);
cudaError_t launch_binning(uint64_t rb, uint64_t re, const uint2* bmeta, const int4* brect, const uint32_t* done,
                           int tiles_x, int ntile, uint32_t* tk, uint32_t* tv, uint64_t capacity, void* scratch,
                           Counters* ctr, cudaStream_t stream, uint64_t* launches);
TileDigits tile_digits(int tile_bits);
// backward (backward.cu)
size_t bwd_splat_bytes();
size_t bwd_partial_bytes();
void launch_finite_check(const double* v, size_t n, int* bad, cudaStream_t s);
void launch_backward(const ScenePlanes& sp, const CamParams& cam, const CfgParams& cfg, const double* axes,
                     const double* bg, int override_degree, uint64_t V, int nchunks, const uint32_t* order,
                     const int4* brect, const uint2* ranges, const uint32_t* keys, void* bs,
                     uint32_t* rank_of, uint32_t* used, double* partial, const double* upstream, double* grads,
                     int stride, cudaStream_t s);
void launch_render_f64(const ScenePlanes& sp, const CamParams& cam, const CfgParams& cfg, const double* axes,
                       const double* bg, int override_degree, uint64_t V, int nchunks, const uint32_t* order,
                       const uint2* ranges, const uint32_t* keys, void* bs, uint32_t* rank_of, double* rgb,
                       double* T, cudaStream_t s);
// image metrics (metrics.cu)
size_t metrics_scratch_doubles(size_t n, bool grad);
void launch_psnr_sum(const void* a, const void* b, bool f64, size_t n, double* scratch, double* d_sum,
                     cudaStream_t s);
void launch_ssim(const void* a, const void* b, bool f64, int W, int H, int C, double* scratch, double* d_sum,
                 double* grad, cudaStream_t s);
void launch_counters_init(Counters* c, cudaStream_t stream);
void launch_counters_publish(const Counters* d, Counters* h_mapped, cudaStream_t stream);
// K6: ranges[t] = [first, last + 1) of tile t's run in the sorted tile ids; the
// count is read from device memory.
void launch_tile_ranges(const unsigned long long* d_count, const uint32_t* tiles, uint2* ranges,
                        cudaStream_t stream);
// K7 over one depth chunk (builds the chunk's work list first). first/last select
// state init / final output; tile_done and state may be null when the frame is a
// single chunk.
cudaError_t launch_composite(const FrameConsts* fc, const CamParams& cam, const CfgParams& cfg,
                             const uint2* ranges, const uint32_t* keys, const SplatRec* rec,
                             const float4* colour, float3 bg, PixelState* state, uint32_t* processed,
                             uint32_t* tile_flags, bool first, bool last, Counters* counters, bool want_stats,
                             uint32_t* tile_emax, uint32_t* work, uint32_t* wctl, cudaStream_t stream);
// K7 work items per tile (64-pixel parts) and the per-tile flag block's size in words
int composite_work_items(int tile_size);
size_t composite_flag_words(uint32_t ntile);
int composite_pixel_chunks(int tile_size);

// capi.cu helpers for group.cu: the last-error text, a context's device and render
// stream, and binding a device blob the scene then owns (freed with it).
sgs_status fail_status(sgs_status code, const std::string& msg);
int context_device(const sgs_context* ctx);
void context_stream(const sgs_context* ctx, cudaStream_t* stream);
sgs_status scene_bind_owned(sgs_context* ctx, const sgs_scene_meta* meta, void* blob, uint64_t bytes,
                            sgs_scene** out);

}  // namespace sgs
