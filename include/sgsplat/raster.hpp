// sgsplat/raster.hpp -- the forward render API, served by the B200 (sm_100a) renderer.
//
// Drop-in for proj/include/sgsplat/raster.hpp:11-62: RenderConfig, the blending
// constants, Splat2D, select_degree, project, RenderResult, render and
// flops_per_gaussian with the reference's signatures. render() and project() run
// the CUDA path through the C-ABI in include/sgs.h (libsgs_b200.so); there is no
// CPU fallback. The reference's detail:: internals (shared with its backward pass)
// are not part of this library.
#pragma once

#include "sgsplat/camera.hpp"
#include "sgsplat/image.hpp"
#include "sgsplat/scene.hpp"

#include <optional>

namespace sgsplat {

struct RenderConfig {
    int tile_size = 16;
    double degree_threshold_lo = 2.0;  // mixed model: radius < lo -> SH degree 0
    double degree_threshold_hi = 8.0;  //              radius < hi -> 1, else 2
    std::optional<int> sh_degree_override;
    double early_stop_transmittance = 1e-4;
    int threads = 0;  // accepted for API parity; the CUDA grid replaces it
};

inline constexpr double kCovarianceDilation = 0.3;
inline constexpr double kSupportMahalanobisSq = 9.0;
inline constexpr double kAlphaClamp = 0.999;
inline constexpr double kAlphaMin = 1.0 / 255.0;

struct Splat2D {
    Vec2 mean2d = Vec2::Zero();
    Vec3 conic = Vec3::Zero();
    double depth = 0.0;
    Vec3 color = Vec3::Zero();
    double opacity = 0.0;
    double radius_px = 0.0;
};

int select_degree(double radius_px, double lo, double hi);

std::optional<Splat2D> project(const GaussianPrimitive& g, const Camera& cam, const Mat3& shared_axes,
                               const RenderConfig& cfg = {});

struct RenderResult {
    Image image;          // H x W x 3 linear RGB
    Image transmittance;  // H x W x 1
};

RenderResult render(const Scene& scene, const Camera& cam, const RenderConfig& cfg = {});

int flops_per_gaussian(ColorModelKind kind, int sh_degree = 3);

}  // namespace sgsplat
