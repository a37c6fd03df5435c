// backward.cu -- GPU backward of render (grad.hpp, grad.cpp:69-246).
//
// d(sum_pixels upstream . rendered) / d(stored parameters), for the reference's
// backward(scene, cam, cfg, upstream). It reuses the forward's exact products: the
// depth order, and the full per-tile lists (one depth chunk) that sgs_debug_tile_grid
// also returns, so every hit decision is the reference's.
//
//   B1 bwd_prep    per visible splat, in FP64: the reference's Splat2D (mean, exact
//                  conic, sigmoid opacity) and its FP64 view-dependent colour
//                  (eval_color, color.cpp:201-235), plus rank_of[gaussian].
//   B2 bwd_pixels  one CTA per tile, one pixel per thread: the per-pixel forward
//                  (grad.cpp:96-121, FP64) finds the last hit, then the reverse walk
//                  (:122-141) rebuilds T before each hit as T / (1 - alpha) and forms
//                  the 9 screen-space partials (colour 3, opacity, mean 2, conic 3).
//                  They are summed over the tile's pixels with a fixed-order warp tree
//                  and a fixed-order sum over warps, into one slot per tile-list entry
//                  -- no float atomics, so the result is deterministic.
//   B3 bwd_splat   per visible splat: sums its entries over the tiles of its rect
//                  (row-major; each found by binary search on rank, the lists being
//                  in depth order), then chains through projection, covariance, the
//                  activations and the colour model (grad.cpp:155-244, grad_color
//                  color.cpp:291-358).
// The arithmetic is FP64 throughout, and this file is compiled without FMA
// contraction (Makefile: -fmad=false), as the reference's x86-64 build rounds; the
// per-splat sums run in different orders than the reference's worker-merged buffers,
// so gradients agree to rounding (tests state the tolerance), not bit for bit.
// The same splats feed render_f64_kernel, the reference's render loop in FP64.
#include "projection.cuh"

namespace sgs {
namespace {

constexpr int kBThreads = 256;
constexpr int kBWarps = kBThreads / 32;
constexpr int kBE = 32;  // tile-list entries per reduction batch
constexpr int kNP = 9;   // partials per (pixel, splat): colour rgb, opacity, mean xy, conic 00 01 11

struct BwdSplat {
    double mx, my, c0, c1, c2, op, cr, cg, cb, pad;
};

struct BwdParams {
    ScenePlanes sp;
    CamParams cam;
    CfgParams cfg;
    double axes[9];
    double bg[3];
    int override_degree;  // -1: adaptive (select_degree)
    int tiles_x;
};

// SH constants (color.hpp:15-26)
__constant__ double kD0 = 0.28209479177387814;
__constant__ double kD1 = 0.4886025119029199;
__constant__ double kD2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                              -1.0925484305920792, 0.5462742152960396};
__constant__ double kD3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                              -0.4570457994644658, 1.445305721320277, -0.5900435899266435};

// eval_sh_basis (color.cpp:99-131)
__device__ void sh_basis(double x, double y, double z, int deg, double* b) {
    b[0] = kD0;
    if (deg >= 1) {
        b[1] = -kD1 * y;
        b[2] = kD1 * z;
        b[3] = -kD1 * x;
    }
    if (deg >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[4] = kD2[0] * x * y;
        b[5] = kD2[1] * y * z;
        b[6] = kD2[2] * (2.0 * zz - xx - yy);
        b[7] = kD2[3] * x * z;
        b[8] = kD2[4] * (xx - yy);
    }
    if (deg >= 3) {
        const double xx = x * x, yy = y * y, zz = z * z;
        b[9] = kD3[0] * y * (3.0 * xx - yy);
        b[10] = kD3[1] * x * y * z;
        b[11] = kD3[2] * y * (4.0 * zz - xx - yy);
        b[12] = kD3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
        b[13] = kD3[4] * x * (4.0 * zz - xx - yy);
        b[14] = kD3[5] * z * (xx - yy);
        b[15] = kD3[6] * x * (xx - 3.0 * yy);
    }
}

// sh_basis_direction_grads (color.cpp:135-161), g[i] = dY_i / d(x, y, z)
__device__ void sh_dbasis(double x, double y, double z, int deg, double (*g)[3]) {
    for (int i = 0; i < 16; ++i) g[i][0] = g[i][1] = g[i][2] = 0.0;
    if (deg >= 1) {
        g[1][1] = -kD1;
        g[2][2] = kD1;
        g[3][0] = -kD1;
    }
    if (deg >= 2) {
        g[4][0] = kD2[0] * y, g[4][1] = kD2[0] * x;
        g[5][1] = kD2[1] * z, g[5][2] = kD2[1] * y;
        g[6][0] = kD2[2] * (-2 * x), g[6][1] = kD2[2] * (-2 * y), g[6][2] = kD2[2] * (4 * z);
        g[7][0] = kD2[3] * z, g[7][2] = kD2[3] * x;
        g[8][0] = kD2[4] * (2 * x), g[8][1] = kD2[4] * (-2 * y);
    }
    if (deg >= 3) {
        const double xx = x * x, yy = y * y, zz = z * z;
        g[9][0] = kD3[0] * (6 * x * y), g[9][1] = kD3[0] * (3 * xx - 3 * yy);
        g[10][0] = kD3[1] * (y * z), g[10][1] = kD3[1] * (x * z), g[10][2] = kD3[1] * (x * y);
        g[11][0] = kD3[2] * (-2 * x * y), g[11][1] = kD3[2] * (4 * zz - xx - 3 * yy), g[11][2] = kD3[2] * (8 * y * z);
        g[12][0] = kD3[3] * (-6 * x * z), g[12][1] = kD3[3] * (-6 * y * z),
        g[12][2] = kD3[3] * (6 * zz - 3 * xx - 3 * yy);
        g[13][0] = kD3[4] * (4 * zz - 3 * xx - yy), g[13][1] = kD3[4] * (-2 * x * y), g[13][2] = kD3[4] * (8 * x * z);
        g[14][0] = kD3[5] * (2 * x * z), g[14][1] = kD3[5] * (-2 * y * z), g[14][2] = kD3[5] * (xx - yy);
        g[15][0] = kD3[6] * (3 * xx - 3 * yy), g[15][1] = kD3[6] * (-6 * x * y);
    }
}

// Flat colour parameter k (color.hpp:121-128 order) of Gaussian i, from the planes
// (fill_blob's layout: SG1 keeps the raw lobe axis in plane 3).
template <int KIND>
__device__ __forceinline__ double cparam(const ScenePlanes& sp, uint64_t i, int k) {
    if (sp.color64) return sp.color64[static_cast<uint64_t>(k) * sp.n + i];  // not f32-exact: FP64 copies
    int slot = k;
    if constexpr (KIND == SGS_MIXED) {
        const int nsh = 3 * (sp.sh_degree + 1) * (sp.sh_degree + 1);
        if (k >= nsh) slot = 4 * ((nsh + 3) / 4) + (k - nsh);
    } else if constexpr (KIND == SGS_SG1) {
        // [diffuse rgb, alpha rgb, log_lambda, mu xyz] -> planes (d, logl) (a, -) (mu_hat, -) (mu, -)
        slot = k < 3 ? k : (k < 6 ? 4 + (k - 3) : (k == 6 ? 3 : 12 + (k - 7)));
    } else if constexpr (KIND == SGS_SG3) {
        slot = k < 3 ? k : 4 + (k - 3);
    }
    const float* plane = reinterpret_cast<const float*>(sp.color + static_cast<uint64_t>(slot >> 2) * sp.n + i);
    return static_cast<double>(plane[slot & 3]);
}

__device__ __forceinline__ double dot3d(const double* a, const double* b) {
    return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2];
}

// SG1 lobe (DiffuseSGModel::lobe, color.cpp:52-59): lambda, unit mu; returns |mu_raw|
template <int KIND>
__device__ double sg1_lobe(const ScenePlanes& sp, uint64_t i, double* mu_hat, double* lambda) {
    const double m[3] = {cparam<KIND>(sp, i, 7), cparam<KIND>(sp, i, 8), cparam<KIND>(sp, i, 9)};
    const double n = sqrt(dot3d(m, m));
    for (int k = 0; k < 3; ++k) mu_hat[k] = n > 1e-12 ? m[k] / n : (k == 0 ? 1.0 : 0.0);
    *lambda = exp(cparam<KIND>(sp, i, 6));
    return n;
}

// pre-clamp colour (pre_clamp_color, color.cpp:244-271)
template <int KIND>
__device__ void pre_colour(const BwdParams& p, uint64_t i, int deg, const double* d, double* pre) {
    const ScenePlanes& sp = p.sp;
    if constexpr (KIND == SGS_SH || KIND == SGS_MIXED) {
        double b[16];
        sh_basis(d[0], d[1], d[2], deg, b);
        double acc[3] = {0.0, 0.0, 0.0};
        const int n = (deg + 1) * (deg + 1);
        for (int k = 0; k < n; ++k)
            for (int c = 0; c < 3; ++c) acc[c] += b[k] * cparam<KIND>(sp, i, 3 * k + c);
        for (int c = 0; c < 3; ++c) pre[c] = 0.5 + acc[c];
        if constexpr (KIND == SGS_MIXED) {
            const int nsh = 3 * (sp.sh_degree + 1) * (sp.sh_degree + 1);
            double lobes[3] = {0.0, 0.0, 0.0};
            for (int l = 0; l < 3; ++l) {
                const double lambda = exp(cparam<KIND>(sp, i, nsh + 4 * l + 3));
                const double e = exp(lambda * (dot3d(p.axes + 3 * l, d) - 1.0));
                for (int c = 0; c < 3; ++c) lobes[c] += cparam<KIND>(sp, i, nsh + 4 * l + c) * e;
            }
            for (int c = 0; c < 3; ++c) pre[c] += lobes[c];
        }
    } else if constexpr (KIND == SGS_SG1) {
        double mu[3], lambda;
        sg1_lobe<KIND>(sp, i, mu, &lambda);
        const double e = exp(lambda * (dot3d(d, mu) - 1.0));
        for (int c = 0; c < 3; ++c) pre[c] = cparam<KIND>(sp, i, c) + cparam<KIND>(sp, i, 3 + c) * e;
    } else {
        double lobes[3] = {0.0, 0.0, 0.0};
        for (int l = 0; l < 3; ++l) {
            const double lambda = exp(cparam<KIND>(sp, i, 3 + 4 * l + 3));
            const double e = exp(lambda * (dot3d(p.axes + 3 * l, d) - 1.0));
            for (int c = 0; c < 3; ++c) lobes[c] += cparam<KIND>(sp, i, 3 + 4 * l + c) * e;
        }
        for (int c = 0; c < 3; ++c) pre[c] = cparam<KIND>(sp, i, c) + lobes[c];
    }
}

// The splat's cached projection quantities (project_cached, raster.cpp:17-80).
struct Proj {
    Geo geo;
    ProjGeo pg;
    double dir[3], dist;
    int deg;
};

template <bool F64, int KIND>
__device__ void project_full(const BwdParams& p, uint64_t g, Proj& q) {
    project_geometry<F64>(p.sp, p.cam, g, q.geo, q.pg);
    exact_conic_opacity(q.geo, q.pg);
    const double off[3] = {q.geo.p[0] - p.cam.C[0], q.geo.p[1] - p.cam.C[1], q.geo.p[2] - p.cam.C[2]};
    q.dist = sqrt(dot3d(off, off));
    for (int k = 0; k < 3; ++k) q.dir[k] = off[k] / q.dist;
    q.deg = p.sp.sh_degree;
    if constexpr (KIND == SGS_MIXED) {
        q.deg = p.override_degree >= 0 ? p.override_degree
                                       : (q.pg.radius < p.cfg.lo ? 0 : (q.pg.radius < p.cfg.hi ? 1 : 2));
    }
}

template <bool F64, int KIND>
__global__ void bwd_prep_kernel(const BwdParams p, uint64_t V, const uint32_t* __restrict__ order,
                                BwdSplat* __restrict__ bs, uint32_t* __restrict__ rank_of) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const uint32_t g = order[r];
    rank_of[g] = static_cast<uint32_t>(r);
    Proj q;
    project_full<F64, KIND>(p, g, q);
    double pre[3];
    pre_colour<KIND>(p, g, q.deg, q.dir, pre);
    BwdSplat s;
    s.mx = q.pg.mx, s.my = q.pg.my;
    s.c0 = q.pg.cona, s.c1 = q.pg.conb, s.c2 = q.pg.conc, s.op = q.pg.opacity;
    s.cr = pre[0] < 0.0 ? 0.0 : pre[0];  // cwiseMax(0)
    s.cg = pre[1] < 0.0 ? 0.0 : pre[1];
    s.cb = pre[2] < 0.0 ? 0.0 : pre[2];
    s.pad = 0.0;
    bs[g] = s;
}

struct Hit {
    bool hit, clamped;
    double alpha, gauss, dx, dy;
};

// One (pixel, splat) blend decision of the backward's forward (grad.cpp:103-118).
__device__ __forceinline__ Hit pixel_hit(const BwdSplat& s, double cx, double cy) {
    Hit h{};
    h.dx = cx - s.mx;
    h.dy = cy - s.my;
    const double m2 = s.c0 * h.dx * h.dx + 2.0 * s.c1 * h.dx * h.dy + s.c2 * h.dy * h.dy;
    if (m2 > kSupportMahalanobisSq) return h;
    h.gauss = exp(-0.5 * m2);
    h.alpha = s.op * h.gauss;
    h.clamped = h.alpha > kAlphaClamp;
    if (h.clamped) h.alpha = kAlphaClamp;
    h.hit = !(h.alpha < kAlphaMin);
    return h;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(kBThreads) bwd_pixels_kernel(
    const BwdParams p, int nchunks, const uint2* __restrict__ ranges, const uint32_t* __restrict__ keys,
    const BwdSplat* __restrict__ bs, const double* __restrict__ upstream, double* __restrict__ partial,
    uint32_t* __restrict__ used) {
    __shared__ double sAcc[kBWarps][kBE][kNP];
    __shared__ int sMax[kBWarps];
    const int tile = blockIdx.x;
    const uint2 range = ranges[tile];
    const int start = static_cast<int>(range.x), end = static_cast<int>(range.y);
    const int ts = p.cfg.tile_size;
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int W = p.cam.width, H = p.cam.height;
    const double stop = p.cfg.early_stop;
    int tile_used = 0;
    for (int ch = 0; ch < nchunks; ++ch) {
        const int pp = ch * kBThreads + threadIdx.x;
        const int lx = pp % ts, ly = pp / ts;
        const int px = tx * ts + lx, py = ty * ts + ly;
        const bool valid = pp < ts * ts && px < W && py < H;
        const double cx = px + 0.5, cy = py + 0.5;
        // forward: the last hit index and the final transmittance
        double T = 1.0;
        int last = start - 1;
        if (valid) {
            for (int j = start; j < end; ++j) {
                const BwdSplat s = bs[keys[j]];
                const Hit h = pixel_hit(s, cx, cy);
                if (!h.hit) continue;
                T *= 1.0 - h.alpha;
                last = j;
                if (T < stop) break;
            }
        }
        int m = last;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) sMax[warp] = m;
        __syncthreads();
        int cta_last = start - 1;
        for (int w = 0; w < kBWarps; ++w) cta_last = max(cta_last, sMax[w]);
        __syncthreads();
        const int prev_used = tile_used;  // entries already holding sums of earlier pixel chunks
        tile_used = max(tile_used, cta_last - start + 1);
        double gup[3] = {0.0, 0.0, 0.0};
        if (valid)
            for (int c = 0; c < 3; ++c) gup[c] = upstream[(static_cast<size_t>(py) * W + px) * 3 + c];
        double suffix[3] = {T * p.bg[0], T * p.bg[1], T * p.bg[2]};
        // reverse walk in batches of kBE entries (descending), CTA-uniform
        for (int hi = cta_last; hi >= start; hi -= kBE) {
            double mine[kNP];  // lane e keeps entry (hi - e)'s warp sums
#pragma unroll
            for (int q = 0; q < kNP; ++q) mine[q] = 0.0;
            for (int e = 0; e < kBE; ++e) {
                const int j = hi - e;
                double c[kNP];
#pragma unroll
                for (int q = 0; q < kNP; ++q) c[q] = 0.0;
                if (j >= start && j <= last) {
                    const BwdSplat s = bs[keys[j]];
                    const Hit h = pixel_hit(s, cx, cy);
                    if (h.hit) {
                        const double Tb = T / (1.0 - h.alpha);  // transmittance before this splat
                        const double weight = h.alpha * Tb;
                        c[0] = weight * gup[0];
                        c[1] = weight * gup[1];
                        c[2] = weight * gup[2];
                        const double gc = (gup[0] * s.cr + gup[1] * s.cg) + gup[2] * s.cb;
                        const double gs = (gup[0] * suffix[0] + gup[1] * suffix[1]) + gup[2] * suffix[2];
                        const double d_alpha = gc * Tb - gs / (1.0 - h.alpha);
                        suffix[0] += weight * s.cr;
                        suffix[1] += weight * s.cg;
                        suffix[2] += weight * s.cb;
                        if (!h.clamped) {
                            c[3] = d_alpha * h.gauss;
                            const double d_m2 = -0.5 * d_alpha * s.op * h.gauss;
                            const double mx = 2.0 * (s.c0 * h.dx + s.c1 * h.dy);
                            const double my = 2.0 * (s.c1 * h.dx + s.c2 * h.dy);
                            c[4] = -(d_m2 * mx);
                            c[5] = -(d_m2 * my);
                            c[6] = d_m2 * (h.dx * h.dx);
                            c[7] = d_m2 * (h.dx * h.dy);
                            c[8] = d_m2 * (h.dy * h.dy);
                        }
                        T = Tb;
                    }
                }
#pragma unroll
                for (int q = 0; q < kNP; ++q) {
                    const double v = warp_sum(c[q]);
                    if (lane == e) mine[q] = v;
                }
            }
#pragma unroll
            for (int q = 0; q < kNP; ++q) sAcc[warp][lane][q] = mine[q];
            __syncthreads();
            for (int k = threadIdx.x; k < kBE * kNP; k += kBThreads) {
                const int e = k / kNP, q = k % kNP;
                const int j = hi - e;
                if (j < start) continue;
                double sum = 0.0;
                for (int w = 0; w < kBWarps; ++w) sum += sAcc[w][e][q];
                double* dst = partial + static_cast<size_t>(j) * kNP + q;
                *dst = j - start < prev_used ? *dst + sum : sum;
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) used[tile] = static_cast<uint32_t>(tile_used);
}

// The reference's per-pixel render loop (raster.cpp:155-186) in FP64 over the full
// tile lists, in its exact operation order (this file is compiled without FMA
// contraction): the exact mode behind sgs_render_f64.
__global__ void __launch_bounds__(kBThreads) render_f64_kernel(const BwdParams p, int nchunks,
                                                               const uint2* __restrict__ ranges,
                                                               const uint32_t* __restrict__ keys,
                                                               const BwdSplat* __restrict__ bs, double* __restrict__ rgb,
                                                               double* __restrict__ Tout) {
    const int tile = blockIdx.x;
    const uint2 range = ranges[tile];
    const int ts = p.cfg.tile_size;
    const int tx = tile % p.tiles_x, ty = tile / p.tiles_x;
    const int W = p.cam.width, H = p.cam.height;
    for (int ch = 0; ch < nchunks; ++ch) {
        const int pp = ch * kBThreads + threadIdx.x;
        const int lx = pp % ts, ly = pp / ts;
        const int px = tx * ts + lx, py = ty * ts + ly;
        if (!(pp < ts * ts && px < W && py < H)) continue;
        const double cx = px + 0.5, cy = py + 0.5;
        double acc[3] = {0.0, 0.0, 0.0};
        double T = 1.0;
        for (uint32_t j = range.x; j < range.y; ++j) {
            const BwdSplat s = bs[keys[j]];
            const double dx = cx - s.mx, dy = cy - s.my;
            const double m2 = s.c0 * dx * dx + 2.0 * s.c1 * dx * dy + s.c2 * dy * dy;
            if (m2 > kSupportMahalanobisSq) continue;
            const double a0 = s.op * exp(-0.5 * m2);
            const double alpha = kAlphaClamp < a0 ? kAlphaClamp : a0;  // std::min(a, 0.999): NaN stays NaN
            if (alpha < kAlphaMin) continue;
            const double w = alpha * T;
            acc[0] += s.cr * w;
            acc[1] += s.cg * w;
            acc[2] += s.cb * w;
            T *= 1.0 - alpha;
            if (T < p.cfg.early_stop) break;
        }
        const size_t pix = static_cast<size_t>(py) * W + px;
        for (int c = 0; c < 3; ++c) {
            acc[c] += T * p.bg[c];
            if (rgb) rgb[pix * 3 + c] = acc[c];
        }
        if (Tout) Tout[pix] = T;
    }
}

// rotation_quat_jacobians (grad.cpp:31-42), (w, x, y, z)
__device__ void quat_jacobians(const double* q, double (*J)[9]) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double j0[9] = {0, -z, y, z, 0, -x, -y, x, 0};
    const double j1[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
    const double j2[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
    const double j3[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
    for (int k = 0; k < 9; ++k) {
        J[0][k] = 2.0 * j0[k];
        J[1][k] = 2.0 * j1[k];
        J[2][k] = 2.0 * j2[k];
        J[3][k] = 2.0 * j3[k];
    }
}

template <bool F64>
__device__ void load_rot_scale(const ScenePlanes& sp, uint64_t i, double* q, double* ls) {
    if constexpr (F64) {
        for (int k = 0; k < 4; ++k) q[k] = sp.g8[3 + k][i];
        for (int k = 0; k < 3; ++k) ls[k] = sp.g8[7 + k][i];
    } else {
        const float4 b = sp.g4[1][i], c = sp.g4[2][i];
        q[0] = b.x, q[1] = b.y, q[2] = b.z, q[3] = b.w;
        ls[0] = c.x, ls[1] = c.y, ls[2] = c.z;
    }
}

// accumulate_lobe_grad (color.cpp:273-287)
__device__ void lobe_grad(const double* alpha, double lambda, const double* mu, const double* d, const double* w,
                          double* params, double* d_mu_unit, double* d_dir) {
    const double e = exp(lambda * (dot3d(d, mu) - 1.0));
    const double t = dot3d(d, mu) - 1.0;
    for (int c = 0; c < 3; ++c) params[c] += e * w[c];
    const double walpha = dot3d(w, alpha);
    params[3] += lambda * t * e * walpha;
    for (int k = 0; k < 3; ++k) {
        if (d_mu_unit) d_mu_unit[k] += lambda * e * walpha * d[k];
        d_dir[k] += lambda * e * walpha * mu[k];
    }
}

template <bool F64, int KIND>
__global__ void bwd_splat_kernel(const BwdParams p, uint64_t V, const uint32_t* __restrict__ order,
                                 const int4* __restrict__ brect, const uint2* __restrict__ ranges,
                                 const uint32_t* __restrict__ keys, const uint32_t* __restrict__ rank_of,
                                 const uint32_t* __restrict__ used, const double* __restrict__ partial,
                                 double* __restrict__ grads, int stride) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= V) return;
    const uint32_t g = order[r];
    const int4 rc = brect[r];
    double acc[kNP] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int ty = rc.z; ty <= rc.w; ++ty)
        for (int tx = rc.x; tx <= rc.y; ++tx) {
            const int tile = ty * p.tiles_x + tx;
            const uint2 range = ranges[tile];
            int lo = static_cast<int>(range.x), hi = static_cast<int>(range.y);
            const int lim = lo + static_cast<int>(used[tile]);
            while (lo < hi) {  // first entry with rank >= r (lists are in depth order)
                const int mid = (lo + hi) >> 1;
                if (rank_of[keys[mid]] < r)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            if (lo < lim && keys[lo] == g)
                for (int q = 0; q < kNP; ++q) acc[q] += partial[static_cast<size_t>(lo) * kNP + q];
        }
    // ---- pass 2 (grad.cpp:155-244) ----
    Proj pj;
    project_full<F64, KIND>(p, g, pj);
    const CamParams& cam = p.cam;
    double* out = grads + static_cast<size_t>(g) * stride;
    double gpos[3] = {0.0, 0.0, 0.0};
    // colour (grad_color, color.cpp:291-358) and the view-direction part of position
    {
        const ScenePlanes& sp = p.sp;
        const double* d = pj.dir;
        double pre[3];
        pre_colour<KIND>(p, g, pj.deg, d, pre);
        double w[3];
        for (int c = 0; c < 3; ++c) w[c] = pre[c] >= 0.0 ? acc[c] : 0.0;
        double ddir[3] = {0.0, 0.0, 0.0};
        double* cp = out + 11;
        if constexpr (KIND == SGS_SH || KIND == SGS_MIXED) {
            double b[16], db[16][3];
            sh_basis(d[0], d[1], d[2], pj.deg, b);
            sh_dbasis(d[0], d[1], d[2], pj.deg, db);
            const int n = (pj.deg + 1) * (pj.deg + 1);
            for (int i = 0; i < n; ++i) {
                for (int c = 0; c < 3; ++c) cp[3 * i + c] = b[i] * w[c];
                const double co[3] = {cparam<KIND>(sp, g, 3 * i), cparam<KIND>(sp, g, 3 * i + 1),
                                      cparam<KIND>(sp, g, 3 * i + 2)};
                const double wd = dot3d(w, co);
                for (int k = 0; k < 3; ++k) ddir[k] += db[i][k] * wd;
            }
            if constexpr (KIND == SGS_MIXED) {
                const int nst = 3 * (sp.sh_degree + 1) * (sp.sh_degree + 1);
                for (int l = 0; l < 3; ++l) {
                    const double al[3] = {cparam<KIND>(sp, g, nst + 4 * l), cparam<KIND>(sp, g, nst + 4 * l + 1),
                                          cparam<KIND>(sp, g, nst + 4 * l + 2)};
                    const double lambda = exp(cparam<KIND>(sp, g, nst + 4 * l + 3));
                    lobe_grad(al, lambda, p.axes + 3 * l, d, w, cp + nst + 4 * l, nullptr, ddir);
                }
            }
        } else if constexpr (KIND == SGS_SG1) {
            for (int c = 0; c < 3; ++c) cp[c] = w[c];
            double mu[3], lambda, dmu[3] = {0.0, 0.0, 0.0};
            const double nrm = sg1_lobe<KIND>(sp, g, mu, &lambda);
            const double al[3] = {cparam<KIND>(sp, g, 3), cparam<KIND>(sp, g, 4), cparam<KIND>(sp, g, 5)};
            lobe_grad(al, lambda, mu, d, w, cp + 3, dmu, ddir);
            const double md = dot3d(mu, dmu);
            for (int c = 0; c < 3; ++c) cp[7 + c] = (dmu[c] - mu[c] * md) / (nrm > 1e-12 ? nrm : 1.0);
        } else {
            for (int c = 0; c < 3; ++c) cp[c] = w[c];
            for (int l = 0; l < 3; ++l) {
                const double al[3] = {cparam<KIND>(sp, g, 3 + 4 * l), cparam<KIND>(sp, g, 4 + 4 * l),
                                      cparam<KIND>(sp, g, 5 + 4 * l)};
                const double lambda = exp(cparam<KIND>(sp, g, 6 + 4 * l));
                lobe_grad(al, lambda, p.axes + 3 * l, d, w, cp + 3 + 4 * l, nullptr, ddir);
            }
        }
        const double dd = dot3d(d, ddir);
        for (int k = 0; k < 3; ++k) gpos[k] += (ddir[k] - d[k] * dd) / pj.dist;
    }
    // opacity activation
    const double op = pj.pg.opacity;
    out[10] = acc[3] * op * (1.0 - op);
    // conic -> 2D covariance: g_cov2d = -K G K (K the conic matrix, G the symmetric gradient)
    const double K[4] = {pj.pg.cona, pj.pg.conb, pj.pg.conb, pj.pg.conc};
    const double G[4] = {acc[6], acc[7], acc[7], acc[8]};
    double KG[4], gc2[4];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) KG[2 * a + b] = K[2 * a] * G[b] + K[2 * a + 1] * G[2 + b];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) gc2[2 * a + b] = -(KG[2 * a] * K[b] + KG[2 * a + 1] * K[2 + b]);
    // 2D covariance -> 3D covariance and the Jacobian
    const double tx = pj.pg.tx, ty = pj.pg.ty, tz = pj.pg.tz;
    const double rx = tx / tz, ry = ty / tz;
    const bool clx = rx < -cam.lim_x || rx > cam.lim_x, cly = ry < -cam.lim_y || ry > cam.lim_y;
    const double txc = fmin(fmax(rx, -cam.lim_x), cam.lim_x) * tz;
    const double tyc = fmin(fmax(ry, -cam.lim_y), cam.lim_y) * tz;
    const double J[6] = {cam.fx / tz, 0.0, -cam.fx * txc / (tz * tz), 0.0, cam.fy / tz, -cam.fy * tyc / (tz * tz)};
    const double* R = cam.R;
    double Tm[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            Tm[3 * a + b] = (J[3 * a] * R[b] + J[3 * a + 1] * R[3 + b]) + J[3 * a + 2] * R[6 + b];
    const double* S6 = pj.geo.S;
    const double S[9] = {S6[0], S6[1], S6[2], S6[1], S6[3], S6[4], S6[2], S6[4], S6[5]};
    // g_cov3d = Tm^T gc2 Tm
    double gTm[6];  // gc2 Tm (2x3)
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) gTm[3 * a + b] = gc2[2 * a] * Tm[b] + gc2[2 * a + 1] * Tm[3 + b];
    double g3[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) g3[3 * a + b] = Tm[a] * gTm[b] + Tm[3 + a] * gTm[3 + b];
    // g_t_mat = 2 gc2 Tm S; g_jac = g_t_mat R^T
    double gT[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            gT[3 * a + b] = 2.0 * ((gTm[3 * a] * S[b] + gTm[3 * a + 1] * S[3 + b]) + gTm[3 * a + 2] * S[6 + b]);
    double gJ[6];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
            gJ[3 * a + b] = (gT[3 * a] * R[3 * b] + gT[3 * a + 1] * R[3 * b + 1]) + gT[3 * a + 2] * R[3 * b + 2];
    double dt[3] = {0.0, 0.0, 0.0};
    dt[2] += gJ[0] * (-cam.fx / (tz * tz));
    dt[2] += gJ[4] * (-cam.fy / (tz * tz));
    if (clx) {
        dt[2] += gJ[2] * (cam.fx * txc / (tz * tz * tz));
    } else {
        dt[0] += gJ[2] * (-cam.fx / (tz * tz));
        dt[2] += gJ[2] * (2.0 * cam.fx * tx / (tz * tz * tz));
    }
    if (cly) {
        dt[2] += gJ[5] * (cam.fy * tyc / (tz * tz * tz));
    } else {
        dt[1] += gJ[5] * (-cam.fy / (tz * tz));
        dt[2] += gJ[5] * (2.0 * cam.fy * ty / (tz * tz * tz));
    }
    // projected mean -> camera-space position (unclamped projection)
    dt[0] += acc[4] * cam.fx / tz;
    dt[1] += acc[5] * cam.fy / tz;
    dt[2] += -acc[4] * cam.fx * tx / (tz * tz) - acc[5] * cam.fy * ty / (tz * tz);
    for (int k = 0; k < 3; ++k) gpos[k] += (R[k] * dt[0] + R[3 + k] * dt[1]) + R[6 + k] * dt[2];
    out[0] = gpos[0];
    out[1] = gpos[1];
    out[2] = gpos[2];
    // 3D covariance -> rotation and log scales: Sigma = M M^T, M = R(q) diag(e^s)
    double qr[4], ls[3];
    load_rot_scale<F64>(p.sp, g, qr, ls);
    const double qn = sqrt(((qr[0] * qr[0] + qr[1] * qr[1]) + qr[2] * qr[2]) + qr[3] * qr[3]);
    const double q[4] = {qr[0] / qn, qr[1] / qn, qr[2] / qn, qr[3] / qn};
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    const double rot[9] = {1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
                           2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
                           2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)};
    const double sa[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    double m3[9], gm3[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) m3[3 * a + b] = rot[3 * a + b] * sa[b];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            gm3[3 * a + b] = 2.0 * ((g3[3 * a] * m3[b] + g3[3 * a + 1] * m3[3 + b]) + g3[3 * a + 2] * m3[6 + b]);
    for (int k = 0; k < 3; ++k)
        out[7 + k] = ((gm3[k] * rot[k] + gm3[3 + k] * rot[3 + k]) + gm3[6 + k] * rot[6 + k]) * sa[k];
    double grot[9];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) grot[3 * a + b] = gm3[3 * a + b] * sa[b];
    double Jq[4][9];
    quat_jacobians(q, Jq);
    double gqn[4];
    for (int k = 0; k < 4; ++k) {
        double sum = 0.0;
        for (int e = 0; e < 9; ++e) sum += grot[e] * Jq[k][e];
        gqn[k] = sum;
    }
    const double qg = ((q[0] * gqn[0] + q[1] * gqn[1]) + q[2] * gqn[2]) + q[3] * gqn[3];
    for (int k = 0; k < 4; ++k) out[3 + k] = (gqn[k] - q[k] * qg) / qn;
}

__global__ void finite_check_kernel(const double* __restrict__ v, size_t n, int* __restrict__ bad) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && !isfinite(v[i])) atomicExch(bad, 1);
}

template <bool F64, int KIND>
void launch_kind_bwd(const BwdParams& p, uint64_t V, int nchunks, int ntile, const uint32_t* order,
                     const int4* brect, const uint2* ranges, const uint32_t* keys, BwdSplat* bs,
                     uint32_t* rank_of, uint32_t* used, double* partial, const double* upstream, double* grads,
                     int stride, cudaStream_t s) {
    const unsigned vb = static_cast<unsigned>((V + 127) / 128);
    if (V) bwd_prep_kernel<F64, KIND><<<vb, 128, 0, s>>>(p, V, order, bs, rank_of);
    if (ntile) bwd_pixels_kernel<<<ntile, kBThreads, 0, s>>>(p, nchunks, ranges, keys, bs, upstream, partial, used);
    if (V)
        bwd_splat_kernel<F64, KIND><<<vb, 128, 0, s>>>(p, V, order, brect, ranges, keys, rank_of, used, partial,
                                                       grads, stride);
}

template <bool F64, int KIND>
void launch_kind_render64(const BwdParams& p, uint64_t V, int nchunks, int ntile, const uint32_t* order,
                          const uint2* ranges, const uint32_t* keys, BwdSplat* bs, uint32_t* rank_of,
                          double* rgb, double* T, cudaStream_t s) {
    if (V) bwd_prep_kernel<F64, KIND><<<static_cast<unsigned>((V + 127) / 128), 128, 0, s>>>(p, V, order, bs, rank_of);
    if (ntile) render_f64_kernel<<<ntile, kBThreads, 0, s>>>(p, nchunks, ranges, keys, bs, rgb, T);
}

}  // namespace

void launch_render_f64(const ScenePlanes& sp, const CamParams& cam, const CfgParams& cfg, const double* axes,
                       const double* bg, int override_degree, uint64_t V, int nchunks, const uint32_t* order,
                       const uint2* ranges, const uint32_t* keys, void* bs, uint32_t* rank_of, double* rgb,
                       double* T, cudaStream_t s) {
    BwdParams p{};
    p.sp = sp;
    p.cam = cam;
    p.cfg = cfg;
    for (int k = 0; k < 9; ++k) p.axes[k] = axes[k];
    for (int k = 0; k < 3; ++k) p.bg[k] = bg[k];
    p.override_degree = override_degree;
    p.tiles_x = cfg.tiles_x;
    const int ntile = cfg.tiles_x * cfg.tiles_y;
    BwdSplat* b = static_cast<BwdSplat*>(bs);
#define SGS_R64(F, K) launch_kind_render64<F, K>(p, V, nchunks, ntile, order, ranges, keys, b, rank_of, rgb, T, s)
    const bool f64 = sp.geometry_f64 != 0;
    switch (sp.kind) {
        case SGS_SH: f64 ? SGS_R64(true, SGS_SH) : SGS_R64(false, SGS_SH); break;
        case SGS_SG1: f64 ? SGS_R64(true, SGS_SG1) : SGS_R64(false, SGS_SG1); break;
        case SGS_SG3: f64 ? SGS_R64(true, SGS_SG3) : SGS_R64(false, SGS_SG3); break;
        default: f64 ? SGS_R64(true, SGS_MIXED) : SGS_R64(false, SGS_MIXED); break;
    }
#undef SGS_R64
}

size_t bwd_splat_bytes() { return sizeof(BwdSplat); }
size_t bwd_partial_bytes() { return kNP * sizeof(double); }

void launch_finite_check(const double* v, size_t n, int* bad, cudaStream_t s) {
    if (n) finite_check_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(v, n, bad);
}

void launch_backward(const ScenePlanes& sp, const CamParams& cam, const CfgParams& cfg, const double* axes,
                     const double* bg, int override_degree, uint64_t V, int nchunks, const uint32_t* order,
                     const int4* brect, const uint2* ranges, const uint32_t* keys, void* bs,
                     uint32_t* rank_of, uint32_t* used, double* partial, const double* upstream, double* grads,
                     int stride, cudaStream_t s) {
    BwdParams p{};
    p.sp = sp;
    p.cam = cam;
    p.cfg = cfg;
    for (int k = 0; k < 9; ++k) p.axes[k] = axes[k];
    for (int k = 0; k < 3; ++k) p.bg[k] = bg[k];
    p.override_degree = override_degree;
    p.tiles_x = cfg.tiles_x;
    const int ntile = cfg.tiles_x * cfg.tiles_y;
    BwdSplat* b = static_cast<BwdSplat*>(bs);
#define SGS_BWD(F, K)                                                                                           \
    launch_kind_bwd<F, K>(p, V, nchunks, ntile, order, brect, ranges, keys, b, rank_of, used, partial, upstream, \
                          grads, stride, s)
    const bool f64 = sp.geometry_f64 != 0;
    switch (sp.kind) {
        case SGS_SH: f64 ? SGS_BWD(true, SGS_SH) : SGS_BWD(false, SGS_SH); break;
        case SGS_SG1: f64 ? SGS_BWD(true, SGS_SG1) : SGS_BWD(false, SGS_SG1); break;
        case SGS_SG3: f64 ? SGS_BWD(true, SGS_SG3) : SGS_BWD(false, SGS_SG3); break;
        default: f64 ? SGS_BWD(true, SGS_MIXED) : SGS_BWD(false, SGS_MIXED); break;
    }
#undef SGS_BWD
}

}  // namespace sgs
