// preprocess.cu -- K1: per-Gaussian cull, EWA projection, degree select, SG+SH colour.
//
// One thread per Gaussian. Replaces project_cached (proj/src/raster.cpp:17-80),
// covariance (proj/src/scene.cpp:81-85), quat_to_rotation (common.hpp:124-134)
// and eval_color (proj/src/color.cpp:99-235).
//
// Numerics. Every decision the reference makes in FP64 (near cull, det <= 0,
// strict bbox cull, |p - C| < 1e-12, degree thresholds, tile rectangle) is made
// here in FP64 with the reference's exact operation order, using the
// round-to-nearest intrinsics (__dmul_rn/__dadd_rn/...) so nvcc cannot contract
// into FMAs. The only libm call on the decision path is exp() in exp(log_scale)
// and sigmoid(); CUDA's is within 1 ulp of glibc's, so a decision can only
// differ within ~1e-16 relative of a boundary (tests count such flips: 0).
// Colour is evaluated in FP32 (tolerance-level quantity).
//
// Memory. Coalesced 16-B loads from float4 SoA planes: geometry 3 planes
// (48 B/Gaussian), colour only the planes the evaluated degree needs
// (MIXED+SH1: 6 planes = 96 B). Outputs per visible splat: 8 B depth key,
// 48 B compositing record, 32 B FP64 guard record, 16 B tile rect, 4 B count.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "projection.cuh"

namespace sgs {
namespace {

// SH constants, color.hpp:15-26 (float copies for the FP32 colour path).
__constant__ float kC0 = 0.28209479177387814f;
__constant__ float kC1 = 0.4886025119029199f;
__constant__ float kC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                             -1.0925484305920792f, 0.5462742152960396f};
__constant__ float kC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                             0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                             -0.5900435899266435f};

constexpr int kK1Threads = 256;

// What one launch stages per Gaussian (float4 slots of kK1Threads each): the
// geometry (F32: pos + logit opacity; F64: two double2), the cached covariance
// (3 x double2) and the colour planes every Gaussian of this launch needs.
struct K1Stage {
    int geo_slots;   // 1 (F32) or 2 (F64)
    int sh_pre;      // SH planes staged, from plane 0
    int lobe_base;   // first lobe plane (MIXED: after the stored SH planes)
    int lobe_pre;    // lobe planes staged (MIXED 3, SG1 3, SG3 4)
    int slots;       // geo_slots + 3 + sh_pre + lobe_pre
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Thread-private staging: each thread copies its own Gaussian's slots (coalesced
// across the warp, slot-major so smem reads are conflict free) and later reads
// only them, so no CTA barrier is needed. Measured against 1D bulk copies
// (cp.async.bulk + mbarriers, the TMA engine) of the same slots at config C: one
// elected thread per CTA moving 4-KB slots with CTA-wide full / empty mbarriers,
// 166 us per launch; lane 0 of every warp moving its 512-B slot parts with per-warp
// mbarriers, 174 us; this per-thread cp.async pipeline, 158 us. K1 is bound by the
// latency of its per-Gaussian FP64 chain at 16 warps per SM, not by issuing loads,
// and the bulk variants' refills wait on slower consumers.
// Staging only geometry + covariance and reading the colour planes at use (32-view
// batch, config C): 0.637 ms/frame at 2 CTAs/SM, 0.606 at 3, 0.614 at 4, against
// 0.594 for the full stage at 2 (and 0.621 for the full stage at 3).
template <bool F64>
__device__ __forceinline__ void stage_item(const ScenePlanes& sp, const K1Stage& st, uint64_t i, float4* buf,
                                           int tid) {
    if constexpr (F64) {
        cp_async8(&buf[tid], &sp.g8[0][i]);
        cp_async8(reinterpret_cast<double*>(&buf[tid]) + 1, &sp.g8[1][i]);
        cp_async8(&buf[kK1Threads + tid], &sp.g8[2][i]);
        cp_async8(reinterpret_cast<double*>(&buf[kK1Threads + tid]) + 1, &sp.g8[10][i]);
    } else {
        cp_async16(&buf[tid], &sp.g4[0][i]);
    }
    float4* b = buf + st.geo_slots * kK1Threads;
#pragma unroll
    for (int k = 0; k < 3; ++k) cp_async16(&b[k * kK1Threads + tid], &sp.cov[k][i]);
    b += 3 * kK1Threads + tid;
    const float4* src = sp.color + i;  // plane p of Gaussian i: src + p n
    for (int p = 0; p < st.sh_pre; ++p, b += kK1Threads, src += sp.n) cp_async16(b, src);
    src = sp.color + static_cast<uint64_t>(st.lobe_base) * sp.n + i;
    for (int p = 0; p < st.lobe_pre; ++p, b += kK1Threads, src += sp.n) cp_async16(b, src);
}

template <bool F64>
__device__ __forceinline__ void geo_from_stage(const float4* buf, int geo_slots, int tid, Geo& g) {
    if constexpr (F64) {
        const double2 a = reinterpret_cast<const double2*>(buf)[tid];
        const double2 b = reinterpret_cast<const double2*>(buf)[kK1Threads + tid];
        g.p[0] = a.x, g.p[1] = a.y, g.p[2] = b.x, g.opl = b.y;
    } else {
        const float4 a = buf[tid];
        g.p[0] = a.x, g.p[1] = a.y, g.p[2] = a.z, g.opl = a.w;
    }
    const double2* c = reinterpret_cast<const double2*>(buf + geo_slots * kK1Threads);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double2 v = c[k * kK1Threads + tid];
        g.S[2 * k] = v.x;
        g.S[2 * k + 1] = v.y;
    }
}

// Colour plane p of Gaussian i: staged copy when the launch staged it, else HBM
// (adaptive degree selection loads the higher SH bands on demand).
struct PlaneFetch {
    const float4* sh;    // staged SH planes (slot-major) or null
    const float4* lobe;  // staged lobe planes
    const float4* color;
    uint64_t n, i;
    int tid, sh_pre, lobe_base;
    __device__ __forceinline__ float4 sh_plane(int p) const {
        return p < sh_pre ? sh[p * kK1Threads + tid] : __ldg(&color[static_cast<uint64_t>(p) * n + i]);
    }
    __device__ __forceinline__ float4 lobe_plane(int p) const { return lobe[p * kK1Threads + tid]; }
};

__device__ __forceinline__ void put4(float* f, float4 v) {
    f[0] = v.x;
    f[1] = v.y;
    f[2] = v.z;
    f[3] = v.w;
}

// sum_i Y_i(d) * c_i for degree `deg` <= MAXD (eval_sh_basis + sh_sum, color.cpp:99-168);
// MAXD bounds the register footprint (MIXED stores degree <= 2)
template <int MAXD>
__device__ __forceinline__ void sh_accumulate_upto(const float* c, int deg, float x, float y, float z,
                                                   float acc[3]) {
    constexpr int kN = (MAXD + 1) * (MAXD + 1);
    float b[kN];
    b[0] = kC0;
    if (MAXD >= 1 && deg >= 1) {
        b[1] = -kC1 * y;
        b[2] = kC1 * z;
        b[3] = -kC1 * x;
    }
    if constexpr (MAXD >= 2) {
        if (deg >= 2) {
            const float xx = x * x, yy = y * y, zz = z * z;
            b[4] = kC2[0] * x * y;
            b[5] = kC2[1] * y * z;
            b[6] = kC2[2] * (2.0f * zz - xx - yy);
            b[7] = kC2[3] * x * z;
            b[8] = kC2[4] * (xx - yy);
            if constexpr (MAXD >= 3) {
                if (deg >= 3) {
                    b[9] = kC3[0] * y * (3.0f * xx - yy);
                    b[10] = kC3[1] * x * y * z;
                    b[11] = kC3[2] * y * (4.0f * zz - xx - yy);
                    b[12] = kC3[3] * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
                    b[13] = kC3[4] * x * (4.0f * zz - xx - yy);
                    b[14] = kC3[5] * z * (xx - yy);
                    b[15] = kC3[6] * x * (xx - 3.0f * yy);
                }
            }
        }
    }
    const int n = (deg + 1) * (deg + 1);
#pragma unroll
    for (int k = 0; k < kN; ++k) {
        if (k < n) {
            acc[0] += b[k] * c[3 * k + 0];
            acc[1] += b[k] * c[3 * k + 1];
            acc[2] += b[k] * c[3 * k + 2];
        }
    }
}

// Three shared-axis lobes (ortho_lobe_sum, color.cpp:171-180). lobes: 3 x (rgb, logl).
__device__ __forceinline__ void lobe_accumulate(const float* lobes, const float* axes, float x,
                                                float y, float z, float acc[3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const float lambda = expf(lobes[4 * i + 3]);
        const float dot = axes[3 * i + 0] * x + axes[3 * i + 1] * y + axes[3 * i + 2] * z;
        const float e = expf(lambda * (dot - 1.0f));
        acc[0] += lobes[4 * i + 0] * e;
        acc[1] += lobes[4 * i + 1] * e;
        acc[2] += lobes[4 * i + 2] * e;
    }
}

__device__ __forceinline__ void raise_error(Counters* ctr, uint64_t i, uint32_t code) {
    atomicMin(&ctr->err, (static_cast<unsigned long long>(i) << 8) | code);
}

// View-dependent colour (eval_color, color.cpp:201-235) in FP32: exactly the colour
// planes the evaluated degree needs. The view direction normalize(p - C)
// (raster.cpp:66-69) is taken in FP32; the reference's FP64 decisions (including the
// unit-direction check) are made by the caller.
template <int KIND>
__device__ __forceinline__ float4 eval_colour(const ScenePlanes& sp, const PlaneFetch& pf, int deg, float fx,
                                              float fy, float fz) {
    float col[3];
    if constexpr (KIND == SGS_SH || KIND == SGS_MIXED) {
        const int need = (3 * (deg + 1) * (deg + 1) + 3) / 4;
        // MIXED stores degree <= 2 (7 planes); SH up to degree 3 (12 planes)
        constexpr int kMaxPlanes = KIND == SGS_MIXED ? 7 : 12;
        float c[4 * kMaxPlanes];
#pragma unroll
        for (int p = 0; p < kMaxPlanes; ++p)
            if (p < need) put4(c + 4 * p, pf.sh_plane(p));
        float acc[3] = {0.f, 0.f, 0.f};
        if constexpr (KIND == SGS_MIXED)
            sh_accumulate_upto<2>(c, deg, fx, fy, fz, acc);
        else
            sh_accumulate_upto<3>(c, deg, fx, fy, fz, acc);
        col[0] = 0.5f + acc[0];
        col[1] = 0.5f + acc[1];
        col[2] = 0.5f + acc[2];
        if constexpr (KIND == SGS_MIXED) {
            float lobes[12];
#pragma unroll
            for (int p = 0; p < 3; ++p) put4(lobes + 4 * p, pf.lobe_plane(p));
            float lacc[3] = {0.f, 0.f, 0.f};
            lobe_accumulate(lobes, sp.axes, fx, fy, fz, lacc);
            col[0] += lacc[0];
            col[1] += lacc[1];
            col[2] += lacc[2];
        }
    } else if constexpr (KIND == SGS_SG1) {
        // diffuse + alpha * exp(lambda (d.mu - 1)) (color.cpp:49-56, :195-199);
        // mu was normalised in FP64 at upload (DiffuseSGModel::lobe).
        float f[12];
#pragma unroll
        for (int p = 0; p < 3; ++p) put4(f + 4 * p, pf.lobe_plane(p));
        const float lambda = expf(f[3]);
        const float e = expf(lambda * (fx * f[8] + fy * f[9] + fz * f[10] - 1.0f));
        col[0] = f[0] + f[4] * e;
        col[1] = f[1] + f[5] * e;
        col[2] = f[2] + f[6] * e;
    } else {
        float f[16];
#pragma unroll
        for (int p = 0; p < 4; ++p) put4(f + 4 * p, pf.lobe_plane(p));
        float lacc[3] = {0.f, 0.f, 0.f};
        lobe_accumulate(f + 4, sp.axes, fx, fy, fz, lacc);
        col[0] = f[0] + lacc[0];
        col[1] = f[1] + lacc[1];
        col[2] = f[2] + lacc[2];
    }
    // cwiseMax(0): std::max(v, 0) keeps NaN
    return make_float4(col[0] < 0.f ? 0.f : col[0], col[1] < 0.f ? 0.f : col[1], col[2] < 0.f ? 0.f : col[2], 0.f);
}

// One view's K1 work for Gaussian i (whose geometry g is loaded): projection,
// decisions, record, rect, colour. Returns the depth key (~0 if culled) and the
// tile count through key / count / visible.
template <int KIND, bool DEBUG>
__device__ __forceinline__ void k1_view(const ScenePlanes& sp, const CfgParams& cfg, const K1Stage& stg,
                                        const K1Out& o, const float4* buf, int tid, uint64_t i, const Geo& g,
                                        DebugSplat& dbg, unsigned long long& key, uint32_t& count, bool& visible) {
    ProjGeo pg;
    const int pstat = project_staged(g, o.cam, pg);
    if (pstat == kProjZeroQuat) raise_error(o.ctr, i, kErrZeroQuaternion);
    do {
        if (pstat != kProjVisible) break;
        const double radius = pg.radius, mx = pg.mx, my = pg.my, tz = pg.tz;
        // view direction, camera.hpp:20 and raster.cpp:66-69
        const double ox = dsub(g.p[0], o.cam.C[0]), oy = dsub(g.p[1], o.cam.C[1]),
                     oz = dsub(g.p[2], o.cam.C[2]);
        const double ss = dadd(dadd(dmul(ox, ox), dmul(oy, oy)), dmul(oz, oz));
        // The direction only feeds the FP32 colour. For |p - C|^2 in (1e-20, 1e30)
        // the reference's distance check (dist < 1e-12) cannot fire and its unit
        // check (color.cpp:10-16) cannot fire either (|norm - 1| ~ 1e-16), so the
        // direction is taken in FP32 with rsqrt; outside that range (or NaN) the
        // exact sqrt, division and checks run.
        const bool safe_dist = ss > 1e-20 && ss < 1e30;
        float fdx, fdy, fdz;
        double dist = 0.0;
        if (safe_dist) {
            const float inv = rsqrtf(static_cast<float>(ss));
            fdx = static_cast<float>(ox) * inv;
            fdy = static_cast<float>(oy) * inv;
            fdz = static_cast<float>(oz) * inv;
        } else {
            dist = __dsqrt_rn(ss);
            if (dist < 1e-12) break;  // raster.cpp:66-69 (NaN continues, as in the reference)
            const float inv = static_cast<float>(1.0 / dist);
            fdx = static_cast<float>(ox) * inv;
            fdy = static_cast<float>(oy) * inv;
            fdz = static_cast<float>(oz) * inv;
        }
        // degree selection and the colour-model error contract (raster.cpp:70-77,
        // color.cpp:201-206, :182-191)
        int deg = sp.sh_degree;
        int deg_used = -1;
        if constexpr (KIND == SGS_MIXED) {
            if (cfg.has_override) {
                deg_used = cfg.override_degree;
            } else {
                if (cfg.lo > cfg.hi) {
                    raise_error(o.ctr, i, kErrThresholds);
                    break;
                }
                deg_used = radius < cfg.lo ? 0 : (radius < cfg.hi ? 1 : 2);
            }
        } else {
            if (cfg.has_override) {
                raise_error(o.ctr, i, kErrOverrideNonMixed);
                break;
            }
        }
        if (!safe_dist) {
            const double dxd = ddiv(ox, dist), dyd = ddiv(oy, dist), dzd = ddiv(oz, dist);
            const double nrm =
                __dsqrt_rn(dadd(dadd(dmul(dxd, dxd), dmul(dyd, dyd)), dmul(dzd, dzd)));
            if (fabs(dsub(nrm, 1.0)) > 1e-6) {
                raise_error(o.ctr, i, kErrDirection);
                break;
            }
        }
        if constexpr (KIND == SGS_MIXED) {
            if (deg_used < 0 || deg_used > sp.sh_degree) {
                raise_error(o.ctr, i, kErrDegreeTooHigh);
                break;
            }
            deg = deg_used;
        }
        // ---- outputs ----
        // conic and opacity only feed FP32 quantities here (the compositor's guard band
        // re-derives the exact FP64 values): one reciprocal instead of three divisions,
        // sigmoid in FP32. The debug dump reports the exact ones.
        double cona, conb, conc, opacity;
        if constexpr (DEBUG) {
            exact_conic_opacity(g, pg);
            cona = pg.cona, conb = pg.conb, conc = pg.conc, opacity = pg.opacity;
        } else {
            const double rdet = 1.0 / pg.det;
            cona = pg.c * rdet;
            conb = -pg.b * rdet;
            conc = pg.a * rdet;
            opacity = 1.0f / (1.0f + __expf(-static_cast<float>(g.opl)));
        }
        visible = true;
        key = depth_key(tz);
        // tile rectangle (raster.cpp:117-122), inclusive, clamped
        const double ts = static_cast<double>(cfg.tile_size);
        // x / ts == x * (1/ts) bit for bit when ts is a power of two (both round the
        // exact quotient once); other tile sizes divide.
        const bool pow2 = (cfg.tile_size & (cfg.tile_size - 1)) == 0;
        const double its = 1.0 / ts;
        const double qx0 = pow2 ? dmul(dsub(mx, radius), its) : ddiv(dsub(mx, radius), ts);
        const double qx1 = pow2 ? dmul(dadd(mx, radius), its) : ddiv(dadd(mx, radius), ts);
        const double qy0 = pow2 ? dmul(dsub(my, radius), its) : ddiv(dsub(my, radius), ts);
        const double qy1 = pow2 ? dmul(dadd(my, radius), its) : ddiv(dadd(my, radius), ts);
        int32_t x0 = to_int_x86(floor(qx0));
        int32_t x1 = to_int_x86(floor(qx1));
        int32_t y0 = to_int_x86(floor(qy0));
        int32_t y1 = to_int_x86(floor(qy1));
        x0 = max(0, x0);
        y0 = max(0, y0);
        x1 = min(cfg.tiles_x - 1, x1);
        y1 = min(cfg.tiles_y - 1, y1);
        if (x1 >= x0 && y1 >= y0)
            count = static_cast<uint32_t>(x1 - x0 + 1) * static_cast<uint32_t>(y1 - y0 + 1);
        // FP32 m2 error bound: 2u S (9 r^2 + 3 r ts) + 1e-6
        const double csum = fabs(cona) + 2.0 * fabs(conb) + fabs(conc);
        const double guard =
            2.0 * 5.9604644775390625e-08 * csum * (9.0 * radius * radius + 3.0 * radius * ts) +
            1e-6;
        // combined cutoff: alpha < 1/255 <=> m2 > 2 ln(255 op) (op > 0); a NaN opacity
        // keeps the support cutoff (the reference blends it: NaN passes std::min and the
        // alpha test)
        const double acut = opacity > 0.0 ? 2.0 * log(255.0 * opacity) : -1.0;
        const double cut = isnan(opacity) ? kSupportMahalanobisSq
                                          : (acut < kSupportMahalanobisSq ? acut : kSupportMahalanobisSq);
        // extents of {d : d^T conic d <= cut + guard} = sqrt(K cov_xx), sqrt(K cov_yy);
        // cov = the dilated 2D covariance (a, b, c), slightly inflated
        const double K = fmax(cut + guard, 0.0);
        SplatRec r;
        r.mx = mx;
        r.my = my;
        r.ca = static_cast<float>(cona);
        r.cb2 = static_cast<float>(2.0 * conb);
        r.cc = static_cast<float>(conc);
        r.lop = opacity > 0.0 ? __log2f(static_cast<float>(opacity)) : -1e30f;
        r.cut = static_cast<float>(cut);
        r.guard = guard < 1e30 ? static_cast<float>(guard) : FLT_MAX;
        r.ext_x = sqrtf(static_cast<float>(K * pg.a)) * (1.0f + 1e-5f) + 1e-3f;
        r.ext_y = sqrtf(static_cast<float>(K * pg.c)) * (1.0f + 1e-5f) + 1e-3f;
        const int4 rect3s = make_int4(x0, x1, y0, y1);  // the reference's 3-sigma rectangle
        if (cfg.tight_rect && x1 >= x0 && y1 >= y0) {
            // Render frames list a splat only in the tiles its cut ellipse's box reaches:
            // every pixel outside it has m2 > cut and is skipped by the reference, so the
            // image is unchanged (the parity dumps and stats frames keep the reference's
            // 3-sigma rectangle, which bounds this one).
            const double ex = r.ext_x, ey = r.ext_y;
            const double ex0 = pow2 ? dmul(dsub(mx, ex), its) : ddiv(dsub(mx, ex), ts);
            const double ex1 = pow2 ? dmul(dadd(mx, ex), its) : ddiv(dadd(mx, ex), ts);
            const double ey0 = pow2 ? dmul(dsub(my, ey), its) : ddiv(dsub(my, ey), ts);
            const double ey1 = pow2 ? dmul(dadd(my, ey), its) : ddiv(dadd(my, ey), ts);
            x0 = max(x0, to_int_x86(floor(ex0)));
            x1 = min(x1, to_int_x86(floor(ex1)));
            y0 = max(y0, to_int_x86(floor(ey0)));
            y1 = min(y1, to_int_x86(floor(ey1)));
            // opacity below 1/255 (cut < 0): alpha < 1/255 at every pixel, no tile at all
            if (cut + guard < 0.0) x1 = x0 - 1;
        }
        o.rects[i] = make_int4(x0, x1, y0, y1);
        // colour (FP32), direction from the FP64 offset
        const float4* sb = buf + (stg.geo_slots + 3) * kK1Threads;
        const PlaneFetch pf{sb, sb + stg.sh_pre * kK1Threads, sp.color, sp.n, i, tid, stg.sh_pre, stg.lobe_base};
        const float4 col = eval_colour<KIND>(sp, pf, deg, fdx, fdy, fdz);
        o.colour[i] = col;
        // A non-finite colour or a NaN opacity must reach exactly the pixels the
        // reference blends it into (it skips the others before touching acc): such a
        // (rare) splat gets an infinite guard band, so every one of its pairs is decided
        // and blended one at a time by the compositor's FP64 path, and its 3-sigma
        // rectangle.
        if (!(isfinite(col.x) && isfinite(col.y) && isfinite(col.z)) || isnan(opacity)) {
            r.guard = INFINITY;
            r.ext_x = r.ext_y = INFINITY;
            o.rects[i] = rect3s;
        }
        if constexpr (DEBUG) {
            dbg.color[0] = col.x;
            dbg.color[1] = col.y;
            dbg.color[2] = col.z;
        }
        o.rec[i] = r;
        if constexpr (DEBUG) {
            dbg.mean2d[0] = mx;
            dbg.mean2d[1] = my;
            dbg.conic[0] = cona;
            dbg.conic[1] = conb;
            dbg.conic[2] = conc;
            dbg.depth = tz;
            dbg.opacity = opacity;
            dbg.radius = radius;
            dbg.degree = KIND == SGS_MIXED ? deg_used : -1;
            dbg.visible = 1;
        }
    } while (false);
}

// K1: persistent CTAs walk the Gaussians with a two-stage cp.async pipeline (the
// next Gaussian's geometry, covariance and colour planes land in shared memory
// while this one is projected), so the FP64 chain overlaps the HBM latency.
// MINB (min resident CTAs per SM) trades registers for occupancy; selected at run
// time by SGS_K1_MINB for tuning (default kDefaultMinB, see profiles/).
template <bool F64, int KIND, int MINB, bool DEBUG>
__global__ void __launch_bounds__(kK1Threads, MINB) preprocess_kernel(
    const ScenePlanes sp, const CfgParams cfg, const K1Stage stg, const K1Out o, DebugSplat* __restrict__ debug) {
    extern __shared__ float4 k1_smem[];
    const int tid = threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kK1Threads;
    const int buf_stride = stg.slots * kK1Threads;
    uint64_t i = static_cast<uint64_t>(blockIdx.x) * kK1Threads + tid;
    if (i < sp.n) stage_item<F64>(sp, stg, i, k1_smem, tid);
    cp_async_commit();
    uint32_t nvis = 0;
    unsigned long long kmin = ~0ULL, kmax = 0ULL;
    for (int it = 0; static_cast<uint64_t>(blockIdx.x) * kK1Threads + static_cast<uint64_t>(it) * stride < sp.n;
         ++it, i += stride) {
        if (i + stride < sp.n) stage_item<F64>(sp, stg, i + stride, k1_smem + ((it + 1) & 1) * buf_stride, tid);
        cp_async_commit();
        cp_async_wait1();
        if (i >= sp.n) continue;
        const float4* buf = k1_smem + (it & 1) * buf_stride;
        Geo g;
        geo_from_stage<F64>(buf, stg.geo_slots, tid, g);
        unsigned long long key = ~0ULL;
        uint32_t count = 0;
        bool visible = false;
        DebugSplat dbg;
        if constexpr (DEBUG) {
            memset(&dbg, 0, sizeof(dbg));
            dbg.degree = -1;
        }
        k1_view<KIND, DEBUG>(sp, cfg, stg, o, buf, tid, i, g, dbg, key, count, visible);
        o.keys[i] = key;
        if constexpr (DEBUG) debug[i] = dbg;
        if (visible) {
            ++nvis;
            kmin = min(kmin, key);
            kmax = max(kmax, key);
        }
    }
    // visible count and depth-key range: one atomic each per warp
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        nvis += __shfl_xor_sync(0xffffffffu, nvis, s);
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, s));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, s));
    }
    if ((tid & 31) == 0 && nvis) {
        atomicAdd(&o.ctr->visible, static_cast<unsigned long long>(nvis));
        atomicMin(&o.ctr->kmin, kmin);
        atomicMax(&o.ctr->kmax, kmax);
    }
}

constexpr int kMaxStageSlots = 10;

K1Stage make_stage(const ScenePlanes& sp, const CfgParams& cfg) {
    K1Stage st{};
    st.geo_slots = sp.geometry_f64 ? 2 : 1;
    const int stored_sh = (3 * (sp.sh_degree + 1) * (sp.sh_degree + 1) + 3) / 4;
    switch (sp.kind) {
        case SGS_SH:
            st.sh_pre = stored_sh;  // SH always evaluates its stored degree
            break;
        case SGS_MIXED: {
            // override: every splat uses that degree; adaptive: degree 0 is staged and
            // higher bands load on demand (an out-of-range override errors in K1)
            int d = cfg.has_override ? cfg.override_degree : 0;
            d = d < 0 ? 0 : (d > sp.sh_degree ? sp.sh_degree : d);
            st.sh_pre = (3 * (d + 1) * (d + 1) + 3) / 4;
            st.lobe_base = stored_sh;
            st.lobe_pre = 3;
            break;
        }
        case SGS_SG1: st.lobe_pre = 3; break;
        default: st.lobe_pre = 4; break;
    }
    st.slots = st.geo_slots + 3 + st.sh_pre + st.lobe_pre;
    // At most kMaxStageSlots slots are staged; the SH planes beyond are read at use. A
    // degree-3 SH scene would otherwise stage 16 (128 KB per CTA, one CTA per SM): config
    // D's K1 0.265 -> 0.212 ms and batch 0.684 -> 0.629 ms/frame with 10 (13: 0.224 /
    // 0.644; 8 also trims config C's stage: 0.605 against 0.586).
    if (st.slots > kMaxStageSlots) {
        const int cut = std::min(st.sh_pre, st.slots - kMaxStageSlots);
        st.sh_pre -= cut;
        st.slots -= cut;
    }
    return st;
}

}  // namespace

struct K1Record {
    const void* func = nullptr;
    dim3 grid, block;
    size_t smem = 0;
    ScenePlanes sp;
    CfgParams cfg;
    K1Stage st;
    K1Out out;
    DebugSplat* debug = nullptr;
};

namespace {

thread_local K1Record t_last_k1;

template <bool F64, int KIND, int MINB, bool DEBUG>
void launch_k1(const ScenePlanes& sp, const CfgParams& cfg, const K1Out& out, DebugSplat* debug,
               cudaStream_t stream) {
    const K1Stage st = make_stage(sp, cfg);
    const size_t smem = static_cast<size_t>(2) * st.slots * kK1Threads * sizeof(float4);
    auto kern = preprocess_kernel<F64, KIND, MINB, DEBUG>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kK1Threads, smem);
    const uint64_t need = (sp.n + kK1Threads - 1) / kK1Threads;
    const uint64_t grid = std::min<uint64_t>(need, static_cast<uint64_t>(sms) * std::max(per_sm, 1));
    t_last_k1 = K1Record{reinterpret_cast<const void*>(kern), dim3(static_cast<unsigned>(grid)), dim3(kK1Threads),
                         smem, sp, cfg, st, out, debug};
    kern<<<static_cast<unsigned>(grid), kK1Threads, smem, stream>>>(sp, cfg, st, out, debug);
}

constexpr int kDefaultMinB = 2;

int k1_minb() {
    static const int v = [] {
        const char* e = std::getenv("SGS_K1_MINB");
        const int m = e ? std::atoi(e) : kDefaultMinB;
        return (m >= 1 && m <= 4) ? m : kDefaultMinB;
    }();
    return v;
}

template <bool F64, int KIND>
void launch_minb(const ScenePlanes& sp, const CfgParams& cfg, const K1Out& out, DebugSplat* debug,
                 cudaStream_t stream) {
    if (debug) {
        launch_k1<F64, KIND, 1, true>(sp, cfg, out, debug, stream);
        return;
    }
    switch (k1_minb()) {
        case 1: launch_k1<F64, KIND, 1, false>(sp, cfg, out, nullptr, stream); break;
        case 3: launch_k1<F64, KIND, 3, false>(sp, cfg, out, nullptr, stream); break;
        case 4: launch_k1<F64, KIND, 4, false>(sp, cfg, out, nullptr, stream); break;
        default: launch_k1<F64, KIND, 2, false>(sp, cfg, out, nullptr, stream); break;
    }
}

template <bool F64>
void launch_kind(const ScenePlanes& sp, const CfgParams& cfg, const K1Out& out, DebugSplat* debug,
                 cudaStream_t stream) {
    switch (sp.kind) {
        case SGS_SH: launch_minb<F64, SGS_SH>(sp, cfg, out, debug, stream); break;
        case SGS_SG1: launch_minb<F64, SGS_SG1>(sp, cfg, out, debug, stream); break;
        case SGS_SG3: launch_minb<F64, SGS_SG3>(sp, cfg, out, debug, stream); break;
        default: launch_minb<F64, SGS_MIXED>(sp, cfg, out, debug, stream); break;
    }
}


// Per-scene cache of the view-independent 3D covariance (projection.cuh).
template <bool F64>
__global__ void cov3d_kernel(const ScenePlanes sp, double2* __restrict__ cov) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= sp.n) return;
    double q[4], ls[3];
    if constexpr (F64) {
        for (int k = 0; k < 4; ++k) q[k] = sp.g8[3 + k][i];
        for (int k = 0; k < 3; ++k) ls[k] = sp.g8[7 + k][i];
    } else {
        const float4 b = __ldg(&sp.g4[1][i]);
        const float4 c = __ldg(&sp.g4[2][i]);
        q[0] = b.x, q[1] = b.y, q[2] = b.z, q[3] = b.w;
        ls[0] = c.x, ls[1] = c.y, ls[2] = c.z;
    }
    double S6[6] = {kZeroQuatMark, 0.0, 0.0, 0.0, 0.0, 0.0};
    covariance3d(q, ls, S6);
    cov[i] = make_double2(S6[0], S6[1]);
    cov[sp.n + i] = make_double2(S6[2], S6[3]);
    cov[2 * sp.n + i] = make_double2(S6[4], S6[5]);
}


}  // namespace

void launch_cov3d(const ScenePlanes& sp, double2* cov, cudaStream_t stream) {
    if (sp.n == 0) return;
    const unsigned blocks = static_cast<unsigned>((sp.n + 255) / 256);
    if (sp.geometry_f64)
        cov3d_kernel<true><<<blocks, 256, 0, stream>>>(sp, cov);
    else
        cov3d_kernel<false><<<blocks, 256, 0, stream>>>(sp, cov);
}


void launch_preprocess(const ScenePlanes& sp, const CamParams& cam, const CfgParams& cfg,
                       unsigned long long* depth_keys, SplatRec* rec, int4* rects,
                       float4* colour, Counters* counters, DebugSplat* debug,
                       cudaStream_t stream) {
    if (sp.n == 0) return;
    const K1Out out{depth_keys, rec, rects, colour, counters, cam};
    if (sp.geometry_f64)
        launch_kind<true>(sp, cfg, out, debug, stream);
    else
        launch_kind<false>(sp, cfg, out, debug, stream);
}

K1Record* k1_last_launch_clone() { return new K1Record(t_last_k1); }

void k1_record_free(K1Record* r) { delete r; }

const void* k1_record_func(const K1Record* r) { return r->func; }

cudaError_t k1_record_patch(cudaGraphExec_t exec, cudaGraphNode_t node, K1Record* r, const CamParams& cam) {
    r->out.cam = cam;
    void* args[] = {&r->sp, &r->cfg, &r->st, &r->out, &r->debug};
    cudaKernelNodeParams p{};
    p.func = const_cast<void*>(r->func);
    p.gridDim = r->grid;
    p.blockDim = r->block;
    p.sharedMemBytes = static_cast<unsigned>(r->smem);
    p.kernelParams = args;
    p.extra = nullptr;
    return cudaGraphExecKernelNodeSetParams(exec, node, &p);
}

}  // namespace sgs
