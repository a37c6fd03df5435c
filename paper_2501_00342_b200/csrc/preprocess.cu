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
#include <cfloat>

#include "sgs_internal.h"

namespace sgs {
namespace {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// ((a0*b0 + a1*b1) + a2*b2): the Eigen-subset left-to-right reduction.
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double b0, double b1,
                                       double b2) {
    return dadd(dadd(dmul(a0, b0), dmul(a1, b1)), dmul(a2, b2));
}

// static_cast<int>(double) as x86-64 executes it (cvttsd2si): out-of-range and
// NaN give INT32_MIN. build_tile_grid (raster.cpp:117-122) depends on it.
__device__ __forceinline__ int32_t to_int_x86(double v) {
    if (!(v > -2147483649.0 && v < 2147483648.0)) return INT32_MIN;
    return static_cast<int32_t>(v);
}

__device__ __forceinline__ unsigned long long depth_key(double z) {
    if (z == 0.0) z = 0.0;  // -0 == +0 in the reference's comparator
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(z));
    return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

// SH constants, color.hpp:15-26 (float copies for the FP32 colour path).
__constant__ float kC0 = 0.28209479177387814f;
__constant__ float kC1 = 0.4886025119029199f;
__constant__ float kC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                             -1.0925484305920792f, 0.5462742152960396f};
__constant__ float kC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                             0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                             -0.5900435899266435f};

// Loads the first `nplanes` colour planes of Gaussian i into f[4*nplanes].
template <int MAXP>
__device__ __forceinline__ void load_planes(const float4* __restrict__ color, uint64_t n,
                                            uint64_t i, int nplanes, float* f) {
#pragma unroll
    for (int p = 0; p < MAXP; ++p) {
        if (p < nplanes) {
            float4 v = __ldg(&color[static_cast<uint64_t>(p) * n + i]);
            f[4 * p + 0] = v.x;
            f[4 * p + 1] = v.y;
            f[4 * p + 2] = v.z;
            f[4 * p + 3] = v.w;
        }
    }
}

// sum_i Y_i(d) * c_i for degree `deg` (eval_sh_basis + sh_sum, color.cpp:99-168).
__device__ __forceinline__ void sh_accumulate(const float* c, int deg, float x, float y, float z,
                                              float acc[3]) {
    float b[16];
    b[0] = kC0;
    if (deg >= 1) {
        b[1] = -kC1 * y;
        b[2] = kC1 * z;
        b[3] = -kC1 * x;
    }
    if (deg >= 2) {
        const float xx = x * x, yy = y * y, zz = z * z;
        b[4] = kC2[0] * x * y;
        b[5] = kC2[1] * y * z;
        b[6] = kC2[2] * (2.0f * zz - xx - yy);
        b[7] = kC2[3] * x * z;
        b[8] = kC2[4] * (xx - yy);
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
    const int n = (deg + 1) * (deg + 1);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
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

struct Geo {
    double p[3], q[4], ls[3], opl;
};

template <bool F64>
__device__ __forceinline__ void load_geo(const ScenePlanes& sp, uint64_t i, Geo& g) {
    if constexpr (F64) {
        g.p[0] = sp.g8[0][i];
        g.p[1] = sp.g8[1][i];
        g.p[2] = sp.g8[2][i];
        g.q[0] = sp.g8[3][i];
        g.q[1] = sp.g8[4][i];
        g.q[2] = sp.g8[5][i];
        g.q[3] = sp.g8[6][i];
        g.ls[0] = sp.g8[7][i];
        g.ls[1] = sp.g8[8][i];
        g.ls[2] = sp.g8[9][i];
        g.opl = sp.g8[10][i];
    } else {
        const float4 a = __ldg(&sp.g4[0][i]);
        const float4 b = __ldg(&sp.g4[1][i]);
        const float4 c = __ldg(&sp.g4[2][i]);
        g.p[0] = a.x;
        g.p[1] = a.y;
        g.p[2] = a.z;
        g.opl = a.w;
        g.q[0] = b.x;
        g.q[1] = b.y;
        g.q[2] = b.z;
        g.q[3] = b.w;
        g.ls[0] = c.x;
        g.ls[1] = c.y;
        g.ls[2] = c.z;
    }
}

__device__ __forceinline__ void raise_error(Counters* ctr, uint64_t i, uint32_t code) {
    atomicMin(&ctr->err, (static_cast<unsigned long long>(i) << 8) | code);
}

template <bool F64, int KIND>
__global__ void __launch_bounds__(256) preprocess_kernel(
    const ScenePlanes sp, const CamParams cam, const CfgParams cfg,
    unsigned long long* __restrict__ depth_keys, uint32_t* __restrict__ iota,
    SplatRec* __restrict__ rec, SplatRec64* __restrict__ rec64, int4* __restrict__ rects,
    uint32_t* __restrict__ ntiles, Counters* __restrict__ ctr, DebugSplat* __restrict__ debug) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    bool visible = false;
    unsigned long long vkey = ~0ULL;
    if (i < sp.n) {
        iota[i] = static_cast<uint32_t>(i);
        unsigned long long key = ~0ULL;
        uint32_t count = 0;
        Geo g;
        load_geo<F64>(sp, i, g);
        DebugSplat dbg;
        if (debug) {
            memset(&dbg, 0, sizeof(dbg));
            dbg.degree = -1;
        }
        // t = R p + t (camera.hpp:19)
        const double* R = cam.R;
        const double tx = dadd(dot3(R[0], R[1], R[2], g.p[0], g.p[1], g.p[2]), cam.t[0]);
        const double ty = dadd(dot3(R[3], R[4], R[5], g.p[0], g.p[1], g.p[2]), cam.t[1]);
        const double tz = dadd(dot3(R[6], R[7], R[8], g.p[0], g.p[1], g.p[2]), cam.t[2]);
        do {
            if (tz < cam.near_plane) break;  // raster.cpp:23
            // quat_to_rotation (common.hpp:124-134)
            const double qn = __dsqrt_rn(
                dadd(dadd(dadd(dmul(g.q[0], g.q[0]), dmul(g.q[1], g.q[1])), dmul(g.q[2], g.q[2])),
                     dmul(g.q[3], g.q[3])));
            if (qn < 1e-12) {
                raise_error(ctr, i, kErrZeroQuaternion);
                break;
            }
            const double w = ddiv(g.q[0], qn), x = ddiv(g.q[1], qn), y = ddiv(g.q[2], qn),
                         z = ddiv(g.q[3], qn);
            const double Rq[9] = {
                dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(z, z)))),
                dmul(2.0, dsub(dmul(x, y), dmul(w, z))),
                dmul(2.0, dadd(dmul(x, z), dmul(w, y))),
                dmul(2.0, dadd(dmul(x, y), dmul(w, z))),
                dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(z, z)))),
                dmul(2.0, dsub(dmul(y, z), dmul(w, x))),
                dmul(2.0, dsub(dmul(x, z), dmul(w, y))),
                dmul(2.0, dadd(dmul(y, z), dmul(w, x))),
                dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y)))),
            };
            // covariance (scene.cpp:81-85): M = Rq diag(exp(s)); S = M M^T
            const double sc[3] = {exp(g.ls[0]), exp(g.ls[1]), exp(g.ls[2])};
            double M[9];
#pragma unroll
            for (int r = 0; r < 3; ++r)
#pragma unroll
                for (int c = 0; c < 3; ++c) M[r * 3 + c] = dmul(Rq[r * 3 + c], sc[c]);
            double S[9];
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    S[a * 3 + b] = dot3(M[a * 3 + 0], M[a * 3 + 1], M[a * 3 + 2], M[b * 3 + 0],
                                        M[b * 3 + 1], M[b * 3 + 2]);
            // EWA Jacobian with the 1.3x frustum clamp (raster.cpp:27-41)
            const double rx = ddiv(tx, tz), ry = ddiv(ty, tz);
            const double crx = rx < -cam.lim_x ? -cam.lim_x : (cam.lim_x < rx ? cam.lim_x : rx);
            const double cry = ry < -cam.lim_y ? -cam.lim_y : (cam.lim_y < ry ? cam.lim_y : ry);
            const double txc = dmul(crx, tz), tyc = dmul(cry, tz);
            const double tz2 = dmul(tz, tz);
            const double J[6] = {ddiv(cam.fx, tz), 0.0, ddiv(dmul(-cam.fx, txc), tz2),
                                 0.0, ddiv(cam.fy, tz), ddiv(dmul(-cam.fy, tyc), tz2)};
            double Tm[6];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    Tm[a * 3 + b] = dot3(J[a * 3 + 0], J[a * 3 + 1], J[a * 3 + 2], R[0 * 3 + b],
                                         R[1 * 3 + b], R[2 * 3 + b]);
            double TS[6];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    TS[a * 3 + b] = dot3(Tm[a * 3 + 0], Tm[a * 3 + 1], Tm[a * 3 + 2], S[0 * 3 + b],
                                         S[1 * 3 + b], S[2 * 3 + b]);
            const double a = dadd(dot3(TS[0], TS[1], TS[2], Tm[0], Tm[1], Tm[2]), kCovarianceDilation);
            const double b = dot3(TS[0], TS[1], TS[2], Tm[3], Tm[4], Tm[5]);
            const double c = dadd(dot3(TS[3], TS[4], TS[5], Tm[3], Tm[4], Tm[5]), kCovarianceDilation);
            const double det = dsub(dmul(a, c), dmul(b, b));
            if (det <= 0.0) break;  // raster.cpp:48 (NaN passes, as in the reference)
            const double mid = dmul(0.5, dadd(a, c));
            const double disc = dsub(dmul(mid, mid), det);
            const double lambda_max = dadd(mid, __dsqrt_rn(0.0 < disc ? disc : 0.0));
            const double radius = dmul(3.0, __dsqrt_rn(lambda_max));
            const double mx = dadd(ddiv(dmul(cam.fx, tx), tz), cam.cx);
            const double my = dadd(ddiv(dmul(cam.fy, ty), tz), cam.cy);
            if (dadd(mx, radius) < 0.0 || dsub(mx, radius) > cam.width ||
                dadd(my, radius) < 0.0 || dsub(my, radius) > cam.height)
                break;  // raster.cpp:56-60
            // view direction, camera.hpp:20 and raster.cpp:66-69
            const double ox = dsub(g.p[0], cam.C[0]), oy = dsub(g.p[1], cam.C[1]),
                         oz = dsub(g.p[2], cam.C[2]);
            const double dist = __dsqrt_rn(dadd(dadd(dmul(ox, ox), dmul(oy, oy)), dmul(oz, oz)));
            if (dist < 1e-12) break;
            const double dxd = ddiv(ox, dist), dyd = ddiv(oy, dist), dzd = ddiv(oz, dist);
            // degree selection and the colour-model error contract (raster.cpp:70-77,
            // color.cpp:201-206, :182-191)
            int deg = sp.sh_degree;
            int deg_used = -1;
            if constexpr (KIND == SGS_MIXED) {
                if (cfg.has_override) {
                    deg_used = cfg.override_degree;
                } else {
                    if (cfg.lo > cfg.hi) {
                        raise_error(ctr, i, kErrThresholds);
                        break;
                    }
                    deg_used = radius < cfg.lo ? 0 : (radius < cfg.hi ? 1 : 2);
                }
            } else {
                if (cfg.has_override) {
                    raise_error(ctr, i, kErrOverrideNonMixed);
                    break;
                }
            }
            {
                const double nrm =
                    __dsqrt_rn(dadd(dadd(dmul(dxd, dxd), dmul(dyd, dyd)), dmul(dzd, dzd)));
                if (fabs(dsub(nrm, 1.0)) > 1e-6) {
                    raise_error(ctr, i, kErrDirection);
                    break;
                }
            }
            if constexpr (KIND == SGS_MIXED) {
                if (deg_used < 0 || deg_used > sp.sh_degree) {
                    raise_error(ctr, i, kErrDegreeTooHigh);
                    break;
                }
                deg = deg_used;
            }
            // ---- colour (FP32) ----
            const float fx = static_cast<float>(dxd), fy = static_cast<float>(dyd),
                        fz = static_cast<float>(dzd);
            float col[3];
            if constexpr (KIND == SGS_SH || KIND == SGS_MIXED) {
                const int stored_planes = (3 * (sp.sh_degree + 1) * (sp.sh_degree + 1) + 3) / 4;
                const int need = (3 * (deg + 1) * (deg + 1) + 3) / 4;
                float c[48];
                load_planes<12>(sp.color, sp.n, i, need, c);
                float acc[3] = {0.f, 0.f, 0.f};
                sh_accumulate(c, deg, fx, fy, fz, acc);
                col[0] = 0.5f + acc[0];
                col[1] = 0.5f + acc[1];
                col[2] = 0.5f + acc[2];
                if constexpr (KIND == SGS_MIXED) {
                    float lobes[12];
                    load_planes<3>(sp.color + static_cast<uint64_t>(stored_planes) * sp.n, sp.n, i, 3,
                                   lobes);
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
                load_planes<3>(sp.color, sp.n, i, 3, f);
                const float lambda = expf(f[3]);
                const float e = expf(lambda * (fx * f[8] + fy * f[9] + fz * f[10] - 1.0f));
                col[0] = f[0] + f[4] * e;
                col[1] = f[1] + f[5] * e;
                col[2] = f[2] + f[6] * e;
            } else {
                float f[16];
                load_planes<4>(sp.color, sp.n, i, 4, f);
                float lacc[3] = {0.f, 0.f, 0.f};
                lobe_accumulate(f + 4, sp.axes, fx, fy, fz, lacc);
                col[0] = f[0] + lacc[0];
                col[1] = f[1] + lacc[1];
                col[2] = f[2] + lacc[2];
            }
            col[0] = fmaxf(col[0], 0.0f);  // cwiseMax(0), NaN-propagating like std::max(v, 0)
            col[1] = fmaxf(col[1], 0.0f);
            col[2] = fmaxf(col[2], 0.0f);

            // ---- outputs ----
            const double cona = ddiv(c, det), conb = ddiv(-b, det), conc = ddiv(a, det);
            const double opacity = ddiv(1.0, dadd(1.0, exp(-g.opl)));  // sigmoid, common.hpp:136
            visible = true;
            key = depth_key(tz);
            // tile rectangle (raster.cpp:117-122), inclusive, clamped
            const double ts = static_cast<double>(cfg.tile_size);
            int32_t x0 = to_int_x86(floor(ddiv(dsub(mx, radius), ts)));
            int32_t x1 = to_int_x86(floor(ddiv(dadd(mx, radius), ts)));
            int32_t y0 = to_int_x86(floor(ddiv(dsub(my, radius), ts)));
            int32_t y1 = to_int_x86(floor(ddiv(dadd(my, radius), ts)));
            x0 = max(0, x0);
            y0 = max(0, y0);
            x1 = min(cfg.tiles_x - 1, x1);
            y1 = min(cfg.tiles_y - 1, y1);
            if (x1 >= x0 && y1 >= y0)
                count = static_cast<uint32_t>(x1 - x0 + 1) * static_cast<uint32_t>(y1 - y0 + 1);
            rects[i] = make_int4(x0, x1, y0, y1);
            // FP32 m2 error bound: 2u S (9 r^2 + 3 r ts) + 1e-6
            const double csum = fabs(cona) + 2.0 * fabs(conb) + fabs(conc);
            const double guard =
                2.0 * 5.9604644775390625e-08 * csum * (9.0 * radius * radius + 3.0 * radius * ts) +
                1e-6;
            SplatRec r;
            r.mx = mx;
            r.my = my;
            r.ca = static_cast<float>(cona);
            r.cb2 = static_cast<float>(2.0 * conb);
            r.cc = static_cast<float>(conc);
            r.op = static_cast<float>(opacity);
            r.r = col[0];
            r.g = col[1];
            r.b = col[2];
            r.guard = guard < 1e30 ? static_cast<float>(guard) : FLT_MAX;
            rec[i] = r;
            SplatRec64 r64;
            r64.ca = cona;
            r64.cb = conb;
            r64.cc = conc;
            r64.op = opacity;
            rec64[i] = r64;
            if (debug) {
                dbg.mean2d[0] = mx;
                dbg.mean2d[1] = my;
                dbg.conic[0] = cona;
                dbg.conic[1] = conb;
                dbg.conic[2] = conc;
                dbg.depth = tz;
                dbg.color[0] = col[0];
                dbg.color[1] = col[1];
                dbg.color[2] = col[2];
                dbg.opacity = opacity;
                dbg.radius = radius;
                dbg.degree = KIND == SGS_MIXED ? deg_used : -1;
                dbg.visible = 1;
            }
        } while (false);
        depth_keys[i] = key;
        vkey = key;
        ntiles[i] = count;
        if (debug) debug[i] = dbg;
    }
    // visible count and depth-key range: one atomic each per warp
    const unsigned vote = __ballot_sync(0xffffffffu, visible);
    if (vote) {
        unsigned long long kmin = visible ? vkey : ~0ULL, kmax = visible ? vkey : 0ULL;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
            kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&ctr->visible, static_cast<unsigned long long>(__popc(vote)));
            atomicMin(&ctr->kmin, kmin);
            atomicMax(&ctr->kmax, kmax);
        }
    }
}

template <bool F64>
void launch_kind(const ScenePlanes& sp, const CamParams& cam, const CfgParams& cfg,
                 unsigned long long* keys, uint32_t* iota, SplatRec* rec, SplatRec64* rec64,
                 int4* rects, uint32_t* ntiles, Counters* ctr, DebugSplat* debug,
                 cudaStream_t stream) {
    const unsigned blocks = static_cast<unsigned>((sp.n + 255) / 256);
    switch (sp.kind) {
        case SGS_SH:
            preprocess_kernel<F64, SGS_SH><<<blocks, 256, 0, stream>>>(sp, cam, cfg, keys, iota, rec,
                                                                     rec64, rects, ntiles, ctr, debug);
            break;
        case SGS_SG1:
            preprocess_kernel<F64, SGS_SG1><<<blocks, 256, 0, stream>>>(sp, cam, cfg, keys, iota, rec,
                                                                      rec64, rects, ntiles, ctr, debug);
            break;
        case SGS_SG3:
            preprocess_kernel<F64, SGS_SG3><<<blocks, 256, 0, stream>>>(sp, cam, cfg, keys, iota, rec,
                                                                      rec64, rects, ntiles, ctr, debug);
            break;
        default:
            preprocess_kernel<F64, SGS_MIXED><<<blocks, 256, 0, stream>>>(
                sp, cam, cfg, keys, iota, rec, rec64, rects, ntiles, ctr, debug);
            break;
    }
}

}  // namespace

void launch_preprocess(const ScenePlanes& sp, const CamParams& cam, const CfgParams& cfg,
                       unsigned long long* depth_keys, uint32_t* iota, SplatRec* rec,
                       SplatRec64* rec64, int4* rects, uint32_t* ntiles, Counters* counters,
                       DebugSplat* debug, cudaStream_t stream) {
    if (sp.n == 0) return;
    if (sp.geometry_f64)
        launch_kind<true>(sp, cam, cfg, depth_keys, iota, rec, rec64, rects, ntiles, counters, debug,
                          stream);
    else
        launch_kind<false>(sp, cam, cfg, depth_keys, iota, rec, rec64, rects, ntiles, counters, debug,
                           stream);
}

}  // namespace sgs
