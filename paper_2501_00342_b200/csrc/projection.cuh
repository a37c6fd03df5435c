// projection.cuh -- the FP64 EWA projection shared by K1 and K7's guard band.
//
// project_cached (proj/src/raster.cpp:17-60), covariance (proj/src/scene.cpp:81-85)
// and quat_to_rotation (proj/include/sgsplat/common.hpp:124-134) in the reference's
// exact operation order, with round-to-nearest intrinsics so nvcc cannot contract
// products into FMAs. K1 calls it once per Gaussian; the compositor calls it again
// for the rare (pixel, splat) pairs inside the FP32 guard band, which reproduces
// the FP64 conic and opacity bit for bit without storing them.
#pragma once

#include "sgs_internal.h"

namespace sgs {

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

// 3D covariance (covariance, scene.cpp:81-85, with quat_to_rotation,
// common.hpp:124-134) in the reference's operation order. It is view independent,
// so it is computed once per scene (cov3d_kernel, at upload/bind) and cached as six
// FP64 planes; K1 and the guard band read it instead of re-deriving it per view.
// Returns false for a zero quaternion (the caller raises the error only when the
// splat survives the near cull, as raster.cpp:23 precedes common.hpp:126).
__device__ __forceinline__ bool covariance3d(const double q[4], const double ls[3], double S6[6]) {
    const double qn = __dsqrt_rn(
        dadd(dadd(dadd(dmul(q[0], q[0]), dmul(q[1], q[1])), dmul(q[2], q[2])), dmul(q[3], q[3])));
    if (qn < 1e-12) return false;
    const double w = ddiv(q[0], qn), x = ddiv(q[1], qn), y = ddiv(q[2], qn), z = ddiv(q[3], qn);
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
    // M = Rq diag(exp(s)); S = M M^T (symmetric bit for bit: dot3 is commutative per term)
    const double sc[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
    double M[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c) M[r * 3 + c] = dmul(Rq[r * 3 + c], sc[c]);
    auto row = [&](int a, int b) {
        return dot3(M[a * 3 + 0], M[a * 3 + 1], M[a * 3 + 2], M[b * 3 + 0], M[b * 3 + 1], M[b * 3 + 2]);
    };
    S6[0] = row(0, 0);
    S6[1] = row(0, 1);
    S6[2] = row(0, 2);
    S6[3] = row(1, 1);
    S6[4] = row(1, 2);
    S6[5] = row(2, 2);
    return true;
}

// Cached covariance planes: cov[0] = (S00, S01), cov[1] = (S02, S11), cov[2] =
// (S12, S22); a zero quaternion is marked by S00 = -1 (a valid S00 is a sum of
// squares: >= 0 or NaN).
constexpr double kZeroQuatMark = -1.0;

struct Geo {
    double p[3], opl;
    double S[6];  // S00 S01 S02 S11 S12 S22
};

template <bool F64>
__device__ __forceinline__ void load_geo(const ScenePlanes& sp, uint64_t i, Geo& g) {
    if constexpr (F64) {
        g.p[0] = sp.g8[0][i];
        g.p[1] = sp.g8[1][i];
        g.p[2] = sp.g8[2][i];
        g.opl = sp.g8[10][i];
    } else {
        const float4 a = __ldg(&sp.g4[0][i]);
        g.p[0] = a.x;
        g.p[1] = a.y;
        g.p[2] = a.z;
        g.opl = a.w;
    }
    const double2 c0 = __ldg(&sp.cov[0][i]);
    const double2 c1 = __ldg(&sp.cov[1][i]);
    const double2 c2 = __ldg(&sp.cov[2][i]);
    g.S[0] = c0.x;
    g.S[1] = c0.y;
    g.S[2] = c1.x;
    g.S[3] = c1.y;
    g.S[4] = c2.x;
    g.S[5] = c2.y;
}

enum ProjStatus { kProjVisible = 0, kProjCulled = 1, kProjZeroQuat = 2 };

struct ProjGeo {
    double tx, ty, tz;
    double mx, my, radius;
    double a, b, c, det;  // dilated 2D covariance
    double cona, conb, conc, opacity;
};

// project_cached's geometry (raster.cpp:17-60) from a loaded Geo (position,
// logit opacity and the cached 3D covariance).
__device__ __forceinline__ int project_staged(const Geo& g, const CamParams& cam, ProjGeo& o) {
    // t = R p + t (camera.hpp:19)
    const double* R = cam.R;
    const double tx = dadd(dot3(R[0], R[1], R[2], g.p[0], g.p[1], g.p[2]), cam.t[0]);
    const double ty = dadd(dot3(R[3], R[4], R[5], g.p[0], g.p[1], g.p[2]), cam.t[1]);
    const double tz = dadd(dot3(R[6], R[7], R[8], g.p[0], g.p[1], g.p[2]), cam.t[2]);
    o.tx = tx;
    o.ty = ty;
    o.tz = tz;
    if (tz < cam.near_plane) return kProjCulled;  // raster.cpp:23
    if (g.S[0] == kZeroQuatMark) return kProjZeroQuat;
    // full symmetric S, row-major
    const double S[9] = {g.S[0], g.S[1], g.S[2], g.S[1], g.S[3], g.S[4], g.S[2], g.S[4], g.S[5]};
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
            Tm[a * 3 + b] = dot3(J[a * 3 + 0], J[a * 3 + 1], J[a * 3 + 2], R[0 * 3 + b], R[1 * 3 + b], R[2 * 3 + b]);
    double TS[6];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            TS[a * 3 + b] = dot3(Tm[a * 3 + 0], Tm[a * 3 + 1], Tm[a * 3 + 2], S[0 * 3 + b], S[1 * 3 + b], S[2 * 3 + b]);
    const double a = dadd(dot3(TS[0], TS[1], TS[2], Tm[0], Tm[1], Tm[2]), kCovarianceDilation);
    const double b = dot3(TS[0], TS[1], TS[2], Tm[3], Tm[4], Tm[5]);
    const double c = dadd(dot3(TS[3], TS[4], TS[5], Tm[3], Tm[4], Tm[5]), kCovarianceDilation);
    const double det = dsub(dmul(a, c), dmul(b, b));
    if (det <= 0.0) return kProjCulled;  // raster.cpp:48 (NaN passes, as in the reference)
    const double mid = dmul(0.5, dadd(a, c));
    const double disc = dsub(dmul(mid, mid), det);
    const double lambda_max = dadd(mid, __dsqrt_rn(0.0 < disc ? disc : 0.0));
    const double radius = dmul(3.0, __dsqrt_rn(lambda_max));
    const double mx = dadd(ddiv(dmul(cam.fx, tx), tz), cam.cx);
    const double my = dadd(ddiv(dmul(cam.fy, ty), tz), cam.cy);
    if (dadd(mx, radius) < 0.0 || dsub(mx, radius) > cam.width || dadd(my, radius) < 0.0 ||
        dsub(my, radius) > cam.height)
        return kProjCulled;  // raster.cpp:56-60
    o.mx = mx;
    o.my = my;
    o.radius = radius;
    o.a = a;
    o.b = b;
    o.c = c;
    o.det = det;
    return kProjVisible;
}

template <bool F64>
__device__ __forceinline__ int project_geometry(const ScenePlanes& sp, const CamParams& cam, uint64_t i,
                                                Geo& g, ProjGeo& o) {
    load_geo<F64>(sp, i, g);
    return project_staged(g, cam, o);
}

// The reference's conic (raster.cpp:62) and activated opacity (scene.hpp:20,
// common.hpp:136), bit for bit. K1 only needs them to FP32 accuracy and uses a
// cheaper form; the compositor's guard band and the debug dump use this one.
__device__ __forceinline__ void exact_conic_opacity(const Geo& g, ProjGeo& o) {
    o.cona = ddiv(o.c, o.det);
    o.conb = ddiv(-o.b, o.det);
    o.conc = ddiv(o.a, o.det);
    o.opacity = ddiv(1.0, dadd(1.0, exp(-g.opl)));
}

}  // namespace sgs
