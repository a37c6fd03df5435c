// host_synth.cpp -- deterministic benchmark/parity inputs (host side of the C-ABI).
//
// make_synthetic_scene (proj/src/synth.cpp:26-106) with the reference's portable
// draws (common.hpp:91-121) and f32 rounding, make_orbit_camera
// (proj/src/camera.cpp:77-100) and make_orbit_cameras (proj/src/synth.cpp:108-118).
// The reference builds each Vec3 as Vec3(f(), f(), f()); g++ evaluates those
// constructor arguments right to left and evaluates the by-value Vec3 operand of
// `radius * cbrt(u) * random_unit_vector()` before the scalar. The draws below are
// written out in that order explicitly (pinned by tests/golden/synth.npz).
// Compiled with -ffp-contract=off so every product/sum rounds as the reference's.
#include <cmath>
#include <cstring>
#include <random>

#include "sgs.h"

namespace {

double uniform01(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
double uniform_range(std::mt19937_64& g, double lo, double hi) { return lo + (hi - lo) * uniform01(g); }
double normal01(std::mt19937_64& g) {
    double u1 = uniform01(g);
    double u2 = uniform01(g);
    if (u1 < 1e-300) u1 = 1e-300;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}
double f32(double v) {
    volatile float f = static_cast<float>(v);
    return static_cast<double>(f);
}
struct V3 {
    double v[3];
};
// Vec3(f(), f(), f()) with right-to-left argument evaluation.
template <typename F>
V3 draw3(F&& f) {
    V3 r;
    r.v[2] = f();
    r.v[1] = f();
    r.v[0] = f();
    return r;
}
V3 random_unit_vector(std::mt19937_64& g) {
    for (;;) {
        V3 r = draw3([&] { return normal01(g); });
        const double n = std::sqrt((r.v[0] * r.v[0] + r.v[1] * r.v[1]) + r.v[2] * r.v[2]);
        if (n > 1e-9) {
            for (double& x : r.v) x = x / n;
            return r;
        }
    }
}
void random_unit_quaternion(std::mt19937_64& g, double q[4]) {
    for (;;) {
        q[3] = normal01(g);
        q[2] = normal01(g);
        q[1] = normal01(g);
        q[0] = normal01(g);
        const double n = std::sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
        if (n > 1e-9) {
            for (int k = 0; k < 4; ++k) q[k] = q[k] / n;
            return;
        }
    }
}
int band_of(int k) { return k == 0 ? 0 : (k < 4 ? 1 : (k < 9 ? 2 : 3)); }
constexpr double kC0 = 0.28209479177387814;

void normalize(double v[3]) {
    const double z = (v[0] * v[0] + v[1] * v[1]) + v[2] * v[2];
    if (z > 0.0) {
        const double n = std::sqrt(z);
        for (int i = 0; i < 3; ++i) v[i] = v[i] / n;
    }
}
void cross(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

}  // namespace

extern "C" {

sgs_status sgs_synth_scene(uint64_t count, uint64_t seed, int32_t kind, int32_t sh_degree,
                           double ls_min, double ls_max, double* params) {
    if (kind < SGS_SH || kind > SGS_MIXED) return SGS_ERR_INVALID_ARGUMENT;
    if (kind == SGS_SH && (sh_degree < 0 || sh_degree > 3)) return SGS_ERR_INVALID_ARGUMENT;
    if (count && !params) return SGS_ERR_INVALID_ARGUMENT;
    // SynthOptions defaults (synth.hpp:10-25)
    const double cluster_radius = 1.0, op_min = 0.3, op_max = 0.95, base_min = 0.25, base_max = 0.75,
                 band_amp = 0.25, band_decay = 0.55, sg_amp = 0.15;
    std::mt19937_64 gen(seed);
    const int deg = kind == SGS_MIXED ? 2 : sh_degree;
    const size_t stride = 11 + static_cast<size_t>(sgs_color_param_count(kind, deg));
    for (uint64_t i = 0; i < count; ++i) {
        double* p = params + i * stride;
        const V3 dir = random_unit_vector(gen);
        const double s = cluster_radius * std::cbrt(uniform01(gen));
        for (int k = 0; k < 3; ++k) p[k] = f32(s * dir.v[k]);
        double q[4];
        random_unit_quaternion(gen, q);
        for (int k = 0; k < 4; ++k) p[3 + k] = f32(q[k]);
        const V3 ls = draw3([&] { return uniform_range(gen, ls_min, ls_max); });
        for (int k = 0; k < 3; ++k) p[7 + k] = f32(ls.v[k]);
        const double op = uniform_range(gen, op_min, op_max);
        p[10] = f32(std::log(op / (1.0 - op)));
        const V3 base = draw3([&] { return uniform_range(gen, base_min, base_max); });
        double* c = p + 11;
        if (kind == SGS_SH || kind == SGS_MIXED) {
            const int ncoef = (deg + 1) * (deg + 1);
            for (int ch = 0; ch < 3; ++ch) c[ch] = f32((base.v[ch] - 0.5) / kC0);
            for (int k = 1; k < ncoef; ++k) {
                const double amp = band_amp * std::pow(band_decay, band_of(k));
                const V3 r = draw3([&] { return uniform_range(gen, -amp, amp); });
                for (int ch = 0; ch < 3; ++ch) c[3 * k + ch] = f32(r.v[ch]);
            }
            if (kind == SGS_MIXED) {
                double* lobes = c + 3 * ncoef;
                for (int l = 0; l < 3; ++l) {
                    const V3 a = draw3([&] { return uniform_range(gen, -sg_amp, sg_amp); });
                    for (int ch = 0; ch < 3; ++ch) lobes[4 * l + ch] = f32(a.v[ch]);
                    lobes[4 * l + 3] = f32(uniform_range(gen, -0.5, 1.5));
                }
            }
        } else if (kind == SGS_SG1) {
            for (int ch = 0; ch < 3; ++ch) c[ch] = f32(base.v[ch]);
            const V3 a = draw3([&] { return uniform_range(gen, -sg_amp, sg_amp); });
            for (int ch = 0; ch < 3; ++ch) c[3 + ch] = f32(a.v[ch]);
            c[6] = f32(uniform_range(gen, -0.5, 1.5));
            const V3 mu = random_unit_vector(gen);
            for (int ch = 0; ch < 3; ++ch) c[7 + ch] = f32(mu.v[ch]);
        } else {
            for (int ch = 0; ch < 3; ++ch) c[ch] = f32(base.v[ch]);
            for (int l = 0; l < 3; ++l) {
                const V3 a = draw3([&] { return uniform_range(gen, -sg_amp, sg_amp); });
                for (int ch = 0; ch < 3; ++ch) c[3 + 4 * l + ch] = f32(a.v[ch]);
                c[3 + 4 * l + 3] = f32(uniform_range(gen, -0.5, 1.5));
            }
        }
    }
    return SGS_OK;
}

sgs_status sgs_synth_sh3_from_mixed(uint64_t count, uint64_t seed, const double* mixed, double* sh3) {
    if (count && (!mixed || !sh3)) return SGS_ERR_INVALID_ARGUMENT;
    const size_t ms = 11 + 39, ss = 11 + 48;
    std::mt19937_64 gen(seed + 1);
    const double amp = 0.25 * std::pow(0.55, 3);
    for (uint64_t i = 0; i < count; ++i) {
        const double* m = mixed + i * ms;
        double* o = sh3 + i * ss;
        std::memcpy(o, m, sizeof(double) * (11 + 27));
        for (int k = 9; k < 16; ++k)
            for (int ch = 0; ch < 3; ++ch) o[11 + 3 * k + ch] = f32(uniform_range(gen, -amp, amp));
    }
    return SGS_OK;
}

sgs_status sgs_orbit_camera(const double* target, double distance, double angle, double elevation,
                            int32_t width, int32_t height, double focal, sgs_camera* cam) {
    if (!target || !cam) return SGS_ERR_INVALID_ARGUMENT;
    const double dir[3] = {std::cos(angle) * std::cos(elevation), std::sin(angle) * std::cos(elevation),
                           std::sin(elevation)};
    double eye[3], fwd[3], up[3] = {0, 0, 1}, right[3], down[3];
    for (int i = 0; i < 3; ++i) eye[i] = target[i] + distance * dir[i];
    for (int i = 0; i < 3; ++i) fwd[i] = target[i] - eye[i];
    normalize(fwd);
    if (std::abs((fwd[0] * up[0] + fwd[1] * up[1]) + fwd[2] * up[2]) > 0.99) {
        up[0] = 0;
        up[1] = 1;
        up[2] = 0;
    }
    cross(fwd, up, right);
    normalize(right);
    cross(fwd, right, down);
    std::memset(cam, 0, sizeof(*cam));
    for (int c = 0; c < 3; ++c) {
        cam->R[c] = right[c];
        cam->R[3 + c] = down[c];
        cam->R[6 + c] = fwd[c];
    }
    for (int r = 0; r < 3; ++r)
        cam->t[r] = ((-cam->R[r * 3]) * eye[0] + (-cam->R[r * 3 + 1]) * eye[1]) + (-cam->R[r * 3 + 2]) * eye[2];
    cam->fx = cam->fy = focal;
    cam->cx = width / 2.0;
    cam->cy = height / 2.0;
    cam->width = width;
    cam->height = height;
    cam->near_plane = 0.01;
    if (focal <= 0 || width < 1 || height < 1) return SGS_ERR_INVALID_ARGUMENT;  // validate()
    return SGS_OK;
}

sgs_status sgs_orbit_cameras(int32_t count, int32_t width, int32_t height, double distance, double focal,
                             double elevation, sgs_camera* out) {
    const double target[3] = {0, 0, 0};
    for (int i = 0; i < count; ++i) {
        const double angle = 2.0 * M_PI * i / count;
        sgs_status st = sgs_orbit_camera(target, distance, angle, elevation, width, height, focal, &out[i]);
        if (st != SGS_OK) return st;
    }
    return SGS_OK;
}

}  // extern "C"
