// sgsplat/common.hpp -- drop-in declarations for the B200 renderer's C++ API.
//
// Same names, types and semantics as the reference's proj/include/sgsplat/common.hpp
// (Eigen aliases :14-18, exception taxonomy :21-42, portable RNG helpers :91-121,
// quat_to_rotation :124-134, sigmoid/logit :136-137), so reference callers compile
// unchanged against libsgsplat_b200.so. Eigen comes from the system if present,
// else from third_party/eigen_subset (layout-compatible fixed-size subset).
#pragma once

#include <Eigen/Dense>

#include <cmath>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>

namespace sgsplat {

using Vec2 = Eigen::Vector2d;
using Vec3 = Eigen::Vector3d;
using Vec4 = Eigen::Vector4d;
using Mat2 = Eigen::Matrix2d;
using Mat3 = Eigen::Matrix3d;

// Contract violations (maps from SGS_ERR_INVALID_ARGUMENT).
struct InvalidArgument : std::runtime_error {
    explicit InvalidArgument(const std::string& what) : std::runtime_error(what) {}
};
// Malformed files.
struct FormatError : std::runtime_error {
    explicit FormatError(const std::string& what) : std::runtime_error(what) {}
};
// I/O failures.
struct IoError : std::runtime_error {
    explicit IoError(const std::string& what) : std::runtime_error(what) {}
};
// Broken numeric invariants (maps from SGS_ERR_NUMERIC).
struct NumericError : std::runtime_error {
    explicit NumericError(const std::string& what) : std::runtime_error(what) {}
};

// 0 -> hardware concurrency. The GPU renderer ignores thread counts; kept for API parity.
inline int resolve_thread_count(int requested) {
    if (requested > 0) return requested;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(hw) : 1;
}

// Portable seeded draws (identical streams to the reference's helpers).
inline double uniform01(std::mt19937_64& gen) { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
inline double uniform_range(std::mt19937_64& gen, double lo, double hi) { return lo + (hi - lo) * uniform01(gen); }
inline double normal01(std::mt19937_64& gen) {
    double u1 = uniform01(gen);
    const double u2 = uniform01(gen);
    if (u1 < 1e-300) u1 = 1e-300;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}
// Note the reference draws these as Vec3(normal01(), normal01(), normal01()); with
// g++ the arguments are evaluated right to left, reproduced here explicitly.
inline Vec3 random_unit_vector(std::mt19937_64& gen) {
    for (;;) {
        const double z = normal01(gen), y = normal01(gen), x = normal01(gen);
        Vec3 v(x, y, z);
        const double n = v.norm();
        if (n > 1e-9) return v / n;
    }
}
inline Vec4 random_unit_quaternion(std::mt19937_64& gen) {
    for (;;) {
        const double d = normal01(gen), c = normal01(gen), b = normal01(gen), a = normal01(gen);
        Vec4 q(a, b, c, d);
        const double n = q.norm();
        if (n > 1e-9) return q / n;
    }
}

// Rotation from a possibly unnormalised (w, x, y, z) quaternion.
Mat3 quat_to_rotation(const Vec4& q);

inline double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }
inline double logit(double p) { return std::log(p / (1.0 - p)); }

}  // namespace sgsplat
