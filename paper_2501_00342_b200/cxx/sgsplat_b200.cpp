// sgsplat_b200.cpp -- the reference's C++ render API (include/sgsplat/*.hpp) served
// by the B200 renderer through the C-ABI (include/sgs.h).
//
// render()/project() convert the caller's Scene (AoS doubles, std::variant colour)
// into the reference's flat parameter layout (Scene::param order, scene.hpp:40-43),
// upload it, and run the sm_100a pipeline; the float32 frame is widened into the
// double Image the reference returns (raster.hpp:49-52). sgs_* error codes are
// rethrown as the reference's exceptions (common.hpp:21-42). The scalar colour /
// scene / camera helpers are host code with the reference's semantics; they are
// utilities, not a render fallback -- render() has no CPU path.
#include "sgs.h"
#include "sgsplat/grad.hpp"
#include "sgsplat/metrics.hpp"
#include "sgsplat/ply.hpp"
#include "sgsplat/raster.hpp"
#include "sgsplat/synth.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <memory>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <sstream>
#include <thread>

namespace sgsplat {

namespace {

[[noreturn]] void rethrow(int status) {
    const std::string msg = sgs_last_error();
    if (status == SGS_ERR_INVALID_ARGUMENT) throw InvalidArgument(msg);
    if (status == SGS_ERR_NUMERIC) throw NumericError(msg);
    if (status == SGS_ERR_IO) throw IoError(msg);
    if (status == SGS_ERR_FORMAT) throw FormatError(msg);
    throw std::runtime_error("B200 renderer: " + msg);
}

void check(int status) {
    if (status != SGS_OK) rethrow(status);
}

sgs_context* context() {
    static std::once_flag once;
    static sgs_context* ctx = nullptr;
    static int status = SGS_OK;
    std::call_once(once, [] {
        const char* dev = std::getenv("SGS_DEVICE");
        status = sgs_create(dev ? std::atoi(dev) : 0, &ctx);
    });
    if (status != SGS_OK) rethrow(status);
    return ctx;
}

int stored_degree(const ColorModel& m) {
    if (auto* s = std::get_if<SHOnlyModel>(&m)) return s->sh.degree;
    if (auto* x = std::get_if<MixedSHSGModel>(&m)) return x->sh.degree;
    return 0;
}

sgs_camera to_c(const Camera& cam) {
    sgs_camera c{};
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) c.R[r * 3 + k] = cam.rotation(r, k);
    for (int r = 0; r < 3; ++r) c.t[r] = cam.translation[r];
    c.fx = cam.fx;
    c.fy = cam.fy;
    c.cx = cam.cx;
    c.cy = cam.cy;
    c.width = cam.width;
    c.height = cam.height;
    c.near_plane = cam.near;
    return c;
}

sgs_render_config to_c(const RenderConfig& cfg) {
    sgs_render_config k{};
    k.tile_size = cfg.tile_size;
    k.has_override = cfg.sh_degree_override.has_value() ? 1 : 0;
    k.override_degree = cfg.sh_degree_override.value_or(0);
    k.threads = cfg.threads;
    k.degree_threshold_lo = cfg.degree_threshold_lo;
    k.degree_threshold_hi = cfg.degree_threshold_hi;
    k.early_stop_transmittance = cfg.early_stop_transmittance;
    return k;
}

// RAII device scene built from a (homogeneous) Scene.
struct DeviceScene {
    sgs_scene* s = nullptr;
    std::vector<double> flat;
    DeviceScene(const std::vector<GaussianPrimitive>& gs, const Mat3& axes, const Vec3& bg) {
        sgs_scene_desc d{};
        d.count = gs.size();
        d.kind = gs.empty() ? SGS_SH : static_cast<int32_t>(kind_of(gs.front().color));
        d.sh_degree = gs.empty() ? 0 : stored_degree(gs.front().color);
        d.dtype = SGS_F64;
        if (!gs.empty()) {
            const std::size_t stride = kGeometryParams + param_count(gs.front().color);
            flat.resize(gs.size() * stride);
            for (std::size_t i = 0; i < gs.size(); ++i) {
                const GaussianPrimitive& g = gs[i];
                double* p = flat.data() + i * stride;
                for (int k = 0; k < 3; ++k) p[k] = g.position[k];
                for (int k = 0; k < 4; ++k) p[3 + k] = g.rotation[k];
                for (int k = 0; k < 3; ++k) p[7 + k] = g.log_scale[k];
                p[10] = g.opacity_logit;
                const int nc = static_cast<int>(stride) - kGeometryParams;
                for (int k = 0; k < nc; ++k) p[kGeometryParams + k] = color_param(g.color, k);
            }
            d.params = flat.data();
        }
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) d.shared_axes[r * 3 + c] = axes(r, c);
        for (int c = 0; c < 3; ++c) d.background[c] = bg[c];
        check(sgs_scene_upload(context(), &d, &s));
    }
    ~DeviceScene() { sgs_scene_free(s); }
};

// ---- the render() fast path -------------------------------------------------
// Host loops over Gaussians / pixels on every core: fn(begin, end).
template <typename Fn>
void parallel_for(std::size_t n, Fn&& fn) {
    const std::size_t hw = std::max<unsigned>(std::thread::hardware_concurrency(), 1u);
    const std::size_t nt = std::min<std::size_t>(hw, n / 32768 + 1);
    if (nt <= 1) {
        fn(std::size_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    const std::size_t per = (n + nt - 1) / nt;
    for (std::size_t t = 0; t < nt; ++t) {
        const std::size_t b = t * per, e = std::min(n, b + per);
        if (b < e) pool.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& th : pool) th.join();
}

// Pinned host staging reused by every render() call (grow-only): scene rows up, frames
// down, both at DMA speed.
struct PinnedBuf {
    void* p = nullptr;
    std::size_t bytes = 0;
    void* get(std::size_t need) {
        if (need > bytes) {
            sgs_host_free(p);
            p = nullptr;
            bytes = 0;
            if (sgs_host_alloc(need, &p) != SGS_OK) throw std::bad_alloc();
            bytes = need;
        }
        return p;
    }
};
std::mutex g_stage_mu;  // render() calls share the staging (the reference is reentrant:
PinnedBuf g_rows, g_frame;  // concurrent calls serialise here, results stay per call)
// The device scene every render() call repacks its scene into (sgs_scene_update: same
// planes, no device allocation per call) while the layout stays the same.
sgs_scene* g_scene = nullptr;

// The colour parameters of one Gaussian in canonical order (one variant visit).
template <typename T>
void pack_color(const ColorModel& model, T* out) {
    std::visit(
        [&](const auto& m) {
            using M = std::decay_t<decltype(m)>;
            int k = 0;
            if constexpr (std::is_same_v<M, SHOnlyModel>) {
                for (const Vec3& c : m.sh.coeffs)
                    for (int j = 0; j < 3; ++j) out[k++] = static_cast<T>(c[j]);
            } else if constexpr (std::is_same_v<M, DiffuseSGModel>) {
                for (int j = 0; j < 3; ++j) out[k++] = static_cast<T>(m.diffuse[j]);
                for (int j = 0; j < 3; ++j) out[k++] = static_cast<T>(m.alpha[j]);
                out[k++] = static_cast<T>(m.log_lambda);
                for (int j = 0; j < 3; ++j) out[k++] = static_cast<T>(m.mu[j]);
            } else if constexpr (std::is_same_v<M, DiffuseOrthoSGModel>) {
                for (int j = 0; j < 3; ++j) out[k++] = static_cast<T>(m.diffuse[j]);
                for (int l = 0; l < 3; ++l) {
                    for (int j = 0; j < 3; ++j) out[k++] = static_cast<T>(m.alpha[static_cast<std::size_t>(l)][j]);
                    out[k++] = static_cast<T>(m.log_lambda[static_cast<std::size_t>(l)]);
                }
            } else {
                for (const Vec3& c : m.sh.coeffs)
                    for (int j = 0; j < 3; ++j) out[k++] = static_cast<T>(c[j]);
                for (int l = 0; l < 3; ++l) {
                    for (int j = 0; j < 3; ++j) out[k++] = static_cast<T>(m.alpha[static_cast<std::size_t>(l)][j]);
                    out[k++] = static_cast<T>(m.log_lambda[static_cast<std::size_t>(l)]);
                }
            }
        },
        model);
}

bool f32_exact(double v) { return static_cast<double>(static_cast<float>(v)) == v; }

// The scene as float32 rows in pinned memory, packed on every core; false when some
// parameter is not f32-exact (the caller then takes the float64 path). *mixed: some
// Gaussian's colour model or stored degree differs from the first one's
// (Scene::check_homogeneous then raises the reference's error).
bool pack_rows_f32(const std::vector<GaussianPrimitive>& gs, std::size_t first, std::size_t count,
                   std::size_t stride, float* rows, bool* mixed) {
    std::atomic<bool> exact{true}, hetero{false};
    const ColorModelKind kind0 = kind_of(gs.front().color);
    const int deg0 = stored_degree(gs.front().color);
    parallel_for(count, [&](std::size_t b, std::size_t e) {
        std::vector<double> c(stride - kGeometryParams);
        bool ok = true;
        for (std::size_t i = first + b; i < first + e && ok; ++i) {
            const GaussianPrimitive& g = gs[i];
            if (kind_of(g.color) != kind0 || stored_degree(g.color) != deg0) {
                hetero.store(true);
                ok = false;
                break;
            }
            double p[kGeometryParams];
            for (int k = 0; k < 3; ++k) p[k] = g.position[k];
            for (int k = 0; k < 4; ++k) p[3 + k] = g.rotation[k];
            for (int k = 0; k < 3; ++k) p[7 + k] = g.log_scale[k];
            p[10] = g.opacity_logit;
            pack_color(g.color, c.data());
            float* r = rows + (i - first) * stride;
            for (int k = 0; k < kGeometryParams; ++k) {
                ok = ok && f32_exact(p[k]);
                r[k] = static_cast<float>(p[k]);
            }
            for (std::size_t k = 0; k < c.size(); ++k) {
                ok = ok && f32_exact(c[k]);
                r[kGeometryParams + k] = static_cast<float>(c[k]);
            }
        }
        if (!ok) exact.store(false);
    });
    *mixed = hetero.load();
    return exact.load();
}

// sgs_scene_update_rows' row producer: packs the caller's Scene block by block while
// the library copies the previous block to the device.
struct RowFill {
    const std::vector<GaussianPrimitive>* gs;
    std::size_t stride;
    bool mixed = false, inexact = false;
    static int32_t call(void* user, float* rows, uint64_t first, uint64_t count) {
        RowFill& f = *static_cast<RowFill*>(user);
        bool mixed = false;
        const bool exact = pack_rows_f32(*f.gs, first, count, f.stride, rows, &mixed);
        f.mixed = f.mixed || mixed;
        f.inexact = f.inexact || !exact;
        return mixed || !exact ? 1 : 0;
    }
};

}  // namespace

// ---------------------------------------------------------------------------- raster

int select_degree(double radius_px, double lo, double hi) {
    int32_t out = 0;
    check(sgs_select_degree(radius_px, lo, hi, &out));
    return out;
}

int flops_per_gaussian(ColorModelKind kind, int sh_degree) {
    int32_t out = 0;
    check(sgs_flops_per_gaussian(static_cast<int32_t>(kind), sh_degree, &out));
    return out;
}

std::optional<Splat2D> project(const GaussianPrimitive& g, const Camera& cam, const Mat3& shared_axes,
                               const RenderConfig& cfg) {
    DeviceScene ds({g}, shared_axes, Vec3::Zero());
    const sgs_camera c = to_c(cam);
    const sgs_render_config k = to_c(cfg);
    sgs_splat out{};
    check(sgs_project(context(), ds.s, &c, &k, &out));
    if (!out.visible) return std::nullopt;
    Splat2D s;
    s.mean2d = Vec2(out.mean2d[0], out.mean2d[1]);
    s.conic = Vec3(out.conic[0], out.conic[1], out.conic[2]);
    s.depth = out.depth;
    s.color = Vec3(out.color[0], out.color[1], out.color[2]);
    s.opacity = out.opacity;
    s.radius_px = out.radius;
    return s;
}

RenderResult render(const Scene& scene, const Camera& cam, const RenderConfig& cfg) {
    if (cfg.tile_size < 1) throw InvalidArgument("tile_size must be >= 1");
    // project_scene's checks (raster.cpp:82-85): the scene's homogeneity -- folded into
    // the packing below -- then the camera
    std::unique_lock<std::mutex> stage(g_stage_mu);
    // SGS_DROPIN_TRACE=1: per-phase wall times of each call on stderr
    static const bool trace = [] {
        const char* e = std::getenv("SGS_DROPIN_TRACE");
        return e && std::atoi(e) != 0;
    }();
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    auto t1 = t0, t2 = t0;
    // the scene: float32 rows packed on every core into pinned memory, scattered into
    // the device planes by a kernel (sgs_scene_upload of an SGS_F32 description) --
    // exactly the planes of the float64 path whenever every value is f32-exact
    // (synthetic scenes and PLY checkpoints are); otherwise the float64 path
    std::unique_ptr<DeviceScene> slow;
    RenderResult out;
    std::thread alloc;
    struct Join {
        std::thread& t;
        ~Join() {
            if (t.joinable()) t.join();
        }
    } join_alloc{alloc};
    // the result images (66 MB at 1080p, zeroed by their constructor: page faults and
    // stores on one core) are allocated while the rows are packed and cross PCIe; an
    // invalid size is left to cam.validate() below
    if (cam.width >= 1 && cam.height >= 1)
        alloc = std::thread([&] {
            out.image = Image(cam.width, cam.height, 3);
            out.transmittance = Image(cam.width, cam.height, 1);
        });
    sgs_scene* dscene = nullptr;
    const std::vector<GaussianPrimitive>& gs = scene.gaussians;
    const std::size_t stride = gs.empty() ? 0 : kGeometryParams + param_count(gs.front().color);
    bool fast = !gs.empty();
    if (fast) {
        sgs_scene_desc d{};
        d.count = gs.size();
        d.kind = static_cast<int32_t>(kind_of(gs.front().color));
        d.sh_degree = stored_degree(gs.front().color);
        d.dtype = SGS_F32;
        for (int r = 0; r < 3; ++r)
            for (int c2 = 0; c2 < 3; ++c2) d.shared_axes[r * 3 + c2] = scene.shared_axes(r, c2);
        for (int c2 = 0; c2 < 3; ++c2) d.background[c2] = scene.background[c2];
        bool streamed = false;
        if (g_scene) {
            // the resident scene takes the new rows in place, packed block by block
            // while the previous block crosses PCIe
            RowFill f{&gs, stride};
            const sgs_status st = sgs_scene_update_rows(context(), g_scene, &d, &RowFill::call, &f);
            if (f.mixed) scene.check_homogeneous();  // throws the reference's InvalidArgument
            streamed = st == SGS_OK;
            if (f.inexact) fast = false;  // (g_scene kept its contents) the float64 path
            // otherwise a different layout: packed and uploaded below as a new scene
        }
        if (fast && !streamed) {
            float* rows = static_cast<float*>(g_rows.get(gs.size() * stride * sizeof(float)));
            bool mixed = false;
            fast = pack_rows_f32(gs, 0, gs.size(), stride, rows, &mixed);
            if (mixed) scene.check_homogeneous();
            if (fast) {
                cam.validate();  // (before the upload, as the reference checks it first)
                d.params = rows;
                sgs_scene_free(g_scene);
                g_scene = nullptr;
                check(sgs_scene_upload(context(), &d, &g_scene));
            }
        }
        t1 = now();
        if (fast) {
            cam.validate();
            dscene = g_scene;
        }
    }
    t2 = now();
    if (!fast) {
        scene.check_homogeneous();
        cam.validate();
        slow = std::make_unique<DeviceScene>(scene.gaussians, scene.shared_axes, scene.background);
        dscene = slow->s;
    }
    const sgs_camera c = to_c(cam);
    const sgs_render_config k = to_c(cfg);
    const std::size_t npx = static_cast<std::size_t>(cam.width) * static_cast<std::size_t>(cam.height);
    if (alloc.joinable()) {
        alloc.join();
    } else {
        out.image = Image(cam.width, cam.height, 3);
        out.transmittance = Image(cam.width, cam.height, 1);
    }
    // SGS_EXACT=1: the reference's FP64 compositing (sgs_render_f64); default: the
    // FP32 throughput path (exact decisions, image within 1e-5)
    static const bool exact = [] {
        const char* e = std::getenv("SGS_EXACT");
        return e && std::atoi(e) != 0;
    }();
    if (exact) {
        check(sgs_render_f64(context(), dscene, &c, &k, out.image.data.data(), out.transmittance.data.data(),
                             SGS_HOST));
        return out;
    }
    // float32 frame into pinned memory, widened to the double Image on every core
    float* rgb = static_cast<float*>(g_frame.get(npx * 4 * sizeof(float)));
    float* T = rgb + npx * 3;
    const auto t3 = now();
    check(sgs_render(context(), dscene, &c, &k, rgb, T, SGS_HOST, nullptr));
    const auto t4 = now();
    parallel_for(npx, [&](std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i) {
            out.image.data[3 * i] = rgb[3 * i];
            out.image.data[3 * i + 1] = rgb[3 * i + 1];
            out.image.data[3 * i + 2] = rgb[3 * i + 2];
            out.transmittance.data[i] = T[i];
        }
    });
    if (trace)
        std::fprintf(stderr, "dropin: scene (pack + upload) %.2f tail %.2f image-wait %.2f render %.2f widen %.2f ms\n",
                     ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, now()));
    return out;
}

// ---------------------------------------------------------------------------- common / scene

Mat3 quat_to_rotation(const Vec4& q_raw) {
    const double n = q_raw.norm();
    if (n < 1e-12) throw NumericError("degenerate rotation: zero quaternion");
    const Vec4 q = q_raw / n;
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    Mat3 r;
    r << 1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),  //
        2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),   //
        2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y);
    return r;
}

Mat3 covariance(const Vec4& rotation, const Vec3& log_scale) {
    const Mat3 m = quat_to_rotation(rotation) * Vec3(log_scale.array().exp()).asDiagonal();
    return m * m.transpose();
}

double gaussian_density(const GaussianPrimitive& g, const Vec3& x) {
    const Mat3 sigma = covariance(g.rotation, g.log_scale) + 1e-9 * Mat3::Identity();
    const double det = sigma.determinant();
    if (!(det > 0.0) || !std::isfinite(det)) throw NumericError("covariance is singular after regularization");
    const Vec3 d = x - g.position;
    return std::exp(-0.5 * d.dot(sigma.inverse() * d));
}

void Scene::check_homogeneous() const {
    if (gaussians.empty()) return;
    const ColorModelKind kind = kind_of(gaussians.front().color);
    const int deg = stored_degree(gaussians.front().color);
    for (std::size_t i = 1; i < gaussians.size(); ++i) {
        const ColorModel& c = gaussians[i].color;
        if (kind_of(c) != kind)
            throw InvalidArgument("scene mixes color model variants (gaussian " + std::to_string(i) + ")");
        if ((kind == ColorModelKind::SHOnly || kind == ColorModelKind::MixedSHSG) && stored_degree(c) != deg)
            throw InvalidArgument("scene mixes SH degrees");
    }
}

ColorModelKind Scene::model_kind() const {
    if (gaussians.empty()) throw InvalidArgument("empty scene has no color model");
    check_homogeneous();
    return kind_of(gaussians.front().color);
}

void Scene::set_shared_axes(const Mat3& axes) {
    validate_ortho_axes(axes);
    shared_axes = axes;
}

std::size_t Scene::params_per_gaussian() const {
    return gaussians.empty() ? 0 : static_cast<std::size_t>(kGeometryParams + param_count(gaussians.front().color));
}

std::size_t Scene::total_params() const { return params_per_gaussian() * gaussians.size(); }

double Scene::param(std::size_t flat_index) const {
    const std::size_t stride = params_per_gaussian();
    if (stride == 0 || flat_index >= total_params()) throw InvalidArgument("parameter index out of range");
    const GaussianPrimitive& g = gaussians[flat_index / stride];
    const int slot = static_cast<int>(flat_index % stride);
    if (slot < 3) return g.position[slot];
    if (slot < 7) return g.rotation[slot - 3];
    if (slot < 10) return g.log_scale[slot - 7];
    if (slot == 10) return g.opacity_logit;
    return color_param(g.color, slot - kGeometryParams);
}

void Scene::set_param(std::size_t flat_index, double value) {
    const std::size_t stride = params_per_gaussian();
    if (stride == 0 || flat_index >= total_params()) throw InvalidArgument("parameter index out of range");
    GaussianPrimitive& g = gaussians[flat_index / stride];
    const int slot = static_cast<int>(flat_index % stride);
    if (slot < 3)
        g.position[slot] = value;
    else if (slot < 7)
        g.rotation[slot - 3] = value;
    else if (slot < 10)
        g.log_scale[slot - 7] = value;
    else if (slot == 10)
        g.opacity_logit = value;
    else
        set_color_param(g.color, slot - kGeometryParams, value);
}

// ---------------------------------------------------------------------------- camera / image

void Camera::validate() const {
    if (fx <= 0 || fy <= 0) throw InvalidArgument("camera focal lengths must be positive");
    if (width < 1 || height < 1) throw InvalidArgument("camera image size must be >= 1");
}

Camera make_orbit_camera(const Vec3& target, double distance, double angle, double elevation, int width,
                         int height, double focal) {
    const double t[3] = {target[0], target[1], target[2]};
    sgs_camera c{};
    const int st = sgs_orbit_camera(t, distance, angle, elevation, width, height, focal, &c);
    Camera cam;
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) cam.rotation(r, k) = c.R[r * 3 + k];
    cam.translation = Vec3(c.t[0], c.t[1], c.t[2]);
    cam.fx = c.fx;
    cam.fy = c.fy;
    cam.cx = c.cx;
    cam.cy = c.cy;
    cam.width = c.width;
    cam.height = c.height;
    cam.near = c.near_plane;
    if (st != SGS_OK) cam.validate();  // throws the reference's message
    return cam;
}

Image Image::clamped01() const {
    Image out = *this;
    for (double& v : out.data) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    return out;
}

// ---------------------------------------------------------------------------- colour

SHCoeffs SHCoeffs::zeros(int degree) {
    if (degree < 0 || degree > 3) {
        std::ostringstream m;
        m << "unsupported SH degree " << degree << " (max 3)";
        throw InvalidArgument(m.str());
    }
    SHCoeffs c;
    c.degree = degree;
    c.coeffs.assign(static_cast<std::size_t>(sh::coeff_count(degree)), Vec3::Zero());
    return c;
}

void validate_ortho_axes(const Mat3& axes, double tol) {
    const double err = (axes * axes.transpose() - Mat3::Identity()).cwiseAbs().maxCoeff();
    if (err > tol) {
        std::ostringstream m;
        m << "axis triple is not orthonormal: |A A^T - I|_max = " << err;
        throw InvalidArgument(m.str());
    }
}

OrthoSGSet::OrthoSGSet(const std::array<SGLobe, 3>& l, const Mat3& a) : lobes(l), axes(a) {
    validate_ortho_axes(axes);
    for (int i = 0; i < 3; ++i) lobes[static_cast<std::size_t>(i)].mu = axes.row(i).transpose();
}

SGLobe DiffuseSGModel::lobe() const {
    SGLobe l;
    l.alpha = alpha;
    l.lambda = std::exp(log_lambda);
    const double n = mu.norm();
    l.mu = n > 1e-12 ? Vec3(mu / n) : Vec3::UnitX();
    return l;
}

SGLobe DiffuseOrthoSGModel::lobe(int i, const Mat3& axes) const {
    return SGLobe{alpha[static_cast<std::size_t>(i)], std::exp(log_lambda[static_cast<std::size_t>(i)]),
                  axes.row(i).transpose()};
}

SGLobe MixedSHSGModel::lobe(int i, const Mat3& axes) const {
    return SGLobe{alpha[static_cast<std::size_t>(i)], std::exp(log_lambda[static_cast<std::size_t>(i)]),
                  axes.row(i).transpose()};
}

ColorModelKind kind_of(const ColorModel& m) { return static_cast<ColorModelKind>(m.index()); }

const char* to_string(ColorModelKind k) {
    static const char* names[] = {"sh", "sg1", "sg3", "mixed"};
    return names[static_cast<int>(k)];
}

ColorModelKind color_model_kind_from_string(const std::string& name) {
    for (int k = 0; k < 4; ++k)
        if (name == to_string(static_cast<ColorModelKind>(k))) return static_cast<ColorModelKind>(k);
    throw InvalidArgument("unknown color model kind: " + name);
}

namespace {
void require_unit(const Vec3& d) {
    if (std::abs(d.norm() - 1.0) > 1e-6) {
        std::ostringstream m;
        m << "direction must be unit length, got |d| = " << d.norm();
        throw InvalidArgument(m.str());
    }
}
}  // namespace

std::vector<double> eval_sh_basis(const Vec3& d, int degree) {
    require_unit(d);
    (void)SHCoeffs::zeros(degree);  // degree check
    const double x = d.x(), y = d.y(), z = d.z();
    std::vector<double> b(static_cast<std::size_t>(sh::coeff_count(degree)));
    b[0] = sh::kC0;
    if (degree >= 1) {
        b[1] = -sh::kC1 * y;
        b[2] = sh::kC1 * z;
        b[3] = -sh::kC1 * x;
    }
    const double xx = x * x, yy = y * y, zz = z * z;
    if (degree >= 2) {
        b[4] = sh::kC2[0] * x * y;
        b[5] = sh::kC2[1] * y * z;
        b[6] = sh::kC2[2] * (2.0 * zz - xx - yy);
        b[7] = sh::kC2[3] * x * z;
        b[8] = sh::kC2[4] * (xx - yy);
    }
    if (degree >= 3) {
        b[9] = sh::kC3[0] * y * (3.0 * xx - yy);
        b[10] = sh::kC3[1] * x * y * z;
        b[11] = sh::kC3[2] * y * (4.0 * zz - xx - yy);
        b[12] = sh::kC3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
        b[13] = sh::kC3[4] * x * (4.0 * zz - xx - yy);
        b[14] = sh::kC3[5] * z * (xx - yy);
        b[15] = sh::kC3[6] * x * (xx - 3.0 * yy);
    }
    return b;
}

Vec3 eval_sg(const SGLobe& lobe, const Vec3& d) {
    require_unit(d);
    return lobe.alpha * std::exp(lobe.lambda * (d.dot(lobe.mu) - 1.0));
}

namespace {
Vec3 sh_part(const SHCoeffs& c, const Vec3& d, int deg) {
    const auto b = eval_sh_basis(d, deg);
    Vec3 acc = Vec3::Zero();
    for (int i = 0; i < sh::coeff_count(deg); ++i) acc += b[static_cast<std::size_t>(i)] * c.coeffs[static_cast<std::size_t>(i)];
    return acc;
}
Vec3 lobes_part(const std::array<Vec3, 3>& alpha, const std::array<double, 3>& ll, const Mat3& axes, const Vec3& d) {
    Vec3 acc = Vec3::Zero();
    for (int i = 0; i < 3; ++i) {
        const double lambda = std::exp(ll[static_cast<std::size_t>(i)]);
        acc += alpha[static_cast<std::size_t>(i)] * std::exp(lambda * (axes.row(i).dot(d) - 1.0));
    }
    return acc;
}
}  // namespace

Vec3 eval_color(const ColorModel& model, const Mat3& axes, const Vec3& d, std::optional<int> ov) {
    require_unit(d);
    if (ov && kind_of(model) != ColorModelKind::MixedSHSG)
        throw InvalidArgument("sh_degree_override is only valid for the mixed SH+SG model");
    Vec3 pre = Vec3::Zero();
    if (auto* m = std::get_if<SHOnlyModel>(&model)) {
        pre = Vec3::Constant(0.5) + sh_part(m->sh, d, m->sh.degree);
    } else if (auto* m1 = std::get_if<DiffuseSGModel>(&model)) {
        pre = m1->diffuse + eval_sg(m1->lobe(), d);
    } else if (auto* m3 = std::get_if<DiffuseOrthoSGModel>(&model)) {
        pre = m3->diffuse + lobes_part(m3->alpha, m3->log_lambda, axes, d);
    } else {
        const auto& mx = std::get<MixedSHSGModel>(model);
        int deg = mx.sh.degree;
        if (ov) {
            if (*ov < 0 || *ov > mx.sh.degree) {
                std::ostringstream m;
                m << "sh degree override " << *ov << " exceeds stored degree " << mx.sh.degree;
                throw InvalidArgument(m.str());
            }
            deg = *ov;
        }
        pre = Vec3::Constant(0.5) + sh_part(mx.sh, d, deg) + lobes_part(mx.alpha, mx.log_lambda, axes, d);
    }
    return pre.cwiseMax(0.0);
}

Vec3 eval_color(const ColorModel& model, const Vec3& d, std::optional<int> ov) {
    return eval_color(model, Mat3::Identity(), d, ov);
}

int param_count(ColorModelKind kind, int deg) { return sgs_color_param_count(static_cast<int32_t>(kind), deg); }

int param_count(const ColorModel& m) { return param_count(kind_of(m), stored_degree(m)); }

int shared_param_count(ColorModelKind kind) {
    return kind == ColorModelKind::DiffuseOrthoSG || kind == ColorModelKind::MixedSHSG ? 3 : 0;
}

namespace {
// canonical order of color.hpp:121-128 (same as sgs.h)
double* param_slot(ColorModel& model, int i) {
    if (i < 0 || i >= param_count(model)) throw InvalidArgument("color parameter index out of range");
    if (auto* m = std::get_if<SHOnlyModel>(&model)) return &m->sh.coeffs[static_cast<std::size_t>(i / 3)][i % 3];
    if (auto* m1 = std::get_if<DiffuseSGModel>(&model)) {
        if (i < 3) return &m1->diffuse[i];
        if (i < 6) return &m1->alpha[i - 3];
        if (i == 6) return &m1->log_lambda;
        return &m1->mu[i - 7];
    }
    if (auto* m3 = std::get_if<DiffuseOrthoSGModel>(&model)) {
        if (i < 3) return &m3->diffuse[i];
        const int l = (i - 3) / 4, s = (i - 3) % 4;
        return s < 3 ? &m3->alpha[static_cast<std::size_t>(l)][s] : &m3->log_lambda[static_cast<std::size_t>(l)];
    }
    auto& mx = std::get<MixedSHSGModel>(model);
    const int nsh = 3 * sh::coeff_count(mx.sh.degree);
    if (i < nsh) return &mx.sh.coeffs[static_cast<std::size_t>(i / 3)][i % 3];
    const int l = (i - nsh) / 4, s = (i - nsh) % 4;
    return s < 3 ? &mx.alpha[static_cast<std::size_t>(l)][s] : &mx.log_lambda[static_cast<std::size_t>(l)];
}
}  // namespace

double color_param(const ColorModel& model, int index) {
    return *param_slot(const_cast<ColorModel&>(model), index);
}

void set_color_param(ColorModel& model, int index, double value) { *param_slot(model, index) = value; }

// ---------------------------------------------------------------------------- synth

namespace {
double f32(double v) {
    volatile float f = static_cast<float>(v);
    return static_cast<double>(f);
}
Vec3 f32(const Vec3& v) { return Vec3(f32(v[0]), f32(v[1]), f32(v[2])); }
// Vec3(f(), f(), f()) with g++'s right-to-left argument evaluation
template <typename F>
Vec3 draw3(F&& f) {
    const double c = f(), b = f(), a = f();
    return Vec3(a, b, c);
}
int band_of(int k) { return k == 0 ? 0 : (k < 4 ? 1 : (k < 9 ? 2 : 3)); }
}  // namespace

Scene make_synthetic_scene(std::size_t count, std::uint64_t seed, const SynthOptions& o) {
    std::mt19937_64 gen(seed);
    Scene scene;
    scene.gaussians.reserve(count);
    auto ur = [&](double lo, double hi) { return uniform_range(gen, lo, hi); };
    for (std::size_t i = 0; i < count; ++i) {
        GaussianPrimitive g;
        const Vec3 dir = random_unit_vector(gen);
        const double s = o.cluster_radius * std::cbrt(uniform01(gen));
        g.position = f32(Vec3(s * dir));
        const Vec4 q = random_unit_quaternion(gen);
        g.rotation = Vec4(f32(q[0]), f32(q[1]), f32(q[2]), f32(q[3]));
        g.log_scale = f32(draw3([&] { return ur(o.log_scale_min, o.log_scale_max); }));
        g.opacity_logit = f32(logit(ur(o.opacity_min, o.opacity_max)));
        const Vec3 base = draw3([&] { return ur(o.base_color_min, o.base_color_max); });
        auto sh_coeffs = [&](int degree) {
            SHCoeffs c = SHCoeffs::zeros(degree);
            c.coeffs[0] = f32(Vec3((base - Vec3::Constant(0.5)) / sh::kC0));
            for (int k = 1; k < sh::coeff_count(degree); ++k) {
                const double amp = o.band_amplitude * std::pow(o.band_decay, band_of(k));
                c.coeffs[static_cast<std::size_t>(k)] = f32(draw3([&] { return ur(-amp, amp); }));
            }
            return c;
        };
        auto lobe_set = [&](std::array<Vec3, 3>& alpha, std::array<double, 3>& ll) {
            for (int l = 0; l < 3; ++l) {
                const double amp = o.sg_alpha_amplitude;
                alpha[static_cast<std::size_t>(l)] = f32(draw3([&] { return ur(-amp, amp); }));
                ll[static_cast<std::size_t>(l)] = f32(ur(-0.5, 1.5));
            }
        };
        switch (o.kind) {
            case ColorModelKind::SHOnly:
                g.color = SHOnlyModel{sh_coeffs(o.sh_degree)};
                break;
            case ColorModelKind::DiffuseSG: {
                DiffuseSGModel m;
                m.diffuse = f32(base);
                const double amp = o.sg_alpha_amplitude;
                m.alpha = f32(draw3([&] { return ur(-amp, amp); }));
                m.log_lambda = f32(ur(-0.5, 1.5));
                m.mu = f32(random_unit_vector(gen));
                g.color = std::move(m);
                break;
            }
            case ColorModelKind::DiffuseOrthoSG: {
                DiffuseOrthoSGModel m;
                m.diffuse = f32(base);
                lobe_set(m.alpha, m.log_lambda);
                g.color = std::move(m);
                break;
            }
            case ColorModelKind::MixedSHSG: {
                MixedSHSGModel m;
                m.sh = sh_coeffs(2);
                lobe_set(m.alpha, m.log_lambda);
                g.color = std::move(m);
                break;
            }
        }
        scene.gaussians.push_back(std::move(g));
    }
    return scene;
}

std::vector<Camera> make_orbit_cameras(int count, int width, int height, double distance, double focal,
                                       double elevation) {
    std::vector<Camera> cams;
    cams.reserve(static_cast<std::size_t>(count));
    for (int i = 0; i < count; ++i)
        cams.push_back(make_orbit_camera(Vec3::Zero(), distance, 2.0 * M_PI * i / count, elevation, width, height,
                                         focal));
    return cams;
}

// ---------------------------------------------------------------------------
// PLY checkpoints (ply.hpp): the C-ABI reader fills the flat parameters, which go
// into the Scene through Scene::set_param.
int ply_floats_per_gaussian(PlyLayout layout, ColorModelKind kind) {
    if (layout == PlyLayout::Reference3DGS) return 59;
    return kind == ColorModelKind::MixedSHSG ? 53 : 29;
}

PlyLayout detect_layout(const Scene& scene) {
    if (scene.gaussians.empty()) return PlyLayout::Reference3DGS;
    return kind_of(scene.gaussians.front().color) == ColorModelKind::SHOnly ? PlyLayout::Reference3DGS
                                                                            : PlyLayout::SGExtended;
}

Scene load_ply(const std::string& path) {
    sgs_ply_info info{};
    check(sgs_ply_read(path.c_str(), &info, nullptr, 0));
    const std::size_t stride = 11 + static_cast<std::size_t>(sgs_color_param_count(info.kind, info.sh_degree));
    std::vector<double> flat(static_cast<std::size_t>(info.count) * stride);
    check(sgs_ply_read(path.c_str(), &info, flat.empty() ? nullptr : flat.data(), flat.size()));
    Scene scene;
    scene.gaussians.resize(static_cast<std::size_t>(info.count));
    for (auto& g : scene.gaussians) {
        switch (static_cast<ColorModelKind>(info.kind)) {
            case ColorModelKind::SHOnly: g.color = SHOnlyModel{SHCoeffs::zeros(info.sh_degree)}; break;
            case ColorModelKind::DiffuseSG: g.color = DiffuseSGModel{}; break;
            case ColorModelKind::DiffuseOrthoSG: g.color = DiffuseOrthoSGModel{}; break;
            default: {
                MixedSHSGModel m;
                m.sh = SHCoeffs::zeros(info.sh_degree);
                g.color = std::move(m);
            }
        }
    }
    for (std::size_t i = 0; i < flat.size(); ++i) scene.set_param(i, flat[i]);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) scene.shared_axes(r, c) = info.shared_axes[3 * r + c];
    scene.background = Vec3(info.background[0], info.background[1], info.background[2]);
    return scene;
}

// ---------------------------------------------------------------------------
// backward (grad.hpp) and metrics (metrics.hpp) through the C-ABI.
namespace {
std::vector<double> flat_params(const Scene& scene) {
    std::vector<double> flat(scene.total_params());
    for (std::size_t i = 0; i < flat.size(); ++i) flat[i] = scene.param(i);
    return flat;
}

sgs_scene* upload_scene(const Scene& scene, std::vector<double>& flat) {
    scene.check_homogeneous();
    flat = flat_params(scene);
    sgs_scene_desc d{};
    d.count = scene.gaussians.size();
    if (d.count) {
        d.kind = static_cast<int32_t>(kind_of(scene.gaussians.front().color));
        d.sh_degree = stored_degree(scene.gaussians.front().color);
    }
    d.dtype = SGS_F64;
    d.params = flat.empty() ? nullptr : flat.data();
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) d.shared_axes[3 * r + c] = scene.shared_axes(r, c);
    for (int k = 0; k < 3; ++k) d.background[k] = scene.background[k];
    sgs_scene* s = nullptr;
    check(sgs_scene_upload(context(), &d, &s));
    return s;
}

void check_image_shapes(const Image& a, const Image& b) {
    if (!a.same_shape(b)) throw InvalidArgument("image dimensions do not match");
}
}  // namespace

double SceneGradients::flat(const Scene& scene, std::size_t flat_index) const {
    const std::size_t stride = scene.params_per_gaussian();
    if (stride == 0 || flat_index >= scene.total_params()) throw InvalidArgument("gradient index out of range");
    const GaussianGrad& g = gaussians[flat_index / stride];
    const int slot = static_cast<int>(flat_index % stride);
    if (slot < 3) return g.position[slot];
    if (slot < 7) return g.rotation[slot - 3];
    if (slot < 10) return g.log_scale[slot - 7];
    if (slot == 10) return g.opacity_logit;
    return g.color[static_cast<std::size_t>(slot - 11)];
}

void SceneGradients::add_scaled(const SceneGradients& other, double scale) {
    for (std::size_t i = 0; i < gaussians.size(); ++i) {
        gaussians[i].position += scale * other.gaussians[i].position;
        gaussians[i].rotation += scale * other.gaussians[i].rotation;
        gaussians[i].log_scale += scale * other.gaussians[i].log_scale;
        gaussians[i].opacity_logit += scale * other.gaussians[i].opacity_logit;
        for (std::size_t k = 0; k < gaussians[i].color.size(); ++k)
            gaussians[i].color[k] += scale * other.gaussians[i].color[k];
    }
}

SceneGradients backward(const Scene& scene, const Camera& cam, const RenderConfig& cfg, const Image& upstream) {
    if (upstream.width != cam.width || upstream.height != cam.height || upstream.channels != 3)
        throw InvalidArgument("upstream image dimensions do not match the render output");
    SceneGradients grads;
    grads.gaussians.resize(scene.gaussians.size());
    for (std::size_t i = 0; i < scene.gaussians.size(); ++i)
        grads.gaussians[i].color.assign(static_cast<std::size_t>(param_count(scene.gaussians[i].color)), 0.0);
    std::vector<double> flat;
    sgs_scene* s = upload_scene(scene, flat);
    std::vector<double> g(flat.size());
    const sgs_camera c = to_c(cam);
    const sgs_render_config k = to_c(cfg);
    const int st = sgs_backward(context(), s, &c, &k, upstream.data.data(), SGS_HOST, g.empty() ? nullptr : g.data());
    sgs_scene_free(s);
    check(st);
    const std::size_t stride = scene.params_per_gaussian();
    for (std::size_t i = 0; i < scene.gaussians.size(); ++i) {
        GaussianGrad& o = grads.gaussians[i];
        const double* p = g.data() + i * stride;
        o.position = Vec3(p[0], p[1], p[2]);
        o.rotation = Vec4(p[3], p[4], p[5], p[6]);
        o.log_scale = Vec3(p[7], p[8], p[9]);
        o.opacity_logit = p[10];
        for (std::size_t k2 = 0; k2 < o.color.size(); ++k2) o.color[k2] = p[11 + k2];
    }
    return grads;
}

double fd_gradient(const Scene& scene, const Camera& cam, const RenderConfig& cfg, const Image& upstream,
                   std::size_t param_index, double h) {
    if (h <= 0.0) throw InvalidArgument("finite-difference step must be positive");
    auto objective = [&](const Scene& s) {
        RenderResult r = render(s, cam, cfg);
        double total = 0.0;
        for (std::size_t i = 0; i < r.image.size(); ++i) total += r.image.data[i] * upstream.data[i];
        return total;
    };
    Scene probe = scene;
    const double original = probe.param(param_index);
    probe.set_param(param_index, original + h);
    const double hi = objective(probe);
    probe.set_param(param_index, original - h);
    const double lo = objective(probe);
    return (hi - lo) / (2.0 * h);
}

double psnr(const Image& a, const Image& b) {
    check_image_shapes(a, b);
    double out = 0.0;
    check(sgs_psnr(context(), a.data.data(), b.data.data(), a.width, a.height, a.channels, SGS_F64, SGS_HOST, &out));
    return out;
}

double ssim(const Image& a, const Image& b) {
    check_image_shapes(a, b);
    double out = 0.0;
    check(sgs_ssim(context(), a.data.data(), b.data.data(), a.width, a.height, a.channels, SGS_F64, SGS_HOST, &out,
                   nullptr));
    return out;
}

SsimResult ssim_with_grad(const Image& a, const Image& b) {
    check_image_shapes(a, b);
    SsimResult r;
    r.grad_a = Image(a.width, a.height, a.channels);
    check(sgs_ssim(context(), a.data.data(), b.data.data(), a.width, a.height, a.channels, SGS_F64, SGS_HOST,
                   &r.value, r.grad_a.data.data()));
    return r;
}

}  // namespace sgsplat
