// ref_harness.cpp -- C harness around the REFERENCE's own render path
// (TEST INFRASTRUCTURE ONLY; see oracle/oracle.h).
//
// Links the reference translation units compiled in place from
// /root/reference/proj/src/{color,scene,camera,raster,synth}.cpp against the
// Eigen subset in third_party/eigen_subset. Nothing here re-implements the
// algorithm: every number comes from sgsplat::render / detail::project_scene /
// detail::build_tile_grid / testing::render_bruteforce themselves.
#include "oracle.h"

#include "sgsplat/grad.hpp"
#include "sgsplat/metrics.hpp"
#include "sgsplat/ply.hpp"
#include "sgsplat/raster.hpp"
#include "sgsplat/synth.hpp"
#include "support/bruteforce.hpp"

#include <cstring>
#include <exception>
#include <string>

using namespace sgsplat;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

#define REF_GUARD(body)                                                    \
    try {                                                                  \
        body                                                               \
    } catch (const InvalidArgument& e) {                                   \
        return fail(e, ORC_INVALID_ARGUMENT);                              \
    } catch (const NumericError& e) {                                      \
        return fail(e, ORC_NUMERIC);                                       \
    } catch (const IoError& e) {                                           \
        return fail(e, ORC_IO);                                            \
    } catch (const FormatError& e) {                                       \
        return fail(e, ORC_FORMAT);                                        \
    } catch (const std::exception& e) {                                    \
        return fail(e, ORC_INTERNAL);                                      \
    }

Camera to_cam(const orc_camera* c) {
    Camera cam;
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) cam.rotation(r, k) = c->R[r * 3 + k];
    cam.translation = Vec3(c->t[0], c->t[1], c->t[2]);
    cam.fx = c->fx;
    cam.fy = c->fy;
    cam.cx = c->cx;
    cam.cy = c->cy;
    cam.width = c->width;
    cam.height = c->height;
    cam.near = c->near_plane;
    return cam;
}

void from_cam(const Camera& cam, orc_camera* c) {
    for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) c->R[r * 3 + k] = cam.rotation(r, k);
    for (int r = 0; r < 3; ++r) c->t[r] = cam.translation[r];
    c->fx = cam.fx;
    c->fy = cam.fy;
    c->cx = cam.cx;
    c->cy = cam.cy;
    c->width = cam.width;
    c->height = cam.height;
    c->near_plane = cam.near;
}

RenderConfig to_cfg(const orc_config* k) {
    RenderConfig cfg;
    cfg.tile_size = k->tile_size;
    cfg.degree_threshold_lo = k->degree_threshold_lo;
    cfg.degree_threshold_hi = k->degree_threshold_hi;
    if (k->has_override) cfg.sh_degree_override = k->override_degree;
    cfg.early_stop_transmittance = k->early_stop_transmittance;
    cfg.threads = k->threads;
    return cfg;
}

int color_params(int kind, int degree) {
    return param_count(static_cast<ColorModelKind>(kind), degree);
}

ColorModel make_model(int kind, int degree) {
    switch (kind) {
        case ORC_SH: return SHOnlyModel{SHCoeffs::zeros(degree)};
        case ORC_SG1: return DiffuseSGModel{};
        case ORC_SG3: return DiffuseOrthoSGModel{};
        default: {
            MixedSHSGModel m;
            m.sh = SHCoeffs::zeros(degree);
            return m;
        }
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_scene_synth(size_t count, uint64_t seed, int kind, int sh_degree, double ls_min,
                      double ls_max) {
    SynthOptions opts;
    opts.kind = static_cast<ColorModelKind>(kind);
    opts.sh_degree = sh_degree;
    opts.log_scale_min = ls_min;
    opts.log_scale_max = ls_max;
    return new Scene(make_synthetic_scene(count, seed, opts));
}

// Builds a Scene from the flat layout through the reference's own parameter
// setters (Scene::set_param, proj/src/scene.cpp:129-137).
void* ref_scene_from_params(size_t count, int kind, int sh_degree, const double* params,
                            const double* axes_rowmajor, const double* background) {
    auto* s = new Scene();
    s->gaussians.resize(count);
    for (auto& g : s->gaussians) g.color = make_model(kind, sh_degree);
    std::size_t stride = s->params_per_gaussian();
    for (std::size_t i = 0; i < count * stride; ++i) s->set_param(i, params[i]);
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) s->shared_axes(r, c) = axes_rowmajor[r * 3 + c];
    s->background = Vec3(background[0], background[1], background[2]);
    return s;
}

void ref_scene_free(void* s) { delete static_cast<Scene*>(s); }

size_t ref_scene_count(void* s) { return static_cast<Scene*>(s)->gaussians.size(); }

size_t ref_scene_stride(void* s) { return static_cast<Scene*>(s)->params_per_gaussian(); }

void ref_scene_params(void* s, double* out) {
    const Scene& sc = *static_cast<Scene*>(s);
    std::size_t n = sc.total_params();
    for (std::size_t i = 0; i < n; ++i) out[i] = sc.param(i);
}

void ref_scene_set_background(void* s, const double* bg) {
    static_cast<Scene*>(s)->background = Vec3(bg[0], bg[1], bg[2]);
}

int ref_color_param_count(int kind, int degree) { return color_params(kind, degree); }

int ref_flops_per_gaussian(int kind, int degree) {
    REF_GUARD(return flops_per_gaussian(static_cast<ColorModelKind>(kind), degree);)
}

int ref_select_degree(double r, double lo, double hi, int* out) {
    REF_GUARD(*out = select_degree(r, lo, hi); return ORC_OK;)
}

void ref_orbit_camera(const double* target, double distance, double angle, double elevation,
                      int width, int height, double focal, orc_camera* out) {
    from_cam(make_orbit_camera(Vec3(target[0], target[1], target[2]), distance, angle, elevation,
                               width, height, focal),
             out);
}

void ref_orbit_cameras(int count, int width, int height, double distance, double focal,
                       double elevation, orc_camera* out) {
    auto cams = make_orbit_cameras(count, width, height, distance, focal, elevation);
    for (int i = 0; i < count; ++i) from_cam(cams[static_cast<std::size_t>(i)], &out[i]);
}

// sgsplat::render (proj/src/raster.cpp:141-188). rgb: H*W*3, T: H*W (either may be null).
int ref_render(void* s, const orc_camera* cam, const orc_config* cfg, double* rgb, double* T) {
    REF_GUARD({
        RenderResult r = render(*static_cast<Scene*>(s), to_cam(cam), to_cfg(cfg));
        if (rgb) std::memcpy(rgb, r.image.data.data(), r.image.data.size() * sizeof(double));
        if (T)
            std::memcpy(T, r.transmittance.data.data(),
                        r.transmittance.data.size() * sizeof(double));
        return ORC_OK;
    })
}

// testing::render_bruteforce (proj/tests/support/bruteforce.hpp:14-57).
int ref_render_bruteforce(void* s, const orc_camera* cam, const orc_config* cfg, double* rgb,
                          double* T) {
    REF_GUARD({
        RenderResult r =
            testing::render_bruteforce(*static_cast<Scene*>(s), to_cam(cam), to_cfg(cfg));
        if (rgb) std::memcpy(rgb, r.image.data.data(), r.image.data.size() * sizeof(double));
        if (T)
            std::memcpy(T, r.transmittance.data.data(),
                        r.transmittance.data.size() * sizeof(double));
        return ORC_OK;
    })
}

// Per-Gaussian detail::project_cached (proj/src/raster.cpp:17-80), serial.
int ref_project_each(void* s, const orc_camera* c, const orc_config* k, orc_splat* out) {
    REF_GUARD({
        const Scene& sc = *static_cast<Scene*>(s);
        Camera cam = to_cam(c);
        RenderConfig cfg = to_cfg(k);
        for (std::size_t i = 0; i < sc.gaussians.size(); ++i) {
            auto pc = detail::project_cached(sc.gaussians[i], cam, sc.shared_axes, cfg, i);
            orc_splat& o = out[i];
            std::memset(&o, 0, sizeof(o));
            o.visible = pc ? 1 : 0;
            o.degree = -1;
            if (!pc) continue;
            const Splat2D& sp = pc->splat;
            o.mean2d[0] = sp.mean2d.x();
            o.mean2d[1] = sp.mean2d.y();
            for (int j = 0; j < 3; ++j) o.conic[j] = sp.conic[j];
            o.depth = sp.depth;
            for (int j = 0; j < 3; ++j) o.color[j] = sp.color[j];
            o.opacity = sp.opacity;
            o.radius = sp.radius_px;
            o.degree = pc->degree_used ? *pc->degree_used : -1;
        }
        return ORC_OK;
    })
}

// detail::project_scene + detail::build_tile_grid (proj/src/raster.cpp:82-130).
// order[rank] = gaussian index (capacity N); offsets: tiles+1 prefix over the
// per-tile lists; entries: concatenated lists of ranks (capacity cap).
int ref_tile_grid(void* s, const orc_camera* c, const orc_config* k, uint32_t* order,
                  size_t* n_visible, uint64_t* offsets, uint32_t* entries, size_t cap,
                  size_t* n_entries) {
    REF_GUARD({
        if (k->tile_size < 1) throw InvalidArgument("tile_size must be >= 1");
        const Scene& sc = *static_cast<Scene*>(s);
        Camera cam = to_cam(c);
        auto sorted = detail::project_scene(sc, cam, to_cfg(k));
        auto grid = detail::build_tile_grid(sorted, cam.width, cam.height, k->tile_size);
        *n_visible = sorted.size();
        if (order)
            for (std::size_t r = 0; r < sorted.size(); ++r)
                order[r] = static_cast<uint32_t>(sorted[r].gaussian_index);
        std::size_t total = 0;
        for (std::size_t t = 0; t < grid.lists.size(); ++t) {
            if (offsets) offsets[t] = total;
            for (uint32_t si : grid.lists[t]) {
                if (entries && total < cap) entries[total] = si;
                ++total;
            }
        }
        if (offsets) offsets[grid.lists.size()] = total;
        *n_entries = total;
        return ORC_OK;
    })
}

// eval_color (proj/src/color.cpp:201-235) on one flat colour record.
int ref_eval_color(int kind, int degree, const double* cparams, const double* axes_rowmajor,
                   const double* dir, int has_override, int override_degree, double* out) {
    REF_GUARD({
        ColorModel model = make_model(kind, degree);
        int n = color_params(kind, degree);
        for (int i = 0; i < n; ++i) set_color_param(model, i, cparams[i]);
        Mat3 axes;
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) axes(r, c) = axes_rowmajor[r * 3 + c];
        std::optional<int> ov;
        if (has_override) ov = override_degree;
        Vec3 col = eval_color(model, axes, Vec3(dir[0], dir[1], dir[2]), ov);
        for (int c = 0; c < 3; ++c) out[c] = col[c];
        return ORC_OK;
    })
}

// sgsplat::load_ply (proj/src/ply.cpp:295-306). *out receives a Scene handle.
int ref_load_ply(const char* path, void** out) {
    REF_GUARD({
        *out = new Scene(load_ply(path));
        return ORC_OK;
    })
}

// sgsplat::save_ply (proj/src/ply.cpp:308-380); layout 0 = Reference3DGS, 1 = SGExtended.
int ref_save_ply(void* s, const char* path, int layout) {
    REF_GUARD({
        save_ply(*static_cast<Scene*>(s), path,
                 layout == 0 ? PlyLayout::Reference3DGS : PlyLayout::SGExtended);
        return ORC_OK;
    })
}

// Colour model kind, stored SH degree (0 for SG-only), axes and background of a scene.
void ref_scene_info(void* s, int* kind, int* degree, double* axes, double* bg) {
    const Scene& sc = *static_cast<Scene*>(s);
    *kind = sc.gaussians.empty() ? -1 : static_cast<int>(kind_of(sc.gaussians.front().color));
    *degree = 0;
    if (!sc.gaussians.empty()) {
        if (auto* m = std::get_if<SHOnlyModel>(&sc.gaussians.front().color)) *degree = m->sh.degree;
        if (auto* m = std::get_if<MixedSHSGModel>(&sc.gaussians.front().color)) *degree = m->sh.degree;
    }
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) axes[3 * r + c] = sc.shared_axes(r, c);
    for (int k = 0; k < 3; ++k) bg[k] = sc.background[k];
}

namespace {
Image image_of(const double* p, int w, int h, int c) {
    Image img(w, h, c);
    std::memcpy(img.data.data(), p, img.size() * sizeof(double));
    return img;
}
}  // namespace

// sgsplat::psnr (proj/src/metrics.cpp:110-121); images H x W x C row-major.
int ref_psnr(const double* a, const double* b, int w, int h, int c, double* out) {
    REF_GUARD({
        *out = psnr(image_of(a, w, h, c), image_of(b, w, h, c));
        return ORC_OK;
    })
}

// sgsplat::ssim / ssim_with_grad (metrics.cpp:125-176); grad may be null.
int ref_ssim(const double* a, const double* b, int w, int h, int c, double* out, double* grad) {
    REF_GUARD({
        if (grad) {
            SsimResult r = ssim_with_grad(image_of(a, w, h, c), image_of(b, w, h, c));
            *out = r.value;
            std::memcpy(grad, r.grad_a.data.data(), r.grad_a.size() * sizeof(double));
        } else {
            *out = ssim(image_of(a, w, h, c), image_of(b, w, h, c));
        }
        return ORC_OK;
    })
}

// sgsplat::backward (proj/src/grad.cpp:69-246): upstream H x W x 3; grads in
// SceneGradients::flat order (count x params_per_gaussian).
int ref_backward(void* s, const orc_camera* cam, const orc_config* cfg, const double* upstream, double* grads) {
    REF_GUARD({
        const Scene& sc = *static_cast<Scene*>(s);
        Camera c = to_cam(cam);
        Image up(c.width, c.height, 3);
        std::memcpy(up.data.data(), upstream, up.size() * sizeof(double));
        SceneGradients g = backward(sc, c, to_cfg(cfg), up);
        for (std::size_t i = 0; i < sc.total_params(); ++i) grads[i] = g.flat(sc, i);
        return ORC_OK;
    })
}

}  // extern "C"
