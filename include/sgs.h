/*
 * sgs.h -- C-ABI of the B200-native SG-Splatting forward renderer.
 *
 * This is the drop-in boundary for the reference's render path. Every entry point
 * takes plain pointers, sizes and POD structs (no C++, no torch types) so the
 * reference's FFI surfaces can bind it directly:
 *
 *   reference interface                                  replaced by
 *   -------------------------------------------------    ------------------------------
 *   sgsplat::render            raster.hpp:56, raster.cpp:141-188   sgs_render / sgs_render_batch
 *   sgsplat::project           raster.hpp:46-47, raster.cpp:134-139 sgs_project
 *   detail::project_scene/build_tile_grid raster.hpp:65-95       sgs_debug_tile_grid
 *   sgsplat::select_degree     raster.hpp:42, raster.cpp:8-13      sgs_select_degree
 *   sgsplat::flops_per_gaussian raster.hpp:62, raster.cpp:190-227  sgs_flops_per_gaussian
 *   sgsplat::param_count       color.hpp:139-140                   sgs_color_param_count
 *   make_synthetic_scene       synth.hpp:29, synth.cpp:26-106      sgs_synth_scene
 *   make_orbit_camera(s)       camera.hpp:34-35, synth.hpp:32-33   sgs_orbit_camera(s)
 *   sgsplat::backward          grad.hpp:32-33, grad.cpp:69-246     sgs_backward
 *   sgsplat::psnr / ssim / ssim_with_grad  metrics.hpp:7-21      sgs_psnr / sgs_ssim
 *   sgsplat::load_ply          ply.hpp:26-29, ply.cpp:295-306      sgs_ply_read (host) /
 *                                                                  sgs_scene_load_ply (device)
 *   python `_core.render`      bindings.cpp:109-121                sgs_render
 *
 * Error contract (proj/include/sgsplat/common.hpp:21-42): every call returns an
 * sgs_status; SGS_ERR_INVALID_ARGUMENT maps to sgsplat::InvalidArgument and
 * SGS_ERR_NUMERIC to sgsplat::NumericError, raised for exactly the inputs the
 * reference raises for (data-dependent cases come from a device error word that
 * keeps the lowest failing Gaussian index, i.e. the reference's serial order).
 * The message is available from sgs_last_error().
 *
 * Threading: contexts are independent; calls on one context are serialised by an
 * internal mutex and run on the context's CUDA stream. Output is bitwise
 * deterministic run to run (no float atomics; stable sorts).
 */
#ifndef SGS_H
#define SGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGS_ABI_VERSION 1

typedef enum {
    SGS_OK = 0,
    SGS_ERR_INVALID_ARGUMENT = 1, /* sgsplat::InvalidArgument */
    SGS_ERR_NUMERIC = 2,          /* sgsplat::NumericError */
    SGS_ERR_CUDA = 3,
    SGS_ERR_NCCL = 4,
    SGS_ERR_OUT_OF_MEMORY = 5,
    SGS_ERR_INTERNAL = 6,
    SGS_ERR_IO = 7,               /* sgsplat::IoError */
    SGS_ERR_FORMAT = 8            /* sgsplat::FormatError */
} sgs_status;

/* Colour model kinds, numbered as ColorModelKind (color.hpp:59). */
typedef enum { SGS_SH = 0, SGS_SG1 = 1, SGS_SG3 = 2, SGS_MIXED = 3 } sgs_color_kind;

typedef enum { SGS_F64 = 0, SGS_F32 = 1 } sgs_dtype;
typedef enum { SGS_HOST = 0, SGS_DEVICE = 1 } sgs_memory;

/* Pinhole camera (camera.hpp:11-23). R is the row-major world-to-camera rotation. */
typedef struct {
    double R[9];
    double t[3];
    double fx, fy, cx, cy;
    int32_t width, height;
    double near_plane;
} sgs_camera;

/* RenderConfig (raster.hpp:11-22). `threads` is accepted and ignored (the CUDA
 * grid replaces the reference's std::thread partition). */
typedef struct {
    int32_t tile_size;
    int32_t has_override;
    int32_t override_degree;
    int32_t threads;
    double degree_threshold_lo;
    double degree_threshold_hi;
    double early_stop_transmittance;
} sgs_render_config;

/* A scene in the reference's flat parameter layout (scene.hpp:40-43): per
 * Gaussian 11 geometry reals [px py pz, qw qx qy qz, lsx lsy lsz, opacity_logit]
 * followed by the colour parameters in the canonical order of color.hpp:121-128:
 *   SH     [coeff rgb x (d+1)^2]                    3(d+1)^2
 *   SG1    [diffuse rgb, alpha rgb, log_lambda, mu]  10
 *   SG3    [diffuse rgb, (alpha rgb, log_lambda)x3]  15
 *   MIXED  [coeff rgb x (d+1)^2, (alpha rgb, log_lambda)x3]  3(d+1)^2+12
 * `params` is count x stride values of `dtype` in host memory. */
typedef struct {
    uint64_t count;
    int32_t kind;
    int32_t sh_degree; /* stored SH degree (SH: 0..3, MIXED: 0..2; ignored for SG1/SG3) */
    int32_t dtype;     /* sgs_dtype of params */
    int32_t reserved;
    const void* params;
    double shared_axes[9]; /* row-major; rows are the shared lobe axes (scene.hpp:30) */
    double background[3];
} sgs_scene_desc;

/* Device layout of an uploaded scene. */
typedef struct {
    uint64_t count;
    int32_t kind;
    int32_t sh_degree;
    int32_t geometry_f64; /* 0: float32 planes (inputs were f32-exact), 1: float64 planes */
    int32_t color_f64;    /* 1: colour parameters not f32-exact: FP64 copies are kept too
                             (read by the exact mode and the backward) */
    uint64_t blob_bytes; /* bytes of the single device allocation holding every plane */
    double shared_axes[9];
    double background[3];
} sgs_scene_meta;

typedef struct sgs_context sgs_context;
typedef struct sgs_scene sgs_scene;

/* Per-render counters and (optionally) per-stage device times. */
typedef struct {
    uint64_t visible;       /* V: splats surviving the culls (raster.cpp:82-106) */
    uint64_t tile_entries;  /* P: (tile, splat) pairs, = sum of TileGrid list sizes */
    uint64_t block_entries; /* E_t: list entries composited before block termination */
    uint64_t guard_hits;    /* pairs recomputed in FP64 by the compositor's guard band */
    int32_t want_timing;    /* in: 1 to record per-stage CUDA-event times */
    int32_t timing_path;    /* in: 1 to run the stats-free render path (tight tile rectangles,
                               no E_t counting) so the stage times are those of a plain
                               render; block_entries stays 0 and tile_entries counts the
                               tight lists */
    float ms_preprocess, ms_depth_sort, ms_binning, ms_tile_sort, ms_composite, ms_total;
} sgs_render_stats;

/* --- context ------------------------------------------------------------------ */
int sgs_abi_version(void);
sgs_status sgs_create(int device, sgs_context** out);
void sgs_destroy(sgs_context* ctx);
/* Thread-local message of the last failing call on this thread. */
const char* sgs_last_error(void);
/* Run on a caller stream (cudaStream_t as void*); NULL restores the context's own. */
sgs_status sgs_set_stream(sgs_context* ctx, void* stream);
sgs_status sgs_synchronize(sgs_context* ctx);
/* Cumulative number of this library's own kernel launches on ctx (every stage K1-K7
 * is the library's own code) and of third-party library kernels (none: always 0),
 * for launch accounting. */
sgs_status sgs_launch_count(sgs_context* ctx, uint64_t* own_kernels, uint64_t* library_kernels);

/* Page-locked host memory (cudaHostAlloc) for callers that stage scenes or frames
 * through host buffers: transfers from / to it run at DMA speed. */
sgs_status sgs_host_alloc(uint64_t bytes, void** out);
void sgs_host_free(void* p);

/* --- scenes ------------------------------------------------------------------- */
/* Validates the desc (homogeneous by construction; scene.cpp:7-25 rules on degree)
 * and fills the device layout it will use. */
sgs_status sgs_scene_plan(const sgs_scene_desc* desc, sgs_scene_meta* meta);
/* Pack the scene into its device layout in HOST memory (meta->blob_bytes bytes):
 * exactly the bytes sgs_scene_upload places in HBM. Used to ship a scene blob
 * through a collective (e.g. NCCL / gloo broadcast) and to test layouts on CPU. */
sgs_status sgs_scene_pack(const sgs_scene_desc* desc, void* host_blob, uint64_t bytes);
/* Upload into a context-owned allocation. */
sgs_status sgs_scene_upload(sgs_context* ctx, const sgs_scene_desc* desc, sgs_scene** out);
/* Upload into caller device memory of meta->blob_bytes (e.g. a torch tensor that
 * NCCL later broadcasts). The scene does not own the memory. */
sgs_status sgs_scene_upload_into(sgs_context* ctx, const sgs_scene_desc* desc,
                                 void* device_blob, uint64_t bytes, sgs_scene** out);
/* Bind an already-populated blob (e.g. received by ncclBroadcast) without copying. */
sgs_status sgs_scene_bind(sgs_context* ctx, const sgs_scene_meta* meta, void* device_blob,
                          uint64_t bytes, sgs_scene** out);
/* The blob of a bound scene changed in place (e.g. a torch tensor the caller owns):
 * recompute what the library caches from it (the 3D covariances). Without this, later
 * renders would use the covariances of the old contents. */
sgs_status sgs_scene_refresh(sgs_context* ctx, sgs_scene* scene);
/* New parameters for an existing device scene with the same layout (count, model,
 * degree, float32/float64 planes): repacked into its blob, caches refreshed; plane
 * addresses do not change, so captured frame graphs stay valid. A different layout
 * is SGS_ERR_INVALID_ARGUMENT (upload a new scene). */
sgs_status sgs_scene_update(sgs_context* ctx, sgs_scene* scene, const sgs_scene_desc* desc);
/* sgs_scene_update with the float32 rows produced block by block, so packing them
 * overlaps their copy to the device: fill(user, rows, first, count) writes rows
 * [first, first + count) -- 11 + colour-parameter floats each, Scene::param order --
 * into a pinned staging block the library owns, which is copied while the caller fills
 * the next one. desc->dtype must be SGS_F32; desc->params is not read. A nonzero
 * return from fill ends the call with SGS_ERR_INVALID_ARGUMENT before the scene is
 * touched (it keeps its previous contents). fill runs on the calling thread while the
 * context is locked: it must not call into the library with this context. The C++
 * drop-in's render() feeds it from the caller's Scene. */
typedef int32_t (*sgs_row_fill_fn)(void* user, float* rows, uint64_t first, uint64_t count);
sgs_status sgs_scene_update_rows(sgs_context* ctx, sgs_scene* scene, const sgs_scene_desc* desc,
                                 sgs_row_fill_fn fill, void* user);
sgs_status sgs_scene_get_meta(const sgs_scene* scene, sgs_scene_meta* meta);
sgs_status sgs_scene_blob(const sgs_scene* scene, void** device_blob, uint64_t* bytes);
sgs_status sgs_scene_set_background(sgs_scene* scene, const double* rgb);
void sgs_scene_free(sgs_scene* scene);

/* --- render path --------------------------------------------------------------- */
/* One view. rgb: H*W*3 float32 row-major (Image layout, image.hpp:12-43); T: H*W
 * float32 transmittance (either may be NULL). out_memory says whether rgb/T are
 * host or device pointers; host outputs are complete when the call returns. */
sgs_status sgs_render(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                      const sgs_render_config* cfg, float* rgb, float* T, int32_t out_memory,
                      sgs_render_stats* stats);
/* n views of one scene; view i writes rgb + i*H*W*3 and T + i*H*W (all cameras must
 * share width/height). Host outputs are copied back on a second stream while the
 * next view renders. stats (optional) accumulates over the views. */
sgs_status sgs_render_batch(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cams,
                            int32_t n, const sgs_render_config* cfg, float* rgb, float* T,
                            int32_t out_memory, sgs_render_stats* stats);

/* Per-Gaussian projection (project_cached, raster.cpp:17-80) computed on the device
 * and copied to host. */
typedef struct {
    double mean2d[2];
    double conic[3];
    double depth;
    double color[3]; /* evaluated in float32, widened */
    double opacity;
    double radius;
    int32_t degree; /* -1 for non-mixed scenes */
    int32_t visible;
} sgs_splat;
sgs_status sgs_project(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                       const sgs_render_config* cfg, sgs_splat* out /* count */);
/* Depth order and TileGrid lists as the reference builds them (raster.cpp:82-130):
 * order[V] = Gaussian index per rank; offsets[tiles+1]; entries[P] = ranks.
 * Call with entries == NULL to query V and P first. */
sgs_status sgs_debug_tile_grid(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                               const sgs_render_config* cfg, uint32_t* order,
                               uint64_t* n_visible, uint64_t* offsets, uint32_t* entries,
                               uint64_t capacity, uint64_t* n_entries);

/* --- scalar helpers (host) ------------------------------------------------------ */
sgs_status sgs_select_degree(double radius_px, double lo, double hi, int32_t* out);
sgs_status sgs_flops_per_gaussian(int32_t kind, int32_t sh_degree, int32_t* out);
int32_t sgs_color_param_count(int32_t kind, int32_t sh_degree);

/* --- synthetic inputs (host) ---------------------------------------------------- */
/* make_synthetic_scene with SynthOptions defaults except kind / sh_degree /
 * log-scale range. params: count * (11 + colour params) doubles. */
sgs_status sgs_synth_scene(uint64_t count, uint64_t seed, int32_t kind, int32_t sh_degree,
                           double log_scale_min, double log_scale_max, double* params);
/* Same geometry, degree-3 SH colours (BASELINE config D): DC + bands 1-2 copied from
 * a MIXED scene, band 3 drawn from mt19937_64(seed + 1). */
sgs_status sgs_synth_sh3_from_mixed(uint64_t count, uint64_t seed, const double* mixed_params,
                                    double* sh3_params);
sgs_status sgs_orbit_camera(const double* target, double distance, double angle,
                            double elevation, int32_t width, int32_t height, double focal,
                            sgs_camera* out);
sgs_status sgs_orbit_cameras(int32_t count, int32_t width, int32_t height, double distance,
                             double focal, double elevation, sgs_camera* out);

/* --- exact mode ------------------------------------------------------------------ */
/* render in the reference's precision: the same culling, depth order and tile lists,
 * then the per-pixel loop (raster.cpp:155-186) in FP64 with the reference's operation
 * order (no FMA contraction). rgb: height x width x 3 doubles, T: height x width
 * (either may be NULL), in host or device memory. Slower than sgs_render; images
 * match the reference to FP64 rounding (CUDA vs glibc exp, <= 1 ulp). */
sgs_status sgs_render_f64(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                          const sgs_render_config* cfg, double* rgb, double* T, int32_t memory);

/* --- backward (grad.hpp, grad.cpp) ------------------------------------------------ */
/* backward (grad.cpp:69-246): d(sum_pixels upstream . rendered) / d(stored params).
 * upstream: height x width x 3 doubles; grads: count x (11 + colour params) doubles in
 * the flat order of Scene::param (SceneGradients::flat); both in host or device
 * memory (memory = SGS_HOST / SGS_DEVICE). Culled Gaussians get zero gradients. A
 * non-finite upstream value is SGS_ERR_NUMERIC ("non-finite upstream gradient"). FP64
 * throughout and deterministic; agrees with the reference to rounding. */
sgs_status sgs_backward(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                        const sgs_render_config* cfg, const double* upstream, int32_t memory,
                        double* grads);

/* --- image metrics (metrics.hpp, metrics.cpp) ------------------------------------ */
/* Images are height x width x channels, row-major (the reference's Image layout),
 * dtype SGS_F64 or SGS_F32 (widened to FP64 exactly), in host or device memory
 * (memory = SGS_HOST / SGS_DEVICE, for both inputs and grad_a). The per-pixel maps
 * are computed on the GPU in FP64 in the reference's operation order; the image
 * means are a fixed-order tree sum. An empty image is SGS_ERR_INVALID_ARGUMENT. */
/* psnr (metrics.cpp:110-121): 10 log10(1 / MSE), 100 dB when MSE < 1e-10. */
sgs_status sgs_psnr(sgs_context* ctx, const void* a, const void* b, int32_t width, int32_t height,
                    int32_t channels, int32_t dtype, int32_t memory, double* out);
/* ssim / ssim_with_grad (metrics.cpp:125-176): 11x11 Gaussian window (sigma 1.5),
 * reflect padding; grad_a (nullable) receives d(mean SSIM)/d(a). */
sgs_status sgs_ssim(sgs_context* ctx, const void* a, const void* b, int32_t width, int32_t height,
                    int32_t channels, int32_t dtype, int32_t memory, double* value, double* grad_a);

/* --- PLY checkpoints (ply.hpp, ply.cpp) ---------------------------------------- */
/* The two layouts of ply.hpp:9-22 (PlyLayout). */
typedef enum { SGS_PLY_REFERENCE3DGS = 0, SGS_PLY_SGEXTENDED = 1 } sgs_ply_layout;

typedef struct {
    uint64_t count;        /* vertices (Gaussians) */
    int32_t kind;          /* sgs_color_kind of the checkpoint */
    int32_t sh_degree;     /* stored SH degree: 3 (Reference3DGS), 2 (mixed), 0 (sg1, sg3) */
    int32_t layout;        /* sgs_ply_layout, detected from the property names */
    int32_t binary;        /* 1: binary_little_endian, 0: ascii */
    double shared_axes[9]; /* row-major; header comment sg_axes, then the .meta sidecar */
    double background[3];  /* header comment sg_background, then the .meta sidecar */
} sgs_ply_info;

/* load_ply (ply.cpp:295-306) on the host: params receives count * (11 + colour
 * params) doubles, the flat order of sgs_scene_desc.params (Scene::param). With params ==
 * NULL the payload is checked but not kept, and *info filled.
 * Errors: SGS_ERR_IO (IoError), SGS_ERR_FORMAT (FormatError), SGS_ERR_INVALID_ARGUMENT
 * (an unknown sg_model name, non-orthonormal sg_axes), with the reference's
 * messages, checked in the reference's order. */
sgs_status sgs_ply_read(const char* path, sgs_ply_info* info, double* params, uint64_t params_capacity);
/* load_ply straight into a device scene: the float rows go to the device once and
 * a kernel scatters them into the scene planes (the same planes sgs_scene_upload
 * builds from sgs_ply_read's parameters, bit for bit). */
sgs_status sgs_scene_load_ply(sgs_context* ctx, const char* path, sgs_ply_info* info, sgs_scene** out);

/* --- multi-GPU ------------------------------------------------ *
 * Replaces the reference's per-view loops (tools/main.cpp:207-216, :280-287) and its
 * std::thread parallel_for (common.hpp:53-77) across GPUs: one rank per GPU over
 * NCCL, the scene replicated by one broadcast, the views block-partitioned, the
 * frames gathered to a root with grouped send/recv overlapped with rendering. Every
 * sgs_group_* call below is collective: each rank makes it (one process per GPU, or
 * one host thread per rank of an sgs_group_create set). NCCL is loaded at run time;
 * without it these calls return SGS_ERR_NCCL. */
typedef struct sgs_group sgs_group;
#define SGS_GROUP_ID_BYTES 128
/* A fresh NCCL unique id (ncclGetUniqueId), made on one rank and shipped to all. */
sgs_status sgs_group_unique_id(uint8_t* id /* SGS_GROUP_ID_BYTES */);
/* Rank `rank` of `nranks` on ctx's device (ncclCommInitRank; one process per GPU). */
sgs_status sgs_group_init_rank(sgs_context* ctx, int32_t nranks, int32_t rank, const uint8_t* id,
                               sgs_group** out);
/* Every rank of one process (ncclCommInitAll over devices[0..ndev)), each with its
 * own context: out[r] is rank r. Drive each rank's collective calls from its own
 * host thread. */
sgs_status sgs_group_create(int32_t ndev, const int32_t* devices, sgs_group** out /* ndev */);
void sgs_group_destroy(sgs_group* group);
/* The rank's render context (owned by the group when made by sgs_group_create). */
sgs_status sgs_group_context(sgs_group* group, sgs_context** ctx);
/* The root uploads desc (ignored elsewhere); its device layout and blob reach every
 * rank by NCCL broadcast; *out is the rank's device scene (free with sgs_scene_free). */
sgs_status sgs_group_broadcast_scene(sgs_group* group, const sgs_scene_desc* desc, int32_t root,
                                     sgs_scene** out);
/* Views [0, n) of cams (the same on every rank), rank r rendering its contiguous
 * block; the root receives every frame: rgb + i*H*W*3 and T + i*H*W (T may be NULL)
 * in out_memory (device buffers on the root's device, or host). Other ranks ignore
 * rgb and the value of T, but T's null-ness must match the root's (it says whether
 * transmittance frames travel). stats (optional) accumulates the rank's own views.
 * The views must share one image size (SGS_ERR_INVALID_ARGUMENT otherwise). Like any
 * collective, an error on one rank leaves the others waiting in NCCL: callers abort
 * the group (sgs_group_destroy on every rank) after a failure. */
sgs_status sgs_group_render_views(sgs_group* group, const sgs_scene* scene, const sgs_camera* cams, int32_t n,
                                  const sgs_render_config* cfg, int32_t root, float* rgb, float* T,
                                  int32_t out_memory, sgs_render_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* SGS_H */
