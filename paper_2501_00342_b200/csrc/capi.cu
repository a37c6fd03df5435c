// capi.cu -- the C-ABI (include/sgs.h): contexts, device scenes, frame orchestration.
//
// Frame pipeline on the context stream:
//   K1 preprocess -> K2 stable radix sort of FP64 depth keys (values: Gaussian index)
//   -> K3 gather per-rank tile counts + exclusive scan -> [one 40-B D2H of the
//   counters: error word, V, P; sizes the tile-key arena] -> K4 emit (tile,index)
//   keys -> K5 stable radix sort on the tile bits -> K6 tile ranges -> K7 composite.
// Radix sorts and the scan use CUB (CUDA 12.9 CCCL) as the library primitive.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "sgs_internal.h"

using namespace sgs;

namespace {

thread_local std::string g_last_error;

sgs_status fail(sgs_status code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define SGS_CUDA(call)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) {                                                             \
            return fail(e_ == cudaErrorMemoryAllocation ? SGS_ERR_OUT_OF_MEMORY : SGS_ERR_CUDA, \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                 \
        }                                                                                    \
    } while (0)

struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t need) {
        if (need <= bytes) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        size_t grow = need + need / 4 + 256;
        cudaError_t e = cudaMalloc(&ptr, grow);
        if (e == cudaSuccess) bytes = grow;
        return e;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
};

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

int color_param_count_impl(int kind, int degree) {
    switch (kind) {
        case SGS_SH: return 3 * (degree + 1) * (degree + 1);
        case SGS_SG1: return 10;
        case SGS_SG3: return 15;
        case SGS_MIXED: return 3 * (degree + 1) * (degree + 1) + 12;
    }
    return -1;
}

}  // namespace

struct sgs_scene {
    sgs_scene_meta meta{};
    sgs_context* ctx = nullptr;
    DevBuf owned;
    void* blob = nullptr;
    ScenePlanes planes{};
};

struct sgs_context {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    std::mutex mu;
    DevBuf keys_a, keys_b, key32_a, key32_b, iota, order, rec, colour, degree, rects, ntiles, brect, bmeta, counts,
        offsets;
    uint64_t iota_n = 0;
    DevBuf buckets;  // K2 bucket histogram / offsets / cursors
    DevBuf work;     // K7 work list (+ 3 control words)
    DevBuf tkeys_a, tkeys_b, ranges, tile_done, pix_state, pix_walked, cub_temp, sort_hist, frame_rgb[2],
        frame_T[2];
    uint64_t tkey_cap = 0;  // tile keys per buffer (grow-only, sized from observed P)
    Counters* d_ctr = nullptr;
    Counters* h_ctr = nullptr;
    Counters* h_ctr_init = nullptr;  // pinned initial counters block (err/kmin = ~0)
    FrameConsts* d_consts = nullptr;  // per-frame scene planes + camera for K7's FP64 path
    FrameConsts* h_consts = nullptr;  // pinned staging copy
    bool chunking = true;
    std::vector<uint64_t> chunk_divs{16, 4};  // depth-chunk boundaries at N/16, N/4
    cudaEvent_t ev[8] = {};
    cudaEvent_t frame_done[2] = {};
    cudaEvent_t slot_free[2] = {};
    // results of the last frame (device pointers into the buffers above)
    const uint32_t* last_order = nullptr;
    const unsigned long long* last_tile_keys = nullptr;
    uint64_t last_v = 0, last_p = 0;
    uint64_t own_launches = 0, lib_launches = 0;
};

namespace {

// ---------------------------------------------------------------------------
// Host-side validation and constants, in the reference's order and arithmetic
// (this TU's host code is compiled with -ffp-contract=off).

sgs_status validate_camera(const sgs_camera* cam) {
    // Camera::validate, camera.cpp:10-13
    if (cam->fx <= 0 || cam->fy <= 0) return fail(SGS_ERR_INVALID_ARGUMENT, "camera focal lengths must be positive");
    if (cam->width < 1 || cam->height < 1) return fail(SGS_ERR_INVALID_ARGUMENT, "camera image size must be >= 1");
    return SGS_OK;
}

CamParams make_cam(const sgs_camera* c) {
    CamParams p{};
    for (int i = 0; i < 9; ++i) p.R[i] = c->R[i];
    for (int i = 0; i < 3; ++i) p.t[i] = c->t[i];
    // center() = -R^T t (camera.hpp:20), left-to-right sums
    for (int i = 0; i < 3; ++i)
        p.C[i] = ((-c->R[0 * 3 + i]) * c->t[0] + (-c->R[1 * 3 + i]) * c->t[1]) + (-c->R[2 * 3 + i]) * c->t[2];
    p.fx = c->fx;
    p.fy = c->fy;
    p.cx = c->cx;
    p.cy = c->cy;
    p.width = c->width;
    p.height = c->height;
    p.near_plane = c->near_plane;
    p.lim_x = 1.3 * (0.5 * c->width / c->fx);  // raster.cpp:29-30
    p.lim_y = 1.3 * (0.5 * c->height / c->fy);
    p.W = c->width;
    p.H = c->height;
    return p;
}

CfgParams make_cfg(const sgs_render_config* cfg, const sgs_camera* cam) {
    CfgParams k{};
    k.tile_size = cfg->tile_size;
    k.tiles_x = (cam->width + cfg->tile_size - 1) / cfg->tile_size;
    k.tiles_y = (cam->height + cfg->tile_size - 1) / cfg->tile_size;
    k.has_override = cfg->has_override;
    k.override_degree = cfg->override_degree;
    k.lo = cfg->degree_threshold_lo;
    k.hi = cfg->degree_threshold_hi;
    k.early_stop = static_cast<float>(cfg->early_stop_transmittance);
    return k;
}

sgs_status device_error(unsigned long long word, const sgs_scene* scene, const sgs_render_config* cfg) {
    const unsigned code = static_cast<unsigned>(word & 0xFF);
    const unsigned long long idx = word >> 8;
    char buf[256];
    switch (code) {
        case kErrZeroQuaternion:
            return fail(SGS_ERR_NUMERIC, "degenerate rotation: zero quaternion");
        case kErrThresholds:
            return fail(SGS_ERR_INVALID_ARGUMENT, "degree thresholds must satisfy lo <= hi");
        case kErrOverrideNonMixed:
            return fail(SGS_ERR_INVALID_ARGUMENT, "sh_degree_override is only valid for mixed scenes");
        case kErrDegreeTooHigh:
            std::snprintf(buf, sizeof(buf), "sh degree override %d exceeds stored degree %d",
                          cfg->has_override ? cfg->override_degree : 2, scene->meta.sh_degree);
            return fail(SGS_ERR_INVALID_ARGUMENT, buf);
        case kErrDirection:
            return fail(SGS_ERR_INVALID_ARGUMENT, "direction must be unit length");
    }
    std::snprintf(buf, sizeof(buf), "device error %u at gaussian %llu", code, idx);
    return fail(SGS_ERR_INTERNAL, buf);
}

int ceil_log2(uint64_t v) {
    int b = 0;
    while ((1ULL << b) < v) ++b;
    return b;
}

enum FrameMode { kRender = 0, kProjectOnly = 1, kTileGrid = 2 };
// run_frame_once results besides sgs_status
constexpr int kRetryWide = 100;  // a run of equal 32-bit depth keys: redo with 64-bit keys
constexpr int kRetryGrow = 101;  // the tile-key arena was too small: grown, redo

// Depth chunking: the first chunk holds the
// nearest ceil(N / kFirstChunkDiv) ranks; tiles whose pixels all terminate inside it
// are finished and receive no keys from the second chunk.
constexpr uint64_t kMinChunkedN = 1 << 16;

sgs_status sort_depth(sgs_context* ctx, uint64_t n, bool wide, cudaStream_t s, const uint32_t** order_out) {
    uint32_t* order = ctx->order.as<uint32_t>();
    size_t temp = 0;
    if (!wide) {
        // K2: exact bucket sort (depth_sort.cu)
        const int log2b = depth_bucket_log2(n);
        const uint32_t nb = 1u << log2b;
        SGS_CUDA(ctx->buckets.ensure(static_cast<size_t>(nb + 1) * 4 * 4));
        uint32_t* hist = ctx->buckets.as<uint32_t>();
        uint32_t* off = hist + (nb + 1);
        uint32_t* cursor = off + (nb + 1);
        SGS_CUDA(cudaMemsetAsync(hist, 0, static_cast<size_t>(nb + 1) * 4, s));
        SGS_CUDA(cudaMemsetAsync(cursor, 0, static_cast<size_t>(nb + 1) * 4, s));
        launch_bucket_hist(n, ctx->keys_a.as<unsigned long long>(), ctx->d_ctr, log2b, hist, s);
        SGS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, hist, off, static_cast<int>(nb + 1), s));
        SGS_CUDA(ctx->cub_temp.ensure(temp));
        SGS_CUDA(cub::DeviceScan::ExclusiveSum(ctx->cub_temp.ptr, temp, hist, off, static_cast<int>(nb + 1), s));
        launch_bucket_scatter(n, ctx->keys_a.as<unsigned long long>(), ctx->d_ctr, log2b, off, cursor, order,
                              ctx->keys_b.as<unsigned long long>(), s);
        launch_bucket_sort(nb, off, ctx->keys_b.as<unsigned long long>(), order, ctx->d_ctr, cursor + (nb + 1), s);
        ctx->own_launches += 4;
        ctx->lib_launches += 2;
    } else {
        // fallback: full 64-bit keys (8 passes); stable, so ties keep index order
        SGS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, ctx->keys_a.as<unsigned long long>(),
                                                 ctx->keys_b.as<unsigned long long>(), ctx->iota.as<uint32_t>(),
                                                 order, static_cast<int>(n), 0, 64, s));
        SGS_CUDA(ctx->cub_temp.ensure(temp));
        SGS_CUDA(cub::DeviceRadixSort::SortPairs(ctx->cub_temp.ptr, temp, ctx->keys_a.as<unsigned long long>(),
                                                 ctx->keys_b.as<unsigned long long>(), ctx->iota.as<uint32_t>(),
                                                 order, static_cast<int>(n), 0, 64, s));
        ctx->lib_launches += 1 + 8;
    }
    SGS_CUDA(cudaGetLastError());
    *order_out = order;
    return SGS_OK;
}

// K3 for ranks [rb, re): counts -> exclusive scan; the total P stays on the device.
sgs_status count_and_scan(sgs_context* ctx, uint64_t rb, uint64_t re, const uint32_t* order, const uint32_t* done,
                          int tiles_x, int ntile, cudaStream_t s) {
    const uint64_t m = re - rb;
    (void)order;
    launch_count_tiles(rb, re, ctx->bmeta.as<uint2>(), ctx->brect.as<int4>(), done, tiles_x, ntile,
                       ctx->counts.as<unsigned long long>(), s);
    size_t temp = 0;
    SGS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, ctx->counts.as<unsigned long long>(),
                                           ctx->offsets.as<unsigned long long>(), static_cast<int>(m + 1), s));
    SGS_CUDA(ctx->cub_temp.ensure(temp));
    SGS_CUDA(cub::DeviceScan::ExclusiveSum(ctx->cub_temp.ptr, temp, ctx->counts.as<unsigned long long>(),
                                           ctx->offsets.as<unsigned long long>(), static_cast<int>(m + 1), s));
    launch_finish_scan(ctx->offsets.as<unsigned long long>() + m, ctx->tkey_cap, ctx->d_ctr, s);
    ctx->own_launches += 2;
    ctx->lib_launches += 2;
    return SGS_OK;
}

// One frame on ctx->stream. Outputs are device pointers (either may be null).
// The whole frame is enqueued without a host round trip (every data-dependent
// size lives on the device); one synchronisation at the end reads the counters,
// reports errors, and -- rarely -- regrows the tile-key arena or falls back to the
// 64-bit depth sort and renders the frame again.
int run_frame_once(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                          const sgs_render_config* cfg, float* d_rgb, float* d_T, sgs_render_stats* stats,
                          DebugSplat* d_debug, FrameMode mode, bool wide_sort) {
    cudaStream_t s = ctx->stream;
    const uint64_t n = scene->meta.count;
    const CamParams cp = make_cam(cam);
    const CfgParams kp = make_cfg(cfg, cam);
    const uint64_t ntile = static_cast<uint64_t>(kp.tiles_x) * static_cast<uint64_t>(kp.tiles_y);
    const uint64_t npx = static_cast<uint64_t>(cam->width) * static_cast<uint64_t>(cam->height);
    const bool timing = stats && stats->want_timing;
    const uint64_t n1 = std::max<uint64_t>(n, 1);

    SGS_CUDA(ctx->keys_a.ensure(n1 * 8));
    SGS_CUDA(ctx->keys_b.ensure(n1 * 8));
    if (ctx->iota.bytes < n1 * 4) ctx->iota_n = 0;
    SGS_CUDA(ctx->iota.ensure(n1 * 4));
    SGS_CUDA(ctx->order.ensure(n1 * 4));
    SGS_CUDA(ctx->rec.ensure(n1 * sizeof(SplatRec)));
    SGS_CUDA(ctx->rects.ensure(n1 * sizeof(int4)));
    SGS_CUDA(ctx->colour.ensure(n1 * sizeof(float4)));
    SGS_CUDA(ctx->ntiles.ensure(n1 * 4));
    SGS_CUDA(ctx->brect.ensure(n1 * sizeof(int4)));
    SGS_CUDA(ctx->bmeta.ensure(n1 * sizeof(uint2)));
    SGS_CUDA(ctx->counts.ensure((n + 1) * 8));
    SGS_CUDA(ctx->offsets.ensure((n + 1) * 8));
    SGS_CUDA(ctx->ranges.ensure(std::max<uint64_t>(ntile, 1) * sizeof(uint2)));
    SGS_CUDA(ctx->sort_hist.ensure(tile_sort_hist_bytes()));
    if (ctx->tkey_cap == 0) ctx->tkey_cap = std::max<uint64_t>(16 * n, 1 << 20);
    SGS_CUDA(ctx->tkeys_a.ensure(ctx->tkey_cap * 8));
    SGS_CUDA(ctx->tkeys_b.ensure(ctx->tkey_cap * 8));

    if (timing) SGS_CUDA(cudaEventRecord(ctx->ev[0], s));
    SGS_CUDA(cudaMemcpyAsync(ctx->d_ctr, ctx->h_ctr_init, sizeof(Counters), cudaMemcpyHostToDevice, s));
    if (mode == kRender) {
        // the pinned staging block is reused every frame; the previous frame has
        // completed (run_frame synchronises at its end)
        ctx->h_consts->sp = scene->planes;
        ctx->h_consts->cam = cp;
        SGS_CUDA(cudaMemcpyAsync(ctx->d_consts, ctx->h_consts, sizeof(FrameConsts), cudaMemcpyHostToDevice, s));
    }

    // K1
    if (ctx->iota_n < n) {  // identity values for the depth sort (kept across frames)
        launch_iota(n, ctx->iota.as<uint32_t>(), s);
        ctx->iota_n = n;
    }
    launch_preprocess(scene->planes, cp, kp, ctx->keys_a.as<unsigned long long>(), ctx->rec.as<SplatRec>(),
                      ctx->rects.as<int4>(), ctx->ntiles.as<uint32_t>(), ctx->colour.as<float4>(), ctx->d_ctr,
                      d_debug, s);
    SGS_CUDA(cudaGetLastError());
    if (n) ctx->own_launches += 1;
    if (timing) SGS_CUDA(cudaEventRecord(ctx->ev[1], s));
    if (mode == kProjectOnly) {
        SGS_CUDA(cudaMemcpyAsync(ctx->h_ctr, ctx->d_ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
        SGS_CUDA(cudaStreamSynchronize(s));
        if (ctx->h_ctr->err != ~0ULL) return device_error(ctx->h_ctr->err, scene, cfg);
        return SGS_OK;
    }

    // K2
    const uint32_t* order = ctx->iota.as<uint32_t>();
    if (n > 1) {
        sgs_status st = sort_depth(ctx, n, wide_sort, s, &order);
        if (st != SGS_OK) return st;
    }
    // rank-ordered binning inputs, gathered once for every chunk
    launch_gather_bins(n, order, ctx->rects.as<int4>(), ctx->ntiles.as<uint32_t>(), ctx->brect.as<int4>(),
                       ctx->bmeta.as<uint2>(), s);
    if (n) ctx->own_launches += 1;
    if (timing) SGS_CUDA(cudaEventRecord(ctx->ev[2], s));

    // depth chunks over ranks (bounds known on the host: culled splats sort last and
    // contribute no tiles, so rank bounds can be taken over N)
    const bool multi = mode == kRender && ctx->chunking && n >= kMinChunkedN &&
                       composite_pixel_chunks(cfg->tile_size) == 1;
    std::vector<uint64_t> bounds{0};
    if (multi) {
        for (uint64_t div : ctx->chunk_divs) {
            const uint64_t b = (n + div - 1) / div;
            if (b > bounds.back() && b < n) bounds.push_back(b);
        }
        SGS_CUDA(ctx->tile_done.ensure((ntile + 31) / 32 * 4 * 2));  // done + touched bitmaps
        SGS_CUDA(ctx->pix_state.ensure(npx * sizeof(PixelState)));
        SGS_CUDA(ctx->pix_walked.ensure(npx * sizeof(uint32_t)));
        SGS_CUDA(cudaMemsetAsync(ctx->tile_done.ptr, 0, (ntile + 31) / 32 * 4 * 2, s));
    }
    bounds.push_back(n);
    const int nchunks = static_cast<int>(bounds.size()) - 1;
    const float3 bg = make_float3(static_cast<float>(scene->meta.background[0]),
                                  static_cast<float>(scene->meta.background[1]),
                                  static_cast<float>(scene->meta.background[2]));
    const int tile_bits = std::max(1, ceil_log2(ntile));
    const uint64_t work_cap = ntile * static_cast<uint64_t>(composite_pixel_chunks(cfg->tile_size));
    SGS_CUDA(ctx->work.ensure((work_cap + 4) * sizeof(uint32_t)));
    // work items: tiles always need a pass at least in the last chunk
    const unsigned long long* d_pc = &ctx->d_ctr->chunk_entries;
    float ms_bin = 0, ms_tsort = 0, ms_comp = 0;
    for (int c = 0; c < nchunks; ++c) {
        const uint64_t rb = bounds[c], re = bounds[c + 1];
        const uint32_t* done = c > 0 ? ctx->tile_done.as<uint32_t>() : nullptr;
        if (timing) SGS_CUDA(cudaEventRecord(ctx->ev[3], s));
        // K3 + K4
        sgs_status st = count_and_scan(ctx, rb, re, order, done, kp.tiles_x, static_cast<int>(ntile), s);
        if (st != SGS_OK) return st;
        launch_emit_tile_keys(rb, re, ctx->bmeta.as<uint2>(), ctx->brect.as<int4>(), done,
                              ctx->offsets.as<unsigned long long>(), kp.tiles_x, static_cast<int>(ntile),
                              ctx->tkeys_a.as<unsigned long long>(), ctx->tkey_cap, s);
        SGS_CUDA(cudaGetLastError());
        if (re > rb) ctx->own_launches += 1;
        if (timing) SGS_CUDA(cudaEventRecord(ctx->ev[4], s));
        // K5 (device-sized stable radix sort on the tile bits)
        const unsigned long long* tkeys = tile_sort(ctx->tkeys_a.as<unsigned long long>(),
                                                    ctx->tkeys_b.as<unsigned long long>(), d_pc, tile_bits,
                                                    ctx->sort_hist.as<uint32_t>(), s, &ctx->own_launches);
        // K6
        SGS_CUDA(cudaMemsetAsync(ctx->ranges.ptr, 0, ntile * sizeof(uint2), s));
        launch_tile_ranges(d_pc, tkeys, ctx->ranges.as<uint2>(), s);
        SGS_CUDA(cudaGetLastError());
        ctx->own_launches += 1;
        if (timing) SGS_CUDA(cudaEventRecord(ctx->ev[5], s));
        ctx->last_order = order;
        ctx->last_tile_keys = tkeys;
        // K7
        if (mode == kRender) {
            launch_composite(ctx->d_consts, cp, kp, ctx->ranges.as<uint2>(), tkeys, ctx->rec.as<SplatRec>(),
                             ctx->colour.as<float4>(), bg, d_rgb, d_T, ctx->pix_state.as<PixelState>(), ctx->pix_walked.as<uint32_t>(),
                             ctx->tile_done.as<uint32_t>(), ctx->tile_done.as<uint32_t>() + (ntile + 31) / 32,
                             c == 0, c == nchunks - 1, ctx->d_ctr, stats != nullptr, ctx->work.as<uint32_t>(),
                             ctx->work.as<uint32_t>() + work_cap, s);
            SGS_CUDA(cudaGetLastError());
            ctx->own_launches += 2;  // work list + persistent compositor
        }
        if (timing) {
            SGS_CUDA(cudaEventRecord(ctx->ev[6], s));
            SGS_CUDA(cudaEventSynchronize(ctx->ev[6]));
            float a = 0, b = 0, d = 0;
            SGS_CUDA(cudaEventElapsedTime(&a, ctx->ev[3], ctx->ev[4]));
            SGS_CUDA(cudaEventElapsedTime(&b, ctx->ev[4], ctx->ev[5]));
            SGS_CUDA(cudaEventElapsedTime(&d, ctx->ev[5], ctx->ev[6]));
            ms_bin += a;
            ms_tsort += b;
            ms_comp += d;
        }
    }
    if (timing) SGS_CUDA(cudaEventRecord(ctx->ev[7], s));
    SGS_CUDA(cudaMemcpyAsync(ctx->h_ctr, ctx->d_ctr, sizeof(Counters), cudaMemcpyDeviceToHost, s));
    SGS_CUDA(cudaStreamSynchronize(s));
    const Counters& hc = *ctx->h_ctr;
    if (hc.err != ~0ULL) return device_error(hc.err, scene, cfg);
    if (hc.tie_overflow && !wide_sort) return kRetryWide;
    if (hc.key_overflow) {
        ctx->tkey_cap = hc.max_chunk_entries + hc.max_chunk_entries / 4 + 1024;
        return kRetryGrow;
    }
    ctx->last_v = hc.visible;
    ctx->last_p = hc.chunk_entries;  // the (single) chunk's P for the debug dump
    if (stats) {
        stats->visible += hc.visible;
        stats->tile_entries += hc.tile_entries;
        stats->block_entries += hc.block_entries;
        stats->guard_hits += hc.guard_hits;
        if (timing) {
            float k1 = 0, k2 = 0, total = 0;
            SGS_CUDA(cudaEventElapsedTime(&k1, ctx->ev[0], ctx->ev[1]));
            SGS_CUDA(cudaEventElapsedTime(&k2, ctx->ev[1], ctx->ev[2]));
            SGS_CUDA(cudaEventElapsedTime(&total, ctx->ev[0], ctx->ev[7]));
            stats->ms_preprocess += k1;
            stats->ms_depth_sort += k2;
            stats->ms_binning += ms_bin;
            stats->ms_tile_sort += ms_tsort;
            stats->ms_composite += ms_comp;
            stats->ms_total += total;
        }
    }
    return SGS_OK;
}

sgs_status run_frame(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                     const sgs_render_config* cfg, float* d_rgb, float* d_T, sgs_render_stats* stats,
                     DebugSplat* d_debug, FrameMode mode) {
    if (cfg->tile_size < 1) return fail(SGS_ERR_INVALID_ARGUMENT, "tile_size must be >= 1");
    sgs_status st = validate_camera(cam);
    if (st != SGS_OK) return st;
    bool wide = false;
    for (int attempt = 0; attempt < 4; ++attempt) {
        const int rc = run_frame_once(ctx, scene, cam, cfg, d_rgb, d_T, stats, d_debug, mode, wide);
        if (rc == kRetryWide) {
            wide = true;
            continue;
        }
        if (rc == kRetryGrow) continue;
        return static_cast<sgs_status>(rc);
    }
    return fail(SGS_ERR_INTERNAL, "frame did not converge after re-sizing");
}

// ---------------------------------------------------------------------------
// Scene layout and upload.

struct Layout {
    size_t geo_off[11];
    size_t color_off;
    size_t bytes;
    int color_planes;
};

Layout make_layout(const sgs_scene_meta& m) {
    Layout L{};
    const size_t n = m.count;
    size_t off = 0;
    if (m.geometry_f64) {
        for (int k = 0; k < 11; ++k) {
            L.geo_off[k] = off;
            off = align_up(off + n * 8, 256);
        }
    } else {
        for (int k = 0; k < 3; ++k) {
            L.geo_off[k] = off;
            off = align_up(off + n * 16, 256);
        }
    }
    L.color_planes = color_plane_count(m.kind, m.sh_degree);
    L.color_off = off;
    off = align_up(off + static_cast<size_t>(L.color_planes) * n * 16, 256);
    L.bytes = std::max<size_t>(off, 256);
    return L;
}

void bind_planes(sgs_scene* sc) {
    const sgs_scene_meta& m = sc->meta;
    Layout L = make_layout(m);
    ScenePlanes& p = sc->planes;
    p = ScenePlanes{};
    p.n = m.count;
    p.kind = m.kind;
    p.sh_degree = m.sh_degree;
    p.geometry_f64 = m.geometry_f64;
    p.color_planes = L.color_planes;
    char* base = static_cast<char*>(sc->blob);
    if (m.geometry_f64) {
        for (int k = 0; k < 11; ++k) p.g8[k] = reinterpret_cast<const double*>(base + L.geo_off[k]);
    } else {
        for (int k = 0; k < 3; ++k) p.g4[k] = reinterpret_cast<const float4*>(base + L.geo_off[k]);
    }
    p.color = reinterpret_cast<const float4*>(base + L.color_off);
    for (int k = 0; k < 9; ++k) p.axes[k] = static_cast<float>(m.shared_axes[k]);
    for (int k = 0; k < 3; ++k) p.bg[k] = static_cast<float>(m.background[k]);
}

double param_at(const sgs_scene_desc* d, size_t idx) {
    if (d->dtype == SGS_F32) return static_cast<double>(static_cast<const float*>(d->params)[idx]);
    return static_cast<const double*>(d->params)[idx];
}

// Host staging of the blob from the reference's flat layout.
void fill_blob(const sgs_scene_desc* d, const sgs_scene_meta& m, std::vector<char>& host) {
    const Layout L = make_layout(m);
    host.assign(L.bytes, 0);
    const size_t n = m.count;
    const int cpc = color_param_count_impl(m.kind, m.sh_degree);
    const size_t stride = 11 + static_cast<size_t>(cpc);
    char* base = host.data();
    std::vector<float> c(static_cast<size_t>(L.color_planes) * 4);
    for (size_t i = 0; i < n; ++i) {
        const size_t o = i * stride;
        if (m.geometry_f64) {
            for (int k = 0; k < 11; ++k) reinterpret_cast<double*>(base + L.geo_off[k])[i] = param_at(d, o + k);
        } else {
            float4* g0 = reinterpret_cast<float4*>(base + L.geo_off[0]);
            float4* g1 = reinterpret_cast<float4*>(base + L.geo_off[1]);
            float4* g2 = reinterpret_cast<float4*>(base + L.geo_off[2]);
            auto f = [&](int k) { return static_cast<float>(param_at(d, o + k)); };
            g0[i] = make_float4(f(0), f(1), f(2), f(10));
            g1[i] = make_float4(f(3), f(4), f(5), f(6));
            g2[i] = make_float4(f(7), f(8), f(9), 0.f);
        }
        std::fill(c.begin(), c.end(), 0.f);
        const size_t co = o + 11;
        switch (m.kind) {
            case SGS_SH:
                for (int k = 0; k < cpc; ++k) c[k] = static_cast<float>(param_at(d, co + k));
                break;
            case SGS_MIXED: {
                const int nsh = 3 * (m.sh_degree + 1) * (m.sh_degree + 1);
                for (int k = 0; k < nsh; ++k) c[k] = static_cast<float>(param_at(d, co + k));
                const int lobe_base = 4 * ((nsh + 3) / 4);
                for (int k = 0; k < 12; ++k) c[lobe_base + k] = static_cast<float>(param_at(d, co + nsh + k));
                break;
            }
            case SGS_SG1: {
                // plane 0 (diffuse rgb, log_lambda), plane 1 (alpha rgb, 0), plane 2 (mu/|mu|, 0);
                // mu normalised in FP64 exactly as DiffuseSGModel::lobe (color.cpp:49-56)
                for (int k = 0; k < 3; ++k) c[k] = static_cast<float>(param_at(d, co + k));
                c[3] = static_cast<float>(param_at(d, co + 6));
                for (int k = 0; k < 3; ++k) c[4 + k] = static_cast<float>(param_at(d, co + 3 + k));
                const double mu[3] = {param_at(d, co + 7), param_at(d, co + 8), param_at(d, co + 9)};
                const double nn = std::sqrt((mu[0] * mu[0] + mu[1] * mu[1]) + mu[2] * mu[2]);
                for (int k = 0; k < 3; ++k)
                    c[8 + k] = static_cast<float>(nn > 1e-12 ? mu[k] / nn : (k == 0 ? 1.0 : 0.0));
                break;
            }
            case SGS_SG3:
                for (int k = 0; k < 3; ++k) c[k] = static_cast<float>(param_at(d, co + k));
                for (int k = 0; k < 12; ++k) c[4 + k] = static_cast<float>(param_at(d, co + 3 + k));
                break;
        }
        float4* cp = reinterpret_cast<float4*>(base + L.color_off);
        for (int pl = 0; pl < L.color_planes; ++pl)
            cp[static_cast<size_t>(pl) * n + i] = make_float4(c[4 * pl], c[4 * pl + 1], c[4 * pl + 2], c[4 * pl + 3]);
    }
}

sgs_status upload_common(sgs_context* ctx, const sgs_scene_desc* desc, void* blob, uint64_t bytes,
                         bool own, sgs_scene** out) {
    if (!ctx || !desc || !out) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    sgs_scene_meta m{};
    sgs_status st = sgs_scene_plan(desc, &m);
    if (st != SGS_OK) return st;
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    auto* sc = new sgs_scene();
    sc->meta = m;
    sc->ctx = ctx;
    if (own) {
        cudaError_t e = sc->owned.ensure(m.blob_bytes);
        if (e != cudaSuccess) {
            delete sc;
            return fail(SGS_ERR_OUT_OF_MEMORY, "scene allocation failed");
        }
        sc->blob = sc->owned.ptr;
    } else {
        if (bytes < m.blob_bytes) {
            delete sc;
            return fail(SGS_ERR_INVALID_ARGUMENT, "device blob smaller than meta.blob_bytes");
        }
        sc->blob = blob;
    }
    std::vector<char> host;
    fill_blob(desc, m, host);
    cudaError_t e = cudaMemcpy(sc->blob, host.data(), host.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        delete sc;
        return fail(SGS_ERR_CUDA, std::string("scene upload: ") + cudaGetErrorString(e));
    }
    bind_planes(sc);
    *out = sc;
    return SGS_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

int sgs_abi_version(void) { return SGS_ABI_VERSION; }

const char* sgs_last_error(void) { return g_last_error.c_str(); }

sgs_status sgs_create(int device, sgs_context** out) {
    if (!out) return fail(SGS_ERR_INVALID_ARGUMENT, "null out");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(SGS_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(SGS_ERR_INVALID_ARGUMENT, "bad device ordinal");
    SGS_CUDA(cudaSetDevice(device));
    auto* ctx = new sgs_context();
    ctx->device = device;
    SGS_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    SGS_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    SGS_CUDA(cudaMalloc(&ctx->d_ctr, sizeof(Counters)));
    SGS_CUDA(cudaMallocHost(&ctx->h_ctr, sizeof(Counters)));
    SGS_CUDA(cudaMallocHost(&ctx->h_ctr_init, sizeof(Counters)));
    SGS_CUDA(cudaMalloc(&ctx->d_consts, sizeof(FrameConsts)));
    SGS_CUDA(cudaMallocHost(&ctx->h_consts, sizeof(FrameConsts)));
    std::memset(ctx->h_ctr_init, 0, sizeof(Counters));
    ctx->h_ctr_init->err = ~0ULL;
    ctx->h_ctr_init->kmin = ~0ULL;
    if (const char* e = std::getenv("SGS_DEPTH_CHUNKING")) ctx->chunking = std::atoi(e) != 0;
    if (const char* e = std::getenv("SGS_DEPTH_CHUNKS")) {  // e.g. "16,4": boundaries at N/16, N/4
        ctx->chunk_divs.clear();
        for (const char* q = e; *q;) {
            char* endp = nullptr;
            const long v = std::strtol(q, &endp, 10);
            if (endp == q) break;
            if (v > 1) ctx->chunk_divs.push_back(static_cast<uint64_t>(v));
            q = *endp ? endp + 1 : endp;
        }
    }
    for (auto& ev : ctx->ev) SGS_CUDA(cudaEventCreate(&ev));
    for (int k = 0; k < 2; ++k) {
        SGS_CUDA(cudaEventCreateWithFlags(&ctx->frame_done[k], cudaEventDisableTiming));
        SGS_CUDA(cudaEventCreateWithFlags(&ctx->slot_free[k], cudaEventDisableTiming));
    }
    *out = ctx;
    return SGS_OK;
}

void sgs_destroy(sgs_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->copy_stream);
    for (DevBuf* b : {&ctx->keys_a, &ctx->keys_b, &ctx->key32_a, &ctx->key32_b, &ctx->iota, &ctx->order,
                      &ctx->rec, &ctx->colour, &ctx->degree, &ctx->rects, &ctx->ntiles, &ctx->brect, &ctx->bmeta, &ctx->counts, &ctx->offsets,
                      &ctx->tkeys_a, &ctx->tkeys_b, &ctx->ranges, &ctx->tile_done, &ctx->pix_state,
                      &ctx->pix_walked, &ctx->cub_temp, &ctx->sort_hist, &ctx->buckets, &ctx->work, &ctx->frame_rgb[0], &ctx->frame_rgb[1],
                      &ctx->frame_T[0], &ctx->frame_T[1]})
        b->release();
    if (ctx->d_ctr) cudaFree(ctx->d_ctr);
    if (ctx->h_ctr) cudaFreeHost(ctx->h_ctr);
    if (ctx->h_ctr_init) cudaFreeHost(ctx->h_ctr_init);
    if (ctx->d_consts) cudaFree(ctx->d_consts);
    if (ctx->h_consts) cudaFreeHost(ctx->h_consts);
    for (auto& ev : ctx->ev) cudaEventDestroy(ev);
    for (int k = 0; k < 2; ++k) {
        cudaEventDestroy(ctx->frame_done[k]);
        cudaEventDestroy(ctx->slot_free[k]);
    }
    cudaStreamDestroy(ctx->own_stream);
    cudaStreamDestroy(ctx->copy_stream);
    delete ctx;
}

sgs_status sgs_set_stream(sgs_context* ctx, void* stream) {
    if (!ctx) return fail(SGS_ERR_INVALID_ARGUMENT, "null context");
    std::lock_guard<std::mutex> lock(ctx->mu);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return SGS_OK;
}

sgs_status sgs_synchronize(sgs_context* ctx) {
    if (!ctx) return fail(SGS_ERR_INVALID_ARGUMENT, "null context");
    SGS_CUDA(cudaStreamSynchronize(ctx->stream));
    SGS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    return SGS_OK;
}

sgs_status sgs_launch_count(sgs_context* ctx, uint64_t* own_kernels, uint64_t* library_kernels) {
    if (!ctx || !own_kernels || !library_kernels) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    std::lock_guard<std::mutex> lock(ctx->mu);
    *own_kernels = ctx->own_launches;
    *library_kernels = ctx->lib_launches;
    return SGS_OK;
}

int32_t sgs_color_param_count(int32_t kind, int32_t sh_degree) { return color_param_count_impl(kind, sh_degree); }

sgs_status sgs_scene_plan(const sgs_scene_desc* d, sgs_scene_meta* m) {
    if (!d || !m) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    if (d->kind < SGS_SH || d->kind > SGS_MIXED) return fail(SGS_ERR_INVALID_ARGUMENT, "unknown color model kind");
    int deg = d->sh_degree;
    if (d->kind == SGS_SG1 || d->kind == SGS_SG3) deg = 0;
    if (d->kind == SGS_SH && (deg < 0 || deg > 3)) return fail(SGS_ERR_INVALID_ARGUMENT, "unsupported SH degree");
    if (d->kind == SGS_MIXED && (deg < 0 || deg > 2))
        return fail(SGS_ERR_INVALID_ARGUMENT, "mixed model stores SH degree 0..2");
    if (d->dtype != SGS_F32 && d->dtype != SGS_F64) return fail(SGS_ERR_INVALID_ARGUMENT, "bad dtype");
    if (d->count && !d->params) return fail(SGS_ERR_INVALID_ARGUMENT, "null params");
    if (d->count > 0xFFFFFFFFULL) return fail(SGS_ERR_INVALID_ARGUMENT, "more than 2^32 Gaussians");
    *m = sgs_scene_meta{};
    m->count = d->count;
    m->kind = d->kind;
    m->sh_degree = deg;
    // float32 geometry planes are lossless iff every geometry real is f32-exact
    int f64 = 0;
    if (d->dtype == SGS_F64) {
        const size_t stride = 11 + static_cast<size_t>(color_param_count_impl(d->kind, deg));
        const double* p = static_cast<const double*>(d->params);
        for (size_t i = 0; i < d->count && !f64; ++i)
            for (int k = 0; k < 11; ++k) {
                const double v = p[i * stride + k];
                if (static_cast<double>(static_cast<float>(v)) != v) {
                    f64 = 1;
                    break;
                }
            }
    }
    m->geometry_f64 = f64;
    for (int k = 0; k < 9; ++k) m->shared_axes[k] = d->shared_axes[k];
    for (int k = 0; k < 3; ++k) m->background[k] = d->background[k];
    m->blob_bytes = make_layout(*m).bytes;
    return SGS_OK;
}

sgs_status sgs_scene_pack(const sgs_scene_desc* desc, void* host_blob, uint64_t bytes) {
    if (!desc || !host_blob) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    sgs_scene_meta m{};
    sgs_status st = sgs_scene_plan(desc, &m);
    if (st != SGS_OK) return st;
    if (bytes < m.blob_bytes) return fail(SGS_ERR_INVALID_ARGUMENT, "host blob smaller than meta.blob_bytes");
    std::vector<char> host;
    fill_blob(desc, m, host);
    std::memcpy(host_blob, host.data(), host.size());
    return SGS_OK;
}

sgs_status sgs_scene_upload(sgs_context* ctx, const sgs_scene_desc* desc, sgs_scene** out) {
    return upload_common(ctx, desc, nullptr, 0, true, out);
}

sgs_status sgs_scene_upload_into(sgs_context* ctx, const sgs_scene_desc* desc, void* device_blob,
                                 uint64_t bytes, sgs_scene** out) {
    if (!device_blob) return fail(SGS_ERR_INVALID_ARGUMENT, "null device blob");
    return upload_common(ctx, desc, device_blob, bytes, false, out);
}

sgs_status sgs_scene_bind(sgs_context* ctx, const sgs_scene_meta* meta, void* device_blob,
                          uint64_t bytes, sgs_scene** out) {
    if (!ctx || !meta || !device_blob || !out) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    sgs_scene_meta m = *meta;
    m.blob_bytes = make_layout(m).bytes;
    if (bytes < m.blob_bytes) return fail(SGS_ERR_INVALID_ARGUMENT, "device blob smaller than layout");
    auto* sc = new sgs_scene();
    sc->meta = m;
    sc->ctx = ctx;
    sc->blob = device_blob;
    bind_planes(sc);
    *out = sc;
    return SGS_OK;
}

sgs_status sgs_scene_get_meta(const sgs_scene* scene, sgs_scene_meta* meta) {
    if (!scene || !meta) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    *meta = scene->meta;
    return SGS_OK;
}

sgs_status sgs_scene_blob(const sgs_scene* scene, void** device_blob, uint64_t* bytes) {
    if (!scene || !device_blob || !bytes) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    *device_blob = scene->blob;
    *bytes = scene->meta.blob_bytes;
    return SGS_OK;
}

sgs_status sgs_scene_set_background(sgs_scene* scene, const double* rgb) {
    if (!scene || !rgb) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    for (int k = 0; k < 3; ++k) scene->meta.background[k] = rgb[k];
    bind_planes(scene);
    return SGS_OK;
}

void sgs_scene_free(sgs_scene* scene) {
    if (!scene) return;
    if (scene->ctx) cudaSetDevice(scene->ctx->device);
    scene->owned.release();
    delete scene;
}

sgs_status sgs_render(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                      const sgs_render_config* cfg, float* rgb, float* T, int32_t out_memory,
                      sgs_render_stats* stats) {
    return sgs_render_batch(ctx, scene, cam, 1, cfg, rgb, T, out_memory, stats);
}

sgs_status sgs_render_batch(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cams,
                            int32_t n, const sgs_render_config* cfg, float* rgb, float* T,
                            int32_t out_memory, sgs_render_stats* stats) {
    if (!ctx || !scene || !cams || !cfg) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    if (n < 0) return fail(SGS_ERR_INVALID_ARGUMENT, "negative view count");
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    if (n == 0) return SGS_OK;
    const int W = cams[0].width, H = cams[0].height;
    for (int i = 1; i < n; ++i)
        if (cams[i].width != W || cams[i].height != H)
            return fail(SGS_ERR_INVALID_ARGUMENT, "all batch cameras must share width/height");
    if (W < 1 || H < 1) return validate_camera(&cams[0]);
    const size_t npx = static_cast<size_t>(W) * static_cast<size_t>(H);
    if (out_memory == SGS_DEVICE) {
        for (int i = 0; i < n; ++i) {
            sgs_status st = run_frame(ctx, scene, &cams[i], cfg, rgb ? rgb + i * npx * 3 : nullptr,
                                      T ? T + i * npx : nullptr, stats, nullptr, kRender);
            if (st != SGS_OK) return st;
        }
        SGS_CUDA(cudaStreamSynchronize(ctx->stream));
        return SGS_OK;
    }
    // Host outputs: render into a double-buffered device frame, copy back on the copy
    // stream while the next view renders.
    for (int k = 0; k < 2; ++k) {
        SGS_CUDA(ctx->frame_rgb[k].ensure(npx * 3 * sizeof(float)));
        SGS_CUDA(ctx->frame_T[k].ensure(npx * sizeof(float)));
        SGS_CUDA(cudaEventRecord(ctx->slot_free[k], ctx->copy_stream));
    }
    for (int i = 0; i < n; ++i) {
        const int k = i & 1;
        SGS_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->slot_free[k], 0));
        sgs_status st = run_frame(ctx, scene, &cams[i], cfg, rgb ? ctx->frame_rgb[k].as<float>() : nullptr,
                                  T ? ctx->frame_T[k].as<float>() : nullptr, stats, nullptr, kRender);
        if (st != SGS_OK) {
            cudaStreamSynchronize(ctx->copy_stream);
            return st;
        }
        SGS_CUDA(cudaEventRecord(ctx->frame_done[k], ctx->stream));
        SGS_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->frame_done[k], 0));
        if (rgb)
            SGS_CUDA(cudaMemcpyAsync(rgb + i * npx * 3, ctx->frame_rgb[k].ptr, npx * 3 * sizeof(float),
                                     cudaMemcpyDeviceToHost, ctx->copy_stream));
        if (T)
            SGS_CUDA(cudaMemcpyAsync(T + i * npx, ctx->frame_T[k].ptr, npx * sizeof(float),
                                     cudaMemcpyDeviceToHost, ctx->copy_stream));
        SGS_CUDA(cudaEventRecord(ctx->slot_free[k], ctx->copy_stream));
    }
    SGS_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    SGS_CUDA(cudaStreamSynchronize(ctx->stream));
    return SGS_OK;
}

sgs_status sgs_project(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                       const sgs_render_config* cfg, sgs_splat* out) {
    if (!ctx || !scene || !cam || !cfg || (!out && scene->meta.count)) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    static_assert(sizeof(sgs_splat) == sizeof(DebugSplat), "debug record layout");
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    const uint64_t n = scene->meta.count;
    DebugSplat* d_dbg = nullptr;
    SGS_CUDA(cudaMalloc(&d_dbg, std::max<uint64_t>(n, 1) * sizeof(DebugSplat)));
    sgs_status st = run_frame(ctx, scene, cam, cfg, nullptr, nullptr, nullptr, d_dbg, kProjectOnly);
    if (st == SGS_OK && n) {
        cudaError_t e = cudaMemcpy(out, d_dbg, n * sizeof(DebugSplat), cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) st = fail(SGS_ERR_CUDA, cudaGetErrorString(e));
    }
    cudaFree(d_dbg);
    return st;
}

sgs_status sgs_debug_tile_grid(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                               const sgs_render_config* cfg, uint32_t* order, uint64_t* n_visible,
                               uint64_t* offsets, uint32_t* entries, uint64_t capacity,
                               uint64_t* n_entries) {
    if (!ctx || !scene || !cam || !cfg || !n_visible || !n_entries)
        return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    sgs_status st = run_frame(ctx, scene, cam, cfg, nullptr, nullptr, nullptr, nullptr, kTileGrid);
    if (st != SGS_OK) return st;
    SGS_CUDA(cudaStreamSynchronize(ctx->stream));
    const uint64_t v = ctx->last_v, p = ctx->last_p;
    *n_visible = v;
    *n_entries = p;
    std::vector<uint32_t> ord(v);
    if (v) SGS_CUDA(cudaMemcpy(ord.data(), ctx->last_order, v * 4, cudaMemcpyDeviceToHost));
    if (order && v) std::memcpy(order, ord.data(), v * 4);
    if (!offsets && !entries) return SGS_OK;
    std::vector<unsigned long long> keys(p);
    if (p) SGS_CUDA(cudaMemcpy(keys.data(), ctx->last_tile_keys, p * 8, cudaMemcpyDeviceToHost));
    const uint64_t ntile = static_cast<uint64_t>((cam->width + cfg->tile_size - 1) / cfg->tile_size) *
                           static_cast<uint64_t>((cam->height + cfg->tile_size - 1) / cfg->tile_size);
    if (offsets) {
        std::vector<uint64_t> cnt(ntile + 1, 0);
        for (uint64_t i = 0; i < p; ++i) cnt[keys[i] >> 32]++;
        uint64_t acc = 0;
        for (uint64_t t = 0; t < ntile; ++t) {
            offsets[t] = acc;
            acc += cnt[t];
        }
        offsets[ntile] = acc;
    }
    if (entries) {
        std::vector<uint32_t> rank_of(scene->meta.count, 0xFFFFFFFFu);
        for (uint64_t r = 0; r < v; ++r) rank_of[ord[r]] = static_cast<uint32_t>(r);
        for (uint64_t i = 0; i < p && i < capacity; ++i) entries[i] = rank_of[static_cast<uint32_t>(keys[i])];
    }
    return SGS_OK;
}

sgs_status sgs_select_degree(double r, double lo, double hi, int32_t* out) {
    if (!out) return fail(SGS_ERR_INVALID_ARGUMENT, "null out");
    if (lo > hi) return fail(SGS_ERR_INVALID_ARGUMENT, "degree thresholds must satisfy lo <= hi");
    *out = r < lo ? 0 : (r < hi ? 1 : 2);
    return SGS_OK;
}

sgs_status sgs_flops_per_gaussian(int32_t kind, int32_t deg, int32_t* out) {
    // flops_per_gaussian, raster.cpp:190-227 (band ops 0/3/15/25, 2 ops per coeff per
    // channel, 8 per lobe, 2 per channel per lobe blend)
    if (!out) return fail(SGS_ERR_INVALID_ARGUMENT, "null out");
    static const int band_ops[4] = {0, 3, 15, 25};
    auto basis = [&](int d) {
        int s = 0;
        for (int l = 1; l <= d; ++l) s += band_ops[l];
        return s;
    };
    switch (kind) {
        case SGS_SH:
            if (deg < 0 || deg > 3) return fail(SGS_ERR_INVALID_ARGUMENT, "SH degree must be 0..3");
            *out = basis(deg) + 2 * (deg + 1) * (deg + 1) * 3;
            return SGS_OK;
        case SGS_SG1: *out = 8 + 2 * 3; return SGS_OK;
        case SGS_SG3: *out = 3 * 8 + 2 * 3 * 3; return SGS_OK;
        case SGS_MIXED:
            if (deg < 0 || deg > 2) return fail(SGS_ERR_INVALID_ARGUMENT, "mixed degree must be 0..2");
            *out = basis(deg) + 2 * (deg + 1) * (deg + 1) * 3 + 3 * 8 + 2 * 3 * 3;
            return SGS_OK;
    }
    return fail(SGS_ERR_INVALID_ARGUMENT, "unknown color model kind");
}

}  // extern "C"
