// capi.cu -- the C-ABI (include/sgs.h): contexts, device scenes, frame orchestration.
//
// Frame pipeline, enqueued on a lane stream with no host
// round trip: K1 preprocess -> K2 exact depth order (radix.cu: 32-bit keys, 4 onesweep
// passes, run fix-up, rank-ordered binning inputs) -> per depth chunk { K3+K4 count,
// look-back scan and emission of (tile, index) pairs -> K5 onesweep passes on the
// tile id -> K6 tile ranges -> K7 persistent compositor } -> the counters (errors,
// overflow retries, stats) written to mapped host memory. Views are dealt over
// lanes (streams with their own arenas). Every kernel is the library's own.
#include <algorithm>
#include <atomic>
#include <iterator>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ply_internal.h"
#include "projection.cuh"
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

// bumped by every (re)allocation: a captured frame graph holds buffer addresses
std::atomic<uint64_t> g_alloc_generation{0};

struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t need) {
        if (need <= bytes) return cudaSuccess;
        g_alloc_generation.fetch_add(1);
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        size_t grow = need + need / 16 + 256;  // (a little slack for sizes that creep up)
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

// Host loops over Gaussians (scene checks and packing) on every core: fn(begin, end).
template <typename Fn>
void parallel_for(size_t n, Fn&& fn) {
    const size_t hw = std::max<unsigned>(std::thread::hardware_concurrency(), 1u);
    const size_t nt = std::min<size_t>(hw, n / 65536 + 1);
    if (nt <= 1) {
        fn(size_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    const size_t per = (n + nt - 1) / nt;
    for (size_t t = 0; t < nt; ++t) {
        const size_t b = t * per, e = std::min(n, b + per);
        if (b < e) pool.emplace_back([&fn, b, e] { fn(b, e); });
    }
    for (auto& th : pool) th.join();
}

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
    DevBuf cov;  // cached 3D covariance planes (computed on the device at upload/bind)
    void* blob = nullptr;
    ScenePlanes planes{};
};

// One frame in flight: a stream plus every per-frame arena. sgs_render_batch deals
// views round-robin over the lanes, so one view's latency-bound sort and scan
// kernels overlap the other view's preprocess and compositing, and the host enqueues
// view i+1 while view i runs.
struct Lane {
    cudaStream_t stream = nullptr;  // the lane's current stream: plain or ranked
    cudaStream_t plain = nullptr, ranked = nullptr;
    cudaEvent_t swap = nullptr;
    DevBuf keys_a, keys_b, order, rec, colour, rects, brect, bmeta;
    DevBuf buckets;     // K2 coarse histogram / offsets
    DevBuf bin_status;  // K3/K4 scratch: per-rank counts, per-CTA sums
    DevBuf work;        // K7 work list (+ control words)
    // (tile id, Gaussian index) pairs, ping-pong for K5; also K2's sort scratch
    DevBuf tk_a, tv_a, tk_b, tv_b;
    DevBuf sort_hist;  // radix sort: per-slice digit histograms
    DevBuf ranges, tile_done, pix_state, pix_walked;
    DevBuf tile_emax;  // stats frames: deepest entry per (tile, pixel chunk) (E_t)
    // host-output frames: kOutSlots device buffers per lane drained by the lane's copy
    // stream, so the lane renders its next views while earlier ones cross PCIe
    static constexpr int kOutSlots = 3;
    DevBuf out_rgb[kOutSlots], out_T[kOutSlots];
    cudaEvent_t rendered[kOutSlots] = {};
    cudaEvent_t copied[kOutSlots] = {};
    cudaStream_t copy_stream = nullptr;
    int out_slot = 0;
    uint64_t tkey_cap = 0;  // tile pairs per buffer (grow-only, sized from observed P)
    Counters* d_ctr = nullptr;
    Counters* h_ctr = nullptr;      // mapped pinned host block the frame's counters land in
    Counters* h_ctr_dev = nullptr;  // its device-side address
    FrameConsts* d_consts = nullptr;  // per-frame scene planes + camera for K7's FP64 path
    FrameConsts* h_consts = nullptr;  // pinned staging copy
    cudaEvent_t ev[8] = {};
    cudaEvent_t done = nullptr;  // the frame's counters have reached h_ctr
    // the frame in flight (valid while busy)
    struct Job {
        const sgs_scene* scene = nullptr;
        sgs_camera cam{};
        sgs_render_config cfg{};
        float* d_rgb = nullptr;  // device outputs the compositor writes
        float* d_T = nullptr;
        float* h_rgb = nullptr;  // host outputs copied back on the lane stream
        float* h_T = nullptr;
        sgs_render_stats* stats = nullptr;
        DebugSplat* d_debug = nullptr;
        int mode = 0;
        float ms_bin = 0, ms_tsort = 0, ms_comp = 0;
    } job;
    bool busy = false;
    // the frame graph (launch_frame_graph): captured on the second frame with the same
    // key, replayed while the key holds
    cudaGraph_t graph = nullptr;  // kept alive: gk1 is one of its nodes
    cudaGraphExec_t gexec = nullptr;
    cudaGraphNode_t gk1 = nullptr;  // the K1 node, whose camera is patched per frame
    K1Record* grec = nullptr;
    std::vector<uint64_t> gkey, gpending;
    uint64_t g_launches = 0, g_lib_launches = 0;
    // results of the last frame (device pointers into the buffers above)
    const uint32_t* last_order = nullptr;
    const uint32_t* last_tiles = nullptr;  // sorted tile ids of the last chunk
    const uint32_t* last_list = nullptr;   // their Gaussian indices (the tile lists)
    uint64_t last_v = 0, last_p = 0;
};

constexpr int kLanes = 8;

struct sgs_context {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;  // the caller's stream: lanes fork from and join back to it
    std::mutex mu;
    Lane lane[kLanes];
    int lanes = 8;                     // lanes of the one-view-per-K1 schedule (SGS_LANES, 1..kLanes; 8 measured best)
    int host_lanes = 6;                // lanes for host-frame batches (SGS_HOST_LANES; fewer frames in flight
                                       // hand the copy engines their first frames sooner)
    Counters* h_ctr_init = nullptr;    // pinned initial counters block (err/kmin = ~0)
    bool chunking = true;
    std::vector<uint64_t> chunk_divs;  // depth-chunk boundaries N/div (SGS_DEPTH_CHUNKS; else by N)
    bool chunk_divs_set = false;
    cudaEvent_t fork = nullptr;
    bool graphs = true;     // frame graphs (SGS_GRAPHS=0 enqueues every frame directly)
    bool tight_rect = true; // render frames bin into the cut ellipse's tiles (SGS_TIGHT_RECT=0: 3-sigma rects)
    bool rank_host = true;  // ranked lane streams for host-frame batches (SGS_RANK_HOST=0 disables)
    bool trace = false;  // SGS_TRACE=1: per-frame lane timeline of each batch on stderr
    bool debug_capture_fail = false;  // SGS_DEBUG_CAPTURE_FAIL=1: a call the capture refuses (tests the fallback)
    struct TraceRec {
        int lane;
        cudaEvent_t ev[3];  // frame start, compositing done, host copies done
    };
    std::vector<TraceRec> trace_recs;
    DevBuf metrics;  // PSNR / SSIM scratch (inputs staged from host, maps, partial sums)
    DevBuf rows;     // float32 scene rows of an SGS_F32 upload (grow-only)
    // sgs_scene_update_rows: two pinned staging blocks (filled by the caller while the
    // other crosses PCIe) and the copy-done events
    void* stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    cudaEvent_t stage_ev[2] = {nullptr, nullptr};
    DevBuf bwd;      // backward scratch (FP64 splats, ranks, per-entry partials, staging)
    uint64_t hbm_bytes = 0;  // the device's memory
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
    // the compositor indexes pixels with 32 bits (the reference would need W H x 32 B)
    if (static_cast<uint64_t>(cam->width) * static_cast<uint64_t>(cam->height) >= (1ULL << 32))
        return fail(SGS_ERR_INVALID_ARGUMENT, "camera image too large: width * height must be < 2^32");
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
constexpr int kRetryGrow = 101;  // the tile-key arena was too small: grown, redo
// the radix sort's counters are 32-bit (kept one bit clear)
constexpr uint64_t kMaxSortKeys = (1ULL << 31) - 1;

// Depth chunking: the first chunk holds the
// nearest ceil(N / div0) ranks; tiles whose pixels all terminate inside it are
// finished and receive no keys from the next chunk. Each chunk costs a fixed chain of
// launches, so the boundaries follow N unless SGS_DEPTH_CHUNKS sets them (measured on
// the B200, 32-view batches: 100K at 800x800 0.164 ms/frame unchunked against 0.19
// with one boundary and 0.25 with two; 1M at 1080p 0.300 with one at N/8, 0.311 with
// N/16 and N/4, 0.372 unchunked; 3M at 1080p 0.624 with N/16 and N/4, 0.659 with N/8).
constexpr uint64_t kMinChunkedN = 1 << 16;  // floor for explicitly requested boundaries
std::vector<uint64_t> default_chunk_divs(uint64_t n) {
    if (n < (1u << 18)) return {};
    if (n < (2u << 20)) return {8};
    return {16, 4};
}

// Enqueue lane L's job on L.stream without a host round trip (every data-dependent
// size lives on the device), ending with a 128-B D2H of the counters and L.done.
// finish_frame() reads the counters, reports errors and -- rarely -- regrows the
// tile-key arena and enqueues the frame again.

// Everything the captured frame depends on besides the per-frame constants (camera,
// outputs) and the K1 camera: a frame whose key differs is enqueued directly; the
// second consecutive frame with one key is captured; later ones replay the graph.
std::vector<uint64_t> frame_graph_key(const sgs_context* ctx, const Lane& L) {
    const Lane::Job& j = L.job;
    auto bits = [](double v) {
        uint64_t u;
        std::memcpy(&u, &v, 8);
        return u;
    };
    std::vector<uint64_t> k{reinterpret_cast<uint64_t>(j.scene), j.scene->meta.count,
                            static_cast<uint64_t>(j.cam.width), static_cast<uint64_t>(j.cam.height),
                            static_cast<uint64_t>(j.cfg.tile_size), static_cast<uint64_t>(j.cfg.has_override),
                            static_cast<uint64_t>(j.cfg.override_degree), bits(j.cfg.degree_threshold_lo),
                            bits(j.cfg.degree_threshold_hi), bits(j.cfg.early_stop_transmittance),
                            (j.stats ? 1u : 0u) | (j.stats && j.stats->timing_path ? 2u : 0u),
                            static_cast<uint64_t>(j.mode), L.tkey_cap, g_alloc_generation.load(),
                            ctx->chunking ? 1u : 0u, ctx->chunk_divs_set ? 1u : 0u};
    for (uint64_t d : ctx->chunk_divs) k.push_back(d);
    // the scene as the captured kernels see it (plane addresses, layout, axes) and
    // its background (a K7 argument): a freed and re-uploaded scene can reuse the host
    // struct's address, so the key holds the contents, not the pointer alone
    uint64_t w[(sizeof(ScenePlanes) + 7) / 8] = {};
    std::memcpy(w, &j.scene->planes, sizeof(ScenePlanes));
    k.insert(k.end(), std::begin(w), std::end(w));
    for (int c = 0; c < 3; ++c) k.push_back(bits(j.scene->meta.background[c]));
    return k;
}

template <typename Body>
sgs_status launch_frame_graph(sgs_context* ctx, Lane& L, const CamParams& cp, Body&& body, bool& capturing) {
    cudaStream_t s = L.stream;
    const std::vector<uint64_t> key = frame_graph_key(ctx, L);
    if (!(L.gexec && key == L.gkey)) {
        if (key != L.gpending) {  // first frame with this key: direct (it sizes the arenas)
            L.gpending = key;
            return body();
        }
        if (L.gexec) {
            cudaGraphExecDestroy(L.gexec);
            L.gexec = nullptr;
        }
        if (L.graph) {
            cudaGraphDestroy(L.graph);
            L.graph = nullptr;
        }
        if (L.grec) {
            k1_record_free(L.grec);
            L.grec = nullptr;
        }
        const uint64_t own0 = ctx->own_launches, lib0 = ctx->lib_launches;
        cudaGraph_t g = nullptr;
        SGS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        capturing = true;
        const sgs_status st = body();
        capturing = false;
        const cudaError_t ec = cudaStreamEndCapture(s, &g);
        if (st != SGS_OK || ec != cudaSuccess || !g) {
            // A capture the driver refused -- at the end, or as a failing call inside the
            // body (StreamCaptureUnsupported / Invalidated): this context enqueues frames
            // directly from now on, starting with this one.
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            ctx->graphs = false;
            ctx->own_launches = own0;
            ctx->lib_launches = lib0;
            return body();
        }
        L.g_launches = ctx->own_launches - own0;
        L.g_lib_launches = ctx->lib_launches - lib0;
        ctx->own_launches = own0;
        ctx->lib_launches = lib0;
        // the K1 node: the kernel node running the recorded K1 function
        L.grec = k1_last_launch_clone();
        size_t nn = 0;
        SGS_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        SGS_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
        L.gk1 = nullptr;
        for (cudaGraphNode_t nd : nodes) {
            cudaGraphNodeType t;
            SGS_CUDA(cudaGraphNodeGetType(nd, &t));
            if (t != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams kp{};
            SGS_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
            if (kp.func == k1_record_func(L.grec)) L.gk1 = nd;
        }
        // (an empty scene launches no K1: nothing to patch)
        if (!L.gk1 && L.job.scene->meta.count > 0) {  // the K1 node was not found: no graphs
            cudaGraphDestroy(g);
            ctx->graphs = false;
            return body();
        }
        const cudaError_t ei = cudaGraphInstantiate(&L.gexec, g, 0);
        if (ei != cudaSuccess) {
            cudaGraphDestroy(g);
            L.gexec = nullptr;
            return fail(SGS_ERR_CUDA, std::string("frame graph: ") + cudaGetErrorString(ei));
        }
        L.graph = g;
        L.gkey = key;
    }
    if (L.gk1) SGS_CUDA(k1_record_patch(L.gexec, L.gk1, L.grec, cp));
    SGS_CUDA(cudaGraphLaunch(L.gexec, s));
    ctx->own_launches += L.g_launches;
    ctx->lib_launches += L.g_lib_launches;
    return SGS_OK;
}

sgs_status enqueue_frame(sgs_context* ctx, Lane& L) {
    Lane::Job& j = L.job;
    cudaStream_t s = L.stream;
    const sgs_scene* scene = j.scene;
    const sgs_camera* cam = &j.cam;
    const sgs_render_config* cfg = &j.cfg;
    const FrameMode mode = static_cast<FrameMode>(j.mode);
    const uint64_t n = scene->meta.count;
    const CamParams cp = make_cam(cam);
    CfgParams kp = make_cfg(cfg, cam);
    // render frames without stats bin each splat into the tiles its cut ellipse reaches
    // (E_t, a stat, is defined over the reference's lists, so stats frames keep them --
    // unless they only time the plain render path)
    const bool count_stats = j.stats && !j.stats->timing_path;
    kp.tight_rect = ctx->tight_rect && mode == kRender && !count_stats ? 1 : 0;
    const uint64_t ntile = static_cast<uint64_t>(kp.tiles_x) * static_cast<uint64_t>(kp.tiles_y);
    const uint64_t npx = static_cast<uint64_t>(cam->width) * static_cast<uint64_t>(cam->height);
    const bool timing = j.stats && j.stats->want_timing;
    const uint64_t n1 = std::max<uint64_t>(n, 1);
    j.ms_bin = j.ms_tsort = j.ms_comp = 0;

    SGS_CUDA(L.keys_a.ensure(n1 * 8));
    SGS_CUDA(L.order.ensure(n1 * 4));
    SGS_CUDA(L.rec.ensure(n1 * sizeof(SplatRec)));
    SGS_CUDA(L.rects.ensure(n1 * sizeof(int4)));
    SGS_CUDA(L.colour.ensure(n1 * sizeof(float4)));
    SGS_CUDA(L.brect.ensure(n1 * sizeof(int4)));
    SGS_CUDA(L.bmeta.ensure(n1 * sizeof(uint2)));
    SGS_CUDA(L.bin_status.ensure(bin_scratch_bytes(n1)));
    SGS_CUDA(L.ranges.ensure(std::max<uint64_t>(ntile, 1) * sizeof(uint2)));
    // tile pairs (grow-only; P above the capacity makes the frame regrow and redo);
    // at least n1, as K2 sorts in these arrays too
    if (L.tkey_cap == 0) L.tkey_cap = std::max<uint64_t>(2 * n, 1 << 20);  // (regrown from the observed P)
    L.tkey_cap = std::min<uint64_t>(std::max<uint64_t>(L.tkey_cap, n1), kMaxSortKeys);
    if (n1 > kMaxSortKeys) return fail(SGS_ERR_INVALID_ARGUMENT, "more than 2^31 - 1 Gaussians in one frame");
    SGS_CUDA(L.tk_a.ensure(L.tkey_cap * 4));
    SGS_CUDA(L.tv_a.ensure(L.tkey_cap * 4));
    SGS_CUDA(L.tk_b.ensure(L.tkey_cap * 4));
    SGS_CUDA(L.tv_b.ensure(L.tkey_cap * 4));
    SGS_CUDA(L.sort_hist.ensure(radix_hist_words() * 4));
    uint32_t* const shist = L.sort_hist.as<uint32_t>();
    float* d_rgb = j.d_rgb;
    float* d_T = j.d_T;
    const int slot = L.out_slot;
    if (j.h_rgb) {
        SGS_CUDA(L.out_rgb[slot].ensure(npx * 3 * sizeof(float)));
        d_rgb = L.out_rgb[slot].as<float>();
    }
    if (j.h_T) {
        SGS_CUDA(L.out_T[slot].ensure(npx * sizeof(float)));
        d_T = L.out_T[slot].as<float>();
    }

    const bool host_out = mode == kRender && (j.h_rgb || j.h_T);
    {
        if (mode == kRender) {
            // the pinned staging block is per lane; the lane's previous frame has
            // completed (finish_frame waits for it before the lane is reused)
            L.h_consts->sp = scene->planes;
            L.h_consts->cam = cp;
            L.h_consts->out_rgb = d_rgb;
            L.h_consts->out_T = d_T;
        }
    }
    if (host_out) {
        // the slot's previous frame must have left the device before K7 rewrites it
        SGS_CUDA(cudaStreamWaitEvent(s, L.copied[slot], 0));
        L.out_slot = (slot + 1) % Lane::kOutSlots;
    }
    sgs_context::TraceRec* tr = nullptr;
    if (ctx->trace && mode == kRender) {
        ctx->trace_recs.push_back(sgs_context::TraceRec{static_cast<int>(&L - ctx->lane), {}});
        tr = &ctx->trace_recs.back();
        for (auto& e : tr->ev) SGS_CUDA(cudaEventCreate(&e));
        SGS_CUDA(cudaEventRecord(tr->ev[0], s));
    }

    // The frame's device work (counters, constants, K1 ... K7, counters published):
    // enqueued directly, or captured once per lane and configuration into a CUDA
    // graph and replayed (one launch per frame instead of ~40 commands, the camera
    // patched into the K1 node; outputs come from the per-frame constants).
    bool capturing = false;
    auto rec_done = [&]() -> cudaError_t {
        return capturing ? cudaEventRecordWithFlags(L.done, s, cudaEventRecordExternal) : cudaEventRecord(L.done, s);
    };
    auto body = [&]() -> sgs_status {
        // (test hook: a stream synchronize is illegal inside a capture, as the driver
        // refusing it mid-body would be)
        if (capturing && ctx->debug_capture_fail) SGS_CUDA(cudaStreamSynchronize(s));
        {
            launch_counters_init(L.d_ctr, s);
            if (mode == kRender)
                SGS_CUDA(cudaMemcpyAsync(L.d_consts, L.h_consts, sizeof(FrameConsts), cudaMemcpyHostToDevice, s));
        }
        // K1
        {
            if (timing) SGS_CUDA(cudaEventRecord(L.ev[0], s));  // brackets K1 alone
            launch_preprocess(scene->planes, cp, kp, L.keys_a.as<unsigned long long>(), L.rec.as<SplatRec>(),
                              L.rects.as<int4>(), L.colour.as<float4>(), L.d_ctr, j.d_debug,
                              s);
            SGS_CUDA(cudaGetLastError());
            if (n) ctx->own_launches += 1;
            if (timing) SGS_CUDA(cudaEventRecord(L.ev[1], s));
        }
        if (mode == kProjectOnly) {
            launch_counters_publish(L.d_ctr, L.h_ctr_dev, s);
            SGS_CUDA(rec_done());
            return SGS_OK;
        }

        // K2: ranks and the rank-ordered binning inputs (depth_sort.cu)
        const uint32_t* order = L.order.as<uint32_t>();
        {
            const int log2c = depth_coarse_log2(n);
            const size_t half = align_up(depth_two_level_scratch(log2c), 256);
            SGS_CUDA(L.buckets.ensure(2 * half));  // histogram, offsets
            SGS_CUDA(L.keys_b.ensure(n1 * 16));  // K2's (key, index) partition
            SGS_CUDA(launch_depth_two_level(n, L.keys_a.as<unsigned long long>(), L.d_ctr, log2c,
                                            L.buckets.as<uint32_t>(), L.buckets.as<uint32_t>() + half / 4,
                                            L.keys_b.ptr, L.order.as<uint32_t>(), L.tk_a.as<uint32_t>(),
                                            L.rects.as<int4>(), L.brect.as<int4>(), L.bmeta.as<uint2>(), s,
                                            &ctx->own_launches));
        }
        if (timing) SGS_CUDA(cudaEventRecord(L.ev[2], s));

        // depth chunks over ranks (bounds known on the host: culled splats sort last and
        // contribute no tiles, so rank bounds can be taken over N)
        const std::vector<uint64_t> divs = ctx->chunk_divs_set ? ctx->chunk_divs : default_chunk_divs(n);
        const bool multi = mode == kRender && ctx->chunking && !divs.empty() && n >= kMinChunkedN &&
                           composite_pixel_chunks(cfg->tile_size) == 1;
        std::vector<uint64_t> bounds{0};
        if (multi) {
            for (uint64_t div : divs) {
                const uint64_t b = (n + div - 1) / div;
                if (b > bounds.back() && b < n) bounds.push_back(b);
            }
            // done, touched and part-done bitmaps
            const size_t flag_bytes = composite_flag_words(static_cast<uint32_t>(ntile)) * 4;
            SGS_CUDA(L.tile_done.ensure(flag_bytes));
            SGS_CUDA(L.pix_state.ensure(npx * sizeof(PixelState)));
            SGS_CUDA(L.pix_walked.ensure(npx * sizeof(uint32_t)));
            SGS_CUDA(cudaMemsetAsync(L.tile_done.ptr, 0, flag_bytes, s));
        }
        bounds.push_back(n);
        const int nchunks = static_cast<int>(bounds.size()) - 1;
        const float3 bg = make_float3(static_cast<float>(scene->meta.background[0]),
                                      static_cast<float>(scene->meta.background[1]),
                                      static_cast<float>(scene->meta.background[2]));
        const TileDigits td = tile_digits(std::max(1, ceil_log2(ntile)));
        const uint64_t work_cap = ntile * static_cast<uint64_t>(composite_work_items(cfg->tile_size));
        if (count_stats) SGS_CUDA(L.tile_emax.ensure(ntile * composite_pixel_chunks(cfg->tile_size) * 4));
        SGS_CUDA(L.work.ensure((7 * work_cap + 8) * sizeof(uint32_t)));  // 6 length classes, 8 control words, background items
        const unsigned long long* d_pc = &L.d_ctr->chunk_entries;
        for (int c = 0; c < nchunks; ++c) {
            const uint64_t rb = bounds[c], re = bounds[c + 1];
            const uint32_t* done = c > 0 ? L.tile_done.as<uint32_t>() : nullptr;
            if (timing) SGS_CUDA(cudaEventRecord(L.ev[3], s));
            // K3 + K4: (tile, index) pairs of the chunk's ranks, in rank order
            SGS_CUDA(launch_binning(rb, re, L.bmeta.as<uint2>(), L.brect.as<int4>(), done, kp.tiles_x,
                                    static_cast<int>(ntile), L.tk_a.as<uint32_t>(), L.tv_a.as<uint32_t>(),
                                    L.tkey_cap, L.bin_status.ptr, L.d_ctr, s, &ctx->own_launches));
            if (timing) SGS_CUDA(cudaEventRecord(L.ev[4], s));
            // K5: stable radix passes on the tile id (device-sized)
            uint32_t* tk = L.tk_a.as<uint32_t>();
            uint32_t* tv = L.tv_a.as<uint32_t>();
            uint32_t* tk2 = L.tk_b.as<uint32_t>();
            uint32_t* tv2 = L.tv_b.as<uint32_t>();
            for (int p = 0; p < td.passes; ++p) {
                SGS_CUDA(launch_radix_pass(tk, tv, tk2, tv2, d_pc, td.shift[p], td.bits[p], shist, s));
                std::swap(tk, tk2);
                std::swap(tv, tv2);
            }
            ctx->own_launches += 3 * td.passes;
            // K6
            SGS_CUDA(cudaMemsetAsync(L.ranges.ptr, 0, ntile * sizeof(uint2), s));
            launch_tile_ranges(d_pc, tk, L.ranges.as<uint2>(), s);
            SGS_CUDA(cudaGetLastError());
            ctx->own_launches += 1;
            const uint32_t* list = tv;  // the compositor's per-tile lists of Gaussian indices
            if (timing) SGS_CUDA(cudaEventRecord(L.ev[5], s));
            L.last_order = order;
            L.last_tiles = tk;
            L.last_list = tv;
            // Every decision the host acts on (device errors, depth-tie and tile-key
            // overflows) is final once the last chunk is binned: without stats the
            // counters are published here, so the host settles this frame and queues the
            // lane's next one while K7 still runs (K7 itself raises nothing).
            const bool early_done = mode == kRender && !j.stats && c == nchunks - 1;
            if (early_done) {
                launch_counters_publish(L.d_ctr, L.h_ctr_dev, s);
                SGS_CUDA(rec_done());
            }
            // K7
            if (mode == kRender) {
                SGS_CUDA(launch_composite(L.d_consts, cp, kp, L.ranges.as<uint2>(), list, L.rec.as<SplatRec>(),
                                          L.colour.as<float4>(), bg, L.pix_state.as<PixelState>(),
                                          L.pix_walked.as<uint32_t>(), L.tile_done.as<uint32_t>(), c == 0,
                                          c == nchunks - 1, L.d_ctr, count_stats, L.tile_emax.as<uint32_t>(),
                                          L.work.as<uint32_t>(),
                                          L.work.as<uint32_t>() + 6 * work_cap, s));
                ctx->own_launches += count_stats && c == nchunks - 1 ? 3 : 2;  // (+ work list, E_t sum)
            }
            if (timing) {
                SGS_CUDA(cudaEventRecord(L.ev[6], s));
                SGS_CUDA(cudaEventSynchronize(L.ev[6]));
                float a = 0, b = 0, d = 0;
                SGS_CUDA(cudaEventElapsedTime(&a, L.ev[3], L.ev[4]));
                SGS_CUDA(cudaEventElapsedTime(&b, L.ev[4], L.ev[5]));
                SGS_CUDA(cudaEventElapsedTime(&d, L.ev[5], L.ev[6]));
                j.ms_bin += a;
                j.ms_tsort += b;
                j.ms_comp += d;
            }
        }
        if (mode != kRender || j.stats) {  // (otherwise published before K7)
            launch_counters_publish(L.d_ctr, L.h_ctr_dev, s);
            SGS_CUDA(rec_done());
        }
        return SGS_OK;
    };
    const bool graph = ctx->graphs && mode == kRender && !timing && !tr && !j.d_debug;
    if (!graph) {
        sgs_status st = body();
        if (st != SGS_OK) return st;
    } else {
        sgs_status st = launch_frame_graph(ctx, L, cp, body, capturing);
        if (st != SGS_OK) return st;
    }
    if (timing) SGS_CUDA(cudaEventRecord(L.ev[7], s));
    if (tr) SGS_CUDA(cudaEventRecord(tr->ev[1], s));
    if (host_out) {
        cudaStream_t cs = L.copy_stream;
        SGS_CUDA(cudaEventRecord(L.rendered[slot], s));
        SGS_CUDA(cudaStreamWaitEvent(cs, L.rendered[slot], 0));
        if (j.h_rgb) SGS_CUDA(cudaMemcpyAsync(j.h_rgb, d_rgb, npx * 3 * sizeof(float), cudaMemcpyDeviceToHost, cs));
        if (j.h_T) SGS_CUDA(cudaMemcpyAsync(j.h_T, d_T, npx * sizeof(float), cudaMemcpyDeviceToHost, cs));
        SGS_CUDA(cudaEventRecord(L.copied[slot], cs));
        if (tr) SGS_CUDA(cudaEventRecord(tr->ev[2], cs));
    } else if (tr) {
        SGS_CUDA(cudaEventRecord(tr->ev[2], s));
    }
    return SGS_OK;
}

// Wait for lane L's frame and check it: SGS_OK / an error status, or kRetryGrow when
// the frame must be enqueued again.
int check_frame(Lane& L) {
    Lane::Job& j = L.job;
    SGS_CUDA(cudaEventSynchronize(L.done));
    const Counters& hc = *L.h_ctr;
    if (hc.err != ~0ULL) return device_error(hc.err, j.scene, &j.cfg);
    if (j.mode == kProjectOnly) return SGS_OK;
    if (hc.key_overflow) {
        if (L.tkey_cap >= kMaxSortKeys) return fail(SGS_ERR_OUT_OF_MEMORY, "more than 2^31 - 1 tile entries in one chunk");
        L.tkey_cap = std::min<uint64_t>(hc.max_chunk_entries + hc.max_chunk_entries / 4 + 1024, kMaxSortKeys);
        return kRetryGrow;
    }
    L.last_v = hc.visible;
    L.last_p = hc.chunk_entries;  // the (single) chunk's P for the debug dump
    if (sgs_render_stats* stats = j.stats) {
        stats->visible += hc.visible;
        stats->tile_entries += hc.tile_entries;
        stats->block_entries += hc.block_entries;
        stats->guard_hits += hc.guard_hits;
        if (stats->want_timing) {
            float k1 = 0, k2 = 0, total = 0;
            SGS_CUDA(cudaEventElapsedTime(&k1, L.ev[0], L.ev[1]));
            SGS_CUDA(cudaEventElapsedTime(&k2, L.ev[1], L.ev[2]));
            SGS_CUDA(cudaEventElapsedTime(&total, L.ev[0], L.ev[7]));
            stats->ms_preprocess += k1;
            stats->ms_depth_sort += k2;
            stats->ms_binning += j.ms_bin;
            stats->ms_tile_sort += j.ms_tsort;
            stats->ms_composite += j.ms_comp;
            stats->ms_total += total;
        }
    }
    return SGS_OK;
}

uint64_t lane_bytes(const Lane& L) {
    uint64_t b = 0;
    for (const DevBuf* d : {&L.keys_a, &L.keys_b, &L.buckets, &L.order, &L.rec, &L.colour, &L.rects, &L.brect,
                            &L.bmeta, &L.bin_status, &L.work, &L.tk_a, &L.tv_a, &L.tk_b, &L.tv_b, &L.sort_hist,
                            &L.ranges, &L.tile_done, &L.pix_state, &L.pix_walked, &L.tile_emax})
        b += d->bytes;
    return b;
}

// How many of the first `lanes` lanes can hold a frame's arenas -- about 170 B per
// Gaussian (K1's keys, records, rectangles and colours, K2's partition and ranks, the
// binning inputs, 2N tile pairs) and 32 B per pixel -- in the free HBM, less a tenth
// kept for the caller (at least one lane; sizes only ever grow, so lanes holding
// arenas count what they already have). A 60M-Gaussian scene takes ~10 GB per lane.
int lanes_that_fit(const sgs_context* ctx, uint64_t n, uint64_t npx, int lanes) {
    const uint64_t per_lane = n * 170 + npx * 32 + (uint64_t{64} << 20);
    // (the free-memory query costs time: only large scenes ask)
    if (lanes <= 1 || per_lane * static_cast<uint64_t>(lanes) <= ctx->hbm_bytes / 4) return lanes;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return lanes;
    }
    uint64_t budget = free_b - free_b / 10;
    int k = 0;
    for (; k < lanes; ++k) {
        const uint64_t held = lane_bytes(ctx->lane[k]);
        const uint64_t need = per_lane > held ? per_lane - held : 0;
        if (k > 0 && need > budget) break;
        budget -= std::min(budget, need);
    }
    return std::max(k, 1);
}

// Settle lane L's frame: check it, re-enqueue on a retry verdict, until it is done.
sgs_status finish_frame(sgs_context* ctx, Lane& L) {
    if (!L.busy) return SGS_OK;
    for (int attempt = 0; attempt < 4; ++attempt) {
        const int rc = check_frame(L);
        if (rc == kRetryGrow) {
            sgs_status st = enqueue_frame(ctx, L);
            if (st != SGS_OK) {
                L.busy = false;
                return st;
            }
            continue;
        }
        L.busy = false;
        return static_cast<sgs_status>(rc);
    }
    L.busy = false;
    return fail(SGS_ERR_INTERNAL, "frame did not converge after re-sizing");
}

// Start a frame on lane L (which must be idle).
sgs_status start_frame(sgs_context* ctx, Lane& L, const sgs_scene* scene, const sgs_camera* cam,
                       const sgs_render_config* cfg, float* d_rgb, float* d_T, float* h_rgb, float* h_T,
                       sgs_render_stats* stats, DebugSplat* d_debug, FrameMode mode) {
    if (cfg->tile_size < 1) return fail(SGS_ERR_INVALID_ARGUMENT, "tile_size must be >= 1");
    sgs_status st = validate_camera(cam);
    if (st != SGS_OK) return st;
    Lane::Job& j = L.job;
    j = Lane::Job{};
    j.scene = scene;
    j.cam = *cam;
    j.cfg = *cfg;
    j.d_rgb = d_rgb;
    j.d_T = d_T;
    j.h_rgb = h_rgb;
    j.h_T = h_T;
    j.stats = stats;
    j.d_debug = d_debug;
    j.mode = mode;
    L.busy = true;
    st = enqueue_frame(ctx, L);
    if (st != SGS_OK) {
        cudaStreamSynchronize(L.stream);
        L.busy = false;
    }
    return st;
}

// Host-frame batches run the lanes on their ranked streams (lane k at priority
// greatest + k): earlier lanes' frames finish first, so the copy engines start
// draining frames early and stay busy, instead of all lanes finishing together and
// their copies piling up at the end of the batch. Measured at config C: e2e 1149 ->
// 1198 frames/s; device-resident batches keep the plain streams (1596 vs 1550).
sgs_status select_lane_streams(sgs_context* ctx, bool ranked) {
    for (Lane& L : ctx->lane) {
        cudaStream_t want = ranked && ctx->rank_host ? L.ranked : L.plain;
        if (L.stream == want) continue;
        SGS_CUDA(cudaEventRecord(L.swap, L.stream));  // the lane's arenas: in order across the swap
        SGS_CUDA(cudaStreamWaitEvent(want, L.swap, 0));
        L.stream = want;
    }
    return SGS_OK;
}

// Lanes start after the work already queued on the caller's stream ...
sgs_status fork_lanes(sgs_context* ctx, int lanes) {
    SGS_CUDA(cudaEventRecord(ctx->fork, ctx->stream));
    for (int k = 0; k < lanes; ++k) SGS_CUDA(cudaStreamWaitEvent(ctx->lane[k].stream, ctx->fork, 0));
    return SGS_OK;
}

// ... and the caller's stream continues after every lane's last frame.
sgs_status join_lanes(sgs_context* ctx, int lanes) {
    for (int k = 0; k < lanes; ++k) {
        Lane& L = ctx->lane[k];
        if (L.busy) finish_frame(ctx, L);
        SGS_CUDA(cudaEventRecord(L.done, L.stream));
        SGS_CUDA(cudaStreamWaitEvent(ctx->stream, L.done, 0));
    }
    return SGS_OK;
}

// One frame on lane 0, synchronously (projection / debug dumps).
sgs_status run_frame(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam, const sgs_render_config* cfg,
                     DebugSplat* d_debug, FrameMode mode) {
    sgs_status st = fork_lanes(ctx, 1);
    if (st != SGS_OK) return st;
    st = start_frame(ctx, ctx->lane[0], scene, cam, cfg, nullptr, nullptr, nullptr, nullptr, nullptr, d_debug, mode);
    if (st == SGS_OK) st = finish_frame(ctx, ctx->lane[0]);
    sgs_status sj = join_lanes(ctx, 1);
    return st != SGS_OK ? st : sj;
}


// ---------------------------------------------------------------------------
// Scene layout and upload.

struct Layout {
    size_t geo_off[11];
    size_t color_off;
    size_t color64_off;  // FP64 colour copies (meta.color_f64)
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
    L.color64_off = off;
    if (m.color_f64) off = align_up(off + static_cast<size_t>(color_param_count_impl(m.kind, m.sh_degree)) * n * 8, 256);
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
    p.color64 = m.color_f64 ? reinterpret_cast<const double*>(base + L.color64_off) : nullptr;
    for (int k = 0; k < 3; ++k) p.cov[k] = sc->cov.ptr ? sc->cov.as<double2>() + k * m.count : nullptr;
    for (int k = 0; k < 9; ++k) p.axes[k] = static_cast<float>(m.shared_axes[k]);
    for (int k = 0; k < 3; ++k) p.bg[k] = static_cast<float>(m.background[k]);
}

// Bind the planes and build the per-scene covariance cache from them, on `stream`
// after the work already queued there (the blob's producer), then wait for it.
sgs_status bind_and_cache(sgs_scene* sc, cudaStream_t stream) {
    SGS_CUDA(sc->cov.ensure(std::max<size_t>(sc->meta.count, 1) * 3 * sizeof(double2)));
    bind_planes(sc);
    launch_cov3d(sc->planes, sc->cov.as<double2>(), stream);
    SGS_CUDA(cudaGetLastError());
    SGS_CUDA(cudaStreamSynchronize(stream));
    return SGS_OK;
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
    parallel_for(n, [&](size_t i0, size_t i1) {
    std::vector<float> c(static_cast<size_t>(L.color_planes) * 4);
    for (size_t i = i0; i < i1; ++i) {
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
                // plane 0 (diffuse rgb, log_lambda), plane 1 (alpha rgb, 0), plane 2 (mu/|mu|, 0),
                // plane 3 (raw mu, 0);
                // mu normalised in FP64 exactly as DiffuseSGModel::lobe (color.cpp:49-56)
                for (int k = 0; k < 3; ++k) c[k] = static_cast<float>(param_at(d, co + k));
                c[3] = static_cast<float>(param_at(d, co + 6));
                for (int k = 0; k < 3; ++k) c[4 + k] = static_cast<float>(param_at(d, co + 3 + k));
                const double mu[3] = {param_at(d, co + 7), param_at(d, co + 8), param_at(d, co + 9)};
                const double nn = std::sqrt((mu[0] * mu[0] + mu[1] * mu[1]) + mu[2] * mu[2]);
                for (int k = 0; k < 3; ++k)
                    c[8 + k] = static_cast<float>(nn > 1e-12 ? mu[k] / nn : (k == 0 ? 1.0 : 0.0));
                for (int k = 0; k < 3; ++k) c[12 + k] = static_cast<float>(mu[k]);  // raw axis (backward)
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
        if (m.color_f64) {
            double* c64 = reinterpret_cast<double*>(base + L.color64_off);
            for (int k = 0; k < cpc; ++k) c64[static_cast<size_t>(k) * n + i] = param_at(d, co + k);
        }
    }
    });
}

cudaError_t upload_rows_f32(sgs_context* ctx, const sgs_scene_desc* desc, const sgs_scene_meta& m, void* blob);

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
    cudaError_t e = cudaSuccess;
    if (desc->dtype == SGS_F32 && m.count) {
        // float32 rows go to the device as they are and a kernel scatters them into the
        // planes (the PLY loader's path with an identity column map)
        e = upload_rows_f32(ctx, desc, m, sc->blob);
    } else {
        std::vector<char> host;
        fill_blob(desc, m, host);
        e = cudaMemcpy(sc->blob, host.data(), host.size(), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        delete sc;
        return fail(SGS_ERR_CUDA, std::string("scene upload: ") + cudaGetErrorString(e));
    }
    st = bind_and_cache(sc, ctx->stream);
    if (st != SGS_OK) {
        sgs_scene_free(sc);
        return st;
    }
    *out = sc;
    return SGS_OK;
}

// ---------------------------------------------------------------------------
// PLY rows -> scene planes (sgs_scene_load_ply). tab[s] gives, for every float slot
// s of the 3 geometry planes and the colour planes, the row column it copies
// (>= 0), zero (-1), or component k of the FP64-normalised SG1 lobe axis (-2 - k),
// exactly as fill_blob lays out the flat parameters.
constexpr int kPlyMaxSlots = 4 * (3 + 12);

__global__ void ply_rows_kernel(uint64_t n, const float* __restrict__ rows, int stride, int nslots,
                                const int32_t* __restrict__ tab, int mu_col, float4* __restrict__ g0,
                                float4* __restrict__ g1, float4* __restrict__ g2, float4* __restrict__ color) {
    __shared__ int32_t s_tab[kPlyMaxSlots];
    for (int k = threadIdx.x; k < nslots; k += blockDim.x) s_tab[k] = tab[k];
    __syncthreads();
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* row = rows + i * static_cast<uint64_t>(stride);
    float mu[3] = {0.f, 0.f, 0.f};
    if (mu_col >= 0) {
        // DiffuseSGModel::lobe (color.cpp:52-59): mu / |mu| in FP64, (1, 0, 0) if |mu| <= 1e-12
        const double m0 = row[mu_col], m1 = row[mu_col + 1], m2 = row[mu_col + 2];
        const double nn = __dsqrt_rn(sgs::dadd(sgs::dadd(sgs::dmul(m0, m0), sgs::dmul(m1, m1)), sgs::dmul(m2, m2)));
        if (nn > 1e-12) {
            mu[0] = static_cast<float>(sgs::ddiv(m0, nn));
            mu[1] = static_cast<float>(sgs::ddiv(m1, nn));
            mu[2] = static_cast<float>(sgs::ddiv(m2, nn));
        } else {
            mu[0] = 1.f;
        }
    }
    for (int p = 0; p < nslots / 4; ++p) {
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = s_tab[4 * p + q];
            v[q] = t >= 0 ? row[t] : (t == -1 ? 0.f : mu[-2 - t]);
        }
        const float4 f = make_float4(v[0], v[1], v[2], v[3]);
        if (p < 3)
            (p == 0 ? g0 : p == 1 ? g1 : g2)[i] = f;
        else
            color[static_cast<uint64_t>(p - 3) * n + i] = f;
    }
}

// The slot table for a resolved checkpoint (mirrors fill_blob's flat -> plane map).
std::vector<int32_t> ply_slot_table(const PlyTable& t, int color_planes, int* mu_col) {
    const std::vector<int32_t>& src = t.src;  // flat parameter -> row column
    std::vector<int32_t> tab(static_cast<size_t>(4 * (3 + color_planes)), -1);
    auto flat = [&](int p) { return src[static_cast<size_t>(p)]; };
    // geometry: (pos, opacity), quaternion, (log scale, 0)
    for (int k = 0; k < 3; ++k) tab[static_cast<size_t>(k)] = flat(k);
    tab[3] = flat(10);
    for (int k = 0; k < 4; ++k) tab[static_cast<size_t>(4 + k)] = flat(3 + k);
    for (int k = 0; k < 3; ++k) tab[static_cast<size_t>(8 + k)] = flat(7 + k);
    int32_t* c = tab.data() + 12;
    const int co = 11;
    const int cpc = color_param_count_impl(t.info.kind, t.info.sh_degree);
    *mu_col = -1;
    switch (t.info.kind) {
        case SGS_SH:
            for (int k = 0; k < cpc; ++k) c[k] = flat(co + k);
            break;
        case SGS_MIXED: {
            const int nsh = 3 * (t.info.sh_degree + 1) * (t.info.sh_degree + 1);
            for (int k = 0; k < nsh; ++k) c[k] = flat(co + k);
            const int lobe_base = 4 * ((nsh + 3) / 4);
            for (int k = 0; k < 12; ++k) c[lobe_base + k] = flat(co + nsh + k);
            break;
        }
        case SGS_SG1:
            for (int k = 0; k < 3; ++k) c[k] = flat(co + k);
            c[3] = flat(co + 6);
            for (int k = 0; k < 3; ++k) c[4 + k] = flat(co + 3 + k);
            for (int k = 0; k < 3; ++k) c[8 + k] = -2 - k;
            for (int k = 0; k < 3; ++k) c[12 + k] = flat(co + 7 + k);  // raw axis (backward)
            *mu_col = flat(co + 7);
            break;
        case SGS_SG3:
            for (int k = 0; k < 3; ++k) c[k] = flat(co + k);
            for (int k = 0; k < 12; ++k) c[4 + k] = flat(co + 3 + k);
            break;
    }
    return tab;
}

// An SGS_F32 description's rows (count x (11 + colour params) floats, Scene::param
// order) into the planes of blob: one copy of the rows, then ply_rows_kernel with the
// identity column map (SG1 lobe axes normalised in FP64 as at every upload).
cudaError_t rows_to_planes(sgs_context* ctx, const sgs_scene_meta& m, void* blob);

cudaError_t upload_rows_f32(sgs_context* ctx, const sgs_scene_desc* desc, const sgs_scene_meta& m, void* blob) {
    const size_t nfloat = static_cast<size_t>(m.count) * static_cast<size_t>(11 + color_param_count_impl(m.kind, m.sh_degree));
    cudaError_t e = ctx->rows.ensure(nfloat * sizeof(float));
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(ctx->rows.ptr, desc->params, nfloat * sizeof(float), cudaMemcpyHostToDevice, ctx->stream);
    return e == cudaSuccess ? rows_to_planes(ctx, m, blob) : e;
}

// The float32 rows in ctx->rows into the planes of blob.
cudaError_t rows_to_planes(sgs_context* ctx, const sgs_scene_meta& m, void* blob) {
    PlyTable t;
    t.count = m.count;
    t.info.kind = m.kind;
    t.info.sh_degree = m.sh_degree;
    const int stride = 11 + color_param_count_impl(m.kind, m.sh_degree);
    t.src.resize(static_cast<size_t>(stride));
    for (int k = 0; k < stride; ++k) t.src[static_cast<size_t>(k)] = k;
    const Layout L = make_layout(m);
    int mu_col = -1;
    const std::vector<int32_t> tab = ply_slot_table(t, L.color_planes, &mu_col);
    DevBuf& d_rows = ctx->rows;
    DevBuf d_tab;
    cudaStream_t s = ctx->stream;
    cudaError_t e = d_tab.ensure(tab.size() * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMemsetAsync(blob, 0, m.blob_bytes, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_tab.ptr, tab.data(), tab.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        char* base = static_cast<char*>(blob);
        ply_rows_kernel<<<static_cast<unsigned>((m.count + 255) / 256), 256, 0, s>>>(
            m.count, d_rows.as<float>(), stride, static_cast<int>(tab.size()), d_tab.as<int32_t>(), mu_col,
            reinterpret_cast<float4*>(base + L.geo_off[0]), reinterpret_cast<float4*>(base + L.geo_off[1]),
            reinterpret_cast<float4*>(base + L.geo_off[2]), reinterpret_cast<float4*>(base + L.color_off));
        e = cudaGetLastError();
        if (e == cudaSuccess) ctx->own_launches += 1;
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    d_tab.release();
    return e;
}

}  // namespace

// ---------------------------------------------------------------------------
// Helpers for group.cu (sgs_internal.h).
namespace sgs {
sgs_status fail_status(sgs_status code, const std::string& msg) { return fail(code, msg); }
int context_device(const sgs_context* ctx) { return ctx->device; }
void context_stream(const sgs_context* ctx, cudaStream_t* stream) { *stream = ctx->stream; }
sgs_status scene_bind_owned(sgs_context* ctx, const sgs_scene_meta* meta, void* blob, uint64_t bytes,
                            sgs_scene** out) {
    sgs_status st = sgs_scene_bind(ctx, meta, blob, bytes, out);
    if (st == SGS_OK) {  // the scene frees the blob with itself
        (*out)->owned.ptr = blob;
        (*out)->owned.bytes = bytes;
    }
    return st;
}
}  // namespace sgs

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
    {
        cudaDeviceProp prop{};
        SGS_CUDA(cudaGetDeviceProperties(&prop, device));
        ctx->hbm_bytes = prop.totalGlobalMem;
    }
    SGS_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;
    SGS_CUDA(cudaMallocHost(&ctx->h_ctr_init, sizeof(Counters)));
    std::memset(ctx->h_ctr_init, 0, sizeof(Counters));
    ctx->h_ctr_init->err = ~0ULL;
    ctx->h_ctr_init->kmin = ~0ULL;
    SGS_CUDA(cudaEventCreateWithFlags(&ctx->fork, cudaEventDisableTiming));
    int prio_least = 0, prio_greatest = 0;
    SGS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
    int lane_k = 0;
    for (Lane& L : ctx->lane) {
        // the ranked stream of lane k runs at priority greatest + k (host-frame batches)
        SGS_CUDA(cudaStreamCreateWithFlags(&L.plain, cudaStreamNonBlocking));
        SGS_CUDA(cudaStreamCreateWithPriority(&L.ranked, cudaStreamNonBlocking,
                                              std::min(prio_least, prio_greatest + lane_k++)));
        SGS_CUDA(cudaEventCreateWithFlags(&L.swap, cudaEventDisableTiming));
        L.stream = L.plain;
        SGS_CUDA(cudaMalloc(&L.d_ctr, sizeof(Counters)));
        SGS_CUDA(cudaHostAlloc(&L.h_ctr, sizeof(Counters), cudaHostAllocMapped));
        SGS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&L.h_ctr_dev), L.h_ctr, 0));
        SGS_CUDA(cudaMalloc(&L.d_consts, sizeof(FrameConsts)));
        SGS_CUDA(cudaMallocHost(&L.h_consts, sizeof(FrameConsts)));
        for (auto& ev : L.ev) SGS_CUDA(cudaEventCreate(&ev));
        SGS_CUDA(cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming));
        SGS_CUDA(cudaStreamCreateWithFlags(&L.copy_stream, cudaStreamNonBlocking));
        for (int k = 0; k < Lane::kOutSlots; ++k) {
            SGS_CUDA(cudaEventCreateWithFlags(&L.rendered[k], cudaEventDisableTiming));
            SGS_CUDA(cudaEventCreateWithFlags(&L.copied[k], cudaEventDisableTiming));
        }
    }
    if (const char* e = std::getenv("SGS_GRAPHS")) ctx->graphs = std::atoi(e) != 0;
    if (const char* e = std::getenv("SGS_TIGHT_RECT")) ctx->tight_rect = std::atoi(e) != 0;
    if (const char* e = std::getenv("SGS_RANK_HOST")) ctx->rank_host = std::atoi(e) != 0;
    if (const char* e = std::getenv("SGS_TRACE")) ctx->trace = std::atoi(e) != 0;
    if (const char* e = std::getenv("SGS_DEBUG_CAPTURE_FAIL")) ctx->debug_capture_fail = std::atoi(e) != 0;
    if (const char* e = std::getenv("SGS_LANES")) ctx->lanes = std::min(std::max(std::atoi(e), 1), kLanes);
    if (const char* e = std::getenv("SGS_HOST_LANES")) ctx->host_lanes = std::min(std::max(std::atoi(e), 1), kLanes);
    if (const char* e = std::getenv("SGS_DEPTH_CHUNKING")) ctx->chunking = std::atoi(e) != 0;
    if (const char* e = std::getenv("SGS_DEPTH_CHUNKS")) {  // e.g. "16,4": boundaries at N/16, N/4
        ctx->chunk_divs.clear();
        ctx->chunk_divs_set = true;
        for (const char* q = e; *q;) {
            char* endp = nullptr;
            const long v = std::strtol(q, &endp, 10);
            if (endp == q) break;
            if (v > 1) ctx->chunk_divs.push_back(static_cast<uint64_t>(v));
            q = *endp ? endp + 1 : endp;
        }
    }
    *out = ctx;
    return SGS_OK;
}

void sgs_destroy(sgs_context* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (Lane& L : ctx->lane) {
        if (L.stream) cudaStreamSynchronize(L.stream);
        for (DevBuf* b : {&L.keys_a, &L.keys_b, &L.buckets, &L.order, &L.rec, &L.colour, &L.rects, &L.brect, &L.bmeta, &L.bin_status,
                          &L.work, &L.tk_a, &L.tv_a, &L.tk_b, &L.tv_b, &L.sort_hist, &L.ranges,
                          &L.tile_done, &L.pix_state, &L.pix_walked, &L.tile_emax})
            b->release();
        if (L.d_ctr) cudaFree(L.d_ctr);
        if (L.h_ctr) cudaFreeHost(L.h_ctr);
        if (L.d_consts) cudaFree(L.d_consts);
        if (L.h_consts) cudaFreeHost(L.h_consts);
        for (auto& ev : L.ev)
            if (ev) cudaEventDestroy(ev);
        if (L.done) cudaEventDestroy(L.done);
        if (L.copy_stream) {
            cudaStreamSynchronize(L.copy_stream);
            cudaStreamDestroy(L.copy_stream);
        }
        for (int k = 0; k < Lane::kOutSlots; ++k) {
            L.out_rgb[k].release();
            L.out_T[k].release();
            if (L.rendered[k]) cudaEventDestroy(L.rendered[k]);
            if (L.copied[k]) cudaEventDestroy(L.copied[k]);
        }
        if (L.gexec) cudaGraphExecDestroy(L.gexec);
        if (L.graph) cudaGraphDestroy(L.graph);
        if (L.grec) k1_record_free(L.grec);
        if (L.plain) cudaStreamDestroy(L.plain);
        if (L.ranked) cudaStreamDestroy(L.ranked);
        if (L.swap) cudaEventDestroy(L.swap);
    }
    ctx->metrics.release();
    ctx->rows.release();
    for (int b = 0; b < 2; ++b) {
        if (ctx->stage[b]) cudaFreeHost(ctx->stage[b]);
        if (ctx->stage_ev[b]) cudaEventDestroy(ctx->stage_ev[b]);
    }
    ctx->bwd.release();
    if (ctx->h_ctr_init) cudaFreeHost(ctx->h_ctr_init);
    if (ctx->fork) cudaEventDestroy(ctx->fork);
    cudaStreamDestroy(ctx->own_stream);
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
    for (Lane& L : ctx->lane) {
        SGS_CUDA(cudaStreamSynchronize(L.stream));
        SGS_CUDA(cudaStreamSynchronize(L.copy_stream));
    }
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

sgs_status sgs_host_alloc(uint64_t bytes, void** out) {
    if (!out) return fail(SGS_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    SGS_CUDA(cudaHostAlloc(out, std::max<uint64_t>(bytes, 1), cudaHostAllocDefault));
    return SGS_OK;
}

void sgs_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

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
        std::atomic<int> any{0};
        parallel_for(d->count, [&](size_t i0, size_t i1) {
            for (size_t i = i0; i < i1 && !any.load(std::memory_order_relaxed); ++i)
                for (int k = 0; k < 11; ++k) {
                    const double v = p[i * stride + k];
                    if (static_cast<double>(static_cast<float>(v)) != v) {
                        any.store(1, std::memory_order_relaxed);
                        break;
                    }
                }
        });
        f64 = any.load();
    }
    m->geometry_f64 = f64;
    // colour: the float planes feed the FP32 compositor; FP64 copies are added when
    // some colour parameter is not f32-exact (the exact mode and the backward read them)
    int cf64 = 0;
    if (d->dtype == SGS_F64) {
        const int cpc = color_param_count_impl(d->kind, deg);
        const size_t stride = 11 + static_cast<size_t>(cpc);
        const double* p = static_cast<const double*>(d->params);
        std::atomic<int> any{0};
        parallel_for(d->count, [&](size_t i0, size_t i1) {
            for (size_t i = i0; i < i1 && !any.load(std::memory_order_relaxed); ++i)
                for (int k = 0; k < cpc; ++k) {
                    const double v = p[i * stride + 11 + k];
                    if (static_cast<double>(static_cast<float>(v)) != v) {
                        any.store(1, std::memory_order_relaxed);
                        break;
                    }
                }
        });
        cf64 = any.load();
    }
    m->color_f64 = cf64;
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
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    sgs_status st = bind_and_cache(sc, ctx->stream);
    if (st != SGS_OK) {
        sgs_scene_free(sc);
        return st;
    }
    *out = sc;
    return SGS_OK;
}

sgs_status sgs_scene_refresh(sgs_context* ctx, sgs_scene* scene) {
    if (!ctx || !scene) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    return bind_and_cache(scene, ctx->stream);
}

sgs_status sgs_scene_update(sgs_context* ctx, sgs_scene* scene, const sgs_scene_desc* desc) {
    if (!ctx || !scene || !desc) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    sgs_scene_meta m{};
    sgs_status st = sgs_scene_plan(desc, &m);
    if (st != SGS_OK) return st;
    const sgs_scene_meta& o = scene->meta;
    if (m.count != o.count || m.kind != o.kind || m.sh_degree != o.sh_degree || m.geometry_f64 != o.geometry_f64 ||
        m.color_f64 != o.color_f64 || m.blob_bytes != o.blob_bytes)
        return fail(SGS_ERR_INVALID_ARGUMENT, "scene update changes the device layout");
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    cudaError_t e = cudaSuccess;
    if (desc->dtype == SGS_F32 && m.count) {
        e = upload_rows_f32(ctx, desc, m, scene->blob);
    } else {
        std::vector<char> host;
        fill_blob(desc, m, host);
        e = cudaMemcpy(scene->blob, host.data(), host.size(), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) return fail(SGS_ERR_CUDA, std::string("scene update: ") + cudaGetErrorString(e));
    scene->meta = m;  // (axes and background may change)
    return bind_and_cache(scene, ctx->stream);
}

sgs_status sgs_scene_update_rows(sgs_context* ctx, sgs_scene* scene, const sgs_scene_desc* desc,
                                 sgs_row_fill_fn fill, void* user) {
    if (!ctx || !scene || !desc || !fill) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    if (desc->dtype != SGS_F32) return fail(SGS_ERR_INVALID_ARGUMENT, "streamed rows are float32 (SGS_F32)");
    sgs_scene_desc d = *desc;
    float unused = 0.0f;
    if (!d.params) d.params = &unused;  // (the rows come from fill)
    sgs_scene_meta m{};
    sgs_status st = sgs_scene_plan(&d, &m);
    if (st != SGS_OK) return st;
    const sgs_scene_meta& o = scene->meta;
    if (m.count != o.count || m.kind != o.kind || m.sh_degree != o.sh_degree || m.geometry_f64 != o.geometry_f64 ||
        m.color_f64 != o.color_f64 || m.blob_bytes != o.blob_bytes)
        return fail(SGS_ERR_INVALID_ARGUMENT, "scene update changes the device layout");
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const uint64_t stride = 11 + static_cast<uint64_t>(color_param_count_impl(m.kind, m.sh_degree));
    if (m.count) {
        // ~64 MB blocks: a few fills per scene, each copy hidden behind the next fill
        constexpr size_t kBlockBytes = size_t{64} << 20;
        const uint64_t per = std::max<uint64_t>(1, kBlockBytes / (stride * sizeof(float)));
        const size_t block_bytes = static_cast<size_t>(std::min<uint64_t>(per, m.count) * stride * sizeof(float));
        if (ctx->stage_bytes < block_bytes) {
            for (int b = 0; b < 2; ++b) {
                if (ctx->stage[b]) SGS_CUDA(cudaFreeHost(ctx->stage[b]));
                ctx->stage[b] = nullptr;
            }
            ctx->stage_bytes = 0;
            for (int b = 0; b < 2; ++b) SGS_CUDA(cudaHostAlloc(&ctx->stage[b], block_bytes, cudaHostAllocDefault));
            ctx->stage_bytes = block_bytes;
        }
        for (int b = 0; b < 2; ++b)
            if (!ctx->stage_ev[b]) SGS_CUDA(cudaEventCreateWithFlags(&ctx->stage_ev[b], cudaEventDisableTiming));
        SGS_CUDA(ctx->rows.ensure(m.count * stride * sizeof(float)));
        float* d_rows = ctx->rows.as<float>();
        uint64_t k = 0;
        for (uint64_t first = 0; first < m.count; first += per, ++k) {
            const uint64_t cnt = std::min<uint64_t>(per, m.count - first);
            float* buf = static_cast<float*>(ctx->stage[k & 1]);
            if (k >= 2) SGS_CUDA(cudaEventSynchronize(ctx->stage_ev[k & 1]));  // its previous copy left
            if (fill(user, buf, first, cnt) != 0) {
                SGS_CUDA(cudaStreamSynchronize(s));  // (the scene's blob was not touched)
                return fail(SGS_ERR_INVALID_ARGUMENT, "scene update aborted by the row producer");
            }
            SGS_CUDA(cudaMemcpyAsync(d_rows + first * stride, buf, cnt * stride * sizeof(float),
                                     cudaMemcpyHostToDevice, s));
            SGS_CUDA(cudaEventRecord(ctx->stage_ev[k & 1], s));
        }
        const cudaError_t e = rows_to_planes(ctx, m, scene->blob);
        if (e != cudaSuccess) return fail(SGS_ERR_CUDA, std::string("scene update: ") + cudaGetErrorString(e));
    }
    scene->meta = m;  // (axes and background may change)
    return bind_and_cache(scene, s);
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
    scene->cov.release();
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
    const bool host = out_memory != SGS_DEVICE;
    const bool timing = stats && stats->want_timing;
    auto outs = [&](int i, float** d_rgb, float** d_T, float** h_rgb, float** h_T) {
        float* o_rgb = rgb ? rgb + i * npx * 3 : nullptr;
        float* o_T = T ? T + i * npx : nullptr;
        *d_rgb = host ? nullptr : o_rgb;
        *d_T = host ? nullptr : o_T;
        *h_rgb = host ? o_rgb : nullptr;
        *h_T = host ? o_T : nullptr;
    };
    sgs_status st = select_lane_streams(ctx, host && n > 1);
    if (st != SGS_OK) return st;
    // per-stage timing reads events mid-frame: one lane keeps the stages unmixed; very
    // large scenes get as many lanes as their arenas fit in HBM
    const int lanes = lanes_that_fit(ctx, scene->meta.count, npx,
                                     std::min<int>(timing ? 1 : (host ? ctx->host_lanes : ctx->lanes), n));
    st = fork_lanes(ctx, lanes);
    if (st != SGS_OK) return st;
    // view i runs on lane i % lanes; a lane's previous view is settled (checked,
    // retried if needed) before the lane is reused, so views complete in order
    for (int i = 0; i < n && st == SGS_OK; ++i) {
        Lane& L = ctx->lane[i % lanes];
        st = finish_frame(ctx, L);
        if (st != SGS_OK) break;
        float *drgb, *dT, *hrgb, *hT;
        outs(i, &drgb, &dT, &hrgb, &hT);
        st = start_frame(ctx, L, scene, &cams[i], cfg, drgb, dT, hrgb, hT, stats, nullptr, kRender);
    }
    for (int k = 0; k < lanes; ++k) {  // settle the views still in flight, in order
        Lane& L = ctx->lane[(n + k) % lanes];
        sgs_status sk = finish_frame(ctx, L);
        if (st == SGS_OK) st = sk;
    }
    sgs_status sj = join_lanes(ctx, lanes);
    // host frames are complete (or abandoned, on an error) once the copies drained
    if (host)
        for (int k = 0; k < lanes; ++k) cudaStreamSynchronize(ctx->lane[k].copy_stream);
    if (ctx->trace && !ctx->trace_recs.empty()) {
        cudaDeviceSynchronize();
        const cudaEvent_t t0 = ctx->trace_recs.front().ev[0];
        std::fprintf(stderr, "sgs trace: frame lane start_ms composite_done_ms copies_done_ms\n");
        int f = 0;
        for (auto& r : ctx->trace_recs) {
            float a = 0, b = 0, c = 0;
            cudaEventElapsedTime(&a, t0, r.ev[0]);
            cudaEventElapsedTime(&b, t0, r.ev[1]);
            cudaEventElapsedTime(&c, t0, r.ev[2]);
            std::fprintf(stderr, "sgs trace: %d %d %.3f %.3f %.3f\n", f++, r.lane, a, b, c);
        }
        for (auto& r : ctx->trace_recs)
            for (auto& e : r.ev) cudaEventDestroy(e);
        ctx->trace_recs.clear();
    }
    if (st != SGS_OK) return st;
    if (sj != SGS_OK) return sj;
    // frames are settled once binned; the call returns with every frame composited
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
    sgs_status st = run_frame(ctx, scene, cam, cfg, d_dbg, kProjectOnly);
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
    sgs_status st = run_frame(ctx, scene, cam, cfg, nullptr, kTileGrid);
    if (st != SGS_OK) return st;
    const Lane& L = ctx->lane[0];
    SGS_CUDA(cudaStreamSynchronize(L.stream));
    const uint64_t v = L.last_v, p = L.last_p;
    *n_visible = v;
    *n_entries = p;
    std::vector<uint32_t> ord(v);
    if (v) SGS_CUDA(cudaMemcpy(ord.data(), L.last_order, v * 4, cudaMemcpyDeviceToHost));
    if (order && v) std::memcpy(order, ord.data(), v * 4);
    if (!offsets && !entries) return SGS_OK;
    std::vector<uint32_t> tiles(p), list(p);
    if (p) SGS_CUDA(cudaMemcpy(tiles.data(), L.last_tiles, p * 4, cudaMemcpyDeviceToHost));
    if (p) SGS_CUDA(cudaMemcpy(list.data(), L.last_list, p * 4, cudaMemcpyDeviceToHost));
    const uint64_t ntile = static_cast<uint64_t>((cam->width + cfg->tile_size - 1) / cfg->tile_size) *
                           static_cast<uint64_t>((cam->height + cfg->tile_size - 1) / cfg->tile_size);
    if (offsets) {
        std::vector<uint64_t> cnt(ntile + 1, 0);
        for (uint64_t i = 0; i < p; ++i) cnt[tiles[i]]++;
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
        for (uint64_t i = 0; i < p && i < capacity; ++i) entries[i] = rank_of[list[i]];
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

sgs_status sgs_ply_read(const char* path, sgs_ply_info* info, double* params, uint64_t params_capacity) {
    if (!path || !info) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    PlyTable t;
    std::string err;
    int st = ply_parse_header(path, t, err);
    if (st != SGS_OK) return fail(static_cast<sgs_status>(st), err);
    std::vector<float> rows;
    if (params) {
        rows.resize(static_cast<size_t>(t.count) * t.props.size());
        st = ply_read_rows(t, rows.data(), err);
    } else {
        st = ply_check_payload(t, err);
    }
    if (st != SGS_OK) return fail(static_cast<sgs_status>(st), err);
    st = ply_resolve(t, err);
    if (st != SGS_OK) return fail(static_cast<sgs_status>(st), err);
    *info = t.info;
    if (params) {
        if (params_capacity < t.count * t.src.size())
            return fail(SGS_ERR_INVALID_ARGUMENT, "params buffer smaller than count * (11 + colour params)");
        ply_rows_to_flat(t, rows.data(), params);
    }
    return SGS_OK;
}

sgs_status sgs_scene_load_ply(sgs_context* ctx, const char* path, sgs_ply_info* info, sgs_scene** out) {
    if (!ctx || !path || !out) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    PlyTable t;
    std::string err;
    int st = ply_parse_header(path, t, err);
    if (st != SGS_OK) return fail(static_cast<sgs_status>(st), err);
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    const size_t nfloat = static_cast<size_t>(t.count) * t.props.size();
    float* h_rows = nullptr;  // pinned: the payload is read straight into DMA-able memory
    SGS_CUDA(cudaMallocHost(&h_rows, std::max<size_t>(nfloat, 1) * sizeof(float)));
    st = ply_read_rows(t, h_rows, err);
    if (st == SGS_OK) st = ply_resolve(t, err);
    if (st != SGS_OK) {
        cudaFreeHost(h_rows);
        return fail(static_cast<sgs_status>(st), err);
    }
    sgs_scene_meta m{};
    m.count = t.count;
    m.kind = t.info.kind;
    m.sh_degree = t.info.sh_degree;
    m.geometry_f64 = 0;  // PLY values are float32
    for (int k = 0; k < 9; ++k) m.shared_axes[k] = t.info.shared_axes[k];
    for (int k = 0; k < 3; ++k) m.background[k] = t.info.background[k];
    const Layout L = make_layout(m);
    m.blob_bytes = L.bytes;
    auto* sc = new sgs_scene();
    sc->meta = m;
    sc->ctx = ctx;
    DevBuf d_rows, d_tab;
    int mu_col = -1;
    const std::vector<int32_t> tab = ply_slot_table(t, L.color_planes, &mu_col);
    cudaError_t e = sc->owned.ensure(m.blob_bytes);
    if (e == cudaSuccess) e = d_rows.ensure(std::max<size_t>(nfloat, 1) * sizeof(float));
    if (e == cudaSuccess) e = d_tab.ensure(tab.size() * sizeof(int32_t));
    if (e == cudaSuccess) {
        sc->blob = sc->owned.ptr;
        cudaStream_t s = ctx->stream;
        e = cudaMemsetAsync(sc->blob, 0, m.blob_bytes, s);
        if (e == cudaSuccess && nfloat)
            e = cudaMemcpyAsync(d_rows.ptr, h_rows, nfloat * sizeof(float), cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(d_tab.ptr, tab.data(), tab.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess && t.count) {
            char* base = static_cast<char*>(sc->blob);
            ply_rows_kernel<<<static_cast<unsigned>((t.count + 255) / 256), 256, 0, s>>>(
                t.count, d_rows.as<float>(), static_cast<int>(t.props.size()), static_cast<int>(tab.size()),
                d_tab.as<int32_t>(), mu_col, reinterpret_cast<float4*>(base + L.geo_off[0]),
                reinterpret_cast<float4*>(base + L.geo_off[1]), reinterpret_cast<float4*>(base + L.geo_off[2]),
                reinterpret_cast<float4*>(base + L.color_off));
            e = cudaGetLastError();
            if (e == cudaSuccess) ctx->own_launches += 1;
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    d_rows.release();
    d_tab.release();
    cudaFreeHost(h_rows);
    if (e != cudaSuccess) {
        sgs_scene_free(sc);
        return fail(e == cudaErrorMemoryAllocation ? SGS_ERR_OUT_OF_MEMORY : SGS_ERR_CUDA,
                    std::string("ply load: ") + cudaGetErrorString(e));
    }
    sgs_status sb = bind_and_cache(sc, ctx->stream);
    if (sb != SGS_OK) {
        sgs_scene_free(sc);
        return sb;
    }
    if (info) *info = t.info;
    *out = sc;
    return SGS_OK;
}

// ---------------------------------------------------------------------------
// Image metrics (metrics.cu).
namespace {
sgs_status run_metric(sgs_context* ctx, const void* a, const void* b, int32_t w, int32_t h, int32_t c,
                      int32_t dtype, int32_t memory, bool ssim, double* out, double* grad) {
    if (!ctx || !a || !b || !out) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    if (w < 0 || h < 0 || c < 0) return fail(SGS_ERR_INVALID_ARGUMENT, "image dimensions do not match");
    if (dtype != SGS_F32 && dtype != SGS_F64) return fail(SGS_ERR_INVALID_ARGUMENT, "bad dtype");
    const size_t n = static_cast<size_t>(w) * static_cast<size_t>(h) * static_cast<size_t>(c);
    if (n == 0) return fail(SGS_ERR_INVALID_ARGUMENT, "empty image");  // check_shapes, metrics.cpp:87-90
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const size_t elem = dtype == SGS_F64 ? 8 : 4;
    const bool host = memory != SGS_DEVICE;
    const size_t work = metrics_scratch_doubles(n, grad != nullptr) * 8;
    const size_t staged = host ? align_up(2 * n * elem, 256) + (grad ? n * 8 : 0) : 0;
    SGS_CUDA(ctx->metrics.ensure(work + staged + 256));
    char* base = static_cast<char*>(ctx->metrics.ptr);
    double* scratch = reinterpret_cast<double*>(base);
    double* d_sum = scratch + metrics_scratch_doubles(n, grad != nullptr) - 1;
    const void* da = a;
    const void* db = b;
    double* dgrad = grad;
    if (host) {
        char* st = base + align_up(work, 256);
        SGS_CUDA(cudaMemcpyAsync(st, a, n * elem, cudaMemcpyHostToDevice, s));
        SGS_CUDA(cudaMemcpyAsync(st + n * elem, b, n * elem, cudaMemcpyHostToDevice, s));
        da = st;
        db = st + n * elem;
        if (grad) dgrad = reinterpret_cast<double*>(st + align_up(2 * n * elem, 256));
    }
    if (ssim) {
        launch_ssim(da, db, dtype == SGS_F64, w, h, c, scratch, d_sum, dgrad, s);
        ctx->own_launches += grad ? 6 : 4;
    } else {
        launch_psnr_sum(da, db, dtype == SGS_F64, n, scratch, d_sum, s);
        ctx->own_launches += 3;
    }
    SGS_CUDA(cudaGetLastError());
    double sum = 0.0;
    SGS_CUDA(cudaMemcpyAsync(&sum, d_sum, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (host && grad) SGS_CUDA(cudaMemcpyAsync(grad, dgrad, n * 8, cudaMemcpyDeviceToHost, s));
    SGS_CUDA(cudaStreamSynchronize(s));
    if (ssim) {
        *out = sum / static_cast<double>(n);
    } else {
        const double mse = sum / static_cast<double>(n);
        *out = mse < 1e-10 ? 100.0 : 10.0 * std::log10(1.0 / mse);
    }
    return SGS_OK;
}
}  // namespace

sgs_status sgs_psnr(sgs_context* ctx, const void* a, const void* b, int32_t width, int32_t height,
                    int32_t channels, int32_t dtype, int32_t memory, double* out) {
    return run_metric(ctx, a, b, width, height, channels, dtype, memory, false, out, nullptr);
}

sgs_status sgs_ssim(sgs_context* ctx, const void* a, const void* b, int32_t width, int32_t height,
                    int32_t channels, int32_t dtype, int32_t memory, double* value, double* grad_a) {
    return run_metric(ctx, a, b, width, height, channels, dtype, memory, true, value, grad_a);
}

sgs_status sgs_backward(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                        const sgs_render_config* cfg, const double* upstream, int32_t memory, double* grads) {
    if (!ctx || !scene || !cam || !cfg || !upstream || (!grads && scene->meta.count))
        return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    if (cfg->tile_size < 1) return fail(SGS_ERR_INVALID_ARGUMENT, "tile_size must be >= 1");
    sgs_status st = validate_camera(cam);
    if (st != SGS_OK) return st;
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const bool host = memory != SGS_DEVICE;
    const uint64_t n = scene->meta.count;
    const int stride = 11 + color_param_count_impl(scene->meta.kind, scene->meta.sh_degree);
    const size_t npx = static_cast<size_t>(cam->width) * static_cast<size_t>(cam->height);
    // grad.cpp:72-75: finite upstream (before any projection error)
    if (host) {
        for (size_t k = 0; k < npx * 3; ++k)
            if (!std::isfinite(upstream[k])) return fail(SGS_ERR_NUMERIC, "non-finite upstream gradient");
    } else {
        SGS_CUDA(ctx->bwd.ensure(256));
        int* d_bad = ctx->bwd.as<int>();
        SGS_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
        launch_finite_check(upstream, npx * 3, d_bad, s);
        int bad = 0;
        SGS_CUDA(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
        SGS_CUDA(cudaStreamSynchronize(s));
        if (bad) return fail(SGS_ERR_NUMERIC, "non-finite upstream gradient");
    }
    if (n == 0) return SGS_OK;
    // the forward's depth order and full tile lists (one chunk), as sgs_debug_tile_grid
    st = run_frame(ctx, scene, cam, cfg, nullptr, kTileGrid);
    if (st != SGS_OK) return st;
    Lane& L = ctx->lane[0];
    const uint64_t V = L.last_v, P = L.last_p;
    const CfgParams kp = make_cfg(cfg, cam);
    const size_t ntile = static_cast<size_t>(kp.tiles_x) * static_cast<size_t>(kp.tiles_y);
    // scratch: FP64 splats | rank_of | used | partials | (host) upstream | (host) grads
    const size_t o_rank = align_up(n * bwd_splat_bytes(), 256);
    const size_t o_used = o_rank + align_up(n * 4, 256);
    const size_t o_part = o_used + align_up(ntile * 4, 256);
    const size_t o_up = o_part + align_up(std::max<uint64_t>(P, 1) * bwd_partial_bytes(), 256);
    const size_t o_gr = o_up + (host ? align_up(npx * 3 * 8, 256) : 0);
    const size_t total = o_gr + (host ? n * stride * 8 : 0) + 256;
    SGS_CUDA(ctx->bwd.ensure(total));
    char* base = static_cast<char*>(ctx->bwd.ptr);
    const double* d_up = upstream;
    double* d_gr = grads;
    if (host) {
        SGS_CUDA(cudaMemcpyAsync(base + o_up, upstream, npx * 3 * 8, cudaMemcpyHostToDevice, s));
        d_up = reinterpret_cast<const double*>(base + o_up);
        d_gr = reinterpret_cast<double*>(base + o_gr);
    }
    SGS_CUDA(cudaMemsetAsync(d_gr, 0, n * stride * 8, s));
    launch_backward(scene->planes, make_cam(cam), kp, scene->meta.shared_axes, scene->meta.background,
                    cfg->has_override ? cfg->override_degree : -1, V, composite_pixel_chunks(cfg->tile_size),
                    L.last_order, L.brect.as<int4>(), L.ranges.as<uint2>(), L.last_list, base,
                    reinterpret_cast<uint32_t*>(base + o_rank), reinterpret_cast<uint32_t*>(base + o_used),
                    reinterpret_cast<double*>(base + o_part), d_up, d_gr, stride, s);
    SGS_CUDA(cudaGetLastError());
    ctx->own_launches += 3;
    if (host) SGS_CUDA(cudaMemcpyAsync(grads, d_gr, n * stride * 8, cudaMemcpyDeviceToHost, s));
    SGS_CUDA(cudaStreamSynchronize(s));
    return SGS_OK;
}

sgs_status sgs_render_f64(sgs_context* ctx, const sgs_scene* scene, const sgs_camera* cam,
                          const sgs_render_config* cfg, double* rgb, double* T, int32_t memory) {
    if (!ctx || !scene || !cam || !cfg) return fail(SGS_ERR_INVALID_ARGUMENT, "null argument");
    if (cfg->tile_size < 1) return fail(SGS_ERR_INVALID_ARGUMENT, "tile_size must be >= 1");
    sgs_status st = validate_camera(cam);
    if (st != SGS_OK) return st;
    std::lock_guard<std::mutex> lock(ctx->mu);
    SGS_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const bool host = memory != SGS_DEVICE;
    const uint64_t n = scene->meta.count;
    const size_t npx = static_cast<size_t>(cam->width) * static_cast<size_t>(cam->height);
    st = run_frame(ctx, scene, cam, cfg, nullptr, kTileGrid);
    if (st != SGS_OK) return st;
    Lane& L = ctx->lane[0];
    const CfgParams kp = make_cfg(cfg, cam);
    const size_t o_rank = align_up(std::max<uint64_t>(n, 1) * bwd_splat_bytes(), 256);
    const size_t o_img = o_rank + align_up(std::max<uint64_t>(n, 1) * 4, 256);
    const size_t o_T = o_img + (host ? align_up(npx * 3 * 8, 256) : 0);
    const size_t total = o_T + (host ? npx * 8 : 0) + 256;
    SGS_CUDA(ctx->bwd.ensure(total));
    char* base = static_cast<char*>(ctx->bwd.ptr);
    double* d_rgb = host ? (rgb ? reinterpret_cast<double*>(base + o_img) : nullptr) : rgb;
    double* d_T = host ? (T ? reinterpret_cast<double*>(base + o_T) : nullptr) : T;
    launch_render_f64(scene->planes, make_cam(cam), kp, scene->meta.shared_axes, scene->meta.background,
                      cfg->has_override ? cfg->override_degree : -1, L.last_v, composite_pixel_chunks(cfg->tile_size),
                      L.last_order, L.ranges.as<uint2>(), L.last_list, base,
                      reinterpret_cast<uint32_t*>(base + o_rank), d_rgb, d_T, s);
    SGS_CUDA(cudaGetLastError());
    ctx->own_launches += 2;
    if (host && rgb) SGS_CUDA(cudaMemcpyAsync(rgb, d_rgb, npx * 3 * 8, cudaMemcpyDeviceToHost, s));
    if (host && T) SGS_CUDA(cudaMemcpyAsync(T, d_T, npx * 8, cudaMemcpyDeviceToHost, s));
    SGS_CUDA(cudaStreamSynchronize(s));
    return SGS_OK;
}

}  // extern "C"
