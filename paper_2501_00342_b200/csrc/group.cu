// group.cu -- multi-GPU rendering through the C-ABI (include/sgs.h).
//
// The reference parallelises only with std::thread (common.hpp:53-77); the renders a
// multi-GPU caller shards are its per-view loops (tools/main.cpp:207-216, :280-287).
// Here the views are the unit: the scene is replicated once by an NCCL broadcast
// over NVLink and the views are block-partitioned across the ranks (one rank per
// GPU); no collective sits on the render path itself. Frames go to a root rank with
// grouped ncclSend / ncclRecv on a separate stream, a sub-batch at a time, so the
// transfer of sub-batch k overlaps the rendering of sub-batch k + 1.
//
// Ranks are NCCL ranks: one process per GPU (sgs_group_init_rank, e.g. under
// torchrun, with the unique id shipped by the caller), or one process driving every
// GPU (sgs_group_create: ncclCommInitAll, then one host thread per rank). Every
// sgs_group_* call is collective: each rank makes it with the same arguments (the
// scene description only on the root).
//
// NCCL is resolved at run time -- the one already in the process (torch's), else
// SGS_NCCL_PATH, else the system's libnccl.so.2 -- so the library itself has no
// link-time NCCL dependency and never loads a second NCCL beside torch's.
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

#include "sgs_internal.h"

namespace {

struct Nccl {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    std::string error;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // an NCCL the process already loaded (e.g. torch's), else SGS_NCCL_PATH, else the
        // system's: never a second copy under the same soname
        n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!n.lib) {
            if (const char* path = std::getenv("SGS_NCCL_PATH")) n.lib = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
        }
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            if (n.lib) break;
            n.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        }
        if (!n.lib) {
            n.error = std::string("NCCL not found: ") + dlerror();
            return;
        }
        auto sym = [&](const char* s) {
            void* p = dlsym(n.lib, s);
            if (!p && n.error.empty()) n.error = std::string("NCCL symbol missing: ") + s;
            return p;
        };
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
        n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(sym("ncclCommInitAll"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
        n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
        n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    });
    return n;
}

// Views per gather sub-batch: the transfer of one overlaps the rendering of the next.
constexpr int kGatherViews = 4;

}  // namespace

struct sgs_group {
    sgs_context* ctx = nullptr;
    bool own_ctx = false;
    int nranks = 1, rank = 0, device = 0;
    ncclComm_t comm = nullptr;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_rendered[2] = {}, ev_sent[2] = {};
    void* stage = nullptr;  // non-root: two slots of kGatherViews frames (RGB, T)
    size_t stage_bytes = 0;
    void* gather = nullptr;  // root with host outputs: every frame on the device
    size_t gather_bytes = 0;
};

namespace {

#define SGS_NCCL(call)                                                                              \
    do {                                                                                            \
        const ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                      \
            return sgs::fail_status(SGS_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
    } while (0)

#define SGS_GCUDA(call)                                                                             \
    do {                                                                                            \
        const cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) return sgs::fail_status(SGS_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

sgs_status check_nccl() {
    const Nccl& n = nccl();
    if (!n.error.empty()) return sgs::fail_status(SGS_ERR_NCCL, n.error);
    return SGS_OK;
}

sgs_status group_setup(sgs_group* g) {
    SGS_GCUDA(cudaSetDevice(g->device));
    SGS_GCUDA(cudaStreamCreateWithFlags(&g->comm_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        SGS_GCUDA(cudaEventCreateWithFlags(&g->ev_rendered[k], cudaEventDisableTiming));
        SGS_GCUDA(cudaEventCreateWithFlags(&g->ev_sent[k], cudaEventDisableTiming));
    }
    return SGS_OK;
}

sgs_status ensure(void** p, size_t* have, size_t need) {
    if (*have >= need) return SGS_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    SGS_GCUDA(cudaMalloc(p, need));
    *have = need;
    return SGS_OK;
}

// [begin, end) of the views rank r renders (contiguous blocks, sizes differ by <= 1).
void shard(int n, int nranks, int r, int* b, int* e) {
    const int base = n / nranks, extra = n % nranks;
    *b = r * base + std::min(r, extra);
    *e = *b + base + (r < extra ? 1 : 0);
}

}  // namespace

extern "C" {

sgs_status sgs_group_unique_id(uint8_t* id) {
    if (!id) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "null id");
    sgs_status st = check_nccl();
    if (st != SGS_OK) return st;
    ncclUniqueId u;
    SGS_NCCL(nccl().GetUniqueId(&u));
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return SGS_OK;
}

sgs_status sgs_group_init_rank(sgs_context* ctx, int32_t nranks, int32_t rank, const uint8_t* id, sgs_group** out) {
    if (!ctx || !id || !out) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "bad rank");
    sgs_status st = check_nccl();
    if (st != SGS_OK) return st;
    auto* g = new sgs_group();
    g->ctx = ctx;
    g->nranks = nranks;
    g->rank = rank;
    g->device = sgs::context_device(ctx);
    st = group_setup(g);
    if (st == SGS_OK) {
        ncclUniqueId u;
        std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        const ncclResult_t r = nccl().CommInitRank(&g->comm, nranks, u, rank);
        if (r != ncclSuccess) st = sgs::fail_status(SGS_ERR_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
    }
    if (st != SGS_OK) {
        sgs_group_destroy(g);
        return st;
    }
    *out = g;
    return SGS_OK;
}

sgs_status sgs_group_create(int32_t ndev, const int32_t* devices, sgs_group** out) {
    if (ndev < 1 || !devices || !out) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "bad device list");
    sgs_status st = check_nccl();
    if (st != SGS_OK) return st;
    std::vector<ncclComm_t> comms(static_cast<size_t>(ndev));
    std::vector<int> devs(devices, devices + ndev);
    SGS_NCCL(nccl().CommInitAll(comms.data(), ndev, devs.data()));
    for (int r = 0; r < ndev; ++r) {
        auto* g = new sgs_group();
        g->nranks = ndev;
        g->rank = r;
        g->device = devices[r];
        g->comm = comms[static_cast<size_t>(r)];
        out[r] = g;
        if (st == SGS_OK) st = sgs_create(devices[r], &g->ctx);
        g->own_ctx = g->ctx != nullptr;
        if (st == SGS_OK) st = group_setup(g);
    }
    if (st != SGS_OK) {
        for (int r = 0; r < ndev; ++r) {
            sgs_group_destroy(out[r]);
            out[r] = nullptr;
        }
    }
    return st;
}

void sgs_group_destroy(sgs_group* g) {
    if (!g) return;
    cudaSetDevice(g->device);
    if (g->comm_stream) cudaStreamSynchronize(g->comm_stream);
    if (g->comm) nccl().CommDestroy(g->comm);
    for (int k = 0; k < 2; ++k) {
        if (g->ev_rendered[k]) cudaEventDestroy(g->ev_rendered[k]);
        if (g->ev_sent[k]) cudaEventDestroy(g->ev_sent[k]);
    }
    if (g->comm_stream) cudaStreamDestroy(g->comm_stream);
    if (g->stage) cudaFree(g->stage);
    if (g->gather) cudaFree(g->gather);
    if (g->own_ctx) sgs_destroy(g->ctx);
    delete g;
}

sgs_status sgs_group_context(sgs_group* g, sgs_context** ctx) {
    if (!g || !ctx) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "null argument");
    *ctx = g->ctx;
    return SGS_OK;
}

sgs_status sgs_group_broadcast_scene(sgs_group* g, const sgs_scene_desc* desc, int32_t root, sgs_scene** out) {
    if (!g || !out) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "null argument");
    if (root < 0 || root >= g->nranks) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "bad root");
    SGS_GCUDA(cudaSetDevice(g->device));
    // the root plans and uploads; the layout (meta) travels first, then the blob
    sgs_scene_meta meta{};
    sgs_scene* scene = nullptr;
    if (g->rank == root) {
        if (!desc) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "null scene description on the root");
        sgs_status st = sgs_scene_upload(g->ctx, desc, &scene);
        if (st != SGS_OK) return st;
        sgs_scene_get_meta(scene, &meta);
    }
    void* d_meta = nullptr;
    SGS_GCUDA(cudaMalloc(&d_meta, sizeof(meta)));
    SGS_GCUDA(cudaMemcpy(d_meta, &meta, sizeof(meta), cudaMemcpyHostToDevice));
    SGS_NCCL(nccl().Broadcast(d_meta, d_meta, sizeof(meta), ncclUint8, root, g->comm, g->comm_stream));
    SGS_GCUDA(cudaMemcpyAsync(&meta, d_meta, sizeof(meta), cudaMemcpyDeviceToHost, g->comm_stream));
    SGS_GCUDA(cudaStreamSynchronize(g->comm_stream));
    cudaFree(d_meta);
    void* blob = nullptr;
    uint64_t bytes = meta.blob_bytes;
    if (g->rank == root) {
        SGS_GCUDA(cudaDeviceSynchronize());  // the upload (its own stream) is complete
        sgs_scene_blob(scene, &blob, &bytes);
    } else {
        SGS_GCUDA(cudaMalloc(&blob, std::max<uint64_t>(bytes, 256)));
    }
    SGS_NCCL(nccl().Broadcast(blob, blob, bytes, ncclUint8, root, g->comm, g->comm_stream));
    SGS_GCUDA(cudaStreamSynchronize(g->comm_stream));
    if (g->rank != root) {
        sgs_status st = sgs::scene_bind_owned(g->ctx, &meta, blob, bytes, &scene);
        if (st != SGS_OK) {
            cudaFree(blob);
            return st;
        }
    }
    *out = scene;
    return SGS_OK;
}

sgs_status sgs_group_render_views(sgs_group* g, const sgs_scene* scene, const sgs_camera* cams, int32_t n,
                                  const sgs_render_config* cfg, int32_t root, float* rgb, float* T,
                                  int32_t out_memory, sgs_render_stats* stats) {
    if (!g || !scene || !cfg || (n > 0 && !cams)) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "null argument");
    if (n < 0) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "negative view count");
    if (root < 0 || root >= g->nranks) return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "bad root");
    if (n == 0) return SGS_OK;
    SGS_GCUDA(cudaSetDevice(g->device));
    const int W = cams[0].width, H = cams[0].height;
    for (int v = 1; v < n; ++v)  // (frames are gathered at one stride)
        if (cams[v].width != W || cams[v].height != H)
            return sgs::fail_status(SGS_ERR_INVALID_ARGUMENT, "group views must share one image size");
    const size_t npx = static_cast<size_t>(W) * static_cast<size_t>(H);
    const bool want_T = T != nullptr;
    const size_t fr_rgb = npx * 3 * sizeof(float), fr_T = want_T ? npx * sizeof(float) : 0;
    int b = 0, e = 0;
    shard(n, g->nranks, g->rank, &b, &e);
    cudaStream_t rs = nullptr;  // the context's render stream
    sgs::context_stream(g->ctx, &rs);
    if (g->rank == root) {
        // frames land in the caller's device buffers, or (host outputs) in a device
        // gather buffer copied out at the end
        float* d_rgb = rgb;
        float* d_T = T;
        if (out_memory != SGS_DEVICE) {
            sgs_status st = ensure(&g->gather, &g->gather_bytes, static_cast<size_t>(n) * (fr_rgb + fr_T));
            if (st != SGS_OK) return st;
            d_rgb = static_cast<float*>(g->gather);
            d_T = want_T ? reinterpret_cast<float*>(static_cast<char*>(g->gather) + n * fr_rgb) : nullptr;
        }
        // every other rank's sub-batches, in the order they are sent
        SGS_NCCL(nccl().GroupStart());
        for (int r = 0; r < g->nranks; ++r) {
            if (r == root) continue;
            int rb = 0, re = 0;
            shard(n, g->nranks, r, &rb, &re);
            for (int v = rb; v < re; v += kGatherViews) {
                const int k = std::min(kGatherViews, re - v);
                SGS_NCCL(nccl().Recv(d_rgb + static_cast<size_t>(v) * npx * 3, k * npx * 3, ncclFloat32, r, g->comm,
                                     g->comm_stream));
                if (want_T)
                    SGS_NCCL(nccl().Recv(d_T + static_cast<size_t>(v) * npx, k * npx, ncclFloat32, r, g->comm,
                                         g->comm_stream));
            }
        }
        SGS_NCCL(nccl().GroupEnd());
        // this rank's own views, while the others' frames arrive
        if (e > b) {
            sgs_status st = sgs_render_batch(g->ctx, scene, cams + b, e - b, cfg, d_rgb + static_cast<size_t>(b) * npx * 3,
                                             want_T ? d_T + static_cast<size_t>(b) * npx : nullptr, SGS_DEVICE, stats);
            if (st != SGS_OK) return st;
        }
        SGS_GCUDA(cudaStreamSynchronize(g->comm_stream));
        if (out_memory != SGS_DEVICE) {
            SGS_GCUDA(cudaMemcpy(rgb, d_rgb, n * fr_rgb, cudaMemcpyDeviceToHost));
            if (want_T) SGS_GCUDA(cudaMemcpy(T, d_T, n * fr_T, cudaMemcpyDeviceToHost));
        }
        return SGS_OK;
    }
    // non-root: render sub-batches into two staging slots; each is sent while the
    // next one renders, and a slot is reused only after its send has left
    const size_t slot_bytes = kGatherViews * (fr_rgb + fr_T);
    sgs_status st = ensure(&g->stage, &g->stage_bytes, 2 * slot_bytes);
    if (st != SGS_OK) return st;
    int slot = 0;
    bool pending[2] = {false, false};
    for (int v = b; v < e; v += kGatherViews, slot ^= 1) {
        const int k = std::min(kGatherViews, e - v);
        char* base = static_cast<char*>(g->stage) + slot * slot_bytes;
        float* s_rgb = reinterpret_cast<float*>(base);
        float* s_T = want_T ? reinterpret_cast<float*>(base + kGatherViews * fr_rgb) : nullptr;
        if (pending[slot]) SGS_GCUDA(cudaStreamWaitEvent(rs, g->ev_sent[slot], 0));
        st = sgs_render_batch(g->ctx, scene, cams + v, k, cfg, s_rgb, s_T, SGS_DEVICE, stats);
        if (st != SGS_OK) return st;
        SGS_GCUDA(cudaEventRecord(g->ev_rendered[slot], rs));
        SGS_GCUDA(cudaStreamWaitEvent(g->comm_stream, g->ev_rendered[slot], 0));
        SGS_NCCL(nccl().GroupStart());
        SGS_NCCL(nccl().Send(s_rgb, k * npx * 3, ncclFloat32, root, g->comm, g->comm_stream));
        if (want_T) SGS_NCCL(nccl().Send(s_T, k * npx, ncclFloat32, root, g->comm, g->comm_stream));
        SGS_NCCL(nccl().GroupEnd());
        SGS_GCUDA(cudaEventRecord(g->ev_sent[slot], g->comm_stream));
        pending[slot] = true;
    }
    SGS_GCUDA(cudaStreamSynchronize(g->comm_stream));
    return SGS_OK;
}

}  // extern "C"
