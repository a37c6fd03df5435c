// radix.cu -- the library's own device radix sort (no CUB on any path), and the
// depth-order stage K2 built on it.
//
// Onesweep LSD radix sort of (u32 key, u32 value) pairs: ONE kernel per digit pass.
// A persistent grid takes 4096-key tiles in ticket order; each CTA ranks its tile
// stably in shared memory (warp match.any + per-warp digit counters), publishes the
// tile's digit counts, finds the counts of all earlier tiles by a decoupled
// look-back over per-tile status words (a warp checks 32 predecessors at once, every
// thread of the CTA then sums its digit over the window), and scatters the tile
// through shared memory so each digit run leaves as one contiguous write. The global
// digit histograms of every pass come from the kernel that produced the keys (K1's
// depth keys via depth_key32_kernel; the binning's tile ids in bin_emit_kernel), so
// a pass count of p costs p launches and no scan kernels.
//
// Status words carry an (epoch, pass) tag -- the epoch is bumped by the producer of
// each sort -- so the per-tile status never needs clearing between sorts; a count of keys
// is read from device memory, so a frame sorts a device-sized list with no host
// round trip.
//
// K2 (raster.cpp:93-101, stable order by (double depth, index)): the 64-bit
// orderable depth keys are reduced to 32 bits as (key - kmin) >> s (s so the range
// fits), sorted in 4 passes with the Gaussian index as value (stable, so equal keys
// stay in index order), and the rare runs of equal 32-bit keys are re-sorted by the
// full (key, index) in depth_rank_kernel, which also writes the ranks and the
// rank-ordered binning inputs. A run longer than kRunCap makes the host redo the
// frame with the full 64-bit sort (8 passes of the same kernel).
#include <algorithm>
#include <cstddef>

#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kOsThreads = 512;
constexpr int kOsWarps = kOsThreads / 32;
constexpr int kOsItems = 8;
constexpr int kOsTile = kOsThreads * kOsItems;  // keys per tile
constexpr uint32_t kStAgg = 1u;  // tile status: aggregate counts published
constexpr uint32_t kStPre = 2u;  // inclusive prefix counts published

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_cg_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// Dynamic shared memory of one onesweep CTA.
struct OsSmem {
    uint32_t wcnt[kOsWarps][257];  // per-warp digit counters -> per-warp digit offsets
    uint32_t tot[256];             // tile digit counts
    uint32_t toff[256];            // tile digit exclusive offsets
    uint32_t gofs[256];            // global position of local position 0 of digit d
    uint32_t gbase[256];           // global digit offsets (exclusive scan of the histogram)
    uint32_t excl[256];            // counts of digit d in all earlier tiles
    uint32_t key[kOsTile];
    uint32_t val[kOsTile];
    uint32_t warp_tmp[kOsWarps];
    uint32_t tile;
    int32_t win_lo, win_pre;  // look-back window [win_lo, win_hi]; win_pre: its lowest tile holds a prefix
};

// Exclusive scan of v[0, 256) by the first 256 threads (warps 0..7) into out.
__device__ __forceinline__ void scan256(const uint32_t* v, uint32_t* out, uint32_t* warp_tmp) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t x = t < 256 ? v[t] : 0u, inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31 && w < 8) warp_tmp[w] = inc;
    __syncthreads();
    if (t < 256) {
        uint32_t add = 0;
        for (int k = 0; k < w; ++k) add += warp_tmp[k];
        out[t] = add + inc - x;
    }
    __syncthreads();
}

template <bool kIota>
__global__ void __launch_bounds__(kOsThreads, 2) onesweep_kernel(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, const unsigned long long* __restrict__ dcount, uint64_t hcount, int shift, int bits,
    SortCtl* __restrict__ ctl, int pass, uint32_t* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char os_raw[];
    OsSmem& S = *reinterpret_cast<OsSmem*>(os_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t n = dcount ? *dcount : hcount;
    const uint32_t radix = 1u << bits, mask = radix - 1;
    const uint32_t ntiles = static_cast<uint32_t>((n + kOsTile - 1) / kOsTile);
    // (epoch, pass) tag of this pass's status words; the low 2 bits of a word are its state
    const uint32_t tag = ((ctl->epoch << 3) | static_cast<uint32_t>(pass)) & 0x3FFFFFFFu;
    // status layout per tile: [0] tag | state word, [1..256] aggregate, [257..512] inclusive prefix
    constexpr int kStride = 1 + 2 * 256;
    if (tid < 256) S.tot[tid] = tid < static_cast<int>(radix) ? ctl->hist[pass][tid] : 0u;
    __syncthreads();
    scan256(S.tot, S.gbase, S.warp_tmp);
    for (;;) {
        if (tid == 0) S.tile = atomicAdd(&ctl->ticket[pass], 1u);
        for (int k = tid; k < kOsWarps * 257; k += kOsThreads) (&S.wcnt[0][0])[k] = 0;
        __syncthreads();
        const uint32_t tile = S.tile;
        if (tile >= ntiles) break;
        const uint64_t t0 = static_cast<uint64_t>(tile) * kOsTile;
        // load: warp w owns keys [t0 + w * 32 kOsItems, +32 kOsItems) in rounds of 32, so
        // the stable order inside the tile is (warp, round, lane) = memory order
        uint32_t key[kOsItems], val[kOsItems], dg[kOsItems], rk[kOsItems];
        const uint64_t w0 = t0 + static_cast<uint64_t>(warp) * (32 * kOsItems) + lane;
#pragma unroll
        for (int j = 0; j < kOsItems; ++j) {
            const uint64_t i = w0 + j * 32;
            const bool ok = i < n;
            key[j] = ok ? kin[i] : 0u;
            val[j] = kIota ? static_cast<uint32_t>(i) : (ok ? vin[i] : 0u);
            dg[j] = ok ? (key[j] >> shift) & mask : 256u;
        }
#pragma unroll
        for (int j = 0; j < kOsItems; ++j) {
            const unsigned peers = __match_any_sync(0xffffffffu, dg[j]);
            const unsigned below = peers & ((1u << lane) - 1u);
            const uint32_t before = S.wcnt[warp][dg[j]];
            rk[j] = before + __popc(below);
            __syncwarp();
            if (below == 0) S.wcnt[warp][dg[j]] = before + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        if (tid < 256) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kOsWarps; ++w) {
                const uint32_t c = S.wcnt[w][tid];
                S.wcnt[w][tid] = run;
                run += c;
            }
            S.tot[tid] = run;
            S.excl[tid] = 0;
        }
        __syncthreads();
        scan256(S.tot, S.toff, S.warp_tmp);
        // publish the tile's aggregate (tile 0: its prefix)
        uint32_t* st = status + static_cast<size_t>(tile) * kStride;
        if (tid < 256) {
            st[1 + tid] = S.tot[tid];
            if (tile == 0) st[257 + tid] = S.tot[tid];
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release_u32(st, tag << 2 | (tile == 0 ? kStPre : kStAgg));
        // decoupled look-back: warp 0 finds, 32 predecessors at a time, the window that
        // ends at the nearest tile with a published prefix; every thread adds its digit
        if (tile > 0) {
            int64_t hi = static_cast<int64_t>(tile) - 1;
            for (;;) {
                if (warp == 0) {
                    const int64_t p = hi - lane;
                    uint32_t s = p >= 0 ? 0u : (tag << 2 | kStPre);
                    for (;;) {
                        if (p >= 0 && (s >> 2) != tag) s = ld_acquire_u32(status + static_cast<size_t>(p) * kStride);
                        const bool ready = p < 0 || ((s >> 2) == tag && (s & 3u) != 0u);
                        if (__all_sync(0xffffffffu, ready)) break;
                    }
                    const unsigned pre = __ballot_sync(0xffffffffu, p >= 0 && (s & 3u) == kStPre);
                    const int stop = pre ? __ffs(pre) - 1 : 31;
                    if (lane == 0) {
                        const int64_t lo = hi - stop;
                        S.win_lo = static_cast<int32_t>(lo < 0 ? 0 : lo);
                        S.win_pre = pre ? 1 : 0;
                    }
                }
                __syncthreads();
                const int64_t lo = S.win_lo;
                const bool has_pre = S.win_pre != 0;
                if (tid < 256) {
                    uint32_t acc = 0;
                    for (int64_t p = hi; p >= lo; --p) {
                        const uint32_t* sp = status + static_cast<size_t>(p) * kStride;
                        acc += ld_cg_u32(sp + ((has_pre && p == lo) ? 257 : 1) + tid);
                    }
                    S.excl[tid] += acc;
                }
                __syncthreads();
                if (has_pre || lo == 0) break;
                hi = lo - 1;
            }
            if (tid < 256) st[257 + tid] = S.excl[tid] + S.tot[tid];
            __threadfence();
            __syncthreads();
            if (tid == 0) st_release_u32(st, tag << 2 | kStPre);
        }
        if (tid < 256) S.gofs[tid] = S.gbase[tid] + S.excl[tid] - S.toff[tid];
        // local scatter into digit order, then contiguous digit runs to global memory
#pragma unroll
        for (int j = 0; j < kOsItems; ++j) {
            if (dg[j] < 256u) {
                const uint32_t lp = S.toff[dg[j]] + S.wcnt[warp][dg[j]] + rk[j];
                S.key[lp] = key[j];
                S.val[lp] = val[j];
            }
        }
        __syncthreads();
        const uint32_t m = static_cast<uint32_t>(n - t0 < static_cast<uint64_t>(kOsTile) ? n - t0 : kOsTile);
        for (uint32_t i = tid; i < m; i += kOsThreads) {
            const uint32_t k = S.key[i];
            const uint32_t pos = S.gofs[(k >> shift) & mask] + i;
            kout[pos] = k;
            vout[pos] = S.val[i];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// K2 producers and the rank writer.

constexpr int kHistThreads = 512;
constexpr int kRunCap = 32;  // longest run of equal 32-bit depth keys fixed up in place

__device__ __forceinline__ int key32_shift(const Counters* ctr) {
    const unsigned long long kmin = ctr->kmin, kmax = ctr->kmax;
    const unsigned long long range = kmax >= kmin ? kmax - kmin : 0ULL;
    const int bits = range ? 64 - __clzll(static_cast<long long>(range)) : 0;
    return bits > 32 ? bits - 32 : 0;
}

// k32[i] = culled ? ~0 : min((key - kmin) >> s, ~0 - 1), and the 4 digit histograms;
// block 0 opens the sort's epoch.
__global__ void __launch_bounds__(kHistThreads) depth_key32_kernel(uint64_t n, const unsigned long long* __restrict__ key,
                                                                   const Counters* __restrict__ ctr,
                                                                   uint32_t* __restrict__ k32, SortCtl* __restrict__ ctl) {
    __shared__ uint32_t h[4 * 256];
    for (int k = threadIdx.x; k < 4 * 256; k += kHistThreads) h[k] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->epoch += 1;
    __syncthreads();
    const unsigned long long kmin = ctr->kmin;
    const int sh = key32_shift(ctr);
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kHistThreads + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kHistThreads) {
        const unsigned long long k = key[i];
        uint32_t v = 0xFFFFFFFFu;
        if (k != ~0ULL) {
            const unsigned long long d = (k - kmin) >> sh;
            v = d < 0xFFFFFFFEULL ? static_cast<uint32_t>(d) : 0xFFFFFFFEu;
        }
        k32[i] = v;
#pragma unroll
        for (int p = 0; p < 4; ++p) atomicAdd(&h[p * 256 + ((v >> (8 * p)) & 255u)], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 4 * 256; k += kHistThreads)
        if (h[k]) atomicAdd(&ctl->hist[k >> 8][k & 255], h[k]);
}

// Wide path: the low (half 0) or high (half 1, gathered through the sorted values)
// 32 bits of the raw 64-bit keys, and their digit histograms (passes 4*half ..).
__global__ void __launch_bounds__(kHistThreads) depth_key_half_kernel(uint64_t n, const unsigned long long* __restrict__ key,
                                                                      const uint32_t* __restrict__ idx, int half,
                                                                      uint32_t* __restrict__ k32, SortCtl* __restrict__ ctl) {
    __shared__ uint32_t h[4 * 256];
    for (int k = threadIdx.x; k < 4 * 256; k += kHistThreads) h[k] = 0;
    if (half == 0 && blockIdx.x == 0 && threadIdx.x == 0) ctl->epoch += 1;
    __syncthreads();
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kHistThreads + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kHistThreads) {
        const uint32_t v = half ? static_cast<uint32_t>(key[idx[i]] >> 32) : static_cast<uint32_t>(key[i]);
        k32[i] = v;
#pragma unroll
        for (int p = 0; p < 4; ++p) atomicAdd(&h[p * 256 + ((v >> (8 * p)) & 255u)], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 4 * 256; k += kHistThreads)
        if (h[k]) atomicAdd(&ctl->hist[4 * half + (k >> 8)][k & 255], h[k]);
}

__device__ __forceinline__ bool less_ki(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

__device__ __forceinline__ void put_rank(uint64_t r, uint32_t g, bool visible, const int4* __restrict__ rects,
                                         uint32_t* __restrict__ order, int4* __restrict__ brect,
                                         uint2* __restrict__ bmeta) {
    order[r] = g;
    if (visible) {  // visible splats always have their rect written by K1
        const int4 rc = rects[g];
        bmeta[r] = make_uint2(g, rect_area(rc));
        brect[r] = rc;
    } else {
        bmeta[r] = make_uint2(g, 0u);
    }
}

// Ranks from the sorted (k32, index) pairs. Narrow keys: a run of equal 32-bit keys
// among the visible splats is re-sorted by (64-bit key, index) by the thread at its
// start (runs are rare: ~n^2 / 2^33 pairs); wide keys are the full key already.
__global__ void depth_rank_kernel(uint64_t n, const uint32_t* __restrict__ sk, const uint32_t* __restrict__ sv,
                                  const unsigned long long* __restrict__ key, int wide,
                                  Counters* __restrict__ ctr, const int4* __restrict__ rects,
                                  uint32_t* __restrict__ order, int4* __restrict__ brect, uint2* __restrict__ bmeta) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t g = sv[r];
    if (wide) {
        put_rank(r, g, r < ctr->visible, rects, order, brect, bmeta);
        return;
    }
    const uint32_t k = sk[r];
    if (k == 0xFFFFFFFFu) {  // culled: after the visible splats, in index order
        put_rank(r, g, false, rects, order, brect, bmeta);
        return;
    }
    const bool same_prev = r > 0 && sk[r - 1] == k;
    const bool same_next = r + 1 < n && sk[r + 1] == k;
    if (!same_prev && !same_next) {
        put_rank(r, g, true, rects, order, brect, bmeta);
        return;
    }
    if (same_prev) return;  // inside a run: its first thread writes it
    uint32_t m = 1;
    while (r + m < n && m <= kRunCap && sk[r + m] == k) ++m;
    if (m > kRunCap) {
        atomicAdd(&ctr->tie_overflow, 1ULL);
        return;
    }
    atomicAdd(&ctr->tie_runs, 1ULL);
    unsigned long long kk[kRunCap];
    uint32_t ii[kRunCap];
    for (uint32_t a = 0; a < m; ++a) {  // insertion sort by (64-bit key, index)
        const uint32_t vi = sv[r + a];
        const unsigned long long vk = key[vi];
        int c = static_cast<int>(a) - 1;
        while (c >= 0 && less_ki(vk, vi, kk[c], ii[c])) {
            kk[c + 1] = kk[c];
            ii[c + 1] = ii[c];
            --c;
        }
        kk[c + 1] = vk;
        ii[c + 1] = vi;
    }
    for (uint32_t a = 0; a < m; ++a) put_rank(r + a, ii[a], true, rects, order, brect, bmeta);
}

size_t onesweep_smem() { return sizeof(OsSmem); }

}  // namespace

size_t sort_status_words(uint64_t capacity) {
    return static_cast<size_t>((capacity + kOsTile - 1) / kOsTile + 1) * (1 + 2 * 256);
}

int onesweep_grid() { return 148 * 2; }

cudaError_t launch_onesweep_pass(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                                 const unsigned long long* dcount, uint64_t hcount, int shift, int bits,
                                 SortCtl* ctl, int pass, uint32_t* status, cudaStream_t stream) {
    static const cudaError_t attr = [] {
        cudaError_t e = cudaFuncSetAttribute(onesweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(onesweep_smem()));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(onesweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(onesweep_smem()));
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    if (vin)
        onesweep_kernel<false><<<onesweep_grid(), kOsThreads, onesweep_smem(), stream>>>(
            kin, vin, kout, vout, dcount, hcount, shift, bits, ctl, pass, status);
    else
        onesweep_kernel<true><<<onesweep_grid(), kOsThreads, onesweep_smem(), stream>>>(
            kin, nullptr, kout, vout, dcount, hcount, shift, bits, ctl, pass, status);
    return cudaGetLastError();
}

// K2: depth order of n splats. Narrow: key32 + 4 passes + rank fix-up (6 launches);
// wide: low half 4 passes, high half 4 passes, ranks (11 launches).
cudaError_t launch_depth_sort(uint64_t n, const unsigned long long* key, Counters* ctr, bool wide, uint32_t* ka,
                              uint32_t* va, uint32_t* kb, uint32_t* vb, SortCtl* ctl, uint32_t* status,
                              const int4* rects, uint32_t* order, int4* brect, uint2* bmeta, cudaStream_t stream,
                              uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(&ctl->ticket[0], 0, sizeof(SortCtl) - offsetof(SortCtl, ticket), stream);
    if (e != cudaSuccess) return e;
    const unsigned hgrid = static_cast<unsigned>(std::min<uint64_t>((n + kHistThreads - 1) / kHistThreads, 148 * 4));
    // 4 passes over 8-bit digits: (ka, iota) -> (kb, vb) -> (ka, va) -> (kb, vb) -> (ka, va)
    auto four = [&](int pass0, bool iota_first) -> cudaError_t {
        cudaError_t ee = cudaSuccess;
        for (int p = 0; p < 4 && ee == cudaSuccess; ++p) {
            const bool even = (p & 1) == 0;
            ee = launch_onesweep_pass(even ? ka : kb, (p == 0 && iota_first) ? nullptr : (even ? va : vb),
                                      even ? kb : ka, even ? vb : va, nullptr, n, 8 * p, 8, ctl, pass0 + p, status,
                                      stream);
        }
        return ee;
    };
    if (!wide) {
        depth_key32_kernel<<<hgrid, kHistThreads, 0, stream>>>(n, key, ctr, ka, ctl);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if ((e = four(0, true)) != cudaSuccess) return e;
        *launches += 6;
    } else {
        depth_key_half_kernel<<<hgrid, kHistThreads, 0, stream>>>(n, key, nullptr, 0, ka, ctl);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if ((e = four(0, true)) != cudaSuccess) return e;
        depth_key_half_kernel<<<hgrid, kHistThreads, 0, stream>>>(n, key, va, 1, ka, ctl);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if ((e = four(4, false)) != cudaSuccess) return e;
        *launches += 11;
    }
    depth_rank_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(n, ka, va, key, wide ? 1 : 0, ctr,
                                                                                  rects, order, brect, bmeta);
    return cudaGetLastError();
}

}  // namespace sgs
