// radix.cu -- the library's own device radix sort (no CUB on any path), and the
// depth-order stage K2 built on it.
//
// Stable LSD radix sort of (u32 key, u32 value) pairs, two kernels per digit pass
// and no scan kernel: the keys are cut into G = 296 contiguous slices (2 CTAs per
// SM); the upsweep writes each slice's digit histogram and adds it to the pass's
// global digit counts; the downsweep CTA of slice g computes its own output offsets
// -- the exclusive scan of the global counts plus the sums of its digits' rows over
// the slices before it (at most 295 counters per digit, coalesced loads all in
// flight at once) -- and walks its slice in order, 4096 keys per step (the next
// step's keys loading meanwhile), ranking equal digits within a warp by match.any +
// popc and across warps by a shared-memory prefix, so the scatter is stable; each
// step is staged in digit order in shared memory and leaves as contiguous runs. No CTA waits for another (nothing spins), so the passes overlap freely
// with the other lanes' kernels. The count of keys is read from device memory: a
// frame sorts a device-sized list with no host round trip.
//
// K2 (raster.cpp:93-101, stable order by (double depth, index)): the 64-bit
// orderable depth keys are reduced to kKeyBits = 24 bits as (key - kmin) >> s (s so
// the range fits), sorted in 3 passes with the Gaussian index as value (stable, so
// equal keys stay in index order), and the runs of equal 24-bit keys are re-sorted by
// the full (key, index) in depth_rank_kernel, which also writes the ranks and the
// rank-ordered binning inputs. At config C (3M splats) 27% of the keys share their
// 24-bit key with another, in runs of at most 8 (32 bits: 1,831 runs, 4 passes;
// measured the extra pass costs more than the fix-up). A run longer than kRunCap
// makes the host redo the frame with the full 64-bit sort (8 passes).
#include <algorithm>
#include <cstddef>

#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kRsThreads = 512;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsPer = 8;                       // keys per thread per step
constexpr int kRsStep = kRsThreads * kRsPer;    // keys per CTA step
constexpr int kSlices = 2 * 148;                // G: slices = CTAs of every pass

__device__ __forceinline__ uint64_t slice_begin(uint64_t n, int g) {
    const uint64_t per = (n + kSlices - 1) / kSlices;
    const uint64_t v = per * static_cast<uint64_t>(g);
    return v < n ? v : n;
}

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

// hist[d * kSlices + g] = keys of slice g with digit d (digit-major, so a digit's row
// over the slices is contiguous); tot[d] += the same (tot zeroed by the sort's memset).
__global__ void __launch_bounds__(kRsThreads) radix_upsweep_kernel(const uint32_t* __restrict__ keys,
                                                                    const unsigned long long* __restrict__ dcount,
                                                                    uint64_t hcount, int shift, int bits,
                                                                    uint32_t* __restrict__ hist,
                                                                    uint32_t* __restrict__ tot) {
    __shared__ uint32_t h[256];
    const int g = blockIdx.x;
    const uint64_t n = dcount ? *dcount : hcount;
    const uint32_t mask = (1u << bits) - 1u;
    if (threadIdx.x < 256) h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t b = slice_begin(n, g), e = slice_begin(n, g + 1);
    for (uint64_t i = b + threadIdx.x; i < e; i += kRsThreads) atomicAdd(&h[(keys[i] >> shift) & mask], 1u);
    __syncthreads();
    if (threadIdx.x < 256) {
        const uint32_t c = h[threadIdx.x];
        hist[threadIdx.x * kSlices + g] = c;
        if (c) atomicAdd(&tot[threadIdx.x], c);
    }
}

// Shared memory of one downsweep CTA.
struct DsSmem {
    uint32_t wcnt[kRsWarps][257];  // per-warp digit counters -> per-warp digit offsets in the step
    uint32_t base[256];            // next global output slot per digit
    uint32_t total[256];           // digit counts of the step
    uint32_t toff[256];            // digit offsets inside the step
    uint32_t warp_tmp[kRsWarps];
    uint32_t key[kRsStep];         // the step in digit order (staged for contiguous writes)
    uint32_t val[kRsStep];
};

template <bool kIota>
__global__ void __launch_bounds__(kRsThreads, 2) radix_downsweep_kernel(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, const unsigned long long* __restrict__ dcount, uint64_t hcount, int shift, int bits,
    const uint32_t* __restrict__ hist, const uint32_t* __restrict__ tot) {
    extern __shared__ __align__(16) unsigned char ds_raw[];
    DsSmem& S = *reinterpret_cast<DsSmem*>(ds_raw);
    const int g = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n = dcount ? *dcount : hcount;
    const uint32_t mask = (1u << bits) - 1u;
    const uint64_t b = slice_begin(n, g), e = slice_begin(n, g + 1);
    // keys of the first step, in flight while the offsets are computed; warp w owns the
    // consecutive keys [t0 + w * 32 kRsPer, +32 kRsPer) in kRsPer rounds of 32, so the
    // stable order inside a step is (warp, round, lane) = memory order
    uint32_t key[kRsPer], val[kRsPer];
    auto load = [&](uint64_t t0) {
        const uint64_t w0 = t0 + static_cast<uint64_t>(warp) * (32 * kRsPer) + lane;
#pragma unroll
        for (int j = 0; j < kRsPer; ++j) {
            const uint64_t i = w0 + j * 32;
            const bool ok = i < e;
            key[j] = ok ? kin[i] : 0u;
            val[j] = kIota ? static_cast<uint32_t>(i) : (ok ? vin[i] : 0u);
        }
    };
    load(b);
    for (int k = threadIdx.x; k < kRsWarps * 257; k += kRsThreads) (&S.wcnt[0][0])[k] = 0;
    // this slice's first output slot per digit: keys of smaller digits anywhere, plus
    // keys of this digit in the slices before g
    if (threadIdx.x < 256) S.total[threadIdx.x] = tot[threadIdx.x];
    __syncthreads();
    scan256(S.total, S.base, S.warp_tmp);
    {
        // warp w sums the rows of digits w, w + 16, ... over the slices before g: every
        // lane issues all of its (independent, coalesced) loads before any reduction
        constexpr int kDig = 256 / kRsWarps, kRows = (kSlices + 31) / 32;
        uint32_t acc[kDig];
#pragma unroll
        for (int i = 0; i < kDig; ++i) {
            acc[i] = 0;
            const uint32_t* row = hist + (warp + i * kRsWarps) * kSlices;
#pragma unroll
            for (int q = 0; q < kRows; ++q) {
                const int p = q * 32 + lane;
                if (p < g) acc[i] += row[p];
            }
        }
#pragma unroll
        for (int i = 0; i < kDig; ++i) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
        }
        if (lane == 0)
#pragma unroll
            for (int i = 0; i < kDig; ++i) S.base[warp + i * kRsWarps] += acc[i];
    }
    for (uint64_t t0 = b; t0 < e; t0 += kRsStep) {
        uint32_t ck[kRsPer], cv[kRsPer], dg[kRsPer], rk[kRsPer];
        const uint64_t w0 = t0 + static_cast<uint64_t>(warp) * (32 * kRsPer) + lane;
#pragma unroll
        for (int j = 0; j < kRsPer; ++j) {
            ck[j] = key[j];
            cv[j] = val[j];
            dg[j] = w0 + j * 32 < e ? (ck[j] >> shift) & mask : 256u;
        }
        if (t0 + kRsStep < e) load(t0 + kRsStep);  // the next step's keys, in flight during this one
        // rank: equal digits within a warp by match.any, in (round, lane) order
#pragma unroll
        for (int j = 0; j < kRsPer; ++j) {
            const unsigned peers = __match_any_sync(0xffffffffu, dg[j]);
            const unsigned below = peers & ((1u << lane) - 1u);
            const uint32_t before = S.wcnt[warp][dg[j]];
            rk[j] = before + __popc(below);
            __syncwarp();
            if (below == 0) S.wcnt[warp][dg[j]] = before + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        // across warps: per-digit exclusive offsets; the step's digit counts
        if (threadIdx.x < 256) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kRsWarps; ++w) {
                const uint32_t c = S.wcnt[w][threadIdx.x];
                S.wcnt[w][threadIdx.x] = run;
                run += c;
            }
            S.total[threadIdx.x] = run;
        }
        __syncthreads();
        scan256(S.total, S.toff, S.warp_tmp);
        // stage the step in digit order, then write each digit's run contiguously
#pragma unroll
        for (int j = 0; j < kRsPer; ++j) {
            if (dg[j] < 256u) {
                const uint32_t lp = S.toff[dg[j]] + S.wcnt[warp][dg[j]] + rk[j];
                S.key[lp] = ck[j];
                S.val[lp] = cv[j];
            }
        }
        __syncthreads();
        const uint32_t m = static_cast<uint32_t>(e - t0 < static_cast<uint64_t>(kRsStep) ? e - t0 : kRsStep);
        for (uint32_t i = threadIdx.x; i < m; i += kRsThreads) {
            const uint32_t k = S.key[i];
            const uint32_t d = (k >> shift) & mask;
            const uint32_t pos = S.base[d] + (i - S.toff[d]);
            kout[pos] = k;
            vout[pos] = S.val[i];
        }
        for (int k = threadIdx.x; k < kRsWarps * 257; k += kRsThreads) (&S.wcnt[0][0])[k] = 0;
        __syncthreads();
        if (threadIdx.x < 256) S.base[threadIdx.x] += S.total[threadIdx.x];
    }
}

// ---------------------------------------------------------------------------
// K2 producers and the rank writer.

constexpr int kKeyBits = 24;  // narrow depth key: 3 passes of 8 bits
constexpr uint32_t kCulledKey = (1u << kKeyBits) - 1u;  // culled splats sort last
constexpr int kRunCap = 32;  // longest run of equal narrow depth keys fixed up in place

__device__ __forceinline__ int key32_shift(const Counters* ctr) {
    const unsigned long long kmin = ctr->kmin, kmax = ctr->kmax;
    const unsigned long long range = kmax >= kmin ? kmax - kmin : 0ULL;
    const int bits = range ? 64 - __clzll(static_cast<long long>(range)) : 0;
    return bits > kKeyBits ? bits - kKeyBits : 0;
}

// k32[i] = culled ? kCulledKey : min((key - kmin) >> s, kCulledKey - 1), and the first pass's upsweep
// (slice histograms of digit 0, global counts into ctl->hist[pass0]).
__global__ void __launch_bounds__(kRsThreads) depth_key32_kernel(uint64_t n, const unsigned long long* __restrict__ key,
                                                                 const Counters* __restrict__ ctr,
                                                                 uint32_t* __restrict__ k32, uint32_t* __restrict__ hist,
                                                                 uint32_t* __restrict__ tot) {
    __shared__ uint32_t h[256];
    if (threadIdx.x < 256) h[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long kmin = ctr->kmin;
    const int sh = key32_shift(ctr);
    const int g = blockIdx.x;
    const uint64_t b = slice_begin(n, g), e = slice_begin(n, g + 1);
    for (uint64_t i = b + threadIdx.x; i < e; i += kRsThreads) {
        const unsigned long long k = key[i];
        uint32_t v = kCulledKey;
        if (k != ~0ULL) {
            const unsigned long long d = (k - kmin) >> sh;
            v = d < kCulledKey - 1 ? static_cast<uint32_t>(d) : kCulledKey - 1;
        }
        k32[i] = v;
        atomicAdd(&h[v & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 256) {
        const uint32_t c = h[threadIdx.x];
        hist[threadIdx.x * kSlices + g] = c;
        if (c) atomicAdd(&tot[threadIdx.x], c);
    }
}

// Wide path: the low (half 0) or high (half 1, gathered through the sorted values)
// 32 bits of the raw 64-bit keys, with the upsweep of their first digit.
__global__ void __launch_bounds__(kRsThreads) depth_key_half_kernel(uint64_t n, const unsigned long long* __restrict__ key,
                                                                    const uint32_t* __restrict__ idx, int half,
                                                                    uint32_t* __restrict__ k32, uint32_t* __restrict__ hist,
                                                                    uint32_t* __restrict__ tot) {
    __shared__ uint32_t h[256];
    if (threadIdx.x < 256) h[threadIdx.x] = 0;
    __syncthreads();
    const int g = blockIdx.x;
    const uint64_t b = slice_begin(n, g), e = slice_begin(n, g + 1);
    for (uint64_t i = b + threadIdx.x; i < e; i += kRsThreads) {
        const uint32_t v = half ? static_cast<uint32_t>(key[idx[i]] >> 32) : static_cast<uint32_t>(key[i]);
        k32[i] = v;
        atomicAdd(&h[v & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 256) {
        const uint32_t c = h[threadIdx.x];
        hist[threadIdx.x * kSlices + g] = c;
        if (c) atomicAdd(&tot[threadIdx.x], c);
    }
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
    if (k == kCulledKey) {  // culled: after the visible splats, in index order
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

}  // namespace

size_t radix_hist_words() { return static_cast<size_t>(kSlices) * 256; }

cudaError_t launch_radix_pass(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                              const unsigned long long* dcount, uint64_t hcount, int shift, int bits, SortCtl* ctl,
                              int pass, uint32_t* hist, bool histogram_ready, cudaStream_t stream) {
    uint32_t* tot = ctl->hist[pass];
    if (!histogram_ready) {
        radix_upsweep_kernel<<<kSlices, kRsThreads, 0, stream>>>(kin, dcount, hcount, shift, bits, hist, tot);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    static const cudaError_t attr = [] {
        cudaError_t e = cudaFuncSetAttribute(radix_downsweep_kernel<false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(DsSmem));
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(radix_downsweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     sizeof(DsSmem));
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    if (vin)
        radix_downsweep_kernel<false><<<kSlices, kRsThreads, sizeof(DsSmem), stream>>>(
            kin, vin, kout, vout, dcount, hcount, shift, bits, hist, tot);
    else
        radix_downsweep_kernel<true><<<kSlices, kRsThreads, sizeof(DsSmem), stream>>>(
            kin, nullptr, kout, vout, dcount, hcount, shift, bits, hist, tot);
    return cudaGetLastError();
}

// K2: depth order of n splats. Narrow: 24-bit keys (+ first upsweep), 3 passes, ranks
// with the run fix-up (7 launches); wide: low half 4 passes, high half 4 passes, ranks.
cudaError_t launch_depth_sort(uint64_t n, const unsigned long long* key, Counters* ctr, bool wide, uint32_t* ka,
                              uint32_t* va, uint32_t* kb, uint32_t* vb, SortCtl* ctl, uint32_t* hist,
                              const int4* rects, uint32_t* order, int4* brect, uint2* bmeta, cudaStream_t stream,
                              uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(&ctl->ticket[0], 0, sizeof(SortCtl) - offsetof(SortCtl, ticket), stream);
    if (e != cudaSuccess) return e;
    // np passes over 8-bit digits, ping-ponging (ka, va) <-> (kb, vb) from (ka, iota); the
    // first pass's histograms come from the key producer. Returns where the result is.
    auto passes = [&](int np, int pass0, bool iota_first, cudaError_t* ee) -> bool {
        *ee = cudaSuccess;
        for (int p = 0; p < np && *ee == cudaSuccess; ++p) {
            const bool even = (p & 1) == 0;
            *ee = launch_radix_pass(even ? ka : kb, (p == 0 && iota_first) ? nullptr : (even ? va : vb),
                                    even ? kb : ka, even ? vb : va, nullptr, n, 8 * p, 8, ctl, pass0 + p, hist,
                                    p == 0, stream);
        }
        return (np & 1) != 0;  // true: in (kb, vb)
    };
    bool in_b = false;
    if (!wide) {
        depth_key32_kernel<<<kSlices, kRsThreads, 0, stream>>>(n, key, ctr, ka, hist, ctl->hist[0]);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        in_b = passes(kKeyBits / 8, 0, true, &e);
        if (e != cudaSuccess) return e;
        *launches += 2 + 2 * (kKeyBits / 8) - 1;
    } else {
        depth_key_half_kernel<<<kSlices, kRsThreads, 0, stream>>>(n, key, nullptr, 0, ka, hist, ctl->hist[0]);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        passes(4, 0, true, &e);
        if (e != cudaSuccess) return e;
        depth_key_half_kernel<<<kSlices, kRsThreads, 0, stream>>>(n, key, va, 1, ka, hist, ctl->hist[4]);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        passes(4, 4, false, &e);
        if (e != cudaSuccess) return e;
        *launches += 17;
    }
    depth_rank_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
        n, in_b ? kb : ka, in_b ? vb : va, key, wide ? 1 : 0, ctr, rects, order, brect, bmeta);
    return cudaGetLastError();
}

}  // namespace sgs
