// radix.cu -- the library's own device radix sort (no CUB on any path), and the
// depth-order stage K2 built on it.
//
// Stable LSD radix sort of (u32 key, u32 value) pairs, three small kernels per digit
// pass and nothing that spins: the keys are cut into G = 296 contiguous slices (2 CTAs
// per SM); the upsweep writes each slice's digit histogram (digit-major); one CTA per
// digit scans its row of slice counts; the downsweep CTA of slice g takes its output
// offsets from that (the exclusive scan of the digit totals plus its row entries) and
// walks its slice in order -- ranking equal digits within a warp by match.any + popc
// and across warps by a shared-memory prefix, so the scatter is stable. Large sorts
// stage each 4096-key step in digit order so each digit's run leaves contiguously;
// a frame's tile-id sorts (about one 2048-key step per slice) scatter straight from
// registers. The count of keys is read from device memory: a frame sorts a
// device-sized list with no host round trip. Measured: a decoupled look-back
// (onesweep) version was 2-3x slower here -- whole waves of tiles start together, so
// the look-backs run deep -- and so was summing the slice counts inside each
// downsweep CTA (every CTA reading the whole 300 KB matrix).
//
// The 64-bit depth sort (K2's fallback, raster.cpp:93-101: stable order by (double
// depth, index)) is built on it: the low then the high 32 bits of the orderable keys,
// 4 passes each, with the Gaussian index as value -- stable, so equal keys stay in
// index order -- then the ranks and rank-ordered binning inputs.
#include <algorithm>
#include <cstddef>

#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kRsThreads = 512;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsStepMax = kRsThreads * 8;     // keys per CTA step (staged variant)
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
// over the slices is contiguous).
__global__ void __launch_bounds__(kRsThreads) radix_upsweep_kernel(const uint32_t* __restrict__ keys,
                                                                    const unsigned long long* __restrict__ dcount,
                                                                    uint64_t hcount, int shift, int bits,
                                                                    uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    const int g = blockIdx.x;
    const uint64_t n = dcount ? *dcount : hcount;
    const uint32_t mask = (1u << bits) - 1u;
    if (threadIdx.x < 256) h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t b = slice_begin(n, g), e = slice_begin(n, g + 1);
    for (uint64_t i = b + threadIdx.x; i < e; i += kRsThreads) atomicAdd(&h[(keys[i] >> shift) & mask], 1u);
    __syncthreads();
    if (threadIdx.x < 256) hist[threadIdx.x * kSlices + g] = h[threadIdx.x];
}

// Row scan: CTA d turns digit d's row of slice counts into exclusive offsets in place
// and writes the digit total to hist[256 * kSlices + d].
constexpr int kRowThreads = (kSlices + 31) / 32 * 32;
__global__ void __launch_bounds__(kRowThreads) radix_rowscan_kernel(uint32_t* __restrict__ hist) {
    __shared__ uint32_t wsum[kRowThreads / 32];
    const int d = blockIdx.x, p = threadIdx.x, lane = p & 31, w = p >> 5;
    uint32_t* row = hist + d * kSlices;
    const uint32_t x = p < kSlices ? row[p] : 0u;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    uint32_t add = 0;
    for (int k = 0; k < w; ++k) add += wsum[k];
    if (p < kSlices) row[p] = add + inc - x;
    if (p == kRowThreads - 1) hist[256 * kSlices + d] = add + inc;
}

// Shared memory of one downsweep CTA.
struct DsSmem {
    uint32_t wcnt[kRsWarps][257];  // per-warp digit counters -> per-warp digit offsets in the step
    uint32_t base[256];            // next global output slot per digit
    uint32_t total[256];           // digit counts of the step
    uint32_t toff[256];            // digit offsets inside the step
    uint32_t warp_tmp[kRsWarps];
    uint32_t key[kRsStepMax];      // the step in digit order (staged variant only)
    uint32_t val[kRsStepMax];
};

// kStage: stage each step in digit order for contiguous writes (large slices); else
// scatter straight from registers (slices of a step or two, where the extra barriers
// and scan cost more than the scattered writes). kPer keys per thread per step.
template <bool kIota, bool kStage, int kPer>
__global__ void __launch_bounds__(kRsThreads, kStage ? 2 : 3) radix_downsweep_kernel(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, const unsigned long long* __restrict__ dcount, uint64_t hcount, int shift, int bits,
    const uint32_t* __restrict__ hist) {
    extern __shared__ __align__(16) unsigned char ds_raw[];
    DsSmem& S = *reinterpret_cast<DsSmem*>(ds_raw);
    constexpr int kStep = kRsThreads * kPer;
    const int g = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n = dcount ? *dcount : hcount;
    const uint32_t mask = (1u << bits) - 1u;
    const uint64_t b = slice_begin(n, g), e = slice_begin(n, g + 1);
    // keys of the first step, in flight while the offsets are computed; warp w owns the
    // consecutive keys [t0 + w * 32 kPer, +32 kPer) in kPer rounds of 32, so the
    // stable order inside a step is (warp, round, lane) = memory order
    uint32_t key[kPer], val[kPer];
    auto load = [&](uint64_t t0) {
        const uint64_t w0 = t0 + static_cast<uint64_t>(warp) * (32 * kPer) + lane;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint64_t i = w0 + j * 32;
            const bool ok = i < e;
            key[j] = ok ? kin[i] : 0u;
            val[j] = kIota ? static_cast<uint32_t>(i) : (ok ? vin[i] : 0u);
        }
    };
    load(b);
    for (int k = threadIdx.x; k < kRsWarps * 257; k += kRsThreads) (&S.wcnt[0][0])[k] = 0;
    // this slice's first output slot per digit: keys of smaller digits anywhere (scan
    // of the digit totals) plus keys of this digit in the slices before g (row scan)
    if (threadIdx.x < 256) S.total[threadIdx.x] = hist[256 * kSlices + threadIdx.x];
    __syncthreads();
    scan256(S.total, S.base, S.warp_tmp);
    if (threadIdx.x < 256) S.base[threadIdx.x] += hist[threadIdx.x * kSlices + g];
    for (uint64_t t0 = b; t0 < e; t0 += kStep) {
        uint32_t ck[kPer], cv[kPer], dg[kPer], rk[kPer];
        const uint64_t w0 = t0 + static_cast<uint64_t>(warp) * (32 * kPer) + lane;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            ck[j] = key[j];
            cv[j] = val[j];
            dg[j] = w0 + j * 32 < e ? (ck[j] >> shift) & mask : 256u;
        }
        if (t0 + kStep < e) load(t0 + kStep);  // the next step's keys, in flight during this one
        // rank: equal digits within a warp by match.any, in (round, lane) order
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
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
        if constexpr (kStage) {
            scan256(S.total, S.toff, S.warp_tmp);
            // stage the step in digit order, then write each digit's run contiguously
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                if (dg[j] < 256u) {
                    const uint32_t lp = S.toff[dg[j]] + S.wcnt[warp][dg[j]] + rk[j];
                    S.key[lp] = ck[j];
                    S.val[lp] = cv[j];
                }
            }
            __syncthreads();
            const uint32_t m = static_cast<uint32_t>(e - t0 < static_cast<uint64_t>(kStep) ? e - t0 : kStep);
            for (uint32_t i = threadIdx.x; i < m; i += kRsThreads) {
                const uint32_t k = S.key[i];
                const uint32_t d = (k >> shift) & mask;
                const uint32_t pos = S.base[d] + (i - S.toff[d]);
                kout[pos] = k;
                vout[pos] = S.val[i];
            }
        } else {
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                if (dg[j] < 256u) {
                    const uint32_t pos = S.base[dg[j]] + S.wcnt[warp][dg[j]] + rk[j];
                    kout[pos] = ck[j];
                    vout[pos] = cv[j];
                }
            }
            __syncthreads();
        }
        for (int k = threadIdx.x; k < kRsWarps * 257; k += kRsThreads) (&S.wcnt[0][0])[k] = 0;
        __syncthreads();
        if (threadIdx.x < 256) S.base[threadIdx.x] += S.total[threadIdx.x];
    }
}

// ---------------------------------------------------------------------------
// K2 producers and the rank writer.

// The low (half 0) or high (half 1, gathered through the sorted values)
// 32 bits of the raw 64-bit keys, with the upsweep of their first digit.
__global__ void __launch_bounds__(kRsThreads) depth_key_half_kernel(uint64_t n, const unsigned long long* __restrict__ key,
                                                                    const uint32_t* __restrict__ idx, int half,
                                                                    uint32_t* __restrict__ k32, uint32_t* __restrict__ hist) {
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
    if (threadIdx.x < 256) hist[threadIdx.x * kSlices + g] = h[threadIdx.x];
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

// Ranks from the sorted (key, index) pairs: order, and the rank-ordered binning inputs.
__global__ void depth_rank_kernel(uint64_t n, const uint32_t* __restrict__ sv, const Counters* __restrict__ ctr,
                                  const int4* __restrict__ rects, uint32_t* __restrict__ order,
                                  int4* __restrict__ brect, uint2* __restrict__ bmeta) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < n) put_rank(r, sv[r], r < ctr->visible, rects, order, brect, bmeta);
}

}  // namespace

size_t radix_hist_words() { return static_cast<size_t>(kSlices + 1) * 256; }

cudaError_t launch_radix_pass(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                              const unsigned long long* dcount, uint64_t hcount, int shift, int bits,
                              uint32_t* hist, bool histogram_ready, cudaStream_t stream) {
    if (!histogram_ready) {
        radix_upsweep_kernel<<<kSlices, kRsThreads, 0, stream>>>(kin, dcount, hcount, shift, bits, hist);
    }
    radix_rowscan_kernel<<<256, kRowThreads, 0, stream>>>(hist);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // staged 4096-key steps for large sorts; direct scatter of 2048-key steps when the
    // count is device-side (a chunk's tile pairs: ~1 step per slice at 1080p)
    constexpr size_t kSmemStaged = sizeof(DsSmem), kSmemDirect = offsetof(DsSmem, key);
    static const cudaError_t attr = [] {
        cudaError_t e = cudaFuncSetAttribute(radix_downsweep_kernel<false, true, 8>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemStaged);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(radix_downsweep_kernel<true, true, 8>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemStaged);
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    if (dcount) {
        if (vin)
            radix_downsweep_kernel<false, false, 4><<<kSlices, kRsThreads, kSmemDirect, stream>>>(
                kin, vin, kout, vout, dcount, hcount, shift, bits, hist);
        else
            radix_downsweep_kernel<true, false, 4><<<kSlices, kRsThreads, kSmemDirect, stream>>>(
                kin, nullptr, kout, vout, dcount, hcount, shift, bits, hist);
    } else if (vin) {
        radix_downsweep_kernel<false, true, 8><<<kSlices, kRsThreads, kSmemStaged, stream>>>(
            kin, vin, kout, vout, dcount, hcount, shift, bits, hist);
    } else {
        radix_downsweep_kernel<true, true, 8><<<kSlices, kRsThreads, kSmemStaged, stream>>>(
            kin, nullptr, kout, vout, dcount, hcount, shift, bits, hist);
    }
    return cudaGetLastError();
}

// K2's fallback: the 64-bit depth sort (low half 4 passes, high half 4 passes, ranks).
cudaError_t launch_depth_sort_wide(uint64_t n, const unsigned long long* key, Counters* ctr, uint32_t* ka,
                                   uint32_t* va, uint32_t* kb, uint32_t* vb, uint32_t* hist,
                                   const int4* rects, uint32_t* order, int4* brect, uint2* bmeta,
                                   cudaStream_t stream, uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    // 4 passes over 8-bit digits, (ka, va) -> (kb, vb) -> ... -> (ka, va); the first
    // pass's histograms come from the key producer
    auto four = [&](bool iota_first) -> cudaError_t {
        cudaError_t ee = cudaSuccess;
        for (int p = 0; p < 4 && ee == cudaSuccess; ++p) {
            const bool even = (p & 1) == 0;
            ee = launch_radix_pass(even ? ka : kb, (p == 0 && iota_first) ? nullptr : (even ? va : vb),
                                   even ? kb : ka, even ? vb : va, nullptr, n, 8 * p, 8, hist,
                                   p == 0, stream);
        }
        return ee;
    };
    depth_key_half_kernel<<<kSlices, kRsThreads, 0, stream>>>(n, key, nullptr, 0, ka, hist);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = four(true)) != cudaSuccess) return e;
    depth_key_half_kernel<<<kSlices, kRsThreads, 0, stream>>>(n, key, va, 1, ka, hist);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = four(false)) != cudaSuccess) return e;
    depth_rank_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(n, va, ctr, rects, order, brect,
                                                                                  bmeta);
    *launches += 17;
    return cudaGetLastError();
}

}  // namespace sgs
