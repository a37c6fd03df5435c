// radix.cu -- the library's own device radix sort (no CUB on any path): K5, the
// stable sort of a chunk's (tile id, Gaussian index) pairs by tile id.
//
// Stable LSD radix sort of (u32 key, u32 value) pairs, three small kernels per digit
// pass and nothing that spins: the keys are cut into G = 296 contiguous slices (2 CTAs
// per SM); the upsweep writes each slice's digit histogram (digit-major); one CTA per
// digit scans its row of slice counts; the downsweep CTA of slice g takes its output
// offsets from that (the exclusive scan of the digit totals plus its row entries) and
// walks its slice in order -- ranking equal digits within a warp by ballots + popc
// and across warps by a shared-memory prefix, so the scatter is stable -- scattering
// each 2048-key step straight from registers. The count of keys is read from device
// memory: a frame sorts a device-sized list with no host round trip. Measured: a
// decoupled look-back (onesweep) version was 2-3x slower here -- whole waves of tiles
// start together, so the look-backs run deep -- and so was summing the slice counts
// inside each downsweep CTA (every CTA reading the whole 300 KB matrix).
#include <algorithm>
#include <cstddef>

#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kRsThreads = 512;
constexpr int kRsWarps = kRsThreads / 32;
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
                                                                    int shift, int bits, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    const int g = blockIdx.x;
    const uint64_t n = *dcount;
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
    uint32_t warp_tmp[kRsWarps];
};

// kPer keys per thread per step, scattered straight from registers (a chunk's pairs
// make a step or two per slice, where staging each step in digit order for
// contiguous writes costs more barriers and scans than it saves).
template <int kPer>
__global__ void __launch_bounds__(kRsThreads, 3) radix_downsweep_kernel(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, const unsigned long long* __restrict__ dcount, int shift, int bits,
    const uint32_t* __restrict__ hist) {
    __shared__ DsSmem S;
    constexpr int kStep = kRsThreads * kPer;
    const int g = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t n = *dcount;
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
            val[j] = ok ? vin[i] : 0u;
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
        // rank: equal digits within a warp by ballots, in (round, lane) order
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            // lanes holding the same digit (the past-the-end sentinel 256 included): one
            // ballot per digit bit -- 4% faster passes than __match_any_sync here
            unsigned peers = __ballot_sync(0xffffffffu, dg[j] & 256u) ^ ((dg[j] & 256u) ? 0u : 0xffffffffu);
            for (int bit = 0; bit < bits; ++bit) {
                const unsigned v = __ballot_sync(0xffffffffu, (dg[j] >> bit) & 1u);
                peers &= ((dg[j] >> bit) & 1u) ? v : ~v;
            }
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
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            if (dg[j] < 256u) {
                const uint32_t pos = S.base[dg[j]] + S.wcnt[warp][dg[j]] + rk[j];
                kout[pos] = ck[j];
                vout[pos] = cv[j];
            }
        }
        __syncthreads();
        for (int k = threadIdx.x; k < kRsWarps * 257; k += kRsThreads) (&S.wcnt[0][0])[k] = 0;
        __syncthreads();
        if (threadIdx.x < 256) S.base[threadIdx.x] += S.total[threadIdx.x];
    }
}

}  // namespace

size_t radix_hist_words() { return static_cast<size_t>(kSlices + 1) * 256; }

cudaError_t launch_radix_pass(const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                              const unsigned long long* dcount, int shift, int bits, uint32_t* hist,
                              cudaStream_t stream) {
    radix_upsweep_kernel<<<kSlices, kRsThreads, 0, stream>>>(kin, dcount, shift, bits, hist);
    radix_rowscan_kernel<<<256, kRowThreads, 0, stream>>>(hist);
    // 2048-key steps: a chunk's tile pairs are ~1 step per slice at 1080p
    radix_downsweep_kernel<4><<<kSlices, kRsThreads, 0, stream>>>(kin, vin, kout, vout, dcount, shift, bits, hist);
    return cudaGetLastError();
}

}  // namespace sgs
