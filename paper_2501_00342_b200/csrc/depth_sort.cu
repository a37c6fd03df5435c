// depth_sort.cu -- K2: the global blending order (depth, index) of raster.cpp:93-101.
//
// Exact bucket sort. The orderable 64-bit depth keys of the visible splats span
// [kmin, kmax] (found by K1). They are split into B = 2^b buckets by their offset
// from kmin (monotone in the key, so bucket order is key order):
//   K2a histogram (global atomics), K2b exclusive scan (CUB), K2c scatter of the
//   Gaussian indices into their buckets (atomics: unordered inside a bucket),
//   K2d one warp per bucket sorts it by (key, index) with a 64-element bitonic
//   network in registers.
// B is chosen so the mean bucket holds <= 4 splats; one thread insertion-sorts a
// bucket of <= kSmall, one warp a bucket of <= kBucketCap; a bucket larger than 64
// (e.g. thousands of splats at one identical depth) sets a flag and the host redoes
// the frame with the 64-bit CUB radix sort (capi.cu, kRetryWide). Culled splats
// (key ~0) go after the visible ones; they own no tiles.
#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kBucketCap = 64;
constexpr int kSmall = 12;

__device__ __forceinline__ uint32_t bucket_of(unsigned long long k, unsigned long long kmin, int shift) {
    return static_cast<uint32_t>((k - kmin) >> shift);
}

__device__ __forceinline__ int bucket_shift(const Counters* ctr, int log2b) {
    const unsigned long long kmin = ctr->kmin, kmax = ctr->kmax;
    const unsigned long long range = kmax >= kmin ? kmax - kmin : 0ULL;
    const int bits = range ? 64 - __clzll(static_cast<long long>(range)) : 0;
    return bits > log2b ? bits - log2b : 0;
}

__global__ void bucket_hist_kernel(uint64_t n, const unsigned long long* __restrict__ key,
                                   const Counters* __restrict__ ctr, int log2b, uint32_t* __restrict__ hist) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = key[i];
    if (k == ~0ULL) return;
    atomicAdd(&hist[bucket_of(k, ctr->kmin, bucket_shift(ctr, log2b))], 1u);
}

// hist now holds exclusive offsets; cursor (zeroed) counts placements per bucket.
__global__ void bucket_scatter_kernel(uint64_t n, const unsigned long long* __restrict__ key,
                                      Counters* __restrict__ ctr, int log2b, const uint32_t* __restrict__ off,
                                      uint32_t* __restrict__ cursor, uint32_t* __restrict__ out,
                                      unsigned long long* __restrict__ out_key) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = key[i];
    uint64_t pos;
    if (k == ~0ULL) {
        pos = ctr->visible + atomicAdd(&ctr->culled_cursor, 1ULL);
    } else {
        const uint32_t b = bucket_of(k, ctr->kmin, bucket_shift(ctr, log2b));
        pos = off[b] + atomicAdd(&cursor[b], 1u);
    }
    out[pos] = static_cast<uint32_t>(i);
    out_key[pos] = k;  // keys travel with the indices: the bucket sort reads them contiguously
}

__device__ __forceinline__ bool less_ki(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// One thread per bucket: insertion sort by (key, index) for buckets of <= kSmall;
// larger buckets are queued for the warp kernel below.
__global__ void bucket_sort_small_kernel(uint32_t nbuckets, const uint32_t* __restrict__ off,
                                         const unsigned long long* __restrict__ skey, uint32_t* __restrict__ order,
                                         Counters* __restrict__ ctr, uint32_t* __restrict__ big) {
    const uint32_t b = static_cast<uint32_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nbuckets) return;
    const uint32_t s = off[b], m = off[b + 1] - s;
    if (m <= 1) return;
    if (m > kSmall) {
        big[atomicAdd(&ctr->big_buckets, 1ULL)] = b;
        return;
    }
    uint32_t idx[kSmall];
    unsigned long long k[kSmall];
    for (uint32_t a = 0; a < m; ++a) {
        const uint32_t vi = order[s + a];
        const unsigned long long vk = skey[s + a];
        int c = static_cast<int>(a) - 1;
        while (c >= 0 && less_ki(vk, vi, k[c], idx[c])) {
            k[c + 1] = k[c];
            idx[c + 1] = idx[c];
            --c;
        }
        k[c + 1] = vk;
        idx[c + 1] = vi;
    }
    for (uint32_t a = 0; a < m; ++a) order[s + a] = idx[a];
}

__device__ void bitonic_bucket(uint32_t b, const uint32_t* __restrict__ off, const unsigned long long* __restrict__ key,
                               uint32_t* __restrict__ order, Counters* __restrict__ ctr, int lane) {
    const uint32_t s = off[b], m = off[b + 1] - s;
    if (m > kBucketCap) {
        if (lane == 0) atomicAdd(&ctr->tie_overflow, 1ULL);
        return;
    }
    uint32_t idx[2];
    unsigned long long k[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t el = h * 32 + lane;
        idx[h] = el < m ? order[s + el] : 0xFFFFFFFFu;
        k[h] = el < m ? key[s + el] : ~0ULL;  // bucket-ordered keys (scatter output)
    }
#pragma unroll
    for (int kk = 2; kk <= 64; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            if (j == 32) {
                // pair (lane, lane + 32) lives in this lane; kk == 64 here: ascending
                if (less_ki(k[1], idx[1], k[0], idx[0])) {
                    const unsigned long long tk = k[0];
                    const uint32_t ti = idx[0];
                    k[0] = k[1];
                    idx[0] = idx[1];
                    k[1] = tk;
                    idx[1] = ti;
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int el = h * 32 + lane;
                    const unsigned long long pk = __shfl_xor_sync(0xffffffffu, k[h], j);
                    const uint32_t pi = __shfl_xor_sync(0xffffffffu, idx[h], j);
                    const bool want_min = ((el & j) == 0) == ((el & kk) == 0);
                    const bool take = want_min ? less_ki(pk, pi, k[h], idx[h]) : less_ki(k[h], idx[h], pk, pi);
                    if (take) {
                        k[h] = pk;
                        idx[h] = pi;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t el = h * 32 + lane;
        if (el < m) order[s + el] = idx[h];
    }
}

// One warp per queued bucket (kSmall < size <= 64): 64-element bitonic sort by
// (key, index), element e held by lane (e & 31) in register half (e >> 5).
__global__ void bucket_sort_big_kernel(const uint32_t* __restrict__ off, const unsigned long long* __restrict__ key,
                                       uint32_t* __restrict__ order, Counters* __restrict__ ctr,
                                       const uint32_t* __restrict__ big) {
    const int lane = threadIdx.x & 31;
    const uint64_t nbig = ctr->big_buckets;
    for (uint64_t w = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < nbig;
         w += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
        bitonic_bucket(big[w], off, key, order, ctr, lane);
    }
}

}  // namespace

int depth_bucket_log2(uint64_t n) {
    int l = 10;
    while (l < 24 && (1ULL << l) * 4 < n) ++l;
    return l;
}

void launch_bucket_hist(uint64_t n, const unsigned long long* key, const Counters* ctr, int log2b, uint32_t* hist,
                        cudaStream_t stream) {
    if (n) bucket_hist_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(n, key, ctr, log2b, hist);
}

void launch_bucket_scatter(uint64_t n, const unsigned long long* key, Counters* ctr, int log2b, const uint32_t* off,
                           uint32_t* cursor, uint32_t* out, unsigned long long* out_key, cudaStream_t stream) {
    if (n)
        bucket_scatter_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(n, key, ctr, log2b, off,
                                                                                        cursor, out, out_key);
}

void launch_bucket_sort(uint32_t nbuckets, const uint32_t* off, const unsigned long long* key, uint32_t* order,
                        Counters* ctr, uint32_t* big, cudaStream_t stream) {
    bucket_sort_small_kernel<<<(nbuckets + 255) / 256, 256, 0, stream>>>(nbuckets, off, key, order, ctr, big);
    bucket_sort_big_kernel<<<148 * 4, 256, 0, stream>>>(off, key, order, ctr, big);
}

}  // namespace sgs
