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
#include <cub/device/device_scan.cuh>

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

// ---------------------------------------------------------------------------
// Two-level exact sort (the default). Level 1 partitions the keys into C coarse
// buckets (uniform in key offset from kmin; culled keys form bucket C): each CTA
// counts its tile in shared memory and adds the counts to the global histogram
// (one atomic per non-empty (CTA, bucket)); after the scan, the scatter CTA
// reserves a contiguous range per (CTA, bucket) with one atomic and places its keys
// by shared-memory offsets. Level 2 gives each coarse bucket (<= kL2Cap keys) to
// one CTA, which sorts it completely in shared memory (fine buckets, then insertion
// sort / warp bitonic by (key, index)) and writes the ranks together with the
// rank-ordered binning inputs. A coarse bucket above kL2Cap or a fine bucket above
// 64 keys raises tie_overflow: the host redoes the frame with the 64-bit CUB sort.

constexpr int kL1Threads = 1024;
constexpr int kL1Per = 8;
constexpr int kL1Tile = kL1Threads * kL1Per;
constexpr int kL2Threads = 512;
constexpr int kL2Cap = 4096;
constexpr int kL2Per = kL2Cap / kL2Threads;
constexpr int kL2MaxFineLog2 = 11;

__device__ __forceinline__ unsigned long long shr64(unsigned long long v, int s) { return s < 64 ? v >> s : 0ULL; }

__device__ __forceinline__ uint32_t coarse_of(unsigned long long k, unsigned long long kmin, int shift, uint32_t C) {
    return k == ~0ULL ? C : static_cast<uint32_t>(shr64(k - kmin, shift));
}

__global__ void __launch_bounds__(kL1Threads) coarse_hist_kernel(uint64_t n, const unsigned long long* __restrict__ key,
                                                                 const Counters* __restrict__ ctr, int log2c,
                                                                 uint32_t* __restrict__ ghist) {
    extern __shared__ uint32_t sh_hist[];
    const uint32_t C = 1u << log2c;
    for (uint32_t b = threadIdx.x; b <= C; b += kL1Threads) sh_hist[b] = 0;
    const unsigned long long kmin = ctr->kmin;
    const int shift = bucket_shift(ctr, log2c);
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kL1Tile + threadIdx.x;
    unsigned long long k[kL1Per];
#pragma unroll
    for (int j = 0; j < kL1Per; ++j) {
        const uint64_t i = base + j * kL1Threads;
        k[j] = i < n ? key[i] : 0ULL;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kL1Per; ++j)
        if (base + j * kL1Threads < n) atomicAdd(&sh_hist[coarse_of(k[j], kmin, shift, C)], 1u);
    __syncthreads();
    for (uint32_t b = threadIdx.x; b <= C; b += kL1Threads)
        if (sh_hist[b]) atomicAdd(&ghist[b], sh_hist[b]);
}

// cur = exclusive offsets of the coarse buckets, advanced to their ends. Visible
// keys go to (part_key, part_idx); culled ones straight to their final ranks
// [V, N) with (index, 0 tiles) metadata.
__global__ void __launch_bounds__(kL1Threads) coarse_scatter_kernel(
    uint64_t n, const unsigned long long* __restrict__ key, const Counters* __restrict__ ctr, int log2c,
    uint32_t* __restrict__ cur, unsigned long long* __restrict__ part_key, uint32_t* __restrict__ part_idx,
    uint2* __restrict__ bmeta) {
    extern __shared__ uint32_t sh[];
    const uint32_t C = 1u << log2c;
    uint32_t* cnt = sh;
    uint32_t* gbase = sh + (C + 1);
    for (uint32_t b = threadIdx.x; b <= C; b += kL1Threads) cnt[b] = 0;
    const unsigned long long kmin = ctr->kmin;
    const int shift = bucket_shift(ctr, log2c);
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kL1Tile + threadIdx.x;
    unsigned long long k[kL1Per];
    uint32_t bk[kL1Per], lo[kL1Per];
#pragma unroll
    for (int j = 0; j < kL1Per; ++j) {
        const uint64_t i = base + j * kL1Threads;
        k[j] = i < n ? key[i] : 0ULL;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kL1Per; ++j) {
        bk[j] = coarse_of(k[j], kmin, shift, C);
        lo[j] = base + j * kL1Threads < n ? atomicAdd(&cnt[bk[j]], 1u) : 0u;
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b <= C; b += kL1Threads)
        if (cnt[b]) gbase[b] = atomicAdd(&cur[b], cnt[b]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kL1Per; ++j) {
        const uint64_t i = base + j * kL1Threads;
        if (i >= n) continue;
        const uint32_t pos = gbase[bk[j]] + lo[j];
        part_idx[pos] = static_cast<uint32_t>(i);
        if (bk[j] == C)
            bmeta[pos] = make_uint2(static_cast<uint32_t>(i), 0u);
        else
            part_key[pos] = k[j];
    }
}

// Exclusive scan of v[0, m) in shared memory (m <= 4 * kL2Threads), in place.
__device__ void block_exclusive_scan(uint32_t* v, int m, uint32_t* warp_tot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t x[4], sum = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int e = tid * 4 + j;
        x[j] = e < m ? v[e] : 0u;
        sum += x[j];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kL2Threads / 32 ? warp_tot[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kL2Threads / 32) warp_tot[lane] = wi - w;
    }
    __syncthreads();
    uint32_t run = warp_tot[warp] + inc - sum;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int e = tid * 4 + j;
        if (e < m) v[e] = run;
        run += x[j];
    }
    __syncthreads();
}

// visible splats always have their rect written by K1: both gathers issue together
__device__ __forceinline__ void put_rank(uint32_t r, uint32_t g, const int4* __restrict__ rects,
                                         uint32_t* __restrict__ order, int4* __restrict__ brect,
                                         uint2* __restrict__ bmeta) {
    const int4 rc = rects[g];
    const uint32_t c = rect_area(rc);
    order[r] = g;
    bmeta[r] = make_uint2(g, c);
    brect[r] = rc;
}

__global__ void __launch_bounds__(kL2Threads) local_sort_kernel(
    const uint32_t* __restrict__ cend, const unsigned long long* __restrict__ part_key, uint32_t* __restrict__ order,
    Counters* __restrict__ ctr, int log2c, const int4* __restrict__ rects,
    int4* __restrict__ brect, uint2* __restrict__ bmeta) {
    extern __shared__ unsigned long long sKey[];  // kL2Cap keys, then kL2Cap indices
    uint32_t* sIdx = reinterpret_cast<uint32_t*>(sKey + kL2Cap);
    __shared__ uint32_t sCur[1 << kL2MaxFineLog2];
    __shared__ uint32_t sBig[kL2Cap / (kSmall + 1) + 1];
    __shared__ uint32_t sWarp[kL2Threads / 32];
    __shared__ uint32_t sNBig;
    const uint32_t b = blockIdx.x;
    const uint32_t s = b ? cend[b - 1] : 0u;
    const uint32_t m = cend[b] - s;
    if (m == 0) return;
    const int tid = threadIdx.x;
    if (m > kL2Cap) {
        if (tid == 0) atomicAdd(&ctr->tie_overflow, 1ULL);
        return;
    }
    const unsigned long long kmin = ctr->kmin;
    const int shiftC = bucket_shift(ctr, log2c);
    int F = 0;
    while (F < kL2MaxFineLog2 && (1u << F) * 2 < m) ++F;
    F = F < shiftC ? F : shiftC;
    const int shiftF = shiftC - F;
    const uint32_t nf = 1u << F, fmask = nf - 1;
    for (uint32_t f = tid; f < nf; f += kL2Threads) sCur[f] = 0;
    if (tid == 0) sNBig = 0;
    unsigned long long k[kL2Per];
    uint32_t ix[kL2Per];
#pragma unroll
    for (int j = 0; j < kL2Per; ++j) {
        const uint32_t e = tid + j * kL2Threads;
        k[j] = e < m ? part_key[s + e] : 0ULL;
        ix[j] = e < m ? order[s + e] : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kL2Per; ++j)
        if (tid + j * kL2Threads < m) atomicAdd(&sCur[static_cast<uint32_t>(shr64(k[j] - kmin, shiftF)) & fmask], 1u);
    __syncthreads();
    block_exclusive_scan(sCur, static_cast<int>(nf), sWarp);
#pragma unroll
    for (int j = 0; j < kL2Per; ++j) {
        if (tid + j * kL2Threads < m) {
            const uint32_t p = atomicAdd(&sCur[static_cast<uint32_t>(shr64(k[j] - kmin, shiftF)) & fmask], 1u);
            sKey[p] = k[j];
            sIdx[p] = ix[j];
        }
    }
    __syncthreads();
    // sCur[f] = end of fine bucket f
    for (uint32_t f = tid; f < nf; f += kL2Threads) {
        const uint32_t fs = f ? sCur[f - 1] : 0u, fe = sCur[f], mf = fe - fs;
        if (mf <= 1) continue;
        if (mf > kBucketCap) {
            atomicAdd(&ctr->tie_overflow, 1ULL);
            continue;
        }
        if (mf > kSmall) {
            sBig[atomicAdd(&sNBig, 1u)] = f;
            continue;
        }
        for (uint32_t a = fs + 1; a < fe; ++a) {
            const unsigned long long vk = sKey[a];
            const uint32_t vi = sIdx[a];
            uint32_t c = a;
            while (c > fs && less_ki(vk, vi, sKey[c - 1], sIdx[c - 1])) {
                sKey[c] = sKey[c - 1];
                sIdx[c] = sIdx[c - 1];
                --c;
            }
            sKey[c] = vk;
            sIdx[c] = vi;
        }
    }
    __syncthreads();
    const int lane = tid & 31;
    for (uint32_t q = tid >> 5; q < sNBig; q += kL2Threads / 32) {
        const uint32_t f = sBig[q];
        const uint32_t fs = f ? sCur[f - 1] : 0u, mf = sCur[f] - fs;
        uint32_t idx[2];
        unsigned long long k[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t el = h * 32 + lane;
            idx[h] = el < mf ? sIdx[fs + el] : 0xFFFFFFFFu;
            k[h] = el < mf ? sKey[fs + el] : ~0ULL;
        }
#pragma unroll
        for (int kk = 2; kk <= 64; kk <<= 1) {
#pragma unroll
            for (int j = kk >> 1; j > 0; j >>= 1) {
                if (j == 32) {
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
                        const bool take =
                            want_min ? less_ki(pk, pi, k[h], idx[h]) : less_ki(k[h], idx[h], pk, pi);
                        if (take) {
                            k[h] = pk;
                            idx[h] = pi;
                        }
                    }
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t el = h * 32 + lane;
            if (el < mf) sIdx[fs + el] = idx[h];
        }
    }
    __syncthreads();
    for (uint32_t e = tid; e < m; e += kL2Threads) put_rank(s + e, sIdx[e], rects, order, brect, bmeta);
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

int depth_coarse_log2(uint64_t n) {
    int l = 0;
    while (l < 14 && (1ULL << l) * 1024 < n) ++l;
    return l;
}

static uint32_t l1_grid(uint64_t n) { return static_cast<uint32_t>((n + kL1Tile - 1) / kL1Tile); }

size_t depth_two_level_scratch(uint64_t n, int log2c) {
    (void)n;
    return static_cast<size_t>((1u << log2c) + 1) * 4;
}

void launch_depth_two_level(uint64_t n, const unsigned long long* key, Counters* ctr, int log2c, uint32_t* ghist,
                            uint32_t* cur, unsigned long long* part_key, uint32_t* order, const int4* rects,
                            int4* brect, uint2* bmeta, void* cub_temp, size_t cub_bytes,
                            cudaStream_t stream) {
    const uint32_t C = 1u << log2c;
    const uint32_t G = l1_grid(n);
    cudaMemsetAsync(ghist, 0, (C + 1) * 4, stream);
    coarse_hist_kernel<<<G, kL1Threads, (C + 1) * 4, stream>>>(n, key, ctr, log2c, ghist);
    cub::DeviceScan::ExclusiveSum(cub_temp, cub_bytes, ghist, cur, static_cast<int>(C + 1), stream);
    coarse_scatter_kernel<<<G, kL1Threads, (C + 1) * 8, stream>>>(n, key, ctr, log2c, cur, part_key, order, bmeta);
    constexpr int kL2Smem = kL2Cap * 12;
    static const bool attr = [] {
        cudaFuncSetAttribute(local_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kL2Smem);
        return true;
    }();
    (void)attr;
    local_sort_kernel<<<C, kL2Threads, kL2Smem, stream>>>(cur, part_key, order, ctr, log2c, rects, brect,
                                                          bmeta);
}

size_t depth_two_level_cub_bytes(uint64_t n, int log2c) {
    (void)n;
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<int>((1u << log2c) + 1));
    return temp;
}

}  // namespace sgs
