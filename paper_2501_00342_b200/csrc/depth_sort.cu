// depth_sort.cu -- K2: the global blending order (depth, index) of raster.cpp:93-101.
//
// Exact two-level bucket sort of the orderable 64-bit depth keys, whose visible range
// [kmin, kmax] K1 found. Buckets are uniform in the key offset from kmin (monotone in
// the key, so bucket order is key order). Culled splats (key ~0) go after the visible
// ones, in index order; they own no tiles. Measured against a 4-pass LSD radix sort
// of 32-bit keys (radix.cu) with an exact fix-up of equal-key runs: 171 against
// 230 us per frame at config C -- one scattered partition plus shared-memory sorts
// move less than four global passes. Dense depth clusters stay on this path: a fine
// bucket past the warp sort's 64 keys sends its coarse bucket to a shared-memory
// bitonic sort, and its CTA sorts a coarse bucket past 4096 keys in global memory
// (runs sorted in shared memory, then merged), so no depth distribution forces a
// slower sort on the whole frame.

#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kBucketCap = 64;
constexpr int kSmall = 12;

__device__ __forceinline__ int bucket_shift(const Counters* ctr, int log2b) {
    const unsigned long long kmin = ctr->kmin, kmax = ctr->kmax;
    const unsigned long long range = kmax >= kmin ? kmax - kmin : 0ULL;
    const int bits = range ? 64 - __clzll(static_cast<long long>(range)) : 0;
    return bits > log2b ? bits - log2b : 0;
}

__device__ __forceinline__ bool less_ki(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
    return ka < kb || (ka == kb && ia < ib);
}

constexpr int kL1Threads = 1024;
constexpr int kL1Per = 8;
constexpr int kL1Tile = kL1Threads * kL1Per;
constexpr int kL2Threads = 512;
constexpr int kL2Cap = 4096;
constexpr int kL2Per = kL2Cap / kL2Threads;
constexpr int kL2MaxFineLog2 = 11;

// A visible splat in K2's partition: its key and index side by side (one 16-B store
// per scattered element instead of two partial-sector ones).
__device__ __forceinline__ void put_part(uint4* part, uint32_t pos, unsigned long long k, uint32_t i) {
    part[pos] = make_uint4(static_cast<uint32_t>(k), static_cast<uint32_t>(k >> 32), i, 0u);
}
__device__ __forceinline__ unsigned long long part_key(const uint4 v) {
    return static_cast<unsigned long long>(v.x) | (static_cast<unsigned long long>(v.y) << 32);
}

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
// keys go to the partition as (key, index) pairs; culled ones straight to their final ranks
// [V, N) with (index, 0 tiles) metadata.
__global__ void __launch_bounds__(kL1Threads) coarse_scatter_kernel(
    uint64_t n, const unsigned long long* __restrict__ key, const Counters* __restrict__ ctr, int log2c,
    uint32_t* __restrict__ cur, uint4* __restrict__ part, uint32_t* __restrict__ order,
    uint2* __restrict__ bmeta) {
    extern __shared__ uint32_t cnt[];  // per-bucket counts, then this CTA's first slot per bucket
    const uint32_t C = 1u << log2c;
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
        if (cnt[b]) cnt[b] = atomicAdd(&cur[b], cnt[b]);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kL1Per; ++j) {
        const uint64_t i = base + j * kL1Threads;
        if (i >= n) continue;
        const uint32_t pos = cnt[bk[j]] + lo[j];
        if (bk[j] == C) {
            order[pos] = static_cast<uint32_t>(i);
            bmeta[pos] = make_uint2(static_cast<uint32_t>(i), 0u);
        } else {
            put_part(part, pos, k[j], static_cast<uint32_t>(i));
        }
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

// Sort (key, index) pairs [0, m) of shared memory in place by (key, index), m <= kL2Cap:
// a CTA-wide bitonic network over the next power of two (padding with (~0, ~0), which
// sorts last). Every thread of the CTA calls it.
__device__ void cta_bitonic_sort(unsigned long long* key, uint32_t* idx, uint32_t m) {
    uint32_t P = 1;
    while (P < m) P <<= 1;
    for (uint32_t e = m + threadIdx.x; e < P; e += blockDim.x) {
        key[e] = ~0ULL;
        idx[e] = 0xFFFFFFFFu;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= P; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < P / 2; i += blockDim.x) {
                const uint32_t a = (i / stride) * 2 * stride + (i % stride), b = a + stride;
                const bool up = (a & size) == 0;
                if (less_ki(key[b], idx[b], key[a], idx[a]) == up) {
                    const unsigned long long tk = key[a];
                    const uint32_t ti = idx[a];
                    key[a] = key[b];
                    idx[a] = idx[b];
                    key[b] = tk;
                    idx[b] = ti;
                }
            }
            __syncthreads();
        }
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

// A coarse bucket with more than kL2Cap keys (dense depth clusters, very large
// scenes), sorted by its CTA by (key, index) in global memory: 4096-pair runs sorted in
// shared memory, then merged pairwise, each pair placed by binary search (keys are
// unique with the index); then its ranks. The runs ping-pong through tmp_key / tmp_idx
// (K1's depth keys and the tile-pair arena, both free while K2 runs).
__device__ __forceinline__ uint32_t count_less(const unsigned long long* key, const uint32_t* idx, uint32_t lo,
                                               uint32_t hi, unsigned long long k, uint32_t i) {
    uint32_t a = lo, b = hi;
    while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (less_ki(key[mid], idx[mid], k, i))
            a = mid + 1;
        else
            b = mid;
    }
    return a - lo;
}

__device__ __noinline__ void sort_big_bucket(uint32_t s, uint32_t m, uint4* part, uint32_t* order,
                                             unsigned long long* tmp_key, uint32_t* tmp_idx,
                                             unsigned long long* sKey, uint32_t* sIdx, const int4* rects,
                                             int4* brect, uint2* bmeta) {
    // the runs ping-pong between tmp and the bucket's own 16m-byte stretch of the
    // partition (8m bytes of keys, then 4m of indices) once it has been read
    unsigned long long* srcK = reinterpret_cast<unsigned long long*>(part + s);
    uint32_t* srcI = reinterpret_cast<uint32_t*>(srcK + m);
    unsigned long long* dstK = tmp_key + s;
    uint32_t* dstI = tmp_idx + s;
    for (uint32_t r0 = 0; r0 < m; r0 += kL2Cap) {
        const uint32_t rm = min(static_cast<uint32_t>(kL2Cap), m - r0);
        for (uint32_t e = threadIdx.x; e < rm; e += kL2Threads) {
            const uint4 v = part[s + r0 + e];
            sKey[e] = part_key(v);
            sIdx[e] = v.z;
        }
        __syncthreads();
        cta_bitonic_sort(sKey, sIdx, rm);
        for (uint32_t e = threadIdx.x; e < rm; e += kL2Threads) {
            dstK[r0 + e] = sKey[e];
            dstI[r0 + e] = sIdx[e];
        }
        __syncthreads();
    }
    // pairwise merges: an element's place is its index in its run plus the number of
    // smaller elements in the other run
    for (uint32_t w = kL2Cap; w < m; w <<= 1) {
        unsigned long long* tk = srcK;
        uint32_t* ti = srcI;
        srcK = dstK, srcI = dstI, dstK = tk, dstI = ti;
        for (uint32_t e = threadIdx.x; e < m; e += kL2Threads) {
            const uint32_t base = e / (2 * w) * (2 * w);
            const uint32_t mid = min(base + w, m), end = min(base + 2 * w, m);
            const unsigned long long k = srcK[e];
            const uint32_t i = srcI[e];
            const uint32_t pos = e < mid ? e + count_less(srcK, srcI, mid, end, k, i)
                                         : e - w + count_less(srcK, srcI, base, mid, k, i);
            dstK[pos] = k;
            dstI[pos] = i;
        }
        __syncthreads();
    }
    for (uint32_t e = threadIdx.x; e < m; e += kL2Threads) put_rank(s + e, dstI[e], rects, order, brect, bmeta);
}

__global__ void __launch_bounds__(kL2Threads) local_sort_kernel(
    const uint32_t* __restrict__ cend, uint4* __restrict__ part, uint32_t* __restrict__ order,
    Counters* __restrict__ ctr, int log2c, const int4* __restrict__ rects,
    int4* __restrict__ brect, uint2* __restrict__ bmeta, unsigned long long* __restrict__ tmp_key,
    uint32_t* __restrict__ tmp_idx) {
    extern __shared__ unsigned long long sKey[];  // kL2Cap keys, then kL2Cap indices
    uint32_t* sIdx = reinterpret_cast<uint32_t*>(sKey + kL2Cap);
    __shared__ uint32_t sCur[1 << kL2MaxFineLog2];
    __shared__ uint32_t sBig[kL2Cap / (kSmall + 1) + 1];
    __shared__ uint32_t sWarp[kL2Threads / 32];
    __shared__ uint32_t sNBig;
    __shared__ uint32_t sFull;  // a fine bucket too large for the warp sort: sort the whole bucket
    const uint32_t b = blockIdx.x;
    const uint32_t s = b ? cend[b - 1] : 0u;
    const uint32_t m = cend[b] - s;
    if (m == 0) return;
    const int tid = threadIdx.x;
    if (m > kL2Cap) {  // more keys than shared memory holds
        sort_big_bucket(s, m, part, order, tmp_key, tmp_idx, sKey, sIdx, rects, brect, bmeta);
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
    if (tid == 0) sNBig = 0, sFull = 0;
    unsigned long long k[kL2Per];
    uint32_t ix[kL2Per];
#pragma unroll
    for (int j = 0; j < kL2Per; ++j) {
        const uint32_t e = tid + j * kL2Threads;
        const uint4 v = e < m ? part[s + e] : make_uint4(0u, 0u, 0u, 0u);
        k[j] = part_key(v);
        ix[j] = v.z;
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
            sFull = 1;
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
    if (sFull) {  // (dense depths: a fine bucket past the warp sort) the whole bucket at once
        cta_bitonic_sort(sKey, sIdx, m);
        for (uint32_t e = tid; e < m; e += kL2Threads) put_rank(s + e, sIdx[e], rects, order, brect, bmeta);
        return;
    }
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


// Exclusive scan of in[0, m) into out (one CTA; m = C + 1 <= 32769).
constexpr int kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) bucket_scan_kernel(const uint32_t* __restrict__ in,
                                                                  uint32_t* __restrict__ out, uint32_t m) {
    __shared__ uint32_t warp_tot[kScanThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t per = (m + kScanThreads - 1) / kScanThreads;
    const uint32_t b = tid * per, e = min(b + per, m);
    uint32_t sum = 0;
    for (uint32_t i = b; i < e; ++i) sum += in[i];
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = warp_tot[lane];
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        warp_tot[lane] = wi - w;
    }
    __syncthreads();
    uint32_t run = warp_tot[warp] + inc - sum;
    for (uint32_t i = b; i < e; ++i) {
        const uint32_t v = in[i];
        out[i] = run;
        run += v;
    }
}
}  // namespace

int depth_coarse_log2(uint64_t n) {
    int l = 0;
    while (l < 15 && (1ULL << l) * 1024 < n) ++l;
    return l;
}

size_t depth_two_level_scratch(int log2c) { return static_cast<size_t>((1u << log2c) + 1) * 4; }  // (per region)

cudaError_t launch_depth_two_level(uint64_t n, unsigned long long* key, Counters* ctr, int log2c,
                                   uint32_t* ghist, uint32_t* cur, void* part_buf, uint32_t* order,
                                   uint32_t* tmp_idx, const int4* rects, int4* brect, uint2* bmeta,
                                   cudaStream_t stream, uint64_t* launches) {
    if (n == 0) return cudaSuccess;
    const uint32_t C = 1u << log2c;
    const uint32_t G = static_cast<uint32_t>((n + kL1Tile - 1) / kL1Tile);
    // shared memory of the level-1 kernels: C + 1 counters, past the default 48 KB above
    // 8M Gaussians (C = 32768 at most: 128 KB)
    static const cudaError_t l1attr = [] {
        constexpr int kMaxL1Smem = ((1 << 15) + 1) * 4;
        cudaError_t a = cudaFuncSetAttribute(coarse_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kMaxL1Smem);
        if (a == cudaSuccess)
            a = cudaFuncSetAttribute(coarse_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxL1Smem);
        return a;
    }();
    if (l1attr != cudaSuccess) return l1attr;
    cudaError_t e = cudaMemsetAsync(ghist, 0, (C + 1) * 4, stream);
    if (e != cudaSuccess) return e;
    coarse_hist_kernel<<<G, kL1Threads, (C + 1) * 4, stream>>>(n, key, ctr, log2c, ghist);
    bucket_scan_kernel<<<1, kScanThreads, 0, stream>>>(ghist, cur, C + 1);
    uint4* part = static_cast<uint4*>(part_buf);
    coarse_scatter_kernel<<<G, kL1Threads, (C + 1) * 4, stream>>>(n, key, ctr, log2c, cur, part, order, bmeta);
    constexpr int kL2Smem = kL2Cap * 12;
    static const cudaError_t attr =
        cudaFuncSetAttribute(local_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kL2Smem);
    if (attr != cudaSuccess) return attr;
    // (the keys are dead once partitioned: K1's key array is the big buckets' scratch)
    local_sort_kernel<<<C, kL2Threads, kL2Smem, stream>>>(cur, part, order, ctr, log2c, rects, brect, bmeta,
                                                           key, tmp_idx);
    *launches += 4;
    return cudaGetLastError();
}

}  // namespace sgs
