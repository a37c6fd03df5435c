// tile_sort.cu -- K5: stable LSD radix sort of the (tile << 32 | index) keys on
// the tile bits, with the item count read from device memory.
//
// K4 writes the keys of a depth chunk in rank order, so a *stable* sort on the tile
// bits alone yields every tile's run in rank order -- the reference's TileGrid list
// (raster.cpp:108-130). The count P of a chunk is only known on the device (it is
// the scan total of K3); this sort reads it from device memory, so the frame needs
// no host round trip between binning and compositing.
//
// One pass per <= 8 digit bits (13 tile bits at 1080p -> 7 + 6): upsweep (per-CTA
// digit histograms, smem atomics), one-CTA exclusive scan over (digit, CTA), and a
// downsweep that walks each CTA's slice in order, 256 keys per step, ranking equal
// digits by warp (match.any + popc) and across warps by a shared-memory prefix, so
// the scatter is stable.
#include <cub/device/device_scan.cuh>

#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kSortThreads = 512;
constexpr int kSortWarps = kSortThreads / 32;

__device__ __forceinline__ uint32_t slice_begin(uint64_t p, int g, int G) {
    const uint64_t per = (p + G - 1) / G;
    const uint64_t v = per * static_cast<uint64_t>(g);
    return static_cast<uint32_t>(v < p ? v : p);
}

__global__ void __launch_bounds__(kSortThreads) upsweep_kernel(const unsigned long long* __restrict__ keys,
                                                                const unsigned long long* __restrict__ count,
                                                                int shift, int radix, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    const int G = gridDim.x, g = blockIdx.x;
    const uint64_t p = *count;
    for (int d = threadIdx.x; d < radix; d += kSortThreads) h[d] = 0;
    __syncthreads();
    const uint32_t b = slice_begin(p, g, G), e = slice_begin(p, g + 1, G);
    for (uint32_t i = b + threadIdx.x; i < e; i += kSortThreads)
        atomicAdd(&h[static_cast<uint32_t>(keys[i] >> shift) & (radix - 1)], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < radix; d += kSortThreads) hist[d * G + g] = h[d];
}

// Each step ranks kStep = kSortThreads * kPerThread keys: warp w owns the
// consecutive keys [t0 + w * 32 kPerThread, +32 kPerThread) in kPerThread rounds of
// 32, so the stable order inside a step is (warp, round, lane). Within a warp,
// equal digits are ranked by match.any + popc on top of the warp's running count;
// across warps by a shared-memory prefix per digit.
constexpr int kPerThread = 4;
constexpr int kStep = kSortThreads * kPerThread;

__global__ void __launch_bounds__(kSortThreads) downsweep_kernel(
    const unsigned long long* __restrict__ in, unsigned long long* __restrict__ out,
    const unsigned long long* __restrict__ count, int shift, int radix, const uint32_t* __restrict__ hist) {
    __shared__ uint32_t base[256];
    __shared__ uint32_t wcnt[kSortWarps][257];
    __shared__ uint32_t total[256];
    const int G = gridDim.x, g = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t p = *count;
    for (int d = threadIdx.x; d < radix; d += kSortThreads) base[d] = hist[d * G + g];
    const uint32_t b = slice_begin(p, g, G), e = slice_begin(p, g + 1, G);
    for (uint32_t t0 = b; t0 < e; t0 += kStep) {
        for (int k = threadIdx.x; k < kSortWarps * 257; k += kSortThreads) (&wcnt[0][0])[k] = 0;
        __syncthreads();
        unsigned long long key[kPerThread];
        uint32_t dg[kPerThread], rk[kPerThread];
        const uint32_t w0 = t0 + warp * (32 * kPerThread) + lane;
#pragma unroll
        for (int j = 0; j < kPerThread; ++j) {
            const uint32_t i = w0 + j * 32;
            key[j] = i < e ? in[i] : 0ULL;
            dg[j] = i < e ? static_cast<uint32_t>(key[j] >> shift) & (radix - 1) : 256u;
        }
#pragma unroll
        for (int j = 0; j < kPerThread; ++j) {
            const unsigned peers = __match_any_sync(0xffffffffu, dg[j]);
            const uint32_t before = wcnt[warp][dg[j]];
            rk[j] = before + __popc(peers & ((1u << lane) - 1u));
            __syncwarp();
            if (__popc(peers & ((1u << lane) - 1u)) == 0) wcnt[warp][dg[j]] = before + __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        for (int dd = threadIdx.x; dd < radix; dd += kSortThreads) {
            uint32_t run = 0;
#pragma unroll
            for (int w = 0; w < kSortWarps; ++w) {
                const uint32_t c = wcnt[w][dd];
                wcnt[w][dd] = run;
                run += c;
            }
            total[dd] = run;
        }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < kPerThread; ++j)
            if (dg[j] < 256u) out[base[dg[j]] + wcnt[warp][dg[j]] + rk[j]] = key[j];
        __syncthreads();
        for (int dd = threadIdx.x; dd < radix; dd += kSortThreads) base[dd] += total[dd];
    }
}

}  // namespace

int tile_sort_grid() { return 2 * 148; }

size_t tile_sort_hist_bytes() {
    // histogram (256 x G) followed by the CUB scan's temporary storage
    size_t temp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  256 * tile_sort_grid());
    return static_cast<size_t>(256) * tile_sort_grid() * sizeof(uint32_t) * 2 + temp + 256;
}

// Sorts keys[0..*d_count) by bits [32, 32 + tile_bits). Returns the buffer holding
// the result (a or b).
unsigned long long* tile_sort(unsigned long long* a, unsigned long long* b, const unsigned long long* d_count,
                              int tile_bits, uint32_t* hist, cudaStream_t stream, uint64_t* launches) {
    const int G = tile_sort_grid();
    unsigned long long* in = a;
    unsigned long long* out = b;
    // digit widths split evenly (13 tile bits -> 7 + 6)
    const int passes = (tile_bits + 7) / 8;
    int shift = 32;
    for (int i = 0; i < passes; ++i) {
        const int db = tile_bits / passes + (i < tile_bits % passes ? 1 : 0);
        const int radix = 1 << db;
        uint32_t* scanned = hist + 256 * G;
        void* temp = scanned + 256 * G;
        size_t temp_bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, hist, scanned, radix * G, stream);
        upsweep_kernel<<<G, kSortThreads, 0, stream>>>(in, d_count, shift, radix, hist);
        cub::DeviceScan::ExclusiveSum(temp, temp_bytes, hist, scanned, radix * G, stream);
        downsweep_kernel<<<G, kSortThreads, 0, stream>>>(in, out, d_count, shift, radix, scanned);
        *launches += 2;
        unsigned long long* t = in;
        in = out;
        out = t;
        shift += db;
    }
    return in;
}

}  // namespace sgs
