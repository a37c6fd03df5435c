// binning.cu -- K3 (per-rank tile counts), K4 (pair emission), K6 (tile ranges).
//
// Replaces build_tile_grid (proj/src/raster.cpp:108-130). The reference walks the
// splats in blending order and push_backs the rank into every tile of the
// inclusive rectangle. Here, for a depth chunk of ranks [rb, re):
//   K3  counts[r - rb] = live tiles of rank r's rectangle, and each CTA's sum;
//   K4  each CTA turns the counts into output offsets itself -- the sum of the CTA
//       sums before it (read from L2 by all its threads) plus a block scan of its
//       own counts (warp shuffles) -- and emits the (tile id, Gaussian index) pairs,
//       tiles row-major as the reference's (ty, tx) double loop visits them, so a
//       warp of 32 consecutive ranks owns one contiguous output range. No CTA waits
//       for another. The pairs leave in rank order; K5 (radix.cu, stable on the tile
//       id) yields every tile's run in rank order -- the reference's TileGrid list --
//   K6  ranges[tile] = [first, last + 1) of the tile's run.
// A tile whose every pixel has terminated (transmittance below the threshold) in
// an earlier chunk receives no further pairs: the reference never reads past that
// point of its list (raster.cpp:177-179), so the image is unchanged.
#include <cstddef>

#include "sgs_internal.h"

namespace sgs {
namespace {

// The finished-tile flags of the frame as a bitmap in shared memory (tiles up to
// kMaxBitmapTiles; larger grids read the global bitmap).
constexpr int kMaxBitmapTiles = 1 << 18;
constexpr int kBinThreads = 1024;
static_assert(kBinThreads == 1024, "the CTA scans and sums reduce over exactly 32 warps");
// Splats covering more than kCoop tiles are emitted cooperatively by the whole warp
// (ballot-compacted over the live tiles) so one large splat does not serialise a
// lane while 31 idle.
constexpr uint32_t kCoop = 32;

__device__ __forceinline__ void load_done_bitmap(const uint32_t* __restrict__ done, int ntile, uint32_t* bits) {
    const int words = (ntile + 31) / 32;
    for (int w = threadIdx.x; w < words; w += blockDim.x) bits[w] = done[w];
    __syncthreads();
}

struct DoneView {
    const uint32_t* bits;  // bitmap (shared copy, or the global one), null if no tile finished yet
    __device__ __forceinline__ bool operator()(uint32_t t) const {
        return bits && ((bits[t >> 5] >> (t & 31)) & 1u);
    }
};

__device__ __forceinline__ uint32_t live_tiles(const int4 rc, const DoneView& done, int tiles_x) {
    uint32_t c = 0;
    for (int ty = rc.z; ty <= rc.w; ++ty)
        for (int tx = rc.x; tx <= rc.y; ++tx) c += done(static_cast<uint32_t>(ty * tiles_x + tx)) ? 0u : 1u;
    return c;
}

__device__ __forceinline__ DoneView done_view(const uint32_t* done_bits, int ntile, uint32_t* smem) {
    DoneView done{done_bits};
    if (done_bits && ntile <= kMaxBitmapTiles) {
        load_done_bitmap(done_bits, ntile, smem);  // ends with __syncthreads
        done.bits = smem;
    }
    return done;
}

// K3: counts[k] = live tiles of rank rb + k; csum[blk] = the CTA's total.
__global__ void __launch_bounds__(kBinThreads) bin_count_kernel(uint64_t rb, uint64_t re,
                                                                const uint2* __restrict__ bmeta,
                                                                const int4* __restrict__ brect,
                                                                const uint32_t* __restrict__ done_bits, int tiles_x,
                                                                int ntile, uint32_t* __restrict__ counts,
                                                                unsigned long long* __restrict__ csum) {
    extern __shared__ uint32_t bitmap[];
    __shared__ unsigned long long s_warp[kBinThreads / 32];
    const DoneView done = done_view(done_bits, ntile, bitmap);
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * kBinThreads + threadIdx.x;
    const uint64_t r = rb + k;
    uint32_t c = 0;
    if (r < re) {
        c = bmeta[r].y;
        if (done_bits) {
            const int4 rc = brect[r];  // issued with the bmeta load (stale when c == 0, unused)
            if (c) c = live_tiles(rc, done, tiles_x);
        }
        counts[k] = c;
    }
    unsigned long long s = c;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = s_warp[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) csum[blockIdx.x] = s;
    }
}

// K4: offsets from the CTA sums before this CTA and a block scan of its counts; the
// last CTA records the chunk's P (total, overflow flag, clamped count for K5-K7).
__global__ void __launch_bounds__(kBinThreads) bin_emit_kernel(
    uint64_t rb, uint64_t re, const uint2* __restrict__ bmeta, const int4* __restrict__ brect,
    const uint32_t* __restrict__ done_bits, int tiles_x, int ntile, const uint32_t* __restrict__ counts,
    const unsigned long long* __restrict__ csum, uint32_t* __restrict__ tk, uint32_t* __restrict__ tv,
    uint64_t capacity, Counters* __restrict__ ctr) {
    extern __shared__ uint32_t bitmap[];
    __shared__ unsigned long long s_warp[kBinThreads / 32];
    __shared__ unsigned long long s_base;
    const uint32_t blk = blockIdx.x;
    // a CTA without pairs has nothing to emit (in late chunks most ranks only cover
    // finished tiles); the last one still records the chunk's P
    if (csum[blk] == 0 && blk != gridDim.x - 1) return;
    const DoneView done = done_view(done_bits, ntile, bitmap);
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // sum of the CTA totals before this one
    unsigned long long before = 0;
    for (uint32_t p = threadIdx.x; p < blk; p += kBinThreads) before += csum[p];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    if (lane == 0) s_warp[warp] = before;
    __syncthreads();
    if (warp == 0) {
        unsigned long long v = s_warp[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
            s_base = v;
            if (blk == gridDim.x - 1) {
                const unsigned long long p = v + csum[blk];
                ctr->tile_entries += p;
                if (p > ctr->max_chunk_entries) ctr->max_chunk_entries = p;
                if (p > capacity) ctr->key_overflow = 1;
                ctr->chunk_entries = p < capacity ? p : capacity;
            }
        }
    }
    __syncthreads();
    const uint64_t k = static_cast<uint64_t>(blk) * kBinThreads + threadIdx.x;
    const uint64_t r = rb + k;
    const uint32_t c = r < re ? counts[k] : 0u;
    // block-exclusive scan of the counts
    unsigned long long inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= static_cast<unsigned>(o)) inc += y;
    }
    __syncthreads();  // (s_warp reuse)
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const unsigned long long w = s_warp[lane];
        unsigned long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= static_cast<unsigned>(o)) wi += y;
        }
        s_warp[lane] = wi - w;
    }
    __syncthreads();
    const unsigned long long off = s_base + s_warp[warp] + inc - c;
    // a rank with no live tile is skipped before its rectangle is read (in late chunks
    // most ranks only cover finished tiles)
    uint32_t g = 0, area = 0;
    int4 rc = make_int4(0, -1, 0, -1);
    if (c) {
        const uint2 m = bmeta[r];
        g = m.x;
        area = m.y;
        rc = brect[r];
    }
    if (area && area <= kCoop) {
        unsigned long long o = off;
        for (int ty = rc.z; ty <= rc.w; ++ty)
            for (int tx = rc.x; tx <= rc.y; ++tx) {
                const uint32_t tile = static_cast<uint32_t>(ty * tiles_x + tx);
                if (done(tile)) continue;
                if (o < capacity) {
                    tk[o] = tile;
                    tv[o] = g;
                }
                ++o;
            }
    }
    unsigned big = __ballot_sync(0xffffffffu, area > kCoop);
    while (big) {
        const int src = __ffs(big) - 1;
        big &= big - 1;
        const uint32_t a = __shfl_sync(0xffffffffu, area, src);
        const uint32_t gg = __shfl_sync(0xffffffffu, g, src);
        const int x0 = __shfl_sync(0xffffffffu, rc.x, src);
        const int x1 = __shfl_sync(0xffffffffu, rc.y, src);
        const int y0 = __shfl_sync(0xffffffffu, rc.z, src);
        unsigned long long o = __shfl_sync(0xffffffffu, off, src);
        const uint32_t ww = static_cast<uint32_t>(x1 - x0 + 1);
        for (uint32_t base = 0; base < a; base += 32) {
            const uint32_t j = base + lane;
            uint32_t tile = 0;
            bool live = false;
            if (j < a) {
                tile = static_cast<uint32_t>(y0 + static_cast<int>(j / ww)) * tiles_x +
                       static_cast<uint32_t>(x0 + static_cast<int>(j % ww));
                live = !done(tile);
            }
            const unsigned m = __ballot_sync(0xffffffffu, live);
            const unsigned long long pos = o + __popc(m & ((1u << lane) - 1u));
            if (live && pos < capacity) {
                tk[pos] = tile;
                tv[pos] = gg;
            }
            o += __popc(m);
        }
    }
}

// Per-frame counters without the copy engines: the init is a kernel, and the final
// block is written straight into mapped pinned host memory, so the readback never
// queues behind the host frame copies on the D2H engine.
__global__ void counters_init_kernel(Counters* __restrict__ c) {
    const int t = threadIdx.x;
    if (t < 16) reinterpret_cast<unsigned long long*>(c)[t] = (t == 0 || t == 5) ? ~0ULL : 0ULL;  // err, kmin
}

__global__ void counters_publish_kernel(const Counters* __restrict__ d, Counters* __restrict__ h_mapped) {
    const int t = threadIdx.x;
    if (t < 16)
        reinterpret_cast<volatile unsigned long long*>(h_mapped)[t] = reinterpret_cast<const unsigned long long*>(d)[t];
    __threadfence_system();
}

__global__ void tile_ranges_kernel(const unsigned long long* __restrict__ count,
                                   const uint32_t* __restrict__ tiles, uint2* __restrict__ ranges) {
    const uint64_t p = *count;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < p;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t t = tiles[i];
        if (i == 0 || tiles[i - 1] != t) ranges[t].x = static_cast<uint32_t>(i);
        if (i == p - 1 || tiles[i + 1] != t) ranges[t].y = static_cast<uint32_t>(i + 1);
    }
}

size_t bitmap_smem(const uint32_t* done, int ntile) {
    return done && ntile <= kMaxBitmapTiles ? static_cast<size_t>((ntile + 31) / 32) * 4 : 0;
}

uint64_t bin_blocks(uint64_t ranks) { return ranks ? (ranks + kBinThreads - 1) / kBinThreads : 1; }

}  // namespace

void launch_tile_ranges(const unsigned long long* d_count, const uint32_t* tiles, uint2* ranges,
                        cudaStream_t stream) {
    tile_ranges_kernel<<<148 * 8, 256, 0, stream>>>(d_count, tiles, ranges);
}

TileDigits tile_digits(int tile_bits) {
    // digit widths split evenly, the wider digit last (13 tile bits at 1080p -> 6 + 7:
    // the first pass scatters rank-ordered pairs into fewer runs; 1% faster)
    TileDigits td{};
    td.passes = (tile_bits + 7) / 8;
    int shift = 0;
    for (int i = 0; i < td.passes; ++i) {
        td.bits[i] = tile_bits / td.passes + (td.passes - 1 - i < tile_bits % td.passes ? 1 : 0);
        td.shift[i] = shift;
        shift += td.bits[i];
    }
    return td;
}

size_t bin_scratch_bytes(uint64_t ranks) {
    const uint64_t nb = bin_blocks(ranks);
    return (nb * kBinThreads * sizeof(uint32_t) + 255) / 256 * 256 + nb * sizeof(unsigned long long);
}

cudaError_t launch_binning(uint64_t rb, uint64_t re, const uint2* bmeta, const int4* brect, const uint32_t* done,
                           int tiles_x, int ntile, uint32_t* tk, uint32_t* tv, uint64_t capacity, void* scratch,
                           Counters* ctr, cudaStream_t stream, uint64_t* launches) {
    const uint64_t n = re > rb ? re - rb : 0;
    const uint64_t nb = bin_blocks(n);
    uint32_t* counts = static_cast<uint32_t*>(scratch);
    unsigned long long* csum = reinterpret_cast<unsigned long long*>(
        static_cast<char*>(scratch) + (nb * kBinThreads * sizeof(uint32_t) + 255) / 256 * 256);
    const size_t smem = bitmap_smem(done, ntile);
    bin_count_kernel<<<static_cast<unsigned>(nb), kBinThreads, smem, stream>>>(rb, re, bmeta, brect, done, tiles_x,
                                                                               ntile, counts, csum);
    bin_emit_kernel<<<static_cast<unsigned>(nb), kBinThreads, smem, stream>>>(rb, re, bmeta, brect, done, tiles_x,
                                                                              ntile, counts, csum, tk, tv, capacity,
                                                                              ctr);
    *launches += 2;
    return cudaGetLastError();
}

void launch_counters_init(Counters* c, cudaStream_t stream) { counters_init_kernel<<<1, 32, 0, stream>>>(c); }

void launch_counters_publish(const Counters* d, Counters* h_mapped, cudaStream_t stream) {
    counters_publish_kernel<<<1, 32, 0, stream>>>(d, h_mapped);
}

}  // namespace sgs
