// binning.cu -- K3+K4 (tile binning in one pass) and K6 (tile ranges).
//
// Replaces build_tile_grid (proj/src/raster.cpp:108-130). The reference walks the
// splats in blending order and push_backs the rank into every tile of the
// inclusive rectangle. Here, for a depth chunk of ranks [rb, re), ONE kernel
// (bin_emit_kernel) counts each rank's live tiles, turns the counts into output
// offsets with a warp-level decoupled look-back scan across the grid (so a warp of 32
// consecutive ranks owns one contiguous output range), and emits the (tile id,
// Gaussian index) pairs, tiles row-major as the reference's (ty, tx) double loop
// visits them. The pairs leave in rank order; K5 (radix.cu, stable on the tile id)
// then yields every tile's run in rank order -- the reference's TileGrid list -- and
// K6 finds each tile's [first, last + 1).
// A tile whose every pixel has terminated (transmittance below the threshold) in
// an earlier chunk receives no further pairs: the reference never reads past that
// point of its list (raster.cpp:177-179), so the image is unchanged.
#include <cstddef>

#include "sgs_internal.h"

namespace sgs {
namespace {

// The finished-tile flags of the frame as a bitmap in shared memory (tiles up to
// kMaxBitmapTiles; larger grids read the byte flags from global memory).
constexpr int kMaxBitmapTiles = 1 << 18;

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

// K3+K4: one pass per chunk counts each rank's live tiles, scans the counts across
// the grid with a decoupled look-back (CTAs take logical block numbers from a
// ticket, so every predecessor a CTA waits on is already resident), and emits the
// pairs at the scanned offsets, adding each tile id's K5 digits to block histograms.
// The last block records the chunk's P (total, overflow flag) and opens the sort's
// epoch.
// status[b] = flag << 62 | value: flag 1 = block aggregate, 2 = inclusive prefix.
constexpr unsigned long long kFlagAgg = 1ULL << 62;
constexpr unsigned long long kFlagPre = 2ULL << 62;
constexpr unsigned long long kValMask = (1ULL << 62) - 1;
constexpr int kBinThreads = 1024;
// Splats covering more than kCoop tiles are emitted cooperatively by the whole warp
// (ballot-compacted over the live tiles) so one large splat does not serialise a
// lane while 31 idle.
constexpr uint32_t kCoop = 32;

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(kBinThreads) bin_emit_kernel(
    uint64_t rb, uint64_t re, const uint2* __restrict__ bmeta, const int4* __restrict__ brect,
    const uint32_t* __restrict__ done_bytes, int tiles_x, int ntile, uint32_t* __restrict__ tk,
    uint32_t* __restrict__ tv, uint64_t capacity, unsigned long long* __restrict__ status, const TileDigits td,
    SortCtl* __restrict__ ctl, Counters* __restrict__ ctr) {
    extern __shared__ uint32_t done_bits[];
    __shared__ uint32_t s_blk;
    __shared__ uint32_t s_hist[4 * 256];
    for (int k = threadIdx.x; k < td.passes * 256; k += kBinThreads) s_hist[k] = 0;
    __shared__ unsigned long long s_warp[kBinThreads / 32];
    __shared__ unsigned long long s_base;
    const unsigned nblk = gridDim.x;
    if (threadIdx.x == 0) s_blk = atomicAdd(reinterpret_cast<unsigned int*>(&status[nblk]), 1u);
    DoneView done{done_bytes};
    if (done_bytes && ntile <= kMaxBitmapTiles) {
        load_done_bitmap(done_bytes, ntile, done_bits);  // ends with __syncthreads
        done.bits = done_bits;
    } else {
        __syncthreads();
    }
    const uint32_t blk = s_blk;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t r = rb + static_cast<uint64_t>(blk) * kBinThreads + threadIdx.x;
    uint32_t g = 0, area = 0;
    int4 rc = make_int4(0, -1, 0, -1);
    unsigned long long c = 0;
    if (r < re) {
        const uint2 m = bmeta[r];
        g = m.x;
        area = m.y;
        if (area) {
            rc = brect[r];
            c = done_bytes ? live_tiles(rc, done, tiles_x) : area;
        }
    }
    // block-exclusive scan of the counts
    unsigned long long inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= static_cast<unsigned>(o)) inc += y;
    }
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
        s_warp[lane] = wi - w;  // exclusive warp offsets
        // wi (lane 31) = block total: publish it, look back over the predecessors a
        // warp-wide window of 32 at a time, publish the inclusive prefix
        const unsigned long long total = __shfl_sync(0xffffffffu, wi, 31);
        if (blk == 0) {
            if (lane == 0) st_release(&status[0], kFlagPre | total);
        } else if (lane == 0) {
            st_release(&status[blk], kFlagAgg | total);
        }
        unsigned long long excl = 0;
        if (blk > 0) {
            int64_t hi = static_cast<int64_t>(blk) - 1;  // window [hi - 31, hi], lane i reads hi - i
            for (;;) {
                const int64_t pb = hi - static_cast<int64_t>(lane);
                unsigned long long v = pb >= 0 ? 0ULL : kFlagPre;  // before block 0: prefix 0
                // every lane of the warp runs this loop until all 32 flags are set
                for (;;) {
                    if (v == 0) v = ld_acquire(&status[pb]);
                    if (__all_sync(0xffffffffu, v != 0)) break;
                }
                const unsigned pre = __ballot_sync(0xffffffffu, (v & kFlagPre) != 0);
                const int stop_lane = pre ? __ffs(pre) - 1 : 31;
                unsigned long long part = static_cast<int>(lane) <= stop_lane ? (v & kValMask) : 0ULL;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                excl += part;
                if (pre) break;
                hi -= 32;
            }
            if (lane == 0) st_release(&status[blk], kFlagPre | (excl + total));
        }
        if (lane == 0) {
            s_base = excl;
            if (blk == nblk - 1) {
                // the chunk's P: total, overflow flag, clamped count for K5-K7
                const unsigned long long p = excl + total;
                ctr->tile_entries += p;
                if (p > ctr->max_chunk_entries) ctr->max_chunk_entries = p;
                if (p > capacity) ctr->key_overflow = 1;
                ctr->chunk_entries = p < capacity ? p : capacity;
                ctl->epoch += 1;  // (the K5 passes of this chunk run after this kernel)
            }
        }
    }
    __syncthreads();
    // emit one (tile, index) pair at slot pos (dropped past the capacity: the frame is redone)
    auto put = [&](unsigned long long pos, uint32_t tile, uint32_t gi) {
        if (pos < capacity) {
            tk[pos] = tile;
            tv[pos] = gi;
            for (int p = 0; p < td.passes; ++p)
                atomicAdd(&s_hist[p * 256 + ((tile >> td.shift[p]) & ((1u << td.bits[p]) - 1u))], 1u);
        }
    };
    const unsigned long long off = s_base + s_warp[warp] + inc - c;
    const uint32_t w = static_cast<uint32_t>(rc.y - rc.x + 1);
    if (area && area <= kCoop) {
        uint32_t o = 0;
        for (uint32_t j = 0; j < area; ++j) {
            const uint32_t tile = static_cast<uint32_t>(rc.z + static_cast<int>(j / w)) * tiles_x +
                                  static_cast<uint32_t>(rc.x + static_cast<int>(j % w));
            if (done(tile)) continue;
            put(off + o, tile, g);
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
            if (live) put(pos, tile, gg);
            o += __popc(m);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < td.passes * 256; k += kBinThreads)
        if (s_hist[k]) atomicAdd(&ctl->hist[k >> 8][k & 255], s_hist[k]);
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

}  // namespace

static size_t bitmap_smem(const uint32_t* done, int ntile) {
    return done && ntile <= kMaxBitmapTiles ? static_cast<size_t>((ntile + 31) / 32) * 4 : 0;
}

void launch_tile_ranges(const unsigned long long* d_count, const uint32_t* tiles, uint2* ranges,
                        cudaStream_t stream) {
    tile_ranges_kernel<<<148 * 8, 256, 0, stream>>>(d_count, tiles, ranges);
}

TileDigits tile_digits(int tile_bits) {
    // digit widths split evenly (13 tile bits at 1080p -> 7 + 6)
    TileDigits td{};
    td.passes = (tile_bits + 7) / 8;
    int shift = 0;
    for (int i = 0; i < td.passes; ++i) {
        td.bits[i] = tile_bits / td.passes + (i < tile_bits % td.passes ? 1 : 0);
        td.shift[i] = shift;
        shift += td.bits[i];
    }
    return td;
}

size_t bin_emit_status_bytes(uint64_t ranks) {
    return ((ranks + kBinThreads - 1) / kBinThreads + 1) * sizeof(unsigned long long);
}

cudaError_t launch_bin_emit(uint64_t rb, uint64_t re, const uint2* bmeta, const int4* brect, const uint32_t* done,
                            int tiles_x, int ntile, uint32_t* tk, uint32_t* tv, uint64_t capacity,
                            unsigned long long* status, const TileDigits& td, SortCtl* ctl, Counters* ctr,
                            cudaStream_t stream) {
    const uint64_t n = re > rb ? re - rb : 0;
    const unsigned grid = static_cast<unsigned>(n ? (n + kBinThreads - 1) / kBinThreads : 1);
    cudaError_t e = cudaMemsetAsync(status, 0, (grid + 1) * sizeof(unsigned long long), stream);
    if (e == cudaSuccess)  // the K5 tickets and histograms this chunk's pairs fill
        e = cudaMemsetAsync(&ctl->ticket[0], 0, sizeof(SortCtl) - offsetof(SortCtl, ticket), stream);
    if (e != cudaSuccess) return e;
    bin_emit_kernel<<<grid, kBinThreads, bitmap_smem(done, ntile), stream>>>(rb, re, bmeta, brect, done, tiles_x,
                                                                             ntile, tk, tv, capacity, status, td,
                                                                             ctl, ctr);
    return cudaGetLastError();
}

void launch_counters_init(Counters* c, cudaStream_t stream) { counters_init_kernel<<<1, 32, 0, stream>>>(c); }

void launch_counters_publish(const Counters* d, Counters* h_mapped, cudaStream_t stream) {
    counters_publish_kernel<<<1, 32, 0, stream>>>(d, h_mapped);
}

}  // namespace sgs
