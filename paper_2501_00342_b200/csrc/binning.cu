// binning.cu -- K3 (per-rank tile counts), K4 (tile-key emission), K6 (tile ranges).
//
// Replaces build_tile_grid (proj/src/raster.cpp:108-130). The reference walks the
// splats in blending order and push_backs the rank into every tile of the
// inclusive rectangle. Here, for a depth chunk of ranks [rb, re):
//   K3  counts[r-rb] = tiles of rect(order[r]) not yet terminated; a device-wide
//       exclusive scan gives each rank its first output slot (so a warp of 32
//       consecutive ranks owns one contiguous output range)
//   K4  keys[off + j] = (tile << 32) | gaussian_index, tiles row-major as the
//       reference's (ty, tx) double loop visits them; keys leave K4 in rank order
//   K5  stable radix sort on the tile bits only (capi.cu) keeps rank order inside a
//       tile, so each tile's run equals the reference's TileGrid list exactly
//   K6  ranges[tile] = [first, last + 1) of the tile's run.
// A tile whose every pixel has terminated (transmittance below the threshold) in
// an earlier chunk receives no further keys: the reference never reads past that
// point of its list (raster.cpp:177-179), so the image is unchanged.
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

// Rank-ordered copy of the binning inputs, gathered once per frame so that every
// chunk's K3/K4 reads them coalesced: brect[r] = rects[order[r]],
// bmeta[r] = (order[r], tiles of its rectangle).
__global__ void gather_bins_kernel(uint64_t n, const uint32_t* __restrict__ order,
                                   const int4* __restrict__ rects, const Counters* __restrict__ ctr,
                                   int4* __restrict__ brect, uint2* __restrict__ bmeta) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t g = order[r];
    // visible splats (ranks below V) carry their rectangle from K1; culled ones none
    const int4 rc = r < ctr->visible ? rects[g] : make_int4(0, -1, 0, -1);
    const uint32_t c = rect_area(rc);
    bmeta[r] = make_uint2(g, c);
    if (c) brect[r] = rc;
}

__global__ void count_tiles_kernel(uint64_t rb, uint64_t re, const uint2* __restrict__ bmeta,
                                   const int4* __restrict__ brect, const uint32_t* __restrict__ done_bytes,
                                   int tiles_x, int ntile, unsigned long long* __restrict__ counts) {
    extern __shared__ uint32_t done_bits[];
    DoneView done{done_bytes};
    if (done_bytes && ntile <= kMaxBitmapTiles) {
        load_done_bitmap(done_bytes, ntile, done_bits);
        done.bits = done_bits;
    }
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t r = rb + k;
    if (r < re) {
        uint32_t c = bmeta[r].y;
        if (done_bytes) {
            const int4 rc = brect[r];  // issued with the bmeta load (stale when c == 0, unused)
            if (c) c = live_tiles(rc, done, tiles_x);
        }
        counts[k] = c;
    } else if (r == re) {
        counts[k] = 0;
    }
}

// One thread per rank writes its splat's keys into its own slot range. Splats
// covering more than kCoop tiles are emitted cooperatively by the whole warp
// (ballot-compacted over the live tiles) so one large splat does not serialise a
// lane while 31 idle.
constexpr uint32_t kCoop = 32;

__global__ void emit_keys_kernel(uint64_t rb, uint64_t re, const uint2* __restrict__ bmeta,
                                 const int4* __restrict__ brect, const uint32_t* __restrict__ done_bytes,
                                 const unsigned long long* __restrict__ offsets, int tiles_x, int ntile,
                                 unsigned long long* __restrict__ keys, uint64_t capacity) {
    extern __shared__ uint32_t done_bits[];
    DoneView done{done_bytes};
    if (done_bytes && ntile <= kMaxBitmapTiles) {
        load_done_bitmap(done_bytes, ntile, done_bits);
        done.bits = done_bits;
    }
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t r = rb + k;
    const unsigned lane = threadIdx.x & 31;
    uint32_t g = 0, area = 0;
    int4 rc = make_int4(0, -1, 0, -1);
    unsigned long long off = 0;
    if (r < re) {
        // the scanned counts tell which ranks emit anything: in late chunks most
        // ranks only cover finished tiles and are skipped before their rect is read
        off = offsets[k];
        if (offsets[k + 1] != off) {
            const uint2 m = bmeta[r];
            g = m.x;
            area = m.y;
            rc = brect[r];
        }
    }
    const uint32_t w = static_cast<uint32_t>(rc.y - rc.x + 1);
    if (area && area <= kCoop) {
        uint32_t o = 0;
        for (uint32_t j = 0; j < area; ++j) {
            const uint32_t tile = static_cast<uint32_t>(rc.z + static_cast<int>(j / w)) * tiles_x +
                                  static_cast<uint32_t>(rc.x + static_cast<int>(j % w));
            if (done(tile)) continue;
            if (off + o < capacity) keys[off + o] = (static_cast<unsigned long long>(tile) << 32) | g;
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
            if (live && pos < capacity) keys[pos] = (static_cast<unsigned long long>(tile) << 32) | gg;
            o += __popc(m);
        }
    }
}

// K3+K4 fused (the default): one pass per chunk counts each rank's live tiles,
// scans the counts across the grid with a decoupled look-back (CTAs take logical
// block numbers from a ticket, so every predecessor a CTA waits on is already
// resident), and emits the keys at the scanned offsets. The last block finishes
// the scan as finish_scan_kernel does (total, overflow flag, chunk count).
// status[b] = flag << 62 | value: flag 1 = block aggregate, 2 = inclusive prefix.
constexpr unsigned long long kFlagAgg = 1ULL << 62;
constexpr unsigned long long kFlagPre = 2ULL << 62;
constexpr unsigned long long kValMask = (1ULL << 62) - 1;
constexpr int kBinThreads = 1024;

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
    const uint32_t* __restrict__ done_bytes, int tiles_x, int ntile, unsigned long long* __restrict__ keys,
    uint64_t capacity, unsigned long long* __restrict__ status, Counters* __restrict__ ctr) {
    extern __shared__ uint32_t done_bits[];
    __shared__ uint32_t s_blk;
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
                // finish the chunk's scan (finish_scan_kernel)
                const unsigned long long p = excl + total;
                ctr->tile_entries += p;
                if (p > ctr->max_chunk_entries) ctr->max_chunk_entries = p;
                if (p > capacity) ctr->key_overflow = 1;
                ctr->chunk_entries = p < capacity ? p : capacity;
            }
        }
    }
    __syncthreads();
    const unsigned long long off = s_base + s_warp[warp] + inc - c;
    const uint32_t w = static_cast<uint32_t>(rc.y - rc.x + 1);
    if (area && area <= kCoop) {
        uint32_t o = 0;
        for (uint32_t j = 0; j < area; ++j) {
            const uint32_t tile = static_cast<uint32_t>(rc.z + static_cast<int>(j / w)) * tiles_x +
                                  static_cast<uint32_t>(rc.x + static_cast<int>(j % w));
            if (done(tile)) continue;
            if (off + o < capacity) keys[off + o] = (static_cast<unsigned long long>(tile) << 32) | g;
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
            if (live && pos < capacity) keys[pos] = (static_cast<unsigned long long>(tile) << 32) | gg;
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
                                   const unsigned long long* __restrict__ keys, uint2* __restrict__ ranges) {
    const uint64_t p = *count;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < p;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t t = static_cast<uint32_t>(keys[i] >> 32);
        if (i == 0 || static_cast<uint32_t>(keys[i - 1] >> 32) != t) ranges[t].x = static_cast<uint32_t>(i);
        if (i == p - 1 || static_cast<uint32_t>(keys[i + 1] >> 32) != t)
            ranges[t].y = static_cast<uint32_t>(i + 1);
    }
}

__global__ void finish_scan_kernel(const unsigned long long* __restrict__ total, uint64_t capacity,
                                   Counters* __restrict__ ctr) {
    const unsigned long long p = *total;
    ctr->tile_entries += p;
    if (p > ctr->max_chunk_entries) ctr->max_chunk_entries = p;
    if (p > capacity) ctr->key_overflow = 1;
    ctr->chunk_entries = p < capacity ? p : capacity;
}

}  // namespace

static size_t bitmap_smem(const uint32_t* done, int ntile) {
    return done && ntile <= kMaxBitmapTiles ? static_cast<size_t>((ntile + 31) / 32) * 4 : 0;
}

void launch_gather_bins(uint64_t n, const uint32_t* order, const int4* rects, const Counters* ctr,
                        int4* brect, uint2* bmeta, cudaStream_t stream) {
    if (n == 0) return;
    gather_bins_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(n, order, rects, ctr,
                                                                                 brect, bmeta);
}

void launch_count_tiles(uint64_t rb, uint64_t re, const uint2* bmeta, const int4* brect,
                        const uint32_t* done, int tiles_x, int ntile, unsigned long long* counts,
                        cudaStream_t stream) {
    const uint64_t n = re - rb + 1;
    // large CTAs amortise the bitmap load
    count_tiles_kernel<<<static_cast<unsigned>((n + 1023) / 1024), 1024, bitmap_smem(done, ntile), stream>>>(
        rb, re, bmeta, brect, done, tiles_x, ntile, counts);
}

void launch_emit_tile_keys(uint64_t rb, uint64_t re, const uint2* bmeta, const int4* brect,
                           const uint32_t* done, const unsigned long long* offsets,
                           int tiles_x, int ntile, unsigned long long* keys, uint64_t capacity,
                           cudaStream_t stream) {
    if (re <= rb) return;
    const uint64_t n = re - rb;
    emit_keys_kernel<<<static_cast<unsigned>((n + 1023) / 1024), 1024, bitmap_smem(done, ntile), stream>>>(
        rb, re, bmeta, brect, done, offsets, tiles_x, ntile, keys, capacity);
}

void launch_tile_ranges(const unsigned long long* d_count, const unsigned long long* keys, uint2* ranges,
                        cudaStream_t stream) {
    tile_ranges_kernel<<<148 * 8, 256, 0, stream>>>(d_count, keys, ranges);
}

void launch_finish_scan(const unsigned long long* total, uint64_t capacity, Counters* ctr,
                        cudaStream_t stream) {
    finish_scan_kernel<<<1, 1, 0, stream>>>(total, capacity, ctr);
}

size_t bin_emit_status_bytes(uint64_t ranks) {
    return ((ranks + kBinThreads - 1) / kBinThreads + 1) * sizeof(unsigned long long);
}

void launch_bin_emit(uint64_t rb, uint64_t re, const uint2* bmeta, const int4* brect, const uint32_t* done,
                     int tiles_x, int ntile, unsigned long long* keys, uint64_t capacity,
                     unsigned long long* status, Counters* ctr, cudaStream_t stream) {
    const uint64_t n = re > rb ? re - rb : 0;
    const unsigned grid = static_cast<unsigned>(n ? (n + kBinThreads - 1) / kBinThreads : 1);
    cudaMemsetAsync(status, 0, (grid + 1) * sizeof(unsigned long long), stream);
    bin_emit_kernel<<<grid, kBinThreads, bitmap_smem(done, ntile), stream>>>(rb, re, bmeta, brect, done, tiles_x,
                                                                             ntile, keys, capacity, status, ctr);
}

void launch_counters_init(Counters* c, cudaStream_t stream) { counters_init_kernel<<<1, 32, 0, stream>>>(c); }

void launch_counters_publish(const Counters* d, Counters* h_mapped, cudaStream_t stream) {
    counters_publish_kernel<<<1, 32, 0, stream>>>(d, h_mapped);
}

}  // namespace sgs
