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

__device__ __forceinline__ uint32_t live_tiles(const int4 rc, const uint8_t* __restrict__ done,
                                               int tiles_x) {
    uint32_t c = 0;
    for (int ty = rc.z; ty <= rc.w; ++ty)
        for (int tx = rc.x; tx <= rc.y; ++tx) c += done[ty * tiles_x + tx] ? 0u : 1u;
    return c;
}

__global__ void count_tiles_kernel(uint64_t rb, uint64_t re, const uint32_t* __restrict__ order,
                                   const uint32_t* __restrict__ ntiles,
                                   const int4* __restrict__ rects, const uint8_t* __restrict__ done,
                                   int tiles_x, unsigned long long* __restrict__ counts) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t r = rb + k;
    if (r < re) {
        const uint32_t g = order[r];
        uint32_t c = ntiles[g];
        if (c && done) c = live_tiles(rects[g], done, tiles_x);
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

__global__ void emit_keys_kernel(uint64_t rb, uint64_t re, const uint32_t* __restrict__ order,
                                 const uint32_t* __restrict__ ntiles,
                                 const int4* __restrict__ rects, const uint8_t* __restrict__ done,
                                 const unsigned long long* __restrict__ offsets, int tiles_x,
                                 unsigned long long* __restrict__ keys) {
    const uint64_t k = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t r = rb + k;
    const unsigned lane = threadIdx.x & 31;
    uint32_t g = 0, area = 0;
    int4 rc = make_int4(0, -1, 0, -1);
    unsigned long long off = 0;
    if (r < re) {
        g = order[r];
        area = ntiles[g];
        if (area) {
            rc = rects[g];
            off = offsets[k];
        }
    }
    const uint32_t w = static_cast<uint32_t>(rc.y - rc.x + 1);
    if (area && area <= kCoop) {
        uint32_t o = 0;
        for (uint32_t j = 0; j < area; ++j) {
            const uint32_t tile = static_cast<uint32_t>(rc.z + static_cast<int>(j / w)) * tiles_x +
                                  static_cast<uint32_t>(rc.x + static_cast<int>(j % w));
            if (done && done[tile]) continue;
            keys[off + o] = (static_cast<unsigned long long>(tile) << 32) | g;
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
                live = !(done && done[tile]);
            }
            const unsigned m = __ballot_sync(0xffffffffu, live);
            if (live) keys[o + __popc(m & ((1u << lane) - 1u))] = (static_cast<unsigned long long>(tile) << 32) | gg;
            o += __popc(m);
        }
    }
}

__global__ void tile_ranges_kernel(uint64_t p, const unsigned long long* __restrict__ keys,
                                   uint2* __restrict__ ranges) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p) return;
    const uint32_t t = static_cast<uint32_t>(keys[i] >> 32);
    if (i == 0 || static_cast<uint32_t>(keys[i - 1] >> 32) != t) ranges[t].x = static_cast<uint32_t>(i);
    if (i == p - 1 || static_cast<uint32_t>(keys[i + 1] >> 32) != t)
        ranges[t].y = static_cast<uint32_t>(i + 1);
}

}  // namespace

void launch_count_tiles(uint64_t rb, uint64_t re, const uint32_t* order, const uint32_t* ntiles,
                        const int4* rects, const uint8_t* done, int tiles_x,
                        unsigned long long* counts, cudaStream_t stream) {
    const uint64_t n = re - rb + 1;
    count_tiles_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
        rb, re, order, ntiles, rects, done, tiles_x, counts);
}

void launch_emit_tile_keys(uint64_t rb, uint64_t re, const uint32_t* order, const uint32_t* ntiles,
                           const int4* rects, const uint8_t* done, const unsigned long long* offsets,
                           int tiles_x, unsigned long long* keys, cudaStream_t stream) {
    if (re <= rb) return;
    const uint64_t n = re - rb;
    emit_keys_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(
        rb, re, order, ntiles, rects, done, offsets, tiles_x, keys);
}

void launch_tile_ranges(uint64_t p, const unsigned long long* keys, uint2* ranges,
                        cudaStream_t stream) {
    if (p == 0) return;
    const unsigned blocks = static_cast<unsigned>((p + 255) / 256);
    tile_ranges_kernel<<<blocks, 256, 0, stream>>>(p, keys, ranges);
}

}  // namespace sgs
