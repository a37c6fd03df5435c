// binning.cu -- K3 (per-rank tile counts), K4 (tile-key emission), K6 (tile ranges).
//
// Replaces build_tile_grid (proj/src/raster.cpp:108-130). The reference walks the
// splats in blending order and push_backs the rank into every tile of the
// inclusive rectangle. Here:
//   K3  counts[r] = ntiles[order[r]]          (gather into rank order; then a
//       device-wide exclusive scan gives each rank its first output slot)
//   K4  keys[off[r] + j] = (tile << 32) | gaussian_index, tiles row-major as the
//       reference's (ty, tx) double loop visits them; keys leave K4 in rank order
//   K5  stable radix sort on the tile bits only (capi.cu) keeps rank order inside a
//       tile, so each tile's run equals the reference's TileGrid list exactly
//   K6  ranges[tile] = [first, last + 1) of the tile's run.
#include "sgs_internal.h"

namespace sgs {
namespace {

__global__ void gather_counts_kernel(uint64_t n, const uint32_t* __restrict__ order,
                                     const uint32_t* __restrict__ ntiles,
                                     unsigned long long* __restrict__ counts) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r < n) counts[r] = ntiles[order[r]];
    if (r == n) counts[r] = 0;  // scan over n+1 items leaves P in offsets[n]
}

// One warp per 32 ranks; each lane emits its splat's tiles. A splat covering many
// tiles is spread over the warp: lanes cooperatively walk the union of the warp's
// rectangles so long rows do not serialise on one lane.
__global__ void emit_keys_kernel(uint64_t n, const uint32_t* __restrict__ order,
                                 const uint32_t* __restrict__ ntiles,
                                 const int4* __restrict__ rects,
                                 const unsigned long long* __restrict__ offsets, int tiles_x,
                                 unsigned long long* __restrict__ keys) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const unsigned lane = threadIdx.x & 31;
    uint32_t g = 0, cnt = 0;
    int4 rc = make_int4(0, -1, 0, -1);
    unsigned long long off = 0;
    if (r < n) {
        g = order[r];
        cnt = ntiles[g];
        if (cnt) {
            rc = rects[g];
            off = offsets[r];
        }
    }
    // Work items: the warp processes each lane's splat in turn, all 32 lanes
    // striding over that splat's cnt tiles (coalesced stores into [off, off+cnt)).
    unsigned pending = __ballot_sync(0xffffffffu, cnt > 0);
    while (pending) {
        const int src = __ffs(pending) - 1;
        pending &= pending - 1;
        const uint32_t c = __shfl_sync(0xffffffffu, cnt, src);
        const uint32_t gg = __shfl_sync(0xffffffffu, g, src);
        const int x0 = __shfl_sync(0xffffffffu, rc.x, src);
        const int x1 = __shfl_sync(0xffffffffu, rc.y, src);
        const int y0 = __shfl_sync(0xffffffffu, rc.z, src);
        const unsigned long long o = __shfl_sync(0xffffffffu, off, src);
        const uint32_t w = static_cast<uint32_t>(x1 - x0 + 1);
        for (uint32_t j = lane; j < c; j += 32) {
            const uint32_t ty = static_cast<uint32_t>(y0) + j / w;
            const uint32_t tx = static_cast<uint32_t>(x0) + j % w;
            const unsigned long long tile = static_cast<unsigned long long>(ty) * tiles_x + tx;
            keys[o + j] = (tile << 32) | gg;
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

void launch_gather_counts(uint64_t n, const uint32_t* order, const uint32_t* ntiles,
                          unsigned long long* counts, cudaStream_t stream) {
    const unsigned blocks = static_cast<unsigned>((n + 1 + 255) / 256);
    gather_counts_kernel<<<blocks, 256, 0, stream>>>(n, order, ntiles, counts);
}

void launch_emit_tile_keys(uint64_t n_visible, const uint32_t* order, const uint32_t* ntiles,
                           const int4* rects, const unsigned long long* offsets, int tiles_x,
                           unsigned long long* keys, cudaStream_t stream) {
    if (n_visible == 0) return;
    const unsigned blocks = static_cast<unsigned>((n_visible + 255) / 256);
    emit_keys_kernel<<<blocks, 256, 0, stream>>>(n_visible, order, ntiles, rects, offsets, tiles_x,
                                                 keys);
}

void launch_tile_ranges(uint64_t p, const unsigned long long* keys, uint2* ranges,
                        cudaStream_t stream) {
    if (p == 0) return;
    const unsigned blocks = static_cast<unsigned>((p + 255) / 256);
    tile_ranges_kernel<<<blocks, 256, 0, stream>>>(p, keys, ranges);
}

}  // namespace sgs
