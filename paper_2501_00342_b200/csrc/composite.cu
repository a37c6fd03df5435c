// composite.cu -- K7: per-tile front-to-back alpha compositing.
//
// Replaces the per-pixel loop of render (proj/src/raster.cpp:155-186) with the
// reference's exact rules (Appendix A of SURVEY.md): pixel centre (px+.5, py+.5),
// m2 = c0 dx^2 + 2 c1 dx dy + c2 dy^2, skip m2 > 9, alpha = min(op e^{-m2/2}, 0.999),
// skip alpha < 1/255, accumulate c * alpha * T, T *= 1 - alpha, stop after the
// splat that pushed T below the threshold, then add T * background.
//
// One CTA per (tile, 256-pixel chunk); for the default 16x16 tile that is one CTA
// per tile, one thread per pixel. The tile's list is streamed through shared
// memory in batches of blockDim records (one coalesced 48-B record gather per
// thread), every thread then walks the batch from shared memory (broadcast LDS.128,
// no bank conflicts). __syncthreads_count ends the tile once every pixel is done.
//
// FP32 fast path with an FP64 guard band: the reference decides m2 > 9 and
// alpha < 1/255 in FP64. Here m2 is evaluated in FP32 from tile-local offsets
// (the FP64 mean is localised once per batch, so dx carries a single rounding), and
// a pair whose FP32 m2 lies within the splat's error bound `guard` of 9 -- or whose
// alpha lies within the matching relative bound of 1/255 -- is recomputed in FP64
// exactly as the reference does (no FMA contraction). Every skip decision therefore
// matches the FP64 reference; only the blended values carry FP32 rounding.
#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kBlock = 256;

// The reference's FP64 decisions for one (pixel, splat) pair (raster.cpp:165-176).
__device__ __noinline__ bool exact_alpha(const SplatRec* __restrict__ rec,
                                         const SplatRec64* __restrict__ rec64, uint32_t g,
                                         double cx, double cy, float* alpha_out) {
    const double mx = rec[g].mx, my = rec[g].my;
    const SplatRec64 r = rec64[g];
    const double dx = __dsub_rn(cx, mx), dy = __dsub_rn(cy, my);
    const double m2 = __dadd_rn(
        __dadd_rn(__dmul_rn(__dmul_rn(r.ca, dx), dx), __dmul_rn(__dmul_rn(__dmul_rn(2.0, r.cb), dx), dy)),
        __dmul_rn(__dmul_rn(r.cc, dy), dy));
    if (m2 > kSupportMahalanobisSq) return false;
    double alpha = __dmul_rn(r.op, exp(__dmul_rn(-0.5, m2)));
    alpha = alpha < kAlphaClamp ? alpha : kAlphaClamp;  // std::min(a, 0.999)
    if (alpha < kAlphaMin) return false;
    *alpha_out = static_cast<float>(alpha);
    return true;
}

__global__ void __launch_bounds__(kBlock) composite_kernel(
    const CamParams cam, const CfgParams cfg, int nchunks, int block_px,
    const uint2* __restrict__ ranges, const unsigned long long* __restrict__ keys,
    const SplatRec* __restrict__ rec, const SplatRec64* __restrict__ rec64, float3 bg,
    float* __restrict__ out_rgb, float* __restrict__ out_T, PixelState* __restrict__ state,
    uint32_t* __restrict__ processed_io, uint8_t* __restrict__ tile_done, int first, int last,
    Counters* __restrict__ ctr, int want_stats) {
    __shared__ float4 sA[kBlock];  // (lmx, lmy, ca, 2cb)
    __shared__ float4 sB[kBlock];  // (cc, op, guard, gaussian index bits)
    __shared__ float4 sC[kBlock];  // (r, g, b, -)
    __shared__ unsigned long long s_red[2][kBlock / 32];

    const int ts = cfg.tile_size;
    const int tile = blockIdx.x / nchunks;
    const int chunk = blockIdx.x - tile * nchunks;
    const int tx = tile % cfg.tiles_x, ty = tile / cfg.tiles_x;
    const int px0 = tx * ts, py0 = ty * ts;
    const int p = chunk * block_px + threadIdx.x;
    const int lx = p % ts, ly = p / ts;
    const int px = px0 + lx, py = py0 + ly;
    const bool valid = threadIdx.x < block_px && p < ts * ts && px < cam.W && py < cam.H;

    // Tiles that terminated in an earlier depth chunk already wrote their output.
    if (!first && tile_done[tile]) return;
    const uint2 range = ranges[tile];
    const uint32_t start = range.x, end = range.y;
    if (!first && !last && start == end) return;  // nothing new for this tile

    // Local pixel centre relative to the tile origin: exact in FP32.
    const float fcx = static_cast<float>(lx) + 0.5f, fcy = static_cast<float>(ly) + 0.5f;
    const float stop = cfg.early_stop;
    const size_t pix = valid ? static_cast<size_t>(py) * cam.W + px : 0;
    float T = 1.0f, ar = 0.f, ag = 0.f, ab = 0.f;
    uint32_t walked = 0;  // list entries walked in earlier chunks
    if (!first && valid) {
        const PixelState ps = state[pix];
        ar = ps.r;
        ag = ps.g;
        ab = ps.b;
        T = ps.T;
        walked = processed_io[pix];
    }
    // a pixel continues while T has not dropped below the threshold (raster.cpp:177)
    bool done = !valid || T < stop;
    uint32_t processed = done ? 0u : end - start;  // entries walked in this chunk
    uint32_t guard_hits = 0;

    for (uint32_t base = start; base < end; base += blockDim.x) {
        if (__syncthreads_count(!done) == 0) break;
        const uint32_t k = base + threadIdx.x;
        if (k < end) {
            const uint32_t g = static_cast<uint32_t>(keys[k]);
            const SplatRec r = rec[g];
            sA[threadIdx.x] = make_float4(static_cast<float>(r.mx - px0), static_cast<float>(r.my - py0),
                                          r.ca, r.cb2);
            sB[threadIdx.x] = make_float4(r.cc, r.op, r.guard, __uint_as_float(g));
            sC[threadIdx.x] = make_float4(r.r, r.g, r.b, 0.f);
        }
        __syncthreads();
        if (!done) {
            const uint32_t nb = min(static_cast<uint32_t>(blockDim.x), end - base);
            for (uint32_t j = 0; j < nb; ++j) {
                const float4 A = sA[j];
                const float dx = fcx - A.x, dy = fcy - A.y;
                const float4 B = sB[j];
                const float m2 = fmaf(fmaf(A.z, dx, A.w * dy), dx, B.x * dy * dy);
                const float G = B.z;
                if (m2 > 9.0f + G) continue;
                float alpha;
                bool exact = m2 >= 9.0f - G;
                if (!exact) {
                    alpha = fminf(B.y * __expf(-0.5f * m2), 0.999f);
                    const float tol = 0.003921568627f * fmaf(0.5f, G, 2e-6f);
                    if (alpha < 0.003921568627f + tol) {
                        if (alpha < 0.003921568627f - tol) continue;
                        exact = true;
                    }
                }
                if (exact) {
                    ++guard_hits;
                    if (!exact_alpha(rec, rec64, __float_as_uint(B.w), px + 0.5, py + 0.5, &alpha))
                        continue;
                }
                const float4 C = sC[j];
                const float w = alpha * T;
                ar += C.x * w;
                ag += C.y * w;
                ab += C.z * w;
                T *= 1.0f - alpha;
                if (T < stop) {
                    done = true;
                    processed = base + j + 1 - start;
                    break;
                }
            }
        }
        __syncthreads();
    }

    const bool all_done = __syncthreads_and(done) != 0;
    const bool finalize = last || all_done;
    if (valid) {
        if (finalize) {
            if (out_rgb) {
                out_rgb[pix * 3 + 0] = ar + T * bg.x;
                out_rgb[pix * 3 + 1] = ag + T * bg.y;
                out_rgb[pix * 3 + 2] = ab + T * bg.z;
            }
            if (out_T) out_T[pix] = T;
        } else {
            state[pix] = PixelState{ar, ag, ab, T};
            processed_io[pix] = walked + processed;
        }
    }
    if (!last && all_done && threadIdx.x == 0) tile_done[tile] = 1;
    if (want_stats) {
        // E_t (block-terminated entries) = max over the tile's pixels of the entries of
        // its full list each pixel walked (counted when the tile finalises); guard hits
        // summed over chunks.
        unsigned long long e = (finalize && valid) ? walked + processed : 0ULL;
        unsigned long long h = guard_hits;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
            h += __shfl_xor_sync(0xffffffffu, h, o);
        }
        const int warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
        if ((threadIdx.x & 31) == 0) {
            s_red[0][warp] = e;
            s_red[1][warp] = h;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long em = 0, hs = 0;
            for (int w = 0; w < nw; ++w) {
                em = max(em, s_red[0][w]);
                hs += s_red[1][w];
            }
            // pixel chunks of one tile (tile_size > 16) each report their own max
            if (em) atomicAdd(&ctr->block_entries, em);
            if (hs) atomicAdd(&ctr->guard_hits, hs);
        }
    }
}

}  // namespace

int composite_pixel_chunks(int ts) {
    const long long tile_px = static_cast<long long>(ts) * ts;
    const int block_px = static_cast<int>(tile_px < kBlock ? ((tile_px + 31) / 32) * 32 : kBlock);
    return static_cast<int>((tile_px + block_px - 1) / block_px);
}

void launch_composite(const CamParams& cam, const CfgParams& cfg, const uint2* ranges,
                      const unsigned long long* keys, const SplatRec* rec,
                      const SplatRec64* rec64, float3 bg, float* rgb, float* T,
                      PixelState* state, uint32_t* processed, uint8_t* tile_done, bool first,
                      bool last, Counters* counters, bool want_stats, cudaStream_t stream) {
    const int ts = cfg.tile_size;
    const long long tile_px = static_cast<long long>(ts) * ts;
    const int block_px = static_cast<int>(tile_px < kBlock ? ((tile_px + 31) / 32) * 32 : kBlock);
    const int nchunks = composite_pixel_chunks(ts);
    const long long ntiles = static_cast<long long>(cfg.tiles_x) * cfg.tiles_y;
    const long long grid = ntiles * nchunks;
    composite_kernel<<<static_cast<unsigned>(grid), block_px, 0, stream>>>(
        cam, cfg, nchunks, block_px, ranges, keys, rec, rec64, bg, rgb, T, state, processed,
        tile_done, first ? 1 : 0, last ? 1 : 0, counters, want_stats ? 1 : 0);
}

}  // namespace sgs
