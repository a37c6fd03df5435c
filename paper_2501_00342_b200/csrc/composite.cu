// composite.cu -- K7: per-tile front-to-back alpha compositing.
//
// Replaces the per-pixel loop of render (proj/src/raster.cpp:155-186) with the
// reference's exact rules: pixel centre (px+.5, py+.5),
// m2 = c0 dx^2 + 2 c1 dx dy + c2 dy^2, skip m2 > 9, alpha = min(op e^{-m2/2}, 0.999),
// skip alpha < 1/255, accumulate c * alpha * T, T *= 1 - alpha, stop after the
// splat that pushed T below the threshold, then add T * background.
//
// composite_kernel: independent warps, each compositing one 64-pixel part of a
// tile (an 8x8 quadrant of a 16x16 tile), two horizontally adjacent pixels per
// thread.
//
// Layout. The tile's list streams through the warp's shared memory in batches of 64
// 64-B records (cp.async gathers, double-buffered). The warp compacts each batch to
// the records whose support box reaches its live pixels (ballot + popc).
//
// Latency. A pixel's walk is inherently sequential, so long lists (tiles on the
// silhouette whose pixels never saturate) sit on the critical path. The walk goes
// in groups of kGroup records: the m2 / alpha of the group are computed
// independently (ILP), then a branch-free blend chain applies them in order; a
// skipped pair, or any pair after the pixel terminated, blends with alpha = 0,
// which leaves T and the colour bit-identical. The warp leaves its part once every
// pixel in it has terminated.
//
// Exactness. The two skip tests are one per-splat cutoff: alpha < 1/255 <=>
// m2 > 2 ln(255 op), so "skip" <=> m2 > cut = min(9, 2 ln(255 op)) (FP64 in K1).
// m2 is evaluated in FP32 from tile-local offsets (the FP64 mean is localised once
// per batch, so dx carries a single rounding) and compared with cut +- guard,
// guard bounding the FP32 error. A group containing a
// pair inside the band is walked one record at a time, that pair decided in FP64
// exactly as the reference does from the FP64 projection re-derived by
// projection.cuh. Every skip decision therefore matches the reference; only the
// blended values carry FP32 rounding.
#include <cstdlib>

#include "projection.cuh"

namespace sgs {
namespace {

constexpr int kChunkPx = 256;  // pixels per K7 work item (one 16x16 tile)

// The reference's FP64 decision for one (pixel, splat) pair (raster.cpp:165-176).
__device__ __noinline__ bool exact_alpha(const FrameConsts* __restrict__ fc, uint32_t g, int px, int py,
                                         float* alpha_out) {
    const double cx = px + 0.5, cy = py + 0.5;  // raster.cpp:165
    Geo geo;
    ProjGeo pg;
    if (fc->sp.geometry_f64)
        project_geometry<true>(fc->sp, fc->cam, g, geo, pg);
    else
        project_geometry<false>(fc->sp, fc->cam, g, geo, pg);
    exact_conic_opacity(geo, pg);
    const double dx = dsub(cx, pg.mx), dy = dsub(cy, pg.my);
    const double m2 = dadd(dadd(dmul(dmul(pg.cona, dx), dx), dmul(dmul(dmul(2.0, pg.conb), dx), dy)),
                           dmul(dmul(pg.conc, dy), dy));
    if (m2 > kSupportMahalanobisSq) return false;
    double alpha = dmul(pg.opacity, exp(dmul(-0.5, m2)));
    alpha = kAlphaClamp < alpha ? kAlphaClamp : alpha;  // std::min(a, 0.999): NaN stays NaN
    if (alpha < kAlphaMin) return false;
    *alpha_out = static_cast<float>(alpha);
    return true;
}

// cp.async of one splat's 48-B record and 16-B colour into a 64-B smem slot:
// [0] (mx, my) [1] (ca, 2cb, cc, log2 op) [2] (cut, guard, ext_x, ext_y) [3] (r, g, b, -)
__device__ __forceinline__ void stage_record(const SplatRec* __restrict__ rec, const float4* __restrict__ colour,
                                             uint32_t g, float4* slot) {
    const char* src = reinterpret_cast<const char*>(rec + g);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(&slot[c]));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + 16 * c));
    }
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(&slot[3]));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(colour + g));
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float fast_alpha(float m2, float lop) {
    // op * exp(-m2/2) = 2^(log2 op - m2 log2(e)/2), clamped at 0.999 (the decision
    // that alpha >= 1/255 was already taken exactly on m2)
    return fminf(ex2_approx(fmaf(m2, -0.72134752044448170f, lop)), 0.999f);
}

constexpr int kWorkCtl = 8;
constexpr int kWorkClasses = 6;  // list-length classes, longest first (LPT order for the persistent CTAs)

__device__ __forceinline__ int work_class(uint32_t len) {
    return len >= 4096 ? 0 : len >= 2048 ? 1 : len >= 1024 ? 2 : len >= 512 ? 3 : len >= 128 ? 4 : 5;
}

// item-th entry of the class-ordered work list (class c's items at work[c * cap ...]).
__device__ __forceinline__ uint32_t work_item(const uint32_t* __restrict__ work, const uint32_t* n_class,
                                              uint32_t cap, uint32_t item) {
#pragma unroll
    for (int c = 0; c < kWorkClasses - 1; ++c) {
        if (item < n_class[c]) return work[static_cast<size_t>(c) * cap + item];
        item -= n_class[c];
    }
    return work[static_cast<size_t>(kWorkClasses - 1) * cap + item];
}

// Background-only (tile, pixel-chunk) items of the last chunk, flat over all CTAs:
// the pixels of a tile that never received an entry are bg (acc 0 + T 1 * bg).
template <int NT>
__device__ __forceinline__ void write_background(int W, int H, const CfgParams& cfg, int nchunks,
                                                 const uint32_t* __restrict__ work_count, float* __restrict__ out_rgb,
                                                 float* __restrict__ out_T, float3 bg) {
    const uint32_t n_bg = work_count[7];
    const uint32_t* bgl = work_count + kWorkCtl;
    const int ts = cfg.tile_size;
    const uint64_t total = static_cast<uint64_t>(n_bg) * 256;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * NT + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * NT) {
        const uint32_t it = bgl[i >> 8];
        const int tile = static_cast<int>(it / nchunks), chunk = static_cast<int>(it % nchunks);
        const int p = chunk * 256 + static_cast<int>(i & 255);
        if (p >= ts * ts) continue;
        const int px = (tile % cfg.tiles_x) * ts + p % ts, py = (tile / cfg.tiles_x) * ts + p / ts;
        if (px >= W || py >= H) continue;
        const size_t pix = static_cast<size_t>(py) * W + px;
        if (out_rgb) {
            out_rgb[pix * 3 + 0] = 0.0f + 1.0f * bg.x;
            out_rgb[pix * 3 + 1] = 0.0f + 1.0f * bg.y;
            out_rgb[pix * 3 + 2] = 0.0f + 1.0f * bg.z;
        }
        if (out_T) out_T[pix] = 1.0f;
    }
}

// ---------------------------------------------------------------------------
// K7. Every warp is an independent compositor: it takes its own (tile, 64-pixel part)
// items from the work list -- on 16x16 tiles one 8x8 quadrant -- and streams the
// tile's list through its own double-buffered shared-memory ring, so no warp ever
// waits for another (the CTA only groups four warps for residency). A thread owns
// two horizontally adjacent pixels (2c, 2c+1) of one row, so a record's dy terms
// (dy, 2b dy, c dy^2) and its shared-memory reads serve both pixels. m2 is formed
// per pixel with the same operations and rounding for both pixels, and the blend
// chain drops the per-step termination bookkeeping: transmittance only decreases, so
// "the pixel stopped before this splat" is T < stop, tested in the chain; the splat
// that stopped it is found afterwards by replaying the group's T products
// (bit-identical), which happens once per pixel. Each record is staged once per warp
// that needs it (4x the L2 reads of a CTA-shared stage, ~200 MB/frame at config C,
// and ~3% more instructions), in exchange for no CTA barrier anywhere in the walk.
constexpr int kThreads = 128;  // four independent warps per CTA
constexpr int kWB = 64;        // records per warp batch (two per lane)
constexpr int kSubPx = 64;     // pixels per warp item (two per lane)
constexpr int kSubsPerChunk = kChunkPx / kSubPx;

// One warp's staging: 64-B records, double-buffered (cp.async). After arrival each
// lane rewrites its records in place as [0] (lmx, lmy, ca, 2cb), [1] (cc, cut + guard,
// cut - guard, log2 op), [2] (r, g, b, gaussian index bits), and the filter box into
// box. Slot kWB of each buffer is a null record (never contributes) that pads the
// compacted lists to whole groups.
struct WarpStage {
    float4 raw[2][kWB + 1][4];
    float4 box[kWB];
    uint32_t idx[kWB + 8];
};
static_assert(sizeof(WarpStage) % 16 == 0, "warp stage alignment");

struct Pix {
    float T, r, g, b;
};

// One blend step (raster.cpp:177-180) unless the pixel already stopped.
__device__ __forceinline__ void step2(Pix& P, float alpha, const float4& C, float stop) {
    const float a = P.T < stop ? 0.0f : alpha;
    const float w = a * P.T;
    P.r = fmaf(C.x, w, P.r);
    P.g = fmaf(C.y, w, P.g);
    P.b = fmaf(C.z, w, P.b);
    P.T = P.T * (1.0f - a);
}

// m2 of both pixels; same formula as mahal2 (dy terms shared when on one row).
template <bool kSameRow>
__device__ __forceinline__ void mahal2x2(const float4& A, float Bx, float fcx0, float fcy0, float fcx1, float fcy1,
                                         float& m0, float& m1) {
    const float dy0 = fcy0 - A.y;
    const float b0 = A.w * dy0, c0 = Bx * dy0 * dy0;
    const float dx0 = fcx0 - A.x, dx1 = fcx1 - A.x;
    m0 = fmaf(fmaf(A.z, dx0, b0), dx0, c0);
    if constexpr (kSameRow) {
        m1 = fmaf(fmaf(A.z, dx1, b0), dx1, c0);
    } else {
        const float dy1 = fcy1 - A.y;
        m1 = fmaf(fmaf(A.z, dx1, A.w * dy1), dx1, Bx * dy1 * dy1);
    }
}

// Flags of a depth-chunked frame: tiles finished (binning skips them); per part
// (bit tile * 4 + part: depth chunking runs on tiles of at most 256 pixels, so a tile
// has at most 4 parts) whether its pixel state was written by an earlier chunk and
// whether it is final. A part's two bits are read and written only by the warp
// compositing it (and by the work-list kernel between launches): the parts of one
// tile run concurrently.
struct TileFlags {
    uint32_t* done;
    uint32_t* touched;
    uint32_t* sub_done;
};

__device__ __forceinline__ bool part_bit(const uint32_t* bits, uint32_t tile, uint32_t part) {
    const uint32_t b = tile * 4u + part;
    return (bits[b >> 5] >> (b & 31)) & 1u;
}

// True only when no point of the box [x0, x1] x [y0, y1] (tile-local pixel centres)
// can reach the record: the minimum over the box of its FP32 quadratic form
// m2(d) = ca dx^2 + 2cb dx dy + cc dy^2 (d = point - mean) exceeds cut + 3 guard (the
// guard bounds the FP32 error of m2 near the cut: once for the walk's per-pixel m2,
// once for this minimum, once to spare) and a relative 1e-4 -- so every live pixel of
// the warp would take the record's skip branch (alpha 0, no exact re-decision) and the
// walk may leave it out. The minimum of the convex form over a box not containing the
// mean lies on an edge, at the edge's clamped 1-D vertex. A degenerate or non-finite
// form never misses.
__device__ __forceinline__ bool ellipse_misses_box(const float4 A, const float4 B, float x0, float x1, float y0,
                                                   float y1) {
    const float ca = A.z, cb2 = A.w, cc = B.x, thr = B.y + (B.y - B.z);  // cut + 3 guard
    const float dx0 = x0 - A.x, dx1 = x1 - A.x, dy0 = y0 - A.y, dy1 = y1 - A.y;
    if (dx0 <= 0.0f && dx1 >= 0.0f && dy0 <= 0.0f && dy1 >= 0.0f) return false;  // the mean is inside
    if (!(ca > 0.0f && cc > 0.0f && thr < 1e30f)) return false;
    const float hc = -0.5f * cb2 / cc, ha = -0.5f * cb2 / ca;
    auto on_x = [&](float X) {  // the edge dx = X, its minimum over dy
        const float y = fminf(fmaxf(hc * X, dy0), dy1);
        return fmaf(fmaf(ca, X, cb2 * y), X, cc * y * y);
    };
    auto on_y = [&](float Y) {  // the edge dy = Y, its minimum over dx
        const float x = fminf(fmaxf(ha * Y, dx0), dx1);
        return fmaf(fmaf(cc, Y, cb2 * x), Y, ca * x * x);
    };
    const float qmin = fminf(fminf(on_x(dx0), on_x(dx1)), fminf(on_y(dy0), on_y(dy1)));
    return qmin * 0.9999f - 1e-4f > thr;
}

template <int kGroup, int MINB, bool kSameRow>
__global__ void __launch_bounds__(kThreads, MINB) composite_kernel(
    const FrameConsts* __restrict__ fc, const int W, const int H, const CfgParams cfg, int nchunks,
    const uint2* __restrict__ ranges, const uint32_t* __restrict__ keys,
    const SplatRec* __restrict__ rec, const float4* __restrict__ colour, float3 bg,
    PixelState* __restrict__ state, uint32_t* __restrict__ processed_io, const TileFlags flags, int first, int last,
    Counters* __restrict__ ctr, int want_stats, uint32_t* __restrict__ tile_emax, const uint32_t* __restrict__ work,
    const uint32_t* __restrict__ work_count, uint32_t* __restrict__ work_next, uint32_t work_cap) {
    extern __shared__ float4 k7_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpStage& S = reinterpret_cast<WarpStage*>(k7_smem)[warp];
    float* const out_rgb = fc->out_rgb;  // the frame's outputs (FrameConsts)
    float* const out_T = fc->out_T;
    if (lane < 8) {
        const int b = lane >> 2, c = lane & 3;
        S.raw[b][kWB][c] = c == 1 ? make_float4(0.f, -1.f, -2.f, -1e30f) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();
    uint32_t n_class[kWorkClasses], n_items = 0;
#pragma unroll
    for (int c = 0; c < kWorkClasses; ++c) n_items += (n_class[c] = work_count[c]);
    // T < stop is the stop test; a threshold above 1 stops every pixel right after
    // its first blended splat, exactly as 1.0 does (T starts at 1 and every blended
    // splat has alpha >= 1/255), and keeps T < stop false for a pixel that has not
    // blended anything yet.
    const float stop = cfg.early_stop > 1.0f ? 1.0f : cfg.early_stop;
    const int nsub = kSubsPerChunk * nchunks;
    const int ts = cfg.tile_size;
    for (;;) {
    uint32_t item = 0;
    if (lane == 0) item = atomicAdd(work_next, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    const uint32_t witem = work_item(work, n_class, work_cap, item);
    const int tile = static_cast<int>(witem / nsub);
    const int sub = static_cast<int>(witem - static_cast<uint32_t>(tile) * nsub);
    const uint2 range = ranges[tile];
    const uint32_t start = range.x, end = range.y;
    const bool touched = !first && part_bit(flags.touched, tile, sub);
    const int tx = tile % cfg.tiles_x, ty = tile / cfg.tiles_x;
    const int px0 = tx * ts, py0 = ty * ts;
    int lx0, ly0, lx1, ly1;
    bool in0, in1;
    if (ts == 16) {
        // part q is the 8x8 quadrant (q & 1, q >> 1): a square strip meets fewer
        // splat boxes per pixel than a 16x4 one
        lx0 = (sub & 1) * 8 + (lane & 3) * 2;
        lx1 = lx0 + 1;
        ly0 = ly1 = (sub >> 1) * 8 + (lane >> 2);
        in0 = in1 = true;
    } else {
        const int p = sub * kSubPx + 2 * lane;
        lx0 = p % ts;
        ly0 = p / ts;
        lx1 = (p + 1) % ts;
        ly1 = (p + 1) / ts;
        in0 = p < ts * ts;
        in1 = p + 1 < ts * ts;
    }
    const int pxa = px0 + lx0, pya = py0 + ly0, pxb = px0 + lx1, pyb = py0 + ly1;
    const bool v0 = in0 && pxa < W && pya < H, v1 = in1 && pxb < W && pyb < H;
    const uint32_t pix0 = v0 ? static_cast<uint32_t>(pya) * W + pxa : 0;  // (W H < 2^32)
    const uint32_t pix1 = v1 ? static_cast<uint32_t>(pyb) * W + pxb : 0;
    const float fcx0 = static_cast<float>(lx0) + 0.5f, fcy0 = static_cast<float>(ly0) + 0.5f;
    const float fcx1 = static_cast<float>(lx1) + 0.5f, fcy1 = static_cast<float>(ly1) + 0.5f;
    Pix P0{1.f, 0.f, 0.f, 0.f}, P1{1.f, 0.f, 0.f, 0.f};
    uint32_t walked0 = 0, walked1 = 0;
    if (touched) {
        if (v0) {
            const PixelState st = state[pix0];
            P0 = Pix{st.T, st.r, st.g, st.b};
            walked0 = processed_io[pix0];
        }
        if (v1) {
            const PixelState st = state[pix1];
            P1 = Pix{st.T, st.r, st.g, st.b};
            walked1 = processed_io[pix1];
        }
    }
    bool live0 = v0 && !(P0.T < stop), live1 = v1 && !(P1.T < stop);
    uint32_t processed0 = live0 ? end - start : 0u, processed1 = live1 ? end - start : 0u;
    int term0 = -1, term1 = -1;  // compacted-walk position of the stopping splat in this batch
    uint32_t guard_hits = 0;

    uint32_t g_next[2], g_cur[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t k = start + lane + h * 32;
        g_next[h] = k < end ? __ldg(&keys[k]) : 0u;
        if (k < end) stage_record(rec, colour, g_next[h], S.raw[0][lane + h * 32]);
    }
    asm volatile("cp.async.commit_group;\n" ::);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        g_cur[h] = g_next[h];
        const uint32_t k = start + kWB + lane + h * 32;
        g_next[h] = k < end ? __ldg(&keys[k]) : 0u;
    }
    int buf = 0;

    for (uint32_t base = start; base < end; base += kWB) {
        if (!__any_sync(0xffffffffu, live0 || live1)) break;
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncwarp();  // every lane's records landed; the previous batch is walked
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rt = lane + h * 32;
            if (base + rt < end) {
                float4* r = S.raw[buf][rt];
                const double2 m = *reinterpret_cast<const double2*>(&r[0]);
                const float4 q1 = r[1];
                const float4 q2 = r[2];
                const float4 q3 = r[3];
                const float lmx = static_cast<float>(m.x - px0), lmy = static_cast<float>(m.y - py0);
                r[0] = make_float4(lmx, lmy, q1.x, q1.y);
                r[1] = make_float4(q1.z, q2.x + q2.y, q2.x - q2.y, q1.w);
                r[2] = make_float4(q3.x, q3.y, q3.z, __uint_as_float(g_cur[h]));
                S.box[rt] = make_float4(lmx, lmy, q2.z, q2.w);
            }
            const uint32_t kn = base + kWB + rt;
            if (kn < end) stage_record(rec, colour, g_next[h], S.raw[buf ^ 1][rt]);
            g_cur[h] = g_next[h];
            g_next[h] = kn + kWB < end ? __ldg(&keys[kn + kWB]) : 0u;
        }
        asm volatile("cp.async.commit_group;\n" ::);
        buf ^= 1;
        __syncwarp();
        const uint32_t nb = min(static_cast<uint32_t>(kWB), end - base);
        const float4(*R)[4] = S.raw[buf ^ 1];
        int cnt = 0;
        {
            // the warp's live-pixel box, shrinking as its pixels stop
            float wx0 = 1e30f, wx1 = -1e30f, wy0 = 1e30f, wy1 = -1e30f;
            if (live0) wx0 = fminf(wx0, fcx0), wx1 = fmaxf(wx1, fcx0), wy0 = fminf(wy0, fcy0), wy1 = fmaxf(wy1, fcy0);
            if (live1) wx0 = fminf(wx0, fcx1), wx1 = fmaxf(wx1, fcx1), wy0 = fminf(wy0, fcy1), wy1 = fmaxf(wy1, fcy1);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                wx0 = fminf(wx0, __shfl_xor_sync(0xffffffffu, wx0, o));
                wx1 = fmaxf(wx1, __shfl_xor_sync(0xffffffffu, wx1, o));
                wy0 = fminf(wy0, __shfl_xor_sync(0xffffffffu, wy0, o));
                wy1 = fmaxf(wy1, __shfl_xor_sync(0xffffffffu, wy1, o));
            }
#pragma unroll
            for (uint32_t j0 = 0; j0 < kWB; j0 += 32) {
                const uint32_t j = j0 + lane;
                bool hit = false;
                if (j < nb) {
                    const float4 F = S.box[j];
                    hit = F.x - F.z <= wx1 && F.x + F.z >= wx0 && F.y - F.w <= wy1 && F.y + F.w >= wy0;
                    if (hit) hit = !ellipse_misses_box(R[j][0], R[j][1], wx0, wx1, wy0, wy1);
                }
                const unsigned m = __ballot_sync(0xffffffffu, hit);
                if (hit) S.idx[cnt + __popc(m & ((1u << lane) - 1u))] = j;
                cnt += __popc(m);
            }
        }
        if (lane < kGroup) S.idx[cnt + lane] = kWB;
        __syncwarp();
        const uint32_t* idx = S.idx;
        // Fast groups until one holds a pair inside the guard band; that group is
        // walked by the cold path below (outside the fast loop, so the FP64 call does
        // not weigh on the fast loop's registers), then the fast loop resumes.
        int q = 0;
        while (q < cnt && (live0 || live1)) {
            for (; q < cnt && (live0 || live1); q += kGroup) {
                float a0[kGroup], a1[kGroup];
                bool guard = false;
#pragma unroll
                for (int k = 0; k < kGroup; ++k) {
                    const int j = idx[q + k];
                    const float4 A = R[j][0];
                    const float4 B = R[j][1];
                    float m0, m1;
                    mahal2x2<kSameRow>(A, B.x, fcx0, fcy0, fcx1, fcy1, m0, m1);
                    guard |= (m0 <= B.y && m0 >= B.z) || (m1 <= B.y && m1 >= B.z);
                    a0[k] = m0 < B.z ? fast_alpha(m0, B.w) : 0.0f;
                    a1[k] = m1 < B.z ? fast_alpha(m1, B.w) : 0.0f;
                }
                if (guard) break;
                const float T0s = P0.T, T1s = P1.T;
#pragma unroll
                for (int k = 0; k < kGroup; ++k) {
                    const float4 C = R[idx[q + k]][2];
                    step2(P0, a0[k], C, stop);
                    step2(P1, a1[k], C, stop);
                }
                if (live0 && P0.T < stop) {  // stopped inside this group: find the splat
                    float tt = T0s;
#pragma unroll
                    for (int k = 0; k < kGroup; ++k) {
                        tt = tt * (1.0f - a0[k]);
                        if (tt < stop) {
                            term0 = q + k;
                            break;
                        }
                    }
                    live0 = false;
                }
                if (live1 && P1.T < stop) {
                    float tt = T1s;
#pragma unroll
                    for (int k = 0; k < kGroup; ++k) {
                        tt = tt * (1.0f - a1[k]);
                        if (tt < stop) {
                            term1 = q + k;
                            break;
                        }
                    }
                    live1 = false;
                }
            }
            if (!(q < cnt && (live0 || live1))) break;
            // the group at q holds a banded pair: one record at a time, banded pairs in FP64
            for (int k = 0; k < kGroup && q + k < cnt && (live0 || live1); ++k) {
                const int j = idx[q + k];
                const float4 A = R[j][0];
                const float4 B = R[j][1];
                const float4 C = R[j][2];
                float m[2];
                mahal2x2<kSameRow>(A, B.x, fcx0, fcy0, fcx1, fcy1, m[0], m[1]);
#pragma unroll 1
                for (int e = 0; e < 2; ++e) {
                    Pix& P = e ? P1 : P0;
                    bool& live = e ? live1 : live0;
                    if (!live || m[e] > B.y) continue;
                    float a;
                    if (m[e] < B.z) {
                        a = fast_alpha(m[e], B.w);
                    } else {  // inside the band (or NaN): the reference's FP64 decision
                        ++guard_hits;
                        if (!exact_alpha(fc, __float_as_uint(C.w), e ? pxb : pxa, e ? pyb : pya, &a)) continue;
                    }
                    step2(P, a, C, stop);
                    if (P.T < stop) {
                        (e ? term1 : term0) = q + k;
                        live = false;
                    }
                }
            }
            q += kGroup;
        }
        if (term0 >= 0) {
            processed0 = base + idx[term0] + 1 - start;
            term0 = -2;
        }
        if (term1 >= 0) {
            processed1 = base + idx[term1] + 1 - start;
            term1 = -2;
        }
    }

    asm volatile("cp.async.wait_all;\n" ::);
    __syncwarp();  // (the next item restages buffer 0)
    const bool all_done = !__any_sync(0xffffffffu, live0 || live1);
    const bool finalize = last || all_done;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const bool v = e ? v1 : v0;
        if (!v) continue;
        const Pix& P = e ? P1 : P0;
        const size_t pix = e ? pix1 : pix0;
        if (finalize) {
            if (out_rgb) {
                out_rgb[pix * 3 + 0] = P.r + P.T * bg.x;
                out_rgb[pix * 3 + 1] = P.g + P.T * bg.y;
                out_rgb[pix * 3 + 2] = P.b + P.T * bg.z;
            }
            if (out_T) out_T[pix] = P.T;
        } else {
            state[pix] = PixelState{P.r, P.g, P.b, P.T};
            processed_io[pix] = (e ? walked1 : walked0) + (e ? processed1 : processed0);
        }
    }
    if (lane == 0) {
        if (!last && all_done) {
            // this part is final; the tile is finished once all its parts are
            const uint32_t b = static_cast<uint32_t>(tile) * 4u + static_cast<uint32_t>(sub);
            const uint32_t old = atomicOr(&flags.sub_done[b >> 5], 1u << (b & 31));
            const int parts = min(4, (ts * ts + kSubPx - 1) / kSubPx);
            const uint32_t need = (1u << parts) - 1u, sh = (static_cast<uint32_t>(tile) * 4u) & 31u;
            const uint32_t before = (old >> sh) & need, after = ((old | (1u << (b & 31))) >> sh) & need;
            if (after == need && before != need) atomicOr(&flags.done[tile >> 5], 1u << (tile & 31));
        }
        if (!finalize && !touched) {
            const uint32_t b = static_cast<uint32_t>(tile) * 4u + static_cast<uint32_t>(sub);
            atomicOr(&flags.touched[b >> 5], 1u << (b & 31));
        }
    }
    if (want_stats) {
        unsigned long long e = 0;
        if (finalize && v0) e = max(e, static_cast<unsigned long long>(walked0 + processed0));
        if (finalize && v1) e = max(e, static_cast<unsigned long long>(walked1 + processed1));
        unsigned long long h = guard_hits;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            e = max(e, __shfl_xor_sync(0xffffffffu, e, o));
            h += __shfl_xor_sync(0xffffffffu, h, o);
        }
        if (lane == 0) {
            // E_t counts the deepest entry of each (tile, 256-pixel chunk)
            if (e) atomicMax(&tile_emax[static_cast<size_t>(tile) * nchunks + sub / kSubsPerChunk],
                             static_cast<uint32_t>(e));
            if (h) atomicAdd(&ctr->guard_hits, h);
        }
    }
    }  // persistent loop
    // background-only items (tiles that never received an entry): T = 1, rgb = bg
    write_background<kThreads>(W, H, cfg, nchunks, work_count, out_rgb, out_T, bg);
}

// Work buffer: kWorkClasses regions of cap items, one per list-length class (the
// persistent warps take the longest lists first); then kWorkCtl control words (the
// class counts, the compositor's cursor [6], the background count [7]); then the
// background-only (tile, pixel chunk) items.
// Work list of a depth chunk: (tile, 64-pixel part) items that still need K7 -- every
// unfinished part in the last chunk (it writes the final pixels), otherwise only
// parts of tiles with entries in this chunk.
__global__ void build_work_kernel(const uint2* __restrict__ ranges, const TileFlags flags, int first, int last,
                                  uint32_t ntile, int nchunks, int tile_px, uint32_t cap, uint32_t* __restrict__ work,
                                  uint32_t* __restrict__ wctl) {
    const uint32_t nsub = static_cast<uint32_t>(kSubsPerChunk * nchunks);
    const uint32_t it = blockIdx.x * blockDim.x + threadIdx.x;
    // the list this item joins: a length class, kWorkClasses for the background list,
    // or none (-1); every lane reaches the warp-aggregated append below
    int dest = -1;
    uint32_t value = 0;
    if (it < ntile * nsub) {
        const uint32_t tile = it / nsub, sub = it - tile * nsub;
        bool skip = static_cast<int>(sub) * kSubPx >= tile_px;  // a part without pixels
        // (a later depth chunk: at most 4 parts per tile)
        skip = skip || (!first && ((flags.done[tile >> 5] >> (tile & 31)) & 1u));
        skip = skip || (!first && part_bit(flags.sub_done, tile, sub));  // final already
        if (!skip) {
            const uint2 r = ranges[tile];
            const uint32_t len = r.y - r.x;
            if (last || len != 0) {
                // A part that is neither final nor touched was never composited: then no
                // part of the tile was (all parts of a tile are queued in the same chunks,
                // and each ends final or touched), and without entries the tile is
                // background, written by the tail loop (one item per 256-pixel chunk).
                if (len == 0 && (first || !part_bit(flags.touched, tile, sub))) {
                    if (sub % kSubsPerChunk == 0) {
                        dest = kWorkClasses;
                        value = tile * nchunks + sub / kSubsPerChunk;
                    }
                } else {
                    dest = work_class(len);
                    value = it;
                }
            }
        }
    }
    // one atomic per (warp, list): lanes bound for the same list take consecutive slots
    const unsigned lane = threadIdx.x & 31;
    const unsigned peers = __match_any_sync(0xffffffffu, dest);
    if (dest < 0) return;
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (static_cast<int>(lane) == leader)
        base = atomicAdd(dest == kWorkClasses ? &wctl[7] : &wctl[dest], static_cast<uint32_t>(__popc(peers)));
    base = __shfl_sync(peers, base, leader) + __popc(peers & ((1u << lane) - 1u));
    if (dest == kWorkClasses)
        wctl[kWorkCtl + base] = value;
    else
        work[static_cast<size_t>(dest) * cap + base] = value;
}

// Stats frames: E_t = the sum of the per-(tile, chunk) deepest entries.
__global__ void emax_sum_kernel(const uint32_t* __restrict__ emax, uint32_t n, Counters* __restrict__ ctr) {
    unsigned long long s = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += emax[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(&ctr->block_entries, s);
}

}  // namespace

int composite_pixel_chunks(int ts) {
    const long long tile_px = static_cast<long long>(ts) * ts;
    return static_cast<int>((tile_px + kChunkPx - 1) / kChunkPx);
}

int composite_work_items(int ts) { return kSubsPerChunk * composite_pixel_chunks(ts); }

namespace {
template <int G, int M, bool ROW>
cudaError_t launch_k7(const FrameConsts* fc, const CamParams& cam, const CfgParams& cfg, int nchunks,
                      const uint2* ranges, const uint32_t* keys, const SplatRec* rec,
                      const float4* colour, float3 bg, PixelState* state, uint32_t* processed, const TileFlags& flags,
                      bool first, bool last, Counters* counters, bool want_stats, uint32_t* emax, uint32_t* work,
                      uint32_t* wctl, uint32_t cap, cudaStream_t stream) {
    constexpr size_t smem = (kThreads / 32) * sizeof(WarpStage);
    static const cudaError_t attr = cudaFuncSetAttribute(composite_kernel<G, M, ROW>,
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         static_cast<int>(smem));
    if (attr != cudaSuccess) return attr;
    // persistent grid: M resident CTAs of four warps per SM
    composite_kernel<G, M, ROW><<<148u * M, kThreads, smem, stream>>>(
        fc, cam.W, cam.H, cfg, nchunks, ranges, keys, rec, colour, bg, state, processed, flags,
        first ? 1 : 0, last ? 1 : 0, counters, want_stats ? 1 : 0, emax, work, wctl, wctl + 6, cap);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_composite(const FrameConsts* fc, const CamParams& cam, const CfgParams& cfg,
                             const uint2* ranges, const uint32_t* keys, const SplatRec* rec,
                             const float4* colour, float3 bg, PixelState* state, uint32_t* processed,
                             uint32_t* tile_flags, bool first, bool last, Counters* counters, bool want_stats,
                             uint32_t* tile_emax, uint32_t* work, uint32_t* wctl, cudaStream_t stream) {
    const int nchunks = composite_pixel_chunks(cfg.tile_size);
    const uint32_t ntile = static_cast<uint32_t>(cfg.tiles_x) * static_cast<uint32_t>(cfg.tiles_y);
    const uint32_t cap = ntile * static_cast<uint32_t>(composite_work_items(cfg.tile_size));
    const uint32_t words = (ntile + 31) / 32;
    const uint32_t part_words = (4 * ntile + 31) / 32;
    const TileFlags flags{tile_flags, tile_flags + words, tile_flags + words + part_words};
    cudaError_t e = cudaMemsetAsync(wctl, 0, kWorkCtl * sizeof(uint32_t), stream);
    if (e != cudaSuccess) return e;
    if (want_stats && first) {
        e = cudaMemsetAsync(tile_emax, 0, static_cast<size_t>(ntile) * nchunks * sizeof(uint32_t), stream);
        if (e != cudaSuccess) return e;
    }
    build_work_kernel<<<(cap + 255) / 256, 256, 0, stream>>>(ranges, flags, first ? 1 : 0, last ? 1 : 0, ntile,
                                                             nchunks, cfg.tile_size * cfg.tile_size, cap, work, wctl);
    if (cfg.tile_size == 16)
        e = launch_k7<4, 4, true>(fc, cam, cfg, nchunks, ranges, keys, rec, colour, bg, state, processed,
                                  flags, first, last, counters, want_stats, tile_emax, work, wctl, cap, stream);
    else
        e = launch_k7<4, 4, false>(fc, cam, cfg, nchunks, ranges, keys, rec, colour, bg, state, processed,
                                   flags, first, last, counters, want_stats, tile_emax, work, wctl, cap, stream);
    if (e != cudaSuccess) return e;
    if (want_stats && last)
        emax_sum_kernel<<<64, 256, 0, stream>>>(tile_emax, ntile * static_cast<uint32_t>(nchunks), counters);
    return cudaGetLastError();
}

// words of the per-tile flag block launch_composite reads (done | touched | part-done)
size_t composite_flag_words(uint32_t ntile) { return (ntile + 31) / 32 + 2 * ((4 * static_cast<size_t>(ntile) + 31) / 32); }

}  // namespace sgs
