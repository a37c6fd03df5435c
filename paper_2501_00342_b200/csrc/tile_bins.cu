// tile_bins.cu -- tile-major binning of a depth chunk (optional: SGS_BIN=tile).
//
// Replaces build_tile_grid (proj/src/raster.cpp:108-130) for the compositor. The
// reference pushes each splat's rank into every tile of its inclusive rectangle in
// blending order, so a tile's list is the ranks covering it, ascending. For the
// ranks [rb, re) of one depth chunk:
//   B1  tb_pairs<count>   one red.add per live (rank, tile) pair into cnt[tile]
//   B2  tb_scan           one CTA: exclusive scan over tiles -> ranges[tile] and
//                         the scatter cursors; the compositor's work list (long
//                         lists first) and the sort work list; P, overflow flags
//   B3  tb_pairs<scatter> list[cursor[tile]++] = rank (order inside a tile is the
//                         order the atomics land in, so:)
//   B4  tb_sort           per tile, sort the ranks in shared memory (warp bitonic
//                         for <= 64 entries, a stable 4-bit LSD block radix sort up
//                         to kSortCap) and write the Gaussian indices order[rank]
// Each tile's list then equals the reference's TileGrid list restricted to the chunk
// (ranks are unique, so the sorted list is exactly the ascending one). A list longer
// than kSortCap raises list_overflow and the host redoes the frame with the
// rank-major path (binning.cu + tile_sort.cu), which has no per-tile limit.
// Compared with that path: 4 launches per chunk instead of 9, 4-B list entries, one
// shared-memory sort per tile instead of two device-wide radix passes. Measured on
// the B200 at config C it is nevertheless slower (per chunk: pairs 32 + scan 21 +
// scatter 63 + sort 54 us, against 100 us for the rank-major path; 0.79 vs 0.72
// ms/frame in the 4-lane batch): the global atomics of the aggregated count and
// scatter run at ~15 G/s whatever their address spread, and mid-sized lists leave
// most of a sorting unit idle. It stays as a tested alternative (bitwise equal).
#include <algorithm>

#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kPairThreads = 512;
constexpr int kSmemTiles = 12288;  // tile grids up to this size aggregate pairs in shared memory
constexpr int kScanThreads = 1024;
constexpr int kSortThreads = 1024;
constexpr int kSortPer = 16;                        // keys per thread in the radix sorts
constexpr int kSortCap = kSortThreads * kSortPer;   // 16384 entries per tile list
constexpr int kGroupThreads = 256;                  // mid lists: 4 groups of 8 warps per CTA
constexpr int kBitonicCap = 64;
constexpr int kMaxBitmapTiles = 1 << 18;
constexpr uint32_t kLongList = 1024;  // compositor: lists this long are scheduled first
constexpr uint32_t kWorkCtlWords = 8;  // composite.cu kWorkCtl: background items follow the control words
// sort classes: 0 warp bitonic (<= 64), 1 warp radix (<= 512), 2 group radix
// (<= 4096), 3 CTA radix (<= kSortCap)
constexpr uint32_t kClassCap[4] = {kBitonicCap, 32 * kSortPer, kGroupThreads * kSortPer, kSortCap};

// padded shared-memory index (one spare word per 32: conflict-free blocked access)
__host__ __device__ constexpr int pad(int e) { return e + (e >> 5); }

struct DoneBits {
    const uint32_t* bits;  // null: no tile finished yet
    __device__ __forceinline__ bool operator()(uint32_t t) const {
        return bits && ((bits[t >> 5] >> (t & 31)) & 1u);
    }
};

// Visit the live tiles of the ranks [r0, r1) owned by this thread (stride: CTA
// size). Rectangles above 32 tiles are walked by the whole warp (one lane per tile)
// so a large splat does not serialise one lane.
template <typename F>
__device__ __forceinline__ void for_pairs(uint64_t r0, uint64_t r1, const uint2* __restrict__ bmeta,
                                          const int4* __restrict__ brect, const DoneBits& done, int tiles_x,
                                          F&& f) {
    const unsigned lane = threadIdx.x & 31;
    for (uint64_t rw = r0 + (threadIdx.x & ~31u); rw < r1; rw += blockDim.x) {
        const uint64_t r = rw + lane;
        uint32_t area = 0;
        int4 rc = make_int4(0, -1, 0, -1);
        if (r < r1) {
            area = bmeta[r].y;
            if (area) rc = brect[r];
        }
        if (area && area <= 32) {
            for (int ty = rc.z; ty <= rc.w; ++ty)
                for (int tx = rc.x; tx <= rc.y; ++tx) {
                    const uint32_t tile = static_cast<uint32_t>(ty * tiles_x + tx);
                    if (!done(tile)) f(tile, static_cast<uint32_t>(r));
                }
        }
        unsigned big = __ballot_sync(0xffffffffu, area > 32);
        while (big) {
            const int src = __ffs(big) - 1;
            big &= big - 1;
            const uint32_t a = __shfl_sync(0xffffffffu, area, src);
            const uint32_t rr = __shfl_sync(0xffffffffu, static_cast<uint32_t>(r), src);
            const int x0 = __shfl_sync(0xffffffffu, rc.x, src);
            const int y0 = __shfl_sync(0xffffffffu, rc.z, src);
            const uint32_t ww = static_cast<uint32_t>(__shfl_sync(0xffffffffu, rc.y, src) - x0 + 1);
            for (uint32_t j = lane; j < a; j += 32) {
                const uint32_t tile = static_cast<uint32_t>(y0 + static_cast<int>(j / ww)) * tiles_x +
                                      static_cast<uint32_t>(x0 + static_cast<int>(j % ww));
                if (!done(tile)) f(tile, rr);
            }
        }
    }
}

__device__ __forceinline__ DoneBits load_done(const uint32_t* done_g, int ntile, uint32_t* s_done) {
    DoneBits done{done_g};
    if (done_g && ntile <= kMaxBitmapTiles) {
        for (int w = threadIdx.x; w < (ntile + 31) / 32; w += blockDim.x) s_done[w] = done_g[w];
        done.bits = s_done;
    }
    return done;
}

// B1 / B3. Each CTA takes a block of consecutive ranks and aggregates its pairs per
// tile in shared memory, so a tile receives one global atomic per CTA, not one per
// pair (hot tiles would serialise on their counter). The scatter reserves each
// tile's block of slots with one atomic and places its pairs behind it.
template <bool kScatter>
__global__ void __launch_bounds__(kPairThreads) tb_pairs_kernel(
    uint64_t rb, uint64_t re, uint32_t ranks_per_cta, const uint2* __restrict__ bmeta,
    const int4* __restrict__ brect, const uint32_t* __restrict__ done_g, int tiles_x, int ntile,
    uint32_t* __restrict__ ctr_tile, uint32_t* __restrict__ list, uint64_t capacity) {
    extern __shared__ uint32_t smem[];
    uint32_t* s_done = smem;
    const int bm_words = (ntile + 31) / 32;
    const uint64_t r0 = rb + static_cast<uint64_t>(blockIdx.x) * ranks_per_cta;
    const uint64_t r1 = r0 + ranks_per_cta < re ? r0 + ranks_per_cta : re;
    const DoneBits done = load_done(done_g, ntile, s_done);
    if (ntile > kSmemTiles) {  // large grids: direct atomics
        __syncthreads();
        for_pairs(r0, r1, bmeta, brect, done, tiles_x, [&](uint32_t tile, uint32_t r) {
            if (kScatter) {
                const uint32_t pos = atomicAdd(&ctr_tile[tile], 1u);
                if (pos < capacity) list[pos] = r;
            } else {
                atomicAdd(&ctr_tile[tile], 1u);
            }
        });
        return;
    }
    uint32_t* s_cnt = smem + bm_words;
    uint32_t* s_base = s_cnt + ntile;
    for (int t = threadIdx.x; t < ntile; t += blockDim.x) s_cnt[t] = 0;
    __syncthreads();
    for_pairs(r0, r1, bmeta, brect, done, tiles_x, [&](uint32_t tile, uint32_t) { atomicAdd(&s_cnt[tile], 1u); });
    __syncthreads();
    for (int t = threadIdx.x; t < ntile; t += blockDim.x) {
        const uint32_t c = s_cnt[t];
        if (!c) continue;
        if (kScatter) {
            s_base[t] = atomicAdd(&ctr_tile[t], c);
            s_cnt[t] = 0;
        } else {
            atomicAdd(&ctr_tile[t], c);
        }
    }
    if (!kScatter) return;
    __syncthreads();
    for_pairs(r0, r1, bmeta, brect, done, tiles_x, [&](uint32_t tile, uint32_t r) {
        const uint32_t pos = s_base[tile] + atomicAdd(&s_cnt[tile], 1u);
        if (pos < capacity) list[pos] = r;
    });
}

// Block-wide exclusive scan of one value per thread; returns the exclusive prefix
// and the block total (through *total). Ends synchronised.
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const uint32_t x = lane < nw ? s_warp[lane] : 0u;
        uint32_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        if (lane < nw) s_warp[lane] = xi - x;
        if (lane == 31) s_warp[32] = xi;
    }
    __syncthreads();
    const uint32_t ex = s_warp[warp] + inc - v;
    *total = s_warp[32];
    __syncthreads();
    return ex;
}

// Warp-aggregated append to one of the shared list counters: returns the slot.
__device__ __forceinline__ uint32_t warp_append(bool take, uint32_t* s_count) {
    const unsigned lane = threadIdx.x & 31;
    const unsigned m = __ballot_sync(0xffffffffu, take);
    uint32_t base = 0;
    const int leader = m ? __ffs(m) - 1 : 0;
    if (m && lane == static_cast<unsigned>(leader)) base = atomicAdd(s_count, static_cast<uint32_t>(__popc(m)));
    base = __shfl_sync(0xffffffffu, base, leader);
    return base + __popc(m & ((1u << lane) - 1u));
}

// B2. cnt holds the chunk's per-tile counts (zeroed here for the next chunk).
// wctl (composite.cu's work layout): [2] long items (class 2), [5] short items (class 5),
// [6] the compositor's cursor, [7] background items.
// sctl: [k] sort items of class k, [4 + k] their cursor.
__global__ void __launch_bounds__(kScanThreads) tb_scan_kernel(
    int ntile, int pchunks, uint32_t* __restrict__ cnt, uint32_t* __restrict__ cur, uint2* __restrict__ ranges,
    const uint32_t* __restrict__ done_g, const uint32_t* __restrict__ touched_g, int first, int last,
    uint64_t capacity, Counters* __restrict__ ctr, uint32_t* __restrict__ work, uint32_t work_cap,
    uint32_t* __restrict__ wctl, uint32_t* __restrict__ sitems, uint32_t* __restrict__ sctl) {
    __shared__ uint32_t s_warp[33];
    __shared__ uint32_t s_n[7];  // long, short work items; sort items per class; background items
    __shared__ uint32_t s_over;
    if (threadIdx.x < 7) s_n[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_over = 0;
    __syncthreads();
    uint64_t carry = 0;
    const DoneBits done{first ? nullptr : done_g};
    for (int base = 0; base < ntile; base += kScanThreads) {
        const int t = base + threadIdx.x;
        const uint32_t len = t < ntile ? cnt[t] : 0u;
        uint32_t tot;
        const uint32_t ex = block_scan(len, s_warp, &tot);
        if (t < ntile) {
            const uint64_t off = carry + ex;
            const uint32_t o32 = static_cast<uint32_t>(off < capacity ? off : capacity);
            const uint32_t e32 = static_cast<uint32_t>(off + len < capacity ? off + len : capacity);
            ranges[t] = make_uint2(o32, e32);
            cur[t] = o32;
            cnt[t] = 0;
            if (len > static_cast<uint32_t>(kSortCap)) s_over = 1;
        }
        carry += tot;
        // sort items: every non-empty list (its ranks become Gaussian indices), by
        // size class; class k's items at sitems[k * ntile ...]
        const bool has = t < ntile && len > 0;
        const int cls = len <= kClassCap[0] ? 0 : len <= kClassCap[1] ? 1 : len <= kClassCap[2] ? 2 : 3;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t slot = warp_append(has && cls == k, &s_n[2 + k]);
            if (has && cls == k) sitems[static_cast<uint32_t>(k) * ntile + slot] = static_cast<uint32_t>(t);
        }
        // compositor work items (build_work_kernel's rules)
        const bool live = t < ntile && (first || !done(static_cast<uint32_t>(t))) && (last || len > 0);
        // a tile that never received an entry only writes background (K7's tail loop)
        const bool bgt = live && len == 0 &&
                         (first || !((touched_g[static_cast<uint32_t>(t) >> 5] >> (t & 31)) & 1u));
        for (int c = 0; c < pchunks; ++c) {
            const uint32_t item = static_cast<uint32_t>(t) * pchunks + c;
            const bool lng = live && !bgt && len >= kLongList;
            const uint32_t pl = warp_append(lng, &s_n[0]);
            const uint32_t ps = warp_append(live && !bgt && !lng, &s_n[1]);
            const uint32_t pb = warp_append(bgt, &s_n[6]);
            if (lng) work[2 * work_cap + pl] = item;  // composite.cu work classes: 2 (>= 1024) and 5
            else if (bgt) wctl[kWorkCtlWords + pb] = item;
            else if (live) work[5 * work_cap + ps] = item;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int c = 0; c < 6; ++c) wctl[c] = 0;
        wctl[2] = s_n[0];
        wctl[5] = s_n[1];
        wctl[6] = 0;
        wctl[7] = s_n[6];
        for (int k = 0; k < 4; ++k) {
            sctl[k] = s_n[2 + k];
            sctl[4 + k] = 0;
        }
        const unsigned long long p = carry;
        ctr->tile_entries += p;
        if (p > ctr->max_chunk_entries) ctr->max_chunk_entries = p;
        if (p > capacity) ctr->key_overflow = 1;
        ctr->chunk_entries = p < capacity ? p : capacity;
        if (s_over) ctr->list_overflow = 1;
    }
}

// Warp: sort up to 64 unique ranks (bitonic in registers, element e in lane e & 31,
// half e >> 5) and write order[rank].
__device__ void warp_bitonic_list(uint32_t* __restrict__ list, uint32_t s, uint32_t L,
                                  const uint32_t* __restrict__ order) {
    const int lane = threadIdx.x & 31;
    uint32_t k0 = static_cast<uint32_t>(lane) < L ? list[s + lane] : 0xFFFFFFFFu;
    uint32_t k1 = static_cast<uint32_t>(lane) + 32 < L ? list[s + 32 + lane] : 0xFFFFFFFFu;
    if (L > 1) {
#pragma unroll
        for (int kk = 2; kk <= 64; kk <<= 1) {
#pragma unroll
            for (int j = kk >> 1; j > 0; j >>= 1) {
                if (j == 32) {
                    // pair (lane, lane + 32) in one lane; kk == 64: ascending
                    const uint32_t lo = min(k0, k1), hi = max(k0, k1);
                    k0 = lo;
                    k1 = hi;
                } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t& k = h ? k1 : k0;
                        const int el = h * 32 + lane;
                        const uint32_t p = __shfl_xor_sync(0xffffffffu, k, j);
                        const bool lower = (el & j) == 0;
                        const bool up = (el & kk) == 0;
                        // the lower element of an ascending pair keeps the min
                        k = lower == up ? min(k, p) : max(k, p);
                    }
                }
            }
        }
    }
    if (static_cast<uint32_t>(lane) < L) list[s + lane] = order[k0];
    if (static_cast<uint32_t>(lane) + 32 < L) list[s + 32 + lane] = order[k1];
}

// A sorting unit of GT contiguous threads (a warp, 8 warps, or the whole CTA) with
// its own barrier: warps sync with __syncwarp, groups of 8 warps with named barrier
// 1 + group, the CTA with __syncthreads.
template <int GT>
struct Unit {
    int id;  // unit index within the CTA
    __device__ __forceinline__ void sync() const {
        if constexpr (GT == 32)
            __syncwarp();
        else if constexpr (GT == kSortThreads)
            __syncthreads();
        else
            asm volatile("bar.sync %0, %1;" ::"r"(id + 1), "r"(GT) : "memory");
    }
    __device__ __forceinline__ int tid() const { return static_cast<int>(threadIdx.x) % GT; }
};

// Exclusive scan of one value per unit thread; red needs GT / 32 + 1 words.
template <int GT>
__device__ __forceinline__ uint32_t unit_scan(const Unit<GT>& u, uint32_t v, uint32_t* red) {
    const int t = u.tid(), lane = t & 31, warp = t >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if constexpr (GT == 32) {
        return inc - v;
    } else {
        constexpr int nw = GT / 32;
        if (lane == 31) red[warp] = inc;
        u.sync();
        if (warp == 0) {
            const uint32_t x = lane < nw ? red[lane] : 0u;
            uint32_t xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
            }
            if (lane < nw) red[lane] = xi - x;
        }
        u.sync();
        const uint32_t ex = red[warp] + inc - v;
        u.sync();
        return ex;
    }
}

template <int GT>
__device__ __forceinline__ void unit_minmax(const Unit<GT>& u, uint32_t& lo, uint32_t& hi, uint32_t* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if constexpr (GT > 32) {
        constexpr int nw = GT / 32;
        const int t = u.tid(), lane = t & 31, warp = t >> 5;
        if (lane == 0) {
            red[warp] = lo;
            red[32 + warp] = hi;
        }
        u.sync();
        lo = 0xFFFFFFFFu;
        hi = 0;
        for (int w = 0; w < nw; ++w) {
            lo = min(lo, red[w]);
            hi = max(hi, red[32 + w]);
        }
        u.sync();
    }
}

// Unit: stable LSD radix sort (4-bit digits) of L <= 16 GT unique ranks in shared
// memory, then list[s + e] = order[rank_e]. Thread t of the first T holds the
// blocked positions [16t, 16t + 16); per-(digit, thread) counters scanned in
// digit-major order give every key its stable destination. Keys are rebased to the
// list's minimum so only the bits of its span are sorted.
template <int GT>
__device__ void unit_radix_list(const Unit<GT>& u, uint32_t* __restrict__ list, uint32_t s, uint32_t L,
                                const uint32_t* __restrict__ order, uint32_t* sk, uint32_t* sc, uint32_t* red) {
    const int tid = u.tid();
    const int T = ((static_cast<int>((L + kSortPer - 1) / kSortPer) + 31) / 32) * 32;
    const bool act = tid < T;
    uint32_t k[kSortPer];
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
#pragma unroll
    for (int j = 0; j < kSortPer; ++j) {
        const uint32_t e = static_cast<uint32_t>(tid * kSortPer + j);
        k[j] = (act && e < L) ? list[s + e] : 0xFFFFFFFFu;
        if (act && e < L) {
            lo = min(lo, k[j]);
            hi = max(hi, k[j]);
        }
    }
    unit_minmax(u, lo, hi, red);
    const uint32_t kmin = lo, span = hi - lo;
    const int bits = span ? 32 - __clz(static_cast<int>(span)) : 1;
#pragma unroll
    for (int j = 0; j < kSortPer; ++j)
        if (k[j] != 0xFFFFFFFFu) k[j] -= kmin;
    for (int sh = 0; sh < bits; sh += 4) {
        // per-key position among the thread's keys of the same digit (< 16): nibbles
        uint32_t loc[kSortPer / 8] = {};
        if (act) {
#pragma unroll
            for (int d = 0; d < 16; ++d) sc[pad(d * T + tid)] = 0;
#pragma unroll
            for (int j = 0; j < kSortPer; ++j) {
                const int c = pad(static_cast<int>((k[j] >> sh) & 15u) * T + tid);
                const uint32_t x = sc[c];
                loc[j >> 3] |= x << (4 * (j & 7));
                sc[c] = x + 1;
            }
        }
        u.sync();
        // exclusive scan of the 16T counters, linear index d * T + t: thread t
        // takes the 16 consecutive entries [16t, 16t + 16)
        uint32_t sum = 0;
        if (act) {
#pragma unroll
            for (int i = 0; i < 16; ++i) sum += sc[pad(tid * 16 + i)];
        }
        uint32_t run = unit_scan(u, act ? sum : 0u, red);
        if (act) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const uint32_t x = sc[pad(tid * 16 + i)];
                sc[pad(tid * 16 + i)] = run;
                run += x;
            }
        }
        u.sync();
        if (act) {
#pragma unroll
            for (int j = 0; j < kSortPer; ++j) {
                const int c = pad(static_cast<int>((k[j] >> sh) & 15u) * T + tid);
                sk[pad(static_cast<int>(sc[c] + ((loc[j >> 3] >> (4 * (j & 7))) & 15u)))] = k[j];
            }
        }
        u.sync();
        if (act) {
#pragma unroll
            for (int j = 0; j < kSortPer; ++j) k[j] = sk[pad(tid * kSortPer + j)];
        }
        u.sync();
    }
    if (act) {
#pragma unroll
        for (int j = 0; j < kSortPer; ++j) {
            const uint32_t e = static_cast<uint32_t>(tid * kSortPer + j);
            if (e < L) list[s + e] = order[k[j] + kmin];
        }
    }
}

// Units of GT threads pull items of one class until it is exhausted.
template <int GT>
__device__ __forceinline__ void sort_class(int cls, int ntile, const uint2* __restrict__ ranges,
                                           uint32_t* __restrict__ list, const uint32_t* __restrict__ order,
                                           const uint32_t* __restrict__ sitems, uint32_t* __restrict__ sctl,
                                           uint32_t* smem, uint32_t* s_item, uint32_t* s_red) {
    const Unit<GT> u{static_cast<int>(threadIdx.x) / GT};
    constexpr int kKeys = pad(GT * kSortPer), kCnt = pad(16 * GT);
    uint32_t* sk = smem + u.id * (kKeys + kCnt);
    uint32_t* sc = sk + kKeys;
    uint32_t* red = s_red + u.id * 66;
    const uint32_t n = sctl[cls];
    for (;;) {
        uint32_t it;
        if constexpr (GT == 32) {
            it = 0;
            if ((threadIdx.x & 31) == 0) it = atomicAdd(&sctl[4 + cls], 1u);
            it = __shfl_sync(0xffffffffu, it, 0);
        } else {
            if (u.tid() == 0) s_item[u.id] = atomicAdd(&sctl[4 + cls], 1u);
            u.sync();
            it = s_item[u.id];
            u.sync();
        }
        if (it >= n) break;
        const uint2 rg = ranges[sitems[static_cast<uint32_t>(cls) * ntile + it]];
        const uint32_t L = rg.y - rg.x;
        if (cls == 0)
            warp_bitonic_list(list, rg.x, L, order);
        else if (L <= static_cast<uint32_t>(GT * kSortPer))  // (class 3 above kSortCap: overflow, skipped)
            unit_radix_list(u, list, rg.x, L, order, sk, sc, red);
        u.sync();
    }
}

// B4: persistent CTAs; the largest lists first (one CTA each), then 8-warp groups,
// then single warps (radix, bitonic).
__global__ void __launch_bounds__(kSortThreads, 1) tb_sort_kernel(
    int ntile, const uint2* __restrict__ ranges, uint32_t* __restrict__ list, const uint32_t* __restrict__ order,
    const uint32_t* __restrict__ sitems, uint32_t* __restrict__ sctl) {
    extern __shared__ uint32_t smem[];
    __shared__ uint32_t s_red[32 * 66];
    __shared__ uint32_t s_item[32];
    sort_class<kSortThreads>(3, ntile, ranges, list, order, sitems, sctl, smem, s_item, s_red);
    sort_class<kGroupThreads>(2, ntile, ranges, list, order, sitems, sctl, smem, s_item, s_red);
    sort_class<32>(1, ntile, ranges, list, order, sitems, sctl, smem, s_item, s_red);
    sort_class<32>(0, ntile, ranges, list, order, sitems, sctl, smem, s_item, s_red);
}

}  // namespace

size_t tb_sort_smem_bytes() { return static_cast<size_t>(pad(kSortCap) + pad(16 * kSortThreads)) * 4; }

void launch_tile_bins(uint64_t rb, uint64_t re, const uint2* bmeta, const int4* brect, const uint32_t* done,
                      const uint32_t* touched, int tiles_x, int ntile, int pchunks, bool first, bool last, const uint32_t* order,
                      uint32_t* cnt, uint32_t* cur, uint2* ranges, uint32_t* list, uint64_t capacity,
                      uint32_t* work, uint32_t work_cap, uint32_t* wctl, uint32_t* sitems, uint32_t* sctl,
                      Counters* ctr, cudaStream_t stream) {
    const uint64_t n = re > rb ? re - rb : 0;
    // ranks per CTA: about two waves of CTAs, 1..16 ranks per thread
    uint64_t per = (n + 2 * 148 - 1) / (2 * 148);
    per = std::min<uint64_t>(std::max<uint64_t>(per, kPairThreads), 16 * kPairThreads);
    per = (per + 31) / 32 * 32;
    const unsigned grid = static_cast<unsigned>(n ? (n + per - 1) / per : 1);
    // (the bitmap slot is reserved even without finished tiles: the counters follow it)
    const size_t bm = ntile <= kMaxBitmapTiles ? static_cast<size_t>((ntile + 31) / 32) * 4 : 0;
    const size_t agg = ntile <= kSmemTiles ? static_cast<size_t>(ntile) * 4 : 0;
    static const bool attr = [] {
        cudaFuncSetAttribute(tb_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(tb_sort_smem_bytes()));
        cudaFuncSetAttribute(tb_pairs_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemTiles * 8 + kMaxBitmapTiles / 8));
        cudaFuncSetAttribute(tb_pairs_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemTiles * 4 + kMaxBitmapTiles / 8));
        return true;
    }();
    (void)attr;
    tb_pairs_kernel<false><<<grid, kPairThreads, bm + agg, stream>>>(rb, re, static_cast<uint32_t>(per), bmeta,
                                                                      brect, done, tiles_x, ntile, cnt, list, capacity);
    tb_scan_kernel<<<1, kScanThreads, 0, stream>>>(ntile, pchunks, cnt, cur, ranges, done, touched,
                                                   first ? 1 : 0, last ? 1 : 0, capacity, ctr, work, work_cap, wctl, sitems, sctl);
    tb_pairs_kernel<true><<<grid, kPairThreads, bm + 2 * agg, stream>>>(rb, re, static_cast<uint32_t>(per), bmeta,
                                                                         brect, done, tiles_x, ntile, cur, list,
                                                                         capacity);
    tb_sort_kernel<<<148, kSortThreads, tb_sort_smem_bytes(), stream>>>(ntile, ranges, list, order, sitems, sctl);
}

}  // namespace sgs
