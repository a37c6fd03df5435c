// depth_sort.cu -- K2: the global blending order (depth, index) of raster.cpp:93-101.
//
// A 64-bit key radix sort costs eight passes over (key, index). The frame's depth
// range is narrow, so the sort runs on 32-bit keys instead: the 64-bit orderable
// depth key minus the frame minimum, shifted right just enough to fit 31 bits
// (never a float32 cast, which would tie a quarter of the splats). That is four
// passes. Keys that collide after the shift form short runs (expected a few
// thousand pairs at 3M splats); K2b re-sorts each run by (full 64-bit key, index),
// which restores the reference's order exactly. Runs longer than kMaxRun are
// reported and the host falls back to the 64-bit sort.
#include "sgs_internal.h"

namespace sgs {
namespace {

constexpr int kMaxRun = 64;

__global__ void make_key32_kernel(uint64_t n, const unsigned long long* __restrict__ key64,
                                  const Counters* __restrict__ ctr, uint32_t* __restrict__ key32) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long kmin = ctr->kmin, kmax = ctr->kmax;
    const unsigned long long range = kmax >= kmin ? kmax - kmin : 0ULL;
    const int bits = range ? 64 - __clzll(static_cast<long long>(range)) : 0;
    const int shift = bits > 31 ? bits - 31 : 0;
    const unsigned long long k = key64[i];
    key32[i] = k == ~0ULL ? 0xFFFFFFFFu : static_cast<uint32_t>((k - kmin) >> shift);
}

// One thread per run head; insertion sort by (key64, index) inside the run.
__global__ void fix_ties_kernel(uint64_t n, const uint32_t* __restrict__ key32,
                                const unsigned long long* __restrict__ key64,
                                uint32_t* __restrict__ order, Counters* __restrict__ ctr) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i + 1 >= n) return;
    const uint32_t k = key32[i];
    if (k == 0xFFFFFFFFu || key32[i + 1] != k) return;
    if (i > 0 && key32[i - 1] == k) return;  // not the head of the run
    uint64_t e = i + 2;
    while (e < n && key32[e] == k && e - i <= kMaxRun) ++e;
    if (e - i > kMaxRun) {
        atomicAdd(&ctr->tie_overflow, 1ULL);
        return;
    }
    const int len = static_cast<int>(e - i);
    uint32_t idx[kMaxRun];
    unsigned long long kk[kMaxRun];
    for (int a = 0; a < len; ++a) {
        idx[a] = order[i + a];
        kk[a] = key64[idx[a]];
    }
    for (int a = 1; a < len; ++a) {
        const uint32_t vi = idx[a];
        const unsigned long long vk = kk[a];
        int b = a - 1;
        while (b >= 0 && (kk[b] > vk || (kk[b] == vk && idx[b] > vi))) {
            idx[b + 1] = idx[b];
            kk[b + 1] = kk[b];
            --b;
        }
        idx[b + 1] = vi;
        kk[b + 1] = vk;
    }
    for (int a = 0; a < len; ++a) order[i + a] = idx[a];
    atomicAdd(&ctr->tie_runs, 1ULL);
}

}  // namespace

void launch_make_key32(uint64_t n, const unsigned long long* key64, const Counters* ctr,
                       uint32_t* key32, cudaStream_t stream) {
    if (n == 0) return;
    make_key32_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(n, key64, ctr, key32);
}

void launch_fix_ties(uint64_t n, const uint32_t* key32, const unsigned long long* key64,
                     uint32_t* order, Counters* ctr, cudaStream_t stream) {
    if (n < 2) return;
    fix_ties_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(n, key32, key64, order, ctr);
}

}  // namespace sgs
