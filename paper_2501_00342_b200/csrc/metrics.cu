// metrics.cu -- GPU PSNR / SSIM / SSIM gradient, the step
// after render in evaluation and training (metrics.hpp, proj/src/metrics.cpp).
//
// Every per-pixel quantity is FP64 in the reference's exact operation order
// (__dmul_rn / __dadd_rn / __ddiv_rn, no FMA contraction), so the blurred moments,
// the SSIM map and the gradient image match the reference bit for bit:
//   * the separable 11-tap Gaussian blur (blur, metrics.cpp:40-60) accumulates the
//     taps left to right, rows then columns, with the reference's reflect();
//   * its adjoint (blur_adjoint, :63-85) is a scatter in the reference; here every
//     output gathers its contributions in the order the scatter visits them
//     (source row / column ascending, then tap ascending), which is the same sum;
//   * the taps are computed on the host with the same libm exp as the reference.
// Only the two image-wide means differ in summation order (a fixed-shape tree,
// deterministic run to run, instead of one serial loop): relative 1e-15-level.
#include <cmath>

#include "projection.cuh"

namespace sgs {
namespace {

constexpr int kWin = 11;
constexpr int kRad = kWin / 2;
constexpr double kC1 = 0.01 * 0.01;
constexpr double kC2 = 0.03 * 0.03;
constexpr int kRedBlocks = 1024;
constexpr int kRedThreads = 256;

__constant__ double c_taps[kWin];

__device__ __forceinline__ int reflect_i(int i, int n) {
    while (i < 0 || i >= n) {
        if (i < 0) i = -i - 1;
        if (i >= n) i = 2 * n - 1 - i;
    }
    return i;
}

template <typename T>
__device__ __forceinline__ double ld(const T* p, size_t i) {
    return static_cast<double>(p[i]);
}

// blur rows of the five moment images a, b, a*a, b*b, a*b (metrics.cpp:104-108)
template <typename T>
__global__ void ssim_rows_kernel(const T* __restrict__ a, const T* __restrict__ b, int W, int H, int C,
                                 double* __restrict__ tmp) {
    const size_t n = static_cast<size_t>(W) * H * C;
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = static_cast<int>(i % C);
    const size_t p = i / C;
    const int x = static_cast<int>(p % W), y = static_cast<int>(p / W);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
#pragma unroll
    for (int k = -kRad; k <= kRad; ++k) {
        const size_t j = (static_cast<size_t>(y) * W + reflect_i(x + k, W)) * C + c;
        const double va = ld(a, j), vb = ld(b, j), w = c_taps[k + kRad];
        s0 = dadd(s0, dmul(w, va));
        s1 = dadd(s1, dmul(w, vb));
        s2 = dadd(s2, dmul(w, dmul(va, va)));
        s3 = dadd(s3, dmul(w, dmul(vb, vb)));
        s4 = dadd(s4, dmul(w, dmul(va, vb)));
    }
    tmp[i] = s0;
    tmp[n + i] = s1;
    tmp[2 * n + i] = s2;
    tmp[3 * n + i] = s3;
    tmp[4 * n + i] = s4;
}

// blur columns, then the SSIM map and (optionally) the three upstream gradient maps
// of ssim_impl (metrics.cpp:126-147)
__global__ void ssim_cols_kernel(const double* __restrict__ tmp, int W, int H, int C, double upstream,
                                 double* __restrict__ smap, double* __restrict__ g) {
    const size_t n = static_cast<size_t>(W) * H * C;
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = static_cast<int>(i % C);
    const size_t p = i / C;
    const int x = static_cast<int>(p % W), y = static_cast<int>(p / W);
    double m[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = -kRad; k <= kRad; ++k) {
        const size_t j = (static_cast<size_t>(reflect_i(y + k, H)) * W + x) * C + c;
        const double w = c_taps[k + kRad];
#pragma unroll
        for (int q = 0; q < 5; ++q) m[q] = dadd(m[q], dmul(w, tmp[q * n + j]));
    }
    const double ma = m[0], mb = m[1];
    const double va = dsub(m[2], dmul(ma, ma));
    const double vb = dsub(m[3], dmul(mb, mb));
    const double cov = dsub(m[4], dmul(ma, mb));
    const double a1 = dadd(dmul(dmul(2.0, ma), mb), kC1);
    const double a2 = dadd(dmul(2.0, cov), kC2);
    const double b1 = dadd(dadd(dmul(ma, ma), dmul(mb, mb)), kC1);
    const double b2 = dadd(dadd(va, vb), kC2);
    const double s = ddiv(dmul(a1, a2), dmul(b1, b2));
    smap[i] = s;
    if (g) {
        const double g_a1 = ddiv(dmul(upstream, a2), dmul(b1, b2));
        const double g_a2 = ddiv(dmul(upstream, a1), dmul(b1, b2));
        const double g_b1 = ddiv(dmul(-upstream, s), b1);
        const double g_b2 = ddiv(dmul(-upstream, s), b2);
        const double g_cov = dmul(2.0, g_a2);
        const double g_va = g_b2;
        // 2 mb g_a1 + 2 ma g_b1 - 2 ma g_va - mb g_cov, left to right
        const double t = dsub(dsub(dadd(dmul(dmul(2.0, mb), g_a1), dmul(dmul(2.0, ma), g_b1)),
                                   dmul(dmul(2.0, ma), g_va)),
                              dmul(mb, g_cov));
        g[i] = t;
        g[n + i] = g_va;
        g[2 * n + i] = g_cov;
    }
}

// blur_adjoint, column stage (metrics.cpp:67-74) as a gather: out(y', x) sums
// w_k v(y, x) over the (y, k) with reflect(y + k) == y', y ascending then k
// ascending -- the scatter's visiting order
__global__ void adjoint_cols_kernel(const double* __restrict__ g, int W, int H, int C, double* __restrict__ t) {
    const size_t n = static_cast<size_t>(W) * H * C;
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = static_cast<int>(i % C);
    const size_t p = i / C;
    const int x = static_cast<int>(p % W), yd = static_cast<int>(p / W);
    const int y0 = H <= 4 * kRad + 2 ? 0 : max(0, yd - 2 * kRad - 1);
    const int y1 = H <= 4 * kRad + 2 ? H - 1 : min(H - 1, yd + 2 * kRad + 1);
    double acc[3] = {0.0, 0.0, 0.0};
    for (int y = y0; y <= y1; ++y) {
        const size_t j = (static_cast<size_t>(y) * W + x) * C + c;
        for (int k = -kRad; k <= kRad; ++k) {
            if (reflect_i(y + k, H) != yd) continue;
            const double w = c_taps[k + kRad];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double v = g[q * n + j];
                if (v != 0.0) acc[q] = dadd(acc[q], dmul(w, v));
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) t[q * n + i] = acc[q];
}

// blur_adjoint, row stage (metrics.cpp:76-84) as a gather, fused with the final
// combination grad_a = back_mu + 2 a back_a2 + b back_ab (metrics.cpp:155-158)
template <typename T>
__global__ void adjoint_rows_kernel(const double* __restrict__ t, const T* __restrict__ a,
                                    const T* __restrict__ b, int W, int H, int C, double* __restrict__ grad) {
    const size_t n = static_cast<size_t>(W) * H * C;
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = static_cast<int>(i % C);
    const size_t p = i / C;
    const int xd = static_cast<int>(p % W), y = static_cast<int>(p / W);
    const int x0 = W <= 4 * kRad + 2 ? 0 : max(0, xd - 2 * kRad - 1);
    const int x1 = W <= 4 * kRad + 2 ? W - 1 : min(W - 1, xd + 2 * kRad + 1);
    double acc[3] = {0.0, 0.0, 0.0};
    for (int x = x0; x <= x1; ++x) {
        const size_t j = (static_cast<size_t>(y) * W + x) * C + c;
        for (int k = -kRad; k <= kRad; ++k) {
            if (reflect_i(x + k, W) != xd) continue;
            const double w = c_taps[k + kRad];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double v = t[q * n + j];
                if (v != 0.0) acc[q] = dadd(acc[q], dmul(w, v));
            }
        }
    }
    grad[i] = dadd(dadd(acc[0], dmul(dmul(2.0, ld(a, i)), acc[1])), dmul(ld(b, i), acc[2]));
}

// squared differences for PSNR (metrics.cpp:116-119)
template <typename T>
__global__ void sqdiff_kernel(const T* __restrict__ a, const T* __restrict__ b, size_t n, double* __restrict__ out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double d = dsub(ld(a, i), ld(b, i));
    out[i] = dmul(d, d);
}

// Deterministic sum: a fixed grid of kRedBlocks blocks, block b owning a fixed
// contiguous range, each thread a fixed strided subset, a fixed shared-memory tree.
__global__ void partial_sum_kernel(const double* __restrict__ v, size_t n, double* __restrict__ partial) {
    __shared__ double sh[kRedThreads];
    const size_t per = (n + kRedBlocks - 1) / kRedBlocks;
    const size_t lo = per * blockIdx.x, hi = min(n, lo + per);
    double acc = 0.0;
    for (size_t i = lo + threadIdx.x; i < hi; i += kRedThreads) acc = dadd(acc, v[i]);
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = dadd(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void final_sum_kernel(const double* __restrict__ partial, double* __restrict__ out) {
    __shared__ double sh[kRedThreads];
    double acc = 0.0;
    for (int i = threadIdx.x; i < kRedBlocks; i += kRedThreads) acc = dadd(acc, partial[i]);
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = dadd(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

// window_taps (metrics.cpp:16-29) with the host libm, as the reference computes them
void upload_taps(cudaStream_t s) {
    static double taps[kWin];
    static const bool once = [] {
        double sum = 0.0;
        for (int i = 0; i < kWin; ++i) {
            const double d = i - kRad;
            taps[i] = std::exp(-d * d / (2.0 * 1.5 * 1.5));
            sum += taps[i];
        }
        for (double& v : taps) v /= sum;
        return true;
    }();
    (void)once;
    cudaMemcpyToSymbolAsync(c_taps, taps, sizeof(taps), 0, cudaMemcpyHostToDevice, s);
}

unsigned blocks_for(size_t n) { return static_cast<unsigned>((n + 255) / 256); }

}  // namespace

size_t metrics_scratch_doubles(size_t n, bool grad) { return (grad ? 9 : 6) * n + kRedBlocks + 2; }

void launch_psnr_sum(const void* a, const void* b, bool f64, size_t n, double* scratch, double* d_sum,
                     cudaStream_t s) {
    if (f64)
        sqdiff_kernel<double><<<blocks_for(n), 256, 0, s>>>(static_cast<const double*>(a),
                                                            static_cast<const double*>(b), n, scratch);
    else
        sqdiff_kernel<float><<<blocks_for(n), 256, 0, s>>>(static_cast<const float*>(a),
                                                           static_cast<const float*>(b), n, scratch);
    partial_sum_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(scratch, n, scratch + n);
    final_sum_kernel<<<1, kRedThreads, 0, s>>>(scratch + n, d_sum);
}

void launch_ssim(const void* a, const void* b, bool f64, int W, int H, int C, double* scratch, double* d_sum,
                 double* grad, cudaStream_t s) {
    const size_t n = static_cast<size_t>(W) * H * C;
    upload_taps(s);
    double* tmp = scratch;          // 5n: row-blurred moments; later 3n adjoint stage
    double* smap = scratch + 5 * n;  // n
    double* g = grad ? scratch + 6 * n : nullptr;  // 3n
    double* partial = scratch + (grad ? 9 : 6) * n;
    if (f64)
        ssim_rows_kernel<double><<<blocks_for(n), 256, 0, s>>>(static_cast<const double*>(a),
                                                               static_cast<const double*>(b), W, H, C, tmp);
    else
        ssim_rows_kernel<float><<<blocks_for(n), 256, 0, s>>>(static_cast<const float*>(a),
                                                              static_cast<const float*>(b), W, H, C, tmp);
    ssim_cols_kernel<<<blocks_for(n), 256, 0, s>>>(tmp, W, H, C, 1.0 / static_cast<double>(n), smap, g);
    partial_sum_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(smap, n, partial);
    final_sum_kernel<<<1, kRedThreads, 0, s>>>(partial, d_sum);
    if (!grad) return;
    adjoint_cols_kernel<<<blocks_for(n), 256, 0, s>>>(g, W, H, C, tmp);
    if (f64)
        adjoint_rows_kernel<double><<<blocks_for(n), 256, 0, s>>>(tmp, static_cast<const double*>(a),
                                                                  static_cast<const double*>(b), W, H, C, grad);
    else
        adjoint_rows_kernel<float><<<blocks_for(n), 256, 0, s>>>(tmp, static_cast<const float*>(a),
                                                                 static_cast<const float*>(b), W, H, C, grad);
}

}  // namespace sgs
