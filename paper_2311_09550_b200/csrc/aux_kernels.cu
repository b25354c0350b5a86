// aux_kernels.cu -- the reference's offline / test-side numerics on the GPU, bit-exact:
//
//   lwc_grid_kernel    ref clip.cpp:55-103 optimize_clipping (LWC grid search, SURVEY §8f
//                      row 4): per channel, every (gamma, beta) candidate pair's
//                      quantization MSE (double, sequential over the row like
//                      mse_for_scale, clip.cpp:40-51), and the reference's tie-break.
//   matmul_f32_kernel  ref tensor.cpp:176-196 matmul_f32 (fixed-order f32 dot, the
//                      reference's float oracle; ody_matmul_f32).
//
// Both are CUDA-core kernels: the reference fixes the accumulation ORDER (sequential
// double / float sums), which any tree or tensor-core reduction would change.  No FMA
// contraction anywhere (__fmul_rn / __dadd_rn ... spell every rounding out).
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "layout.h"

namespace odyb200 {

namespace {

constexpr int kLwcThreads = 256;
constexpr int kMaxCand = 1024;  // candidates per axis the grid may hold

// ref clip.cpp:11-24 ClipGrid::candidates: min + i*step (f32, no FMA) while < 1 - 1e-6,
// then 1.0
__device__ int lwc_candidates(float gmin, float step, float* out) {
    int n = 0;
    for (int i = 0; n < kMaxCand - 1; ++i) {
        const float v = __fadd_rn(gmin, __fmul_rn(static_cast<float>(i), step));
        if (v >= 1.0f - 1e-6f) break;
        out[n++] = v;
    }
    out[n++] = 1.0f;
    return n;
}

// ref clip.cpp:40-51 mse_for_scale: sum over the row, in order, of
// (double(v) - double(clamp(round(v / s))) * double(s))^2, / K
__device__ double lwc_mse(const float* w, int K, float s, float lo, float hi) {
    double acc = 0.0;
    for (int k = 0; k < K; ++k) {
        const float v = w[k];
        float c = roundf(__fdiv_rn(v, s));
        c = fminf(fmaxf(c, lo), hi);
        const double e = __dsub_rn(static_cast<double>(v), __dmul_rn(static_cast<double>(c), static_cast<double>(s)));
        acc = __dadd_rn(acc, __dmul_rn(e, e));
    }
    return __ddiv_rn(acc, static_cast<double>(K));
}

// (mse, -(g+b), -g) lexicographic: the candidate the reference's sequential scan keeps
// (clip.cpp:81-90) -- its "better" relation is this strict order, so any reduction
// order picks the same winner.
__device__ __forceinline__ bool lwc_better(double m1, float g1, float b1, double m2, float g2, float b2) {
    if (m1 != m2) return m1 < m2;
    const float s1 = __fadd_rn(g1, b1), s2 = __fadd_rn(g2, b2);
    if (s1 != s2) return s1 > s2;
    return g1 > g2;
}

__global__ void __launch_bounds__(kLwcThreads) lwc_grid_kernel(const float* __restrict__ w, int N, int K, int bits,
                                                               float gmin, float step, float* gamma, float* beta,
                                                               float* mse_before, float* mse_after) {
    extern __shared__ float row[];  // K floats
    __shared__ float cand[kMaxCand];
    __shared__ double r_mse[kLwcThreads];
    __shared__ float r_g[kLwcThreads], r_b[kLwcThreads];
    __shared__ float s_max, s_min;
    __shared__ int s_nc;
    __shared__ double s_ident;
    const int r = blockIdx.x;
    const float* src = w + static_cast<size_t>(r) * K;
    for (int k = threadIdx.x; k < K; k += kLwcThreads) row[k] = src[k];
    if (threadIdx.x == 0) s_nc = lwc_candidates(gmin, step, cand);
    __syncthreads();
    if (threadIdx.x == 0) {  // ref clip.cpp:68-72 (max / min, in order: exact either way)
        float mx = row[0], mn = row[0];
        for (int k = 1; k < K; ++k) {
            mx = fmaxf(mx, row[k]);
            mn = fminf(mn, row[k]);
        }
        s_max = mx;
        s_min = mn;
    }
    __syncthreads();
    const int nc = s_nc;
    const float qmax = static_cast<float>((1 << (bits - 1)) - 1);
    const float lo = static_cast<float>(-(1 << (bits - 1)));
    double best = 0.0;
    float bg = 1.0f, bb = 1.0f;
    bool have = false;
    for (int c = threadIdx.x; c < nc * nc; c += kLwcThreads) {
        const float g = cand[c / nc], b = cand[c % nc];
        float s = __fdiv_rn(fmaxf(fabsf(__fmul_rn(g, s_max)), fabsf(__fmul_rn(b, s_min))), qmax);
        if (!(s > 0.0f)) s = kMinScale;
        const double m = lwc_mse(row, K, s, lo, qmax);
        if (g == 1.0f && b == 1.0f) s_ident = m;
        if (!have || lwc_better(m, g, b, best, bg, bb)) {
            best = m;
            bg = g;
            bb = b;
            have = true;
        }
    }
    r_mse[threadIdx.x] = have ? best : 1.0 / 0.0;
    r_g[threadIdx.x] = bg;
    r_b[threadIdx.x] = bb;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = r_mse[0];
        float g = r_g[0], b = r_b[0];
        for (int t = 1; t < kLwcThreads; ++t)
            if (lwc_better(r_mse[t], r_g[t], r_b[t], m, g, b)) {
                m = r_mse[t];
                g = r_g[t];
                b = r_b[t];
            }
        gamma[r] = g;
        beta[r] = b;
        mse_before[r] = static_cast<float>(s_ident);
        mse_after[r] = static_cast<float>(m);
    }
}

// ref tensor.cpp:176-196: out[i][j] = ((0 + a0*b0) + a1*b1) + ..., f32, no FMA.
__global__ void matmul_f32_kernel(const float* __restrict__ a, const float* __restrict__ bt, int M, int N, int K,
                                  float* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= N) return;
    const float* ai = a + static_cast<size_t>(i) * K;
    const float* bj = bt + static_cast<size_t>(j) * K;
    float acc = 0.0f;
    for (int k = 0; k < K; ++k) acc = __fadd_rn(acc, __fmul_rn(ai[k], bj[k]));
    out[static_cast<size_t>(i) * N + j] = acc;
}

}  // namespace

int lwc_max_candidates() { return kMaxCand; }

cudaError_t launch_lwc_grid(const float* w, int N, int K, int bits, float grid_min, float grid_step, float* gamma,
                            float* beta, float* mse_before, float* mse_after, cudaStream_t st) {
    const size_t smem = static_cast<size_t>(K) * sizeof(float);
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        const cudaError_t e =
            cudaFuncSetAttribute(lwc_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    lwc_grid_kernel<<<N, kLwcThreads, smem, st>>>(w, N, K, bits, grid_min, grid_step, gamma, beta, mse_before,
                                                  mse_after);
    return cudaGetLastError();
}

cudaError_t launch_matmul_f32(const float* a, const float* bt, int M, int N, int K, float* out, cudaStream_t st) {
    dim3 grid((N + 127) / 128, M);
    matmul_f32_kernel<<<grid, 128, 0, st>>>(a, bt, M, N, K, out);
    return cudaGetLastError();
}

}  // namespace odyb200
