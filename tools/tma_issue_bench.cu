// tma_issue_bench.cu -- cost of ISSUING 1-D bulk copies (cp.async.bulk) from one thread:
// clock64 around each issue, for 1 CTA and for a full grid (diagnostics; GPU box only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_09550_b200/csrc \
//        tools/tma_issue_bench.cu -o tools/tma_issue_bench
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"
using namespace odyb200;

__global__ void issue_kernel(const uint8_t* src, size_t per_cta, int chunk, int n, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 12 * 16384);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint8_t* base = src + per_cta * blockIdx.x;
    const uint64_t pol = l2_policy_evict_first();
    mbar_expect_tx(bar, static_cast<uint32_t>(n) * chunk);
    unsigned long long t0 = clock64(), tmax = 0;
    for (int i = 0; i < n; ++i) {
        const unsigned long long a = clock64();
        bulk_g2s(smem + (i % 12) * 16384, base + static_cast<size_t>(i) * chunk, chunk, bar, pol);
        const unsigned long long b = clock64();
        if (b - a > tmax) tmax = b - a;
    }
    const unsigned long long t1 = clock64();
    mbar_wait(bar, 0);
    const unsigned long long t2 = clock64();
    if (blockIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = tmax;
        out[2] = t2 - t0;
    }
}

int main() {
    uint8_t* buf;
    cudaMalloc(&buf, size_t(1) << 30);
    cudaMemset(buf, 1, size_t(1) << 30);
    unsigned long long* out;
    cudaMalloc(&out, 64);
    cudaFuncSetAttribute(issue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 13 * 16384);
    for (int grid : {1, 148})
        for (int chunk : {4096, 16384})
            for (int n : {4, 12}) {
                for (int rep = 0; rep < 2; ++rep)
                    issue_kernel<<<grid, 32, 13 * 16384>>>(buf + rep * (size_t(1) << 28), size_t(1) << 20, chunk, n, out);
                cudaDeviceSynchronize();
                unsigned long long h[3];
                cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
                std::printf("grid %3d chunk %5d n %2d: issue all %6llu cyc (%5llu/copy, max %5llu), landed %6llu cyc -> %.1f B/clk\n",
                            grid, chunk, n, h[0], h[0] / n, h[1], h[2], double(n) * chunk / h[2]);
            }
    return 0;
}
