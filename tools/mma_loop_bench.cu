// mma_loop_bench.cu -- cycles per iteration of a decode-style MMA-warp loop on one SM:
// try_wait on two already-complete mbarriers, 8 x tcgen05.mma.kind::i8 128x16x32 (A from
// TMEM, B from smem), then `commits` tcgen05.commit arrivals (diagnostics).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_loop_bench tools/mma_loop_bench.cu
#include <cstdint>
#include <cstdio>

#include "../paper_2311_09550_b200/csrc/ptx.cuh"

using namespace odyb200;

__device__ __forceinline__ uint64_t desc128(uint32_t a) {
    return static_cast<uint64_t>((a >> 4) & 0x3FFFu) | (static_cast<uint64_t>(64) << 32) |
           (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}

__global__ void bench(int iters, int mmas, int commits, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bars[8];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc(&slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (2u << 17) | (8u << 24);  // N=16, M=128
    if (warp == 1) {
        // complete phase 0 of bars[0..1] once: the loop's waits on parity 0 pass at once
        if (threadIdx.x == 32) {
            mbar_arrive(&bars[0]);
            mbar_arrive(&bars[1]);
        }
        __syncwarp();
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            mbar_wait(&bars[0], 0);
            mbar_wait(&bars[1], 0);
            tc_fence_after();
            if (elect_one()) {
                for (int c = 0; c < mmas; ++c)
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
                        "r"(tmem + 256 + 8 * (c & 7)), "l"(desc128(smem_u32(smem) + 32 * (c & 3))), "r"(idesc),
                        "r"(c > 0 ? 1u : 0u)
                        : "memory");
                for (int c = 0; c < commits; ++c) mma_commit(&bars[2 + (c & 3)]);
            }
            __syncwarp();
        }
        long long t1 = clock64();
        if (threadIdx.x == 32) out[0] = (t1 - t0) / iters;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    printf("| MMAs per iteration | commits per iteration | cycles per iteration |\n|---|---|---|\n");
    for (int mmas : {0, 8})
        for (int commits : {0, 1, 2, 3}) {
            bench<<<1, 128, 64 * 1024>>>(2000, mmas, commits, d);
            long long h = 0;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("| %d | %d | %lld |\n", mmas, commits, h);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
