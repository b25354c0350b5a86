// mma_bench.cu -- microbenchmark of tcgen05.mma.kind::i8 issue/execute rates on one SM
// (diagnostics for the FastGEMM design; not part of the library).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu
//
// For each (A source, N, chains): one elected thread issues R MMAs of 128xNx32 into
// `chains` independent TMEM accumulators, commits, and waits; reports cycles per MMA.
#include <cstdint>
#include <cstdio>

#include "../paper_2311_09550_b200/csrc/ptx.cuh"

using namespace odyb200;

__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ uint64_t desc128(uint32_t smem_addr) {
    return static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(64) << 32) |
           (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}

__global__ void bench(int n, int chains, int ss, int reps, int mdim, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
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
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
                           (static_cast<uint32_t>(mdim >> 4) << 24);
    const uint32_t base = smem_u32(smem);
    long long t0 = 0, t1 = 0;
    if (warp == 1) {
        for (int pass = 0; pass < 2; ++pass) {
            __syncwarp();
            t0 = clock64();
            if (elect_one()) {
                const uint64_t bd = desc128(base + 32768);
                const uint64_t ad = desc128(base);
                if (ss) {
                    for (int i = 0; i < reps; i += 8) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) mma_i8_ss(tmem + (j % chains) * n, ad, bd, idesc, 1);
                    }
                } else {
                    for (int i = 0; i < reps; i += 8) {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            mma_i8_ts(tmem + (j % chains) * n, tmem + 256 + 8 * j, bd, idesc, 1);
                    }
                }
                mma_commit(&bar);
            }
            __syncwarp();
            mbar_wait(&bar, pass & 1);
            t1 = clock64();
        }
        if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8 * 148);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    const int reps = 512;
    printf("%-4s %4s %4s %6s %10s %12s\n", "src", "M", "N", "chains", "cyc/MMA", "MAC/cyc");
    for (int mdim : {128, 64}) {
        for (int ss = 0; ss < 2; ++ss) {
            for (int n : {16, 32, 64, 128, 256}) {
                for (int chains : {1, 4}) {
                    if (chains * n > 256) continue;
                    bench<<<1, 128, 96 * 1024>>>(n, chains, ss, reps, mdim, d);
                    long long h = 0;
                    cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                    if (e != cudaSuccess) {
                        printf("error %s\n", cudaGetErrorString(e));
                        return 1;
                    }
                    const double cyc = static_cast<double>(h) / reps;
                    printf("%-4s %4d %4d %6d %10.1f %12.0f\n", ss ? "SS" : "TS", mdim, n, chains, cyc,
                           static_cast<double>(mdim) * n * 32 / cyc);
                }
            }
        }
    }
    return 0;
}
