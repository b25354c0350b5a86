// i8_peak.cu -- whole-GPU dense INT8 tensor peak of this B200 (tcgen05.mma.kind::i8),
// the denominator BASELINE.md §2 asks for beside the 4.5 POPS datasheet figure.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_peak tools/i8_peak.cu
//   tools/i8_peak [seconds]
//
// One CTA per SM; an elected thread issues SS MMAs of 128 x 256 x 32 (s8 x s8 -> s32,
// the shape that runs at the per-SM peak in tools/mma_bench.cu) from pseudo-random
// operand tiles in shared memory into two TMEM accumulators, for a fixed count sized
// to ~0.2 s per launch (sustained clocks, not a burst).  TOPS = 2*M*N*K*MMAs / time.
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../paper_2311_09550_b200/csrc/ptx.cuh"

using namespace odyb200;

__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
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

constexpr int kN = 256;
constexpr int kABytes = 128 * 128, kBBytes = kN * 128;

__global__ void __launch_bounds__(128, 1) peak_kernel(long long mmas, unsigned seed, int* sink) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    // pseudo-random operands (data-dependent power: not zeros)
    uint32_t x = seed ^ (blockIdx.x * 0x9E3779B9u) ^ (threadIdx.x * 0x85EBCA6Bu);
    for (int i = threadIdx.x; i < (kABytes + kBBytes) / 4; i += blockDim.x) {
        x ^= x << 13;
        x ^= x >> 17;
        x ^= x << 5;
        reinterpret_cast<uint32_t*>(smem)[i] = x;
    }
    fence_proxy_async_shared();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) {
        tmem_alloc(&slot, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(kN >> 3) << 17) |
                           (static_cast<uint32_t>(128 >> 4) << 24);
    if (threadIdx.x < 32) {
        if (elect_one()) {
            const uint32_t a0 = smem_u32(smem), b0 = a0 + kABytes;
            for (long long i = 0; i < mmas; i += 8) {
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    mma_i8_ss(tmem + (c & 1) * kN, desc128(a0 + 32 * (c & 3)), desc128(b0 + 32 * (c & 3)), idesc,
                              i > 0 || c > 1 ? 1u : 0u);
            }
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        tc_fence_after();
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem, v);
        tmem_wait_ld();
        if (v[0] == 0x12345678u) atomicAdd(sink, 1);  // keep the result live
        tc_fence_before();
    }
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

int main(int argc, char** argv) {
    const double seconds = argc > 1 ? atof(argv[1]) : 0.2;
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const int smem = kABytes + kBBytes + 2048;
    cudaFuncSetAttribute(peak_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int* sink;
    cudaMalloc(&sink, 4);
    // ~64 cycles per 128x256x32 MMA at the per-SM peak: size the count to `seconds`
    const long long mmas = static_cast<long long>(seconds * clk * 1e3 / 64.0) / 8 * 8;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    peak_kernel<<<sms, 128, smem>>>(mmas / 20, 1u, sink);  // warm-up
    cudaDeviceSynchronize();
    double best = 0, sum = 0;
    const int runs = 5;
    for (int r = 0; r < runs; ++r) {
        cudaEventRecord(a);
        peak_kernel<<<sms, 128, smem>>>(mmas, 7u + r, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double tops = 2.0 * 128 * kN * 32 * static_cast<double>(mmas) * sms / (ms * 1e-3) / 1e12;
        best = tops > best ? tops : best;
        sum += tops;
        printf("run %d: %.3f ms  %.1f TOPS\n", r, ms, tops);
    }
    const cudaError_t e = cudaGetLastError();
    printf("{\"i8_dense_tops_sustained_mean\": %.1f, \"i8_dense_tops_best\": %.1f, \"sms\": %d, "
           "\"max_clock_mhz\": %d, \"mma\": \"128x%dx32 SS kind::i8\", \"seconds_per_run\": %.2f, \"err\": \"%s\"}\n",
           sum / runs, best, sms, clk / 1000, kN, seconds, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
