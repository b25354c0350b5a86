// icache_probe.cu -- cost of cold instruction fetch on this B200 (diagnostic for the
// decode kernel's per-launch ramp: ~0.6 us between trace marks a few instructions apart).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/icache_probe tools/icache_probe.cu
//   tools/icache_probe
//
// One warp per CTA runs a long straight-line block of independent ALU instructions
// (kBlocks x 64 unrolled IADDs, 16 B each) twice, timing each pass with globaltimer:
// pass 0 fetches the code cold (first launch) or from whatever the previous launch
// left cached; pass 1 is warm.  Launched several times back to back, with and without
// a "flush" kernel of different code in between, and with all SMs busy streaming HBM.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// 8 independent chains: issue-bound (~1 instruction per cycle), so fetch stalls show
template <int N>
__device__ __forceinline__ uint32_t straight(uint32_t a, uint32_t b) {
    uint32_t r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a + j;
#pragma unroll
    for (int i = 0; i < N / 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("add.u32 %0, %0, %1;" : "+r"(r[j]) : "r"(b));
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) x ^= r[j];
    return x;
}
// the same amount of code cut into 32 blocks, each behind a data-dependent branch whose
// taken target is the far side of a skipped block (cold code on every jump)
template <int N>
__device__ __forceinline__ uint32_t branchy(uint32_t a, uint32_t b, const int* flags) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
        if (__ldg(flags + k)) a = straight<N / 64>(a, b + k);
        else a = straight<N / 64>(a ^ k, b);
    }
    return a;
}

constexpr int kInstr = 2048;  // x2 instructions x 16 B = 64 KiB of code per pass

__global__ void probe(unsigned long long* out, uint32_t seed, const uint4* hbm, size_t n, const int* flags) {
    if (threadIdx.x >= 32) {  // other warps: stream HBM (load) while warp 0 runs
        uint4 acc = {};
        for (size_t i = blockIdx.x * (blockDim.x - 32) + threadIdx.x - 32; i < n; i += gridDim.x * (blockDim.x - 32)) {
            const uint4 v = __ldcs(hbm + i);
            acc.x ^= v.x;
        }
        if (acc.x == 0x12345678u) out[1023] = acc.x;
        return;
    }
    uint32_t a = seed + threadIdx.x, b = seed * 3;
    unsigned long long t[8];
    for (int pass = 0; pass < 2; ++pass) {
        t[2 * pass] = gt();
        a = straight<kInstr>(a, b);
        t[2 * pass + 1] = gt();
        b ^= a;
    }
    for (int pass = 0; pass < 2; ++pass) {
        t[4 + 2 * pass] = gt();
        a = branchy<kInstr>(a, b, flags);
        t[4 + 2 * pass + 1] = gt();
        b ^= a;
    }
    if (threadIdx.x == 0) {
        out[4 * blockIdx.x + 0] = t[1] - t[0];
        out[4 * blockIdx.x + 1] = t[3] - t[2];
        out[4 * blockIdx.x + 2] = t[5] - t[4];
        out[4 * blockIdx.x + 3] = t[7] - t[6];
        if (a == 0x7654321u) out[1023] = a;
    }
}

template <int KB>  // KB KiB of straight-line code
__global__ void other(unsigned long long* out, uint32_t seed) {
    uint32_t a = seed + threadIdx.x, b = seed * 5;
    a = straight<KB * 1024 / 32>(a, b);
    if (a == 0x1234567u) out[0] = a;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *d, h[4 * 1024];
    cudaMalloc(&d, 8 * 4 * 1024);
    const size_t n = (size_t(1) << 30) / 16;  // 1 GiB to stream
    int* flags;
    cudaMalloc(&flags, 64 * 4);
    cudaMemset(flags, 0, 64 * 4);
    uint4* hbm;
    cudaMalloc(&hbm, n * 16);
    cudaMemset(hbm, 1, n * 16);
    const char* names[] = {"first launch", "repeat", "repeat", "after 8 KiB kernel", "after 32 KiB kernel",
                           "after 64 KiB kernel", "after 96 KiB kernel", "after 128 KiB kernel",
                           "loaded: repeat", "loaded: after 32 KiB"};
    for (int r = 0; r < 10; ++r) {
        if (r == 3) other<8><<<sms, 32>>>(d + 2048, 7);
        if (r == 4 || r == 9) other<32><<<sms, 32>>>(d + 2048, 7);
        if (r == 5) other<64><<<sms, 32>>>(d + 2048, 7);
        if (r == 6) other<96><<<sms, 32>>>(d + 2048, 7);
        if (r == 7) other<128><<<sms, 32>>>(d + 2048, 7);
        const bool load = r >= 8;
        probe<<<sms, load ? 32 + 256 : 32>>>(d, 11u + r, hbm, load ? n : 0, flags);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8 * 4 * sms, cudaMemcpyDeviceToHost);
        double p[4] = {0, 0, 0, 0};
        for (int c = 0; c < sms; ++c)
            for (int q = 0; q < 4; ++q) p[q] += h[4 * c + q];
        printf("%-22s straight pass0 %6.2f pass1 %6.2f us | 32 far branches pass0 %6.2f pass1 %6.2f us "
               "(mean over %d CTAs)\n", names[r], p[0] / sms / 1e3, p[1] / sms / 1e3, p[2] / sms / 1e3,
               p[3] / sms / 1e3, sms);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
