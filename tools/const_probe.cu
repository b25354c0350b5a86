// const_probe.cu -- latency of kernel-parameter (constant bank) loads on this B200: the
// decode kernel's producer reaches its first weight copy through ~4 levels of dependent
// run-time-indexed parameter loads (diagnostic).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/const_probe tools/const_probe.cu
//   tools/const_probe
//
// Per CTA, thread 0 times (globaltimer): a dependent chain of 4 indexed loads into cold
// parameter lines; the same after warming every line with immediate-offset (uniform)
// loads; and a chain into lines already touched.
#include <cstdint>
#include <cstdio>

struct Big {
    int v[1024];  // 4 KiB of parameters
};

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int keep(int v) {
    int r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}

// v[i] = index of the next load (a pointer chase through the parameter bank)
__global__ void chase(const __grid_constant__ Big b, unsigned long long* out, int start, int warm) {
    if (threadIdx.x != 0) return;
    if (warm) {
        const uint32_t* pw = reinterpret_cast<const uint32_t*>(&b);
        uint32_t acc = 0;
#pragma unroll
        for (int i = 0; i < 64; ++i) acc ^= pw[16 * i];
        keep(static_cast<int>(acc));
    }
    const unsigned long long t0 = gt();
    int i = start;
    i = keep(b.v[i]);
    i = keep(b.v[i]);
    i = keep(b.v[i]);
    i = keep(b.v[i]);
    const unsigned long long t1 = gt();
    // same lines again (warm)
    int j = start;
    j = keep(b.v[j]);
    j = keep(b.v[j]);
    j = keep(b.v[j]);
    j = keep(b.v[j]);
    const unsigned long long t2 = gt();
    out[3 * blockIdx.x] = t1 - t0;
    out[3 * blockIdx.x + 1] = t2 - t1;
    out[3 * blockIdx.x + 2] = i + j;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    static Big b;
    // chain 0 -> 300 -> 600 -> 900 -> 100 (distinct 64-byte lines)
    for (int i = 0; i < 1024; ++i) b.v[i] = 0;
    b.v[0] = 300;
    b.v[300] = 600;
    b.v[600] = 900;
    b.v[900] = 100;
    unsigned long long *d, h[3 * 1024];
    cudaMalloc(&d, 8 * 3 * 1024);
    for (int r = 0; r < 6; ++r) {
        const int warm = r >= 3;
        chase<<<sms, 32>>>(b, d, 0, warm);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 8 * 3 * sms, cudaMemcpyDeviceToHost);
        double c0 = 0, c1 = 0;
        for (int c = 0; c < sms; ++c) {
            c0 += h[3 * c];
            c1 += h[3 * c + 1];
        }
        printf("%s launch %d: 4 dependent indexed param loads %.3f us, again (same lines) %.3f us\n",
               warm ? "warmed (64 uniform loads first)" : "cold", r, c0 / sms / 1e3, c1 / sms / 1e3);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
