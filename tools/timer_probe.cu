// Resolution of %globaltimer vs clock64 on the box (diagnostics).
#include <cstdio>
__global__ void k(unsigned long long* out) {
    unsigned long long prev, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
    int n = 0;
    long long c0 = clock64();
    while (n < 16) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t != prev) { out[n * 2] = t - prev; out[n * 2 + 1] = clock64() - c0; prev = t; ++n; }
    }
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 256 * 8);
    k<<<1, 1>>>(d); cudaDeviceSynchronize();
    unsigned long long h[32]; cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 16; ++i) printf("step %llu ns at clk %llu\n", h[2 * i], h[2 * i + 1]);
}
