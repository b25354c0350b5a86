// stream_bench.cu -- upper bounds for the decode GEMM's weight stream (diagnostics; GPU box only).
//
//  part 1: how fast can CTAs pull contiguous bytes -> smem with 1-D bulk copies (UBLKCP)
//          into an S-stage ring, from HBM (rotating pool) and from L2 (same buffer,
//          evict_normal), per grid / chunk / stage count;
//  part 2: a chain of 4 "layer" kernels (39/13/71/35 MB, the LLaMA-13B linears) launched
//          back to back with and without PDL, where each kernel streams its first ring
//          before griddepcontrol.wait and optionally L2-prefetches more -- the best
//          step time a kernel-per-linear design can reach.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_09550_b200/csrc \
//        tools/stream_bench.cu -o tools/stream_bench && tools/stream_bench
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"
using namespace odyb200;

struct SP {
    const uint8_t* src;
    size_t per_cta;
    int chunk, stages, policy, pdl, pf_bytes, hold;  // hold: pdl-wait after first ring
    unsigned long long* sink;
};

__global__ void stream_kernel(const SP p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * p.chunk);
    if (p.pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int i = 0; i < p.stages; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const uint8_t* base = p.src + p.per_cta * blockIdx.x;
    const int n = static_cast<int>(p.per_cta / p.chunk);
    uint64_t pol;
    if (p.policy == 0) pol = l2_policy_evict_first();
    else if (p.policy == 2) pol = l2_policy_evict_last();
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    int issued = 0;
    unsigned long long acc = 0;
    for (; issued < p.stages && issued < n; ++issued) {
        mbar_expect_tx(&full[issued], p.chunk);
        bulk_g2s(smem + issued * p.chunk, base + static_cast<size_t>(issued) * p.chunk, p.chunk,
                 &full[issued], pol);
    }
    if (p.pf_bytes > 0) {
        const size_t lo = static_cast<size_t>(issued) * p.chunk;
        const size_t hi = lo + p.pf_bytes < p.per_cta ? lo + p.pf_bytes : p.per_cta;
        for (size_t off = lo; off < hi; off += 16384) {
            const uint32_t b = static_cast<uint32_t>(hi - off < 16384 ? hi - off : 16384);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(b) : "memory");
        }
    }
    if (p.hold) asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int u = 0; u < n; ++u) {
        const int s = u % p.stages;
        mbar_wait(&full[s], (u / p.stages) & 1);
        acc += lds32(smem_u32(smem + s * p.chunk));
        if (issued < n) {
            mbar_expect_tx(&full[s], p.chunk);
            bulk_g2s(smem + s * p.chunk, base + static_cast<size_t>(issued) * p.chunk, p.chunk, &full[s], pol);
            ++issued;
        }
    }
    p.sink[blockIdx.x] = acc;
}

static void launch(const SP& p, int grid, int smem, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, stream_kernel, p);
}

int main() {
    const size_t total_max = size_t(2) << 30;  // 2 GiB rotating pool (>> L2)
    uint8_t* buf;
    cudaMalloc(&buf, total_max);
    cudaMemset(buf, 1, total_max);
    unsigned long long* sink;
    cudaMalloc(&sink, 4096 * 8);
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time_it = [&](auto&& body, int reps) {
        for (int i = 0; i < 3; ++i) body(i);
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i) body(i);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        return ms * 1e3 / reps;
    };
    // ---- part 1: L2-resident bandwidth (same buffer, evict_normal / evict_last) ----
    for (size_t mb : {12, 24, 39, 60})
        for (int grid : {148, 296})
            for (int pol : {1, 2}) {
                const int chunk = 16384, stages = grid == 148 ? 8 : 4;
                const size_t per = ((mb << 20) / grid) / chunk * chunk;
                SP p = {buf, per, chunk, stages, pol, 0, 0, 0, sink};
                const int smem = chunk * stages + 1024;
                const double us = time_it([&](int) { launch(p, grid, smem, false); }, 40);
                std::printf("L2 %3zu MB grid %3d pol %d: %7.2f us %6.0f GB/s\n", mb, grid, pol, us,
                            per * grid / us / 1e3);
            }
    // ---- part 2: 4-kernel layer chain (qkv, o, gate_up, down weight bytes) ----
    const size_t layer_mb[4] = {39321600, 13107200, 70778880, 35389440};
    size_t step_bytes = 0;
    for (size_t b : layer_mb) step_bytes += b;
    const int copies = static_cast<int>(total_max / step_bytes);
    struct C2 { int grid, chunk, stages, pdl, pf_kb; };
    std::vector<C2> c2s = {{148, 16384, 12, 0, 0},  {148, 16384, 12, 1, 0},  {148, 16384, 12, 1, 256},
                           {148, 16384, 6, 1, 0},   {148, 16384, 6, 1, 256}, {296, 16384, 6, 1, 0},
                           {296, 16384, 6, 1, 128}, {296, 16384, 4, 1, 128}, {296, 8192, 8, 1, 128},
                           {120, 16384, 12, 1, 256}};
    for (const C2& c : c2s) {
        const int smem = c.chunk * c.stages + 1024;
        const double us = time_it(
            [&](int it) {
                const uint8_t* base = buf + static_cast<size_t>(it % copies) * step_bytes;
                for (int l = 0; l < 4; ++l) {
                    const size_t per = (layer_mb[l] / c.grid) / c.chunk * c.chunk;
                    SP p = {base, per, c.chunk, c.stages, 0, c.pdl, c.pf_kb * 1024, c.pdl, sink};
                    launch(p, c.grid, smem, c.pdl);
                    base += layer_mb[l];
                }
            },
            30);
        std::printf("chain grid %3d chunk %5d stages %2d pdl %d pf %3d KB: %7.2f us/step %6.0f GB/s\n", c.grid,
                    c.chunk, c.stages, c.pdl, c.pf_kb, us, step_bytes / us / 1e3);
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
