// quant_probe.cu -- throughput of the exact activation quantizer (quant16) on one CTA
// of 64 threads, staged in smem like the self-quantizer (diagnostic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2311_09550_b200/csrc \
//        -o tools/quant_probe tools/quant_probe.cu && tools/quant_probe
#include <vector>

#include "../paper_2311_09550_b200/csrc/decode_kernel.cu"

namespace odyb200 {
// link stubs for the host planner pulled in with decode_kernel.cu (unused here)
int device_sm_count() { return 148; }
cudaError_t launch_act_quant(const void*, int, size_t, int, int, int8_t*, float*, const float*, float*, bool,
                             cudaStream_t) {
    return cudaErrorNotSupported;
}
namespace {
__global__ void qprobe(const uint4* in, uint4* out, float sc, unsigned long long* tm, int reps, int bf, int dbg) {
    __shared__ uint4 xs[64 * 16];
    const int tid = threadIdx.x;
    for (int i = tid; i < 64 * 16; i += blockDim.x) xs[i] = in[i];
    __syncthreads();
    const float rcp = 1.0f / sc;
    uint4 acc = make_uint4(0, 0, 0, 0);
    const unsigned long long t0 = globaltimer();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint4 r0 = xs[(tid * 8 + i) * 2 % 1024], r1 = xs[((tid * 8 + i) * 2 + 1) % 1024];
            const uint4 v = bf ? quant16<true>(r0, r1, sc, rcp, dbg) : quant16<false>(r0, r1, sc, rcp, dbg);
            acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
        }
    }
    const unsigned long long t1 = globaltimer();
    out[tid] = acc;
    if (tid == 0) tm[blockIdx.x] = t1 - t0;
}
}  // namespace
}  // namespace odyb200

int main() {
    using namespace odyb200;
    std::vector<unsigned short> h(64 * 16 * 8);
    uint32_t s = 12345;
    for (auto& v : h) {
        s = s * 1664525u + 1013904223u;
        const float f = ((s >> 8) & 0xFFFF) / 65535.0f * 12.0f - 6.0f;
        v = __half_as_ushort(__float2half(f));
    }
    uint4 *in, *out;
    unsigned long long* tm;
    cudaMalloc(&in, h.size() * 2);
    cudaMalloc(&out, 64 * 16);
    cudaMalloc(&tm, 8 * 148);
    cudaMemcpy(in, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    const char* names[] = {"f16 (fix16 check)", "f16 no fix16 (dbg 2)", "bf16 (fix16 check)"};
    const int cfg[3][2] = {{0, 0}, {0, 2}, {1, 0}};
    for (int pass = 0; pass < 6; ++pass) {
        const int reps = 100;
        const int v = pass % 3;
        qprobe<<<1, 64>>>(in, out, 6.0f / 127.0f, tm, reps, cfg[v][0], cfg[v][1]);
        unsigned long long t;
        cudaDeviceSynchronize();
        cudaMemcpy(&t, tm, 8, cudaMemcpyDeviceToHost);
        printf("quant16 %-22s: %7.1f ns per 8 chunks per thread (2 warps), %s\n", names[v], t / double(reps),
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
