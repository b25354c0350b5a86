// quant_kernels.cu -- K1 (per-token INT8 activation quantization) and K2 (per-channel
// INT4 weight quantization + prepack into the w4 tile layout), plus the layout
// converters used by checkpoint ingest/export and the parity suite.
//
// Bit-exactness contract with the reference (ref quantize.cpp:12-47,113-132):
//   S = max(|g*max|,|b*min|) / qmax  (IEEE f32 division), S <= 0 -> 2^-24
//   code = clamp(roundf(x / S))       (IEEE division, round half away from zero)
// Built WITHOUT --use_fast_math so '/' is IEEE round-to-nearest and no FTZ.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "kernels.h"
#include "layout.h"
#include "ptx.cuh"
#include "quant_common.cuh"

namespace odyb200 {

namespace {

constexpr int kActThreads = 128;
constexpr int kActBatch = 8;

// K1: per-token INT8 quantization, one CTA of NT threads per token row; every thread
// keeps its MC 16-element chunks in registers across both passes.  Pass 1: row
// max|x| (warp shuffle -> smem).  Pass 2: codes clamp(roundf(x/S)) (exact fast path
// above), one 128-bit store per chunk into the swizzled a8 k-block layout.
// absmax_in (optional) supplies the row max (row-parallel TP: the all-reduced global
// max of a K-sharded row); absmax_out (optional) exports it.  With PDL the kernel
// lets its consumer launch immediately and waits for its producer before touching x.
template <typename T, int NT, int MC>
__device__ __forceinline__ void act_quant_row(const T* __restrict__ row, int t, int K, int Kp, int Mp,
                                              int8_t* __restrict__ q, float* __restrict__ s,
                                              const float* __restrict__ absmax_in,
                                              float* __restrict__ absmax_out, float* red,
                                              unsigned long long* __restrict__ trace) {
    const int nchunks = Kp / 16;
    float v[MC][16];
    float mx = 0.0f;
#pragma unroll
    for (int i = 0; i < MC; ++i) {
        const int c = threadIdx.x + i * NT;
        if (c < nchunks) {
            load16(row, c * 16, K, v[i]);
#pragma unroll
            for (int e = 0; e < 16; ++e) mx = fmaxf(mx, fabsf(v[i][e]));
        }
    }
    float scale;
    if (absmax_in) {
        scale = absmax_in[t] / 127.0f;
    } else {
        mx = warp_max(mx);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        __syncthreads();
        float m = red[0];
#pragma unroll
        for (int i = 1; i < NT / 32; ++i) m = fmaxf(m, red[i]);
        // max(|max|,|min|) == max|x| for finite rows (ref quantize.cpp:27-33)
        scale = m / 127.0f;
        if (threadIdx.x == 0 && absmax_out) absmax_out[t] = m;
    }
    if (!(scale > 0.0f)) scale = kMinScale;
    if (threadIdx.x == 0) s[t] = scale;
    if (trace && threadIdx.x == 0) trace[blockIdx.x * 8 + 3] = globaltimer();
    const float rcp = 1.0f / scale;
    const bool exact = !(rcp < INFINITY);

#pragma unroll
    for (int i = 0; i < MC; ++i) {
        const int c = threadIdx.x + i * NT;
        if (c < nchunks) {
            uint32_t tb[16];
            bool redo = exact;
#pragma unroll
            for (int e = 0; e < 16; ++e) tb[e] = quant_byte_fast(v[i][e], rcp, redo);
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                w[j] = pack4_low_bytes(tb[4 * j], tb[4 * j + 1], tb[4 * j + 2], tb[4 * j + 3]);
            if (redo) {  // rare: a near-half-integer quotient or non-finite 1/S
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint32_t acc = 0;
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int32_t code = quant_code_i8(v[i][j * 4 + b], scale, rcp, true);
                        acc |= (static_cast<uint32_t>(code) & 0xFFu) << (8 * b);
                    }
                    w[j] = acc;
                }
            }
            const size_t off = a8_offset(static_cast<size_t>(t), static_cast<size_t>(c) * 16, Mp);
            *reinterpret_cast<uint4*>(q + off) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

template <typename T, int NT, int MC>
__global__ void __launch_bounds__(NT)
act_quant_kernel(const T* __restrict__ x, size_t ldx, int M, int K, int Kp, int Mp,
                 int8_t* __restrict__ q, float* __restrict__ s,
                 const float* __restrict__ absmax_in, float* __restrict__ absmax_out,
                 int pdl, unsigned long long* __restrict__ trace) {
    if (trace && threadIdx.x == 0) trace[blockIdx.x * 8] = globaltimer();
    if (pdl) {
        pdl_launch_dependents();  // let the consumer GEMM start streaming its weights now
        pdl_wait();
    }
    if (trace && threadIdx.x == 0) trace[blockIdx.x * 8 + 2] = globaltimer();
    __shared__ float red[NT / 32];
    const int t = blockIdx.x;
    act_quant_row<T, NT, MC>(x + static_cast<size_t>(t) * ldx, t, K, Kp, Mp, q, s, absmax_in, absmax_out, red,
                             trace);
    if (trace) {
        __syncthreads();
        if (threadIdx.x == 0) trace[blockIdx.x * 8 + 1] = globaltimer();
    }
}

// K1 for a batch of up to kActBatch activation matrices (the external inputs of a
// linear program) in ONE launch: CTA b quantizes global row b of the concatenation.
struct ActBatch {
    const void* x[kActBatch];
    size_t ldx[kActBatch];
    int dtype[kActBatch], M[kActBatch], K[kActBatch];
    int8_t* q[kActBatch];
    float* s[kActBatch];
    int n, pdl;
};

template <int NT, int MC>
__global__ void __launch_bounds__(NT) act_quant_batch_kernel(const __grid_constant__ ActBatch b) {
    if (b.pdl) {
        pdl_launch_dependents();
        pdl_wait();
    }
    __shared__ float red[NT / 32];
    int i = 0, t = blockIdx.x;
    while (i + 1 < b.n && t >= b.M[i]) t -= b.M[i++];
    const int K = b.K[i], Kp = static_cast<int>(pad_k(K)), Mp = static_cast<int>(pad_m(b.M[i]));
    switch (b.dtype[i]) {
        case kDtypeF32:
            act_quant_row<float, NT, MC>(static_cast<const float*>(b.x[i]) + t * b.ldx[i], t, K, Kp, Mp, b.q[i],
                                         b.s[i], nullptr, nullptr, red, nullptr);
            break;
        case kDtypeF16:
            act_quant_row<__half, NT, MC>(static_cast<const __half*>(b.x[i]) + t * b.ldx[i], t, K, Kp, Mp, b.q[i],
                                          b.s[i], nullptr, nullptr, red, nullptr);
            break;
        default:
            act_quant_row<__nv_bfloat16, NT, MC>(static_cast<const __nv_bfloat16*>(b.x[i]) + t * b.ldx[i], t, K,
                                                 Kp, Mp, b.q[i], b.s[i], nullptr, nullptr, red, nullptr);
            break;
    }
}

// Per-row scale for per-channel weights: ref quantize.cpp:22-35.  One warp per row.
__global__ void w_scale_kernel(const float* __restrict__ w, int N, int K, int bits,
                               const float* __restrict__ gamma, const float* __restrict__ beta,
                               float* __restrict__ s, int* __restrict__ err) {
    const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= N) return;
    const float* r = w + static_cast<size_t>(row) * K;
    float mx = r[0], mn = r[0];
    for (int k = lane; k < K; k += 32) {
        mx = fmaxf(mx, r[k]);
        mn = fminf(mn, r[k]);
    }
    mx = warp_max(mx);
    mn = warp_min(mn);
    if (lane == 0) {
        const float g = gamma ? gamma[row] : 1.0f;
        const float b = beta ? beta[row] : 1.0f;
        if (err && !(g > 0.0f && g <= 1.0f && b > 0.0f && b <= 1.0f)) atomicExch(err, 1);
        const float qmax = static_cast<float>((1 << (bits - 1)) - 1);
        float sc = fmaxf(fabsf(__fmul_rn(g, mx)), fabsf(__fmul_rn(b, mn))) / qmax;
        s[row] = sc > 0.0f ? sc : kMinScale;
    }
}

// K2 (quantize + prepack): one thread per (row, 32-k chunk); writes one 16-byte
// row chunk of the w4 tile layout.  Rows >= N and k >= K are zero codes.
__global__ void w4_quant_prepack_kernel(const float* __restrict__ w, int N, int K, int Np, int Kp,
                                        const float* __restrict__ s, uint8_t* __restrict__ out) {
    const size_t chunks_per_row = Kp / 32;
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<size_t>(Np) * chunks_per_row) return;
    const int r = static_cast<int>(idx / chunks_per_row);
    const int cc = static_cast<int>(idx % chunks_per_row);
    int8_t code[32];
    if (r < N) {
        const float sc = s[r];
        const float* row = w + static_cast<size_t>(r) * K;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const int k = cc * 32 + e;
            code[e] = k < K ? static_cast<int8_t>(clamp_code(row[k] / sc, -8, 7)) : int8_t(0);
        }
    } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) code[e] = 0;
    }
    uint32_t word[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t lo = static_cast<uint32_t>(code[8 * j + b]) & 0xFu;
            const uint32_t hi = static_cast<uint32_t>(code[8 * j + 4 + b]) & 0xFu;
            v |= (lo | (hi << 4)) << (8 * b);
        }
        word[j] = v;
    }
    int high;
    const size_t off = w4_offset(r, static_cast<size_t>(cc) * 32, Kp / kBlockK, &high);
    *reinterpret_cast<uint4*>(out + off) = make_uint4(word[0], word[1], word[2], word[3]);
}

// K2 (prepack only): reference flat PackedInt4Buffer (ref tensor.hpp:43-64) -> tile layout.
__global__ void w4_prepack_flat_kernel(const uint8_t* __restrict__ flat, int N, int K, int Np,
                                       int Kp, uint8_t* __restrict__ out) {
    const size_t chunks_per_row = Kp / 32;
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<size_t>(Np) * chunks_per_row) return;
    const int r = static_cast<int>(idx / chunks_per_row);
    const int cc = static_cast<int>(idx % chunks_per_row);
    uint32_t nib[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) {
        const int k = cc * 32 + e;
        if (r < N && k < K) {
            const size_t i = static_cast<size_t>(r) * K + k;
            const uint8_t byte = flat[i / 2];
            nib[e] = (i % 2 == 0) ? (byte & 0xFu) : (byte >> 4);
        } else {
            nib[e] = 0;
        }
    }
    uint32_t word[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint32_t v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) v |= (nib[8 * j + b] | (nib[8 * j + 4 + b] << 4)) << (8 * b);
        word[j] = v;
    }
    int high;
    const size_t off = w4_offset(r, static_cast<size_t>(cc) * 32, Kp / kBlockK, &high);
    *reinterpret_cast<uint4*>(out + off) = make_uint4(word[0], word[1], word[2], word[3]);
}

__device__ __forceinline__ uint32_t w4_nibble(const uint8_t* __restrict__ packed, size_t i, int K,
                                              size_t kblocks) {
    const size_t r = i / K, k = i % K;
    int high;
    const size_t off = w4_offset(r, k, kblocks, &high);
    const uint8_t b = packed[off];
    return high ? (b >> 4) : (b & 0xFu);
}

// Tile layout -> reference flat PackedInt4Buffer bytes (odd tail high nibble 0).
__global__ void w4_unpack_flat_kernel(const uint8_t* __restrict__ packed, int N, int K, int Kp,
                                      uint8_t* __restrict__ flat) {
    const size_t count = static_cast<size_t>(N) * K;
    const size_t nbytes = (count + 1) / 2;
    const size_t b = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (b >= nbytes) return;
    const size_t kblocks = Kp / kBlockK;
    uint32_t lo = w4_nibble(packed, 2 * b, K, kblocks);
    uint32_t hi = (2 * b + 1 < count) ? w4_nibble(packed, 2 * b + 1, K, kblocks) : 0u;
    flat[b] = static_cast<uint8_t>(lo | (hi << 4));
}

// Dequantize weights: out[r][k] = code * S_r  (ref quantize.cpp:134-146).
__global__ void w4_dequant_kernel(const uint8_t* __restrict__ packed, const float* __restrict__ s,
                                  int N, int K, int Kp, float* __restrict__ out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<size_t>(N) * K) return;
    uint32_t nib = w4_nibble(packed, i, K, Kp / kBlockK);
    const int code = nib >= 8 ? static_cast<int>(nib) - 16 : static_cast<int>(nib);
    out[i] = static_cast<float>(code) * s[i / K];
}

// Activation codes -> row-major int8 (and optional dequantized f32).
__global__ void a8_unpack_kernel(const int8_t* __restrict__ q, const float* __restrict__ s, int M,
                                 int K, int Mp, int8_t* __restrict__ codes,
                                 float* __restrict__ deq) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<size_t>(M) * K) return;
    const size_t t = i / K, k = i % K;
    const int8_t c = q[a8_offset(t, k, Mp)];
    if (codes) codes[i] = c;
    if (deq) deq[i] = static_cast<float>(c) * s[t];
}

// Dequantizing epilogue on int32 accumulators (row-parallel TP: after the int32 SUM
// all-reduce of the K-sharded partial accumulators).  ref gemm.cpp:269-273.
__global__ void dequant_epilogue_kernel(const int32_t* __restrict__ acc, const float* __restrict__ sa,
                                        const float* __restrict__ sw, int M, int N, int out_dtype,
                                        void* __restrict__ out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<size_t>(M) * N) return;
    const int t = static_cast<int>(i / N), n = static_cast<int>(i % N);
    const float v = __fmul_rn(__int2float_rn(acc[i] >> 4), __fmul_rn(sa[t], sw[n]));
    if (out_dtype == kDtypeF32)
        static_cast<float*>(out)[i] = v;
    else if (out_dtype == kDtypeF16)
        static_cast<__half*>(out)[i] = __float2half_rn(v);
    else
        static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
}

// Row absmax only (for row-parallel TP: local max before the MAX all-reduce).
template <typename T>
__global__ void __launch_bounds__(kActThreads)
row_absmax_kernel(const T* __restrict__ x, size_t ldx, int K, float* __restrict__ out) {
    const T* row = x + static_cast<size_t>(blockIdx.x) * ldx;
    __shared__ float red[kActThreads / 32];
    float mx = 0.0f;
    for (int k0 = threadIdx.x * 16; k0 < K; k0 += kActThreads * 16) {
        float v[16];
        load16(row, k0, K, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) mx = fmaxf(mx, fabsf(v[i]));
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = red[0];
        for (int i = 1; i < kActThreads / 32; ++i) m = fmaxf(m, red[i]);
        out[blockIdx.x] = m;
    }
}

unsigned long long* g_act_trace = nullptr;  // diagnostics: [cta][entry, exit]

}  // namespace

void set_act_trace(unsigned long long* buf) { g_act_trace = buf; }

template <int NT, int MC>
cudaError_t launch_act_quant_cfg(cudaLaunchConfig_t& cfg, const void* x, int dtype, size_t ldx,
                                 int M, int K, int Kp, int Mp, int8_t* q, float* s,
                                 const float* absmax_in, float* absmax_out, int p) {
    cfg.blockDim = dim3(NT);
    switch (dtype) {
        case kDtypeF32:
            return cudaLaunchKernelEx(&cfg, act_quant_kernel<float, NT, MC>,
                                      static_cast<const float*>(x), ldx, M, K, Kp, Mp, q, s,
                                      absmax_in, absmax_out, p, g_act_trace);
        case kDtypeF16:
            return cudaLaunchKernelEx(&cfg, act_quant_kernel<__half, NT, MC>,
                                      static_cast<const __half*>(x), ldx, M, K, Kp, Mp, q, s,
                                      absmax_in, absmax_out, p, g_act_trace);
        case kDtypeBF16:
            return cudaLaunchKernelEx(&cfg, act_quant_kernel<__nv_bfloat16, NT, MC>,
                                      static_cast<const __nv_bfloat16*>(x), ldx, M, K, Kp, Mp, q,
                                      s, absmax_in, absmax_out, p, g_act_trace);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_act_quant_batch(int n, const void* const* x, const int* dtype, const size_t* ldx,
                                   const int* M, const int* K, int8_t* const* q, float* const* s, bool pdl,
                                   cudaStream_t st) {
    if (n < 1 || n > kActBatch) return cudaErrorInvalidValue;
    ActBatch b = {};
    int rows = 0, kmax = 0;
    for (int i = 0; i < n; ++i) {
        b.x[i] = x[i];
        b.ldx[i] = ldx[i];
        b.dtype[i] = dtype[i];
        b.M[i] = M[i];
        b.K[i] = K[i];
        b.q[i] = q[i];
        b.s[i] = s[i];
        rows += M[i];
        kmax = std::max(kmax, K[i]);
    }
    b.n = n;
    b.pdl = pdl ? 1 : 0;
    const int chunks = static_cast<int>(pad_k(kmax) / 16);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(rows);
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = pdl ? 1 : 0;
    // 256-thread CTAs (<= 16K registers, ~1 KiB smem): they stay co-resident with the decode
    // program kernel running before them, so the PDL chain program -> act quant -> program
    // lets the next program's CTAs start on every SM the previous one frees
    cfg.blockDim = dim3(256);
    if (chunks <= 512) return cudaLaunchKernelEx(&cfg, act_quant_batch_kernel<256, 2>, b);
    if (chunks <= 1024) return cudaLaunchKernelEx(&cfg, act_quant_batch_kernel<256, 4>, b);
    return cudaErrorInvalidValue;  // K > 16384: the per-linear act_quant handles it
}

cudaError_t launch_act_quant(const void* x, int dtype, size_t ldx, int M, int K, int8_t* q,
                             float* s, const float* absmax_in, float* absmax_out, bool pdl,
                             cudaStream_t st) {
    const int Kp = static_cast<int>(pad_k(K)), Mp = static_cast<int>(pad_m(M));
    const int chunks = Kp / 16;  // 16-element chunks per row, held in registers
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(M);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    const int p = pdl ? 1 : 0;
    if (chunks <= 128)
        return launch_act_quant_cfg<128, 1>(cfg, x, dtype, ldx, M, K, Kp, Mp, q, s, absmax_in,
                                            absmax_out, p);
    if (chunks <= 256)
        return launch_act_quant_cfg<256, 1>(cfg, x, dtype, ldx, M, K, Kp, Mp, q, s, absmax_in,
                                            absmax_out, p);
    if (chunks <= 512)
        return launch_act_quant_cfg<512, 1>(cfg, x, dtype, ldx, M, K, Kp, Mp, q, s, absmax_in,
                                            absmax_out, p);
    if (chunks <= 1024)
        return launch_act_quant_cfg<512, 2>(cfg, x, dtype, ldx, M, K, Kp, Mp, q, s, absmax_in,
                                            absmax_out, p);
    if (chunks <= 4096)
        return launch_act_quant_cfg<512, 8>(cfg, x, dtype, ldx, M, K, Kp, Mp, q, s, absmax_in,
                                            absmax_out, p);
    if (chunks <= 8192)
        return launch_act_quant_cfg<1024, 8>(cfg, x, dtype, ldx, M, K, Kp, Mp, q, s, absmax_in,
                                             absmax_out, p);
    return cudaErrorInvalidValue;  // K > 131072 (beyond the reference's 2^17 bound)
}

cudaError_t launch_row_absmax(const void* x, int dtype, size_t ldx, int M, int K, float* out,
                              cudaStream_t st) {
    switch (dtype) {
        case kDtypeF32:
            row_absmax_kernel<float><<<M, kActThreads, 0, st>>>(static_cast<const float*>(x), ldx,
                                                                K, out);
            break;
        case kDtypeF16:
            row_absmax_kernel<__half><<<M, kActThreads, 0, st>>>(static_cast<const __half*>(x),
                                                                 ldx, K, out);
            break;
        case kDtypeBF16:
            row_absmax_kernel<__nv_bfloat16><<<M, kActThreads, 0, st>>>(
                static_cast<const __nv_bfloat16*>(x), ldx, K, out);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_w4_quant_prepack(const float* w, int N, int K, int bits, const float* gamma,
                                    const float* beta, uint8_t* packed, float* s, int* err,
                                    cudaStream_t st, bool scales_given) {
    const int Np = static_cast<int>(pad_n(N)), Kp = static_cast<int>(pad_k(K));
    if (!scales_given) w_scale_kernel<<<(N + 7) / 8, 256, 0, st>>>(w, N, K, bits, gamma, beta, s, err);
    const size_t total = static_cast<size_t>(Np) * (Kp / 32);
    w4_quant_prepack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
        w, N, K, Np, Kp, s, packed);
    return cudaGetLastError();
}

cudaError_t launch_w_scale(const float* w, int N, int K, int bits, const float* gamma, const float* beta,
                           float* s, int* err, cudaStream_t st) {
    w_scale_kernel<<<(N + 7) / 8, 256, 0, st>>>(w, N, K, bits, gamma, beta, s, err);
    return cudaGetLastError();
}

size_t w8_bytes(size_t n, size_t k) { return pad_n(n) * pad_k(k); }

cudaError_t launch_w4_prepack_flat(const uint8_t* flat, int N, int K, uint8_t* packed,
                                   cudaStream_t st) {
    const int Np = static_cast<int>(pad_n(N)), Kp = static_cast<int>(pad_k(K));
    const size_t total = static_cast<size_t>(Np) * (Kp / 32);
    w4_prepack_flat_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
        flat, N, K, Np, Kp, packed);
    return cudaGetLastError();
}

cudaError_t launch_w4_unpack_flat(const uint8_t* packed, int N, int K, uint8_t* flat,
                                  cudaStream_t st) {
    const size_t nbytes = (static_cast<size_t>(N) * K + 1) / 2;
    w4_unpack_flat_kernel<<<static_cast<unsigned>((nbytes + 255) / 256), 256, 0, st>>>(
        packed, N, K, static_cast<int>(pad_k(K)), flat);
    return cudaGetLastError();
}

cudaError_t launch_w4_dequant(const uint8_t* packed, const float* s, int N, int K, float* out,
                              cudaStream_t st) {
    const size_t total = static_cast<size_t>(N) * K;
    w4_dequant_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
        packed, s, N, K, static_cast<int>(pad_k(K)), out);
    return cudaGetLastError();
}

cudaError_t launch_dequant_epilogue(const int32_t* acc, const float* sa, const float* sw, int M,
                                    int N, int out_dtype, void* out, cudaStream_t st) {
    const size_t total = static_cast<size_t>(M) * N;
    dequant_epilogue_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
        acc, sa, sw, M, N, out_dtype, out);
    return cudaGetLastError();
}

cudaError_t launch_a8_unpack(const int8_t* q, const float* s, int M, int K, int8_t* codes,
                             float* deq, cudaStream_t st) {
    const size_t total = static_cast<size_t>(M) * K;
    a8_unpack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(
        q, s, M, K, static_cast<int>(pad_m(M)), codes, deq);
    return cudaGetLastError();
}

}  // namespace odyb200
