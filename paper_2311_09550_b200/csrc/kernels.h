// kernels.h -- launch entry points of the sm_100a kernels (internal C++ API used by
// the C-ABI layer in capi.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace odyb200 {

enum : int { kDtypeF32 = 0, kDtypeF16 = 1, kDtypeBF16 = 2 };

// K1: per-token INT8 quantization into the a8 k-block layout (layout.h).
cudaError_t launch_act_quant(const void* x, int dtype, size_t ldx, int M, int K, int8_t* q,
                             float* s, const float* absmax_in, float* absmax_out, bool pdl,
                             cudaStream_t st);
void set_act_trace(unsigned long long* buf);  // diagnostics: per-CTA entry/exit globaltimer
cudaError_t launch_row_absmax(const void* x, int dtype, size_t ldx, int M, int K, float* out,
                              cudaStream_t st);

// K2: per-channel INT4 quantization + prepack; flat-nibble prepack / unpack; dequant.
// scales_given: s already holds the per-row scales (row-parallel TP shards quantize
// with the scale of the FULL row), only the codes are produced.
cudaError_t launch_w4_quant_prepack(const float* w, int N, int K, int bits, const float* gamma,
                                    const float* beta, uint8_t* packed, float* s, int* err,
                                    cudaStream_t st, bool scales_given = false);
// int32 accumulators -> float(acc>>4)*(sa*sw) as f32/f16/bf16 (row-parallel TP epilogue).
cudaError_t launch_dequant_epilogue(const int32_t* acc, const float* sa, const float* sw, int M,
                                    int N, int out_dtype, void* out, cudaStream_t st);
cudaError_t launch_w4_prepack_flat(const uint8_t* flat, int N, int K, uint8_t* packed,
                                   cudaStream_t st);
cudaError_t launch_w4_unpack_flat(const uint8_t* packed, int N, int K, uint8_t* flat,
                                  cudaStream_t st);
cudaError_t launch_w4_dequant(const uint8_t* packed, const float* s, int N, int K, float* out,
                              cudaStream_t st);
cudaError_t launch_a8_unpack(const int8_t* q, const float* s, int M, int K, int8_t* codes,
                             float* deq, cudaStream_t st);

// K3+K4: FastGEMM with fused dequantizing epilogue.
struct GemmArgs {
    const int8_t* qa;     // a8 k-block layout, M x K
    const float* sa;      // M per-token scales
    const uint8_t* wp;    // w4 tile layout, N x K
    const float* sw;      // N per-channel scales
    void* out;            // M x N row-major, out_dtype (may be null if acc_out given)
    int out_dtype;
    int32_t* acc_out;     // optional: M x N pre-shift int32 accumulators (exactness suite)
    void* workspace;      // >= gemm_workspace_bytes(M,N,K), zero-initialised once
    size_t workspace_bytes;
    int M, N, K;
    int max_ctas;         // 0 = number of SMs
    bool pdl;             // programmatic dependent launch
    unsigned long long* trace;  // optional: 8 globaltimer slots per CTA (diagnostics)
};
size_t gemm_workspace_bytes(int M, int N, int K, int num_sms);
cudaError_t launch_w4a8_gemm(const GemmArgs& a, cudaStream_t st);

// The W4A8 linear y = x W^T end to end from unquantized activations: K1 fused into the
// GEMM (decode widths, one kernel) or act_quant + GEMM.  workspace: linear_scratch_bytes.
struct LinearArgs {
    const void* x;        // M x K, row stride ldx elements, dtype x_dtype
    int x_dtype;
    size_t ldx;
    const uint8_t* wp;    // w4 tile layout
    const float* sw;
    void* out;            // M x N row-major, out_dtype
    int out_dtype;
    float* sa_out;        // optional: the M per-token scales
    void* workspace;
    size_t workspace_bytes;
    int M, N, K;
    int max_ctas;
    bool pdl;
    unsigned long long* trace;
};
size_t linear_scratch_bytes(int M, int N, int K, int num_sms);
bool linear_is_fused(int M, int N, int K, int num_sms);
void set_linear_mode(int mode);  // 0: act_quant + GEMM (default); 1: K1 fused when eligible
cudaError_t launch_w4a8_linear(const LinearArgs& a, cudaStream_t st);

int device_sm_count();

}  // namespace odyb200
