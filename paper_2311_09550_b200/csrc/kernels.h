// kernels.h -- launch entry points of the sm_100a kernels (internal C++ API used by
// the C-ABI layer in capi.cu).
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

// Diagnostic / ablation switches read from the environment (ODY_DBG_*, ODY_PREFILL_*,
// ODY_DYN_*, ODY_PLAN_LOG, ...) exist only in a -DODY_DIAG build (make diag, used by
// tools/).  The product library never reads the environment, so a stray variable can
// neither change numerics nor inflate performance.
#ifdef ODY_DIAG
#define ODY_DIAG_ENV(name) std::getenv(name)
#else
#define ODY_DIAG_ENV(name) (static_cast<const char*>(nullptr))
#endif

namespace odyb200 {

enum : int { kDtypeF32 = 0, kDtypeF16 = 1, kDtypeBF16 = 2 };

// K1: per-token INT8 quantization into the a8 k-block layout (layout.h).
cudaError_t launch_act_quant(const void* x, int dtype, size_t ldx, int M, int K, int8_t* q,
                             float* s, const float* absmax_in, float* absmax_out, bool pdl,
                             cudaStream_t st);
void set_act_trace(unsigned long long* buf);
// K1 over up to 8 activation matrices in one launch (CTA per token row; K <= 16384).
cudaError_t launch_act_quant_batch(int n, const void* const* x, const int* dtype, const size_t* ldx,
                                   const int* M, const int* K, int8_t* const* q, float* const* s, bool pdl,
                                   cudaStream_t st);  // diagnostics: per-CTA entry/exit globaltimer
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
// Prefill widths (M >= 65, or ODY_PREFILL=<min M>; ODY_PREFILL=0 disables): the 2-SM
// cta_group::2 FastGEMM (prefill_kernel.cu).  launch_w4a8_gemm dispatches to it.
bool prefill_eligible(int M, int N, int K);
void set_prefill_min_m(int m);  // 0 disables
cudaError_t launch_w4a8_prefill(const GemmArgs& a, cudaStream_t st);
// Decode widths (M <= 64) on pre-quantized 128-row a8 activations: the dynamic decode
// kernel as a one-linear program (decode_kernel.cu).  scratch: gemm_prequant_scratch_bytes,
// its first program_zero_bytes() zeroed once (left zeroed).
bool gemm_prequant_eligible(int M, int N, int K);
size_t gemm_prequant_scratch_bytes(int M, int N, int K, int max_ctas);
cudaError_t launch_w4a8_gemm_prequant(const GemmArgs& a, void* scratch, size_t scratch_bytes, cudaStream_t st);

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
    const uint8_t* next_wp;  // optional L2 prefetch hint: the next linear's packed weights
    size_t next_bytes;
    unsigned long long* trace;
    const float* absmax_in;  // optional: per-token row max overriding max|x| (row-parallel TP)
    int32_t* acc_out;        // optional: M x N int32 pre-shift accumulators INSTEAD of out
};
size_t linear_scratch_bytes(int M, int N, int K, int num_sms);
bool linear_is_fused(int M, int N, int K, int num_sms);
// Linear lowering: 0 act_quant + GEMM; 1 K1 fused into the GEMM prologue (cluster code
// all-gather); 2 (default) the cluster split-K decode kernel when eligible, else 0.
void set_linear_mode(int mode);
int linear_mode();
cudaError_t launch_w4a8_linear(const LinearArgs& a, cudaStream_t st);

// Decode-width (M <= 16) linear as one kernel: fused K1 over each CTA's k-slice,
// cluster split-K, DSMEM reduce-scatter epilogue (decode_kernel.cu).
struct DecodePlan {
    int S, C, grid;  // cluster size, clusters, CTAs (S == 0: not eligible)
};
DecodePlan plan_decode(int M, int N, int K, int sms);
bool decode_eligible(int M, int N, int K, int x_dtype, int num_sms);
cudaError_t launch_w4a8_decode(const LinearArgs& a, cudaStream_t st);
// A "linear program": up to 8 decode-width linears in ONE persistent launch (the weight
// stream never drains between them).  deps[l] (or NULL: all -1) = index of an earlier
// linear whose output is linear l's x (quantized in-kernel after a grid-wide wait);
// external activations are quantized by one batched act-quant launch first.  scratch:
// program_scratch_bytes(), its first kProgramCounterRegion bytes zeroed once (the launch
// leaves them zeroed).  Of a[]'s launch fields only a[0].max_ctas and a[0].trace are used.
constexpr int kProgramMaxLinears = 8;
constexpr size_t kProgramCounterRegion = 4096 + 65536;  // counters + chain done/absmax (decode_kernel.cu)
constexpr size_t kProgramMaxTiles = 1024;  // 128-row weight tiles per program (8 MiB of split-K sums)
constexpr size_t kLinearGemmCounters = 4096;  // == the GEMM workspace's counter region
// Bytes at the start of a program scratch that must stay zero (counters, accumulators);
// shape-independent, so one scratch buffer can serve programs/linears of any shape.
size_t program_zero_bytes();
DecodePlan plan_program(const LinearArgs* a, const int* deps, int L, int sms);
bool program_eligible(const LinearArgs* a, const int* deps, int L, int num_sms);
size_t program_scratch_bytes(const LinearArgs* a, const int* deps, int L);
// A dependency chain as one launch per linear (decode_kernel.cu "chain links"): dependent
// linears quantize their x in-kernel from the row maxima their producer launch's
// epilogues accumulated.  Same scratch as launch_w4a8_program.
bool chain_links_eligible(const LinearArgs* a, const int* deps, int L);
cudaError_t launch_w4a8_chain_links(const LinearArgs* a, const int* deps, int L, void* scratch,
                                    size_t scratch_bytes, bool pdl, cudaStream_t st);
cudaError_t launch_w4a8_program(const LinearArgs* a, const int* deps, int L, void* scratch, size_t scratch_bytes,
                                bool pdl, const uint8_t* next_wp, size_t next_bytes, cudaStream_t st);

int device_sm_count();

// engine_kernel.cu: the reference's comparison engines (ref gemm.cpp:100-311) on tcgen05.
enum : int { kEngineFast = 0, kEngineAsym = 1, kEngineW8A8 = 2, kEngineFine = 3 };
struct EngineArgs {
    int mode;
    const uint8_t* w;     // W4 tile layout (FAST/FINE), its UINT4+8 twin (ASYM), W8 layout (W8A8)
    const float* sw;      // [N], or [N][K/group] (FINE)
    const int8_t* qa;     // a8 k-block layout
    const float* sa;
    float* out;           // M x N f32 row-major
    int M, N, K;
    int group;            // FINE: group size (multiple of 32, divides K)
    void* workspace;      // engine_workspace_bytes, zeroed once (left zeroed)
    size_t workspace_bytes;
};
int engine_splits(int mode, int M, int N, int K);
size_t engine_workspace_bytes(int mode, int M, int N, int K);
cudaError_t launch_engine_gemm(const EngineArgs& a, cudaStream_t st);
// per-row symmetric scale (ref quantize.cpp:22-35), bits 4 or 8; err set on bad gamma/beta
cudaError_t launch_w_scale(const float* w, int N, int K, int bits, const float* gamma, const float* beta,
                           float* s, int* err, cudaStream_t st);
// per-group INT4 weights (scales [N][K/g]) into the W4 tile layout
cudaError_t launch_wg_quant_prepack(const float* w, int N, int K, int g, int bits, const float* gamma,
                                    const float* beta, uint8_t* packed, float* s, cudaStream_t st);
// per-channel INT8 weights into the W8 layout (a8 k-block layout over the padded rows)
size_t w8_bytes(size_t n, size_t k);
cudaError_t launch_w8_quant(const float* w, int N, int K, const float* gamma, const float* beta, int8_t* codes,
                            float* s, int* err, cudaStream_t st);
cudaError_t launch_w4_offset(const uint8_t* packed, int N, int K, uint8_t* out, cudaStream_t st);
// FINEGRAINED with g % 32 != 0: W4 tiles and a8 codes re-laid out over K' = (K/g)*ceil32(g)
cudaError_t launch_regroup(const uint8_t* w4, const int8_t* qa, int M, int N, int K, int g, uint8_t* w4_out,
                           int8_t* qa_out, cudaStream_t st);
cudaError_t launch_wg_dequant(const uint8_t* packed, const float* s, int N, int K, int g, float* out,
                              cudaStream_t st);
cudaError_t launch_w4a16(const float* a, const uint8_t* packed, const float* s, int M, int N, int K, int g,
                         float* out, cudaStream_t st);

// aux_kernels.cu: the reference's offline / float-oracle numerics, bit-exact.
// LWC grid search (ref clip.cpp:55-103): w is N x K f32 on the device; per-row outputs.
int lwc_max_candidates();
cudaError_t launch_lwc_grid(const float* w, int N, int K, int bits, float grid_min, float grid_step, float* gamma,
                            float* beta, float* mse_before, float* mse_after, cudaStream_t st);
// matmul_f32 (ref tensor.cpp:176-196): out = a (M x K) . bt (N x K)^T, sequential f32 dots.
cudaError_t launch_matmul_f32(const float* a, const float* bt, int M, int N, int K, float* out, cudaStream_t st);

}  // namespace odyb200
