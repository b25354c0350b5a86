/*
 * odyssey_b200.h -- C ABI of libodyssey_b200.so, the B200 (sm_100a) drop-in for the
 * reference's W4A8 FastGEMM hot path.
 *
 * Part 1 re-declares, with IDENTICAL names, signatures, status codes and ownership
 * rules, the hot-path subset of the reference ABI (/root/reference/proj/include/
 * odyssey/odyssey.h).  A program linked against libodyssey.so for these calls links
 * against libodyssey_b200.so unchanged; the work runs on the GPU, never on a CPU
 * fallback.  Each declaration cites the reference declaration it replaces.
 *
 * Part 2 is the device-pointer, stream-ordered API underneath (the "thin C-ABI
 * layer" of the north star): plain pointers, sizes and a cudaStream_t passed as
 * void*, no torch types.  Part 3 holds the parity/inspection accessors the
 * reference ABI lacks (ref odyssey.h:79-94 has no code/scale accessors).
 *
 * Conventions (ref odyssey.h:1-10): every call returns ody_status, ODY_OK == 0;
 * on failure ody_last_error() returns a thread-local message; handles are opaque
 * and released with their *_free function.
 */
#ifndef ODYSSEY_B200_H
#define ODYSSEY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ================================================================ part 1 */

/* ref odyssey.h:21-27 (+ ODY_EDEVICE: CUDA runtime / launch failure) */
typedef enum ody_status {
    ODY_OK = 0,
    ODY_EINVAL = 1,
    ODY_EIO = 2,
    ODY_EPARSE = 3,
    ODY_ENUMERIC = 4,
    ODY_EDEVICE = 5,
} ody_status;

/* ref odyssey.h:29-34 */
typedef enum ody_granularity {
    ODY_PER_TENSOR = 0,
    ODY_PER_CHANNEL = 1,
    ODY_PER_TOKEN = 2,
    ODY_PER_GROUP = 3,
} ody_granularity;

/* ref odyssey.h:36-42.  Every engine runs on the GPU (FAST: the FastGEMM kernels; the
 * comparison engines W8A8 / ASYMMETRIC / FINEGRAINED / W4A16: engine_kernel.cu), bit-exact
 * with the reference's gemm.cpp; there is never a CPU fallback. */
typedef enum ody_engine {
    ODY_ENGINE_W4A16 = 0,
    ODY_ENGINE_FINEGRAINED = 1,
    ODY_ENGINE_ASYMMETRIC = 2,
    ODY_ENGINE_FAST = 3,
    ODY_ENGINE_W8A8 = 4,
} ody_engine;

typedef struct ody_tensor ody_tensor;   /* ref odyssey.h:44 -- host row-major f32 */
typedef struct ody_qtensor ody_qtensor; /* ref odyssey.h:45 -- device-resident codes+scales */

/* ref odyssey.h:47-52 */
typedef struct ody_gemm_counters {
    uint64_t int8_mac_ops;
    uint64_t dequant_events;
    uint64_t zero_point_sub_ops;
    uint64_t final_scale_ops;
} ody_gemm_counters;

const char* ody_last_error(void);                 /* ref odyssey.h:55 */
void ody_string_free(char* s);                    /* ref odyssey.h:57 */
void ody_set_threads(int n);                      /* ref odyssey.h:61 -- here: the host threads
                                                   * of the ABI's host copies (<= 0: auto) */

ody_status ody_tensor_create(size_t rows, size_t cols, const float* data,
                             ody_tensor** out);   /* ref odyssey.h:65 */
/* Extension: the same from a row-strided host matrix (row r at data + r * ld), so a column
 * slice of a larger matrix needs no intermediate contiguous copy. */
ody_status ody_tensor_create_strided(size_t rows, size_t cols, size_t ld, const float* data,
                                     ody_tensor** out);
void ody_tensor_free(ody_tensor* t);              /* ref odyssey.h:66 */
ody_status ody_tensor_dims(const ody_tensor* t, size_t* rows, size_t* cols); /* :67 */
ody_status ody_tensor_data(const ody_tensor* t, const float** data);        /* :69 */

void ody_qtensor_free(ody_qtensor* q);                                        /* :79 */
ody_status ody_qtensor_dims(const ody_qtensor* q, size_t* rows, size_t* cols); /* :82 */

/* ref odyssey.h:87-89.  Hot path: bits == 4, ODY_PER_CHANNEL; also bits == 4
 * ODY_PER_GROUP (group_size | cols; the FINEGRAINED / W4A16 engines) and bits == 8
 * ODY_PER_CHANNEL (the W8A8 engine).  Optional per-row clip_gamma / clip_beta in (0,1].
 * Quantizes on the GPU straight into the kernels' layouts. */
ody_status ody_quantize_weights(const ody_tensor* w, int bits, ody_granularity granularity,
                                size_t group_size, const float* clip_gamma,
                                const float* clip_beta, ody_qtensor** out);

/* ref odyssey.h:92 -- dynamic symmetric per-token INT8, on the GPU. */
ody_status ody_quantize_activations(const ody_tensor* a, ody_qtensor** out);

/* ref odyssey.h:94 */
ody_status ody_dequantize(const ody_qtensor* q, ody_tensor** out);

/* ref odyssey.h:120-121 -- any engine (ref gemm.cpp:313-333 run_engine, same validation
 * order and counter formulas); returns a new host f32 tensor. */
ody_status ody_gemm(ody_engine engine, const ody_tensor* a_dense, const ody_qtensor* a_q,
                    const ody_qtensor* w_q, ody_gemm_counters* counters, ody_tensor** out);
/* ody_gemm on device memory, stream-ordered (no host copies, no synchronization): out_dev
 * (m x n f32, device) <- engine(a_q, w_q).  W4A16 takes device f32 activations a_dev
 * (a_rows x w cols) instead of a_q.  stream NULL = the library stream.  Calls share the
 * library's workspaces: order them on one stream. */
ody_status ody_gemm_dev(ody_engine engine, const float* a_dev, size_t a_rows, const ody_qtensor* a_q,
                        const ody_qtensor* w_q, float* out_dev, ody_gemm_counters* counters, void* stream);

/* Reference OTF files and float oracles (ref odyssey.h:71-75, 80-81, 100-101).
 * ody_qtensor_read builds the DEVICE qtensor straight from an `odyssey quantize` output
 * directory (payload.otf packed-i4 + scales.otf + scheme.txt, ref otf.cpp:121-202):
 * per-channel 4-bit weights are prepacked into the kernel layout, per-token 8-bit
 * activations into the a8 layout.  ody_optimize_clipping is the LWC grid search
 * (ref clip.cpp:55-103) run on the GPU, bit-exact.  ody_matmul_f32 is the reference's
 * fixed-order f32 matmul (its test oracle), on the GPU. */
ody_status ody_tensor_write(const ody_tensor* t, const char* path);          /* ref odyssey.h:71 */
ody_status ody_tensor_read(const char* path, ody_tensor** out);              /* :72 */
ody_status ody_matmul_f32(const ody_tensor* a, const ody_tensor* b_transposed, ody_tensor** out); /* :75 */
ody_status ody_qtensor_write(const ody_qtensor* q, const char* dir);         /* :80 */
ody_status ody_qtensor_read(const char* dir, ody_qtensor** out);             /* :81 */
ody_status ody_optimize_clipping(const ody_tensor* w, int bits, float grid_min, float grid_step,
                                 float* gamma, float* beta, float* mse_before, float* mse_after); /* :100 */

/* ================================================================ part 2 */

typedef enum ody_dtype { ODY_DTYPE_F32 = 0, ODY_DTYPE_F16 = 1, ODY_DTYPE_BF16 = 2 } ody_dtype;

/* Byte sizes of the device layouts (see paper_2311_09550_b200/csrc/layout.h). */
size_t ody_dev_a8_bytes(size_t m, size_t k);          /* per-token INT8 codes, k-block layout */
size_t ody_dev_w4_bytes(size_t n, size_t k);          /* prepacked INT4 tile layout */
size_t ody_dev_workspace_bytes(size_t m, size_t n, size_t k); /* stream-K partial sums */

/* K1 (replaces ref quantize.cpp:113-132): x is m x k row-major with row stride ldx
 * elements; q receives ody_dev_a8_bytes(m,k) bytes, s receives m f32 scales.
 * absmax_in (optional, m floats) overrides the row max -- row-parallel TP passes
 * the all-reduced global max of a K-sharded row.  absmax_out (optional) exports it. */
ody_status ody_dev_act_quant(const void* x, ody_dtype dtype, size_t ldx, size_t m, size_t k,
                             void* q, float* s, const float* absmax_in, float* absmax_out,
                             int pdl, void* stream);
/* Row max|x| only (the local half of the row-parallel scale all-reduce). */
ody_status ody_dev_row_absmax(const void* x, ody_dtype dtype, size_t ldx, size_t m, size_t k,
                              float* absmax, void* stream);

/* K2 (replaces ref quantize.cpp:75-111 per-channel, tensor.cpp:30-60 packing):
 * w is n x k f32 on the device; writes ody_dev_w4_bytes(n,k) bytes and n scales.
 * gamma/beta optional per-row device arrays. bits must be 4. */
ody_status ody_dev_w4_quantize(const float* w, size_t n, size_t k, const float* gamma,
                               const float* beta, void* w_packed, float* s_w, void* stream);
/* K2 with caller-supplied per-row scales (device array s_w, n floats): only the codes
 * clamp(round(w/s), -8, 7) are produced.  Row-parallel TP quantizes each K-shard with
 * the scale of the FULL row so the shards concatenate to the unsharded codes. */
ody_status ody_dev_w4_quantize_with_scales(const float* w, size_t n, size_t k, const float* s_w,
                                           void* w_packed, void* stream);
/* K4 alone: out = float(acc >> 4) * (s_a[i] * s_w[j]) from int32 accumulators (the
 * row-parallel TP epilogue after the bit-exact int32 SUM all-reduce). */
ody_status ody_dev_dequant_epilogue(const int32_t* acc, const float* s_a, const float* s_w,
                                    size_t m, size_t n, ody_dtype out_dtype, void* out,
                                    void* stream);
/* K2 prepack only: reference flat PackedInt4Buffer bytes ((n*k+1)/2, element 2i low
 * nibble) -> tile layout; and the inverse for export / parity. */
ody_status ody_dev_w4_prepack(const void* flat_nibbles, size_t n, size_t k, void* w_packed,
                              void* stream);
ody_status ody_dev_w4_unpack(const void* w_packed, size_t n, size_t k, void* flat_nibbles,
                             void* stream);

/* K3+K4 (replaces ref gemm.cpp:229-279): out[i][j] = float((sum a*16w) >> 4) * (sa*sw).
 * out (m x n row-major, out_dtype) and/or acc_out (m x n int32 pre-shift accumulators,
 * ref gemm_w4a8_fast_accumulators) may be NULL but not both.  workspace must hold
 * ody_dev_workspace_bytes(m,n,k) bytes, zeroed once (ody_dev_workspace_init); the
 * kernel leaves it zeroed.  max_ctas 0 = all SMs.  Requires k <= 2^17. */
ody_status ody_dev_w4a8_gemm(const void* q, const float* s_a, const void* w_packed,
                             const float* s_w, size_t m, size_t n, size_t k, ody_dtype out_dtype,
                             void* out, int32_t* acc_out, void* workspace,
                             size_t workspace_bytes, int max_ctas, int pdl, void* stream);
ody_status ody_dev_workspace_init(void* workspace, size_t bytes, void* stream);

/* K1+K3+K4: the whole W4A8 linear y = x W^T from unquantized activations x (m x k,
 * dtype x_dtype, row stride ldx).  For decode widths (m <= 16) the per-token INT8
 * quantization runs inside the GEMM kernel: each CTA of a thread-block cluster
 * quantizes its own k-slice, the cluster combines the per-token maxima through DSMEM
 * and reduce-scatters the int32 partial tiles through DSMEM -- one launch per linear;
 * otherwise act quant + GEMM.  Results are identical to
 * ody_dev_act_quant + ody_dev_w4a8_gemm.  s_a_out (optional, m floats) receives the
 * per-token scales.  workspace: ody_dev_linear_workspace_bytes(m,n,k), zeroed once. */
ody_status ody_dev_w4a8_linear(const void* x, ody_dtype x_dtype, size_t ldx, const void* w_packed,
                               const float* s_w, size_t m, size_t n, size_t k, ody_dtype out_dtype,
                               void* out, float* s_a_out, void* workspace, size_t workspace_bytes,
                               int max_ctas, int pdl, void* stream);
/* Same, plus a cross-kernel L2 prefetch hint: once this linear's own weight loads are
 * issued, its CTAs prefetch next_w[0, next_w_bytes) (the packed weights of the linear
 * the caller launches next) into L2, so HBM keeps streaming through the kernel boundary
 * and the next linear's activation prologue.  A pure hint: results never depend on it;
 * next_w may be NULL. */
ody_status ody_dev_w4a8_linear_pf(const void* x, ody_dtype x_dtype, size_t ldx, const void* w_packed,
                                  const float* s_w, size_t m, size_t n, size_t k, ody_dtype out_dtype,
                                  void* out, float* s_a_out, void* workspace, size_t workspace_bytes,
                                  int max_ctas, int pdl, const void* next_w, size_t next_w_bytes,
                                  void* stream);
size_t ody_dev_linear_workspace_bytes(size_t m, size_t n, size_t k);

/* A "linear program": up to 8 W4A8 linears run by ONE persistent kernel launch when every
 * linear is decode-width (m <= 16, 16-bit x): the weight stream never drains between
 * the linears, and a linear whose x is the output of an earlier linear of the program
 * (dep = that index; -1 = x is an external input) waits for it through grid-wide
 * completion counters in the workspace.  Otherwise the linears run one after another
 * (ody_dev_w4a8_linear each; stream order honours the deps).  Results are identical
 * to running ody_dev_w4a8_linear on each linear in order.  workspace:
 * ody_dev_program_workspace_bytes(lin, count) bytes, zeroed once (left zeroed). */
typedef struct ody_linear_desc {
    const void* x;           /* m x k, row stride ldx elements */
    ody_dtype x_dtype;
    size_t ldx;
    const void* w_packed;    /* ody_dev_w4_quantize / ody_dev_w4_prepack output */
    const float* s_w;
    size_t m, n, k;
    void* out;               /* m x n row-major */
    ody_dtype out_dtype;
    float* s_a_out;          /* optional: the m per-token scales */
    int dep;                 /* -1, or index < this one whose out is this x */
    const float* absmax_in;  /* optional (external x only): per-token row max overriding
                              * max|x| -- a row-parallel TP shard passes the all-reduced max */
    int32_t* acc_out;        /* optional: m x n int32 pre-shift accumulators written INSTEAD
                              * of out (out may then be NULL) -- the row-parallel TP partial
                              * that the int32 SUM all-reduce combines */
} ody_linear_desc;
size_t ody_dev_program_workspace_bytes(const ody_linear_desc* lin, int count);
ody_status ody_dev_w4a8_linear_program(const ody_linear_desc* lin, int count, void* workspace,
                                       size_t workspace_bytes, int max_ctas, int pdl,
                                       const void* next_w, size_t next_w_bytes, void* stream);
/* A dependency chain (deps set as for a program) run as ONE LAUNCH PER LINEAR: a dependent
 * linear's x is quantized from the per-token row maxima its producer launch's epilogues
 * accumulated (a reduction-free act quant spread over 4 CTAs per token row); external
 * linears keep the row-reducing act-quant kernel.  Eligible (ody_dev_chain_is_links) when every dependent
 * x is a column slice of its producer's 16-bit output and m <= 64; otherwise it runs as
 * ody_dev_w4a8_linear_program.  Results are identical to the program's.  Same workspace
 * (ody_dev_program_workspace_bytes, zeroed once, left zeroed). */
ody_status ody_dev_w4a8_linear_chain(const ody_linear_desc* lin, int count, void* workspace,
                                     size_t workspace_bytes, int max_ctas, int pdl, void* stream);
int ody_dev_chain_is_links(const ody_linear_desc* lin, int count);
/* 1 if ody_dev_w4a8_linear_program runs these linears as one kernel launch. */
int ody_dev_program_is_fused(const ody_linear_desc* lin, int count);
int ody_dev_linear_is_fused(size_t m, size_t n, size_t k); /* 1: single fused kernel */
/* Linear lowering: 0 = act-quant kernel + FastGEMM (PDL-chained); 1 = act quant fused
 * into the GEMM prologue (cluster code all-gather) where eligible; 2 (default) = the
 * cluster split-K decode kernel (K1 per k-slice + K3 + K4 in one launch) where eligible
 * (m <= 16, 16-bit x), else 0. */
void ody_dev_set_linear_mode(int mode);
/* FastGEMM kernel choice by width: m >= min_m (default 65; env ODY_PREFILL) runs the
 * 2-SM cta_group::2 prefill kernel (256 weight rows x 256 tokens per CTA pair), smaller m
 * the 1-SM tile GEMM.  0 disables the prefill kernel.  Results are identical either way. */
void ody_dev_set_prefill_min_m(int min_m);
/* Diagnostics: when buf (device, >= 8 * #CTAs u64) is non-NULL, subsequent
 * ody_dev_w4a8_gemm launches record a per-CTA %globaltimer timeline into it:
 * [entry, setup done, first data at MMA, last MMA commit, epilogue done, exit,
 *  producer done, units | segments << 32].  NULL disables (the default). */
void ody_dev_set_trace(void* buf);
/* Diagnostics: act-quant launches record [entry, exit] %globaltimer per CTA (NULL = off). */
void ody_dev_set_act_trace(void* buf);

/* Inspection: activation codes back to row-major int8 (and/or dequantized f32). */
ody_status ody_dev_a8_unpack(const void* q, const float* s, size_t m, size_t k, int8_t* codes,
                             float* dequant, void* stream);

/* ================================================================ part 3 */

/* Host copies of a qtensor's content in the REFERENCE layouts: activations and 8-bit
 * weights -> rows*cols int8 codes; 4-bit weights -> (n*k+1)/2 flat PackedInt4Buffer
 * bytes; plus scales (rows x groups per row). */
ody_status ody_qtensor_export(const ody_qtensor* q, void* codes_or_nibbles, float* scales);
/* Build a weight qtensor from reference-layout packed nibbles + scales (e.g. an OTF
 * payload.otf / scales.otf pair, ref otf.cpp:121-153). */
ody_status ody_qtensor_import_w4(size_t n, size_t k, const void* flat_nibbles,
                                 const float* scales, ody_qtensor** out);
/* Build an activation qtensor from reference-layout int8 codes + scales. */
ody_status ody_qtensor_import_a8(size_t m, size_t k, const int8_t* codes, const float* scales,
                                 ody_qtensor** out);
/* ref gemm.cpp:229-249: int32 accumulators before the >>4, m*n row-major. */
/* The scheme of a qtensor (the reference keeps it in QuantizedTensor::scheme, tensor.hpp:76-109):
 * bits 4/8, granularity (PER_TOKEN activations, PER_CHANNEL / PER_GROUP weights), group_size. */
ody_status ody_qtensor_scheme(const ody_qtensor* q, int* bits, ody_granularity* granularity, size_t* group_size);
ody_status ody_gemm_accumulators(const ody_qtensor* a_q, const ody_qtensor* w_q, int32_t* acc);
/* Library/device identification, e.g. "libodyssey_b200 sm_100a NVIDIA B200 (148 SMs)". */
const char* ody_b200_version(void);

/* ================================================================ part 4 */
/* Tensor parallelism (the paper's 70B runs).
 * ody_comm wraps an NCCL communicator (bound at run time from libnccl.so.2) over the
 * calling thread's current CUDA device; one rank per GPU.  Rank 0 makes the unique id
 * and the caller distributes its ODY_COMM_ID_BYTES bytes to every rank. */
#define ODY_COMM_ID_BYTES 128
typedef struct ody_comm ody_comm;
ody_status ody_comm_unique_id(void* id);
ody_status ody_comm_init(int nranks, int rank, const void* id, ody_comm** out);
ody_status ody_comm_free(ody_comm* comm);
ody_status ody_comm_dims(const ody_comm* comm, int* nranks, int* rank);

/* Megatron linear shards.  COLUMN: W split along N (this rank's n rows), x replicated,
 * out = this rank's [m, n] column block, no collective.  ROW: W and x split along K (this
 * rank's k_local columns; W quantized with the FULL rows' scales,
 * ody_dev_w4_quantize_with_scales): local row max -> all-reduce(MAX) -> K-shard FastGEMM
 * into int32 pre-shift partials -> all-reduce(SUM, int32: exact and order-free) -> K4, so
 * out ([m, n], replicated) is bit-identical to the unsharded linear.  Stream-ordered and
 * CUDA-graph capturable.  workspace: ody_tp_linear_workspace_bytes, zeroed once. */
typedef enum ody_tp_kind { ODY_TP_COLUMN = 0, ODY_TP_ROW = 1 } ody_tp_kind;
size_t ody_tp_linear_workspace_bytes(ody_tp_kind kind, size_t m, size_t n, size_t k_local);
ody_status ody_tp_linear(ody_comm* comm, ody_tp_kind kind, const void* x, ody_dtype x_dtype, size_t ldx,
                         const void* w_packed, const float* s_w, size_t m, size_t n, size_t k_local,
                         ody_dtype out_dtype, void* out, void* workspace, size_t workspace_bytes,
                         void* stream);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* ODYSSEY_B200_H */
