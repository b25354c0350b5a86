// decode_kernel.cu -- decode-width (M <= 16) W4A8 linears as ONE persistent kernel: a
// "linear program" of up to kMaxLin linears y_l = x_l W_l^T, each with per-token INT8
// activation quantization (K1), the FastGEMM mainloop (K3) and the dequantizing
// epilogue (K4), from unquantized fp16/bf16 activations.  A single linear is a program
// of length 1 (ody_dev_w4a8_linear).
//
// Reference semantics (bit-exact):
//   S_t   = max_k |x[t,k]| / 127   (0 -> 2^-24)          ref quantize.cpp:22-35, 113-132
//   q     = clamp(roundf(x / S_t), -128, 127)             ref quantize.cpp:12-18, 44
//   acc16 = sum_k q[t,k] * (16 * w[n,k])                  ref gemm.cpp:229-249 (high-nibble lanes)
//   y     = float(acc16 >> 4) * (S_t * S_w[n])            ref gemm.cpp:251-279
//
// Partition ("cluster split-K"): the grid is C clusters of S CTAs (S uniform over the
// program).  For linear l, cluster c owns the 128-row weight tiles v, v+C, v+2C, ...
// (v = (c + rot_l) mod C: independent linears rotate, so the program's tiles spread
// evenly over the clusters); rank r owns k-blocks [r*kb/S, (r+1)*kb/S) of every tile.
//   * a CTA needs only its own k-slice of x_l: it loads x[:, slice], takes the per-token
//     partial max|x|, exchanges the S partial maxima over DSMEM (st.async -> the peers'
//     mbarrier) and quantizes its slice straight into a resident, MMA-ready smem B;
//   * the S int32 partial tiles are reduced by a DSMEM reduce-scatter: rank j owns rows
//     [j*R, (j+1)*R) of each tile, the other ranks st.async those rows to it, and it adds
//     them (integer addition: exact in any order) and runs the epilogue on its rows.
// The weight stream never waits for activations: the producer walks the WHOLE program's
// weight units from the first instruction (no griddepcontrol.wait on that path), with an
// L2 prefetch window ahead of the smem ring, so HBM keeps streaming through every
// linear's activation prologue and epilogue tail.  A linear whose x is the output of an
// earlier linear of the program (dep >= 0) waits for that linear's grid-wide completion
// counter before loading x; the counters reset themselves at the end of the launch.
//
// Warp roles (12 warps, one CTA per SM; 168 registers per thread):
//   0      producer: 1-D bulk copies (UBLKCP) of 16 KiB packed-INT4 weight units and of
//          the per-tile channel scales
//   1      MMA: tcgen05.mma.cta_group::1.kind::i8, A (widened weights) from TMEM,
//          B (resident activation codes) from smem, int32 D in TMEM (double-buffered)
//   2      TMEM allocator; warps 2..11: the activation-quantization prologue of each linear
//   4..7   converters (one warp per TMEM sub-partition): smem packed INT4 ->
//          (w<<4)&0xF0F0F0F0 / w&0xF0F0F0F0 int8 lanes (the paper's SINT4->S8 trick) ->
//          tcgen05.st
//   8..11  epilogue: tcgen05.ld D -> DSMEM reduce-scatter -> >>4, scale, store
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "kernels.h"
#include "layout.h"
#include "ptx.cuh"
#include "quant_common.cuh"

namespace odyb200 {

namespace {

constexpr int kThreads = 384;
constexpr int kWarpProducer = 0;
constexpr int kWarpMma = 1;
constexpr int kWarpAlloc = 2;
constexpr int kWarpConv0 = 4;
constexpr int kConvGroups = 1;
constexpr int kWarpEpi0 = 8;
constexpr int kBN = 16;                 // tokens per tile (MMA N); decode widths M <= 16
constexpr int kUnitBlocks = 2;          // k-blocks per pipeline unit (16 KiB of weights)
constexpr int kUnitBytes = kUnitBlocks * kWBlockBytes;
constexpr int kBN_ = 16;
constexpr int kStageBytes = kUnitBytes + kUnitBlocks * kBN_ * 128;  // weights + pre-quantized B tiles
constexpr int kAStages = 4;             // TMEM A stages (64 columns each)
constexpr int kAStageCols = kUnitBlocks * kBlockK / 4;
constexpr int kAColBase = 256;
constexpr int kDBufs = 4;               // TMEM accumulator buffers (tiles in flight to the epilogue)
constexpr int kTmemCols = 512;
constexpr int kMaxSplit = 8;            // portable cluster size
constexpr int kMaxKbPerCta = 28;        // resident B: 28 k-blocks x 16 tokens x 128 B = 56 KiB
constexpr int kBBlockBytes = kBN * 128;
constexpr int kResBBytes = kMaxKbPerCta * kBBlockBytes;
constexpr int kQThreads = 320;          // warps 2..11 quantize the activations
constexpr int kQHold = 3;              // 16-element activation chunks held per thread per batch
constexpr int kStages = 7;
constexpr int kMaxLin = 8;
constexpr int kSmemBytes = kStages * kStageBytes + kResBBytes + 16 /*finalise flag*/ +
                           kMaxSplit * kBN * 4 /*peer maxima*/ + 3 * kBN * 4 /*max, scale, rcp*/ +
                           1024 /*barriers*/ + 1024 /*alignment*/;
static_assert(kSmemBytes <= 227 * 1024, "smem budget");
static_assert(kAColBase + kAStages * kAStageCols <= kTmemCols, "TMEM budget");
static_assert(4 * 16 <= 256, "D buffers below the A stages");
// kind::i8, D=s32, A=B=s8 signed, K-major both, N=16, M=128
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) |
                            (static_cast<uint32_t>(kBN >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
constexpr int kAmaxStride = 32;  // u32: per-token row maxima one 128-byte line apart
constexpr int kTraceCta = 32;  // [entry, setup, -, -, -, exit, producer done, meta, per linear 4 x 6]

struct LinDesc {
    const void* x;        // M x K, row stride ldx elements, f16 or bf16
    size_t ldx;
    const uint8_t* wp;    // w4 tile layout
    const float* sw;
    void* out;            // M x N row-major
    float* sa_out;        // optional per-token scales
    int x_bf16, out_dtype;
    int M, N, K, kblocks, n_tiles;
    const int8_t* qa;     // pre-quantized activations (a8 k-block layout, Mp rows) or NULL:
    const float* sa;      //   then B tiles ride in the ring stages and no prologue runs
    int Mp;
    int dep;              // x is the output of linear `dep` of this program (-1: external)
    int signal;           // a later linear depends on this one: publish its completion
    int rot;              // tile rotation (independent linears spread over the clusters)
    // dynamic schedule (w4a8_decode_dyn_kernel): work items = (tile, k-split) pairs
    int split;            // k-splits per tile (tiles [0, t1))
    int t1, split2;       // tiles [t1, n_tiles): the last partial wave, split2 k-splits each
    int items;            // work items of this linear: t1 * split + (n_tiles - t1) * split2
    int off;              // static chain schedule: CTA of this linear's item 0
    int ibase;            // first work item of this linear
    int tbase;            // first tile of this linear in the program's tile numbering
    // dynamic-schedule dependency chain (w4a8_decode_dyn_kernel)
    int32_t* acc_out;     // optional: final int32 pre-shift accumulators (M x N) INSTEAD of out
    uint32_t* done;       // items of this linear finished (a later linear depends on it), or NULL
    uint32_t* amax_dst;   // per-token max |y| (f32 bits) over the output columns [amax_c0, amax_c1)
    int amax_c0, amax_c1; //   that the dependent linear reads as its x
    const uint32_t* dep_done;  // dependent linear: its producer's `done`, complete at dep_target
    uint32_t dep_target;
    const uint32_t* amax_src;  // dependent linear: per-token max |x| (its producer's amax_dst)
    uint32_t* qdone;      // dependent linear: k-blocks of x quantized into qa (grid-wide), or NULL
    uint32_t qtarget;     //   complete at kblocks
    uint32_t* amax_reset; // row maxima this launch's last CTA re-zeroes (the chain program: its
                          // amax_dst; a chain link launch: the amax_src its x was quantized with)
    uint32_t* amax_zero;  // chain link: the row maxima its act quant consumed, re-zeroed by CTA 0
                          // once griddepcontrol.wait returned (the act quant completed)
};

constexpr int kRowThreads = 1024;  // one 16-element chunk per thread: the row quantizes in one pass
constexpr int kRowChunks = 1;  // K <= 1024 * 16 = 16384
struct RowBatch {
    const unsigned short* x[kMaxLin];
    size_t ldx[kMaxLin];
    int M[kMaxLin], K[kMaxLin], Mp[kMaxLin], bf16[kMaxLin];
    int8_t* q[kMaxLin];
    float* s[kMaxLin];
    const float* amax_in[kMaxLin];  // optional row max override (row-parallel TP: all-reduced max)
    int n, pdl;
    unsigned long long* trace;  // diagnostics: [cta][entry, griddepcontrol.wait returned, done, -]
    const uint32_t* amax_src[kMaxLin];  // act_quant_premax_kernel: the producer's per-token maxima
};

struct PParams {
    LinDesc lin[kMaxLin];
    int L;
    int S, C;             // cluster size (split-K factor), clusters
    uint32_t* ctr;        // [kMaxLin] completion counters + [kMaxLin] exit counter (zeroed)
    int32_t* acc;         // [program tiles][BN][128] split-K accumulators in L2 (zeroed)
    int32_t* part;        // dynamic schedule: [items][BN][128] split partials (scratch)
    int n_items;          // dynamic schedule: work items of the whole program
    uint32_t* work;       // dynamic schedule: next-item counter (zeroed; reset by the last CTA)
    int reset_at_exit;    // the last CTA out re-arms the work counter / chain state (else
                          // nothing to re-arm: static deal, no chain state)
    int chain_static;     // dependency chain: items dealt round-robin over the CTAs in program
                          // order (CTA c: items c - off, + C, ... of each linear), no counter
    uint32_t* tile_cnt;   // [program tiles] split arrivals (zeroed)
    int pdl;
    int pf_units;         // L2 prefetch window past the smem ring (units)
    int no_item_pf;       // a dependent item does not L2-prefetch its weights while x is quantized
    int rest_pf;          // a CTA whose ring filled before griddepcontrol.wait L2-prefetches the
                          // rest of its first item
    const uint8_t* next_wp;  // cross-kernel hint: L2-prefetch this slice of the next weights
    size_t next_bytes;
    int dbg;              // diagnostics (ODY_DBG_DECODE): 1 store raw x (no quant math), 2 no IEEE redo
    unsigned long long* trace;
};

// A value the compiler must keep in a register (a volatile move cannot be rematerialised
// from the kernel parameters).
__device__ __forceinline__ int ld_keep(int v) {
    int r;
    asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
    return r;
}
__device__ __forceinline__ void stg_b16(void* p, unsigned short v) {
    asm volatile("st.global.b16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}
__device__ __forceinline__ void stg_b32(void* p, uint32_t v) {
    asm volatile("st.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// The same stores with no compiler memory barrier (the epilogue's independent per-token
// stores may interleave with the next token's arithmetic).
__device__ __forceinline__ void stg_b16_free(void* p, unsigned short v) {
    asm("st.global.b16 [%0], %1;" ::"l"(p), "h"(v));
}
__device__ __forceinline__ void stg_b32_free(void* p, uint32_t v) {
    asm("st.global.b32 [%0], %1;" ::"l"(p), "r"(v));
}
template <typename T>
__device__ __forceinline__ T* ld_keep_ptr(T* v) {
    unsigned long long r;
    asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(reinterpret_cast<unsigned long long>(v)));
    return reinterpret_cast<T*>(r);
}

__device__ __forceinline__ uint64_t b_desc(uint32_t smem_addr) {
    // K-major SWIZZLE_128B: start>>4, SBO = 1024 B (8 rows x 128 B), version 1, swizzle 128B.
    return static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(64) << 32) |
           (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}

// ---- DSMEM helpers local to this kernel ----
__device__ __forceinline__ void st_async_u32(uint32_t remote_addr, uint32_t v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];"
                 ::"r"(remote_addr), "r"(v), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, uint32_t a, uint32_t b, uint32_t c,
                                            uint32_t d, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];"
                 ::"r"(remote_addr), "r"(a), "r"(b), "r"(c), "r"(d), "r"(remote_bar)
                 : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ float half_bits_to_f32(uint32_t w, int hi, bool bf16) {
    const unsigned short h = hi ? static_cast<unsigned short>(w >> 16) : static_cast<unsigned short>(w);
    return bf16 ? __uint_as_float(static_cast<uint32_t>(h) << 16) : __half2float(__ushort_as_half(h));
}

// Elements whose fast quotient lies within 6e-5 of a half-integer (flag bit e) are
// recomputed with the reference's IEEE division and roundf (ref quantize.cpp:44).
// Rare (~1e-4 of elements): kept out of line, and only the flagged bytes are redone.
// Out-of-line slow path of quant16 (a lane of the chunk is within 7e-5 of a half-integer,
// ~1e-4 of elements, or 1/S overflowed): find those lanes and redo them with the
// reference's IEEE division and roundf (ref quantize.cpp:12-18, 44).
__device__ __noinline__ uint4 fix16(uint4 q, uint4 r0, uint4 r1, float scale, float rcp, bool bf16) {
    uint32_t o[4] = {q.x, q.y, q.z, q.w};
    const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    const bool all = !(rcp < INFINITY);
    for (int e = 0; e < 16; ++e) {
        const float x = half_bits_to_f32(w[e >> 1], e & 1, bf16);
        const uint32_t byte = (o[e >> 2] >> (8 * (e & 3))) & 0xFFu;
        const float r = static_cast<float>(static_cast<int8_t>(byte));
        if (!all && fabsf(__fmaf_rn(x, rcp, -r)) < 0.49993f) continue;
        const int32_t code = clamp_code(x / scale, -128, 127);
        const int sh = 8 * (e & 3);
        o[e >> 2] = (o[e >> 2] & ~(0xFFu << sh)) | ((static_cast<uint32_t>(code) & 0xFFu) << sh);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

struct uint4x2 {
    uint4 a, b;
};

// ---- packed f32x2 arithmetic (FFMA2 / FADD2 on sm_100) ----
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void upk2(unsigned long long v, uint32_t& a, uint32_t& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(v));
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long fsub2(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

template <bool BF16>
__device__ __forceinline__ void unpack2(uint32_t w, float& lo, float& hi) {
    if (BF16) {
        lo = __uint_as_float(w << 16);
        hi = __uint_as_float(w & 0xFFFF0000u);
    } else {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w));
        lo = f.x;
        hi = f.y;
    }
}

// 16 packed 16-bit values -> 16 INT8 codes, bit-exact with clamp(roundf(fl(x / S))):
//   t = RN(x*rcp + 1.5*2^23)   rounds the EXACT product x*rcp to an integer r (low byte of
//                              t = r, two's complement; |x*rcp| <= 127.0001 needs no clamp)
//   d = RN(x*rcp - r)          its distance to r, accurate to 2^-25
// |x*rcp - x/S| <= |x/S| * 2^-24 < 7.6e-6 and |fl(x/S) - x/S| < 7.6e-6, so whenever
// |d| < 0.49993 both the exact and the reference's rounded quotient round to r.  The
// check d*d - 0.49993^2 < 0 is folded over all 16 lanes with sign-bit ANDs; a chunk with
// any lane at or past the threshold (~1e-4 of elements) is redone element by element
// through the IEEE division (fix16).  Two lanes per instruction: ~4.3 ops per element.
// The fast path alone; `ok` false: the chunk must be redone by fix16 (callers that
// quantize several chunks per thread run every fast path first, then the rare fix-ups,
// so the chunks' independent arithmetic interleaves -- an out-of-line call inside each
// chunk serialises them: measured ~0.15-0.25 us per chunk for a lone warp).
template <bool BF16>
__device__ __forceinline__ uint4 quant16_fast(uint4 r0, uint4 r1, float rcp, bool& ok) {
    const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    const unsigned long long RCP = pk2(rcp, rcp);
    const unsigned long long MAGIC = pk2(12582912.0f, 12582912.0f);
    const unsigned long long THR = pk2(-0.2499300049f, -0.2499300049f);  // -(0.49993^2)
    uint32_t t[16];
    uint32_t sign_and = 0xFFFFFFFFu;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float lo, hi;
        unpack2<BF16>(w[i], lo, hi);
        const unsigned long long X = pk2(lo, hi);
        const unsigned long long T = ffma2(X, RCP, MAGIC);
        const unsigned long long NR = fsub2(MAGIC, T);     // -r
        const unsigned long long D = ffma2(X, RCP, NR);    // x*rcp - r
        const unsigned long long U = ffma2(D, D, THR);     // d^2 - 0.49993^2 (< 0: safe)
        upk2(T, t[2 * i], t[2 * i + 1]);
        uint32_t u0, u1;
        upk2(U, u0, u1);
        sign_and &= u0 & u1;
    }
    ok = (sign_and >> 31) && rcp < INFINITY;
    return make_uint4(pack4_low_bytes(t[0], t[1], t[2], t[3]), pack4_low_bytes(t[4], t[5], t[6], t[7]),
                      pack4_low_bytes(t[8], t[9], t[10], t[11]), pack4_low_bytes(t[12], t[13], t[14], t[15]));
}
template <bool BF16>
__device__ __forceinline__ uint4 quant16(uint4 r0, uint4 r1, float scale, float rcp, int dbg) {
    bool ok;
    const uint4 q = quant16_fast<BF16>(r0, r1, rcp, ok);
    if (dbg != 2 && !ok) return fix16(q, r0, r1, scale, rcp, BF16);
    return q;
}

// Largest |x| bit pattern of 16 packed 16-bit floats as f32 bits (non-negative floats
// order like their bits; NaN stays NaN): sign-masked 16-bit magnitudes, packed max.
template <bool BF16>
__device__ __forceinline__ uint32_t absmax16_bits(uint4 r0, uint4 r1) {
    uint32_t m2 = __vmaxu2(__vmaxu2(r0.x & 0x7FFF7FFFu, r0.y & 0x7FFF7FFFu),
                           __vmaxu2(r0.z & 0x7FFF7FFFu, r0.w & 0x7FFF7FFFu));
    m2 = __vmaxu2(m2, __vmaxu2(__vmaxu2(r1.x & 0x7FFF7FFFu, r1.y & 0x7FFF7FFFu),
                               __vmaxu2(r1.z & 0x7FFF7FFFu, r1.w & 0x7FFF7FFFu)));
    const uint32_t m = max(m2 & 0xFFFFu, m2 >> 16);
    return BF16 ? (m << 16) : __float_as_uint(__half2float(__ushort_as_half(static_cast<unsigned short>(m))));
}

// Row tail (k0 + 16 > K): element loads, zero past K.  Out of line: it runs for at most
// one chunk per token row and would otherwise be inlined into every unrolled chunk.
__device__ __noinline__ uint4x2 load16_tail(const unsigned short* row, int k0, int K) {
    uint32_t h[8];
    for (int i = 0; i < 8; ++i) {
        const uint32_t lo = k0 + 2 * i < K ? row[k0 + 2 * i] : 0u;
        const uint32_t hi = k0 + 2 * i + 1 < K ? row[k0 + 2 * i + 1] : 0u;
        h[i] = lo | (hi << 16);
    }
    return {make_uint4(h[0], h[1], h[2], h[3]), make_uint4(h[4], h[5], h[6], h[7])};
}

__device__ __forceinline__ void load16_raw(const unsigned short* row, int k0, int K, bool cg, uint4& r0,
                                           uint4& r1) {
    if (k0 + 16 <= K) {
        const uint4* src = reinterpret_cast<const uint4*>(row + k0);
        if (cg) {  // x written earlier in this launch by other CTAs: coherent L2 loads
            r0 = __ldcg(src);
            r1 = __ldcg(src + 1);
        } else {
            r0 = __ldg(src);
            r1 = __ldg(src + 1);
        }
    } else {
        const uint4x2 v = load16_tail(row, k0, K);
        r0 = v.a;
        r1 = v.b;
    }
}

// Shared-memory carve-up of one CTA.
struct Smem {
    uint8_t* ring;
    uint8_t* resb;
    float* swr;          // [4]: the epilogue's "this CTA finalises the tile" broadcast
    uint32_t* peer_max;  // [kMaxSplit][BN] partial maxima pushed by the cluster peers
    uint32_t* tmax;      // [BN] this CTA's partial maxima
    float* tscale;       // [BN]
    float* trcp;         // [BN]
    uint64_t *w_full, *w_empty, *b_full, *a_full, *a_empty, *d_full, *d_empty, *b_ready, *max_full;
    uint32_t* tmem_slot;
};

__device__ __forceinline__ Smem carve(uint8_t* smem) {
    Smem m;
    m.ring = smem;
    m.resb = m.ring + kStages * kStageBytes;
    m.swr = reinterpret_cast<float*>(m.resb + kResBBytes);
    m.peer_max = reinterpret_cast<uint32_t*>(m.swr + 4);
    m.tmax = m.peer_max + kMaxSplit * kBN;
    m.tscale = reinterpret_cast<float*>(m.tmax + kBN);
    m.trcp = m.tscale + kBN;
    uint64_t* bars = reinterpret_cast<uint64_t*>(m.trcp + kBN);
    m.w_full = bars;
    m.w_empty = m.w_full + kStages;
    m.b_full = m.w_empty + kStages;
    m.a_full = m.b_full + kStages;
    m.a_empty = m.a_full + kAStages;
    m.d_full = m.a_empty + kAStages;
    m.d_empty = m.d_full + kDBufs;
    m.b_ready = m.d_empty + kDBufs;
    m.max_full = m.b_ready + 1;
    m.tmem_slot = reinterpret_cast<uint32_t*>(m.max_full + 1);
    return m;
}

// Geometry of linear l for this CTA: k-slice, tiles, pipeline units.
struct LGeo {
    int kb_lo, kb_hi, nkb, upt, ntiles, units, vcl, C;
    __device__ __forceinline__ int tile(int i) const { return vcl + i * C; }
    __device__ __forceinline__ int unit_kb(int k) const { return kb_lo + kUnitBlocks * (k % upt); }
    __device__ __forceinline__ int unit_nb(int k) const { return min(kUnitBlocks, kb_hi - unit_kb(k)); }
};
__device__ __forceinline__ LGeo lgeo(const PParams& p, int l, int crank, int cl) {
    const LinDesc& d = p.lin[l];
    LGeo g;
    g.kb_lo = crank * d.kblocks / p.S;
    g.kb_hi = (crank + 1) * d.kblocks / p.S;
    g.nkb = g.kb_hi - g.kb_lo;
    g.upt = (g.nkb + kUnitBlocks - 1) / kUnitBlocks;
    g.C = p.C;
    g.vcl = (cl + d.rot) % p.C;
    g.ntiles = g.vcl < d.n_tiles ? (d.n_tiles - 1 - g.vcl) / p.C + 1 : 0;
    g.units = g.ntiles * g.upt;
    return g;
}

// Converter warp q of one group widens global unit u (nb k-blocks): smem packed INT4 ->
// int8 lanes (value*16) -> TMEM A stage.  The ring stage is handed back once read.
__device__ __forceinline__ void convert_unit(const Smem& m, uint32_t tmem, int q, int lane, int u, int nb,
                                             unsigned long long* utr) {
    const int r = 32 * q + lane;
    const int s = u % kStages;
    const int as = u % kAStages;
    mbar_wait(&m.w_full[s], (u / kStages) & 1);
    if (utr && u < 64 && r == 0) utr[8 * u] = clock64();
    const uint32_t src = smem_u32(m.ring) + s * kStageBytes + r * 16;
    uint32_t lanes8[kUnitBlocks][32];
#pragma unroll
    for (int b = 0; b < kUnitBlocks; ++b) {
        if (b < nb) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint4 v = lds128(src + b * kWBlockBytes + c * 2048);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    lanes8[b][c * 8 + 2 * jj] = (w[jj] << 4) & 0xF0F0F0F0u;  // k 8jj+0..3
                    lanes8[b][c * 8 + 2 * jj + 1] = w[jj] & 0xF0F0F0F0u;     // k 8jj+4..7
                }
            }
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&m.w_empty[s]);
    mbar_wait(&m.a_empty[as], ((u / kAStages) & 1) ^ 1);
    tc_fence_after();
    const uint32_t dst = tmem + (static_cast<uint32_t>(32 * q) << 16) + kAColBase + as * kAStageCols;
    tmem_st_32x32b_x32(dst, lanes8[0]);
    if (nb > 1) tmem_st_32x32b_x32(dst + 32, lanes8[1]);
    tmem_wait_st();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&m.a_full[as]);
    if (utr && u < 64 && r == 0) utr[8 * u + 1] = clock64();
}

// K1 of linear l over this CTA's k-slice, by the kQThreads threads of warps 2..11:
// (wait for the producing linear if any) load x[:, slice] (all loads in flight at once,
// held packed in registers), per-token partial max|x| (warp-reduced per token, one
// shared atomic per token and warp), all-to-all of the partial maxima over the cluster
// (DSMEM st.async completing on the peers' max_full), S = max/127 (ref
// quantize.cpp:22-35), codes into the resident, MMA-ready B (SWIZZLE_128B K-major), then
// b_ready.  The MMAs of linear l-1 are complete when it writes B: the epilogue warps,
// which join the first barrier, have drained all of its accumulators.
template <bool BF16>
__device__ __forceinline__ void quantize_slice(const PParams& p, const Smem& m, int l, int qi, const LGeo& g,
                                               int crank, int qt, unsigned long long* trc) {
    const LinDesc& d = p.lin[l];
    const int lane = qt & 31;
    if (d.dep >= 0) {  // x_l is linear dep's output: wait for its grid-wide completion
        if (qt == 0) {
            while (ld_acquire_u32(p.ctr + d.dep) < gridDim.x) __nanosleep(64);
        }
        named_bar_sync(2, kQThreads);
    }
    if (trc && qt == 0 && l < 6) trc[8 + 4 * l] = globaltimer();
    const bool cg = d.dep >= 0;
    const unsigned short* x = static_cast<const unsigned short*>(d.x);
    const int nch = g.nkb * (kBlockK / 16);  // 16-element chunks per token row
    if (qt < kBN) m.tmax[qt] = 0u;
    // Chunk j of this thread is c = qt + j * kQThreads -> (token t = c / nch, 16-element
    // chunk k = c % nch); t >= M: none.  Chunks are processed in batches of kQHold held
    // packed in registers: the max pass walks every batch, the quantize pass keeps the
    // last batch and reloads the others (large k-slices only; L2 hits).
    const int nbatch = max(1, (d.M * nch - qt + kQThreads * kQHold - 1) / (kQThreads * kQHold));
    const int dt = nch > 0 ? kQThreads / nch : 0, dk = kQThreads - dt * nch;
    const unsigned short* xs = x + g.kb_lo * kBlockK;
    const int kx = d.K - g.kb_lo * kBlockK;
    uint4 raw[kQHold][2];
    auto batch_start = [&](int b, int& t, int& k) {
        const int c = qt + b * kQHold * kQThreads;
        t = nch > 0 ? c / nch : d.M;
        k = nch > 0 ? c - t * nch : 0;
    };
    auto load_batch = [&](int b) {
        int t, k;
        batch_start(b, t, k);
#pragma unroll
        for (int i = 0; i < kQHold; ++i) {
            if (t < d.M) load16_raw(xs + static_cast<size_t>(t) * d.ldx, k * 16, kx, cg, raw[i][0], raw[i][1]);
            t += dt;
            k += dk;
            if (k >= nch) {
                k -= nch;
                ++t;
            }
        }
    };
    const uint32_t tmax_s = smem_u32(m.tmax);
    for (int b = 0; b < nbatch; ++b) {
        load_batch(b);
        if (b == 0) named_bar_sync(2, kQThreads);  // tmax zeroed; linear l-1's MMAs all complete
        int t, k;
        batch_start(b, t, k);
#pragma unroll
        for (int i = 0; i < kQHold; ++i) {
            const bool live = t < d.M;
            const int tt = live ? t : -1;
            const uint32_t v = live ? absmax16_bits<BF16>(raw[i][0], raw[i][1]) : 0u;
            const uint32_t grp = __match_any_sync(0xffffffffu, tt);
            const uint32_t mx = __reduce_max_sync(grp, v);
            if (live && lane == __ffs(grp) - 1) atom_max_shared_u32(tmax_s + t * 4, mx);
            t += dt;
            k += dk;
            if (k >= nch) {
                k -= nch;
                ++t;
            }
        }
    }
    named_bar_sync(2, kQThreads);
    if (p.S > 1) {  // all-to-all of the partial maxima over the cluster (DSMEM)
        if (qt < p.S * kBN) {
            const int dst = qt / kBN, t = qt % kBN;
            if (dst != crank)
                st_async_u32(mapa_shared(smem_u32(m.peer_max + crank * kBN + t), dst), lds32(tmax_s + t * 4),
                             mapa_shared(smem_u32(m.max_full), dst));
        }
        mbar_wait_cluster(m.max_full, qi & 1);
    }
    if (qt < kBN) {
        uint32_t mx = lds32(tmax_s + qt * 4);
        for (int s = 0; s < p.S; ++s)
            if (s != crank) mx = max(mx, lds32(smem_u32(m.peer_max) + (s * kBN + qt) * 4));
        float sc = __uint_as_float(mx) / 127.0f;  // ref quantize.cpp:22-35 (IEEE division)
        if (!(sc > 0.0f)) sc = kMinScale;
        m.tscale[qt] = sc;
        m.trcp[qt] = 1.0f / sc;
        if (d.sa_out && blockIdx.x == 0 && qt < d.M) d.sa_out[qt] = sc;
    }
    // every thread has passed the max_full wait: re-arm it for the next linear's maxima
    if (p.S > 1 && qt == 0) mbar_expect_tx(m.max_full, (p.S - 1) * kBN * 4);  // next in-kernel linear
    named_bar_sync(2, kQThreads);
    const uint32_t rb = smem_u32(m.resb);
    const uint32_t sc_s = smem_u32(m.tscale), rc_s = smem_u32(m.trcp);
    for (int b = nbatch - 1; b >= 0; --b) {
        if (b != nbatch - 1) load_batch(b);  // earlier batches were not kept
        int t, k;
        batch_start(b, t, k);
#pragma unroll
        for (int i = 0; i < kQHold; ++i) {
            if (t < d.M) {
                const float scale = __uint_as_float(lds32(sc_s + t * 4));
                const float rcp = __uint_as_float(lds32(rc_s + t * 4));
                const uint4 qv = p.dbg == 1 ? raw[i][0] : quant16<BF16>(raw[i][0], raw[i][1], scale, rcp, p.dbg);
                sts128(rb + (k >> 3) * kBBlockBytes + t * 128 + ((((k & 7) ^ (t & 7)) & 7) * 16), qv);
            }
            t += dt;
            k += dk;
            if (k >= nch) {
                k -= nch;
                ++t;
            }
        }
    }
    for (int c = d.M * nch + qt; c < kBN * nch; c += kQThreads) {  // padding tokens: zero codes
        const int t = c / nch, k = c - t * nch;
        sts128(rb + (k >> 3) * kBBlockBytes + t * 128 + ((((k & 7) ^ (t & 7)) & 7) * 16), make_uint4(0, 0, 0, 0));
    }
    fence_proxy_async_shared();  // generic smem writes -> visible to tcgen05.mma
    named_bar_sync(2, kQThreads);
    if (qt == 0) mbar_arrive(m.b_ready);
    if (trc && qt == 0 && l < 6) trc[9 + 4 * l] = globaltimer();
}

// Runs linear l's prologue unless its activations arrive pre-quantized; qi counts the
// in-kernel-quantized linears (their b_ready / max_full phases).
__device__ __forceinline__ void quantize_slice_any(const PParams& p, const Smem& m, int l, int& qi, const LGeo& g,
                                                   int crank, int qt, unsigned long long* trc) {
    if (p.lin[l].qa) return;
    if (p.lin[l].x_bf16)
        quantize_slice<true>(p, m, l, qi, g, crank, qt, trc);
    else
        quantize_slice<false>(p, m, l, qi, g, crank, qt, trc);
    ++qi;
}

__global__ void __launch_bounds__(kThreads, 1) w4a8_decode_kernel(const __grid_constant__ PParams p) {
    extern __shared__ uint8_t smem_raw[];
    const Smem m = carve(reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                    ~static_cast<uintptr_t>(1023)));
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int S = p.S;
    const int crank = S > 1 ? static_cast<int>(cluster_rank()) : 0;
    const int cl = blockIdx.x / S;
    int total_tiles = 0;  // this cluster's tiles over the whole program (same on every rank)
    bool any_signal = false;
    for (int l = 0; l < p.L; ++l) {
        total_tiles += lgeo(p, l, crank, cl).ntiles;
        any_signal |= p.lin[l].signal != 0;
    }
    unsigned long long* trc = p.trace ? p.trace + blockIdx.x * kTraceCta : nullptr;
    // CTA 0 only: per-unit clock64 [converter start, converter done, MMA ready, MMA issued]
    unsigned long long* utr = p.trace && blockIdx.x == 0 ? p.trace + 148 * kTraceCta : nullptr;
    if (trc && threadIdx.x == 0) trc[0] = globaltimer();
    if (p.pdl) pdl_launch_dependents();

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&m.w_full[i], 1);
            mbar_init(&m.w_empty[i], 5);  // the 4 converter warps + the MMA commit (B tiles)
            mbar_init(&m.b_full[i], 1);
        }
        for (int i = 0; i < kAStages; ++i) {
            mbar_init(&m.a_full[i], 4);
            mbar_init(&m.a_empty[i], 1);
        }
        for (int i = 0; i < kDBufs; ++i) {
            mbar_init(&m.d_full[i], 1);
            mbar_init(&m.d_empty[i], 4);
        }
        mbar_init(m.b_ready, 1);
        mbar_init(m.max_full, 1);
        fence_mbar_init();
        if (S > 1) mbar_expect_tx(m.max_full, (S - 1) * kBN * 4);  // peers' partial maxima
    }
    if (warp == kWarpAlloc) {
        tmem_alloc(m.tmem_slot, kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    if (S > 1) cluster_sync();  // every peer's barriers are armed before any DSMEM traffic
    tc_fence_after();
    const uint32_t tmem = lds32(smem_u32(m.tmem_slot));
    if (trc && threadIdx.x == 0) trc[1] = globaltimer();

    if (warp == kWarpProducer) {
        // Weights and channel scales are constant: the only griddepcontrol.wait on this
        // path guards the pre-quantized B tiles.
        if (lane < 2) {
            const uint64_t pol = l2_policy_evict_first();
            // L2 prefetch window: units [kStages, U + kStages + pf_units) ahead of the load
            // position U, walking across the program's linears.
            int pl = 0, pk = 0, PU = 0;
            LGeo pg = lgeo(p, 0, crank, cl);
            auto pf_step = [&](bool issue) -> bool {
                while (pl < p.L && pk >= pg.units) {
                    if (++pl < p.L) pg = lgeo(p, pl, crank, cl);
                    pk = 0;
                }
                if (pl >= p.L) return false;
                if (issue) {
                    const LinDesc& d = p.lin[pl];
                    const int nt = pg.tile(pk / pg.upt);
                    bulk_prefetch_l2(d.wp + (static_cast<size_t>(nt) * d.kblocks + pg.unit_kb(pk)) * kWBlockBytes,
                                     pg.unit_nb(pk) * kWBlockBytes);
                }
                ++pk;
                ++PU;
                return true;
            };
            // Pre-quantized B tiles come from the previous kernel (the act quant): the
            // first ring of weight units is issued before griddepcontrol.wait, their B
            // tiles after it.
            const uint64_t pol_b = l2_policy_evict_last();
            auto issue_b = [&](const LinDesc& d, int s, int kb, int nb) {
                mbar_expect_tx(&m.b_full[s], nb * kBBlockBytes);
                for (int b = 0; b < nb; ++b)
                    bulk_g2s(m.ring + s * kStageBytes + kUnitBytes + b * kBBlockBytes,
                             d.qa + static_cast<size_t>(kb + b) * d.Mp * 128, kBBlockBytes, &m.b_full[s], pol_b);
            };
            bool waited = p.pdl == 0;
            auto flush_deferred = [&](int upto) {  // B tiles of units [0, upto)
                int u = 0;
                for (int l = 0; l < p.L && u < upto; ++l) {
                    const LinDesc& d = p.lin[l];
                    const LGeo g = lgeo(p, l, crank, cl);
                    for (int k = 0; k < g.units && u < upto; ++k, ++u)
                        if (d.qa) issue_b(d, u % kStages, g.unit_kb(k), g.unit_nb(k));
                }
            };
            // Two lanes issue alternate units of each tile in SIMT lockstep, halving the
            // producer's per-unit overhead (waits, barrier arrivals, copy issue).
            int U = 0, J = 0;
            for (int l = 0; l < p.L; ++l) {
                const LinDesc& d = p.lin[l];
                const LGeo g = lgeo(p, l, crank, cl);
                const uint8_t* wp = d.wp;
                const size_t kbl = static_cast<size_t>(d.kblocks);
                const bool pre = d.qa != nullptr;
                for (int i = 0; i < g.ntiles; ++i, ++J) {
                    const int nt = g.tile(i);
                    const uint8_t* wtile = wp + static_cast<size_t>(nt) * kbl * kWBlockBytes;
                    for (int k0 = 0; k0 < g.upt; k0 += 2) {
                        if (!waited && U + k0 + 1 >= kStages) {
                            // the ring's first units are in flight: wait for the act quant,
                            // then send the B tiles of every unit issued so far
                            pdl_wait();
                            waited = true;
                            if (lane == 0) flush_deferred(U + k0);
                        }
                        const int k = k0 + lane;
                        if (k < g.upt) {
                            const int Uk = U + k;
                            const int s = Uk % kStages;
                            const int kb = g.kb_lo + kUnitBlocks * k;
                            const int nb = min(kUnitBlocks, g.kb_hi - kb);
                            if (lane == 0 && p.pf_units > 0)
                                while (PU < Uk + kStages + p.pf_units && pf_step(PU >= kStages)) {
                                }
                            if (utr && Uk < 64) utr[8 * Uk + 4] = clock64();
                            if (Uk >= kStages) mbar_wait(&m.w_empty[s], ((Uk / kStages) & 1) ^ 1);
                            if (utr && Uk < 64) utr[8 * Uk + 5] = clock64();
                            mbar_expect_tx(&m.w_full[s], nb * kWBlockBytes);
                            bulk_g2s(m.ring + s * kStageBytes, wtile + static_cast<size_t>(kb) * kWBlockBytes,
                                     nb * kWBlockBytes, &m.w_full[s], pol);
                            if (utr && Uk < 64) utr[8 * Uk + 6] = clock64();
                            if (pre && waited) issue_b(d, s, kb, nb);
                            if (utr && Uk < 64) utr[8 * Uk + 7] = clock64();
                        }
                        __syncwarp(0x3u);
                    }
                    U += g.upt;
                }
            }
            if (!waited) {  // the whole program fit in one ring
                pdl_wait();
                if (lane == 0) flush_deferred(U);
            }
            if (p.next_bytes > 0 && lane == 0) {
                // every own load is issued: stream this CTA's share of the next launch's
                // weights into L2 (evict-normal; that kernel reads them evict-first)
                const size_t share = (p.next_bytes / gridDim.x + 16383) & ~static_cast<size_t>(16383);
                const size_t lo = share * blockIdx.x;
                const size_t hi = min(p.next_bytes, lo + share);
                for (size_t off = lo; off < hi; off += 16384)
                    bulk_prefetch_l2(p.next_wp + off, static_cast<uint32_t>(min(static_cast<size_t>(16384), hi - off)));
            }
            if (trc && lane == 0) trc[6] = globaltimer();
        }
    } else if (warp == kWarpMma) {
        const uint32_t rb = smem_u32(m.resb);
        int U = 0, JD = 0, qi = 0;
        for (int l = 0; l < p.L; ++l) {
            const LGeo g = lgeo(p, l, crank, cl);
            const bool pre = p.lin[l].qa != nullptr;  // B tiles ride in the ring stages
            if (!pre) {
                mbar_wait(m.b_ready, qi & 1);
                tc_fence_after();
                ++qi;
            }
            for (int i = 0; i < g.ntiles && g.upt > 0; ++i, ++JD) {
                const int db = JD % kDBufs;
                const uint32_t d_tmem = tmem + db * kBN;
                mbar_wait(&m.d_empty[db], ((JD / kDBufs) & 1) ^ 1);
                tc_fence_after();
                for (int k = i * g.upt; k < (i + 1) * g.upt; ++k, ++U) {
                    const int kb = g.unit_kb(k), nb = g.unit_nb(k);
                    const int as = U % kAStages;
                    const int s = U % kStages;
                    mbar_wait(&m.a_full[as], (U / kAStages) & 1);
                    if (pre) mbar_wait(&m.b_full[s], (U / kStages) & 1);
                    tc_fence_after();
                    if (utr && U < 64 && lane == 0) utr[8 * U + 2] = clock64();
                    if (trc && lane == 0 && l < 6 && k == 0) trc[10 + 4 * l] = globaltimer();
                    const uint32_t a_tmem = tmem + kAColBase + as * kAStageCols;
                    const uint32_t b0 = pre ? smem_u32(m.ring) + s * kStageBytes + kUnitBytes
                                            : rb + (kb - g.kb_lo) * kBBlockBytes;
                    if (elect_one()) {
#pragma unroll
                        for (int c = 0; c < 4 * kUnitBlocks; ++c)
                            if (c < 4 * nb)
                                mma_i8_ts(d_tmem, a_tmem + 8 * c, b_desc(b0 + (c / 4) * kBBlockBytes + 32 * (c % 4)),
                                          kIdesc, (kb > g.kb_lo || c > 0) ? 1u : 0u);
                        mma_commit(&m.a_empty[as]);
                        mma_commit(&m.w_empty[s]);  // the stage's B tiles are consumed
                        if (utr && U < 64) utr[8 * U + 3] = clock64();
                        if (kb + nb == g.kb_hi) mma_commit(&m.d_full[db]);  // tile complete
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // Warps 2..11: every linear starts with its activation prologue (all 10 warps);
        // then the converters widen the linear's units and warps 8..11 run its epilogue.
        const bool conv = warp >= kWarpConv0 && warp < kWarpConv0 + 4 * kConvGroups;
        const bool epi = warp >= kWarpEpi0;
        const int qt = threadIdx.x - kWarpAlloc * 32;
        if (p.pdl) pdl_wait();  // the activations may come from the previous kernel
        if (conv) {
            const int grp = (warp - kWarpConv0) / 4;
            const int q = warp & 3;  // TMEM sub-partition: lanes 32q..32q+31
            int U = 0, qi = 0;
            for (int l = 0; l < p.L; ++l) {
                const LGeo g = lgeo(p, l, crank, cl);
                quantize_slice_any(p, m, l, qi, g, crank, qt, trc);
                for (int k = 0; k < g.units; ++k, ++U)
                    if (U % kConvGroups == grp) convert_unit(m, tmem, q, lane, U, g.unit_nb(k), utr);
            }
        } else if (!epi) {
            int qi = 0;
            for (int l = 0; l < p.L; ++l) quantize_slice_any(p, m, l, qi, lgeo(p, l, crank, cl), crank, qt, trc);
        } else {
            const int q = warp & 3;
            const int r = 32 * q + lane;  // tile row (TMEM lane) of this thread
            const uint32_t t_lane = tmem + (static_cast<uint32_t>(32 * q) << 16);
            uint32_t* flag = reinterpret_cast<uint32_t*>(m.swr);  // "this CTA finalises" broadcast
            int JD = 0, qi = 0, tbase = 0;
            for (int l = 0; l < p.L; ++l) {
                const LinDesc& d = p.lin[l];
                const LGeo g = lgeo(p, l, crank, cl);
                quantize_slice_any(p, m, l, qi, g, crank, qt, trc);
                // ---------------- epilogue.  With S > 1 the S partial tiles meet in L2:
                // every rank red.adds its int32 partial into the tile's accumulator and
                // bumps the tile's arrival counter; the LAST rank to arrive finalises the
                // whole tile (integer addition: exact in any order) and re-zeroes it.  No
                // rank ever waits for another.
                float sa[kBN];
#pragma unroll
                for (int t = 0; t < kBN; ++t)
                    sa[t] = !d.qa ? m.tscale[t] : (t < d.M ? __ldg(d.sa + t) : 0.0f);
                for (int i = 0; i < g.ntiles; ++i) {
                    const int nt = g.tile(i);
                    const int n = nt * kTileN + r;
                    const float sw_n = n < d.N ? __ldg(d.sw + n) : 0.0f;  // in flight during the wait
                    uint32_t v[kBN];
                    if (g.upt > 0) {
                        const int db = JD % kDBufs;
                        mbar_wait(&m.d_full[db], (JD / kDBufs) & 1);
                        tc_fence_after();
                        tmem_ld_32x32b_x16(t_lane + db * kBN, v);
                        tmem_wait_ld();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&m.d_empty[db]);
                        ++JD;
                    } else {
#pragma unroll
                        for (int t = 0; t < kBN; ++t) v[t] = 0u;  // empty k-slice: zero partial
                    }
                    bool fin = true;
                    int32_t* acc = p.acc + (static_cast<size_t>(tbase + nt) * kBN) * kTileN;  // [t][row]
                    if (S > 1) {
                        if (g.upt > 0)
#pragma unroll
                            for (int t = 0; t < kBN; ++t)
                                if (t < d.M) red_add_s32(acc + t * kTileN + r, static_cast<int32_t>(v[t]));
                        named_bar_sync(3, 128);  // this CTA's partial is issued
                        if (r == 0) {
                            __threadfence();
                            const uint32_t prev = atomicAdd(p.tile_cnt + tbase + nt, 1u);
                            *flag = prev == static_cast<uint32_t>(S - 1) ? 1u : 0u;
                        }
                        named_bar_sync(3, 128);
                        fin = *flag != 0u;
                        if (fin) {
                            __threadfence();  // every rank's partial is visible (acquire side)
#pragma unroll
                            for (int t = 0; t < kBN; ++t)
                                if (t < d.M) {
                                    v[t] = static_cast<uint32_t>(__ldcg(acc + t * kTileN + r));
                                    __stcg(acc + t * kTileN + r, 0);  // re-zero for the next launch
                                }
                            if (r == 0) p.tile_cnt[tbase + nt] = 0u;
                        }
                    }
                    if (fin && n < d.N) {
#pragma unroll
                        for (int t = 0; t < kBN; ++t) {
                            if (t < d.M) {
                                const int32_t sh = static_cast<int32_t>(v[t]) >> 4;  // exact (ref gemm.cpp:269)
                                const float y = __fmul_rn(__int2float_rn(sh), __fmul_rn(sa[t], sw_n));
                                const size_t idx = static_cast<size_t>(t) * d.N + n;
                                if (d.out_dtype == kDtypeF32)
                                    static_cast<float*>(d.out)[idx] = y;
                                else if (d.out_dtype == kDtypeF16)
                                    static_cast<__half*>(d.out)[idx] = __float2half_rn(y);
                                else
                                    static_cast<__nv_bfloat16*>(d.out)[idx] = __float2bfloat16_rn(y);
                            }
                        }
                    }
                }
                tbase += d.n_tiles;
                if (d.signal) {
                    // every output of linear l stored by this CTA -> publish (release, gpu scope)
                    named_bar_sync(3, 128);
                    if (r == 0) {
                        __threadfence();
                        red_release_add_u32(p.ctr + l, 1u);
                    }
                }
                if (trc && r == 0 && l < 6) trc[11 + 4 * l] = globaltimer();
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kWarpAlloc) tmem_dealloc(tmem, kTmemCols);
    if (threadIdx.x == 0) {
        if (any_signal) {
            // the last CTA out resets the completion counters for the next launch
            __threadfence();
            if (atomicAdd(p.ctr + kMaxLin, 1u) == gridDim.x - 1) {
                for (int l = 0; l < p.L; ++l) p.ctr[l] = 0u;
                p.ctr[kMaxLin] = 0u;
                __threadfence();
            }
        }
        if (trc) {
            trc[5] = globaltimer();
            trc[7] = static_cast<unsigned long long>(S) | (static_cast<unsigned long long>(p.C) << 16) |
                     (static_cast<unsigned long long>(p.L) << 32);
        }
    }
}

// ===================================================================== dynamic schedule
// w4a8_decode_dyn_kernel: the same data path for a program whose activations all arrive
// pre-quantized, but the work -- (linear, 128-row tile, k-split) items, in program order
// -- is handed out at run time from one global counter: each CTA's producer grabs the
// next item whenever its ring has room, so SMs that stream faster simply take more items
// (measured: the static assignment left some CTAs ~2x behind on every linear).  A
// split tile's partials meet in L2: each item stores its int32 partial, bumps the tile's
// arrival counter, and the last item to arrive sums the S partials and runs the
// epilogue.  No clusters, no DSMEM; the grid is one CTA per SM.

constexpr int kDynThreads = 512;        // 16 warps: two converter groups (4..7, 8..11), epilogue 12..15
constexpr int kDynConvGroups = 2;
constexpr int kDynEpi0 = 12;
constexpr int kItemSlots = 8;
// Per-BN configuration of the dynamic kernel (BN = 16/32/64 tokens per MMA N).
template <int BN, bool DEP, int UB = 2>
struct DynCfg {
    // Pipeline unit: UB k-blocks (UB * 8 KiB of packed weights, a UB*32-column TMEM A stage).
    // The MMA warp's per-unit fixed cost (two mbarrier waits ~100 cycles each even when
    // already complete, commits, loop: ~350 cycles, tools/mma_loop_bench.cu) is amortised
    // over UB k-blocks: UB = 4 for a lone linear (config 1: 18.2 -> 12.1 us), UB = 2 for
    // multi-linear programs, whose deeper rings and A-stage count measured faster (37.5 vs
    // 41.3 us for the layer's 4 linears).
    static constexpr int kUB = UB;
    static constexpr int kUBytes = kUB * kWBlockBytes;
    static constexpr int kAStageColsD = kUB * kBlockK / 4;
    static constexpr int kBBlock = BN * 128;                            // one B k-block tile
    static constexpr int kStageBytes = kUBytes + kUB * kBBlock;         // weights + B tiles
    static constexpr int kStages = (220 * 1024 - 3072) / kStageBytes < 10 ? (220 * 1024 - 3072) / kStageBytes : 10;
    static constexpr int kSmem = kStages * kStageBytes + 2048 /*barriers, items*/ + 1024 /*alignment*/;
    // TMEM: kDBufs accumulator buffers (BN columns each) at column 0, then as many 64-column
    // A stages as fit.  The converter -> MMA -> commit -> converter handshake has ~1 us of
    // round-trip latency, so the unit rate is A stages / that latency (measured: 0.32 us per
    // unit with 4 stages, unchanged with the MMAs and TMEM stores removed).
    static constexpr int kAColBase = kDBufs * BN;
    static constexpr int kAStages = (kTmemCols - kAColBase) / kAStageColsD;
    // kind::i8, D=s32, A=B=s8 signed, K-major both, N=BN, M=128
    static constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                       (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
    static_assert(kSmem <= 227 * 1024, "smem budget");
    static_assert(kDBufs * BN <= kAColBase, "D buffers below the A stages");
};


// One item's outputs from thread r's accumulators (output column n, BN tokens), specialised
// per output format so the token loop is straight-line and the tokens' conversions and
// stores overlap: with the format switched at run time inside the loop every token cost
// ~5 branches and a serial convert->store chain (measured ~0.1 us per token, 1.6 us per
// 16-token item on the critical path of every linear).  ODT -1: int32 pre-shift
// accumulators (acc_out).  AMX: also reduce max |stored value| per token into the CTA's
// smem maxima (the dependent linear's x scale).
// One row-batch entry's fields, read from the kernel parameters ONCE (and kept in
// registers: a parameter indexed by a run-time entry number compiles to an indexed
// constant load, whose cold miss costs ~0.3 us on a fresh SM -- measured, several of them
// serialised were most of the act quant's run time after its loads landed).
struct RowArgs {
    const unsigned short* x;
    size_t ldx;
    int K, Mp;
    int8_t* q;
    float* s;
    const float* amax_in;
};
__device__ __forceinline__ size_t ld_keep_u64(size_t v) {
    unsigned long long r;
    asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(static_cast<unsigned long long>(v)));
    return static_cast<size_t>(r);
}

template <bool BF16>
__device__ __forceinline__ void quant_row(const RowArgs& ra, int t, float* red, bool dry,
                                          unsigned long long* trc = nullptr) {
    const unsigned short* row = ra.x + static_cast<size_t>(t) * ra.ldx;
    const int K = ra.K;
    const int nch = static_cast<int>(pad_k(K) / 16);
    uint4 raw[kRowChunks][2];
    uint32_t mb = 0u;
#pragma unroll
    for (int j = 0; j < kRowChunks; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        if (c < nch) {
            load16_raw(row, c * 16, K, false, raw[j][0], raw[j][1]);
            mb = max(mb, absmax16_bits<BF16>(raw[j][0], raw[j][1]));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    if ((threadIdx.x & 31) == 0) reinterpret_cast<uint32_t*>(red)[threadIdx.x >> 5] = mb;
    __syncthreads();
    if (trc && !dry && threadIdx.x == 0) trc[3] = globaltimer();  // every load of the row landed
    // the CTA max: one shared load per lane + a shuffle tree (32 dependent shared loads
    // per thread measured ~0.5 us)
    const int lane = threadIdx.x & 31;
    uint32_t m = lane < kRowThreads / 32 ? reinterpret_cast<uint32_t*>(red)[lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (ra.amax_in) m = __float_as_uint(ra.amax_in[t]);  // the global max of a K-sharded row
    if (trc && !dry && threadIdx.x == 0) trc[4] = globaltimer() + (m == 0x7fffffffu);  // row max
    float sc = __uint_as_float(m) / 127.0f;  // ref quantize.cpp:22-35 (IEEE division)
    if (!(sc > 0.0f)) sc = kMinScale;
    const float rcp = 1.0f / sc;
    if (trc && !dry && threadIdx.x == 0) trc[5] = globaltimer() + (rcp == 3.0f);  // scale
    if (threadIdx.x == 0 && !dry) ra.s[t] = sc;
    uint4 qv[kRowChunks];
    bool ok[kRowChunks];
#pragma unroll
    for (int j = 0; j < kRowChunks; ++j) qv[j] = quant16_fast<BF16>(raw[j][0], raw[j][1], rcp, ok[j]);
    if (trc && !dry && threadIdx.x == 0) trc[6] = globaltimer() + (qv[0].x == 0x7fffffffu);  // codes
#pragma unroll
    for (int j = 0; j < kRowChunks; ++j) {
        const int c = threadIdx.x + j * kRowThreads;
        if (c < nch) {
            if (!ok[j]) qv[j] = fix16(qv[j], raw[j][0], raw[j][1], sc, rcp, BF16);
            if (!dry)
                *reinterpret_cast<uint4*>(ra.q + a8_offset(static_cast<size_t>(t), static_cast<size_t>(c) * 16,
                                                           ra.Mp)) = qv[j];
        }
    }
}

__device__ __forceinline__ void act_quant_rows_body(const RowBatch& b) {
    unsigned long long* trc = (b.trace && blockIdx.x < 64) ? b.trace + 8 * blockIdx.x : nullptr;
    if (trc && threadIdx.x == 0) trc[0] = globaltimer();
    if (b.pdl) pdl_launch_dependents();
    __shared__ float red[kRowThreads / 32];
    int i = 0, t = blockIdx.x;
    while (i + 1 < b.n && t >= b.M[i]) t -= b.M[i++];
    // Under PDL the CTA is resident long before its input exists: pass 0 runs the whole
    // row quantization dry (x as it is now, no stores) so its instructions are fetched
    // into the SM's instruction cache while waiting; the real pass then runs warm.  Cold
    // fetch of this straight-line code measured 1.5-3 us per launch (trace marks), most
    // of the act quant's time between two dependent linears.  One copy of the code
    // (`unroll 1`): the dry pass must warm the very instructions the real pass runs.
    RowArgs ra;
    ra.x = ld_keep_ptr(b.x[i]);
    ra.ldx = ld_keep_u64(b.ldx[i]);
    ra.K = ld_keep(b.K[i]);
    ra.Mp = ld_keep(b.Mp[i]);
    ra.q = ld_keep_ptr(b.q[i]);
    ra.s = ld_keep_ptr(b.s[i]);
    ra.amax_in = ld_keep_ptr(b.amax_in[i]);
    const int bf16 = ld_keep(b.bf16[i]);
    const int pdl = ld_keep(b.pdl);
#pragma unroll 1
    for (int pass = pdl ? 0 : 1; pass < 2; ++pass) {
        if (pass == 1) {
            if (pdl) pdl_wait();
            if (trc && threadIdx.x == 0) trc[1] = globaltimer();
        }
        if (bf16)
            quant_row<true>(ra, t, red, pass == 0, trc);
        else
            quant_row<false>(ra, t, red, pass == 0, trc);
    }
    if (trc) {
        __syncthreads();
        if (threadIdx.x == 0) trc[2] = globaltimer();
    }
}


__global__ void __launch_bounds__(kRowThreads, 1) act_quant_rows_kernel(const __grid_constant__ RowBatch b) {
    act_quant_rows_body(b);
}

// K1 of a dependent chain link: the token row maxima come from the producer launch's
// epilogues (per-token atomicMax of the stored |y|, f32 bits -- the same value the row
// reduction would find), so a row needs no reduction and is spread over kPreCtas CTAs of
// 256 threads, one 16-element chunk per thread.  Bit-exact with act_quant_rows_kernel.
constexpr int kPreCtas = 4;
constexpr int kPreThreads = 256;
static_assert(kPreCtas * kPreThreads * 16 >= kRowThreads * kRowChunks * 16, "premax covers every external K");
__global__ void __launch_bounds__(kPreThreads, 4) act_quant_premax_kernel(const __grid_constant__ RowBatch b) {
    if (b.pdl) pdl_launch_dependents();
    int i = 0, t = blockIdx.x / kPreCtas;
    const int part = blockIdx.x % kPreCtas;
    while (i + 1 < b.n && t >= b.M[i]) t -= b.M[i++];
    const unsigned short* row = ld_keep_ptr(b.x[i]) + static_cast<size_t>(t) * ld_keep_u64(b.ldx[i]);
    const int K = ld_keep(b.K[i]);
    const int Mp = ld_keep(b.Mp[i]);
    int8_t* const q = ld_keep_ptr(b.q[i]);
    float* const s = ld_keep_ptr(b.s[i]);
    const uint32_t* const am = ld_keep_ptr(b.amax_src[i]);
    const int bf16 = ld_keep(b.bf16[i]);
    const int pdl = ld_keep(b.pdl);
    const int nch = static_cast<int>(pad_k(K) / 16);
    const int c = part * kPreThreads + threadIdx.x;
    // pass 0 runs dry before griddepcontrol.wait (warm instruction / constant caches)
#pragma unroll 1
    for (int pass = pdl ? 0 : 1; pass < 2; ++pass) {
        if (pass == 1 && pdl) pdl_wait();
        const bool dry = pass == 0;
        const uint32_t m = __ldcg(am + t * kAmaxStride);
        float sc = __uint_as_float(m) / 127.0f;  // ref quantize.cpp:22-35 (IEEE division)
        if (!(sc > 0.0f)) sc = kMinScale;
        const float rcp = 1.0f / sc;
        if (threadIdx.x == 0 && part == 0 && !dry) s[t] = sc;
        if (c < nch) {
            uint4 r0, r1;
            load16_raw(row, c * 16, K, true, r0, r1);
            bool ok;
            uint4 v = bf16 ? quant16_fast<true>(r0, r1, rcp, ok) : quant16_fast<false>(r0, r1, rcp, ok);
            if (!ok || dry) v = fix16(v, r0, r1, sc, rcp, bf16 != 0);
            if (!dry) *reinterpret_cast<uint4*>(q + a8_offset(static_cast<size_t>(t), static_cast<size_t>(c) * 16, Mp)) = v;
        }
    }
}

template <int BN, int ODT, bool AMX>
__device__ __forceinline__ void epi_store(const uint32_t (&v)[BN], const float* tsc, float sw_n, int m_rows,
                                          int n_cols, int n, bool own, bool amx, void* outv, uint32_t emax_a,
                                          int lane) {
#pragma unroll
    for (int t0 = 0; t0 < BN; t0 += 16) {
        float sat[16];  // the token scales of 16 tokens at a time, loaded ahead of the stores
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
            const uint4 s4 = lds128(smem_u32(tsc + t0 + 4 * q4));
            sat[4 * q4] = __uint_as_float(s4.x);
            sat[4 * q4 + 1] = __uint_as_float(s4.y);
            sat[4 * q4 + 2] = __uint_as_float(s4.z);
            sat[4 * q4 + 3] = __uint_as_float(s4.w);
        }
#pragma unroll
        for (int tt = 0; tt < 16; ++tt) {
            const int t = t0 + tt;
            if (t >= m_rows) break;  // warp-uniform
            const size_t idx = static_cast<size_t>(t) * n_cols + n;
            if constexpr (ODT < 0) {
                if (own) stg_b32_free(static_cast<uint32_t*>(outv) + idx, v[t]);  // pre-shift (TP all-reduce)
            } else {
                const int32_t sh = static_cast<int32_t>(v[t]) >> 4;  // exact (ref gemm.cpp:269)
                const float y = __fmul_rn(__int2float_rn(sh), __fmul_rn(sat[tt], sw_n));
                uint32_t mag = 0u;  // |stored value| as f32 bits (the dependent linear's x)
                if constexpr (ODT == kDtypeF32) {
                    if (own) stg_b32_free(static_cast<float*>(outv) + idx, __float_as_uint(y));
                } else if constexpr (ODT == kDtypeF16) {
                    const __half h = __float2half_rn(y);
                    if (own) stg_b16_free(static_cast<__half*>(outv) + idx, __half_as_ushort(h));
                    mag = __float_as_uint(fabsf(__half2float(h)));
                } else {
                    const __nv_bfloat16 h = __float2bfloat16_rn(y);
                    if (own) stg_b16_free(static_cast<__nv_bfloat16*>(outv) + idx, __bfloat16_as_ushort(h));
                    mag = __float_as_uint(fabsf(__bfloat162float(h)));
                }
                if constexpr (AMX) {  // every lane joins the reduction
                    mag = __reduce_max_sync(0xffffffffu, (own && amx) ? mag : 0u);
                    if (lane == 0 && mag != 0u) atom_max_shared_u32(emax_a + 4 * t, mag);
                }
            }
        }
    }
}

struct DynItem {
    int l, nt, kb_lo, kb_hi, r;
    int s, i0;  // the tile's k-split count, its split 0's item index within the linear
};
__device__ __forceinline__ DynItem dyn_item(const PParams& p, const LinDesc* lin, int it) {
    DynItem x;
    int l = 0;
    while (l + 1 < p.L && it >= lin[l + 1].ibase) ++l;
    const LinDesc& d = lin[l];
    const int rel = it - d.ibase;
    x.l = l;
    const int head = d.t1 * d.split;
    if (rel < head) {
        x.s = d.split;
        x.nt = rel / x.s;
        x.r = rel - x.nt * x.s;
        x.i0 = x.nt * x.s;
    } else {
        x.s = d.split2;
        const int t = (rel - head) / x.s;
        x.r = rel - head - t * x.s;
        x.nt = d.t1 + t;
        x.i0 = head + t * x.s;
    }
    x.kb_lo = x.r * d.kblocks / x.s;
    x.kb_hi = (x.r + 1) * d.kblocks / x.s;
    return x;
}

template <int BN, bool DEP, int UB>
__global__ void __launch_bounds__(kDynThreads, 1) w4a8_decode_dyn_kernel(const __grid_constant__ PParams p) {
    using C = DynCfg<BN, DEP, UB>;
    constexpr int kDynStages = C::kStages;
    constexpr int kStageBytes = C::kStageBytes;
    constexpr int kBBlockBytes = C::kBBlock;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kDynStages * kStageBytes);
    uint64_t* w_full = bars;
    uint64_t* w_empty = w_full + kDynStages;
    uint64_t* b_full = w_empty + kDynStages;
    uint64_t* a_full = b_full + kDynStages;
    uint64_t* a_empty = a_full + C::kAStages;
    uint64_t* d_full = a_empty + C::kAStages;
    uint64_t* d_empty = d_full + kDBufs;
    uint64_t* i_full = d_empty + kDBufs;
    uint64_t* i_empty = i_full + kItemSlots;
    int* items = reinterpret_cast<int*>(i_empty + kItemSlots);
    uint32_t* flag = reinterpret_cast<uint32_t*>(items + kItemSlots);
    uint32_t* tmem_slot = flag + 1;
    uint32_t* emax = tmem_slot + 1;  // [BN] the CTA's per-token max |y| of the current item
    // [2][64] token scales of the item (parity), 16-byte aligned for ld.shared.v4
    float* ssc = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(emax + 64) + 15) & ~uintptr_t(15));
    // [64] the B-quantizers' token row maxima (one global load per token per CTA: the
    // whole grid reading them per chunk hot-spotted their few L2 lines)
    uint32_t* qam = reinterpret_cast<uint32_t*>(ssc + 128);
    static_assert((3 * kDynStages + 2 * C::kAStages + 2 * kDBufs + 2 * kItemSlots) * 8 + kItemSlots * 4 + 8 + 64 * 4 +
                          16 + 128 * 4 + 64 * 4 <= 2048,
                  "barrier / item / scale region");
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    unsigned long long* trc = p.trace ? p.trace + blockIdx.x * kTraceCta : nullptr;
    // diagnostics: per-unit timeline of the LAST CTA (first 64 units, 8 slots each)
    unsigned long long* utr = (p.trace && blockIdx.x == gridDim.x - 1) ? p.trace + 148 * kTraceCta : nullptr;
    if (trc && threadIdx.x == 0) trc[0] = globaltimer();
    if (p.pdl) pdl_launch_dependents();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kDynStages; ++i) {
            mbar_init(&w_full[i], 1);
            mbar_init(&w_empty[i], 5);  // 4 converter warps read W, the MMA consumed B
            mbar_init(&b_full[i], 1);
        }
        for (int i = 0; i < C::kAStages; ++i) {
            mbar_init(&a_full[i], 4);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < kDBufs; ++i) {
            mbar_init(&d_full[i], 1);
            mbar_init(&d_empty[i], 4);
        }
        for (int i = 0; i < kItemSlots; ++i) {
            mbar_init(&i_full[i], 1);
            mbar_init(&i_empty[i], 1 + 4 * kDynConvGroups + 4);  // MMA, converter, epilogue warps
        }
        fence_mbar_init();
    }
    if (warp == kWarpAlloc) {
        tmem_alloc(tmem_slot, kTmemCols);
        tmem_relinquish();
    }
    if (threadIdx.x < BN) emax[threadIdx.x] = 0u;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = lds32(smem_u32(tmem_slot));
    if (trc && threadIdx.x == 0) trc[1] = globaltimer();

    if (warp == kWarpProducer) {
        // Lanes 0 and 1 issue alternate units of each item in SIMT lockstep (halves the
        // per-unit producer overhead); lane 0 fetches the items.
        if (lane < 2) {
            if (trc && lane == 0) trc[2] = globaltimer();
            const uint64_t pol = l2_policy_evict_first();
            const uint64_t pol_b = l2_policy_evict_last();
            // B tiles come from the act-quant kernel: units issued before griddepcontrol.wait
            // get their B tiles once it returns (each lane records its own)
            bool waited = p.pdl == 0;
            int dq[kDynStages], dst[kDynStages], dkb[kDynStages], dnb[kDynStages], ndef = 0;
            // programs quantize into a compact a8 layout (Mp == BN rows per k-block), so the B
            // tiles of a unit are one contiguous run
            auto issue_b = [&](const LinDesc& d, int s, int kb, int nb) {
                mbar_expect_tx(&b_full[s], nb * kBBlockBytes);
                if (d.Mp == BN) {  // compact a8 (BN rows per k-block): one contiguous run
                    bulk_g2s(ring + s * kStageBytes + C::kUBytes, d.qa + static_cast<size_t>(kb) * d.Mp * 128,
                             nb * kBBlockBytes, &b_full[s], pol_b);
                } else {           // 128-row padded a8 (an ody_qtensor): rows 0..BN-1 per k-block
                    for (int b = 0; b < nb; ++b)
                        bulk_g2s(ring + s * kStageBytes + C::kUBytes + b * kBBlockBytes,
                                 d.qa + static_cast<size_t>(kb + b) * d.Mp * 128, kBBlockBytes, &b_full[s], pol_b);
                }
            };
            auto release_deferred = [&]() {
                // The ring is full and the B tiles wait for the act quant (i.e. for the
                // previous launch to finish): keep HBM busy by pulling the weights of the
                // items most likely handed out next (second round) into L2 meanwhile.
                if (lane == 0)
                    for (int r2 = 1; r2 <= p.pf_units; ++r2) {
                        const int it2 = static_cast<int>(blockIdx.x + r2 * gridDim.x);
                        if (it2 >= p.n_items) break;
                        const DynItem y = dyn_item(p, p.lin, it2);
                        const LinDesc& d2 = p.lin[y.l];
                        bulk_prefetch_l2(d2.wp + (static_cast<size_t>(y.nt) * d2.kblocks + y.kb_lo) * kWBlockBytes,
                                         static_cast<uint32_t>(y.kb_hi - y.kb_lo) * kWBlockBytes);
                    }
                pdl_wait();
                waited = true;
                if (trc && lane == 0) trc[8] = globaltimer();
                for (int i = 0; i < ndef; ++i) issue_b(p.lin[dq[i]], dst[i], dkb[i], dnb[i]);
            };
            // DEP: the B tiles of a dependent linear come from its a8 buffer, which the
            // B-quantizer warps of every CTA fill once the producer linear completed (its
            // `qdone` reaches the k-block count -- only trusted after griddepcontrol.wait,
            // the previous launch re-arms the counters); until then the copies are deferred
            // and the weight stream keeps going.  Every blocking wait below polls so that a
            // released linear's copies go out meanwhile.
            int xq[DEP ? kDynStages : 1], xst[DEP ? kDynStages : 1], xkb[DEP ? kDynStages : 1],
                xnb[DEP ? kDynStages : 1], nx = 0;
            uint32_t rel_mask = 0u;
            auto released = [&](int l) -> bool {
                if ((rel_mask >> l) & 1u) return true;
                if (!waited) return false;
                const LinDesc& dl = p.lin[l];
                if (ld_acquire_u32(dl.qdone) < dl.qtarget) return false;
                fence_proxy_async_global();  // the quantizers' generic writes -> our bulk copies
                rel_mask |= 1u << l;
                if (trc && l < 4) trc[26 + l] = globaltimer();
                return true;
            };
            auto flush_x = [&]() {
                int keep = 0;
                for (int i = 0; i < nx; ++i) {
                    if (released(xq[i])) {
                        issue_b(p.lin[xq[i]], xst[i], xkb[i], xnb[i]);
                    } else {
                        xq[keep] = xq[i];
                        xst[keep] = xst[i];
                        xkb[keep] = xkb[i];
                        xnb[keep] = xnb[i];
                        ++keep;
                    }
                }
                nx = keep;
            };
            // Both issuing lanes wait TOGETHER (called convergently; `need` false for a lane
            // with nothing to wait on): each keeps flushing its own deferred copies while the
            // other waits, so neither can sit at the warp barrier holding a copy the other
            // lane's ring slot depends on.
            // The dependency counters are polled by lane 0 ONLY, with back-off: with most
            // CTAs waiting on one linear, per-role polling at ~100 ns saturated the L2 slice
            // holding the counter and slowed every CTA still streaming (trace: 2 us/unit).
            auto wait_poll = [&](uint64_t* bar, uint32_t par, bool need) {
                if (!DEP) {
                    if (need) mbar_wait(bar, par);
                    return;
                }
                uint32_t ns = 128;
                while (true) {
                    const bool ok = !need || mbar_test(bar, par);
                    if (__all_sync(0x3u, ok)) break;
                    const uint32_t want = nx ? (1u << xq[0]) : 0u;
                    const uint32_t want_all = (want | __shfl_xor_sync(0x3u, want, 1)) & ~rel_mask;
                    uint32_t newly = 0u;
                    if (lane == 0 && waited)
                        for (uint32_t m = want_all; m; m &= m - 1) {
                            const int l = __ffs(m) - 1;
                            if (ld_acquire_u32(p.lin[l].qdone) >= p.lin[l].qtarget) newly |= 1u << l;
                        }
                    newly = __shfl_sync(0x3u, newly, 0);
                    if (newly) {
                        fence_proxy_async_global();  // the quantizers' writes -> our bulk copies
                        rel_mask |= newly;
                        if (trc)
                            for (uint32_t m = newly; m; m &= m - 1)
                                if (__ffs(m) - 1 < 4) trc[26 + __ffs(m) - 1] = globaltimer();
                        flush_x();
                        ns = 128;
                    } else {
                        __nanosleep(ns);
                        ns = ns < 256 ? 2 * ns : 256;
                    }
                }
            };
            int U = 0;
            int cl = 0, ci = -1;  // static chain schedule: current linear, its item index
            for (int j = 0;; ++j) {
                const int is = j % kItemSlots;
                wait_poll(&i_empty[is], ((j / kItemSlots) & 1) ^ 1, j >= kItemSlots);
                // item 0 of every CTA is static (blockIdx.x), so the weight stream starts at
                // once; the shared counter is only touched after griddepcontrol.wait, i.e.
                // once the previous launch (which re-arms it) has completed
                int it = static_cast<int>(blockIdx.x);
                if (p.chain_static) {
                    // every linear runs alone between grid-wide completions: deal its items
                    // evenly (a dynamic grab lets idle CTAs hoard the next linear's items)
                    it = -1;
                    while (cl < p.L) {
                        const LinDesc& dl = p.lin[cl];
                        const int nl = dl.items;
                        const int C = static_cast<int>(gridDim.x);
                        const int i = ci < 0 ? ((static_cast<int>(blockIdx.x) - dl.off) % C + C) % C : ci + C;
                        if (i < nl) {
                            ci = i;
                            it = dl.ibase + i;
                            break;
                        }
                        ++cl;
                        ci = -1;
                    }
                    if (j > 0 && !waited) release_deferred();
                } else if (j > 0) {
                    if (!waited) release_deferred();
                    if (lane == 0) it = static_cast<int>(gridDim.x + atomicAdd(p.work, 1u));
                    it = __shfl_sync(0x3u, it, 0);
                }
                if (it >= p.n_items) it = -1;
                if (lane == 0) {
                    items[is] = it;
                    mbar_arrive(&i_full[is]);  // release: the item id is visible to the consumers
                }
                if (it < 0) break;
                if (trc && j == 0 && lane == 0) trc[3] = globaltimer();
                const DynItem x = dyn_item(p, p.lin, it);
                const LinDesc& d = p.lin[x.l];
                const uint8_t* wtile = d.wp + static_cast<size_t>(x.nt) * d.kblocks * kWBlockBytes;
                const int nunits = (x.kb_hi - x.kb_lo + C::kUB - 1) / C::kUB;
                if (trc && j == 0 && lane == 0) trc[30] = globaltimer() + (ld_keep(nunits) == -7 ? 1 : 0);
                // A dependent linear's B tiles are quantized in-kernel by the converters once
                // its producer linear completes.  While it has not, keep HBM streaming: pull
                // this whole item's weights into L2 (the ring then refills from L2).
                const bool depi = d.qdone != nullptr;
                if (depi && !p.no_item_pf && lane == 0 && ld_acquire_u32(d.qdone) < d.qtarget)
                    bulk_prefetch_l2(wtile + static_cast<size_t>(x.kb_lo) * kWBlockBytes,
                                     static_cast<uint32_t>(x.kb_hi - x.kb_lo) * kWBlockBytes);
                for (int k0 = 0; k0 < nunits; k0 += 2) {
#ifdef ODY_DIAG
                    // dbg 2048 / 4096: weights streamed before griddepcontrol.wait capped at
                    // 0 / 2 units (does the ring fill starve the act quant of memory bandwidth?)
                    if (!waited && (p.dbg & 2048)) release_deferred();
                    if (!waited && (p.dbg & 4096) && U + k0 >= 2) release_deferred();
#endif
                    if (!waited && U + k0 + 1 >= kDynStages) {
                        // the ring is full and the B tiles wait on the act quant (i.e. on the
                        // previous launch): pull the rest of this item into L2 meanwhile
                        if (p.rest_pf && lane == 0 && k0 + 2 < nunits) {
                            const int kb_r = x.kb_lo + C::kUB * (k0 + 2);
                            bulk_prefetch_l2(wtile + static_cast<size_t>(kb_r) * kWBlockBytes,
                                             static_cast<uint32_t>(x.kb_hi - kb_r) * kWBlockBytes);
                        }
                        release_deferred();
                    }
                    const int k = k0 + lane;
                    {
                        const int Uk = U + k;
                        wait_poll(&w_empty[Uk % kDynStages], ((Uk / kDynStages) & 1) ^ 1,
                                  k < nunits && Uk >= kDynStages);
                    }
                    if (k < nunits) {
                        const int Uk = U + k;
                        const int s = Uk % kDynStages;
                        const int kb = x.kb_lo + C::kUB * k;
                        const int nb = min(C::kUB, x.kb_hi - kb);
                        mbar_expect_tx(&w_full[s], nb * kWBlockBytes);
                        bulk_g2s(ring + s * kStageBytes, wtile + static_cast<size_t>(kb) * kWBlockBytes,
                                 nb * kWBlockBytes, &w_full[s], pol);
                        if (utr && Uk < 64) utr[8 * Uk + 0] = globaltimer();
                        if (trc && Uk == 0) trc[31] = globaltimer();
                        if (DEP && depi) {
                            if (released(x.l)) {
                                issue_b(d, s, kb, nb);
                            } else {
                                xq[nx] = x.l;
                                xst[nx] = s;
                                xkb[nx] = kb;
                                xnb[nx] = nb;
                                ++nx;
                            }
                        } else if (waited) {
                            issue_b(d, s, kb, nb);
                        } else {
                            dq[ndef] = x.l;
                            dst[ndef] = s;
                            dkb[ndef] = kb;
                            dnb[ndef] = nb;
                            ++ndef;
                        }
                    }
                    __syncwarp(0x3u);
                }
                U += nunits;
            }
            if (!waited) release_deferred();
            for (uint32_t ns = 128; nx;) {
                flush_x();
                if (nx) {
                    __nanosleep(ns);
                    ns = ns < 1024 ? 2 * ns : 1024;
                }
            }
            if (p.next_bytes > 0 && lane == 0) {
                // every own load is issued: stream this CTA's share of the NEXT launch's
                // weights (the caller's hint, e.g. the next linear of the layer) into L2,
                // so its ramp reads L2 and the HBM keeps streaming through this kernel's
                // drain, epilogues and the act quant in between
                const size_t share = (p.next_bytes / gridDim.x + 16383) & ~static_cast<size_t>(16383);
                const size_t lo = share * blockIdx.x;
                const size_t hi = min(p.next_bytes, lo + share);
                for (size_t off = lo; off < hi; off += 16384)
                    bulk_prefetch_l2(p.next_wp + off, static_cast<uint32_t>(min(static_cast<size_t>(16384), hi - off)));
            }
            if (trc && lane == 0) trc[6] = globaltimer();
        }
    } else if (warp == kWarpMma) {
        int U = 0, JD = 0;
        for (int j = 0;; ++j) {
            const int is = j % kItemSlots;
            mbar_wait(&i_full[is], (j / kItemSlots) & 1);
            const int it = items[is];
            __syncwarp();
            if (lane == 0) mbar_arrive(&i_empty[is]);
            if (it < 0) break;
            const DynItem x = dyn_item(p, p.lin, it);
            if (x.kb_hi <= x.kb_lo) continue;
            if (trc && lane == 0 && x.l < 4 && trc[10 + 4 * x.l] == 0) trc[10 + 4 * x.l] = globaltimer();
            const int db = JD % kDBufs;
            const uint32_t d_tmem = tmem + db * BN;
            mbar_wait(&d_empty[db], ((JD / kDBufs) & 1) ^ 1);
            tc_fence_after();
            for (int kb = x.kb_lo; kb < x.kb_hi; kb += C::kUB, ++U) {
                const int nb = min(C::kUB, x.kb_hi - kb);
                const int as = U % C::kAStages;
                const int s = U % kDynStages;
                mbar_wait(&a_full[as], (U / C::kAStages) & 1);
                if (utr && lane == 0 && U < 64) utr[8 * U + 1] = globaltimer();
                mbar_wait(&b_full[s], (U / kDynStages) & 1);
                if (utr && lane == 0 && U < 64) utr[8 * U + 6] = globaltimer();
                if (trc && lane == 0 && U == 0) trc[9] = globaltimer();  // first B tiles landed
                tc_fence_after();
                const uint32_t a_tmem = tmem + C::kAColBase + as * C::kAStageColsD;
                const uint32_t b0 = smem_u32(ring) + s * kStageBytes + C::kUBytes;
                if (elect_one()) {
#pragma unroll
                    for (int c = 0; c < 4 * C::kUB; ++c)
                        if (c < 4 * nb && !((p.dbg & 128) && (kb > x.kb_lo || c > 0)))  // dbg 128: first MMA only
                            mma_i8_ts(d_tmem, a_tmem + 8 * c, b_desc(b0 + (c / 4) * kBBlockBytes + 32 * (c % 4)),
                                      C::kIdesc, (kb > x.kb_lo || c > 0) ? 1u : 0u);
                    mma_commit(&a_empty[as]);
                    mma_commit(&w_empty[s]);
                    if (kb + nb >= x.kb_hi) mma_commit(&d_full[db]);
                }
                __syncwarp();
            }
            ++JD;
        }
    } else if (!DEP && warp == kWarpAlloc + 1) {
        // chain link: re-zero the row maxima this launch's act quant consumed (it completed:
        // griddepcontrol.wait) before the producer of the next step accumulates into them
        if (blockIdx.x == 0 && p.lin[0].amax_zero) {
            if (p.pdl) pdl_wait();
            for (int t = lane; t < p.lin[0].M; t += 32) p.lin[0].amax_zero[t * kAmaxStride] = 0u;
        }
    } else if (DEP && (warp == kWarpAlloc || warp == kWarpAlloc + 1)) {
        // B-quantizer (warps 2-3, idle once TMEM is allocated).  A DEPENDENT linear's x
        // is an earlier linear's 16-bit output.  Once that linear completed, x is
        // quantized ONCE for the whole grid: CTA c quantizes k-blocks c, c + grid, ... of
        // it (quant16: bit-exact with the act-quant kernel) into the linear's compact a8
        // buffer, then bumps its `qdone`; every item of the linear bulk-copies its B tiles
        // from there like an external linear's.  Token scale S = max/127 (IEEE; 0 -> 2^-24,
        // ref quantize.cpp:22-35) from the row maxima the producer linear's epilogues
        // accumulated.
        const int qt = threadIdx.x - kWarpAlloc * 32;  // 0..63
        if (p.pdl) pdl_wait();  // the counters are re-armed by the previous launch
        for (int l = 0; l < p.L; ++l) {
            const LinDesc& d = p.lin[l];
            if (d.qdone == nullptr) continue;
            if (qt == 0) {
                uint32_t ns = 64;
                while (ld_acquire_u32(d.dep_done) < d.dep_target) {
                    __nanosleep(ns);
                    ns = ns < 256 ? 2 * ns : 256;
                }
                if (trc && l < 4) trc[12 + 4 * l] = globaltimer();
            }
            named_bar_sync(4, 64);  // the producer completed (qt 0 acquired dep_done)
            if (qt < BN) qam[qt] = qt < d.M ? __ldcg(d.amax_src + qt * kAmaxStride) : 0u;
            named_bar_sync(4, 64);
            // CTA c owns an even share [lo, hi) of the x's kblocks x BN x 8 sixteen-element
            // chunks (a k-block per CTA left most CTAs idle and made the grid wait on the
            // few that quantized: ~1-2 chunks per thread is one L2 round trip)
            const int nchunks = d.kblocks * BN * 8;
            const int lo = static_cast<int>((static_cast<long long>(nchunks) * blockIdx.x) / gridDim.x);
            const int hi = static_cast<int>((static_cast<long long>(nchunks) * (blockIdx.x + 1)) / gridDim.x);
            {
                for (int task0 = lo; task0 < hi; task0 += 4 * 64) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int task = task0 + u * 64 + qt;
                    if (task >= hi) break;
                    const int kb = task / (BN * 8);
                    const int t = (task >> 3) % BN, c = task & 7;
                    const int k0 = kb * kBlockK + c * 16;
                    uint4 v = make_uint4(0u, 0u, 0u, 0u);
                    if (t < d.M && k0 < d.K) {
                        float sc = __uint_as_float(qam[t]) / 127.0f;
                        if (!(sc > 0.0f)) sc = kMinScale;
                        const unsigned short* row = static_cast<const unsigned short*>(d.x) + static_cast<size_t>(t) * d.ldx;
                        uint4 r0, r1;
                        if (k0 + 16 <= d.K) {
                            r0 = __ldcg(reinterpret_cast<const uint4*>(row + k0));
                            r1 = __ldcg(reinterpret_cast<const uint4*>(row + k0 + 8));
                        } else {
                            uint32_t w[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) {
                                const uint32_t lo = k0 + 2 * e < d.K ? __ldcg(row + k0 + 2 * e) : 0u;
                                const uint32_t hi = k0 + 2 * e + 1 < d.K ? __ldcg(row + k0 + 2 * e + 1) : 0u;
                                w[e] = lo | (hi << 16);
                            }
                            r0 = make_uint4(w[0], w[1], w[2], w[3]);
                            r1 = make_uint4(w[4], w[5], w[6], w[7]);
                        }
                        v = d.x_bf16 ? quant16<true>(r0, r1, sc, 1.0f / sc, 0) : quant16<false>(r0, r1, sc, 1.0f / sc, 0);
                    }
                    if (trc && p.L == 1 && qt == 0 && u == 0 && task0 == lo) trc[14] = globaltimer() + (v.x == 0x7fffffffu);
                    *reinterpret_cast<uint4*>(const_cast<int8_t*>(d.qa) + static_cast<size_t>(kb) * BN * 128 + t * 128 +
                                              ((c ^ (t & 7)) << 4)) = v;
                }
                }
            }
            // no writer-side proxy fence: each consumer orders its bulk copies (async proxy)
            // after its acquire of qdone with fence.proxy.async (the `released` check); the
            // release below publishes these generic stores at gpu scope.  Every CTA counts
            // once (qtarget = the grid).
            if (trc && p.L == 1 && qt == 0) trc[15] = globaltimer();
            named_bar_sync(4, 64);
            if (trc && p.L == 1 && qt == 0) trc[16] = globaltimer();
            if (qt == 0) red_release_add_u32(d.qdone, 1u);
            if (trc && qt == 0 && l < 4) trc[13 + 4 * l] = globaltimer();
        }
    } else if (warp >= kWarpConv0 && warp < kWarpConv0 + 4 * kDynConvGroups) {
        const int q = warp & 3;
        const int r = 32 * q + lane;
        const int grp = (warp - kWarpConv0) / 4;
        int U = 0;
        for (int j = 0;; ++j) {
            const int is = j % kItemSlots;
            mbar_wait(&i_full[is], (j / kItemSlots) & 1);
            const int it = items[is];
            __syncwarp();
            if (lane == 0) mbar_arrive(&i_empty[is]);
            if (it < 0) break;
            const DynItem x = dyn_item(p, p.lin, it);
            for (int kb = x.kb_lo; kb < x.kb_hi; kb += C::kUB, ++U) {
                // the group owning ring stage U % kDynStages widens this unit (stage
                // ownership keeps every w_full waiter in phase order on odd-length rings)
                if ((U % kDynStages) % kDynConvGroups != grp) continue;
                const int nb = min(C::kUB, x.kb_hi - kb);
                const int s = U % kDynStages;
                const int as = U % C::kAStages;
                mbar_wait(&w_full[s], (U / kDynStages) & 1);
                if (utr && r == 0 && U < 64) utr[8 * U + 4] = globaltimer();
                const uint32_t src = smem_u32(ring) + s * kStageBytes + r * 16;
                mbar_wait(&a_empty[as], ((U / C::kAStages) & 1) ^ 1);
                tc_fence_after();
                const uint32_t dst = tmem + (static_cast<uint32_t>(32 * q) << 16) + C::kAColBase + as * C::kAStageColsD;
                // two k-blocks at a time (64 words in registers), each straight to TMEM
#pragma unroll
                for (int h = 0; h < C::kUB; h += 2) {
                    if (h < nb) {
                        uint32_t lanes8[2][32];
#pragma unroll
                        for (int b2 = 0; b2 < 2; ++b2) {
                            const int b = h + b2;
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                const uint4 v = (b < nb && !(p.dbg & 512)) ? lds128(src + b * kWBlockBytes + c * 2048)
                                                                           : make_uint4(0u, 0u, 0u, 0u);
                                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                                for (int jj = 0; jj < 4; ++jj) {
                                    lanes8[b2][c * 8 + 2 * jj] = (w[jj] << 4) & 0xF0F0F0F0u;  // k 8jj+0..3
                                    lanes8[b2][c * 8 + 2 * jj + 1] = w[jj] & 0xF0F0F0F0u;     // k 8jj+4..7
                                }
                            }
                        }
                        if (!(p.dbg & 256)) {  // dbg 256 (diag build): no TMEM stores
                            tmem_st_32x32b_x32(dst + 32 * h, lanes8[0]);
                            if (h + 1 < nb) tmem_st_32x32b_x32(dst + 32 * h + 32, lanes8[1]);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&w_empty[s]);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[as]);
                if (utr && lane == 0 && U < 64) utr[8 * U + (q == 0 ? 5 : (q == 1 ? 2 : (q == 2 ? 3 : 7)))] = globaltimer();
            }
        }
    } else if (warp >= kDynEpi0) {
        const int q = warp & 3;
        const int r = 32 * q + lane;
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(32 * q) << 16);
        int JD = 0, cur_l = -1;
        // diagnostics: per-item epilogue timeline of the LAST CTA (first 32 items, 8 slots)
        unsigned long long* etr = utr ? utr + 64 * 8 : nullptr;
        auto emark = [&](int j2, int slot) {
            if (etr && r == 0 && j2 < 32) etr[16 * j2 + slot] = globaltimer();
        };
        for (int j = 0;; ++j) {
            const int is = j % kItemSlots;
            mbar_wait(&i_full[is], (j / kItemSlots) & 1);
            const int it = items[is];
            __syncwarp();
            if (lane == 0) mbar_arrive(&i_empty[is]);
            if (it < 0) break;
            const DynItem x = dyn_item(p, p.lin, it);
            const LinDesc& d = p.lin[x.l];
            if (cur_l < 0 && p.pdl) pdl_wait();  // token scales come from the act-quant kernel
            cur_l = x.l;
            const int n = x.nt * kTileN + r;
            const float sw_n = n < d.N ? __ldg(d.sw + n) : 0.0f;  // in flight during the wait
            uint32_t v[BN];
            if (x.kb_hi > x.kb_lo) {
                const int db = JD % kDBufs;
                mbar_wait(&d_full[db], (JD / kDBufs) & 1);
                emark(j, 0);
                tc_fence_after();
#pragma unroll
                for (int tc = 0; tc < BN; tc += 16) {
                    uint32_t w16[16];
                    tmem_ld_32x32b_x16(t_lane + db * BN + tc, w16);
                    tmem_wait_ld();
#pragma unroll
                    for (int t = 0; t < 16; ++t) v[tc + t] = w16[t];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&d_empty[db]);
                ++JD;
            } else {
#pragma unroll
                for (int t = 0; t < BN; ++t) v[t] = 0u;
            }
            // Token scales, staged once per item in smem (a per-token global load inside the
            // store loop below cannot be hoisted past the output stores: 16 serial L2 round
            // trips).  A dependent linear's scales follow from its producer's row maxima exactly
            // as the B-quantizers derived them (complete by now: the MMAs consumed B tiles
            // quantized after the producer finished; one acquire).
            emark(j, 1);
            const bool depi = d.qdone != nullptr;
            float* tsc = ssc + (j & 1) * 64;
            if (depi) {
                // no acquire needed here: the producer linear's row-max atomics precede its
                // `done` release, which the B-quantizers acquired before releasing `qdone`,
                // which the producer warp acquired before the B copies this item's MMAs
                // consumed (mbarrier chain to d_full): the maxima are final in L2
                if (r < d.M) {
                    float sc = __uint_as_float(__ldcg(d.amax_src + r * kAmaxStride)) / 127.0f;
                    if (!(sc > 0.0f)) sc = kMinScale;
                    tsc[r] = sc;
                }
            } else if (r < d.M) {
                tsc[r] = __ldg(d.sa + r);
            }
            emark(j, 2);
            bool fin = true;
            if (x.s > 1) {
                // Per-ROW last-arriver reduction, no barrier and no waiting: thread r stores
                // its row's partial into this item's slot, then an acq_rel increment of the
                // row's counter (release: the store is visible before the count; acquire:
                // the last arriver sees every other split's row).  The thread that arrives
                // last for row r adds the other splits' rows and stores the outputs.  The
                // row counters live in the program's zero region (p.acc, unused by this
                // kernel) and are re-zeroed by their last arriver.
                int32_t* part = p.part + static_cast<size_t>(it) * BN * kTileN;  // [t][row]
#pragma unroll
                for (int t = 0; t < BN; ++t)
                    if (t < d.M) __stcg(part + t * kTileN + r, static_cast<int32_t>(v[t]));
                uint32_t* rc = reinterpret_cast<uint32_t*>(p.acc) + static_cast<size_t>(d.tbase + x.nt) * kTileN + r;
                const uint32_t old = atom_add_acq_rel_u32(rc, 1u);
                fin = old == static_cast<uint32_t>(x.s - 1);
                emark(j, 3);
                if (fin) {
                    // the other splits' rows, kPer splits' loads in flight per round trip
                    constexpr int kPer = BN >= 32 ? 1 : 32 / BN;
                    const int32_t* p0 = p.part + static_cast<size_t>(d.ibase + x.i0) * BN * kTileN;
#pragma unroll 1
                    for (int s0 = 0; s0 < x.s; s0 += kPer) {
                        uint32_t add[kPer][BN];
#pragma unroll
                        for (int j2 = 0; j2 < kPer; ++j2) {
                            const int s2 = s0 + j2;
                            const bool use = s2 < x.s && s2 != x.r;
#pragma unroll
                            for (int t = 0; t < BN; ++t)
                                add[j2][t] = (use && t < d.M)
                                                 ? static_cast<uint32_t>(__ldcg(p0 + (s2 * BN + t) * kTileN + r))
                                                 : 0u;
                        }
#pragma unroll
                        for (int j2 = 0; j2 < kPer; ++j2)
#pragma unroll
                            for (int t = 0; t < BN; ++t) v[t] += add[j2][t];
                    }
                    *rc = 0u;  // every split of this row arrived: re-armed for the next launch
                }
            }
            emark(j, 4);
            named_bar_sync(3, 128);  // tsc complete (the other parity buffer is still in use)
            emark(j, 8);
            // The descriptor fields used per token, hoisted into registers once: read through a
            // run-time linear index they compile to indexed LDC, re-issued for every token
            // (rematerialised rather than kept live) at ~0.3 us per token on this path.
            const int m_rows = ld_keep(d.M);
            const int n_cols = ld_keep(d.N);
            const int odt = ld_keep(d.out_dtype);
            uint8_t* const outp = ld_keep_ptr(static_cast<uint8_t*>(d.out));
            int32_t* const accp = ld_keep_ptr(d.acc_out);
            float* const sa_outp = (depi && x.nt == 0 && r == 0) ? ld_keep_ptr(d.sa_out) : nullptr;
            emark(j, 9);
            const bool amx_on = d.amax_dst != nullptr;
            const bool own = fin && n < n_cols;
            const bool amx = amx_on && n >= d.amax_c0 && n < d.amax_c1;
            if (sa_outp && own)
                for (int t = 0; t < m_rows; ++t) stg_b32(sa_outp + t, __float_as_uint(tsc[t]));
            const uint32_t emax_a = smem_u32(emax);
            if (accp) {
                epi_store<BN, -1, false>(v, tsc, sw_n, m_rows, n_cols, n, own, false, accp, emax_a, lane);
            } else if (odt == kDtypeF32) {
                epi_store<BN, kDtypeF32, false>(v, tsc, sw_n, m_rows, n_cols, n, own, false, outp, emax_a, lane);
            } else if (odt == kDtypeF16) {
                if (amx_on)
                    epi_store<BN, kDtypeF16, true>(v, tsc, sw_n, m_rows, n_cols, n, own, amx, outp, emax_a, lane);
                else
                    epi_store<BN, kDtypeF16, false>(v, tsc, sw_n, m_rows, n_cols, n, own, false, outp, emax_a, lane);
            } else {
                if (amx_on)
                    epi_store<BN, kDtypeBF16, true>(v, tsc, sw_n, m_rows, n_cols, n, own, amx, outp, emax_a, lane);
                else
                    epi_store<BN, kDtypeBF16, false>(v, tsc, sw_n, m_rows, n_cols, n, own, false, outp, emax_a, lane);
            }
            emark(j, 5);
            if (trc && r == 0 && x.l < 4) trc[11 + 4 * x.l] = globaltimer();
            if (d.done != nullptr || amx_on) {
                // publish: every store (and row-max contribution) of this item happens
                // before the release increment the dependent linear acquires.  One global
                // atomicMax per token per item, each token on its own 128-byte line (the
                // whole grid's items hit these few addresses: same-line atomics serialise).
                // A chain link launch (no `done`: its consumer is the NEXT launch, ordered
                // by kernel completion) only contributes the row maxima.
                named_bar_sync(3, 128);
                if (amx_on && r < d.M) {
                    const uint32_t m = emax[r];
                    emax[r] = 0u;
                    if (m != 0u) atomicMax(d.amax_dst + r * kAmaxStride, m);
                }
                if (amx_on) named_bar_sync(3, 128);
                emark(j, 6);
                if (r == 0 && d.done) red_release_add_u32(d.done, 1u);  // cumulative over the CTA barrier
                emark(j, 7);
            }
        }
        if (trc && r == 0) trc[4] = globaltimer();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kWarpAlloc) tmem_dealloc(tmem, kTmemCols);
    if (threadIdx.x == 0 && p.reset_at_exit) {
        // the last CTA out re-arms the item counter for the next launch (a lone linear is
        // dealt statically and skips this: the exit atomic is an L2 round trip every CTA
        // pays before the grid can complete)
        __threadfence();
        if (atomicAdd(p.ctr + kMaxLin, 1u) == gridDim.x - 1) {
            *p.work = 0u;
            p.ctr[kMaxLin] = 0u;
            for (int l = 0; l < p.L; ++l) {  // chain state of this launch (zero region)
                if (p.lin[l].done) *p.lin[l].done = 0u;
                if (p.lin[l].qdone) *p.lin[l].qdone = 0u;
                if (p.lin[l].amax_reset)
                    for (int t = 0; t < p.lin[l].M; ++t) p.lin[l].amax_reset[t * kAmaxStride] = 0u;
            }
            __threadfence();
        }
    }
    if (trc && threadIdx.x == 0) trc[5] = globaltimer();
}

// K1 for the external activations of a program: one 128-thread CTA per token row,
// each thread holding its <= 7 sixteen-element chunks PACKED (8 registers per chunk) across
// the max pass and the quantize pass (quant16: the exact fast path + IEEE redo).  Small
// enough (<= 80 registers x 128 threads, no shared arrays beyond 16 B) to stay
// co-resident with a running decode program CTA, so in the PDL chain program -> K1 ->
// program the next program's CTAs take every SM the previous one frees.
template <int BN, bool DEP, int UB>
cudaError_t ensure_dyn_attr() {
    static std::once_flag once;
    static cudaError_t err = cudaSuccess;
    std::call_once(once, [] {
        err = cudaFuncSetAttribute(w4a8_decode_dyn_kernel<BN, DEP, UB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   DynCfg<BN, DEP, UB>::kSmem);
    });
    return err;
}

// rb != NULL: first the batched activation quant (rb_rows token rows, act_quant_rows_kernel),
// then the GEMM, PDL-chained.  (Measured: the same act quant as a mode of this kernel
// function -- warm instruction caches for the GEMM launch -- made no difference.)
// Dynamic shared memory the act-quant kernel reserves so it never shares an SM with a
// decode CTA (launch_dyn); diagnostics: ODY_ACT_SMEM overrides (0 = co-reside).
size_t act_excl_smem() {
    static const char* env = ODY_DIAG_ENV("ODY_ACT_SMEM");
    static const size_t v = env ? static_cast<size_t>(std::atoi(env)) : 0;
    return v;
}

cudaError_t launch_premax(const RowBatch& rb, int rows, cudaStream_t st) {
    cudaLaunchConfig_t acfg = {};
    acfg.gridDim = dim3(rows * kPreCtas);
    acfg.blockDim = dim3(kPreThreads);
    acfg.stream = st;
    cudaLaunchAttribute aattr;
    aattr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    aattr.val.programmaticStreamSerializationAllowed = 1;
    acfg.attrs = &aattr;
    acfg.numAttrs = rb.pdl ? 1 : 0;
    return cudaLaunchKernelEx(&acfg, act_quant_premax_kernel, rb);
}

template <int BN, bool DEP, int UB>
cudaError_t launch_dyn(const PParams& p, bool pdl, cudaStream_t st, const RowBatch* rb = nullptr, int rb_rows = 0) {
    const cudaError_t ed = ensure_dyn_attr<BN, DEP, UB>();
    if (ed != cudaSuccess) return ed;
    if (rb) {
        cudaLaunchConfig_t acfg = {};
        acfg.gridDim = dim3(rb_rows);
        acfg.blockDim = dim3(kRowThreads);
        acfg.stream = st;
        // Keep the act quant off SMs that hold a decode CTA: its x loads would queue behind
        // that CTA's ring fill (~160 KiB per SM at the SM's HBM share: ~3.6 us).  Reserving
        // more shared memory than a decode CTA leaves free places it on idle SMs only.
        acfg.dynamicSmemBytes = act_excl_smem();
        cudaLaunchAttribute aattr;
        aattr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
        aattr.val.programmaticStreamSerializationAllowed = 1;
        acfg.attrs = &aattr;
        acfg.numAttrs = rb->pdl ? 1 : 0;
        const cudaError_t ea = cudaLaunchKernelEx(&acfg, act_quant_rows_kernel, *rb);
        if (ea != cudaSuccess) return ea;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.C);
    cfg.blockDim = dim3(kDynThreads);
    cfg.dynamicSmemBytes = DynCfg<BN, DEP, UB>::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, w4a8_decode_dyn_kernel<BN, DEP, UB>, p);
}

int dyn_bn(int M) { return M <= 16 ? 16 : (M <= 32 ? 32 : 64); }

cudaError_t ensure_decode_attr() {
    static std::once_flag once;
    static cudaError_t err = cudaSuccess;
    std::call_once(once, [] {
        err = cudaFuncSetAttribute(w4a8_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    });
    return err;
}

// How many clusters of S decode CTAs (one per SM) can be co-resident: clusters must fit
// inside one GPC, so e.g. S = 7 leaves SMs of every GPC idle.  Cached per S.
int max_active_clusters(int S) {
    static int cache[kMaxSplit + 1] = {-1, -1, -1, -1, -1, -1, -1, -1, -1};
    if (S < 1 || S > kMaxSplit) return 0;
    if (cache[S] >= 0) return cache[S];
    int n = 0;
    if (ensure_decode_attr() == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(S * 64);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kSmemBytes;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = S;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&n, w4a8_decode_kernel, &cfg) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
    }
    static const bool plan_log = ODY_DIAG_ENV("ODY_PLAN_LOG") != nullptr;
    if (plan_log) std::fprintf(stderr, "[ody] decode: max active clusters of %d = %d\n", S, n);
    cache[S] = n;
    return n;
}

// Decode-width linear the program kernels accept: M <= 64 (the dynamic kernel; the
// cluster kernel that quantizes dependent activations in-kernel takes M <= 16).
bool lin_ok(const LinearArgs& a, bool external = true) {
    // external x goes through the batched act-quant kernel (K <= 14336); a dependent
    // linear's x is quantized in-kernel by the B-quantizer warps (any K <= 2^17)
    return a.M >= 1 && a.M <= 64 && a.N >= 1 && a.K >= 1 &&
           (!external || a.K <= kRowThreads * kRowChunks * 16) &&
           (a.x_dtype == kDtypeF16 || a.x_dtype == kDtypeBF16) &&
           (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && (a.ldx * 2) % 16 == 0 &&
           (reinterpret_cast<uintptr_t>(a.sw) & 15) == 0;
}

}  // namespace

static size_t program_tiles(const LinearArgs* a, int L) {
    size_t t = 0;
    for (int l = 0; l < L; ++l) t += pad_n(a[l].N) / kTileN;
    return t;
}
constexpr size_t kAccOffset = kProgramCounterRegion + kProgramMaxTiles * 4;
// chain state inside the counter region: done[kMaxLin] at u32 64, row maxima [kMaxLin][64]
constexpr int kChainDoneU32 = 64;
constexpr size_t kChainAmaxOffset = 4096;
constexpr int kChainMaxM = 64;
static_assert(kChainAmaxOffset + kMaxLin * kChainMaxM * kAmaxStride * 4 <= kProgramCounterRegion, "counter region");
// the last 4 KiB of the zero region are the two-kernel GEMM's stream-K counters when the
// same scratch serves ody_dev_w4a8_linear's fallback (kLinearGemmCounters)
constexpr size_t kZeroRegion = kAccOffset + kProgramMaxTiles * kBN * kTileN * 4 + kLinearGemmCounters;
size_t program_zero_bytes() { return kZeroRegion; }

// A dependency chain runs on the dynamic kernel when every dependent linear's x is a
// column slice [c0, c0 + K) of its producer's 16-bit output (same tokens, row stride = the
// producer's N) and every producer feeds one dependent linear: the producer's epilogues
// then accumulate the slice's per-token max and the consumer quantizes in-kernel.
static bool dyn_chain_slice(const LinearArgs* a, const int* deps, int L, int l, int* c0) {
    const int d = deps[l];
    if (d < 0 || d >= l) return false;
    const LinearArgs& x = a[l];
    const LinearArgs& y = a[d];
    if (y.acc_out || x.absmax_in) return false;
    if (x.x_dtype != y.out_dtype || (x.x_dtype != kDtypeF16 && x.x_dtype != kDtypeBF16)) return false;
    if (x.M != y.M || x.ldx != static_cast<size_t>(y.N)) return false;
    const std::ptrdiff_t off = static_cast<const uint8_t*>(x.x) - static_cast<const uint8_t*>(y.out);
    if (off < 0 || off % 2 != 0) return false;
    const std::ptrdiff_t col = off / 2;
    if (col + x.K > y.N) return false;
    *c0 = static_cast<int>(col);
    return true;
}
static bool dyn_chain_ok(const LinearArgs* a, const int* deps, int L) {
    if (!deps) return true;
    int consumers[kMaxLin] = {};
    for (int l = 0; l < L; ++l) {
        if (deps[l] < 0) continue;
        int c0;
        if (!dyn_chain_slice(a, deps, L, l, &c0)) return false;
        if (++consumers[deps[l]] > 1) return false;
    }
    return true;
}

// Cluster split S (uniform over the program) and cluster count C: minimise the busiest
// CTA's k-blocks -- per linear for a dependency chain, over the whole program (tiles
// rotated across clusters) for independent linears -- plus a small activation-prologue
// term per linear; subject to the resident-B bound ceil(kb / S) <= kMaxKbPerCta.
DecodePlan plan_program(const LinearArgs* a, const int* deps, int L, int sms) {
    DecodePlan best = {};
    if (L < 1 || L > kMaxLin) return best;
    bool chain = false;
    int max_tiles = 0;
    if (program_tiles(a, L) > kProgramMaxTiles) return best;
    for (int l = 0; l < L; ++l) {
        if (!lin_ok(a[l], !(deps && deps[l] >= 0))) return best;
        chain |= deps && deps[l] >= 0;
        max_tiles = std::max(max_tiles, static_cast<int>(pad_n(a[l].N) / kTileN));
    }
    static const char* dyn_env = ODY_DIAG_ENV("ODY_PROGRAM_DYN");  // diagnostics: 0 = static schedule
    const bool dyn_allowed = !(dyn_env && dyn_env[0] == '0');
    if (chain && !(dyn_allowed && dyn_chain_ok(a, deps, L))) {
        for (int l = 0; l < L; ++l)  // the static cluster kernel: in-kernel K1 for M <= 16,
            if (a[l].M > kBN || a[l].absmax_in || a[l].acc_out) return best;  // f16/bf16 out only
    }
    if (!chain || (dyn_allowed && dyn_chain_ok(a, deps, L))) {  // dynamic schedule: one CTA per SM
        best = {1, std::min(sms, 1 << 20), std::min(sms, 1 << 20)};
        return best;
    }
    double best_cost = 0;
    for (int S = 1; S <= kMaxSplit; ++S) {
        bool ok = true;
        for (int l = 0; l < L; ++l)
            ok &= (static_cast<int>(pad_k(a[l].K) / kBlockK) + S - 1) / S <= kMaxKbPerCta;
        if (!ok) continue;
        int C = sms / S;
        if (C < 1) break;
        if (sms >= device_sm_count()) C = std::min(C, max_active_clusters(S));  // one wave
        C = std::min(C, max_tiles);
        if (C < 1) continue;
        double cost = 0, total = 0;
        for (int l = 0; l < L; ++l) {
            const int kb = static_cast<int>(pad_k(a[l].K) / kBlockK);
            const int nt = static_cast<int>(pad_n(a[l].N) / kTileN);
            const int kbpc = (kb + S - 1) / S;
            const double pro = 0.25 * a[l].M / 16.0 * kbpc;  // activation prologue, per linear
            if (chain)
                cost += static_cast<double>((nt + C - 1) / C) * kbpc + pro;
            else {
                total += static_cast<double>(nt) * kbpc;
                cost += pro;
            }
        }
        if (!chain) cost += std::ceil(total / C);
        if (best.S == 0 || cost < best_cost - 1e-9) {
            best = {S, C, S * C};
            best_cost = cost;
        }
    }
    return best;
}

// Dynamic schedule: k-splits per tile so a work item streams <= 48 k-blocks (384 KiB).
static int dyn_split(int kblocks) {
    static const char* env = ODY_DIAG_ENV("ODY_DYN_KB");  // diagnostics: target k-blocks per item
    // measured (tools/program_trace.py, LLaMA-13B layer): whole 40-block tiles for
    // K = 5120 and 3 splits of 36 blocks for K = 13824 beat finer splits, whose L2 partial
    // round trips make the epilogue the bottleneck
    static const int target = env ? std::max(1, std::atoi(env)) : 56;
    return std::max(1, (kblocks + target - 1) / target);
}
// A linear that runs alone (a lone launch, or a chain link between two grid-wide
// completions) is split along K only as far as ONE wave of items allows: s = floor(CTAs /
// tiles), at least 1, and items of >= 4 k-blocks.  Measured per forced split
// (tools/single_linear_ab.py, M = 16, us): 4096^2 12.7 / 11.3 / 11.1 / 10.8 (s = 4 = 148/32)
// / 15.1; o 14.4 / 13.0 / 12.0 (s = 3) / 16.1; qkv and gate_up best unsplit (15.6, 23.0;
// 17.7, 26.5 at s = 2); down 27.8 / 21.9 / 19.1 (s = 3) / 22.8 -- a second item per CTA
// costs more (its pipeline ramp and epilogue round trips) than the balance it buys.
static int chain_split(int n_tiles, int kblocks, int sms) {
    static const char* env = ODY_DIAG_ENV("ODY_CHAIN_SPLIT");  // diagnostics: fixed split
    if (env) return std::max(1, std::min(std::atoi(env), kblocks));
    return std::max(1, std::min({sms / std::max(n_tiles, 1), kblocks / 4, 8}));
}
// Uniform k-split s for every tile of d.
static int split_uniform(LinDesc& d, int s) {
    d.split = s;
    d.t1 = d.n_tiles;
    d.split2 = 1;
    d.items = d.n_tiles * s;
    return d.items;
}
// A linear that runs alone, dealt round-robin over `sms` CTAs: chain_split's k-split, and
// when it leaves a partial last wave of whole tiles (n_tiles > sms, e.g. gate_up's 216
// tiles on 148 SMs: 68 CTAs stream two whole tiles while 80 stream one) the tiles of that
// wave are cut into split2 pieces spread over all CTAs -- the busiest CTA streams
// kb + ceil(R * s2 / sms) * kb / s2 blocks instead of 2 * kb.
static int split_alone(LinDesc& d, int sms) {
    const int s = chain_split(d.n_tiles, d.kblocks, sms);
    split_uniform(d, s);
    static const char* env = ODY_DIAG_ENV("ODY_TAIL_SPLIT");  // diagnostics: 0 = off, n = forced split2
    const int forced = env ? std::atoi(env) : -1;
    if (s != 1 || d.n_tiles <= sms || d.n_tiles % sms == 0 || forced == 0) return d.items;
    const int R = d.n_tiles % sms;
    int best = 1;
    long long best_cost = static_cast<long long>((R + sms - 1) / sms) * d.kblocks;
    for (int s2 = 2; s2 <= 8 && d.kblocks / s2 >= 4; ++s2) {
        const long long cost = static_cast<long long>((R * s2 + sms - 1) / sms) * ((d.kblocks + s2 - 1) / s2);
        if (cost < best_cost) {
            best_cost = cost;
            best = s2;
        }
    }
    if (forced > 0) best = std::min(forced, std::min(8, d.kblocks));
    d.t1 = d.n_tiles - R;
    d.split2 = best;
    d.items = d.t1 + R * best;
    return d.items;
}
static size_t dyn_items(const LinearArgs* a, int L) {
    // upper bound over the tail refinement (any linear may be the tail one, <= 12-block
    // items) and the chain split (<= 8)
    size_t n = 0;
    for (int l = 0; l < L; ++l) {
        const int kb = static_cast<int>(pad_k(a[l].K) / kBlockK);
        const int nt = static_cast<int>(pad_n(a[l].N) / kTileN);
        n += static_cast<size_t>(nt) * std::max(std::max(dyn_split(kb), (kb + 11) / 12), std::min(8, kb));
    }
    return n;
}

DecodePlan plan_decode(int M, int N, int K, int sms) {
    LinearArgs a = {};
    a.M = M;
    a.N = N;
    a.K = K;
    a.x_dtype = kDtypeF16;
    static const float dummy_sw[4] = {0, 0, 0, 0};
    a.sw = dummy_sw;
    static const uint4 dummy_x = {};
    a.x = &dummy_x;
    a.ldx = 8;
    return plan_program(&a, nullptr, 1, sms);
}

bool decode_eligible(int M, int N, int K, int x_dtype, int num_sms) {
    if (x_dtype != kDtypeF16 && x_dtype != kDtypeBF16) return false;
    const int sms = num_sms > 0 ? num_sms : device_sm_count();
    return plan_decode(M, N, K, sms).S > 0;
}

bool program_eligible(const LinearArgs* a, const int* deps, int L, int num_sms) {
    const int sms = num_sms > 0 ? num_sms : device_sm_count();
    return plan_program(a, deps, L, sms).S > 0;
}

// Scratch: [dependency counters][split-K arrival counters][split-K accumulators] -- a
// FIXED-size zero region (zeroed once; every launch leaves it zeroed), so scratch
// shared by programs of different shapes never lands transient data in it --
// [a8 codes + scales of the external x].
size_t program_scratch_bytes(const LinearArgs* a, const int* deps, int L) {
    int mmax = 1;
    for (int l = 0; l < L; ++l) mmax = std::max(mmax, a[l].M);
    size_t b = kZeroRegion + dyn_items(a, L) * dyn_bn(mmax) * kTileN * 4;  // + split partials
    for (int l = 0; l < L; ++l) {
        if (!deps || deps[l] < 0)
            b += round_up(a8_bytes(a[l].M, a[l].K), 256) + round_up(pad_m(a[l].M) * 4, 256);
        else  // dependency chain: the quantized x (compact a8, BN rows) + its token scales
            b += round_up(static_cast<size_t>(dyn_bn(mmax)) * pad_k(a[l].K), 256) + round_up(pad_m(a[l].M) * 4, 256);
    }
    return b;
}

cudaError_t launch_w4a8_program(const LinearArgs* a, const int* deps, int L, void* scratch, size_t scratch_bytes,
                                bool pdl, const uint8_t* next_wp, size_t next_bytes, cudaStream_t st) {
    const int sms = a[0].max_ctas > 0 ? a[0].max_ctas : device_sm_count();
    const DecodePlan pl = plan_program(a, deps, L, sms);
    if (pl.S == 0) return cudaErrorInvalidValue;
    if (!scratch || scratch_bytes < program_scratch_bytes(a, deps, L)) return cudaErrorInvalidValue;
    const cudaError_t e = ensure_decode_attr();
    if (e != cudaSuccess) return e;
    PParams p = {};
    p.L = L;
    p.S = pl.S;
    p.C = pl.C;
    bool chain = false;
    for (int l = 0; l < L; ++l) chain |= deps && deps[l] >= 0;
    // External activations are quantized up front by ONE batched K1 launch into the
    // scratch (a8 layout); the program kernel then streams their B tiles with the weights.
    if (program_tiles(a, L) > kProgramMaxTiles) return cudaErrorInvalidValue;
    p.tile_cnt = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + kProgramCounterRegion);
    p.acc = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(scratch) + kAccOffset);
    p.part = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(scratch) + kZeroRegion);
    int mmax_s = 1;
    for (int l = 0; l < L; ++l) mmax_s = std::max(mmax_s, a[l].M);
    uint8_t* cursor = static_cast<uint8_t*>(scratch) + kZeroRegion + dyn_items(a, L) * dyn_bn(mmax_s) * kTileN * 4;
    int nb = 0;
    const void* bx[kMaxLin];
    int bdt[kMaxLin], bm[kMaxLin], bk[kMaxLin];
    size_t bld[kMaxLin];
    int8_t* bq[kMaxLin];
    float* bs[kMaxLin];
    const float* bam[kMaxLin];
    bool batch_ok = true;
    int rot = 0;
    int mmax_b = 1;
    for (int l = 0; l < L; ++l) mmax_b = std::max(mmax_b, a[l].M);
    static const char* dynb_env = ODY_DIAG_ENV("ODY_PROGRAM_DYN");
    const bool dyn_chain = chain && dyn_chain_ok(a, deps, L) && !(dynb_env && dynb_env[0] == '0');
    const int b_rows = (chain && !dyn_chain) ? kBN : dyn_bn(mmax_b);
    for (int l = 0; l < L; ++l) {
        LinDesc& d = p.lin[l];
        d.x = a[l].x;
        d.ldx = a[l].ldx;
        d.x_bf16 = a[l].x_dtype == kDtypeBF16 ? 1 : 0;
        d.wp = a[l].wp;
        d.sw = a[l].sw;
        d.out = a[l].out;
        d.out_dtype = a[l].out_dtype;
        d.sa_out = a[l].sa_out;
        d.M = a[l].M;
        d.N = a[l].N;
        d.K = a[l].K;
        d.kblocks = static_cast<int>(pad_k(a[l].K) / kBlockK);
        d.n_tiles = static_cast<int>(pad_n(a[l].N) / kTileN);
        d.dep = deps ? deps[l] : -1;
        d.acc_out = a[l].acc_out;
        if (d.dep >= l) return cudaErrorInvalidValue;  // only earlier linears
        d.rot = chain ? 0 : rot % pl.C;
        rot += d.n_tiles;
        static const char* pq_env = ODY_DIAG_ENV("ODY_PROGRAM_PREQUANT");  // diagnostics: 0 = in-kernel K1
        const bool prequant = !(pq_env && pq_env[0] == '0');
        if (d.dep < 0 && prequant) {
            int8_t* q = reinterpret_cast<int8_t*>(cursor);
            cursor += round_up(a8_bytes(d.M, d.K), 256);
            float* sa = a[l].sa_out ? a[l].sa_out : reinterpret_cast<float*>(cursor);
            cursor += round_up(pad_m(d.M) * 4, 256);
            d.qa = q;
            d.sa = sa;
            d.Mp = b_rows;  // compact a8 layout: BN rows per k-block
            bx[nb] = a[l].x;
            bdt[nb] = a[l].x_dtype;
            bld[nb] = a[l].ldx;
            bm[nb] = d.M;
            bk[nb] = d.K;
            bq[nb] = q;
            bs[nb] = sa;
            bam[nb] = a[l].absmax_in;
            batch_ok &= d.K <= kRowThreads * kRowChunks * 16 && (a[l].x_dtype == kDtypeF16 || a[l].x_dtype == kDtypeBF16);
            ++nb;
        }
    }
    uint32_t* counters = static_cast<uint32_t*>(scratch);
    (void)counters;
    for (int l = 0; l < L; ++l)
        if (p.lin[l].dep >= 0) p.lin[p.lin[l].dep].signal = 1;
    bool prog_pdl = pdl;
    RowBatch rb_pending = {};
    int rb_rows = 0;
    bool has_rb = false;
    if (nb > 0) {
        cudaError_t ea = cudaSuccess;
        if (batch_ok) {
            RowBatch rb = {};
            int rows = 0;
            for (int i = 0; i < nb; ++i) {
                rb.x[i] = static_cast<const unsigned short*>(bx[i]);
                rb.ldx[i] = bld[i];
                rb.M[i] = bm[i];
                rb.K[i] = bk[i];
                rb.Mp[i] = b_rows;
                rb.bf16[i] = bdt[i] == kDtypeBF16 ? 1 : 0;
                rb.q[i] = bq[i];
                rb.s[i] = bs[i];
                rb.amax_in[i] = bam[i];
                rows += bm[i];
            }
            rb.n = nb;
            rb.pdl = pdl ? 1 : 0;
            rb.trace = a[0].trace ? a[0].trace + 148 * kTraceCta + 512 : nullptr;
            // launched right before the GEMM below (launch_dyn)
            rb_pending = rb;
            rb_rows = rows;
            has_rb = true;
        } else {
            for (int i = 0; i < nb && ea == cudaSuccess; ++i)
                ea = launch_act_quant(bx[i], bdt[i], bld[i], bm[i], bk[i], bq[i], bs[i], bam[i], nullptr,
                                      pdl || i > 0, st);
        }
        if (ea != cudaSuccess) return ea;
        prog_pdl = true;  // stream the weights while the act quant runs
    }
    p.ctr = counters;
    p.pdl = prog_pdl ? 1 : 0;
    p.next_wp = next_wp;
    p.next_bytes = next_wp ? (next_bytes & ~static_cast<size_t>(15)) : 0;
    p.trace = a[0].trace;
    static const char* pf_env = ODY_DIAG_ENV("ODY_DECODE_PF");
    p.pf_units = pf_env ? std::atoi(pf_env) : 0;
    static const char* dbg_env = ODY_DIAG_ENV("ODY_DBG_DECODE");
    p.dbg = dbg_env ? std::atoi(dbg_env) : 0;
    static const bool plan_log = ODY_DIAG_ENV("ODY_PLAN_LOG") != nullptr;
    if (plan_log) {
        std::fprintf(stderr, "[ody] decode program L=%d: S %d C %d grid %d%s:", L, pl.S, pl.C, pl.grid,
                     chain ? " (chain)" : "");
        for (int l = 0; l < L; ++l) std::fprintf(stderr, " %dx%dx%d", a[l].M, a[l].N, a[l].K);
        std::fprintf(stderr, "\n");
    }
    static const char* dyn_env = ODY_DIAG_ENV("ODY_PROGRAM_DYN");  // diagnostics: 0 = static schedule
    int n_ext = 0;
    for (int l = 0; l < L; ++l) n_ext += p.lin[l].dep < 0 ? 1 : 0;
    const bool dyn = nb == n_ext && (!chain || dyn_chain_ok(a, deps, L)) && !(dyn_env && dyn_env[0] == '0');
    const RowBatch* rbp = has_rb ? &rb_pending : nullptr;
    if (has_rb && !dyn) {  // the cluster kernel: the stand-alone act-quant kernel
        cudaLaunchConfig_t acfg = {};
        acfg.gridDim = dim3(rb_rows);
        acfg.blockDim = dim3(kRowThreads);
        acfg.stream = st;
        cudaLaunchAttribute aattr;
        aattr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
        aattr.val.programmaticStreamSerializationAllowed = 1;
        acfg.attrs = &aattr;
        acfg.numAttrs = rb_pending.pdl ? 1 : 0;
        const cudaError_t ea = cudaLaunchKernelEx(&acfg, act_quant_rows_kernel, rb_pending);
        if (ea != cudaSuccess) return ea;
    }
    if (dyn && chain) {
        // Dependency chain on the dynamic kernel: items in PROGRAM order (a producer's items
        // are all handed out before its dependent's), per-linear completion counters and
        // per-token row maxima in the zero region (re-armed by the launch's last CTA).
        uint32_t* done = counters + kChainDoneU32;
        uint32_t* qdone = done + kMaxLin;
        uint32_t* amax = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + kChainAmaxOffset);
        int mmax_c = 1;
        for (int l = 0; l < L; ++l) mmax_c = std::max(mmax_c, a[l].M);
        const int bn = dyn_bn(mmax_c);
        int ib = 0, tb = 0;
        for (int l = 0; l < L; ++l) {
            LinDesc& d = p.lin[l];
            split_alone(d, std::min(sms, device_sm_count()));
            d.off = ib;  // round-robin continues across linears (reduced mod C in the kernel)
            d.ibase = ib;
            d.tbase = tb;
            ib += d.items;
            tb += d.n_tiles;
        }
        for (int l = 0; l < L; ++l) {
            LinDesc& d = p.lin[l];
            if (d.dep < 0) continue;
            int c0 = 0;
            dyn_chain_slice(a, deps, L, l, &c0);
            LinDesc& y = p.lin[d.dep];
            y.done = done + d.dep;
            y.amax_dst = amax + d.dep * kChainMaxM * kAmaxStride;
            y.amax_c0 = c0;
            y.amax_c1 = c0 + d.K;
            y.amax_reset = y.amax_dst;
            d.dep_done = y.done;
            d.dep_target = static_cast<uint32_t>(y.items);
            d.amax_src = y.amax_dst;
            // the grid-wide quantized x (compact a8: BN rows per k-block), after the
            // external linears' buffers in the scratch
            d.qa = reinterpret_cast<const int8_t*>(cursor);
            cursor += round_up(static_cast<size_t>(bn) * pad_k(d.K), 256);
            d.Mp = bn;
            d.qdone = qdone + l;
        }
        p.n_items = ib;
        p.work = counters + kMaxLin + 1;
        p.pf_units = 0;
        p.S = 1;
        p.C = std::min(sms, ib);
        for (int l = 0; l < L; ++l)  // every CTA quantizes a share of each dependent x
            if (p.lin[l].qdone) p.lin[l].qtarget = static_cast<uint32_t>(p.C);
        static const char* st_env = ODY_DIAG_ENV("ODY_CHAIN_DYNAMIC");  // diagnostics: 1 = counter
        p.chain_static = (st_env && st_env[0] == '1') ? 0 : 1;
        p.reset_at_exit = 1;  // done / qdone / row maxima (and the counter when dynamic)
        for (int l = 0; l < L; ++l) p.lin[l].off %= p.C;
        if (plan_log) std::fprintf(stderr, "[ody] dynamic chain: %d items over %d CTAs\n", ib, p.C);
        switch (bn) {
            case 16: return launch_dyn<16, true, 2>(p, prog_pdl, st, rbp, rb_rows);
            case 32: return launch_dyn<32, true, 2>(p, prog_pdl, st, rbp, rb_rows);
            default: return launch_dyn<64, true, 2>(p, prog_pdl, st, rbp, rb_rows);
        }
    }
    if (dyn) {
        // Independent linears: hand the items out largest first (LPT), and end with the
        // linear of fewest bytes cut into ~12-block items, so the last items -- whose
        // duration is the tail -- are small.
        int order[kMaxLin];
        for (int l = 0; l < L; ++l) order[l] = l;
        auto bytes_of = [&](int l) { return static_cast<long long>(p.lin[l].n_tiles) * p.lin[l].kblocks; };
        std::sort(order, order + L, [&](int x, int y) { return bytes_of(x) > bytes_of(y); });
        static const char* tail_env = ODY_DIAG_ENV("ODY_DYN_TAIL_KB");  // diagnostics: 0 = off
        const int tail_kb = tail_env ? std::atoi(tail_env) : 0;  // measured: finer tails cost more (L2 partials)
        LinDesc sorted[kMaxLin];
        for (int l = 0; l < L; ++l) sorted[l] = p.lin[order[l]];
        int ib = 0, tb = 0;
        for (int l = 0; l < L; ++l) {
            LinDesc& d = sorted[l];
            // a lone linear is split like a chain link (all SMs, short last wave); in a
            // program the other linears' items fill the machine
            if (L == 1) {
                split_alone(d, std::min(sms, device_sm_count()));
            } else {
                int s = dyn_split(d.kblocks);
                if (l == L - 1 && tail_kb > 0) s = std::max(s, (d.kblocks + tail_kb - 1) / tail_kb);
                split_uniform(d, s);
            }
            d.ibase = ib;
            d.tbase = tb;
            ib += d.items;
            tb += d.n_tiles;
        }
        for (int l = 0; l < L; ++l) p.lin[l] = sorted[l];
        p.n_items = ib;
        p.work = counters + kMaxLin + 1;
        // a lone linear: static deal (items <= ~2 per CTA, balanced), nothing to re-arm
        p.chain_static = L == 1 ? 1 : 0;
        p.reset_at_exit = L == 1 ? 0 : 1;
        static const char* pfi_env = ODY_DIAG_ENV("ODY_DYN_PF_ITEMS");  // second-round items to L2
        p.pf_units = pfi_env ? std::atoi(pfi_env) : 0;  // measured: guessing next items costs more
        static const char* rpf_env = ODY_DIAG_ENV("ODY_REST_PF");  // diagnostics: 1 = on
        p.rest_pf = (rpf_env && rpf_env[0] == '1') ? 1 : 0;
        p.S = 1;
        p.C = std::min(sms, ib);
        if (plan_log) std::fprintf(stderr, "[ody] dynamic schedule: %d items over %d CTAs\n", ib, p.C);
        int mmax = 1;
        for (int l = 0; l < L; ++l) mmax = std::max(mmax, a[l].M);
        switch (dyn_bn(mmax)) {
            case 16: return (L == 1 ? launch_dyn<16, false, 4>(p, prog_pdl, st, rbp, rb_rows)
                                    : launch_dyn<16, false, 2>(p, prog_pdl, st, rbp, rb_rows));
            case 32: return (L == 1 ? launch_dyn<32, false, 4>(p, prog_pdl, st, rbp, rb_rows)
                                    : launch_dyn<32, false, 2>(p, prog_pdl, st, rbp, rb_rows));
            default: return (L == 1 ? launch_dyn<64, false, 4>(p, prog_pdl, st, rbp, rb_rows)
                                    : launch_dyn<64, false, 2>(p, prog_pdl, st, rbp, rb_rows));
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = pl.S;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (prog_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, w4a8_decode_kernel, p);
}

// A dependency chain as ONE LAUNCH PER LINEAR ("chain links"): each linear is a lone
// linear on the dynamic kernel (its own balanced split, static deal), and the kernel
// boundary replaces the chain program's grid-wide `done` counter.  A producer's epilogues
// accumulate its consumer's per-token row maxima (as in the chain program); the consumer
// launch, once griddepcontrol.wait returned (the producer grid completed, its maxima
// final), quantizes its x grid-wide in-kernel (B-quantizer warps, `qdone`) while its
// weights already stream -- no act-quant kernel and no second kernel boundary between
// two linears.  The consumer's last CTA re-zeroes its qdone and the row maxima it read.
// External linears keep the act-quant kernel.  Same scratch as launch_w4a8_program.
bool chain_links_eligible(const LinearArgs* a, const int* deps, int L) {
    if (!deps || L < 1 || L > kMaxLin || !dyn_chain_ok(a, deps, L)) return false;
    for (int l = 0; l < L; ++l) {
        if (!lin_ok(a[l], deps[l] < 0) || a[l].M > kChainMaxM) return false;
        if (pad_n(a[l].N) / kTileN > kProgramMaxTiles) return false;
    }
    return true;
}

cudaError_t launch_w4a8_chain_links(const LinearArgs* a, const int* deps, int L, void* scratch,
                                    size_t scratch_bytes, bool pdl, cudaStream_t st) {
    if (!chain_links_eligible(a, deps, L)) return cudaErrorInvalidValue;
    if (!scratch || scratch_bytes < program_scratch_bytes(a, deps, L)) return cudaErrorInvalidValue;
    const int sms = std::min(a[0].max_ctas > 0 ? a[0].max_ctas : device_sm_count(), device_sm_count());
    int mmax = 1;
    for (int l = 0; l < L; ++l) mmax = std::max(mmax, a[l].M);
    const int bn = dyn_bn(mmax);
    uint32_t* counters = static_cast<uint32_t*>(scratch);
    uint32_t* amax = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + kChainAmaxOffset);
    uint8_t* cursor = static_cast<uint8_t*>(scratch) + kZeroRegion + dyn_items(a, L) * bn * kTileN * 4;
    int consumer[kMaxLin];
    for (int l = 0; l < L; ++l) consumer[l] = -1;
    for (int l = 0; l < L; ++l)
        if (deps[l] >= 0) consumer[deps[l]] = l;
    for (int l = 0; l < L; ++l) {
        PParams p = {};
        p.L = 1;
        LinDesc& d = p.lin[0];
        d.x = a[l].x;
        d.ldx = a[l].ldx;
        d.x_bf16 = a[l].x_dtype == kDtypeBF16 ? 1 : 0;
        d.wp = a[l].wp;
        d.sw = a[l].sw;
        d.out = a[l].out;
        d.out_dtype = a[l].out_dtype;
        d.sa_out = a[l].sa_out;
        d.M = a[l].M;
        d.N = a[l].N;
        d.K = a[l].K;
        d.kblocks = static_cast<int>(pad_k(a[l].K) / kBlockK);
        d.n_tiles = static_cast<int>(pad_n(a[l].N) / kTileN);
        d.dep = -1;  // the producer is an earlier LAUNCH, not a linear of this one
        d.acc_out = a[l].acc_out;
        const bool dep = deps[l] >= 0;
        RowBatch rb = {};
        if (!dep) {
            int8_t* q = reinterpret_cast<int8_t*>(cursor);
            cursor += round_up(a8_bytes(d.M, d.K), 256);
            float* sa = a[l].sa_out ? a[l].sa_out : reinterpret_cast<float*>(cursor);
            cursor += round_up(pad_m(d.M) * 4, 256);
            d.qa = q;
            d.sa = sa;
            d.Mp = bn;  // compact a8 layout: BN rows per k-block
            rb.x[0] = static_cast<const unsigned short*>(a[l].x);
            rb.ldx[0] = a[l].ldx;
            rb.M[0] = d.M;
            rb.K[0] = d.K;
            rb.Mp[0] = bn;
            rb.bf16[0] = d.x_bf16;
            rb.q[0] = q;
            rb.s[0] = sa;
            rb.amax_in[0] = a[l].absmax_in;
            rb.n = 1;
            rb.pdl = (pdl || l > 0) ? 1 : 0;
        } else {
            // the act quant reads the row maxima the producer launch's epilogues accumulated
            // (act_quant_premax_kernel: no row reduction, 4 CTAs per token row); this
            // launch's CTA 0 re-zeroes them after its griddepcontrol.wait
            int8_t* q = reinterpret_cast<int8_t*>(cursor);
            cursor += round_up(static_cast<size_t>(bn) * pad_k(d.K), 256);
            float* sa = a[l].sa_out ? a[l].sa_out : reinterpret_cast<float*>(cursor);
            cursor += round_up(pad_m(d.M) * 4, 256);
            d.qa = q;
            d.sa = sa;
            d.Mp = bn;
            uint32_t* src = amax + deps[l] * kChainMaxM * kAmaxStride;
            d.amax_zero = src;
            rb.x[0] = static_cast<const unsigned short*>(a[l].x);
            rb.ldx[0] = a[l].ldx;
            rb.M[0] = d.M;
            rb.K[0] = d.K;
            rb.Mp[0] = bn;
            rb.bf16[0] = d.x_bf16;
            rb.q[0] = q;
            rb.s[0] = sa;
            rb.amax_src[0] = src;
            rb.n = 1;
            rb.pdl = 1;
        }
        if (consumer[l] >= 0) {
            int c0 = 0;
            dyn_chain_slice(a, deps, L, consumer[l], &c0);
            d.amax_dst = amax + l * kChainMaxM * kAmaxStride;
            d.amax_c0 = c0;
            d.amax_c1 = c0 + a[consumer[l]].K;
        }
        p.n_items = split_alone(d, sms);
        p.ctr = counters;
        p.work = counters + kMaxLin + 1;
        p.tile_cnt = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + kProgramCounterRegion);
        p.acc = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(scratch) + kAccOffset);
        p.part = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(scratch) + kZeroRegion);
        p.S = 1;
        p.C = std::min(sms, p.n_items);
        p.chain_static = 1;
        p.reset_at_exit = 0;  // static deal, nothing to re-arm
        p.pdl = 1;            // every link overlaps its act quant
        // diagnostics: one trace block per link (the per-CTA slots + the last CTA's units)
        p.trace = a[l].trace ? a[l].trace + static_cast<size_t>(l) * (148 * kTraceCta + 1536) : nullptr;
        cudaError_t e = cudaSuccess;
        const RowBatch* rbp = dep ? nullptr : &rb;  // lin_ok: an external K fits the row kernel
        if (dep) {
            e = launch_premax(rb, d.M, st);
            if (e != cudaSuccess) return e;
        }
        switch (bn) {
            case 16: e = launch_dyn<16, false, 4>(p, true, st, rbp, rbp ? d.M : 0); break;
            case 32: e = launch_dyn<32, false, 4>(p, true, st, rbp, rbp ? d.M : 0); break;
            default: e = launch_dyn<64, false, 4>(p, true, st, rbp, rbp ? d.M : 0); break;
        }
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_w4a8_decode(const LinearArgs& a, cudaStream_t st) {
    return launch_w4a8_program(&a, nullptr, 1, a.workspace, a.workspace_bytes, a.pdl, a.next_wp, a.next_bytes,
                               st);
}


// ody_gemm's decode widths (M <= 64) on pre-quantized activations (an ody_qtensor: the
// 128-row padded a8 layout): the dynamic decode kernel as a program of ONE linear, its
// k-split chosen like a chain link's so every SM streams weights.
size_t gemm_prequant_scratch_bytes(int M, int N, int K, int max_ctas) {
    const int sms = std::min(max_ctas > 0 ? max_ctas : device_sm_count(), device_sm_count());
    LinDesc d = {};
    d.kblocks = static_cast<int>(pad_k(K) / kBlockK);
    d.n_tiles = static_cast<int>(pad_n(N) / kTileN);
    return kZeroRegion + static_cast<size_t>(split_alone(d, sms)) * dyn_bn(M) * kTileN * 4;
}

bool gemm_prequant_eligible(int M, int N, int K) {
    return M >= 1 && M <= 64 && N >= 1 && K >= 1 && pad_n(N) / kTileN <= kProgramMaxTiles;
}

cudaError_t launch_w4a8_gemm_prequant(const GemmArgs& g, void* scratch, size_t scratch_bytes, cudaStream_t st) {
    if (!gemm_prequant_eligible(g.M, g.N, g.K)) return cudaErrorInvalidValue;
    if (!scratch || scratch_bytes < gemm_prequant_scratch_bytes(g.M, g.N, g.K, g.max_ctas)) return cudaErrorInvalidValue;
    const int sms = std::min(g.max_ctas > 0 ? g.max_ctas : device_sm_count(), device_sm_count());
    PParams p = {};
    p.L = 1;
    LinDesc& d = p.lin[0];
    d.wp = g.wp;
    d.sw = g.sw;
    d.out = g.out;
    d.out_dtype = g.out_dtype;
    d.acc_out = g.acc_out;
    d.M = g.M;
    d.N = g.N;
    d.K = g.K;
    d.kblocks = static_cast<int>(pad_k(g.K) / kBlockK);
    d.n_tiles = static_cast<int>(pad_n(g.N) / kTileN);
    d.qa = g.qa;
    d.sa = g.sa;
    d.Mp = static_cast<int>(pad_m(g.M));
    d.dep = -1;
    p.n_items = split_alone(d, sms);
    uint32_t* counters = static_cast<uint32_t*>(scratch);
    p.ctr = counters;
    p.work = counters + kMaxLin + 1;
    p.tile_cnt = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + kProgramCounterRegion);
    p.acc = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(scratch) + kAccOffset);
    p.part = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(scratch) + kZeroRegion);
    p.S = 1;
    p.C = std::min(sms, p.n_items);
    p.chain_static = 1;  // static deal of the lone linear's items: no counter to re-arm
    p.reset_at_exit = 0;
    p.pdl = g.pdl ? 1 : 0;
    p.trace = g.trace;
    switch (dyn_bn(g.M)) {
        case 16: return launch_dyn<16, false, 4>(p, g.pdl, st);
        case 32: return launch_dyn<32, false, 4>(p, g.pdl, st);
        default: return launch_dyn<64, false, 4>(p, g.pdl, st);
    }
}

}  // namespace odyb200
