// gemm_kernel.cu -- K3+K4: the W4A8 FastGEMM core with its fused dequantizing epilogue.
//
// Reference semantics (ref gemm.cpp:251-279):
//     acc  = sum_k a[i][k] * (16 * w[j][k])        (int32, exact)
//     acc >>= 4                                     (exact: every addend is a multiple of 16)
//     out[i][j] = float(acc) * (sa[i] * sw[j])
//
// B200 mapping (swap-AB, weights are the MMA "A" operand, tokens the MMA "N"):
//   * producer warp: 1-D bulk copies (cp.async.bulk -> UBLKCP) of up to two 8 KiB
//     packed-INT4 weight blocks (128 rows x 128 k each, contiguous) and the matching
//     activation k-blocks (BN tokens x 128 B, pre-swizzled SWIZZLE_128B) into an S-stage
//     smem ring.  A "unit" is one or two k-blocks;
//   * converter warps (2 groups x 4 warps, one warp per TMEM sub-partition): read the
//     packed blocks from smem, widen SINT4 -> S8 with the paper's high-nibble trick
//     ((w<<4)&0xF0F0F0F0 and w&0xF0F0F0F0 -- lanes hold value*16, no per-group scale
//     multiply), and tcgen05.st the int8 lanes straight into TMEM as the A operand;
//   * MMA warp (one elected lane, warp-uniform control flow): tcgen05.mma.kind::i8 with
//     A from TMEM, B from smem, int32 accumulators in TMEM (double-buffered, split over
//     independent chains so back-to-back MMAs do not serialise on one accumulator);
//   * epilogue warps: tcgen05.ld D, sum chains, >>4, *(sa*sw) with IEEE RN multiplies,
//     store f32/f16/bf16 -- or, for stream-K partial tiles, red.add.s32 into an
//     L2-resident workspace; the CTA that completes a tile's K range finalises it
//     (integer addition is associative, so split-K is bit-exact) and re-zeroes it.
//   * scheduling: persistent grid of <= #SMs CTAs; full waves of (n_tile, m_tile)
//     tiles are data-parallel, the remainder (all tiles for decode shapes) is split
//     stream-K over 128-k blocks, so every SM streams the same number of weight bytes.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>

#include "kernels.h"
#include "layout.h"
#include "ptx.cuh"
#include "quant_common.cuh"

namespace odyb200 {

namespace {

constexpr int kNumThreads = 512;   // 16 warps
constexpr int kWarpProducer = 0;
constexpr int kWarpMma = 1;
constexpr int kWarpAlloc = 2;
constexpr int kWarpFixup = 3;      // gathers other CTAs' stream-K partials for owned tiles
constexpr int kWarpConv0 = 4;      // warps 4..11: two converter groups of 4
constexpr int kConvGroups = 2;
constexpr int kWarpEpi0 = 12;      // warps 12..15
constexpr int kUnitBlocks = 2;     // k-blocks per pipeline unit (256 k, 16 KiB of weights)
constexpr int kAStages = 4;        // TMEM A stages (64 columns each)
constexpr int kAStageCols = kUnitBlocks * kBlockK / 4;
constexpr int kTmemCols = 512;
constexpr int kAColBase = 256;     // A stages live at columns 256..511
constexpr int kSmemBudget = 200 * 1024;
// diagnostics layout of the trace buffer (ody_dev_set_trace)
constexpr int kTraceCta = 8;                         // [cta][8] globaltimer slots
constexpr int kTraceUnits = 148 * kTraceCta;         // CTA 0: per-unit converter clock64 x4
constexpr int kTraceEpi = kTraceUnits + 64 * 4;      // per CTA, per segment epilogue x4
constexpr int kTraceMma = kTraceEpi + 148 * 16;      // (epi: 3 segs x 4 + fixup slot 15)
                                                     // CTA 0: per-unit MMA clock64 x4
constexpr int kTraceDbg = kTraceMma + 64 * 4;        // per CTA: epilogue clock64 checkpoints
static_assert(kAColBase + kAStages * kAStageCols <= kTmemCols, "TMEM budget");

template <int BN, bool FUSE = false>
struct Cfg {
    static constexpr int kBBytes = BN * 128;                          // one activation k-block
    // FUSE: activations are quantized inside the kernel into a resident smem B (all of
    // this CTA's k-range), so pipeline stages carry weights only.
    static constexpr int kStageBytes = FUSE ? kUnitBlocks * kWBlockBytes
                                            : kUnitBlocks * (kBBytes + kWBlockBytes);
    static constexpr int kWOff = FUSE ? 0 : kUnitBlocks * kBBytes;   // weights after B tiles
    static constexpr int kResBBytes = FUSE ? 96 * 1024 : 0;
    static constexpr int kTokBytes = FUSE ? (2 + 8) * BN * 4 : 0;  // max, scale, peers' maxima
    // Owned stream-K tile: the fixup warp bulk-copies the other contributors' partial
    // sums (kSlotBytes each, kStageSlots at a time) into smem and adds them into
    // fix_buf.  For BN=128 (prefill remainder tiles) the owner reads them directly.
    static constexpr int kSlotBytes = BN * kTileN * 4;
    static constexpr bool kBulkFix = BN <= 64;
    static constexpr int kStageSlots = BN == 16 ? 4 : (BN == 32 ? 2 : 1);
    static constexpr int kFixBytes =
        FUSE ? kSlotBytes * 2 : (kBulkFix ? kSlotBytes * (1 + kStageSlots) : 0);
    // Epilogue scales of the first kSegPre segments, prefetched at kernel start: loads
    // issued during the weight stream queue behind it for microseconds.
    static constexpr int kSegPre = 4;
    static constexpr int kScaleBytes = kSegPre * (kTileN + BN) * 4;
    // Output tile staged in smem and written with bulk async stores (one per token row)
    // instead of 2-byte scattered stores.
    static constexpr int kOutBytes = BN <= 64 ? BN * kTileN * 4 : 0;
    static constexpr int kBudget = FUSE ? 220 * 1024 : kSmemBudget;
    static constexpr int kStages = std::min(
        12, (kBudget - kResBBytes - kFixBytes - kScaleBytes - kOutBytes - kTokBytes) / kStageBytes);
    // Accumulator chains (chunk c -> chain c % kChains, summed in the epilogue).  The
    // tensor pipe pipelines dependent kind::i8 accumulations (measured: 10 cycles per
    // 128x16x32 MMA with 1 or 4 chains, tools/mma_bench.cu), so one chain suffices.
    static constexpr int kChains = 1;
    static constexpr int kBarrierBytes = 1024;
    static constexpr int kSmemBytes = kStages * kStageBytes + kResBBytes + kFixBytes + kScaleBytes +
                                      kOutBytes + kTokBytes + kBarrierBytes + 1024;
    // kind::i8, D=s32, A=B=s8 signed, K-major both, N=BN, M=128
    static constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                       (static_cast<uint32_t>(BN >> 3) << 17) |
                                       (static_cast<uint32_t>(128 >> 4) << 24);
    static_assert(BN % 16 == 0 && BN >= 16 && BN <= 128, "BN");
    static_assert(kBBytes % 1024 == 0 && kStageBytes % 1024 == 0, "swizzle atom alignment");
    static_assert(!FUSE || BN == 16, "in-kernel activation quantization is a decode (M<=16) path");
};

struct Params {
    const int8_t* qa;
    const float* sa;
    const uint8_t* wp;
    const float* sw;
    void* out;
    int32_t* acc_out;
    int32_t* ws_slots;   // [sk tile][contributor slot][BN][128] int32 partial sums
    uint32_t* ws_cnt;    // [sk tile] k-blocks published by non-owners (owner resets to 0)
    int max_contrib;     // contributor slots per stream-K tile
    int out_dtype;
    int M, N, K, Mp;
    int kblocks, m_tiles, tiles, dp_tiles, sk_units;
    int bulk_out;        // outputs may be staged in smem and bulk-stored (16 B aligned rows)
    // FUSE: quantize x (M x K, dtype x_dtype, row stride ldx) in-kernel; sa_out optional
    const void* x;
    int x_dtype;
    size_t ldx;
    float* sa_out;
    int split;           // 0: stream-K; >= 1: DP waves + remainder tiles split over
                         // clusters of `split` CTAs, reduced through DSMEM
    int cluster;         // cluster size (>= split; FUSE: activation share groups)
    int pdl;
    int dbg;             // diagnostics (ODY_DBG_FUSE): 1 hold weights until B quantized, 2 skip quant math
    unsigned long long* trace;  // optional timeline, see ody_dev_set_trace
};

// Walks this CTA's segments: data-parallel tiles first, then its stream-K block range.
// The stream-K range is walked BACKWARDS, so a CTA's final segment is the one that
// holds the last k-block of its tile: that CTA is the tile's owner, and the other
// contributors covered the tile's first blocks as the FIRST work of their own ranges,
// i.e. long before the owner finishes.  The owner then only adds their (already
// published) partial sums to its own accumulators -- no fixup after the mainloop.
//
// "DP + cluster split" mode (p.split >= 1, decode widths): full waves of tiles are
// data-parallel; each remaining tile r goes to cluster r, whose S CTAs each take 1/S of
// its k-blocks and reduce through distributed shared memory -- no global fixup at all.
struct SegIter {
    int tile, kb0, kb1;
    int dp_next, u_lo, u;
    int split_left;  // DP+split mode: the remainder segment of this CTA not yet returned
    bool is_split;   // the current segment is a cluster-split remainder segment
    __device__ void init(const Params& p) {
        const int P = gridDim.x, b = blockIdx.x;
        dp_next = b;
        const long long su = p.sk_units;
        u_lo = static_cast<int>(su * b / P);
        u = static_cast<int>(su * (b + 1) / P);
        split_left = (p.split >= 1 && b / p.split < p.tiles - p.dp_tiles) ? 1 : 0;
        is_split = false;
    }
    __device__ bool next(const Params& p) {
        is_split = false;
        if (dp_next < p.dp_tiles) {
            tile = dp_next;
            kb0 = 0;
            kb1 = p.kblocks;
            dp_next += gridDim.x;
            return true;
        }
        if (p.split >= 1) {  // rank r of cluster c owns k-blocks [r*kb/S, (r+1)*kb/S) of tile c
            if (!split_left) return false;
            split_left = 0;
            const int r = blockIdx.x % p.split;
            tile = p.dp_tiles + blockIdx.x / p.split;
            kb0 = r * p.kblocks / p.split;
            kb1 = (r + 1) * p.kblocks / p.split;
            is_split = p.split > 1;
            return true;
        }
        if (dp_next < p.dp_tiles) {
            tile = dp_next;
            kb0 = 0;
            kb1 = p.kblocks;
            dp_next += gridDim.x;
            return true;
        }
        if (u <= u_lo) return false;
        const int t = (u - 1) / p.kblocks;
        const int base = t * p.kblocks;
        tile = p.dp_tiles + t;
        kb0 = max(u_lo, base) - base;
        kb1 = u - base;
        u = base + kb0;
        return true;
    }
};

// Stream-K partition: CTA b owns units [lo(b), lo(b+1)).
__device__ __forceinline__ int sk_lo(const Params& p, int b) {
    return static_cast<int>(static_cast<long long>(p.sk_units) * b / gridDim.x);
}
__device__ __forceinline__ int sk_cta_of_unit(const Params& p, int u) {
    int b = static_cast<int>(static_cast<long long>(u) * gridDim.x / p.sk_units);
    while (b + 1 < static_cast<int>(gridDim.x) && sk_lo(p, b + 1) <= u) ++b;
    while (b > 0 && sk_lo(p, b) > u) --b;
    return b;
}

__device__ __forceinline__ uint64_t b_desc(uint32_t smem_addr) {
    // K-major SWIZZLE_128B: start>>4, LBO unused, SBO = 1024 B (8 rows x 128 B),
    // version 1 (sm_100), layout type 2 = SWIZZLE_128B.
    return static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(64) << 32) |
           (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}

// sa_t / sw_n are loaded before the accumulators are ready (off the critical path).
__device__ __forceinline__ void store_out(const Params& p, int t, int n, int32_t acc, float sa_t,
                                          float sw_n) {
    const size_t idx = static_cast<size_t>(t) * p.N + n;
    if (p.acc_out) p.acc_out[idx] = acc;
    if (p.out) {
        const int32_t sh = acc >> 4;  // exact (ref gemm.cpp:269)
        const float v = __fmul_rn(__int2float_rn(sh), __fmul_rn(sa_t, sw_n));
        if (p.out_dtype == kDtypeF32)
            static_cast<float*>(p.out)[idx] = v;
        else if (p.out_dtype == kDtypeF16)
            static_cast<__half*>(p.out)[idx] = __float2half_rn(v);
        else
            static_cast<__nv_bfloat16*>(p.out)[idx] = __float2bfloat16_rn(v);
    }
}

// FUSE quantization geometry.  The CTAs of a cluster that consume the same activation
// k-range (a "share class": the whole cluster when every CTA owns a data-parallel
// tile, the CTAs with the same split rank when the tiles are cluster-split) quantize
// disjoint sub-slices of it and push their codes into each other's resident B, so each
// activation byte is loaded and quantized once per class rather than once per CTA.
struct FuseGeom {
    int klo, khi;  // class k-block range (this CTA's resident B)
    int slo, shi;  // this CTA's sub-slice, quantized here
    int crank;     // rank in the cluster
    int seff;      // class stride in cluster ranks (1, or the split S)
    int D, j;      // class size, this CTA's index in it
};
__device__ __forceinline__ FuseGeom fuse_geom(const Params& p) {
    FuseGeom g;
    const int G = p.cluster;
    g.crank = static_cast<int>(blockIdx.x) % G;
    g.seff = (p.dp_tiles == 0 && p.split > 1) ? p.split : 1;
    const int s = g.crank % g.seff;
    g.D = G / g.seff;
    g.j = g.crank / g.seff;
    g.klo = s * p.kblocks / g.seff;  // == SegIter's split slice of rank s
    g.khi = (s + 1) * p.kblocks / g.seff;
    const int nb = g.khi - g.klo;
    g.slo = g.klo + g.j * nb / g.D;
    g.shi = g.klo + (g.j + 1) * nb / g.D;
    return g;
}

// FUSE prologue, run by the 384 threads of warps 4..15 before their pipeline roles:
// the per-token max|x| over this CTA's k-range (combined across the cluster's ranks
// through DSMEM when the tile is split, so every rank sees the max over ALL of K --
// ref quantize.cpp:113-132), then the INT8 codes of that k-range straight into the
// resident smem B operand in the swizzled K-major layout.  tok[0..BN) = scales.
// 16-bit activations are held packed (16 values = 2 x uint4) in registers between the
// max pass and the quantize pass: every x load of the CTA is issued at once, so the
// prologue costs one memory round trip even while the weight stream is in flight.
constexpr int kFuseThreads = 448;  // warps 2..15
constexpr int kFuseChunks = 6;     // 16-element chunks per thread (M * sub-slice <= 43008)

template <typename T>
__device__ __forceinline__ void load_chunk_raw(const T* row, int k0, int K, uint4 (&r)[2]) {
    if (k0 + 16 <= K) {
        r[0] = __ldg(reinterpret_cast<const uint4*>(row + k0));
        r[1] = __ldg(reinterpret_cast<const uint4*>(row + k0 + 8));
    } else {
        unsigned short h[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
            h[i] = k0 + i < K ? reinterpret_cast<const unsigned short*>(row)[k0 + i] : 0;
        r[0] = make_uint4(h[0] | (h[1] << 16), h[2] | (h[3] << 16), h[4] | (h[5] << 16),
                          h[6] | (h[7] << 16));
        r[1] = make_uint4(h[8] | (h[9] << 16), h[10] | (h[11] << 16), h[12] | (h[13] << 16),
                          h[14] | (h[15] << 16));
    }
}

__device__ __forceinline__ float unpack16(uint32_t w, int hi, bool bf16) {
    const unsigned short h = hi ? static_cast<unsigned short>(w >> 16) : static_cast<unsigned short>(w);
    return bf16 ? __uint_as_float(static_cast<uint32_t>(h) << 16) : __half2float(__ushort_as_half(h));
}

// 16 packed 16-bit values -> 16 INT8 codes through the IEEE-division path (the rare
// chunks holding a near-half-integer quotient, or a non-finite reciprocal).
__device__ __noinline__ uint4 quant16_exact(uint4 r0, uint4 r1, float scale, float rcp, bool bf16) {
    const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    uint32_t out[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const int32_t code = quant_code_i8(unpack16(w[e >> 1], e & 1, bf16), scale, rcp, true);
        out[e >> 2] |= (static_cast<uint32_t>(code) & 0xFFu) << (8 * (e & 3));
    }
    return make_uint4(out[0], out[1], out[2], out[3]);
}

// Fast path (quant_byte_fast): ~7 instructions per element, no branches.
__device__ __forceinline__ uint4 quant16_packed(uint4 r0, uint4 r1, float scale, float rcp, bool exact,
                                                bool bf16) {
    const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    uint32_t t[16];
    bool redo = exact;
#pragma unroll
    for (int e = 0; e < 16; ++e) t[e] = quant_byte_fast(unpack16(w[e >> 1], e & 1, bf16), rcp, redo);
    if (redo) return quant16_exact(r0, r1, scale, rcp, bf16);
    return make_uint4(pack4_low_bytes(t[0], t[1], t[2], t[3]), pack4_low_bytes(t[4], t[5], t[6], t[7]),
                      pack4_low_bytes(t[8], t[9], t[10], t[11]),
                      pack4_low_bytes(t[12], t[13], t[14], t[15]));
}

__device__ __forceinline__ float absmax16_packed(uint4 r0, uint4 r1, bool bf16) {
    const uint32_t w[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    float m = 0.0f;
#pragma unroll
    for (int e = 0; e < 16; ++e) m = fmaxf(m, fabsf(unpack16(w[e >> 1], e & 1, bf16)));
    return m;
}

// FUSE prologue, run by the 448 threads of warps 2..15 before their pipeline roles:
// per-token max|x| over this CTA's sub-slice, combined over the whole cluster through
// DSMEM (the cluster's sub-slices tile all of K, so every CTA sees the max over ALL of
// K -- ref quantize.cpp:113-132), then the INT8 codes of the sub-slice into the resident
// smem B (swizzled K-major), pushed to the share class with DSMEM bulk copies that
// complete on the peers' b_ready.  The 16-bit activations stay packed in registers
// between the max pass and the quantize pass: every load is issued at once.
template <int BN>
__device__ __forceinline__ void fused_act_quant(const Params& p, const FuseGeom& g, uint32_t resb,
                                                float* tok, uint64_t* max_ready, uint64_t* b_ready,
                                                int qt, bool kBf16) {
    constexpr int kQ = kFuseThreads;
    constexpr uint32_t kBlk = BN * 128;  // one resident B k-block
    const __half* x = static_cast<const __half*>(p.x);  // raw 16-bit payload (f16 or bf16)
    const int nch = (g.shi - g.slo) * (kBlockK / 16);  // 16-element chunks per token row
    const int total = p.M * nch;
    const int G = p.cluster;
    uint32_t* tmax = reinterpret_cast<uint32_t*>(tok + BN);  // [BN] as float bits (>= 0)
    float* peer = tok + 2 * BN;                               // [8][BN] cluster ranks' maxima
    if (qt < BN) tmax[qt] = 0u;
    uint4 raw[kFuseChunks][2];
#pragma unroll
    for (int i = 0; i < kFuseChunks; ++i) {  // all loads in flight together
        const int c = qt + i * kQ;
        if (c < total) {
            const int t = c / nch, kc = c - t * nch;
            load_chunk_raw(x + static_cast<size_t>(t) * p.ldx, g.slo * kBlockK + kc * 16, p.K, raw[i]);
        }
    }
    named_bar_sync(2, kQ);  // tmax zeroed
    unsigned long long* dbg = p.trace ? p.trace + kTraceDbg + blockIdx.x * 8 : nullptr;
    if (dbg && qt == 0) dbg[0] = globaltimer();
#pragma unroll
    for (int i = 0; i < kFuseChunks; ++i) {
        const int c = qt + i * kQ;
        if (c < total) {
            const float m = absmax16_packed(raw[i][0], raw[i][1], kBf16);
            atom_max_shared_u32(smem_u32(tmax + c / nch), __float_as_uint(m));  // floats >= 0
        }
    }
    named_bar_sync(2, kQ);
    if (dbg && qt == 0) dbg[1] = globaltimer();
    if (G > 1) {  // all-to-all of the partial maxima over the cluster (DSMEM)
        // Thread (d, token) stores one token's maximum into rank d and arrives there with
        // release semantics (orders its own store; no fence), all pairs in parallel.
        if (qt < G * BN) {
            const int d = qt / BN, tk = qt % BN;
            if (d != g.crank) {
                st_dsmem_u32(mapa_shared(smem_u32(peer + g.crank * BN + tk), d), tmax[tk]);
                mbar_arrive_remote(mapa_shared(smem_u32(max_ready), d));
            }
        }
        if (dbg && qt == 0) dbg[4] = globaltimer();
        mbar_wait_cluster(max_ready, 0);
        if (dbg && qt == 0) dbg[5] = globaltimer();
        if (qt < BN) {
            uint32_t m = tmax[qt];
            for (int d = 0; d < G; ++d)
                if (d != g.crank) m = max(m, __float_as_uint(peer[d * BN + qt]));
            tmax[qt] = m;
        }
        named_bar_sync(2, kQ);
    }
    float* trcp = peer;  // reuse: per-token reciprocal (thread qt only overwrites column qt)
    if (qt < BN) {
        float sc = __uint_as_float(tmax[qt]) / 127.0f;  // ref quantize.cpp:22-35
        if (!(sc > 0.0f)) sc = kMinScale;
        tok[qt] = sc;
        trcp[qt] = 1.0f / sc;
        if (p.sa_out && blockIdx.x == 0 && qt < p.M) p.sa_out[qt] = sc;
    }
    named_bar_sync(2, kQ);
    if (dbg && qt == 0) dbg[2] = globaltimer();
    const uint32_t mine = resb + (g.slo - g.klo) * kBlk;
#pragma unroll
    for (int i = 0; i < kFuseChunks; ++i) {
        const int c = qt + i * kQ;
        if (c < total) {
            const int t = c / nch, kc = c - t * nch;
            const float scale = __uint_as_float(lds32(smem_u32(tok + t)));
            const float rcp = __uint_as_float(lds32(smem_u32(trcp + t)));
            const bool exact = !(rcp < INFINITY);
            const uint4 q = p.dbg == 2 ? raw[i][0] : quant16_packed(raw[i][0], raw[i][1], scale, rcp, exact, kBf16);
            const int kb = kc / 8, chunk = kc % 8;  // block (relative to slo), 16-byte chunk
            sts128(mine + kb * kBlk + t * 128 + (((chunk ^ (t & 7)) & 7) * 16), q);
        }
    }
    for (int c = total + qt; c < BN * nch; c += kQ) {  // padding tokens M..BN-1: zero codes
        const int t = c / nch, kc = c - t * nch;
        const int kb = kc / 8, chunk = kc % 8;
        sts128(mine + kb * kBlk + t * 128 + (((chunk ^ (t & 7)) & 7) * 16), make_uint4(0, 0, 0, 0));
    }
    if (dbg && qt == 0) dbg[6] = globaltimer();
    fence_proxy_async_shared();  // generic smem writes -> async proxy (tcgen05, bulk copies)
    named_bar_sync(2, kQ);
    if (qt == 0) {
        const uint32_t bytes = (g.shi - g.slo) * kBlk;
        if (bytes > 0)
            for (int jj = 0; jj < g.D; ++jj) {
                if (jj == g.j) continue;
                const uint32_t rk = g.crank % g.seff + jj * g.seff;
                bulk_s2peer(mapa_shared(mine, rk), mine, bytes, mapa_shared(smem_u32(b_ready), rk));
            }
        // own arrival + the bytes the class peers push into this CTA
        mbar_expect_tx(b_ready, (g.khi - g.klo - (g.shi - g.slo)) * kBlk);
    }
    if (dbg && qt == 0) dbg[3] = globaltimer();
}

template <int BN, bool FUSE>
__global__ void __launch_bounds__(kNumThreads, 1) w4a8_gemm_kernel(const Params p) {
    using C = Cfg<BN, FUSE>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* stages = smem;
    uint8_t* resb_ptr = smem + C::kStages * C::kStageBytes;  // FUSE: resident B (1 KiB aligned)
    uint8_t* after_b = resb_ptr + C::kResBBytes;
    int32_t* fix_buf = reinterpret_cast<int32_t*>(after_b);
    float* scl = reinterpret_cast<float*>(after_b + C::kFixBytes);
    uint8_t* out_stage = after_b + C::kFixBytes + C::kScaleBytes;
    float* tok = reinterpret_cast<float*>(out_stage + C::kOutBytes);  // FUSE: token scales
    uint64_t* bars = reinterpret_cast<uint64_t*>(out_stage + C::kOutBytes + C::kTokBytes);
    uint64_t* w_full = bars;
    uint64_t* w_empty = w_full + C::kStages;
    uint64_t* a_full = w_empty + C::kStages;
    uint64_t* a_empty = a_full + kAStages;
    uint64_t* d_full = a_empty + kAStages;
    uint64_t* d_empty = d_full + 2;
    uint64_t* fix_full = d_empty + 2;
    uint64_t* fix_tx = fix_full + 1;
    uint64_t* recv_full = fix_tx + 1;  // cluster split-K: partials of ranks 1..S-1 landed
    uint64_t* b_ready = recv_full + 1;  // FUSE: resident B quantized
    uint64_t* max_ready = b_ready + 1;  // FUSE + cluster: the other ranks' token maxima landed
    uint64_t* push_done = max_ready + 1;  // FUSE: class peers received this CTA's codes
    uint64_t* b_full = push_done + 1;  // !FUSE: [kStages] activation tile of the stage landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_full + C::kStages);
    const uint32_t stage_base = smem_u32(stages);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    unsigned long long* trc = p.trace;
    if (trc && threadIdx.x == 0) trc[blockIdx.x * kTraceCta + 0] = globaltimer();
    // PDL: let the next kernel in the stream get scheduled immediately; it only
    // prefetches independent data before its own griddepcontrol.wait, which waits
    // for this grid's completion (and memory flush), so this is always safe.
    if (p.pdl) pdl_launch_dependents();

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::kStages; ++i) {
            mbar_init(&w_full[i], 1);
            mbar_init(&b_full[i], 1);
            mbar_init(&w_empty[i], 1);  // MMA commit (converters finished reading before MMA)
        }
        for (int i = 0; i < kAStages; ++i) {
            mbar_init(&a_full[i], 4);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&d_full[i], 1);
            mbar_init(&d_empty[i], 4);
        }
        mbar_init(fix_full, 1);
        mbar_init(fix_tx, 1);
        mbar_init(recv_full, p.split > 1 ? 4 * (p.split - 1) : 1);
        mbar_init(b_ready, 1);
        mbar_init(max_ready, p.cluster > 1 ? (p.cluster - 1) * BN : 1);
        mbar_init(push_done, p.cluster > 1 ? p.cluster - 1 : 1);
        fence_mbar_init();
    }
    if (warp == kWarpAlloc) {
        tmem_alloc(tmem_slot, kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    if (p.cluster > 1) cluster_sync();  // peers' barriers are initialised before any DSMEM traffic
    tc_fence_after();
    const uint32_t tmem = lds32(smem_u32(tmem_slot));
    if (trc && threadIdx.x == 0) trc[blockIdx.x * kTraceCta + 1] = globaltimer();

    SegIter it;
    it.init(p);

    if (FUSE && warp >= kWarpAlloc) {
        if (p.pdl) pdl_wait();  // x is produced by the previous kernel
        const int qt = threadIdx.x - kWarpAlloc * 32;
        fused_act_quant<BN>(p, fuse_geom(p), smem_u32(resb_ptr), tok, max_ready, b_ready, qt,
                            p.x_dtype == kDtypeBF16);
    }

    if (warp == kWarpProducer) {
        if (lane == 0) {
            const uint64_t pol_w = l2_policy_evict_first();
            const uint64_t pol_a = l2_policy_evict_last();
            // Weights do not depend on the previous kernel: with PDL, stream the first
            // ring's worth of weight blocks while the producer of the activations is
            // still finishing, then wait for it and fetch the activation tiles.
            int pre = 0;
            if (FUSE && p.dbg == 1) mbar_wait(b_ready, 0);
            if (p.pdl) {
                SegIter ip = it;
                bool more = true;
                while (more && pre < C::kStages && ip.next(p)) {
                    const int nt = ip.tile / p.m_tiles;
                    for (int kb = ip.kb0; kb < ip.kb1; kb += kUnitBlocks) {
                        if (pre >= C::kStages) {
                            more = false;
                            break;
                        }
                        const int nb = min(kUnitBlocks, ip.kb1 - kb);
                        mbar_expect_tx(&w_full[pre], nb * kWBlockBytes);
                        bulk_g2s(stages + pre * C::kStageBytes + C::kWOff,
                                 p.wp + (static_cast<size_t>(nt) * p.kblocks + kb) * kWBlockBytes,
                                 nb * kWBlockBytes, &w_full[pre], pol_w);
                        ++pre;
                    }
                }
                if (!FUSE) pdl_wait();
            }
            int u = 0;
            while (it.next(p)) {
                const int nt = it.tile / p.m_tiles, mt = it.tile % p.m_tiles;
                const uint8_t* wsrc = p.wp + (static_cast<size_t>(nt) * p.kblocks) * kWBlockBytes;
                const int8_t* asrc = p.qa + static_cast<size_t>(mt) * BN * 128;
                for (int kb = it.kb0; kb < it.kb1; kb += kUnitBlocks, ++u) {
                    const int nb = min(kUnitBlocks, it.kb1 - kb);
                    const int s = u % C::kStages;
                    uint8_t* st = stages + s * C::kStageBytes;
                    if (u >= pre) {
                        mbar_wait(&w_empty[s], ((u / C::kStages) & 1) ^ 1);
                        mbar_expect_tx(&w_full[s], nb * kWBlockBytes);
                        bulk_g2s(st + C::kWOff, wsrc + static_cast<size_t>(kb) * kWBlockBytes,
                                 nb * kWBlockBytes, &w_full[s], pol_w);
                    }
                    if (!FUSE) {  // own barrier: converters widen weights before B lands
                        mbar_expect_tx(&b_full[s], nb * C::kBBytes);
                        for (int b = 0; b < nb; ++b)
                            bulk_g2s(st + b * C::kBBytes,
                                     asrc + static_cast<size_t>(kb + b) * p.Mp * 128, C::kBBytes,
                                     &b_full[s], pol_a);
                    }
                }
            }
            if (trc) trc[blockIdx.x * kTraceCta + 6] = globaltimer();
        }
    } else if (warp == kWarpMma) {
        // Whole warp runs the (warp-uniform) loop; one elected lane issues tcgen05.
        int u = 0, j = 0;
        int klo = 0, khi = 0;
        if (FUSE) {
            const FuseGeom g = fuse_geom(p);
            klo = g.klo;
            khi = g.khi;
            mbar_wait(b_ready, 0);
            tc_fence_after();
            if (trc && lane == 0) trc[kTraceDbg + blockIdx.x * 8 + 7] = globaltimer();
            // every class peer's codes have landed here: tell them their pushes are done
            if (p.cluster > 1 && elect_one()) {
                for (int d = 0; d < p.cluster; ++d)
                    if (d != g.crank) mbar_arrive_remote(mapa_shared(smem_u32(push_done), d));
            }
            __syncwarp();
        }
        const uint32_t resb = smem_u32(resb_ptr);
        while (it.next(p)) {
            const int db = j & 1;
            mbar_wait(&d_empty[db], ((j >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem + db * C::kChains * BN;
            for (int kb = it.kb0; kb < it.kb1; kb += kUnitBlocks, ++u) {
                const int nb = min(kUnitBlocks, it.kb1 - kb);
                const int s = u % C::kStages;
                const int as = u % kAStages;
                const bool mtr = trc && blockIdx.x == 0 && u < 64 && lane == 0;
                if (mtr) trc[kTraceMma + u * 4 + 0] = clock64();
                // a_full(u): the converters observed w_full(u) and widened it into TMEM;
                // the stage's activation tile has its own barrier.
                mbar_wait(&a_full[as], (u / kAStages) & 1);
                if (!FUSE) mbar_wait(&b_full[s], (u / C::kStages) & 1);
                if (mtr) trc[kTraceMma + u * 4 + 1] = clock64();
                if (u == 0 && trc && lane == 0) trc[blockIdx.x * kTraceCta + 2] = globaltimer();
                if (mtr) trc[kTraceUnits + u * 4 + 3] = clock64();
                tc_fence_after();
                const uint32_t b_addr =
                    FUSE ? resb + (kb - klo) * C::kBBytes : stage_base + s * C::kStageBytes;
                const uint32_t a_tmem = tmem + kAColBase + as * kAStageCols;
                if (elect_one()) {
#pragma unroll
                    for (int c = 0; c < 4 * kUnitBlocks; ++c) {
                        if (c < 4 * nb)
                            mma_i8_ts(d_tmem + (c % C::kChains) * BN, a_tmem + 8 * c,
                                      b_desc(b_addr + (c / 4) * C::kBBytes + 32 * (c % 4)),
                                      C::kIdesc, (kb > it.kb0 || c >= C::kChains) ? 1u : 0u);
                    }
                    mma_commit(&a_empty[as]);
                    mma_commit(&w_empty[s]);
                }
                __syncwarp();
                if (mtr) trc[kTraceMma + u * 4 + 2] = clock64();
            }
            if (elect_one()) mma_commit(&d_full[db]);
            __syncwarp();
            ++j;
        }
        if (trc && lane == 0) {
            trc[blockIdx.x * kTraceCta + 3] = globaltimer();
            trc[blockIdx.x * kTraceCta + 7] =
                static_cast<unsigned long long>(u) | (static_cast<unsigned long long>(j) << 32);
        }
    } else if (warp >= kWarpConv0 && warp < kWarpConv0 + 4 * kConvGroups) {
        const int g = (warp - kWarpConv0) / 4;
        const int q = warp & 3;  // TMEM sub-partition: lanes 32q..32q+31
        const int r = 32 * q + lane;
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(32 * q) << 16);
        int u = 0;
        while (it.next(p)) {
            for (int kb = it.kb0; kb < it.kb1; kb += kUnitBlocks, ++u) {
                // a group owns the ring STAGES s with s % kConvGroups == g: alternating units
                // over an odd-length ring let a group wait on w_full one phase ahead (an
                // mbarrier parity wait then passes on the previous phase and widens stale
                // weights -- seen as whole wrong tiles at BN = 64, 3 stages)
                if (((u % C::kStages) % kConvGroups) != g) continue;
                const int nb = min(kUnitBlocks, it.kb1 - kb);
                const int s = u % C::kStages;
                const int as = u % kAStages;
                mbar_wait(&w_full[s], (u / C::kStages) & 1);
                const bool tr = trc && blockIdx.x == 0 && u < 64 && q == 0 && lane == 0;
                if (tr) trc[kTraceUnits + u * 4 + 0] = clock64();
                const uint32_t src = stage_base + s * C::kStageBytes + C::kWOff + r * 16;
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
                mbar_wait(&a_empty[as], ((u / kAStages) & 1) ^ 1);
                if (tr) trc[kTraceUnits + u * 4 + 1] = clock64();
                tc_fence_after();
                const uint32_t dst = t_lane + kAColBase + as * kAStageCols;
                tmem_st_32x32b_x32(dst, lanes8[0]);
                if (nb > 1) tmem_st_32x32b_x32(dst + 32, lanes8[1]);
                tmem_wait_st();
                if (tr) trc[kTraceUnits + u * 4 + 2] = clock64();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[as]);
            }
        }
    } else if (warp == kWarpFixup) {
        // Gather the partial sums other CTAs published for the tile this CTA owns (its
        // first stream-K segment in forward order, when that segment ends the tile and
        // does not start it).  Runs concurrently with the mainloop: bulk copies bring the
        // contributors' slots into smem and the warp adds them into fix_buf, so when the
        // owner's accumulators are ready only one smem add remains.
        const int b = blockIdx.x;
        if (C::kBulkFix && p.sk_units > 0) {
            const int lo = sk_lo(p, b), hi = sk_lo(p, b + 1);
            const int t = lo / p.kblocks;
            const int kb0 = lo - t * p.kblocks;
            if (hi > lo && kb0 > 0 && hi >= (t + 1) * p.kblocks) {
                const int bf = sk_cta_of_unit(p, t * p.kblocks);
                const int nslots = b - bf;
                if (p.pdl) pdl_wait();  // the previous launch has released the workspace
                if (lane == 0) {
                    while (ld_acquire_u32(p.ws_cnt + t) < static_cast<uint32_t>(kb0)) __nanosleep(64);
                    fence_proxy_async_global();  // generic-proxy writes -> async-proxy reads
                }
                __syncwarp();
                const uint8_t* src = reinterpret_cast<const uint8_t*>(
                    p.ws_slots + static_cast<size_t>(t) * p.max_contrib * BN * kTileN);
                uint8_t* stage_slots = reinterpret_cast<uint8_t*>(fix_buf) + C::kSlotBytes;
                const uint32_t fb = smem_u32(fix_buf), sb = smem_u32(stage_slots);
                constexpr int n4 = C::kSlotBytes / 16;
                uint32_t phase = 0;
                for (int c0 = 0; c0 < nslots; c0 += C::kStageSlots) {
                    const int nb = min(C::kStageSlots, nslots - c0);
                    if (lane == 0) {
                        mbar_expect_tx(fix_tx, nb * C::kSlotBytes);
                        for (int i = 0; i < nb; ++i)
                            bulk_g2s(stage_slots + i * C::kSlotBytes,
                                     src + static_cast<size_t>(c0 + i) * C::kSlotBytes, C::kSlotBytes,
                                     fix_tx, l2_policy_evict_first());
                    }
                    mbar_wait(fix_tx, phase);
                    phase ^= 1;
                    for (int i = lane; i < n4; i += 32) {
                        uint4 acc = c0 == 0 ? make_uint4(0, 0, 0, 0) : lds128(fb + i * 16);
                        for (int k = 0; k < nb; ++k) {
                            const uint4 v = lds128(sb + k * C::kSlotBytes + i * 16);
                            acc.x += v.x;
                            acc.y += v.y;
                            acc.z += v.z;
                            acc.w += v.w;
                        }
                        sts128(fb + i * 16, acc);
                    }
                    __syncwarp();
                }
                if (lane == 0) {
                    p.ws_cnt[t] = 0u;  // every contribution is consumed
                    mbar_arrive(fix_full);
                }
                if (trc && lane == 0) trc[kTraceEpi + blockIdx.x * 16 + 15] = globaltimer();
            }
        }
    } else if (warp >= kWarpEpi0) {
        // Epilogue.  Three segment kinds:
        //   full     -- all k-blocks of the tile are this CTA's: store directly;
        //   partial  -- publish the int32 partial sums into this CTA's slot of the tile
        //               (plain stores), then a release increment of the tile's counter;
        //   owner    -- holds the tile's last k-block (its final segment): add the other
        //               contributors' sum (gathered into smem by the fixup warp) to its
        //               own accumulators and store.
        const int q = warp & 3;
        const int r = 32 * q + lane;
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(32 * q) << 16);
        const uint32_t fix_base = smem_u32(fix_buf);
        if (p.pdl) pdl_wait();
        {  // prefetch the scales of the first kSegPre segments before the stream saturates
            SegIter ip = it;
            for (int jj = 0; jj < C::kSegPre && ip.next(p); ++jj) {
                const int nt = ip.tile / p.m_tiles, mt = ip.tile % p.m_tiles;
                const int n = nt * kTileN + r;
                float* sc = scl + jj * (kTileN + BN);
                sc[r] = n < p.N ? __ldg(p.sw + n) : 0.0f;
                if (r < BN)
                    sc[kTileN + r] = FUSE ? tok[r]
                                          : (mt * BN + r < p.M ? __ldg(p.sa + mt * BN + r) : 0.0f);
            }
            named_bar_sync(1, 128);
        }
        int j = 0;
        while (it.next(p)) {
            const int db = j & 1;
            const int nt = it.tile / p.m_tiles, mt = it.tile % p.m_tiles;
            const int n = nt * kTileN + r;
            const int t0 = mt * BN;
            const bool csplit = it.is_split;
            const int crank = csplit ? static_cast<int>(blockIdx.x % p.split) : 0;
            // cluster rank of this split group's rank 0 (clusters may hold several groups)
            const uint32_t sbase = csplit ? static_cast<uint32_t>(blockIdx.x % p.cluster - crank) : 0u;
            const bool full = csplit ? crank == 0 : (it.kb0 == 0 && it.kb1 == p.kblocks);
            const bool owner = !csplit && !full && it.kb1 == p.kblocks;
            const int skt = it.tile - p.dp_tiles;
            const bool etr = trc && warp == kWarpEpi0 && lane == 0 && j < 3;
            unsigned long long* et = trc + kTraceEpi + blockIdx.x * 16 + j * 4;
            // scales for this tile, fetched while the MMAs finish
            constexpr int kPre = BN < 32 ? BN : 32;
            const float* sc = scl + j * (kTileN + BN);
            const bool pref = j < C::kSegPre;
            const float sw_n = !(full || owner) ? 0.0f
                               : pref           ? sc[r]
                               : (n < p.N ? __ldg(p.sw + n) : 0.0f);
            float sa_pre[kPre];
#pragma unroll
            for (int i = 0; i < kPre; ++i)
                sa_pre[i] = !(full || owner) ? 0.0f
                            : pref           ? sc[kTileN + i]
                            : FUSE           ? tok[i]
                            : (t0 + i < p.M ? __ldg(p.sa + t0 + i) : 0.0f);
            const bool stage_out = C::kOutBytes > 0 && p.bulk_out && (full || owner) &&
                                   (nt + 1) * kTileN <= p.N;
            const uint32_t ostage = smem_u32(out_stage);
            int32_t* slot = nullptr;
            if (!full && !owner && !csplit) {
                const int c = blockIdx.x - sk_cta_of_unit(p, skt * p.kblocks);
                slot = p.ws_slots + (static_cast<size_t>(skt) * p.max_contrib + c) * BN * kTileN;
            }
            mbar_wait(&d_full[db], (j >> 1) & 1);
            if (etr) et[0] = globaltimer();
            if (owner && C::kBulkFix) {
                mbar_wait(fix_full, 0);
                if (etr) et[2] = globaltimer();
            }
            if (csplit && crank == 0) {
                mbar_wait_cluster(recv_full, 0);
                if (etr) et[2] = globaltimer();
            }
            int nslots_direct = 0;
            const int32_t* slots_direct = nullptr;
            if (owner && !C::kBulkFix) {  // BN=128: read the other contributors' slots here
                if (warp == kWarpEpi0 && lane == 0)
                    while (ld_acquire_u32(p.ws_cnt + skt) < static_cast<uint32_t>(it.kb0))
                        __nanosleep(64);
                named_bar_sync(1, 128);
                fence_acq_rel_gpu();
                nslots_direct = blockIdx.x - sk_cta_of_unit(p, skt * p.kblocks);
                slots_direct = p.ws_slots + static_cast<size_t>(skt) * p.max_contrib * BN * kTileN;
            }
            tc_fence_after();
#pragma unroll
            for (int tc = 0; tc < BN; tc += 16) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(t_lane + db * C::kChains * BN + tc, v);
#pragma unroll
                for (int ch = 1; ch < C::kChains; ++ch) {
                    uint32_t w[16];
                    tmem_ld_32x32b_x16(t_lane + (db * C::kChains + ch) * BN + tc, w);
                    tmem_wait_ld();
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] += w[i];  // exact int32 (mod 2^32)
                }
                tmem_wait_ld();
                if (full || owner) {
                    if (csplit) {
                        for (int c = 0; c < p.split - 1; ++c) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                v[i] += lds32(fix_base + ((c * BN + tc + i) * kTileN + r) * 4);
                        }
                    }
                    if (owner && C::kBulkFix) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            v[i] += lds32(fix_base + ((tc + i) * kTileN + r) * 4);
                    } else if (owner) {
                        for (int c = 0; c < nslots_direct; ++c) {
                            const int32_t* sl = slots_direct + static_cast<size_t>(c) * BN * kTileN;
                            int32_t w[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i) w[i] = __ldcg(sl + (tc + i) * kTileN + r);
#pragma unroll
                            for (int i = 0; i < 16; ++i) v[i] += static_cast<uint32_t>(w[i]);
                        }
                    }
                    if (stage_out) {
                        // value of (token tc+i, row r) into the smem tile [token][128 rows]
                        float val[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const float sa_t = tc + i < kPre ? sa_pre[tc + i < kPre ? tc + i : 0]
                                                             : __ldg(p.sa + min(t0 + tc + i, p.M - 1));
                            val[i] = __fmul_rn(__int2float_rn(static_cast<int32_t>(v[i]) >> 4),
                                               __fmul_rn(sa_t, sw_n));  // ref gemm.cpp:269-273
                        }
                        const uint32_t e0 = static_cast<uint32_t>(tc * kTileN + r);
                        if (p.out_dtype == kDtypeF32) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                sts32(ostage + (e0 + i * kTileN) * 4, __float_as_uint(val[i]));
                        } else if (p.out_dtype == kDtypeF16) {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                sts16(ostage + (e0 + i * kTileN) * 2, __half_as_ushort(__float2half_rn(val[i])));
                        } else {
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                sts16(ostage + (e0 + i * kTileN) * 2,
                                      __bfloat16_as_ushort(__float2bfloat16_rn(val[i])));
                        }
                    } else if (n < p.N) {
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            const int t = t0 + tc + i;
                            if (t < p.M) {
                                const float sa_t = tc + i < kPre ? sa_pre[tc + i < kPre ? tc + i : 0]
                                                                 : __ldg(p.sa + t);
                                store_out(p, t, n, static_cast<int32_t>(v[i]), sa_t, sw_n);
                            }
                        }
                    }
                } else if (csplit) {  // rank > 0: partials into rank 0's smem (DSMEM)
                    const uint32_t dst0 =
                        mapa_shared(fix_base + (((crank - 1) * BN + tc) * kTileN + r) * 4, sbase);
#pragma unroll
                    for (int i = 0; i < 16; ++i) st_dsmem_u32(dst0 + i * kTileN * 4, v[i]);
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        __stcg(slot + (tc + i) * kTileN + r, static_cast<int32_t>(v[i]));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&d_empty[db]);
            if (stage_out) {  // the staged tile leaves as coalesced 16-byte row pieces
                named_bar_sync(1, 128);
                const int esz = p.out_dtype == kDtypeF32 ? 4 : 2;
                const int per_row = kTileN * esz / 16;  // 16-byte pieces per token row
                const int rows = min(BN, p.M - t0);
                for (int c = r; c < rows * per_row; c += 128) {
                    const int t = c / per_row, piece = c % per_row;
                    const uint4 val = lds128(ostage + (t * kTileN * esz) + piece * 16);
                    *reinterpret_cast<uint4*>(static_cast<uint8_t*>(p.out) +
                                              (static_cast<size_t>(t0 + t) * p.N + nt * kTileN) * esz +
                                              piece * 16) = val;
                }
                named_bar_sync(1, 128);  // staging reusable by the next segment
            }
            if (etr) et[1] = globaltimer();
            if (csplit && crank > 0) {
                fence_acq_rel_cluster();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(mapa_shared(smem_u32(recv_full), sbase));
            } else if (!full && !owner) {
                __threadfence();  // this thread's partials are visible before the count
                named_bar_sync(1, 128);
                if (warp == kWarpEpi0 && lane == 0)
                    red_release_add_u32(p.ws_cnt + skt, static_cast<uint32_t>(it.kb1 - it.kb0));
            } else if (owner && !C::kBulkFix) {
                named_bar_sync(1, 128);  // all 128 threads read their slots
                if (warp == kWarpEpi0 && lane == 0) p.ws_cnt[skt] = 0u;
            }
            if (etr) et[3] = globaltimer() | (static_cast<unsigned long long>(owner) << 63);
            ++j;
        }
        if (trc && warp == kWarpEpi0 && lane == 0) trc[blockIdx.x * kTraceCta + 4] = globaltimer();
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kWarpAlloc) tmem_dealloc(tmem, kTmemCols);
    // FUSE: this CTA's smem is the source of DSMEM bulk pushes; stay resident until every
    // cluster peer has received them.
    if (FUSE && p.cluster > 1 && threadIdx.x == 0) mbar_wait_cluster(push_done, 0);
    if (trc && threadIdx.x == 0) trc[blockIdx.x * kTraceCta + 5] = globaltimer();
}

template <int BN, bool FUSE = false>
cudaError_t ensure_attr() {
    using C = Cfg<BN, FUSE>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(w4a8_gemm_kernel<BN, FUSE>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    });
    return attr_err;
}

template <int BN, bool FUSE = false>
cudaError_t launch_bn(const Params& p, int grid, bool pdl, cudaStream_t st) {
    using C = Cfg<BN, FUSE>;
    static_assert(C::kFixBytes == 0 || C::kFixBytes >= C::kSlotBytes, "fix region");
    const cudaError_t attr_err = ensure_attr<BN, FUSE>();
    if (attr_err != cudaSuccess) return attr_err;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kNumThreads);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (p.cluster > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = p.cluster;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, w4a8_gemm_kernel<BN, FUSE>, p);
}

int pick_bn(int M) {
    if (M <= 16) return 16;
    if (M <= 32) return 32;
    if (M <= 64) return 64;
    return 128;
}

}  // namespace

int device_sm_count() {
    static int sms = [] {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    }();
    return sms;
}

// Workspace = [fixed counter region | contributor slots].  The counter region never moves
// with the shape, so slot data of one launch can never land on another's counters.
constexpr size_t kCounterBytes = 4096;  // up to 1024 stream-K tiles (<= #CTAs)

// Stream-K geometry shared by the launcher and the workspace sizing.
struct SkPlan {
    int bn, kblocks, m_tiles, tiles, P, dp_tiles, sk_units, sk_tiles, max_contrib, split;
};

// Largest cluster split S with (S-1) partial tiles fitting the receive region.
static int max_split_for_bn(int bn, bool fused = false) {
    if (fused) return bn == 16 ? Cfg<16, true>::kFixBytes / Cfg<16, true>::kSlotBytes + 1 : 1;
    switch (bn) {
        case 16: return Cfg<16>::kFixBytes / Cfg<16>::kSlotBytes + 1;
        case 32: return Cfg<32>::kFixBytes / Cfg<32>::kSlotBytes + 1;
        case 64: return Cfg<64>::kFixBytes / Cfg<64>::kSlotBytes + 1;
        default: return 1;
    }
}

static SkPlan plan_for(int M, int N, int K, int sms, bool fused = false) {
    SkPlan s = {};
    s.bn = pick_bn(M);
    s.kblocks = static_cast<int>(pad_k(K) / kBlockK);
    const int n_tiles = static_cast<int>(pad_n(N) / kTileN);
    s.m_tiles = (M + s.bn - 1) / s.bn;
    s.tiles = n_tiles * s.m_tiles;
    const long long units = static_cast<long long>(s.tiles) * s.kblocks;
    s.split = 0;
    static const char* mode_env = ODY_DIAG_ENV("ODY_GEMM_SCHED");  // "sk" forces stream-K
    const bool force_sk = mode_env && std::string(mode_env) == "sk";
    const int max_split =
        std::min({max_split_for_bn(s.bn, fused), 8, std::max(1, s.kblocks / 2)});
    if (!force_sk && max_split >= 1 && s.bn <= 64) {
        // DP waves over P' = floor(P/S)*S CTAs, then the R remaining tiles each split over
        // a cluster of S = min(P'/R, max) CTAs.  Choose S to minimise the busiest CTA's
        // k-blocks (DP waves * kb + kb / S).
        int best_s = 1;
        double best_cost = 1e30;
        for (int S = 1; S <= max_split; ++S) {
            const int Pp = (sms / S) * S;
            if (Pp == 0) break;
            const int W = s.tiles / Pp;
            const int R = s.tiles - W * Pp;
            if (R * S > Pp) continue;
            const double cost = W * s.kblocks + (R > 0 ? static_cast<double>(s.kblocks) / S : 0.0);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best_s = S;
            }
        }
        const int Pp = (sms / best_s) * best_s;
        const int W = s.tiles / Pp;
        const int R = s.tiles - W * Pp;
        s.split = best_s;
        s.dp_tiles = W * Pp;
        s.P = W > 0 ? Pp : R * best_s;
        s.sk_units = 0;
        s.sk_tiles = 0;
        s.max_contrib = 1;
        return s;
    }
    s.P = static_cast<int>(std::min<long long>(sms, units));
    s.dp_tiles = (s.tiles / s.P) * s.P;
    s.sk_tiles = s.tiles - s.dp_tiles;
    s.sk_units = s.sk_tiles * s.kblocks;
    s.max_contrib = 1;
    if (s.sk_units > 0) {
        auto lo = [&](int b) { return static_cast<int>(static_cast<long long>(s.sk_units) * b / s.P); };
        auto cta_of = [&](int u) {
            int b = static_cast<int>(static_cast<long long>(u) * s.P / s.sk_units);
            while (b + 1 < s.P && lo(b + 1) <= u) ++b;
            while (b > 0 && lo(b) > u) --b;
            return b;
        };
        for (int t = 0; t < s.sk_tiles; ++t) {
            const int c = cta_of((t + 1) * s.kblocks - 1) - cta_of(t * s.kblocks);
            s.max_contrib = std::max(s.max_contrib, c);
        }
    }
    return s;
}

static size_t sk_workspace_bytes(int M, int N, int K, int sms) {
    const SkPlan s = plan_for(M, N, K, sms);
    return kCounterBytes + static_cast<size_t>(std::max(s.sk_tiles, 1)) * s.max_contrib * s.bn *
                               kTileN * sizeof(int32_t);
}

// num_sms > 0: the workspace of a launch on that many CTAs.  num_sms == 0 (the size
// queries of the C ABI): the maximum over every CTA budget 1..#SMs, so a buffer sized by
// the query is large enough whatever max_ctas the caller later passes (the stream-K
// remainder does not shrink monotonically with the budget).
size_t gemm_workspace_bytes(int M, int N, int K, int num_sms) {
    if (num_sms > 0) return sk_workspace_bytes(M, N, K, num_sms);
    static std::mutex mu;
    static std::map<std::tuple<int, int, int>, size_t> cache;  // the queries run per call
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(M, N, K);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    size_t b = 0;
    for (int P = 1; P <= device_sm_count(); ++P) b = std::max(b, sk_workspace_bytes(M, N, K, P));
    cache.emplace(key, b);
    return b;
}

cudaError_t launch_w4a8_gemm(const GemmArgs& a, cudaStream_t st) {
    if (a.M <= 0 || a.N <= 0 || a.K <= 0) return cudaErrorInvalidValue;
    if (prefill_eligible(a.M, a.N, a.K)) return launch_w4a8_prefill(a, st);  // prefill_kernel.cu
    const int sms = a.max_ctas > 0 ? a.max_ctas : device_sm_count();
    const SkPlan s = plan_for(a.M, a.N, a.K, sms);
    Params p = {};
    p.qa = a.qa;
    p.sa = a.sa;
    p.wp = a.wp;
    p.sw = a.sw;
    p.out = a.out;
    p.acc_out = a.acc_out;
    p.out_dtype = a.out_dtype;
    p.M = a.M;
    p.N = a.N;
    p.K = a.K;
    p.Mp = static_cast<int>(pad_m(a.M));
    p.kblocks = s.kblocks;
    p.m_tiles = s.m_tiles;
    p.tiles = s.tiles;
    p.dp_tiles = s.dp_tiles;
    p.sk_units = s.sk_units;
    p.max_contrib = s.max_contrib;
    p.split = s.split;
    p.cluster = s.split > 1 ? s.split : 1;
    {
        const size_t esz = a.out_dtype == kDtypeF32 ? 4 : 2;
        p.bulk_out = (a.out && !a.acc_out && (static_cast<size_t>(a.N) * esz) % 16 == 0 &&
                      (reinterpret_cast<uintptr_t>(a.out) & 15) == 0)
                         ? 1
                         : 0;
    }
    if (a.workspace_bytes < gemm_workspace_bytes(a.M, a.N, a.K, sms) || s.sk_tiles > 1024)
        return cudaErrorInvalidValue;
    p.ws_cnt = static_cast<uint32_t*>(a.workspace);
    p.ws_slots = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(a.workspace) + kCounterBytes);
    p.pdl = a.pdl ? 1 : 0;
    p.trace = a.trace;
    switch (s.bn) {
        case 16: return launch_bn<16>(p, s.P, a.pdl, st);
        case 32: return launch_bn<32>(p, s.P, a.pdl, st);
        case 64: return launch_bn<64>(p, s.P, a.pdl, st);
        default: return launch_bn<128>(p, s.P, a.pdl, st);
    }
}

// How many clusters of G fused-kernel CTAs (one per SM) can be resident at once.
static int max_active_clusters_fused(int G) {
    static int cache[9] = {-1, -1, -1, -1, -1, -1, -1, -1, -1};
    if (G < 1 || G > 8) return 0;
    if (cache[G] >= 0) return cache[G];
    int n = 0;
    if (ensure_attr<16, true>() == cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(G * 64);
        cfg.blockDim = dim3(kNumThreads);
        cfg.dynamicSmemBytes = Cfg<16, true>::kSmemBytes;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = G;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&n, w4a8_gemm_kernel<16, true>, &cfg) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
    }
    cache[G] = n;
    return n;
}

// Cluster size of the fused launch: the largest G <= 8 that is a multiple of the split S,
// divides the grid and keeps every cluster co-resident (one CTA per SM); the share
// classes then load and quantize 1/(G/S_eff) of the activations each.
static int fused_cluster(const SkPlan& s) {
    const int S = std::max(1, s.split);
    static const char* env = ODY_DIAG_ENV("ODY_FUSE_CLUSTER");  // diagnostics override
    const int forced = env ? std::atoi(env) : 0;
    for (int G = 8; G >= 2; --G) {
        if (forced > 0 && G != forced) continue;
        if (G % S != 0 || s.P % G != 0) continue;
        if (max_active_clusters_fused(G) < s.P / G) continue;
        return G;
    }
    return S;
}

// K1 fused into K3+K4 for decode widths (M <= 16): one kernel per linear.  Falls back to
// act_quant + GEMM (two kernels, codes in the caller's a8 scratch) when not eligible.
size_t linear_scratch_bytes(int M, int N, int K, int num_sms) {
    // One buffer serves both lowerings, with every zero-invariant region at a fixed,
    // shape-independent offset: [decode-program zero region, whose last 4 KiB are the
    // GEMM's stream-K counters][transient: GEMM slots / program partials + a8 ...]; the
    // two-kernel path's a8 codes + scales sit at the very end.
    static_assert(kLinearGemmCounters == kCounterBytes, "GEMM counter region");
    LinearArgs a = {};
    a.M = M;
    a.N = N;
    a.K = K;
    const size_t gemm_path = program_zero_bytes() - kCounterBytes + gemm_workspace_bytes(M, N, K, num_sms) +
                             round_up(a8_bytes(M, K), 256) + round_up(pad_m(M) * sizeof(float), 256);
    return std::max(gemm_path, program_scratch_bytes(&a, nullptr, 1));
}

static thread_local int g_linear_mode = 2;  // see kernels.h; per calling thread, like the CUDA current device
void set_linear_mode(int mode) { g_linear_mode = mode; }
int linear_mode() { return g_linear_mode; }

bool linear_is_fused(int M, int N, int K, int num_sms) {
    if (g_linear_mode == 2) return decode_eligible(M, N, K, kDtypeF16, num_sms);
    if (g_linear_mode != 1) return false;
    const int sms = num_sms > 0 ? num_sms : device_sm_count();
    const SkPlan s = plan_for(M, N, K, sms, true);
    if (s.bn != 16 || s.split < 1) return false;
    const int G = fused_cluster(s);
    const int seff = (s.dp_tiles == 0 && s.split > 1) ? s.split : 1;
    const int D = G / seff;
    const int span = (s.kblocks + seff - 1) / seff;  // class range (resident B)
    const int sub = (span + D - 1) / D;               // per-CTA quantized sub-slice
    return static_cast<long long>(span) * 16 * 128 <= Cfg<16, true>::kResBBytes &&
           static_cast<long long>(M) * sub * (kBlockK / 16) <= kFuseThreads * kFuseChunks;
}

cudaError_t launch_w4a8_linear(const LinearArgs& a, cudaStream_t st) {
    if (a.M <= 0 || a.N <= 0 || a.K <= 0) return cudaErrorInvalidValue;
    const int sms = a.max_ctas > 0 ? a.max_ctas : device_sm_count();
    if (a.workspace_bytes < linear_scratch_bytes(a.M, a.N, a.K, sms)) return cudaErrorInvalidValue;
    const size_t esz_x = a.x_dtype == kDtypeF32 ? 4 : 2;
    const bool aligned = (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && (a.ldx * esz_x) % 16 == 0;
    uint8_t* ws = static_cast<uint8_t*>(a.workspace);
    const size_t gws = gemm_workspace_bytes(a.M, a.N, a.K, sms);
    if (g_linear_mode == 2 && aligned && decode_eligible(a.M, a.N, a.K, a.x_dtype, sms))
        return launch_w4a8_decode(a, st);  // the whole buffer is its program scratch
    uint8_t* gemm_ws = ws + program_zero_bytes() - kCounterBytes;
    const bool tp_io = a.absmax_in != nullptr || a.acc_out != nullptr;  // row-parallel TP shard
    if (tp_io || !(aligned && a.x_dtype != kDtypeF32 && linear_is_fused(a.M, a.N, a.K, sms))) {
        const size_t a8_off = linear_scratch_bytes(a.M, a.N, a.K, sms) - round_up(a8_bytes(a.M, a.K), 256) -
                              round_up(pad_m(a.M) * sizeof(float), 256);
        int8_t* q = reinterpret_cast<int8_t*>(ws + a8_off);
        float* sa = a.sa_out ? a.sa_out : reinterpret_cast<float*>(ws + a8_off + round_up(a8_bytes(a.M, a.K), 256));
        cudaError_t e = launch_act_quant(a.x, a.x_dtype, a.ldx, a.M, a.K, q, sa, a.absmax_in, nullptr,
                                         a.pdl, st);
        if (e != cudaSuccess) return e;
        GemmArgs g = {};
        g.qa = q;
        g.sa = sa;
        g.wp = a.wp;
        g.sw = a.sw;
        g.out = a.acc_out ? nullptr : a.out;
        g.acc_out = a.acc_out;
        g.out_dtype = a.out_dtype;
        g.workspace = gemm_ws;
        g.workspace_bytes = gws;
        g.M = a.M;
        g.N = a.N;
        g.K = a.K;
        g.max_ctas = a.max_ctas;
        g.pdl = a.pdl;
        g.trace = a.trace;
        return launch_w4a8_gemm(g, st);
    }
    const SkPlan s = plan_for(a.M, a.N, a.K, sms, true);
    Params p = {};
    p.wp = a.wp;
    p.sw = a.sw;
    p.out = a.out;
    p.out_dtype = a.out_dtype;
    p.M = a.M;
    p.N = a.N;
    p.K = a.K;
    p.Mp = static_cast<int>(pad_m(a.M));
    p.kblocks = s.kblocks;
    p.m_tiles = s.m_tiles;
    p.tiles = s.tiles;
    p.dp_tiles = s.dp_tiles;
    p.sk_units = 0;
    p.max_contrib = 1;
    p.split = s.split;
    p.cluster = fused_cluster(s);
    static const bool plan_log = ODY_DIAG_ENV("ODY_PLAN_LOG") != nullptr;
    if (plan_log)
        std::fprintf(stderr, "[ody] fused %dx%dx%d: grid %d split %d dp_tiles %d cluster %d (max active %d)\n",
                     a.M, a.N, a.K, s.P, s.split, s.dp_tiles, p.cluster,
                     max_active_clusters_fused(p.cluster));
    const size_t esz = a.out_dtype == kDtypeF32 ? 4 : 2;
    p.bulk_out = ((static_cast<size_t>(a.N) * esz) % 16 == 0 &&
                  (reinterpret_cast<uintptr_t>(a.out) & 15) == 0)
                     ? 1
                     : 0;
    p.x = a.x;
    p.x_dtype = a.x_dtype;
    p.ldx = a.ldx;
    p.sa_out = a.sa_out;
    p.ws_cnt = reinterpret_cast<uint32_t*>(gemm_ws);
    p.ws_slots = reinterpret_cast<int32_t*>(gemm_ws + kCounterBytes);
    p.pdl = a.pdl ? 1 : 0;
    static const char* dbg_env = ODY_DIAG_ENV("ODY_DBG_FUSE");
    p.dbg = dbg_env ? std::atoi(dbg_env) : 0;
    p.trace = a.trace;
    return launch_bn<16, true>(p, s.P, a.pdl, st);
}

}  // namespace odyb200
