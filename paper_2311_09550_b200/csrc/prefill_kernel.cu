// prefill_kernel.cu -- K3+K4 for prefill widths (M > 64): the W4A8 FastGEMM on 2-SM
// tcgen05 MMAs (cta_group::2), 256 weight rows x BT tokens per CTA pair.
//
// Reference semantics (ref gemm.cpp:251-279), unchanged from the tile GEMM:
//     acc  = sum_k a[i][k] * (16 * w[j][k]);  acc >>= 4;  out = float(acc) * (sa[i] * sw[j])
//
// Why a separate kernel.  At M = 1024 the 1-SM tile GEMM (gemm_kernel.cu: 128 weight rows
// x 128 tokens, A widened into TMEM once per (n, m) tile) moves 24 KiB of operands per
// 256 MMA cycles per SM and re-widens every weight tile for every token tile; it reaches
// 0.14-0.30 of the INT8 peak.  Here a CTA PAIR runs one 256 x BT x 32 MMA per
// instruction: each CTA stages its own 128 weight rows (8 KiB INT4) and HALF of the
// BT-token activation tile, and the pair's MMA reads both CTAs' shared memory -- 24 KiB
// per 512 MMA cycles per SM at BT = 256 -- and each weight k-block is widened once per
// 256 tokens instead of once per 128.
//
//   * producer (warp 0, each CTA): 1-D bulk copies of the CTA's half activation k-block
//     into an S-stage ring; a stage is [B half tile | A tile];
//   * converters (warps 4..11, each CTA): warp g owns stage g.  It loads the 8 KiB INT4
//     block of its next k-block straight from L2 into registers (one k-block ahead: W
//     never passes through shared memory, whose bandwidth the bulk copies, the A tiles and
//     the MMA operand reads share), widens it with the paper's high-nibble trick
//     ((w<<4)&0xF0F0F0F0, w&0xF0F0F0F0 -> value*16, no scale multiply) into the stage's A
//     tile (SWIZZLE_128B K-major canonical layout), fence.proxy.async, and after its CTA's
//     B landed arrives (cluster scope) on the LEADER's ready[s].  Stage ownership keeps
//     every barrier's waiter single and in order while the warps' latencies overlap;
//   * MMA (warp 1 of the leader CTA only): tcgen05.mma.cta_group::2.kind::i8, M=256
//     (both CTAs' weight rows), N=BT (both CTAs' token halves), K=32, accumulators in a
//     double-buffered TMEM tile; commits multicast to both CTAs' stage / tile barriers;
//   * epilogue (warps 12..15, each CTA): tcgen05.ld its 128 rows x 32 tokens at a time,
//     exact >>4, __fmul_rn(float(acc), __fmul_rn(sa, sw)) in the reference's order, RN
//     f16/bf16 conversion two at a time, staged [token][row] in smem and written as
//     16-byte row pieces (or the raw int32 accumulators for the exactness suite).
// Tiles (pair n-tile, token tile) are assigned round-robin over the persistent clusters,
// token tile fastest, so the clusters in flight read each weight tile at about the same
// time (L2 hits) and the whole activation matrix stays L2-resident (evict_last).
//
// Measured (B200, M = 1024, LLaMA-13B shapes): 0.36-0.64 of the 4.5 POPS INT8 dense
// peak (layer 276 us); the k-block pipeline is bound by shared-memory traffic (~64 KiB
// per k-block per SM: B bulk-copy write + A tile write + both MMA operand reads) and by
// the stage round trip.  Explored and rejected: A in TMEM (TS MMA),
// separate W/B/A rings, two warps per k-block, register-direct epilogue stores, 4-CTA
// clusters with the activation tile multicast to both pairs (CL = 4 below, opt-in).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "kernels.h"
#include "layout.h"
#include "ptx.cuh"

namespace odyb200 {

namespace {

constexpr int kPThreads = 512;  // 16 warps
constexpr int kPWarpProducer = 0;
constexpr int kPWarpMma = 1;
constexpr int kPWarpAlloc = 2;
constexpr int kPWarpConv0 = 4;   // warps 4..11: converters
constexpr int kPConvWarps = 8;
constexpr int kPWarpEpi0 = 12;   // warps 12..15
constexpr int kPTmemCols = 512;
constexpr int kATileBytes = kTileN * kBlockK;  // 16 KiB of widened int8 weights
constexpr int kEpiTok = 32;                    // tokens per epilogue chunk (tcgen05.ld x32)
constexpr int kOutStageBytes = kEpiTok * kTileN * 4;
// trace layout: [cta 0/1][k-block u < 256][4: producer past empty, converter past full,
// converter arrived, MMA past ready], then [cta][tile j < 16][2: epilogue start, end]
constexpr int kTrK = 256;
__device__ __forceinline__ void trk(unsigned long long* t, int slot, int u) {
    if (t && blockIdx.x < 2 && u < kTrK) t[(blockIdx.x * kTrK + u) * 4 + slot] = globaltimer();
}
// epilogue phases of CTA 0 / warp kPWarpEpi0, tile 0: [chunk < 8][5]
__device__ __forceinline__ void trp(unsigned long long* t, int chunk, int ph) {
    if (t && blockIdx.x == 0 && chunk < 8) t[2 * kTrK * 4 + 64 + chunk * 5 + ph] = clock64();
}
__device__ __forceinline__ void tre(unsigned long long* t, int slot, int j) {
    if (t && blockIdx.x < 2 && j < 16) t[2 * kTrK * 4 + (blockIdx.x * 16 + j) * 2 + slot] = globaltimer();
}

template <int BT>
struct PCfg {
    static constexpr int kHalfT = BT / 2;                  // tokens of B staged per CTA
    static constexpr int kBBytes = kHalfT * kBlockK;       // 16 / 8 KiB
    // one ring; a stage = [B half tile | packed W block] (landed by the producer) + the
    // widened A tile (written by the converter group that owns the stage), all released
    // together by the MMA commit
    // stage = [B half tile | A tile]; the producer lands the packed W block in the first
    // 8 KiB of the A tile and the converter warp, holding all of W in registers, widens it
    // in place -- so a stage costs kBBytes + 16 KiB, not + 24 KiB
    static constexpr int kLoadBytes = kBBytes + kATileBytes;
    static constexpr int kLoadStages = (216 * 1024 - kOutStageBytes) / kLoadBytes;
    static constexpr int kAStages = kLoadStages;
    static constexpr int kScaleBytes = 2 * BT * 4;         // per-token scales, per D buffer
    static constexpr int kSmemBytes = kLoadStages * kLoadBytes + kOutStageBytes +
                                      kScaleBytes + 1024 + 1024;
    // kind::i8, D=s32, A=B=s8 signed, K-major both, N=BT, M=256 (2 CTAs)
    static constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                       (static_cast<uint32_t>(BT >> 3) << 17) |
                                       (static_cast<uint32_t>(256 >> 4) << 24);
    static_assert(BT % 16 == 0 && BT >= 64 && BT <= 256, "BT: 2-SM MMA N granularity, 8-row swizzle atoms");
    static_assert(2 * BT <= kPTmemCols, "TMEM: two accumulator buffers");
    static_assert(kLoadBytes % 1024 == 0 && kBBytes % 1024 == 0, "swizzle atom alignment");
    static_assert(kSmemBytes <= 227 * 1024, "smem");
};

struct PParams {
    const int8_t* qa;
    const float* sa;
    const uint8_t* wp;
    const float* sw;
    void* out;
    int32_t* acc_out;
    int out_dtype;
    int M, N, K, Mp;
    int kblocks, n_tiles, pair_tiles, m_tiles, tiles;
    int split_r;  // the last split_r tiles run as 2 half-width items each (filling the final round)
    int items;    // tiles + split_r
    int pdl;
    int vec_out;  // output rows are 16-byte aligned (N * esz % 16 == 0, aligned base)
    unsigned long long* trace;  // diagnostics: CTAs 0/1, per k-block globaltimer (kTrK slots)
    int wreg;  // 1: converter warps load W straight into registers (no smem pass for W)
    int dbg;  // diagnostics (ODY_PREFILL_DBG bits): 1 no loads, 4 no MMAs, 8 no stores
};

// ---------------------------------------------------------------- 2-SM PTX
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "r"(ncols));
}
__device__ __forceinline__ void tmem_relinquish2() {
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
// D[tmem] (+)= A[smem] * B[smem]^T over the CTA pair; issued by the leader CTA.
__device__ __forceinline__ void mma2_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on the mbarrier at the same smem offset in every CTA of `mask` once all prior
// tcgen05 ops of this thread complete.
__device__ __forceinline__ void mma2_commit_mc(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;" ::"r"(smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// Global -> shared 1-D bulk copy delivered to the same smem offset (and completing tx
// bytes on the same-offset mbarrier) in every CTA of ctaMask.
__device__ __forceinline__ void bulk_g2s_mc(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint16_t mask, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4, %5;" ::"r"(smem_u32(dst_smem)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr) {
    // K-major SWIZZLE_128B: start>>4, LBO unused, SBO = 1024 B (8 rows x 128 B), version 1.
    return static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(64) << 32) |
           (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}
__device__ __forceinline__ unsigned short lds16(uint32_t addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr) : "memory");
    return v;
}
// 32 lanes x 32 consecutive 32-bit columns.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr)
        : "memory");
}

// CL = CTAs per cluster: 2 (one pair) or 4 (two pairs on adjacent weight tiles, same
// tokens): each CTA then bulk-loads 1/(CL/2) of its activation half tile and multicasts
// it to the same-rank CTA of every pair, cutting the per-SM L2 read bytes.
// A work item: a whole (pair n-tile, token tile), or -- for the last split_r tiles, so
// the final round of the persistent grid is not left mostly idle -- one token half of it.
struct PItem {
    int tile;  // cluster tile index: np-major, token tile fastest
    int t0;    // first token
    int bt;    // tokens (MMA N)
};
template <int BT>
__device__ __forceinline__ PItem prefill_item(const PParams& p, int it) {
    const int full = p.tiles - p.split_r;
    if (it < full) return {it, (it % p.m_tiles) * BT, BT};
    const int h = it - full;
    const int tile = full + (h >> 1);
    return {tile, (tile % p.m_tiles) * BT + (h & 1) * (BT / 2), BT / 2};
}

template <int BT, int CL>
__global__ void __launch_bounds__(kPThreads, 1) w4a8_prefill_kernel(const PParams p) {
    using C = PCfg<BT>;
    constexpr int NP = CL / 2;                          // pairs per cluster
    constexpr uint16_t kAllMask = (1u << CL) - 1u;
    constexpr int LS = C::kLoadStages, AS = C::kAStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* lring = smem;                                   // [LS][B | W -> A]
    uint8_t* ostage = lring + LS * C::kLoadBytes;            // epilogue staging
    float* sbuf = reinterpret_cast<float*>(ostage + kOutStageBytes);  // [2][BT]
    uint64_t* bars = reinterpret_cast<uint64_t*>(ostage + kOutStageBytes + C::kScaleBytes);
    uint64_t* full = bars;                // [LS] producer tx (local)
    uint64_t* empty = full + LS;          // [LS] MMA commit (multicast to the pair)
    uint64_t* ready = empty + LS;         // [AS] leader: both CTAs' converter warps
    uint64_t* d_full = ready + AS;        // [2] MMA commit (multicast)
    uint64_t* d_empty = d_full + 2;       // [2] leader: both CTAs' epilogue warps (count 8)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + 2);
    const uint32_t l_base = smem_u32(lring);
    const uint32_t a_base = l_base + C::kBBytes;  // A tile of stage s at a_base + s * kLoadBytes

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t crank = cluster_ctarank();
    const uint32_t rank = crank & 1u;             // rank in the pair; 0 = leader (issues the MMAs)
    const int pi = static_cast<int>(crank >> 1);  // pair index in the cluster
    const uint32_t leader = crank & ~1u;
    const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pi));
    uint16_t peer_mask = 0;                       // same pair rank in every pair (B multicast)
#pragma unroll
    for (int q = 0; q < NP; ++q) peer_mask |= static_cast<uint16_t>(1u << (2 * q + rank));
    const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
    if (p.pdl) pdl_launch_dependents();

    if (threadIdx.x == 0) {
        for (int i = 0; i < LS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NP);  // every pair's MMAs released the stage
        }
        for (int i = 0; i < AS; ++i) mbar_init(&ready[i], 2);  // both CTAs' converter warp
        for (int i = 0; i < 2; ++i) {
            mbar_init(&d_full[i], 1);
            mbar_init(&d_empty[i], 8);
        }
        fence_mbar_init();
    }
    if (warp == kPWarpAlloc) {
        tmem_alloc2(tmem_slot, kPTmemCols);
        tmem_relinquish2();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the peer's barriers are initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem = lds32(smem_u32(tmem_slot));

    if (warp == kPWarpProducer) {
        if (lane == 0) {
            const uint64_t pol_w = l2_policy_evict_normal();
            const uint64_t pol_a = l2_policy_evict_last();
            if (p.pdl) pdl_wait();  // activations come from the previous kernel
            int u = 0;
            constexpr int kSlice = C::kBBytes / NP;  // this CTA's multicast share of B
            for (int itx = cid; itx < p.items; itx += ncl) {
                const PItem im = prefill_item<BT>(p, itx);
                const int np = (im.tile / p.m_tiles) * NP + pi;
                const int nt = 2 * np + static_cast<int>(rank);
                const int half_t = im.bt / 2;  // tokens of B this CTA stages
                const int tok0 = im.t0 + static_cast<int>(rank) * half_t;
                const bool has_w = nt < p.n_tiles;
                // activation rows inside the a8 buffer (the last token tile may overhang Mp
                // when BT does not divide it; the overhanging MMA columns are never stored)
                const int brows = NP == 1 ? max(0, min(half_t, p.Mp - tok0)) : (tok0 < p.Mp ? half_t : 0);
                const bool has_b = brows > 0;
                const uint8_t* wsrc = p.wp + static_cast<size_t>(nt) * p.kblocks * kWBlockBytes;
                const int8_t* bsrc = p.qa + static_cast<size_t>(tok0) * kBlockK;
                for (int kb = 0; kb < p.kblocks; ++kb, ++u) {
                    const int s = u % LS;
                    uint8_t* st = lring + s * C::kLoadBytes;
                    mbar_wait(&empty[s], ((u / LS) & 1) ^ 1);
                    trk(p.trace, 0, u);
                    if (p.dbg & 1) {
                        mbar_arrive(&full[s]);
                        continue;
                    }
                    const bool tma_w = has_w && !p.wreg;
                    mbar_expect_tx(&full[s], (tma_w ? kWBlockBytes : 0) + brows * kBlockK);
                    if (tma_w)
                        bulk_g2s(st + C::kBBytes, wsrc + static_cast<size_t>(kb) * kWBlockBytes,
                                 kWBlockBytes, &full[s], pol_w);
                    if (has_b) {
                        const int8_t* src = bsrc + static_cast<size_t>(kb) * p.Mp * kBlockK + pi * kSlice;
                        if (NP == 1)
                            bulk_g2s(st, src, brows * kBlockK, &full[s], pol_a);
                        else
                            bulk_g2s_mc(st + pi * kSlice, src, kSlice, &full[s], peer_mask, pol_a);
                    }
                }
            }
        }
    } else if (warp == kPWarpMma) {
        if (rank == 0) {
            const uint16_t all_mask = kAllMask;
            int u = 0, j = 0;
            for (int itx = cid; itx < p.items; itx += ncl, ++j) {
                const PItem im = prefill_item<BT>(p, itx);
                // MMA N = the item's token count (instruction-descriptor bits 17..22)
                const uint32_t idesc = (C::kIdesc & ~(0x3Fu << 17)) | (static_cast<uint32_t>(im.bt >> 3) << 17);
                const int db = j & 1;
                mbar_wait(&d_empty[db], ((j >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + db * BT;
                for (int kb = 0; kb < p.kblocks; ++kb, ++u) {
                    const int s = u % LS, as = u % AS;
                    mbar_wait(&ready[as], (u / AS) & 1);
                    if (lane == 0) trk(p.trace, 3, u);
                    tc_fence_after();
                    const uint32_t ab = a_base + as * C::kLoadBytes, bb = l_base + s * C::kLoadBytes;
                    if (elect_one()) {
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (!(p.dbg & 4))
                                mma2_i8_ss(d_tmem, sw128_desc(ab + 32 * c), sw128_desc(bb + 32 * c), idesc,
                                           (kb > 0 || c > 0) ? 1u : 0u);
                        mma2_commit_mc(&empty[s], all_mask);  // B slices came from every pair
                    }
                    __syncwarp();
                }
                if (elect_one()) mma2_commit_mc(&d_full[db], pair_mask);
                __syncwarp();
            }
        }
    } else if (warp >= kPWarpConv0 && warp < kPWarpConv0 + kPConvWarps) {
        // One warp widens one k-block (128 rows).  Warp g OWNS the stages s with
        // s % kPConvWarps == g and takes their k-blocks in order (so no waiter ever runs a
        // phase ahead on a barrier), while the warps' per-k-block widening + fence +
        // cluster-arrive latencies overlap.
        const int g = warp - kPWarpConv0;
        const uint32_t ready_leader = mapa_shared(smem_u32(ready), leader);
        const int total = ((p.items - cid + ncl - 1) / ncl) * p.kblocks;  // this pair's k-blocks
        const uint32_t sw = static_cast<uint32_t>(lane & 7);  // == row & 7 for rows 32*rr + lane
        if (p.wreg) {
            // W straight from global (L2) into registers, one k-block ahead: W never passes
            // through shared memory, which the bulk copies, the widened A tiles and the MMA
            // operand reads otherwise share (~80 KiB of smem traffic per k-block -> ~64).
            // Warp g owns stage g (LS <= kPConvWarps) and its k-blocks g, g+LS, ...
            const int g0 = g;
            auto load_w = [&](int u, uint4 (&v)[4][4]) {
                const int ti = u / p.kblocks, kb = u - ti * p.kblocks;
                const int tile = prefill_item<BT>(p, cid + ti * ncl).tile;
                const int nt = 2 * ((tile / p.m_tiles) * NP + pi) + static_cast<int>(rank);
                if (nt >= p.n_tiles) {
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                        for (int c = 0; c < 4; ++c) v[rr][c] = make_uint4(0, 0, 0, 0);
                    return;
                }
                const uint4* src = reinterpret_cast<const uint4*>(
                                       p.wp + (static_cast<size_t>(nt) * p.kblocks + kb) * kWBlockBytes) + lane;
#pragma unroll
                for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                    for (int c = 0; c < 4; ++c) v[rr][c] = __ldg(src + c * 128 + rr * 32);
            };
            if (g0 < LS && g0 < total) {
                uint4 v[4][4];
                load_w(g0, v);
                for (int u = g0; u < total; u += LS) {
                    const int s = g0, as = s;
                    mbar_wait(&empty[s], ((u / LS) & 1) ^ 1);  // A tile free: MMA of u - LS done
                    if (lane == 0) trk(p.trace, 1, u);
#pragma unroll
                    for (int rr = 0; rr < 4; ++rr) {
                        const uint32_t dst = a_base + as * C::kLoadBytes + (rr * 32 + lane) * 128;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint4 w = v[rr][c];
                            const uint4 lo = make_uint4((w.x << 4) & 0xF0F0F0F0u, w.x & 0xF0F0F0F0u,
                                                        (w.y << 4) & 0xF0F0F0F0u, w.y & 0xF0F0F0F0u);
                            const uint4 hi = make_uint4((w.z << 4) & 0xF0F0F0F0u, w.z & 0xF0F0F0F0u,
                                                        (w.w << 4) & 0xF0F0F0F0u, w.w & 0xF0F0F0F0u);
                            sts128(dst + (((2 * c) ^ sw) << 4), lo);      // k 32c .. 32c+15
                            sts128(dst + (((2 * c + 1) ^ sw) << 4), hi);  // k 32c+16 .. 32c+31
                        }
                    }
                    fence_proxy_async_shared();  // generic smem writes -> tensor-core reads
                    mbar_wait(&full[s], (u / LS) & 1);  // this CTA's B landed (the leader's MMA reads it)
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote(ready_leader + as * 8);
                    if (lane == 0) trk(p.trace, 2, u);
                    if (u + LS < total) load_w(u + LS, v);
                }
            }
        } else
        for (int u = 0; u < total; ++u) {
            const int s = u % LS, as = s;
            if (s % kPConvWarps != g) continue;
            mbar_wait(&full[s], (u / LS) & 1);
            if (lane == 0) trk(p.trace, 1, u);
            const uint32_t src = l_base + s * C::kLoadBytes + C::kBBytes + lane * 16;
            uint4 v[4][4];  // all 16 loads in flight before the first widening
#pragma unroll
            for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                for (int c = 0; c < 4; ++c) v[rr][c] = lds128(src + rr * 512 + c * 2048);
            __syncwarp();  // every lane has read W before any lane overwrites it with A
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
                const uint32_t dst = a_base + as * C::kLoadBytes + (rr * 32 + lane) * 128;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    // word j of the row chunk: k = 32c+8j+0..3 low nibbles, +4..7 high nibbles
                    const uint4 w = v[rr][c];
                    const uint4 lo = make_uint4((w.x << 4) & 0xF0F0F0F0u, w.x & 0xF0F0F0F0u,
                                                (w.y << 4) & 0xF0F0F0F0u, w.y & 0xF0F0F0F0u);
                    const uint4 hi = make_uint4((w.z << 4) & 0xF0F0F0F0u, w.z & 0xF0F0F0F0u,
                                                (w.w << 4) & 0xF0F0F0F0u, w.w & 0xF0F0F0F0u);
                    sts128(dst + (((2 * c) ^ sw) << 4), lo);      // k 32c .. 32c+15
                    sts128(dst + (((2 * c + 1) ^ sw) << 4), hi);  // k 32c+16 .. 32c+31
                }
            }
            fence_proxy_async_shared();  // generic smem writes -> tensor-core reads
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(ready_leader + as * 8);
            if (lane == 0) trk(p.trace, 2, u);
        }
    } else if (warp >= kPWarpEpi0) {
        const int q = warp & 3;
        const int r = 32 * q + lane;
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(32 * q) << 16);
        const uint32_t d_empty_leader = mapa_shared(smem_u32(d_empty), leader);
        const int esz = (p.acc_out || p.out_dtype == kDtypeF32) ? 4 : 2;
        const uint32_t ob = smem_u32(ostage);
        if (p.pdl) pdl_wait();
        int j = 0;
        for (int itx = cid; itx < p.items; itx += ncl, ++j) {
            const PItem im = prefill_item<BT>(p, itx);
            const int db = j & 1;
            const int np = (im.tile / p.m_tiles) * NP + pi;
            const int n0 = (2 * np + static_cast<int>(rank)) * kTileN;
            const int n = n0 + r;
            const int t0 = im.t0;
            const float sw_n = n < p.N ? __ldg(p.sw + n) : 0.0f;
            float* sc = sbuf + db * BT;
            for (int i = r; i < im.bt; i += 128) sc[i] = t0 + i < p.M ? __ldg(p.sa + t0 + i) : 0.0f;
            named_bar_sync(1, 128);
            mbar_wait(&d_full[db], (j >> 1) & 1);
            if (r == 0) tre(p.trace, 0, j);
            tc_fence_after();
            const int tn = min(im.bt, p.M - t0);  // valid tokens of this item
            const int nn = min(kTileN, p.N - n0);  // valid weight rows (may be <= 0)
            // 16-byte pieces per staged token row
            const int per_row = kTileN * esz / 16;
#pragma unroll 1
            for (int tc = 0; tc < im.bt; tc += kEpiTok) {
                uint32_t v[32];
                __syncwarp();  // tcgen05.ld is .sync.aligned: the whole warp, converged
                const bool ptr = j == 0 && r == 0;
                if (ptr) trp(p.trace, tc / kEpiTok, 0);
                tmem_ld_32x32b_x32(t_lane + db * BT + tc, v);
                tmem_wait_ld();
                if (ptr) trp(p.trace, tc / kEpiTok, 1);
                if (tc >= tn || nn <= 0 || (p.dbg & 8)) continue;  // uniform over the CTA
                // stage [token][row] so each token row leaves as contiguous 16-byte pieces.
                // All 32 results are computed before the first smem store (the asm
                // stores are ordered memory ops: interleaving them with the scale loads
                // serialises every element on a load latency).
                uint32_t ov[32];
                if (p.acc_out) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) ov[i] = v[i];
                } else {
                    float o[32];
                    const uint32_t sca = smem_u32(sc + tc);
#pragma unroll
                    for (int i4 = 0; i4 < 8; ++i4) {
                        const uint4 s4 = lds128(sca + 16 * i4);
                        o[4 * i4 + 0] = __uint_as_float(s4.x);
                        o[4 * i4 + 1] = __uint_as_float(s4.y);
                        o[4 * i4 + 2] = __uint_as_float(s4.z);
                        o[4 * i4 + 3] = __uint_as_float(s4.w);
                    }
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int32_t sh = static_cast<int32_t>(v[i]) >> 4;  // exact (ref gemm.cpp:269)
                        o[i] = __fmul_rn(__int2float_rn(sh), __fmul_rn(o[i], sw_n));
                    }
                    // RN conversions, two per packed ALU instruction (same rounding as the
                    // scalar __float2half_rn / __float2bfloat16_rn)
                    if (p.out_dtype == kDtypeF16) {
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const __half2 h = __floats2half2_rn(o[i], o[i + 1]);
                            const uint32_t u = *reinterpret_cast<const uint32_t*>(&h);
                            ov[i] = u & 0xFFFFu;
                            ov[i + 1] = u >> 16;
                        }
                    } else if (p.out_dtype == kDtypeBF16) {
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const __nv_bfloat162 h = __floats2bfloat162_rn(o[i], o[i + 1]);
                            const uint32_t u = *reinterpret_cast<const uint32_t*>(&h);
                            ov[i] = u & 0xFFFFu;
                            ov[i + 1] = u >> 16;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) ov[i] = __float_as_uint(o[i]);
                    }
                }
                if (esz == 4) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) sts32(ob + (i * kTileN + r) * 4, ov[i]);
                } else {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        sts16(ob + (i * kTileN + r) * 2, static_cast<unsigned short>(ov[i]));
                }
                if (ptr) trp(p.trace, tc / kEpiTok, 2);
                named_bar_sync(1, 128);
                if (ptr) trp(p.trace, tc / kEpiTok, 3);
                uint8_t* dst = p.acc_out ? reinterpret_cast<uint8_t*>(p.acc_out) : static_cast<uint8_t*>(p.out);
                const int rows = min(kEpiTok, tn - tc);
                for (int c = r; c < rows * per_row; c += 128) {
                    const int t = c / per_row, piece = c % per_row;
                    const int e0 = piece * 16 / esz;  // first row (n) of the piece
                    uint8_t* g = dst + (static_cast<size_t>(t0 + tc + t) * p.N + n0 + e0) * esz;
                    const uint32_t sa_ = ob + (t * kTileN + e0) * esz;
                    if (p.vec_out && e0 + 16 / esz <= nn) {
                        *reinterpret_cast<uint4*>(g) = lds128(sa_);
                    } else {
                        for (int e = 0; e < 16 / esz && e0 + e < nn; ++e) {
                            if (esz == 4)
                                reinterpret_cast<uint32_t*>(g)[e] = lds32(sa_ + 4 * e);
                            else
                                reinterpret_cast<unsigned short*>(g)[e] = lds16(sa_ + 2 * e);
                        }
                    }
                }
                if (ptr) trp(p.trace, tc / kEpiTok, 4);
                named_bar_sync(1, 128);  // staging reusable
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(d_empty_leader + db * 8);
            if (r == 0) tre(p.trace, 1, j);
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();  // no CTA leaves while its peer may still signal or read it
    tc_fence_after();
    if (warp == kPWarpAlloc) tmem_dealloc2(tmem, kPTmemCols);
}

template <int BT, int CL>
cudaError_t prefill_attr() {
    static std::once_flag once;
    static cudaError_t err = cudaSuccess;
    std::call_once(once, [] {
        err = cudaFuncSetAttribute(w4a8_prefill_kernel<BT, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   PCfg<BT>::kSmemBytes);
    });
    return err;
}

template <int BT, int CL>
int prefill_max_clusters() {
    static int n = [] {
        if (prefill_attr<BT, CL>() != cudaSuccess) return 0;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CL * (148 / CL));
        cfg.blockDim = dim3(kPThreads);
        cfg.dynamicSmemBytes = PCfg<BT>::kSmemBytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int c = 0;
        if (cudaOccupancyMaxActiveClusters(&c, w4a8_prefill_kernel<BT, CL>, &cfg) != cudaSuccess || c <= 0) {
            cudaGetLastError();
            c = device_sm_count() / CL;
        }
        return c;
    }();
    return n;
}

template <int BT, int CL>
cudaError_t launch_prefill_bt(PParams p, int max_ctas, cudaStream_t st) {
    const cudaError_t e = prefill_attr<BT, CL>();
    if (e != cudaSuccess) return e;
    p.m_tiles = (p.M + BT - 1) / BT;
    p.tiles = ((p.pair_tiles + CL / 2 - 1) / (CL / 2)) * p.m_tiles;  // cluster tiles
    int clusters = prefill_max_clusters<BT, CL>();
    if (max_ctas > 0) clusters = std::min(clusters, std::max(1, max_ctas / CL));
    clusters = std::min(clusters, p.tiles);
    // a final round with few tiles: split each of them into two token halves when the
    // halves still fit one round (BT/2 keeps the 2-SM N and swizzle-row granularity)
    {
        const int r = p.tiles % clusters;
        p.split_r = (CL == 2 && BT % 32 == 0 && r > 0 && 2 * r <= clusters && p.tiles > clusters) ? r : 0;
        static const char* nosplit = ODY_DIAG_ENV("ODY_PREFILL_NOSPLIT");
        if (nosplit && std::atoi(nosplit)) p.split_r = 0;
        p.items = p.tiles + p.split_r;
    }
    static const bool plan_log = ODY_DIAG_ENV("ODY_PLAN_LOG") != nullptr;
    if (plan_log)
        std::fprintf(stderr, "[ody] prefill %dx%dx%d: BT %d CL %d tiles %d (+%d split) clusters %d stages %d\n", p.M,
                     p.N, p.K, BT, CL, p.tiles, p.split_r, clusters, PCfg<BT>::kLoadStages);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * clusters);
    cfg.blockDim = dim3(kPThreads);
    cfg.dynamicSmemBytes = PCfg<BT>::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    int na = 1;
    if (p.pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, w4a8_prefill_kernel<BT, CL>, p);
}

}  // namespace

// Per calling thread (like the CUDA current device): a switch set by one host thread
// never changes the kernel choice of a launch issued concurrently by another.
static int default_prefill_min_m() {
    const char* env = ODY_DIAG_ENV("ODY_PREFILL");
    return env ? std::atoi(env) : 65;  // M = 128 / 192 / 256: 1.7-2.5x the tile GEMM; M = 64: the tile GEMM wins
}
static thread_local int g_prefill_min_m = default_prefill_min_m();
void set_prefill_min_m(int m) { g_prefill_min_m = m; }
bool prefill_eligible(int M, int N, int K) {
    return g_prefill_min_m > 0 && M >= g_prefill_min_m && N > 0 && K > 0;
}

// Token-tile width: the candidate minimising the modelled makespan -- rounds of items
// over the persistent CTA pairs (a final round of half-width split items counted as 0.6)
// times a per-item cost of BT + 60 token-columns (fitted to the measured M = 1024 LLaMA
// shapes: BT 256 for qkv / gate_up, 160 for the N = 5120 shapes, whose 20 pair tiles
// leave a BT = 256 grid mostly idle in its second round).
int pick_prefill_bt(int M, int pair_tiles) {
    static const int kCand[] = {256, 224, 192, 176, 160, 128};
    const int pairs = std::max(1, device_sm_count() / 2);
    int best = 256;
    double best_cost = 1e30;
    for (int bt : kCand) {
        const long long tiles = static_cast<long long>(pair_tiles) * ((M + bt - 1) / bt);
        const long long r = tiles % pairs;
        const bool split = bt % 32 == 0 && r > 0 && 2 * r <= pairs && tiles > pairs;  // as the launcher
        const double rounds = static_cast<double>(tiles / pairs) + (r == 0 ? 0.0 : (split ? 0.6 : 1.0));
        const double cost = rounds * (bt + 60);
        if (cost < best_cost * 0.999) {
            best_cost = cost;
            best = bt;
        }
    }
    return best;
}

cudaError_t launch_w4a8_prefill(const GemmArgs& a, cudaStream_t st) {
    if (a.M <= 0 || a.N <= 0 || a.K <= 0) return cudaErrorInvalidValue;
    PParams p = {};
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
    p.kblocks = static_cast<int>(pad_k(a.K) / kBlockK);
    p.n_tiles = static_cast<int>(pad_n(a.N) / kTileN);
    p.pair_tiles = (p.n_tiles + 1) / 2;
    p.pdl = a.pdl ? 1 : 0;
    p.trace = a.trace;
    {
        const size_t esz = (a.acc_out || a.out_dtype == kDtypeF32) ? 4 : 2;
        const void* o = a.acc_out ? static_cast<const void*>(a.acc_out) : a.out;
        p.vec_out = ((static_cast<size_t>(a.N) * esz) % 16 == 0 && (reinterpret_cast<uintptr_t>(o) & 15) == 0) ? 1 : 0;
    }
    static const char* wreg_env = ODY_DIAG_ENV("ODY_PREFILL_WREG");
    p.wreg = wreg_env ? std::atoi(wreg_env) : 1;
    static const char* dbg_env = ODY_DIAG_ENV("ODY_PREFILL_DBG");
    p.dbg = dbg_env ? std::atoi(dbg_env) : 0;
    static const char* cl_env = ODY_DIAG_ENV("ODY_PREFILL_CL");
    if (cl_env && std::atoi(cl_env) == 4) return launch_prefill_bt<256, 4>(p, a.max_ctas, st);
    static const char* bt_env = ODY_DIAG_ENV("ODY_PREFILL_BT");
    const int bt = bt_env ? std::atoi(bt_env) : pick_prefill_bt(p.M, p.pair_tiles);
    switch (bt) {
        case 128: return launch_prefill_bt<128, 2>(p, a.max_ctas, st);
        case 160: return launch_prefill_bt<160, 2>(p, a.max_ctas, st);
        case 176: return launch_prefill_bt<176, 2>(p, a.max_ctas, st);
        case 192: return launch_prefill_bt<192, 2>(p, a.max_ctas, st);
        case 224: return launch_prefill_bt<224, 2>(p, a.max_ctas, st);
        default: return launch_prefill_bt<256, 2>(p, a.max_ctas, st);
    }
}

}  // namespace odyb200
