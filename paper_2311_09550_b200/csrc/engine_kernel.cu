// engine_kernel.cu -- the reference's comparison GEMM engines on tcgen05 (the paper's
// Fig. 7 ablation), behind ody_gemm(engine, ...):
//
//   ODY_ENGINE_W8A8         ref gemm.cpp:281-311   acc = sum a*w (int8 x int8),        out = float(acc)*(sa*sw)
//   ODY_ENGINE_ASYMMETRIC   ref gemm.cpp:163-202   w stored as UINT4 + 8 (ref :56-75), the kernel
//                                                  subtracts the zero point per lane, out as W8A8
//   ODY_ENGINE_FINEGRAINED  ref gemm.cpp:123-161   per group g: sub = sum a*w (int32), leaves the
//                                                  integer domain: acc += float(sub)*(sa*s_g)
//   ODY_ENGINE_FAST (here)  ref gemm.cpp:251-279   the same kernel with the high-nibble widening,
//                                                  so the four dequant schemes run on one data path
//   ODY_ENGINE_W4A16        ref gemm.cpp:100-121   f32 activations x dequantized weights, one
//                                                  thread per output, the reference's sequential
//                                                  f32 order (w4a16_kernel below)
//
// One CTA = 128 weight rows (MMA M) x BN tokens (MMA N) over a k-range, SS operands:
//   warp 0       producer: 1-D bulk copies of the k-block's weight tile (8 KiB packed INT4
//                or 16 KiB INT8) and activation tile (BN x 128 B, SWIZZLE_128B) per stage
//   warp 1       MMA: tcgen05.mma.cta_group::1.kind::i8, A and B from smem, D in TMEM
//   warp 2       TMEM allocator
//   warps 4..7   converters (INT4 modes): widen the packed row chunk to 128 int8 lanes into
//                a SWIZZLE_128B A tile -- FAST/FINE: (w<<4)&0xF0F0F0F0 | w&0xF0F0F0F0 (x16);
//                ASYM: ((u>>4j)&0x0F0F0F0F) - 0x08080808 per byte (the zero-point subtract)
//   warps 8..11  epilogue: tcgen05.ld, the engine's dequant, f32 row-major store
// Integer engines split K over up to 8 CTAs (exact int32 red.add into an L2 workspace;
// the last CTA of a tile finalises it).  FINEGRAINED is never split: its float
// accumulation runs group by group in the reference's order (a TMEM ring of per-group
// int32 sums feeds the epilogue while the next groups accumulate).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "kernels.h"
#include "layout.h"
#include "ptx.cuh"
#include "quant_common.cuh"

namespace odyb200 {

namespace {

constexpr int kEThreads = 384;
constexpr int kEWarpProd = 0, kEWarpMma = 1, kEWarpAlloc = 2, kEWarpConv0 = 4, kEWarpEpi0 = 8;
constexpr int kFineBufs = 4;  // TMEM ring of per-group accumulators

template <int MODE, int BN>
struct ECfg {
    static constexpr bool kW8 = MODE == kEngineW8A8;
    static constexpr bool kFine = MODE == kEngineFine;
    static constexpr int kWBytes = kW8 ? 16384 : kWBlockBytes;     // one k-block of the tile
    static constexpr int kBBytes = BN * 128;
    static constexpr int kABytes = kW8 ? 0 : 16384;               // widened A tile
    static constexpr int kStageBytes = kWBytes + kBBytes + kABytes;
    static constexpr int kStages = (200 * 1024) / kStageBytes < 6 ? (200 * 1024) / kStageBytes : 6;
    static constexpr int kSmem = kStages * kStageBytes + 1024 /*barriers*/ + 1024 /*align*/;
    static constexpr int kAccCols = kFine ? kFineBufs * BN : BN;
    static constexpr int kTmemCols = kAccCols <= 32 ? 32 : (kAccCols <= 64 ? 64 : (kAccCols <= 128 ? 128 : (kAccCols <= 256 ? 256 : 512)));
    // kind::i8, D=s32, A=B=s8 signed, K-major both, N=BN, M=128
    static constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                       (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
    static_assert(kStages >= 2, "stages");
    static_assert(kStageBytes % 1024 == 0, "swizzle atoms");
};

struct EParams {
    const uint8_t* w;   // W4 tile layout (FAST/FINE), its UINT4+8 twin (ASYM) or the W8 layout
    const float* sw;    // [N] per-channel, or [N][groups] (FINE)
    const int8_t* qa;   // a8 k-block layout, Mp rows
    const float* sa;
    float* out;         // M x N f32
    int M, N, K, Mp, Np, kblocks;
    int g, groups;      // FINE: group size (a multiple of 32) and groups per row
    int splits;         // integer engines: CTAs per tile along K
    int32_t* ws;        // splits > 1: M x N int32 sums (zeroed; left zeroed)
    uint32_t* cnt;      // splits > 1: per-tile arrivals (zeroed; left zeroed)
};

__device__ __forceinline__ uint64_t e_desc(uint32_t smem_addr) {
    // K-major SWIZZLE_128B: start>>4, SBO = 1024 B (8 rows x 128 B), version 1, swizzle 128B.
    return static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(64) << 32) |
           (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}
__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

template <int MODE>
__device__ __forceinline__ void widen(uint32_t w, uint32_t& lo, uint32_t& hi) {
    if (MODE == kEngineAsym) {  // UINT4 + 8 nibbles: subtract the zero point per lane
        lo = __vsub4(w & 0x0F0F0F0Fu, 0x08080808u);
        hi = __vsub4((w >> 4) & 0x0F0F0F0Fu, 0x08080808u);
    } else {                    // SINT4 -> S8 high-nibble trick: lanes hold value x 16
        lo = (w << 4) & 0xF0F0F0F0u;
        hi = w & 0xF0F0F0F0u;
    }
}

template <int MODE, int BN>
__global__ void __launch_bounds__(kEThreads, 1) engine_gemm_kernel(const __grid_constant__ EParams p) {
    using C = ECfg<MODE, BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* a_full = empty + C::kStages;
    uint64_t* d_full = a_full + C::kStages;     // [kFineBufs] (non-FINE: [0])
    uint64_t* d_empty = d_full + kFineBufs;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(d_empty + kFineBufs);
    uint32_t* last_flag = tmem_slot + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = blockIdx.x, mt = blockIdx.y, sp = blockIdx.z;
    const int kb0 = sp * p.kblocks / p.splits, kb1 = (sp + 1) * p.kblocks / p.splits;
    if (threadIdx.x == 0) {
        for (int i = 0; i < C::kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
            mbar_init(&a_full[i], 4);
        }
        for (int i = 0; i < kFineBufs; ++i) {
            mbar_init(&d_full[i], 1);
            mbar_init(&d_empty[i], 4);
        }
        fence_mbar_init();
    }
    if (warp == kEWarpAlloc) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = lds32(smem_u32(tmem_slot));

    if (warp == kEWarpProd) {
        if (lane == 0) {
            const uint64_t pol_w = l2_policy_evict_first();
            const uint64_t pol_b = l2_policy_evict_last();
            for (int kb = kb0, u = 0; kb < kb1; ++kb, ++u) {
                const int s = u % C::kStages;
                if (u >= C::kStages) mbar_wait(&empty[s], ((u / C::kStages) & 1) ^ 1);
                uint8_t* st = ring + s * C::kStageBytes;
                mbar_expect_tx(&full[s], C::kWBytes + C::kBBytes);
                const uint8_t* wsrc = C::kW8 ? p.w + static_cast<size_t>(kb) * p.Np * 128 + static_cast<size_t>(nt) * 16384
                                             : p.w + (static_cast<size_t>(nt) * p.kblocks + kb) * kWBlockBytes;
                bulk_g2s(st, wsrc, C::kWBytes, &full[s], pol_w);
                bulk_g2s(st + C::kWBytes, p.qa + static_cast<size_t>(kb) * p.Mp * 128 + static_cast<size_t>(mt) * BN * 128,
                         C::kBBytes, &full[s], pol_b);
            }
        }
    } else if (warp == kEWarpMma) {
        int fb = 0;  // FINE: group buffers handed out
        for (int kb = kb0, u = 0; kb < kb1; ++kb, ++u) {
            const int s = u % C::kStages;
            const uint32_t ph = (u / C::kStages) & 1;
            mbar_wait(&full[s], ph);
            if (!C::kW8) mbar_wait(&a_full[s], ph);
            tc_fence_after();
            const uint32_t st = smem_u32(ring + s * C::kStageBytes);
            const uint32_t a0 = C::kW8 ? st : st + C::kWBytes + C::kBBytes;
            const uint32_t b0 = st + C::kWBytes;
            if (elect_one()) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int k = kb * kBlockK + c * 32;
                    if (C::kFine) {
                        if (k >= p.K) break;  // K padding: no group past K
                        const bool first = k % p.g == 0;
                        const int buf = fb % kFineBufs;
                        if (first && fb >= kFineBufs) mbar_wait(&d_empty[buf], ((fb / kFineBufs) & 1) ^ 1);
                        if (first) tc_fence_after();
                        mma_i8_ss(tmem + buf * BN, e_desc(a0 + 32 * c), e_desc(b0 + 32 * c), C::kIdesc, first ? 0u : 1u);
                        if ((k + 32) % p.g == 0) {
                            mma_commit(&d_full[buf]);
                            ++fb;
                        }
                    } else {
                        mma_i8_ss(tmem, e_desc(a0 + 32 * c), e_desc(b0 + 32 * c), C::kIdesc,
                                  (kb > kb0 || c > 0) ? 1u : 0u);
                    }
                }
                mma_commit(&empty[s]);
                if (!C::kFine && kb + 1 == kb1) mma_commit(&d_full[0]);
            }
            __syncwarp();
        }
    } else if (!C::kW8 && warp >= kEWarpConv0 && warp < kEWarpConv0 + 4) {
        const int r = 32 * (warp - kEWarpConv0) + lane;  // weight row of the tile
        for (int kb = kb0, u = 0; kb < kb1; ++kb, ++u) {
            const int s = u % C::kStages;
            mbar_wait(&full[s], (u / C::kStages) & 1);
            const uint32_t st = smem_u32(ring + s * C::kStageBytes);
            const uint32_t at = st + C::kWBytes + C::kBBytes + r * 128;
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // 32 k per packed 16-byte row chunk
                const uint4 v = lds128(st + c * 2048 + r * 16);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                uint32_t l[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) widen<MODE>(w[j], l[2 * j], l[2 * j + 1]);  // k 8j..8j+3, 8j+4..8j+7
                sts128(at + (((2 * c) ^ (r & 7)) << 4), make_uint4(l[0], l[1], l[2], l[3]));
                sts128(at + (((2 * c + 1) ^ (r & 7)) << 4), make_uint4(l[4], l[5], l[6], l[7]));
            }
            fence_proxy_async_shared();  // generic smem writes -> the MMA's async proxy
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_full[s]);
        }
    } else if (warp >= kEWarpEpi0) {
        const int q = warp - kEWarpEpi0;
        const int r = 32 * q + lane;
        const int n = nt * kTileN + r;
        const uint32_t t_lane = tmem + (static_cast<uint32_t>(32 * q) << 16);
        const int t0 = mt * BN;
        const int tm = min(BN, p.M - t0);  // tokens of this tile
        uint32_t v[BN];
        auto load_acc = [&](uint32_t col) {
#pragma unroll
            for (int tc = 0; tc < BN; tc += 16) {
                uint32_t w16[16];
                tmem_ld_32x32b_x16(t_lane + col + tc, w16);
                tmem_wait_ld();
#pragma unroll
                for (int t = 0; t < 16; ++t) v[tc + t] = w16[t];
            }
        };
        if (C::kFine) {
            // ref gemm.cpp:141-153: per group, sub leaves the integer domain, f32 accumulate
            float acc[BN];
#pragma unroll
            for (int t = 0; t < BN; ++t) acc[t] = 0.0f;
            const float* sg = p.sw + static_cast<size_t>(n < p.N ? n : 0) * p.groups;
            for (int gi = 0; gi < p.groups; ++gi) {
                const int buf = gi % kFineBufs;
                mbar_wait(&d_full[buf], (gi / kFineBufs) & 1);
                tc_fence_after();
                load_acc(buf * BN);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&d_empty[buf]);
                const float s_g = n < p.N ? __ldg(sg + gi) : 0.0f;
#pragma unroll
                for (int t = 0; t < BN; ++t) {
                    if (t < tm) {
                        const int32_t sub = static_cast<int32_t>(v[t]) >> 4;  // lanes were x16: exact
                        acc[t] = __fadd_rn(acc[t], __fmul_rn(__int2float_rn(sub), __fmul_rn(__ldg(p.sa + t0 + t), s_g)));
                    }
                }
            }
            if (n < p.N)
#pragma unroll
                for (int t = 0; t < BN; ++t)
                    if (t < tm) p.out[static_cast<size_t>(t0 + t) * p.N + n] = acc[t];
        } else {
            mbar_wait(&d_full[0], 0);
            tc_fence_after();
            load_acc(0);
            tc_fence_before();
            bool fin = true;
            if (p.splits > 1) {
                // exact split-K: int32 sums meet in L2, the tile's last CTA finalises
                int32_t* wsr = p.ws + static_cast<size_t>(t0) * p.N + n;
                if (n < p.N)
#pragma unroll
                    for (int t = 0; t < BN; ++t)
                        if (t < tm) red_add_s32(wsr + static_cast<size_t>(t) * p.N, static_cast<int32_t>(v[t]));
                named_bar_sync(1, 128);
                if (r == 0) {
                    __threadfence();
                    const uint32_t tile = static_cast<uint32_t>(mt) * gridDim.x + nt;
                    const uint32_t old = atomicAdd(p.cnt + tile, 1u);
                    const bool last = old == static_cast<uint32_t>(p.splits - 1);
                    if (last) p.cnt[tile] = 0u;  // every split arrived: re-armed
                    *last_flag = last ? 1u : 0u;
                    __threadfence();
                }
                named_bar_sync(1, 128);
                fin = *reinterpret_cast<volatile uint32_t*>(last_flag) != 0u;
                if (fin && n < p.N)
#pragma unroll
                    for (int t = 0; t < BN; ++t)
                        if (t < tm) {
                            v[t] = static_cast<uint32_t>(__ldcg(wsr + static_cast<size_t>(t) * p.N));
                            wsr[static_cast<size_t>(t) * p.N] = 0;
                        }
            }
            if (fin && n < p.N) {
                const float sw_n = __ldg(p.sw + n);
#pragma unroll
                for (int t = 0; t < BN; ++t) {
                    if (t < tm) {
                        // FAST lanes carry x16: >>4 is exact (ref gemm.cpp:269); the others are plain
                        const int32_t acc = MODE == kEngineFast ? static_cast<int32_t>(v[t]) >> 4 : static_cast<int32_t>(v[t]);
                        p.out[static_cast<size_t>(t0 + t) * p.N + n] =
                            __fmul_rn(__int2float_rn(acc), __fmul_rn(__ldg(p.sa + t0 + t), sw_n));
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kEWarpAlloc) tmem_dealloc(tmem, C::kTmemCols);
}

template <int MODE, int BN>
cudaError_t launch_engine_t(const EParams& p, int n_tiles, int m_tiles, cudaStream_t st) {
    using C = ECfg<MODE, BN>;
    static std::once_flag once;
    static cudaError_t attr = cudaSuccess;
    std::call_once(once, [] {
        attr = cudaFuncSetAttribute(engine_gemm_kernel<MODE, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    });
    if (attr != cudaSuccess) return attr;
    engine_gemm_kernel<MODE, BN><<<dim3(n_tiles, m_tiles, p.splits), kEThreads, C::kSmem, st>>>(p);
    return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_engine_bn(const EParams& p, int bn, int n_tiles, int m_tiles, cudaStream_t st) {
    switch (bn) {
        case 16: return launch_engine_t<MODE, 16>(p, n_tiles, m_tiles, st);
        case 32: return launch_engine_t<MODE, 32>(p, n_tiles, m_tiles, st);
        default: return MODE == kEngineFine ? cudaErrorInvalidValue : launch_engine_t<MODE, 64>(p, n_tiles, m_tiles, st);
    }
}

// ---------------------------------------------------------------- weight formats
// Per-(row, group) scale (ref quantize.cpp:22-35 over each group span): one warp each.
__global__ void wg_scale_kernel(const float* __restrict__ w, int N, int K, int g, int bits,
                                const float* __restrict__ gamma, const float* __restrict__ beta,
                                float* __restrict__ s) {
    const int groups = K / g;
    const int item = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (item >= N * groups) return;
    const int row = item / groups, gi = item % groups;
    const float* r = w + static_cast<size_t>(row) * K + static_cast<size_t>(gi) * g;
    float mx = r[0], mn = r[0];
    for (int k = lane; k < g; k += 32) {
        mx = fmaxf(mx, r[k]);
        mn = fminf(mn, r[k]);
    }
    mx = warp_max(mx);
    mn = warp_min(mn);
    if (lane == 0) {
        const float ga = gamma ? gamma[row] : 1.0f;
        const float be = beta ? beta[row] : 1.0f;
        const float qmax = static_cast<float>((1 << (bits - 1)) - 1);
        const float sc = fmaxf(fabsf(__fmul_rn(ga, mx)), fabsf(__fmul_rn(be, mn))) / qmax;
        s[item] = sc > 0.0f ? sc : kMinScale;
    }
}

// Per-group INT4 codes (scale of the element's group) into the W4 tile layout: one
// thread per (row, 32-k chunk), one 16-byte row chunk.
__global__ void wg_quant_prepack_kernel(const float* __restrict__ w, int N, int K, int g, int Np, int Kp,
                                        const float* __restrict__ s, uint8_t* __restrict__ out) {
    const size_t chunks = Kp / 32;
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<size_t>(Np) * chunks) return;
    const int r = static_cast<int>(idx / chunks);
    const int cc = static_cast<int>(idx % chunks);
    const int groups = K / g;
    uint32_t word[4] = {0u, 0u, 0u, 0u};
    if (r < N) {
        const float* row = w + static_cast<size_t>(r) * K;
#pragma unroll 4
        for (int e = 0; e < 32; ++e) {
            const int k = cc * 32 + e;
            if (k >= K) break;
            const int32_t code = clamp_code(row[k] / s[static_cast<size_t>(r) * groups + k / g], -8, 7);
            const int j = e / 8, b = e % 4, hi = (e % 8) >= 4;
            word[j] |= (static_cast<uint32_t>(code) & 0xFu) << (8 * b + 4 * hi);
        }
    }
    int high;
    const size_t off = w4_offset(r, static_cast<size_t>(cc) * 32, Kp / kBlockK, &high);
    *reinterpret_cast<uint4*>(out + off) = make_uint4(word[0], word[1], word[2], word[3]);
}

// Per-channel INT8 codes into the W8 layout (the a8 k-block layout over Np weight rows:
// a 128-row tile of one k-block is one contiguous, MMA-ready SWIZZLE_128B 16 KiB block).
// One thread per (row, 16-k chunk).
__global__ void w8_quant_kernel(const float* __restrict__ w, int N, int K, int Np, int Kp,
                                const float* __restrict__ s, int8_t* __restrict__ out) {
    const size_t chunks = Kp / 16;
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<size_t>(Np) * chunks) return;
    const int r = static_cast<int>(idx / chunks);
    const int cc = static_cast<int>(idx % chunks);
    uint32_t word[4] = {0u, 0u, 0u, 0u};
    if (r < N) {
        const float sc = s[r];
        const float* row = w + static_cast<size_t>(r) * K;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int k = cc * 16 + e;
            const int32_t code = k < K ? clamp_code(row[k] / sc, -128, 127) : 0;
            word[e / 4] |= (static_cast<uint32_t>(code) & 0xFFu) << (8 * (e % 4));
        }
    }
    *reinterpret_cast<uint4*>(out + a8_offset(r, static_cast<size_t>(cc) * 16, Np)) =
        make_uint4(word[0], word[1], word[2], word[3]);
}

// W4 tile layout -> its UINT4 + 8 twin (ref pack_uint4_offset, gemm.cpp:56-75): a
// two's-complement nibble q maps to q + 8 = q ^ 8.
__global__ void w4_offset_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n16) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n16) return;
    uint4 v = in[i];
    v.x ^= 0x88888888u;
    v.y ^= 0x88888888u;
    v.z ^= 0x88888888u;
    v.w ^= 0x88888888u;
    out[i] = v;
}

__device__ __forceinline__ int8_t w4_code_at(const uint8_t* packed, size_t r, size_t k, size_t kblocks) {
    int high;
    const uint8_t byte = packed[w4_offset(r, k, kblocks, &high)];
    return static_cast<int8_t>(static_cast<uint8_t>((high ? byte : byte << 4) & 0xF0)) >> 4;
}

// Dequantize per-group W4 (ref quantize.cpp:134-146): q * S of the element's group.
__global__ void wg_dequant_kernel(const uint8_t* __restrict__ packed, const float* __restrict__ s, int N, int K,
                                  int g, int Kp, float* __restrict__ out) {
    const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<size_t>(N) * K) return;
    const size_t r = i / K, k = i % K;
    out[i] = __fmul_rn(static_cast<float>(w4_code_at(packed, r, k, Kp / kBlockK)), s[r * (K / g) + k / g]);
}

// ODY_ENGINE_W4A16 (ref gemm.cpp:100-121): out[i][j] = sum_k a[i][k] * (q[j][k] * S(j,k)),
// one thread per output in the reference's sequential f32 order (IEEE RN multiply, then
// add: the reference's x86-64 build has no FMA contraction).  Threads of a block share
// the weight row j (one block column per j), tokens i across threads.
__global__ void w4a16_kernel(const float* __restrict__ a, const uint8_t* __restrict__ packed,
                             const float* __restrict__ s, int M, int N, int K, int g, int Kp,
                             float* __restrict__ out) {
    const int j = blockIdx.x;
    const int i = blockIdx.y * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const float* ai = a + static_cast<size_t>(i) * K;
    const size_t kblocks = Kp / kBlockK;
    const int groups = K / g;
    float acc = 0.0f;
    for (int k = 0; k < K; ++k) {
        const float wf = __fmul_rn(static_cast<float>(w4_code_at(packed, j, k, kblocks)),
                                   s[static_cast<size_t>(j) * groups + k / g]);
        acc = __fadd_rn(acc, __fmul_rn(ai[k], wf));
    }
    out[static_cast<size_t>(i) * N + j] = acc;
}

// FINEGRAINED with a group size that is not a multiple of the MMA's 32-k step: both
// operands are re-laid out over K' = groups * g32 (g32 = g rounded up to 32), group gi
// at k' = gi*g32 .. gi*g32+g-1 and zero codes after it, so every group is whole MMA
// steps; the zero lanes add nothing to the group's exact int32 sum.
__global__ void regroup_w4_kernel(const uint8_t* __restrict__ src, int N, int K, int g, int g32, int Kq,
                                  uint8_t* __restrict__ dst) {
    const int Np = static_cast<int>(pad_n(N)), Kqp = static_cast<int>(pad_k(Kq));
    const size_t chunks = Kqp / 32;
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<size_t>(Np) * chunks) return;
    const int r = static_cast<int>(idx / chunks);
    const int cc = static_cast<int>(idx % chunks);
    const size_t kb_src = pad_k(K) / kBlockK;
    uint32_t word[4] = {0u, 0u, 0u, 0u};
    for (int e = 0; e < 32; ++e) {
        const int kq = cc * 32 + e, gi = kq / g32, off = kq - gi * g32;
        if (r >= N || kq >= Kq || off >= g) continue;
        const int32_t code = w4_code_at(src, r, static_cast<size_t>(gi) * g + off, kb_src);
        const int j = e / 8, b = e % 4, hi = (e % 8) >= 4;
        word[j] |= (static_cast<uint32_t>(code) & 0xFu) << (8 * b + 4 * hi);
    }
    int high;
    const size_t o = w4_offset(r, static_cast<size_t>(cc) * 32, Kqp / kBlockK, &high);
    *reinterpret_cast<uint4*>(dst + o) = make_uint4(word[0], word[1], word[2], word[3]);
}
__global__ void regroup_a8_kernel(const int8_t* __restrict__ src, int M, int K, int g, int g32, int Kq,
                                  int8_t* __restrict__ dst) {
    const size_t Mp = pad_m(M), Kqp = pad_k(Kq);
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= Mp * Kqp) return;
    const size_t t = idx / Kqp, kq = idx % Kqp;
    const size_t gi = kq / g32, off = kq - gi * g32;
    int8_t v = 0;
    if (t < static_cast<size_t>(M) && kq < static_cast<size_t>(Kq) && off < static_cast<size_t>(g))
        v = src[a8_offset(t, gi * g + off, Mp)];
    dst[a8_offset(t, kq, Mp)] = v;
}

}  // namespace

cudaError_t launch_regroup(const uint8_t* w4, const int8_t* qa, int M, int N, int K, int g, uint8_t* w4_out,
                           int8_t* qa_out, cudaStream_t st) {
    const int g32 = (g + 31) / 32 * 32, Kq = (K / g) * g32;
    const size_t wt = pad_n(N) * (pad_k(Kq) / 32);
    regroup_w4_kernel<<<static_cast<unsigned>((wt + 255) / 256), 256, 0, st>>>(w4, N, K, g, g32, Kq, w4_out);
    const size_t at = pad_m(M) * pad_k(Kq);
    regroup_a8_kernel<<<static_cast<unsigned>((at + 255) / 256), 256, 0, st>>>(qa, M, K, g, g32, Kq, qa_out);
    return cudaGetLastError();
}

cudaError_t launch_wg_quant_prepack(const float* w, int N, int K, int g, int bits, const float* gamma,
                                    const float* beta, uint8_t* packed, float* s, cudaStream_t st) {
    const int Np = static_cast<int>(pad_n(N)), Kp = static_cast<int>(pad_k(K));
    const int items = N * (K / g);
    wg_scale_kernel<<<(items + 7) / 8, 256, 0, st>>>(w, N, K, g, bits, gamma, beta, s);
    const size_t total = static_cast<size_t>(Np) * (Kp / 32);
    wg_quant_prepack_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(w, N, K, g, Np, Kp, s, packed);
    return cudaGetLastError();
}

cudaError_t launch_w8_quant(const float* w, int N, int K, const float* gamma, const float* beta, int8_t* codes,
                            float* s, int* err, cudaStream_t st) {
    const int Np = static_cast<int>(pad_n(N)), Kp = static_cast<int>(pad_k(K));
    cudaError_t e = launch_w_scale(w, N, K, 8, gamma, beta, s, err, st);
    if (e != cudaSuccess) return e;
    const size_t total = static_cast<size_t>(Np) * (Kp / 16);
    w8_quant_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(w, N, K, Np, Kp, s, codes);
    return cudaGetLastError();
}

cudaError_t launch_w4_offset(const uint8_t* packed, int N, int K, uint8_t* out, cudaStream_t st) {
    const size_t n16 = w4_packed_bytes(N, K) / 16;
    w4_offset_kernel<<<static_cast<unsigned>((n16 + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const uint4*>(packed), reinterpret_cast<uint4*>(out), n16);
    return cudaGetLastError();
}

cudaError_t launch_wg_dequant(const uint8_t* packed, const float* s, int N, int K, int g, float* out,
                              cudaStream_t st) {
    const size_t total = static_cast<size_t>(N) * K;
    wg_dequant_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, st>>>(packed, s, N, K, g,
                                                                                   static_cast<int>(pad_k(K)), out);
    return cudaGetLastError();
}

cudaError_t launch_w4a16(const float* a, const uint8_t* packed, const float* s, int M, int N, int K, int g,
                         float* out, cudaStream_t st) {
    const int tpb = M < 128 ? ((M + 31) / 32) * 32 : 128;
    w4a16_kernel<<<dim3(N, (M + tpb - 1) / tpb), tpb, 0, st>>>(a, packed, s, M, N, K, g,
                                                                static_cast<int>(pad_k(K)), out);
    return cudaGetLastError();
}

int engine_splits(int mode, int M, int N, int K) {
    if (mode == kEngineFine) return 1;
    const int bn = M <= 16 ? 16 : (M <= 32 ? 32 : 64);
    const int tiles = static_cast<int>(pad_n(N) / kTileN) * ((M + bn - 1) / bn);
    const int kblocks = static_cast<int>(pad_k(K) / kBlockK);
    return std::max(1, std::min({8, kblocks, (device_sm_count() + tiles - 1) / tiles}));
}

size_t engine_workspace_bytes(int mode, int M, int N, int K) {
    if (engine_splits(mode, M, N, K) <= 1) return 0;
    return round_up(static_cast<size_t>(M) * N * 4, 256) + 4 * pad_n(N) / kTileN * ((M + 15) / 16);
}

cudaError_t launch_engine_gemm(const EngineArgs& a, cudaStream_t st) {
    if (a.M <= 0 || a.N <= 0 || a.K <= 0) return cudaErrorInvalidValue;
    EParams p = {};
    p.w = a.w;
    p.sw = a.sw;
    p.qa = a.qa;
    p.sa = a.sa;
    p.out = a.out;
    p.M = a.M;
    p.N = a.N;
    p.K = a.K;
    p.Mp = static_cast<int>(pad_m(a.M));
    p.Np = static_cast<int>(pad_n(a.N));
    p.kblocks = static_cast<int>(pad_k(a.K) / kBlockK);
    p.g = a.mode == kEngineFine ? a.group : a.K;
    if (a.mode == kEngineFine && (p.g <= 0 || p.g % 32 != 0 || a.K % p.g != 0)) return cudaErrorInvalidValue;
    p.groups = a.K / p.g;
    // BN <= 64 (the epilogue holds BN accumulators per thread; FINE also BN partial sums)
    const int bn = a.M <= 16 ? 16 : (a.M <= 32 || a.mode == kEngineFine ? 32 : 64);
    const int n_tiles = p.Np / kTileN, m_tiles = (a.M + bn - 1) / bn;
    p.splits = engine_splits(a.mode, a.M, a.N, a.K);
    if (p.splits > 1) {
        if (!a.workspace || a.workspace_bytes < engine_workspace_bytes(a.mode, a.M, a.N, a.K))
            return cudaErrorInvalidValue;
        p.ws = static_cast<int32_t*>(a.workspace);
        p.cnt = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(a.workspace) +
                                            round_up(static_cast<size_t>(a.M) * a.N * 4, 256));
    }
    switch (a.mode) {
        case kEngineFast: return launch_engine_bn<kEngineFast>(p, bn, n_tiles, m_tiles, st);
        case kEngineAsym: return launch_engine_bn<kEngineAsym>(p, bn, n_tiles, m_tiles, st);
        case kEngineW8A8: return launch_engine_bn<kEngineW8A8>(p, bn, n_tiles, m_tiles, st);
        case kEngineFine: return launch_engine_bn<kEngineFine>(p, bn, n_tiles, m_tiles, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace odyb200
