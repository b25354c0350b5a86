// quant_common.cuh -- device helpers shared by K1 (act quant) and the fused K1+K3 GEMM.
// Bit-exactness contract with the reference (ref quantize.cpp:12-47,113-132).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

namespace odyb200 {

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// ref quantize.cpp:12-18
__device__ __forceinline__ int32_t clamp_code(float x, int32_t lo, int32_t hi) {
    float r = roundf(x);
    if (r < static_cast<float>(lo)) return lo;
    if (r > static_cast<float>(hi)) return hi;
    return static_cast<int32_t>(r);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Load 16 consecutive row elements starting at k0 (zero beyond K).
template <typename T>
__device__ __forceinline__ void load16(const T* __restrict__ row, int k0, int K, float (&v)[16]) {
    if (k0 + 16 <= K && (reinterpret_cast<uintptr_t>(row + k0) & 15) == 0) {
        constexpr int kPer = 16 / sizeof(T);
#pragma unroll
        for (int i = 0; i < 16; i += kPer) {
            uint4 raw = __ldg(reinterpret_cast<const uint4*>(row + k0 + i));
            const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
            for (int j = 0; j < kPer; ++j) v[i + j] = to_f32(e[j]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = (k0 + i < K) ? to_f32(row[k0 + i]) : 0.0f;
    }
}

// Exact fast path for clamp(roundf(fl(x / S))): with r = RN(1/S), q' = RN(x * r) is
// within |x/S| * 1.8e-7 <= 2.3e-5 of fl(x/S) (|x/S| <= 127.0001 since S = max|x|/127).
// roundf(q') can only differ from roundf(fl(x/S)) when a half-integer lies within that
// distance, so those rare elements (and a non-finite r) take the IEEE division.
__device__ __forceinline__ int32_t quant_code_i8(float x, float scale, float rcp, bool exact) {
    const float qa = __fmul_rn(x, rcp);
    const float a = fabsf(qa);
    const float f = a - truncf(a);
    if (exact || fabsf(f - 0.5f) < 6.0e-5f) return clamp_code(x / scale, -128, 127);
    return clamp_code(qa, -128, 127);
}

// Same contract, branch-free for the common case: q' + 1.5*2^23 rounds q' to the
// nearest integer (ties-to-even) and leaves it, two's complement, in the low mantissa
// byte; d = q' - round(q') flags the near-half-integer (and non-finite) cases, which
// the caller redoes through quant_code_i8's IEEE division.  |q'| <= 127.0001 (every
// |x| <= max|x| = 127*S), so no clamp is needed on the fast path.
__device__ __forceinline__ uint32_t quant_byte_fast(float x, float rcp, bool& redo) {
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
    const float qa = __fmul_rn(x, rcp);
    const float t = __fadd_rn(qa, kMagic);
    const float d = __fsub_rn(qa, __fsub_rn(t, kMagic));
    redo |= !(fabsf(d) <= 0.49994f);  // also true for NaN
    return __float_as_uint(t);         // low byte = code
}
// Four codes (low bytes of a..d) -> one word, byte 0 = a.
__device__ __forceinline__ uint32_t pack4_low_bytes(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

}  // namespace odyb200
