// layout.h -- HBM layouts of the two quantized operands (host + device).
//
// Prepacked INT4 weights ("w4 tile layout"), for an N x K per-channel W4 matrix:
//   rows padded to Np = ceil(N/128)*128, k padded to Kp = ceil(K/128)*128 (zero codes);
//   one 8 KiB block per (n_tile, k_block) of 128 rows x 128 k, blocks in
//   n_tile-major order, so one 1-D bulk copy moves one pipeline stage;
//   inside a block: 4 chunks (32 k each) x 128 rows x 16 bytes;
//   inside a 16-byte row chunk, word j (k = 8j..8j+7) holds in byte b the code of
//   k = 8j+b in its LOW nibble and k = 8j+4+b in its HIGH nibble, so
//       (w << 4) & 0xF0F0F0F0  ->  4 int8 lanes  k = 8j..8j+3    (value * 16)
//        w       & 0xF0F0F0F0  ->  4 int8 lanes  k = 8j+4..8j+7  (value * 16)
//   -- the paper's SINT4 -> S8 "high nibble" widening (ref gemm.cpp:49-54) with
//   the nibble order permuted so each result word is 4 consecutive K lanes.
//
// Quantized activations ("a8 k-block layout"), for an M x K per-token INT8 matrix:
//   rows padded to Mp = ceil(M/128)*128, k padded to Kp (zero codes);
//   k-block major: block kb holds all Mp rows x 128 bytes, row-contiguous, with the
//   16-byte chunk index XOR-swizzled by (row % 8) -- the tcgen05 SWIZZLE_128B
//   K-major canonical layout.  Any run of 8-aligned rows of one k-block is one
//   contiguous, 1024-byte-aligned span, copied by a single 1-D bulk copy.
#pragma once
#include <cstddef>
#include <cstdint>

#ifdef __CUDACC__
#define ODY_HD __host__ __device__ __forceinline__
#else
#define ODY_HD inline
#endif

namespace odyb200 {

constexpr int kTileN = 128;         // weight rows per tile (MMA M)
constexpr int kBlockK = 128;        // k per pipeline unit
constexpr int kWBlockBytes = kTileN * kBlockK / 2;  // 8192
constexpr int kRowPadM = 128;       // activation row padding
constexpr float kMinScale = 0x1.0p-24f;  // ref tensor.hpp:14
constexpr std::size_t kMaxK = std::size_t{1} << 17;  // ref gemm.cpp:14

ODY_HD std::size_t round_up(std::size_t x, std::size_t m) { return (x + m - 1) / m * m; }
ODY_HD std::size_t pad_k(std::size_t k) { return round_up(k, kBlockK); }
ODY_HD std::size_t pad_n(std::size_t n) { return round_up(n, kTileN); }
ODY_HD std::size_t pad_m(std::size_t m) { return round_up(m, kRowPadM); }

ODY_HD std::size_t w4_packed_bytes(std::size_t n, std::size_t k) { return pad_n(n) * pad_k(k) / 2; }
ODY_HD std::size_t a8_bytes(std::size_t m, std::size_t k) { return pad_m(m) * pad_k(k); }

// Byte offset and nibble (0 low, 1 high) of weight code (r, k).
ODY_HD std::size_t w4_offset(std::size_t r, std::size_t k, std::size_t kblocks, int* high) {
    std::size_t nt = r / kTileN, rr = r % kTileN;
    std::size_t kb = k / kBlockK, kk = k % kBlockK;
    std::size_t c = kk / 32, e = kk % 32, j = e / 8, p = e % 8;
    *high = p >= 4 ? 1 : 0;
    std::size_t b = p & 3;
    return ((nt * kblocks + kb) * 4 + c) * 2048 + rr * 16 + j * 4 + b;
}

// Byte offset of activation code (t, k).
ODY_HD std::size_t a8_offset(std::size_t t, std::size_t k, std::size_t mp) {
    std::size_t kb = k / kBlockK, kk = k % kBlockK;
    std::size_t chunk = kk / 16, byte = kk % 16;
    return kb * mp * 128 + t * 128 + (((chunk ^ (t & 7)) & 7) * 16) + byte;
}

}  // namespace odyb200
