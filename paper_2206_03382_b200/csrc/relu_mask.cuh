// Layout of the ReLU mask [h > 0]: one 64-bit word per (capacity row, 64-column block),
// written by the up-GEMM epilogue, patched by the fp64 fix-up, read by the dgrad x mask epilogue.
//
// Words are interleaved by 32-row groups, [rows / 32][V / 64][32]: the epilogues map one row to
// each lane, so a warp's 32 words of one column block are 256 contiguous bytes (one coalesced
// store / load instead of 32 scattered sectors). Allocation: relu_mask_words(rows, V / 64).
//
// The order inside each 32-column half is chosen for the two epilogues' instruction counts, not
// for readability: column pair p (columns 2p, 2p + 1 of the half) has its even column at bit
// (p & 7) + 16 * (p >> 3) and its odd column 8 bits above. The consumer then turns one shifted
// copy of the half into the bf16-pair masks of pairs p and p + 8 with two byte permutes (sign
// replication of bytes 0 / 1 and 2 / 3), and the producer gathers the 32 sign bits of a half in
// this order with one funnel shift per column.
#pragma once

#include <cstdint>

namespace moe {

// word of (global capacity row, 64-column block) with nblk blocks per row
__host__ __device__ __forceinline__ size_t relu_mask_word(size_t row, uint32_t blk, uint32_t nblk) {
  return ((row >> 5) * nblk + blk) * 32 + (row & 31);
}

// bit index (0..63) of column c (0..63) of a 64-column block
__host__ __device__ constexpr uint32_t relu_mask_bit(uint32_t c) {
  return 32u * (c >> 5) + (((c & 31u) >> 1) & 7u) + 8u * (c & 1u) + 16u * ((c & 31u) >> 4);
}

// inverse within a 32-column half: the column stored at bit b (0..31)
__host__ __device__ constexpr uint32_t relu_mask_col(uint32_t b) {
  return 2u * ((b & 7u) + 8u * (b >> 4)) + ((b >> 3) & 1u);
}

static_assert(relu_mask_bit(0) == 0 && relu_mask_bit(1) == 8 && relu_mask_bit(16) == 16 &&
                  relu_mask_bit(17) == 24 && relu_mask_bit(31) == 31 && relu_mask_bit(32) == 32,
              "mask layout");
static_assert(relu_mask_col(relu_mask_bit(13)) == 13 && relu_mask_col(relu_mask_bit(30)) == 30 &&
                  relu_mask_col(relu_mask_bit(7)) == 7 && relu_mask_col(relu_mask_bit(22)) == 22,
              "mask layout inverse");

// the 32 masks of a 64-column block's bf16 pairs: pair j (columns 2j, 2j + 1) -> 0x0000ffff per
// set even bit | 0xffff0000 per set odd bit
__device__ __forceinline__ void relu_mask_pairs(unsigned long long mk, uint32_t (&m)[32]) {
#pragma unroll
  for (uint32_t h = 0; h < 2; ++h) {
    const uint32_t x = static_cast<uint32_t>(mk >> (32 * h));
#pragma unroll
    for (uint32_t p = 0; p < 8; ++p) {
      const uint32_t y = x << (7 - p);  // bits p, p+8, p+16, p+24 -> the four byte sign bits
      uint32_t a, b;
      asm("prmt.b32 %0, %1, 0, 0x9988;" : "=r"(a) : "r"(y));
      asm("prmt.b32 %0, %1, 0, 0xBBAA;" : "=r"(b) : "r"(y));
      m[16 * h + p] = a;
      m[16 * h + p + 8] = b;
    }
  }
}

}  // namespace moe
