// Grouped expert GEMM (tcgen05/TMEM/TMA, sm_100a). See gemm_sm100.cu.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "peer_flags.h"

namespace moe {

enum GemmKind : int {
  kGemmUp = 0,         // act[g,(s,r),:V] = relu(X[g,(s,r),:M] . W1[g])          (bf16 out)
  kGemmDown = 1,       // Y[g,(s,r),:M]   = act . W2[g]                          (bf16 out)
  kGemmDgradMask = 2,  // dh = (dY . W2[g]^T) * [act > 0]                       (bf16 out)
  kGemmDgrad = 3,      // dX = dh . W1[g]^T                                     (bf16 out)
  kGemmWgrad = 4,      // dW[g] = A[g]^T . B[g], reduction over all token rows  (fp32 out)
};

enum EpiKind : int { kEpiBf16 = 0, kEpiReluBf16 = 1, kEpiMaskBf16 = 2, kEpiF32 = 3 };

// Token-indexed output (single-rank fused decode / encode-backward; GemmArgs::idx_mode bits). A
// slot row (segment s, row r) maps to token row_token[s * seg_rows + r] (< 0: empty slot).
enum IdxMode : uint32_t {
  kIdxScatterD = 4,  // row-M: D rows are written to token rows of D:[gather_rows][N]
  kIdxScaleRow = 8,  // row-M: output row scaled by row_scale[slot] (the slot's gate)
  // row-M, expert-parallel combine fused into the epilogue: segment (chunk, src, g) of the
  // receive layout is stored straight into rank src's combine buffer (peer memory over NVLink),
  // at its [chunk][E][cap chunk][N] position (collectives.cpp:116-162 combine, reversed plan).
  kIdxPeerD = 16,
};
constexpr int kMaxPeers = 8;

struct GemmArgs {
  uint32_t G;         // groups (local experts)
  uint32_t S;         // capacity segments per group (pipeline chunks x source ranks)
  uint32_t seg_rows;  // token rows per segment (capacity chunk cc)
  uint32_t seg_base;  // first segment of this launch inside the segment buffer
  uint32_t N;         // output columns
  uint32_t K;         // reduction length (row-M kinds)
  uint32_t Mo;        // output rows (wgrad)
  const void* aux;    // SIMT kGemmDgradMask: saved activation, same layout as D
  // ReLU bitmask [nseg * seg_rows][N / 64] (bit i of word w <-> column 64 w + i): written by the
  // tcgen05 kGemmUp epilogue (if non-null), read by the tcgen05 kGemmDgradMask epilogue.
  unsigned long long* relu_mask;
  void* d_ptr;        // set by gemm_fwd: output base
  // kGemmUp ReLU-mask certificate (optional): outputs with |h| < tau = 2^-18 * rownorm[row] *
  // colnorm[g][col] are appended to fix_list for an fp64 sign re-decision (relu_fixup).
  const float* rownorm;            // [nseg * seg_rows] |X[row, :]|_2 (rounded up)
  const float* colnorm;            // [G][N] |W1[g][:, col]|_2 (rounded up)
  const float* colnorm_blk;        // [G][N / 64] max of colnorm over each 64-column block
  unsigned long long* fix_list;   // packed (seg << 44) | (row << 24) | col
  unsigned int* fix_count;
  unsigned int fix_cap;
  // token-indexed output (IdxMode)
  uint32_t idx_mode;
  uint32_t gather_rows;       // token rows of the scattered tensor
  const int32_t* row_token;   // [nseg * seg_rows]
  const float* row_scale;     // [nseg * seg_rows]
  // row-M sub-range (pipelined first chunk): rows [row0, row0 + nrows) of every segment (nrows = 0:
  // all; row0 and nrows multiples of the tile height unless the range ends at seg_rows), and one
  // segment index of [0, S] skipped (skip_seg < 0: none; S then counts the segments processed)
  uint32_t row0 = 0, nrows = 0;
  int32_t skip_seg = -1;
  // W > 1: peers' ready (or freed) flags the kernel polls before its first load -- the receive
  // wait fused into the GEMM (wait.base == nullptr: none). Row norms (certificate) written by the
  // peers before the flags are then read coherently.
  FlagWait wait;
  // kIdxPeerD: destination combine buffer of every rank (this rank's own for src == rank)
  uint32_t peer_world, peer_rank, peer_out_segs;  // out_segs = chunks * E
  void* peer_d[kMaxPeers];
  // Kernel span (measurement): [0] = min over CTAs of %globaltimer once the kernel may start
  // work (after the programmatic-dependent-launch wait), [1] = max at CTA exit; [2] / [3] = CTA
  // 0's clock64 cycles / nanoseconds over its lifetime (the effective SM clock). Null: off.
  unsigned long long* span = nullptr;
};

// Pack / unpack of one ReLU-fixup entry.
__host__ __device__ inline unsigned long long fix_pack(uint32_t seg, uint32_t row, uint32_t col) {
  return (static_cast<unsigned long long>(seg) << 44) | (static_cast<unsigned long long>(row) << 24) |
         col;
}
constexpr float kReluTauScale = 1.0f / 262144.0f;  // 2^-18

// 64-bit words of a ReLU mask over `rows` capacity rows with nblk = ceil(V / 64) column blocks
// per row (32-row interleaved layout, relu_mask.cuh; the fix-up indexes with the same nblk, so a
// partial last block -- SIMT shapes, whose dgrad reads the activation instead -- stays in bounds)
inline size_t relu_mask_words(size_t rows, size_t nblk) { return (rows + 31) / 32 * 32 * nblk; }

int gemm_validate(const GemmArgs& a, int kind);

int gemm_fwd(GemmKind kind, const void* A, const void* B, void* D, const GemmArgs& args,
             int nseg_total, int num_sms, cudaStream_t stream);

// 3-D tensor map, box {b0, b1, 1}, 128-byte swizzle (0 on success).
int tensor_map_3d(CUtensorMap* m, const void* base, bool f32, uint64_t d0, uint64_t d1, uint64_t d2,
                  uint32_t b0, uint32_t b1);

}  // namespace moe
