// Internal launch interfaces of the non-GEMM kernels (gating, dispatch, rng).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "peer_flags.h"

#include <cstdint>

namespace moe {

// Launch-error bookkeeping: cudaGetLastError() clears the error, so launch helpers record it
// here for the caller's message (returns 0 on success, -2 on failure).
cudaError_t& last_launch_error();

// One-time per-(kernel, device) opt-in to > 48 KiB dynamic shared memory: function attributes
// are per device, so a process driving several GPUs sets them once on each.
bool smem_optin_raw(const void* kern, int bytes);
template <typename F>
inline bool smem_optin(F* kern, int bytes) {
  return smem_optin_raw(reinterpret_cast<const void*>(kern), bytes);
}
inline int launch_status() {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return 0;
  last_launch_error() = e;
  return -2;
}

struct GatingArgs {
  const void* x;       // [blocks*T, M] bf16 or f32
  int x_is_f32;
  const double* wg;    // [M, E] fp64
  int blocks, T, M, E, k;
  int cap_kind;        // 0 fixed, 1 auto, 2 bounded
  int cap_formula;     // expert_capacity(k, f, T, E) (fixed) or at max_factor (bounded)
  int bpr;
  // RouterKind::Cosine (moe_layer.hpp:10, gating.cpp:37-56); router == 0: linear (wg)
  int router;
  const double* cos_proj;  // [M][D]
  const double* cos_ct;    // [D][E]: the expert embeddings transposed
  const double* cos_en;    // [E]: |C_e|
  double cos_tau;          // max(temperature, 0.01)
  int cos_dim;             // D
  double* cos_buf;         // [blocks*T][D] fp64 scratch: x . P
  int32_t* err;            // set to 1 on a zero-norm projected token
  // Certified tensor-core gate (gate_tc.cu; linear router, bf16 x): set -> used when the shape
  // allows it and no probs are requested; null -> the fp64 DMMA gate
  const void* wg_pieces = nullptr;    // [2][E][M] bf16 hi / lo split of wg
  const float* wg_norm_max = nullptr; // max_e |wg[:, e]|_2
  int32_t* gate_fixups = nullptr;     // += tokens re-decided in fp64
  int32_t* gate_flags = nullptr;      // [blocks*T] scratch: uncertified tokens
  int32_t* gate_flag_count = nullptr; // [2], zero at rest (the fixup kernel resets it)
};

bool gate_tc_supported(int M, int E, int k);
int gate_tc_prepare_device(const double* wg, int M, int E, void* pieces, float* wn_max,
                           cudaStream_t st);
int gate_tc_device(const void* x, const void* pieces, const double* wg, const float* wn_max,
                   int blocks, int T, int M, int E, int k, int32_t* idxs, double* gates,
                   int32_t* hist, int32_t* fixups, int32_t* flag_list, int32_t* flag_count,
                   cudaStream_t st);

// Cosine router weights: ct = C^T, en[e] = |C_e|; err = 2 if an expert row has zero norm.
int cosine_prep_device(const double* ce, int E, int D, double* ct, double* en, int32_t* err,
                       cudaStream_t st);

struct GatingBuffers {
  int32_t* idxs;        // [blocks*T, k]
  double* gates;        // [blocks*T, k]
  int32_t* locations;   // [blocks*T, k]
  int32_t* hist;        // [blocks*cta_per_block, E]
  int32_t* offs;        // [blocks*cta_per_block, E]
  int32_t* demand;      // [blocks, E]
  int32_t* list_base;   // [blocks, E]
  int32_t* fill;        // [blocks, E]
  int32_t* list;        // [blocks*T*k]
  int32_t* cap;         // [1] resolved capacity
  int32_t* drops;       // [1]
  int32_t* slot_token;  // [blocks, E, cap]
  float* slot_gate;     // [blocks, E, cap]
  double* probs;        // optional [blocks*T, E]
  // resolve_capacity in the capacity scan's last CTA: a zeroed counter (reset by that CTA);
  // null: a separate finalize kernel
  int32_t* scan_done = nullptr;
  // BPR chunked ranking scratch ([blocks*T*k] each); null: the one-CTA-per-list sort
  unsigned long long* bpr_keys = nullptr;
  int32_t* bpr_pos = nullptr;
};

int gate_cta_per_block(int T);
// Router GEMM + softmax + top-k + histogram + capacity resolution (device scalar g.cap).
int run_gating_device(const GatingArgs& a, const GatingBuffers& g, cudaStream_t st);
// Capacity from a (global, all-reduced) per-expert demand vector.
int resolve_capacity_device(const int32_t* demand, int E, int cap_kind, int cap_formula,
                            int32_t* cap_out, cudaStream_t st);
// Location assignment (FIFO or BPR) + slot tables. cap_bound >= resolved capacity.
int run_assign_device(const GatingArgs& a, const GatingBuffers& g, int cap_bound, cudaStream_t st);

// Capacity-slot geometry of one source block: degree d chunks of cc slots (cap <= d*cc).
// Row of slot (b, e, c) in a [blocks][d][E][cc][M] buffer:
//   b*d*E*cc + ((c / cc) * E + e) * cc + c % cc
struct SlotGeom {
  int blocks, T, E, M, k, cap, cc, degree;
};

// Optional side task of the slot-major gathers: zero the [T][row_bytes] rows of tokens whose k
// assignments were all dropped (the fused decode / encode-backward path never writes them).
struct DropZero {
  const int32_t* locations = nullptr;  // [T][k]
  int T = 0, k = 0;
  void* out = nullptr;                 // [T] rows of row_bytes (multiple of 16)
  size_t row_bytes = 0;
};

// W > 1 peer backend: this rank's own experts' rows go straight into its receive buffer
// ([chunk][W][dE][cc] layout, source = rank) instead of the send buffer -- the local block of
// the all-to-all is never copied.
struct LocalDest {
  void* recv = nullptr;
  int W = 1, rank = 0, dE = 0;
  float* recv_norm = nullptr;  // encode: the own rows' norms go here (receive-row index)
  // Fused dispatch (all_peers): EVERY expert's rows are stored straight into its owner's
  // receive buffer over NVLink -- peer_recv[p] / peer_norm[p] are rank p's receive buffer / norm
  // array mapped into this process (p == rank: the local ones) -- after polling `freed` (every
  // peer released its buffer). No send buffer, no copy-engine push: the stream publishes the
  // ready flags after the kernel (which fences its stores system-wide).
  bool all_peers = false;
  void* peer_recv[8] = {};
  float* peer_norm[8] = {};
  FlagWait freed;
};

// dtype: 0 = bf16, 1 = f32 (x, z, y share the layer dtype). rownorm (optional, [z rows]):
// |z[row]|_2 (rounded up) for the ReLU-mask certificate.
// reset (optional): a counter zeroed by the pass (the ReLU-fixup count; no memset node).
int encode_device(const SlotGeom& g, int dtype, const void* x, const int32_t* slot_token, void* z,
                  cudaStream_t st, float* rownorm = nullptr, const DropZero& dzero = DropZero{},
                  unsigned int* reset = nullptr, const LocalDest& local = LocalDest{});
// wait (optional): peers' ready flags polled by the kernel before it reads z (fused receive wait)
int decode_device(const SlotGeom& g, int dtype, const void* z, const int32_t* idxs,
                  const int32_t* locations, const double* gates, void* y, cudaStream_t st,
                  const FlagWait* wait = nullptr);
int decode_backward_device(const SlotGeom& g, int dtype, const void* dy,
                           const int32_t* slot_token, const float* slot_gate, void* dz,
                           cudaStream_t st, const DropZero& dzero = DropZero{},
                           const LocalDest& local = LocalDest{});
// k = 1 combine, slot-major (layer path): out[token of slot] = (slot_gate ? g : 1) * src[slot row]
// for every kept slot of the [blocks][degree][E][cc] rows; dropped tokens' rows zeroed (dzero).
int slot_scatter_device(const SlotGeom& g, int dtype, const void* src, const int32_t* slot_token,
                        const float* slot_gate, void* out, const DropZero& dzero, cudaStream_t st,
                        const FlagWait* wait = nullptr);
// Optional d_gates[t, j] = <Z[e, loc], dy[t]> (dispatch.cpp:143-156); 0 for dropped.
int decode_backward_gates_device(const SlotGeom& g, int dtype, const void* z, const void* dy,
                                 const int32_t* idxs, const int32_t* locations, double* dgates,
                                 cudaStream_t st);
int encode_backward_device(const SlotGeom& g, int dtype, const void* dz, const int32_t* idxs,
                           const int32_t* locations, void* dx, cudaStream_t st,
                           const FlagWait* wait = nullptr);
// Sharded P2 combine: out[b] = sum over q < s of part[b][q] (blocks of blk elements, dtype 0 bf16
// / 1 f32, fp32 accumulate in q order).
int shard_sum_device(const void* part, void* out, int64_t nblk, int s, int64_t blk, int dtype,
                     cudaStream_t st);

int build_slots_device(int blocks, int T, int k, int E, int cap, const int32_t* idxs,
                       const int32_t* locations, const double* gates, int32_t* slot_token,
                       float* slot_gate, cudaStream_t st);

// splitmix64 counter stream (core.cpp:66-83): value n (0-based) = lo + (hi-lo) * u(seed, n+1).
int fill_uniform_device(void* dst, int dtype /*0 bf16, 1 f32, 2 f64*/, int64_t n, uint64_t seed,
                        uint64_t offset, double lo, double hi, cudaStream_t st);
// Same stream, strided gather: dst[i*cols + j] = draw(offset + i*src_stride + j) for a sub-block.
int fill_uniform_2d_device(void* dst, int dtype, int64_t rows, int64_t cols, int64_t src_stride,
                           uint64_t seed, uint64_t offset, double lo, double hi, cudaStream_t st);

// ReLU-mask certificate support (relu_fix.cu).
int weight_stats_device(const void* w1, int G, int M, int V, float* colnorm, float* colnorm_blk,
                        void* w1t, cudaStream_t st);
int relu_mask_from_act_device(const void* act, int64_t rows, int V, unsigned long long* mask,
                              cudaStream_t st);
// wait: optional fused receive wait (peer flags, see peer_flags.cuh); reset: optional counter
// zeroed by the kernel (the ReLU fixup count)
// Rows [row0, row0 + nrows) of segments [seg_begin, seg_begin + nsegs) (seg_rows apart), the
// segments [skip_begin, skip_begin + skip_count) skipped over (nsegs counts processed segments).
struct RowSet {
  int64_t seg_begin = 0, nsegs = 0, seg_rows = 1, row0 = 0, nrows = 0;
  int64_t skip_begin = 0, skip_count = 0;
};
int rownorm_device(const void* x, int M, float* rownorm, const RowSet& rs, cudaStream_t st,
                   const FlagWait* wait = nullptr, unsigned int* reset = nullptr);
int wait_flags_device(const FlagWait& w, cudaStream_t st);
int relu_fixup_device(const void* x, const void* w1t, int G, int seg_rows, int M, int V,
                      const unsigned long long* list, const unsigned int* count, unsigned int cap,
                      void* act, unsigned long long* relu_mask, cudaStream_t st);

// fp32 SIMT GEMM path (the 1e-5 fp32 layer): same kinds/addressing as the bf16 tcgen05 GEMM.
struct GemmArgs;
int gemm_f32(int kind, const float* A, const float* B, float* D, const GemmArgs& args,
             cudaStream_t st);
int gemm_bf16_simt(int kind, const void* A, const void* B, void* D, const GemmArgs& args,
                   cudaStream_t st);

}  // namespace moe
