// Internal C++ layer object behind the C ABI (include/moe_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "moe_b200.h"
#include "gemm_sm100.h"
#include "kernels.h"
#include "peer_a2a.h"
#include "strategy.h"

namespace moe {

struct MoeError : std::runtime_error {
  int code;
  MoeError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct DevMem {
  void* p = nullptr;
  size_t bytes = 0;
  DevMem() = default;
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  ~DevMem();
  void alloc(size_t n);
};

uint16_t bf16_bits_rne(double x);

// Flexible all-to-all plan for pipeline chunk `chunk` (flex_all2all, collectives.cpp:116-162):
// element offsets of the block sent to / received from each peer p and the block size.
// phase 0 (dispatch): send [chunk][E][cc][M] experts [p*dE,(p+1)*dE) -> recv [chunk][W][dE][cc][M]
// phase 1 (combine):  the inverse.
void a2a_plan(int64_t W, int64_t E, int64_t cc, int64_t M, int64_t chunk, int phase,
              int64_t* send_off, int64_t* recv_off, int64_t* elems);
int64_t expert_capacity(int64_t k, double f, int64_t tokens, int64_t experts);
void validate(const moe_config& c);
// select_parallelism (parallelism.cpp:288-308): MOE_PARALLEL_P1 iff comm_cost_p1 <= comm_cost_p2.
int32_t select_parallelism(double local_experts, int64_t gathered_capacity, int64_t model_dim,
                           double param_bytes, int64_t n_sharded);

// Phases timed with CUDA events on the compute stream when profiling is on (Timeline tracing,
// pipeline.hpp:36-46 / pipeline.cpp:68-76, with measured instead of simulated intervals).
enum Phase : int {
  kPhGate = 0, kPhEncode, kPhUp, kPhDown, kPhDecode, kPhDecodeBwd, kPhDgradMask, kPhDgrad,
  kPhWgrad1, kPhWgrad2, kPhEncodeBwd, kPhA2aFwd, kPhA2aBwd, kPhAssign, kPhReluFix,
  kPhXferDispatch, kPhXferCombine, kPhWeightStats, kNumPhases
};

class Layer {
 public:
  Layer(const moe_config& cfg, int rank, const uint8_t* nccl_id, int device);
  ~Layer();

  void init_params(uint64_t seed);
  void set_router(const double* wg);
  void set_cosine_router(const double* proj, const double* experts, double temperature);
  void set_capacity_factor(double f);
  void set_expert(int64_t le, const double* w1, const double* w2);
  void set_expert_slices(const double* w1s, const double* w2s);
  void forward(const void* x, void* y, cudaStream_t st);
  void backward(const void* dy, void* dx, float* dw1, float* dw2, cudaStream_t st);
  void forward_host(const void* xh, void* yh, cudaStream_t st);
  void backward_host(const void* dyh, void* dxh, cudaStream_t st);
  // Pipelined host-buffer calls: return after enqueueing; the input upload (H2D stream) and the
  // result download (D2H stream) overlap the neighbouring steps' compute through double-buffered
  // device staging. Host buffers must stay untouched / unread until host_sync().
  void forward_host_async(const void* xh, void* yh, cudaStream_t st);
  void backward_host_async(const void* dyh, void* dxh, cudaStream_t st);
  void host_sync();
  void get_routing(int32_t* idxs, int32_t* locs, double* gates, int64_t* capacity);
  void get_metrics(moe_step_metrics* m);
  void get_grads(float* dw1, float* dw2);
  void grad_slices(float* w1s, float* w2s, cudaStream_t st);
  void* w1() { return w1_.p; }
  void* w2() { return w2_.p; }
  // resident weights changed in place: rebuild the derived state (W1^T, column norms, W1 slice)
  void weights_updated() { stats_dirty_ = true; }
  // Kernel spans of the tcgen05 expert GEMMs (device %globaltimer; no events, so programmatic
  // dependent launch stays intact): per phase, the summed span in ms and the launch count.
  void set_kernel_spans(bool on);
  void take_kernel_spans(double* ms, int64_t* counts, int n);
  double span_mhz() const { return span_mhz_; }
  int64_t launches() const { return launches_; }
  void set_profiling(bool on) { prof_ = on; }
  // Sums (ms) and counts per phase since the last call; synchronizes.
  void take_profile(double* ms, int64_t* counts, int n);

  std::string err;

 private:
  uint64_t expert_draw_offset(int64_t e) const;
  void upload_weights(void* dst, const double* src, size_t n);
  bool tc_ok(int kind, const GemmArgs& a) const;
  void gemm(int kind, const void* A, const void* B, void* D, const GemmArgs& a, int nseg,
            cudaStream_t st);
  GatingArgs gating_args(const void* x) const;
  GatingBuffers gating_buffers();
  SlotGeom geom() const;
  void exchange(const void* send, void* recv, int chunk, int phase);
  void exchange_2dh(const char* send, char* recv, size_t block_bytes, ncclDataType_t dt, int64_t elems);
  DevMem a2a_tmp_;  // 2DH staging (two W-block buffers)
  void peer_push(int ch, const void* src, int chunk, int phase, uint32_t epoch, cudaEvent_t local_done);
  void peer_push_rows(int ch, const void* src, int chunk, int phase, int slot, uint32_t row0,
                      uint32_t nrows, uint32_t epoch);
  double allreduce_max_host(double v);
  void sync_comm(cudaStream_t s, const char* what);  // polls NCCL async errors, times out
  void check_comm(const char* what);                 // throws MOE_ECOMM on an NCCL async error
  // Sharded placement (W = E*s, moe_layer.cpp:17-108): grouped NCCL exchanges of chunk `chunk`,
  // dir 0 = dispatch (z order -> [chunk][nsrc][cc] receive order), dir 1 = combine (inverse; P2
  // lands the s partials in [chunk][E][s][cc] order for shard_sum).
  void shard_exchange(const void* send, void* recv, int chunk, int dir, bool p2);
  void sharded_forward(GemmArgs up, GemmArgs down, bool cert, cudaStream_t st);
  void sharded_backward(GemmArgs dgm, GemmArgs dg, GemmArgs wg1, GemmArgs wg2, float* gw1,
                        float* gw2, cudaStream_t st);
  void refresh_slices(cudaStream_t st);
  void ensure_io();
  void alloc_capacity(int cap);
  void prof_mark(int phase, bool begin, cudaStream_t st);
  // MOE_TIMELINE=1 (debug): event timeline of one forward + backward, printed after backward.
  void tl_mark(const std::string& name, cudaStream_t st);
  void tl_flush();
  bool tl_on_ = false;
  std::vector<std::pair<std::string, cudaEvent_t>> tl_;

  moe_config cfg_;
  int rank_, device_;
  int W_, E_, dE_, M_, V_, T_, k_, esz_;
  // sharded placement: s_ ranks per expert; this rank computes expert rank/s_ and holds slice
  // rank%s_ (h = V/s_ hidden columns); parallel_ is the last forward's ParallelChoice
  bool sharded_ = false;
  int s_ = 1;
  int parallel_ = MOE_PARALLEL_P1;
  ncclComm_t group_comm_ = nullptr;  // the s_ ranks sharing this rank's expert
  DevMem w1s_, ypart_, dws1_, dws2_;  // P2: W1 slice (M, h), partial outputs, slice grads
  int cap_, cap_alloc_ = 0, cap_formula_ = 0;
  int32_t* cap_host_ = nullptr;
  int degree_ = 1, cc_ = 1;
  int num_sms_ = 148;
  double f_ = 1.0;
  Strategy strategy_;
  StrategySearch search_;
  // (f, strategy) -> executions so far and the fastest timed one (the first is not timed)
  std::map<std::pair<double, int>, std::pair<int, double>> trials_;
  bool fwd_done_ = false, metrics_valid_ = false;
  int64_t launches_ = 0, bwd_launches_ = 0;
  double comm_bytes_ = 0.0;
  float* last_dw1_ = nullptr;
  float* last_dw2_ = nullptr;

  cudaStream_t comm_stream_ = nullptr;
  ncclComm_t comm_ = nullptr;
  cudaEvent_t ev_fwd_start_{}, ev_fwd_end_{}, ev_sync_{}, ev_comm_done_{};
  cudaEvent_t ev_a_[8]{}, ev_b_[8]{}, ev_c_[8]{};
  cudaEvent_t ev_freed_[PeerExchange::kChannels]{};
  std::unique_ptr<PeerExchange> peer_;
  uint32_t epoch_[PeerExchange::kChannels] = {0, 0, 0, 0};
  bool bwd_pending_ = false;  // last forward's receive buffer still held for a backward

  DevMem wg_, w1_, w2_, dw1_, dw2_;
  // certified tensor-core gate: bf16 hi/lo split of Wg, max column norm, re-decision counter
  DevMem wg_pieces_, wg_nmax_, gate_fix_, gate_flags_;
  DevMem bpr_keys_, bpr_pos_;  // chunked BPR ranking scratch
  DevMem scan_done_;           // capacity scan: last-CTA counter
  DevMem kspan_;                 // [kMaxSpans][4] u64 kernel spans (set_kernel_spans)
  std::vector<int> kspan_phase_;
  double span_mhz_ = 0.0;  // effective SM clock inside the spanned GEMMs (last take)
  bool kspan_on_ = false;
  int64_t simt_gemms_ = 0;  // SIMT fallback GEMM launches since the last forward began
  int cur_phase_ = -1;
  bool gate_tc_ = false, wg_dirty_ = true;
  // peer transport: dispatch fused into encode / decode-backward (NVLink stores, MOE_DISPATCH=fused)
  bool fused_dispatch_ = false;
  // cosine router (RouterParams, gating.hpp:25-30): P [M][256], C [E][256], C^T, |C_e|, x . P
  DevMem cos_p_, cos_ce_, cos_ct_, cos_en_, cos_buf_, gate_err_;
  double cos_tau_ = 1.0;
  void check_gate_error();
  DevMem idxs_, gates_, locs_, hist_, offs_, demand_, demand_max_, list_base_, fill_, list_, capd_,
      drops_;
  DevMem slot_token_, slot_gate_;
  DevMem z_, recv_, act_, yexp_, ycomb_, dz_, drecv_, dh_, dxe_, dxcomb_;
  DevMem io_x_, io_y_, io_dy_, io_dx_;
  struct HostPipe {
    DevMem in[2], out[2];
    cudaEvent_t in_ready[2]{}, in_free[2]{}, out_ready[2]{}, out_free[2]{};
    int slot = 0;
  };
  HostPipe pipe_[2];  // [forward, backward]
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr;
  void pipe_call(int dir, const void* inh, void* outh, cudaStream_t st);
  void host_copy(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t st);
  size_t host_chunk_ = 0;
  void pipe_mark(const std::string& name, cudaStream_t st);
  bool pipe_tl_on_ = false;
  std::vector<std::pair<std::string, cudaEvent_t>> pipe_tl_;
  // ReLU-mask certificate state (relu_fix.cu)
  DevMem colnorm_, colnorm_blk_, w1t_, rownorm_, fix_list_, fix_count_, relu_mask_;
  // W > 1 peer backend: row norms of the send buffer (z order); pushed with the rows into the
  // peers' rownorm_ (receive order), so no receiver-side norm pass is needed
  DevMem znorm_;
  bool sender_norms_ = false;
  unsigned int fix_cap_ = 0;
  bool stats_dirty_ = true;
  void prepare_up(GemmArgs& up);
  // Single-rank fused path (W = 1, k = 1, bf16 tcgen05 shapes): decode runs in the down GEMM's
  // epilogue (gate scale + TMA row scatter to token rows) and encode-backward in the dgrad
  // GEMM's epilogue (row scatter), so expert-output rows are never materialised.
  bool fused_ = false;
  // W > 1 peer backend: combine (fwd) / dx combine (bwd) fused into the down / dgrad GEMM
  // epilogues, which store straight into the source ranks' buffers over NVLink.
  bool fused_combine_ = false;
  bool local_first_ = true;  // W > 1: chunk 0 computes this rank's own source segment first
  GemmArgs peer_args(const GemmArgs& a, int ch) const;

  struct ProfRec {
    int phase;
    cudaEvent_t a, b;
  };
  bool prof_ = false;
  std::vector<ProfRec> prof_recs_;
  std::vector<cudaEvent_t> ev_pool_;
  cudaEvent_t prof_open_[kNumPhases]{};
};

}  // namespace moe
