// Per-rank MoE layer: gate -> encode -> flexible all-to-all -> expert FFN -> all-to-all ->
// decode, and the reverse pass. One handle per GPU; NCCL grouped send/recv over NVLink for the
// exchanges; capacity-chunk pipelining on a compute stream and a comm stream.
//
// Restates LayerState / forward / backward of /root/reference/proj/src/moe_layer.cpp:
//   init draw order          :144-163     forward  :171-244     backward :246-319
// Per-rank placement P1 (moe_layer.cpp:138-140): experts are resident full-width on their owner
// (gathered once from ZeRO slices, parallelism.cpp:149-206) instead of re-gathered per step;
// nothing updates weights between steps, so this is numerically identical.
#include "layer.h"

#include <chrono>
#include <thread>

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <set>
#include <map>
#include <mutex>
#include <vector>

#include "gemm_sm100.h"
#include "kernels.h"
#include "peer_flags.h"

namespace moe {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw MoeError(MOE_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void ckr(int rc, const char* what) {
  if (rc == -1) throw MoeError(MOE_EINVAL, std::string(what) + ": invalid arguments");
  if (rc != 0) {
    cudaError_t e = last_launch_error();
    if (e == cudaSuccess) e = cudaGetLastError();
    last_launch_error() = cudaSuccess;
    throw MoeError(MOE_ECUDA, std::string(what) + ": launch failed (" + cudaGetErrorString(e) + ")");
  }
}
void ckn(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw MoeError(MOE_ECOMM, std::string(what) + ": " + ncclGetErrorString(r));
}

}  // namespace

bool smem_optin_raw(const void* kern, int bytes) {
  // per (kernel, device): the largest dynamic shared memory size set so far (a later, larger
  // request -- e.g. a second layer with a larger M -- raises it again)
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({kern, dev});
  if (it != done.end() && it->second >= bytes) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return false;
  done[{kern, dev}] = bytes;
  return true;
}

cudaError_t& last_launch_error() {
  static thread_local cudaError_t e = cudaSuccess;
  return e;
}

// Round-to-nearest-even double -> bf16 bits without passing through fp32 (no double rounding).
uint16_t bf16_bits_rne(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  if ((u & 0x7FF0000000000000ULL) != 0x7FF0000000000000ULL) {
    const uint64_t lsb = (u >> 45) & 1;
    u += (1ULL << 44) - 1 + lsb;
    u &= ~((1ULL << 45) - 1);
  }
  double r;
  std::memcpy(&r, &u, 8);
  const float f = static_cast<float>(r);  // exact: r has <= 8 significant bits
  uint32_t fb;
  std::memcpy(&fb, &f, 4);
  return static_cast<uint16_t>(fb >> 16);
}

void a2a_plan(int64_t W, int64_t E, int64_t cc, int64_t M, int64_t chunk, int phase,
              int64_t* send_off, int64_t* recv_off, int64_t* elems) {
  const int64_t dE = E / W;
  const int64_t blk = dE * cc * M;
  for (int64_t p = 0; p < W; ++p) {
    const int64_t zoff = (chunk * E + p * dE) * cc * M;  // [chunk][E][cc] block of peer p
    const int64_t roff = (chunk * W + p) * blk;           // [chunk][W][dE][cc] block of peer p
    send_off[p] = phase == 0 ? zoff : roff;
    recv_off[p] = phase == 0 ? roff : zoff;
  }
  *elems = blk;
}

int64_t expert_capacity(int64_t k, double f, int64_t tokens, int64_t experts) {
  if (k < 1 || tokens < 1 || experts < 1 || !(f > 0.0))
    throw MoeError(MOE_EINVAL, "expert_capacity: inputs must be positive");
  const double q = static_cast<double>(k) * f * static_cast<double>(tokens) / static_cast<double>(experts);
  const int64_t cap = static_cast<int64_t>(std::ceil(q - 1e-9));
  return std::max<int64_t>(cap, 1);
}

void validate(const moe_config& c) {
  if (c.world_size < 1 || c.gpus_per_node < 1) throw MoeError(MOE_EINVAL, "Dims: W and m must be >= 1");
  if (c.world_size % c.gpus_per_node != 0)
    throw MoeError(MOE_EINVAL, "Dims: world size must be a multiple of gpus per node");
  if (c.global_experts < 1) throw MoeError(MOE_EINVAL, "Dims: E must be >= 1");
  if (c.top_k < 1 || c.top_k > c.global_experts) throw MoeError(MOE_EINVAL, "Dims: need 1 <= k <= E");
  if (c.model_dim < 1 || c.hidden_dim < 1 || c.tokens_per_step < 1)
    throw MoeError(MOE_EINVAL, "Dims: M, V, T must be >= 1");
  if (c.global_experts < c.world_size) {  // RanksPerExpert{s}: W = E*s
    if (c.world_size % c.global_experts != 0)
      throw MoeError(MOE_EINVAL, "Dims: RanksPerExpert(s) requires W = E*s");
    if (c.hidden_dim % (c.world_size / c.global_experts) != 0)
      throw MoeError(MOE_EINVAL, "ExpertParams: hidden dim must divide into parameter slices");
  } else {
    if (c.global_experts % c.world_size != 0)
      throw MoeError(MOE_EINVAL, "Dims: ExpertsPerRank(x) requires E = W*x");
    if (c.hidden_dim % c.world_size != 0)
      throw MoeError(MOE_EINVAL, "ExpertParams: hidden dim must divide into parameter slices");
  }
  if (c.parallel < MOE_PARALLEL_P1 || c.parallel > MOE_PARALLEL_ADAPTIVE)
    throw MoeError(MOE_EINVAL, "parallel control");
  if (c.gate_precision != MOE_GATE_AUTO && c.gate_precision != MOE_GATE_FP64)
    throw MoeError(MOE_EINVAL, "gate_precision must be MOE_GATE_AUTO or MOE_GATE_FP64");
  if (c.a2a_algo != MOE_A2A_LINEAR && c.a2a_algo != MOE_A2A_2DH)
    throw MoeError(MOE_EINVAL, "all-to-all algorithm");
  if (c.top_k > 32) throw MoeError(MOE_EINVAL, "top_k > 32 unsupported");
  if (c.global_experts > 256) throw MoeError(MOE_EINVAL, "E > 256 unsupported by the gate kernel");
  if (c.dtype != MOE_DTYPE_BF16 && c.dtype != MOE_DTYPE_F32) throw MoeError(MOE_EINVAL, "dtype");
  if (c.router != MOE_ROUTER_LINEAR && c.router != MOE_ROUTER_COSINE)
    throw MoeError(MOE_EINVAL, "router kind");
  if (c.router == MOE_ROUTER_COSINE && (c.global_experts > 64 || c.global_experts % 2 != 0))
    throw MoeError(MOE_EINVAL, "cosine router: E <= 64 (even) supported");
  if (c.capacity_kind < 0 || c.capacity_kind > 2) throw MoeError(MOE_EINVAL, "capacity kind");
  if (c.capacity_kind != MOE_CAP_AUTO && !(c.capacity_factor > 0.0))
    throw MoeError(MOE_EINVAL, "capacity factor must be positive");
  if (c.degree != 1 && c.degree != 2 && c.degree != 4 && c.degree != 8)
    throw MoeError(MOE_EINVAL, "pipelining degree must be 1, 2, 4 or 8");
  if (c.model_dim > (1 << 20) || c.hidden_dim > (1 << 20) || c.tokens_per_step > (1 << 26))
    throw MoeError(MOE_EINVAL, "dims too large");
}

// comm_cost_p1 / comm_cost_p2 / select_parallelism (parallelism.cpp:288-308), same operation order.
int32_t select_parallelism(double local_experts, int64_t gathered_capacity, int64_t model_dim,
                           double param_bytes, int64_t n_sharded) {
  if (n_sharded < 1) throw MoeError(MOE_EINVAL, "comm_cost_p2: n_sharded must be >= 1");
  const double p1 = 8.0 * local_experts * static_cast<double>(gathered_capacity) *
                        static_cast<double>(model_dim) +
                    param_bytes;
  const double p2 = 8.0 * static_cast<double>(n_sharded) * local_experts *
                    static_cast<double>(gathered_capacity) * static_cast<double>(model_dim);
  return p1 <= p2 ? MOE_PARALLEL_P1 : MOE_PARALLEL_P2;
}

DevMem::~DevMem() {
  if (p) cudaFree(p);
}
void DevMem::alloc(size_t n) {
  if (n <= bytes) return;
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
  ck(cudaMalloc(&p, n), "cudaMalloc");
  bytes = n;
}

Layer::Layer(const moe_config& cfg, int rank, const uint8_t* nccl_id, int device)
    : cfg_(cfg), rank_(rank), device_(device) {
  validate(cfg);
  W_ = static_cast<int>(cfg.world_size);
  E_ = static_cast<int>(cfg.global_experts);
  dE_ = E_ / W_;
  sharded_ = E_ < W_;
  if (sharded_) {
    s_ = W_ / E_;
    dE_ = 1;  // the one computed expert, rank / s
  }
  M_ = static_cast<int>(cfg.model_dim);
  V_ = static_cast<int>(cfg.hidden_dim);
  T_ = static_cast<int>(cfg.tokens_per_step);
  k_ = static_cast<int>(cfg.top_k);
  esz_ = cfg.dtype == MOE_DTYPE_BF16 ? 2 : 4;
  if (rank < 0 || rank >= W_) throw MoeError(MOE_EINVAL, "rank out of range");
  if (cfg.gpus_per_node == cfg.world_size) search_.restrict_to({0, 1, 2, 3});  // linear x {1,2,4,8}
  // Fixed: the formula; Bounded: its formula at max_factor bounds every step; Auto: start at the
  // f = 1 capacity and grow (collectively) when a step's max demand exceeds the allocation.
  if (cfg.capacity_kind == MOE_CAP_AUTO)
    cap_ = static_cast<int>(expert_capacity(k_, 1.0, T_, E_));
  else
    cap_ = static_cast<int>(expert_capacity(k_, cfg.capacity_factor, T_, E_));
  cap_formula_ = cfg.capacity_kind == MOE_CAP_AUTO ? 0 : cap_;

  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) throw MoeError(MOE_ECUDA, "no such CUDA device");
  ck(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop{};
  ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10) throw MoeError(MOE_ECUDA, "sm_100 (B200) device required");
  num_sms_ = prop.multiProcessorCount;
  {
    const char* t = std::getenv("MOE_TIMELINE");
    tl_on_ = t && t[0] == '1';
  }
  {
    const char* pt = std::getenv("MOE_PIPE_TIMELINE");
    pipe_tl_on_ = pt && pt[0] == '1';
    const char* hc = std::getenv("MOE_HOST_CHUNK_MB");
    host_chunk_ = hc ? static_cast<size_t>(std::atol(hc)) << 20 : 0;
  }
  {
    const char* lf = std::getenv("MOE_LOCAL_FIRST");  // =0: chunk 0 waits for every source
    local_first_ = !(lf && lf[0] == '0');
    const char* e = std::getenv("MOE_FUSED");  // MOE_FUSED=0: unfused single-rank path (A/B runs)
    fused_ = !(e && e[0] == '0') && W_ == 1 && k_ == 1 && cfg.dtype == MOE_DTYPE_BF16 &&
             M_ % 256 == 0 && V_ % 256 == 0;
  }

  ck(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "stream");
  ck(cudaEventCreateWithFlags(&ev_fwd_start_, cudaEventDefault), "event");
  ck(cudaEventCreateWithFlags(&ev_fwd_end_, cudaEventDefault), "event");
  ck(cudaEventCreateWithFlags(&ev_sync_, cudaEventDisableTiming), "event");
  for (int i = 0; i < 8; ++i) {
    ck(cudaEventCreateWithFlags(&ev_a_[i], cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_b_[i], cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&ev_c_[i], cudaEventDisableTiming), "event");
  }
  for (int c = 0; c < PeerExchange::kChannels; ++c)
    ck(cudaEventCreateWithFlags(&ev_freed_[c], cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&ev_comm_done_, cudaEventDisableTiming), "event");

  if (W_ > 1) {
    if (!nccl_id) throw MoeError(MOE_EINVAL, "W > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ckn(ncclCommInitRank(&comm_, W_, id, rank_), "ncclCommInitRank");
    if (sharded_)  // the expert's sharing group: dW replica sums (P1) / slice gathers (P2)
      ckn(ncclCommSplit(comm_, rank_ / s_, rank_ % s_, &group_comm_, nullptr), "ncclCommSplit");
  }

  const size_t Tk = static_cast<size_t>(T_) * k_;
  const size_t cpb = gate_cta_per_block(T_);
  wg_.alloc(sizeof(double) * M_ * E_);
  gate_tc_ = cfg_.gate_precision != MOE_GATE_FP64 && cfg_.dtype == MOE_DTYPE_BF16 &&
             cfg_.router == MOE_ROUTER_LINEAR && !cfg_.bpr && gate_tc_supported(M_, E_, k_);
  if (gate_tc_) {
    wg_pieces_.alloc(static_cast<size_t>(2) * E_ * M_ * 2);
    wg_nmax_.alloc(sizeof(float));
    gate_fix_.alloc(3 * sizeof(int32_t));  // [0] metrics counter, [1..2] flag list size / CTAs done
    ck(cudaMemset(gate_fix_.p, 0, 3 * sizeof(int32_t)), "memset");
    gate_flags_.alloc(sizeof(int32_t) * static_cast<size_t>(T_));
  }
  gate_err_.alloc(sizeof(int32_t));
  ck(cudaMemset(gate_err_.p, 0, sizeof(int32_t)), "memset");
  if (cfg_.router == MOE_ROUTER_COSINE) {
    const size_t D = MOE_COSINE_DIM;
    cos_p_.alloc(sizeof(double) * M_ * D);
    cos_ce_.alloc(sizeof(double) * E_ * D);
    cos_ct_.alloc(sizeof(double) * E_ * D);
    cos_en_.alloc(sizeof(double) * E_);
    cos_buf_.alloc(sizeof(double) * static_cast<size_t>(T_) * D);
  }
  w1_.alloc(static_cast<size_t>(esz_) * dE_ * M_ * V_);
  w2_.alloc(static_cast<size_t>(esz_) * dE_ * V_ * M_);
  dw1_.alloc(sizeof(float) * dE_ * M_ * V_);
  dw2_.alloc(sizeof(float) * dE_ * V_ * M_);
  ck(cudaMemset(wg_.p, 0, wg_.bytes), "memset");
  ck(cudaMemset(w1_.p, 0, w1_.bytes), "memset");
  ck(cudaMemset(w2_.p, 0, w2_.bytes), "memset");
  if (sharded_) {
    const size_t mh = static_cast<size_t>(M_) * (V_ / s_);
    w1s_.alloc(static_cast<size_t>(esz_) * mh);
    dws1_.alloc(sizeof(float) * (mh + static_cast<size_t>(M_) * V_));  // slice + gathered slices
    dws2_.alloc(sizeof(float) * mh);
  }

  idxs_.alloc(4 * Tk);
  gates_.alloc(8 * Tk);
  locs_.alloc(4 * Tk);
  hist_.alloc(4 * cpb * E_);
  offs_.alloc(4 * cpb * E_);
  demand_.alloc(4 * E_);
  demand_max_.alloc(4 * E_);
  list_base_.alloc(4 * E_);
  fill_.alloc(4 * E_);
  list_.alloc(4 * Tk);
  scan_done_.alloc(sizeof(int32_t));
  ck(cudaMemset(scan_done_.p, 0, sizeof(int32_t)), "memset");
  if (cfg.bpr) {  // chunked BPR ranking scratch
    bpr_keys_.alloc(8 * Tk);
    bpr_pos_.alloc(4 * Tk);
  }
  capd_.alloc(4);
  drops_.alloc(4);
  ck(cudaMallocHost(&cap_host_, sizeof(int32_t)), "cudaMallocHost");
  if (cfg.dtype == MOE_DTYPE_BF16) {
    colnorm_.alloc(sizeof(float) * dE_ * V_);
    colnorm_blk_.alloc(sizeof(float) * dE_ * (V_ / 64 + 1));
    w1t_.alloc(static_cast<size_t>(esz_) * dE_ * M_ * V_);
    // list size, fixup CTAs done, last list size, largest list since the last metrics read
    fix_count_.alloc(4 * sizeof(unsigned int));
    ck(cudaMemset(fix_count_.p, 0, 4 * sizeof(unsigned int)), "memset");
  }
  if (W_ > 1 && cfg.a2a_backend != MOE_A2A_BACKEND_PEER && cfg.a2a_backend != MOE_A2A_BACKEND_NCCL)
    throw MoeError(MOE_EINVAL, "unknown all-to-all backend");
  alloc_capacity(cap_);
}

// (Re)allocates every capacity-sized buffer for capacity `cap` (and every pipelining degree's
// padding), and for the peer all-to-all re-exports the receive buffers. Collective when W > 1 and
// the peer backend is used: every rank reaches it at the same step (the capacity is global).
void Layer::alloc_capacity(int cap) {
  int ca = 0;
  for (int d : {1, 2, 4, 8}) ca = std::max(ca, d * ((cap + d - 1) / d));
  if (ca <= cap_alloc_) return;
  ck(cudaDeviceSynchronize(), "sync before realloc");
  peer_.reset();
  cap_alloc_ = ca;
  slot_token_.alloc(4 * static_cast<size_t>(E_) * cap_alloc_);
  slot_gate_.alloc(4 * static_cast<size_t>(E_) * cap_alloc_);
  // rows in z order are E * cap; the sharded receive order holds up to W * cap rows (P2)
  const size_t rows_all = static_cast<size_t>(std::max(E_, W_)) * cap_alloc_;
  const size_t rowsM = rows_all * M_ * esz_;
  const size_t rowsV = rows_all * V_ * esz_;
  act_.alloc(rowsV);
  dh_.alloc(rowsV);
  z_.alloc(rowsM);
  dz_.alloc(rowsM);
  if (!fused_) {  // the fused path never materialises expert-output rows
    yexp_.alloc(rowsM);
    dxe_.alloc(rowsM);
  }
  if (cfg_.dtype == MOE_DTYPE_BF16) {
    relu_mask_.alloc(sizeof(unsigned long long) * relu_mask_words(rows_all, (V_ + 63) / 64));
    rownorm_.alloc(sizeof(float) * rows_all);
    if (W_ > 1) znorm_.alloc(sizeof(float) * rows_all);
    fix_cap_ = static_cast<unsigned int>(std::max<size_t>(1 << 16, rows_all * V_ / 256));
    fix_list_.alloc(sizeof(unsigned long long) * fix_cap_);
  }
  if (W_ > 1) {
    recv_.alloc(rowsM);
    ycomb_.alloc(rowsM);
    drecv_.alloc(rowsM);
    dxcomb_.alloc(rowsM);
    if (sharded_) ypart_.alloc(rowsM);  // P2: the s partials of every expert, [chunk][E][s][cc]
    if (cfg_.a2a_backend == MOE_A2A_BACKEND_PEER && !sharded_) {
      void* bufs[PeerExchange::kChannels] = {recv_.p, ycomb_.p, drecv_.p, dxcomb_.p};
      const bool cert = cfg_.dtype == MOE_DTYPE_BF16;
      peer_ = std::make_unique<PeerExchange>(rank_, W_, comm_, bufs, cert ? rownorm_.p : nullptr);
      // copy-engine transfer spans (channels 0 / 2 dispatch, 1 / 3 combine) for the profile
      peer_->probe = [this](int ch, cudaStream_t s, bool begin) {
        if (prof_ || tl_on_) prof_mark(ch % 2 == 0 ? kPhXferDispatch : kPhXferCombine, begin, s);
      };
      const char* e = std::getenv("MOE_FUSED_COMBINE");  // =0: copy-engine combine (A/B runs)
      fused_combine_ = !(e && e[0] == '0') && cfg_.dtype == MOE_DTYPE_BF16 && W_ <= kMaxPeers &&
                       M_ % 256 == 0 && V_ % 64 == 0;
      // certificate row norms computed by the sender and pushed with the rows (tcgen05 path:
      // the up GEMM then takes the receive wait itself)
      sender_norms_ = cert && fused_combine_;
      // MOE_DISPATCH=fused: encode / decode-backward store every row straight into its owner's
      // receive buffer over NVLink (no send buffer, no copy-engine push); default: copy engines
      const char* dm = std::getenv("MOE_DISPATCH");
      fused_dispatch_ = dm && std::string(dm) == "fused" && fused_combine_ && W_ <= 8;
      for (auto& e : epoch_) e = 0;  // fresh flag block on every rank
      bwd_pending_ = false;
    }
  }
  fwd_done_ = false;
}

void Layer::tl_mark(const std::string& name, cudaStream_t st) {
  if (!tl_on_) return;
  cudaEvent_t e;
  ck(cudaEventCreateWithFlags(&e, cudaEventDefault), "event");
  ck(cudaEventRecord(e, st), "event");
  tl_.emplace_back(name, e);
}

void Layer::tl_flush() {
  if (!tl_on_ || tl_.empty()) return;
  ck(cudaDeviceSynchronize(), "sync");
  for (auto& [n, e] : tl_) {
    float t = 0.0f;
    ck(cudaEventElapsedTime(&t, tl_.front().second, e), "elapsed");
    std::fprintf(stderr, "[timeline r%d] %9.3f ms  %s\n", rank_, t, n.c_str());
  }
  for (auto& pe : tl_) cudaEventDestroy(pe.second);
  tl_.clear();
}

void Layer::prof_mark(int phase, bool begin, cudaStream_t st) {
  cur_phase_ = begin ? phase : -1;
  if (tl_on_) {
    static const char* names[] = {"gate", "encode", "gemm_up", "gemm_down", "decode", "decode_bwd",
                                  "gemm_dgrad_mask", "gemm_dgrad", "gemm_wgrad1", "gemm_wgrad2",
                                  "encode_bwd", "a2a_fwd", "a2a_bwd", "assign", "relu_fixup",
                                  "xfer_dispatch", "xfer_combine", "weight_stats"};
    tl_mark(std::string(phase < kNumPhases ? names[phase] : "?") + (begin ? " >" : " <") +
                (st == comm_stream_ ? " [comm]" : ""),
            st);
  }
  if (!prof_) return;
  cudaEvent_t e;
  if (!ev_pool_.empty()) {
    e = ev_pool_.back();
    ev_pool_.pop_back();
  } else {
    ck(cudaEventCreateWithFlags(&e, cudaEventDefault), "event");
  }
  ck(cudaEventRecord(e, st), "event");
  if (begin) {
    prof_open_[phase] = e;
  } else {
    prof_recs_.push_back({phase, prof_open_[phase], e});
    prof_open_[phase] = nullptr;
  }
}

void Layer::take_profile(double* ms, int64_t* counts, int n) {
  for (int i = 0; i < n; ++i) {
    ms[i] = 0.0;
    counts[i] = 0;
  }
  for (const auto& r : prof_recs_) {
    ck(cudaEventSynchronize(r.b), "event sync");
    float t = 0.0f;
    ck(cudaEventElapsedTime(&t, r.a, r.b), "elapsed");
    if (r.phase < n) {
      ms[r.phase] += t;
      counts[r.phase] += 1;
    }
    ev_pool_.push_back(r.a);
    ev_pool_.push_back(r.b);
  }
  prof_recs_.clear();
}

Layer::~Layer() {
  cudaSetDevice(device_);
  if (comm_stream_) cudaStreamSynchronize(comm_stream_);
  if (d2h_) cudaStreamSynchronize(d2h_);
  for (auto& p : pipe_)
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t e : {p.in_ready[i], p.in_free[i], p.out_ready[i], p.out_free[i]})
        if (e) cudaEventDestroy(e);
  if (h2d_) cudaStreamDestroy(h2d_);
  if (d2h_) cudaStreamDestroy(d2h_);
  peer_.reset();
  if (cap_host_) cudaFreeHost(cap_host_);
  for (const auto& r : prof_recs_) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (cudaEvent_t e : ev_pool_) cudaEventDestroy(e);
  if (group_comm_) ncclCommDestroy(group_comm_);
  if (comm_) ncclCommDestroy(comm_);
  if (comm_stream_) cudaStreamDestroy(comm_stream_);
  cudaEventDestroy(ev_fwd_start_);
  cudaEventDestroy(ev_fwd_end_);
  cudaEventDestroy(ev_sync_);
  cudaEventDestroy(ev_comm_done_);
  for (int i = 0; i < 8; ++i) {
    cudaEventDestroy(ev_a_[i]);
    cudaEventDestroy(ev_b_[i]);
    cudaEventDestroy(ev_c_[i]);
  }
  for (int c = 0; c < PeerExchange::kChannels; ++c) cudaEventDestroy(ev_freed_[c]);
}

uint64_t Layer::expert_draw_offset(int64_t e) const {
  return static_cast<uint64_t>(M_) * E_ + 256ULL * (M_ + E_) + static_cast<uint64_t>(e) * 2 * M_ * V_;
}

void Layer::init_params(uint64_t seed) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  ckr(fill_uniform_device(wg_.p, MOE_DTYPE_F64, static_cast<int64_t>(M_) * E_, seed, 0, -1.0, 1.0, 0),
      "init router");
  wg_dirty_ = true;
  const int dt = cfg_.dtype == MOE_DTYPE_BF16 ? 0 : 1;
  const size_t mv = static_cast<size_t>(M_) * V_;
  for (int le = 0; le < dE_; ++le) {
    const uint64_t o = expert_draw_offset(sharded_ ? rank_ / s_ : static_cast<int64_t>(rank_) * dE_ + le);
    ckr(fill_uniform_device(static_cast<char*>(w1_.p) + le * mv * esz_, dt, mv, seed, o, -0.5, 0.5, 0),
        "init w1");
    ckr(fill_uniform_device(static_cast<char*>(w2_.p) + le * mv * esz_, dt, mv, seed, o + mv, -0.5, 0.5, 0),
        "init w2");
  }
  if (cfg_.router == MOE_ROUTER_COSINE) {
    // RouterParams draws (moe_layer.cpp:154-160): cosine_proj (M x 256), cosine_experts (E x 256)
    const int64_t D = MOE_COSINE_DIM;
    const uint64_t o = static_cast<uint64_t>(M_) * E_;
    ckr(fill_uniform_device(cos_p_.p, MOE_DTYPE_F64, static_cast<int64_t>(M_) * D, seed, o, -1.0, 1.0, 0),
        "init cosine proj");
    ckr(fill_uniform_device(cos_ce_.p, MOE_DTYPE_F64, static_cast<int64_t>(E_) * D, seed,
                            o + static_cast<uint64_t>(M_) * D, -1.0, 1.0, 0),
        "init cosine experts");
    cos_tau_ = 1.0;  // RouterParams::temperature at init
    ckr(cosine_prep_device(static_cast<const double*>(cos_ce_.p), E_, static_cast<int>(D),
                           static_cast<double*>(cos_ct_.p), static_cast<double*>(cos_en_.p),
                           static_cast<int32_t*>(gate_err_.p), 0),
        "cosine prep");
  }
  ck(cudaDeviceSynchronize(), "init_params");
  stats_dirty_ = true;
}

void Layer::set_capacity_factor(double f) {
  if (cfg_.capacity_kind != MOE_CAP_FIXED)
    throw MoeError(MOE_ESTATE, "set_capacity_factor: layer capacity policy is not Fixed");
  if (!(f > 0.0)) throw MoeError(MOE_EINVAL, "capacity factor must be positive");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  cfg_.capacity_factor = f;
  cap_ = static_cast<int>(expert_capacity(k_, f, T_, E_));
  cap_formula_ = cap_;
  alloc_capacity(cap_);  // collective growth when needed
}

void Layer::set_cosine_router(const double* proj, const double* experts, double temperature) {
  if (cfg_.router != MOE_ROUTER_COSINE) throw MoeError(MOE_ESTATE, "set_cosine_router: layer uses the linear router");
  const int64_t D = MOE_COSINE_DIM;
  for (int64_t e = 0; e < E_; ++e) {
    double s = 0.0;
    for (int64_t d = 0; d < D; ++d) s += experts[e * D + d] * experts[e * D + d];
    if (s == 0.0) throw MoeError(MOE_EINVAL, "gate_cosine: zero-norm expert row");
  }
  ck(cudaSetDevice(device_), "cudaSetDevice");
  ck(cudaMemcpy(cos_p_.p, proj, sizeof(double) * M_ * D, cudaMemcpyHostToDevice), "set_cosine_router");
  ck(cudaMemcpy(cos_ce_.p, experts, sizeof(double) * E_ * D, cudaMemcpyHostToDevice), "set_cosine_router");
  cos_tau_ = std::max(temperature, 0.01);  // clamped as gating.cpp:42
  ckr(cosine_prep_device(static_cast<const double*>(cos_ce_.p), E_, static_cast<int>(D),
                         static_cast<double*>(cos_ct_.p), static_cast<double*>(cos_en_.p),
                         static_cast<int32_t*>(gate_err_.p), 0),
      "cosine prep");
  ck(cudaDeviceSynchronize(), "set_cosine_router");
}

// The cosine gate flags a zero-norm projected token on the device (no host sync in forward);
// the reference throws invalid_argument from gate_cosine -- reported at the next host read.
void Layer::check_gate_error() {
  int32_t err = 0;
  ck(cudaMemcpy(&err, gate_err_.p, sizeof(err), cudaMemcpyDeviceToHost), "copy");
  if (err) {
    ck(cudaMemset(gate_err_.p, 0, sizeof(int32_t)), "memset");
    throw MoeError(MOE_EINVAL, err == 2 ? "gate_cosine: zero-norm expert row"
                                        : "gate_cosine: zero-norm projected token");
  }
}

void Layer::set_router(const double* wg) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  ck(cudaMemcpy(wg_.p, wg, sizeof(double) * M_ * E_, cudaMemcpyHostToDevice), "set_router");
  wg_dirty_ = true;
}

void Layer::upload_weights(void* dst, const double* src, size_t n) {
  if (cfg_.dtype == MOE_DTYPE_BF16) {
    std::vector<uint16_t> buf(n);
    for (size_t i = 0; i < n; ++i) buf[i] = bf16_bits_rne(src[i]);
    ck(cudaMemcpy(dst, buf.data(), 2 * n, cudaMemcpyHostToDevice), "upload");
  } else {
    std::vector<float> buf(n);
    for (size_t i = 0; i < n; ++i) buf[i] = static_cast<float>(src[i]);
    ck(cudaMemcpy(dst, buf.data(), 4 * n, cudaMemcpyHostToDevice), "upload");
  }
}

void Layer::set_expert(int64_t le, const double* w1, const double* w2) {
  if (le < 0 || le >= dE_) throw MoeError(MOE_EINVAL, "set_expert: local expert out of range");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  const size_t mv = static_cast<size_t>(M_) * V_;
  upload_weights(static_cast<char*>(w1_.p) + le * mv * esz_, w1, mv);
  upload_weights(static_cast<char*>(w2_.p) + le * mv * esz_, w2, mv);
  stats_dirty_ = true;
}

// gather_computed_experts (parallelism.cpp:149-206) for per-rank placement: rank q holds slice q
// (w1 cols / w2 rows [q*h, (q+1)*h), h = V/W) of every expert; one grouped exchange sends each
// destination its experts' slices (w1 slice row-major, then w2 slice), then the owner assembles.
void Layer::set_expert_slices(const double* w1s, const double* w2s) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  if (sharded_) {
    // Sharded placement (parallelism.cpp:155-175): this rank holds slice rank%s of expert rank/s;
    // the sharing group all-gathers the s slices and every member assembles the full expert.
    const int h = V_ / s_;
    const size_t slice = static_cast<size_t>(2) * M_ * h;
    std::vector<double> packed(slice);
    std::memcpy(packed.data(), w1s, sizeof(double) * M_ * h);
    std::memcpy(packed.data() + static_cast<size_t>(M_) * h, w2s, sizeof(double) * h * M_);
    DevMem send, recv;
    send.alloc(slice * esz_);
    recv.alloc(slice * s_ * esz_);
    upload_weights(send.p, packed.data(), slice);
    const ncclDataType_t dt = cfg_.dtype == MOE_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32;
    ckn(ncclAllGather(send.p, recv.p, slice, dt, group_comm_, comm_stream_), "allgather");
    sync_comm(comm_stream_, "gather sync");
    for (int q = 0; q < s_; ++q) {
      const char* base = static_cast<const char*>(recv.p) + static_cast<size_t>(q) * slice * esz_;
      ck(cudaMemcpy2D(static_cast<char*>(w1_.p) + static_cast<size_t>(q) * h * esz_,
                      static_cast<size_t>(V_) * esz_, base, static_cast<size_t>(h) * esz_,
                      static_cast<size_t>(h) * esz_, M_, cudaMemcpyDeviceToDevice),
         "assemble w1");
      ck(cudaMemcpy(static_cast<char*>(w2_.p) + static_cast<size_t>(q) * h * M_ * esz_,
                    base + static_cast<size_t>(M_) * h * esz_, static_cast<size_t>(h) * M_ * esz_,
                    cudaMemcpyDeviceToDevice),
         "assemble w2");
    }
    ck(cudaDeviceSynchronize(), "set_expert_slices");
    stats_dirty_ = true;
    return;
  }
  const int h = V_ / W_;
  const size_t slice = static_cast<size_t>(2) * M_ * h;  // elements per (expert, slice)
  // Pack my slices of every expert in destination order (experts are rank-major).
  std::vector<double> packed(static_cast<size_t>(E_) * slice);
  for (int e = 0; e < E_; ++e) {
    std::memcpy(&packed[e * slice], w1s + static_cast<size_t>(e) * M_ * h, sizeof(double) * M_ * h);
    std::memcpy(&packed[e * slice + static_cast<size_t>(M_) * h], w2s + static_cast<size_t>(e) * h * M_,
                sizeof(double) * h * M_);
  }
  DevMem send, recv;
  send.alloc(packed.size() * esz_);
  recv.alloc(packed.size() * esz_);
  upload_weights(send.p, packed.data(), packed.size());
  const size_t per_peer = static_cast<size_t>(dE_) * slice;
  if (W_ == 1) {
    ck(cudaMemcpy(recv.p, send.p, per_peer * esz_, cudaMemcpyDeviceToDevice), "gather");
  } else {
    const ncclDataType_t dt = cfg_.dtype == MOE_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32;
    ckn(ncclGroupStart(), "group");
    for (int p = 0; p < W_; ++p) {
      ckn(ncclSend(static_cast<char*>(send.p) + p * per_peer * esz_, per_peer, dt, p, comm_, comm_stream_), "send");
      ckn(ncclRecv(static_cast<char*>(recv.p) + p * per_peer * esz_, per_peer, dt, p, comm_, comm_stream_), "recv");
    }
    ckn(ncclGroupEnd(), "group");
    sync_comm(comm_stream_, "gather sync");
  }
  // recv block q = slice q of my dE experts -> full weights (strided 2-D copies).
  const size_t mv = static_cast<size_t>(M_) * V_;
  for (int q = 0; q < W_; ++q)
    for (int le = 0; le < dE_; ++le) {
      const char* base = static_cast<const char*>(recv.p) + (q * per_peer + le * slice) * esz_;
      char* w1 = static_cast<char*>(w1_.p) + le * mv * esz_;
      char* w2 = static_cast<char*>(w2_.p) + le * mv * esz_;
      // w1 slice (M, h) -> columns [q*h, (q+1)*h) of (M, V)
      ck(cudaMemcpy2D(w1 + static_cast<size_t>(q) * h * esz_, static_cast<size_t>(V_) * esz_, base,
                      static_cast<size_t>(h) * esz_, static_cast<size_t>(h) * esz_, M_,
                      cudaMemcpyDeviceToDevice),
         "assemble w1");
      // w2 slice (h, M) -> rows [q*h, (q+1)*h) of (V, M)
      ck(cudaMemcpy(w2 + static_cast<size_t>(q) * h * M_ * esz_, base + static_cast<size_t>(M_) * h * esz_,
                    static_cast<size_t>(h) * M_ * esz_, cudaMemcpyDeviceToDevice),
         "assemble w2");
    }
  ck(cudaDeviceSynchronize(), "set_expert_slices");
  stats_dirty_ = true;
}

// Enables the ReLU-mask certificate on an up-GEMM launch (bf16 path only).
void Layer::prepare_up(GemmArgs& up) {
  if (cfg_.dtype != MOE_DTYPE_BF16) return;
  up.rownorm = static_cast<const float*>(rownorm_.p);
  up.colnorm = static_cast<const float*>(colnorm_.p);
  up.colnorm_blk = static_cast<const float*>(colnorm_blk_.p);
  up.relu_mask = static_cast<unsigned long long*>(relu_mask_.p);
  up.fix_list = static_cast<unsigned long long*>(fix_list_.p);
  up.fix_count = static_cast<unsigned int*>(fix_count_.p);
  up.fix_cap = fix_cap_;
}

bool Layer::tc_ok(int kind, const GemmArgs& a) const {
  if (cfg_.dtype != MOE_DTYPE_BF16) return false;
  if (a.N % 256 != 0) return false;
  if (kind == kGemmWgrad) return a.Mo % 128 == 0;
  return a.K % 64 == 0;
}

void Layer::gemm(int kind, const void* A, const void* B, void* D, const GemmArgs& a, int nseg,
                 cudaStream_t st) {
  int rc;
  if (cfg_.dtype == MOE_DTYPE_F32)
    rc = gemm_f32(kind, static_cast<const float*>(A), static_cast<const float*>(B),
                  static_cast<float*>(D), a, st);
  else if (tc_ok(kind, a)) {
    constexpr int kMaxSpans = 4096;
    if (kspan_on_ && static_cast<int>(kspan_phase_.size()) < kMaxSpans) {
      GemmArgs b = a;
      b.span = static_cast<unsigned long long*>(kspan_.p) + 4 * kspan_phase_.size();
      kspan_phase_.push_back(cur_phase_);
      rc = gemm_fwd(static_cast<GemmKind>(kind), A, B, D, b, nseg, num_sms_, st);
    } else {
      rc = gemm_fwd(static_cast<GemmKind>(kind), A, B, D, a, nseg, num_sms_, st);
    }
  }
  else {
    // shape not tcgen05-eligible: ~10x slower SIMT kernel, counted in moe_step_metrics.simt_gemms
    static bool warned = false;
    if (!warned) {
      warned = true;
      std::fprintf(stderr, "moe_b200: expert GEMM N=%u K=%u Mo=%u is not tcgen05-eligible (N %% 256, "
                           "K %% 64, wgrad rows %% 128); using the SIMT kernel\n", a.N, a.K, a.Mo);
    }
    ++simt_gemms_;
    rc = gemm_bf16_simt(kind, A, B, D, a, st);
  }
  ckr(rc, "expert gemm");
  ++launches_;
}

GatingArgs Layer::gating_args(const void* x) const {
  GatingArgs g{};
  g.x = x;
  g.x_is_f32 = cfg_.dtype == MOE_DTYPE_F32;
  g.wg = static_cast<const double*>(wg_.p);
  g.blocks = 1;
  g.T = T_;
  g.M = M_;
  g.E = E_;
  g.k = k_;
  g.cap_kind = cfg_.capacity_kind;
  g.cap_formula = cfg_.capacity_kind == MOE_CAP_FIXED ? cap_ : cap_formula_;
  g.bpr = cfg_.bpr;
  g.router = cfg_.router;
  if (cfg_.router == MOE_ROUTER_COSINE) {
    g.cos_proj = static_cast<const double*>(cos_p_.p);
    g.cos_ct = static_cast<const double*>(cos_ct_.p);
    g.cos_en = static_cast<const double*>(cos_en_.p);
    g.cos_tau = cos_tau_;
    g.cos_dim = MOE_COSINE_DIM;
    g.cos_buf = static_cast<double*>(cos_buf_.p);
  }
  g.err = static_cast<int32_t*>(gate_err_.p);
  if (gate_tc_) {
    g.wg_pieces = wg_pieces_.p;
    g.wg_norm_max = static_cast<const float*>(wg_nmax_.p);
    g.gate_fixups = static_cast<int32_t*>(gate_fix_.p);
    g.gate_flags = static_cast<int32_t*>(gate_flags_.p);
    g.gate_flag_count = static_cast<int32_t*>(gate_fix_.p) + 1;
  }
  return g;
}

GatingBuffers Layer::gating_buffers() {
  GatingBuffers b{};
  b.idxs = static_cast<int32_t*>(idxs_.p);
  b.gates = static_cast<double*>(gates_.p);
  b.locations = static_cast<int32_t*>(locs_.p);
  b.hist = static_cast<int32_t*>(hist_.p);
  b.offs = static_cast<int32_t*>(offs_.p);
  b.demand = static_cast<int32_t*>(demand_.p);
  b.list_base = static_cast<int32_t*>(list_base_.p);
  b.fill = static_cast<int32_t*>(fill_.p);
  b.list = static_cast<int32_t*>(list_.p);
  b.cap = static_cast<int32_t*>(capd_.p);
  b.drops = static_cast<int32_t*>(drops_.p);
  b.slot_token = static_cast<int32_t*>(slot_token_.p);
  b.slot_gate = static_cast<float*>(slot_gate_.p);
  b.probs = nullptr;
  b.scan_done = static_cast<int32_t*>(scan_done_.p);
  if (cfg_.bpr) {
    b.bpr_keys = static_cast<unsigned long long*>(bpr_keys_.p);
    b.bpr_pos = static_cast<int32_t*>(bpr_pos_.p);
  }
  return b;
}

SlotGeom Layer::geom() const {
  SlotGeom g{};
  g.blocks = 1;
  g.T = T_;
  g.E = E_;
  g.M = M_;
  g.k = k_;
  g.cap = cap_;
  g.cc = cc_;
  g.degree = degree_;
  return g;
}

// One grouped exchange of chunk `chunk` (all2all_linear, collectives.cpp:48-56): block p of
// `send` -> rank p, block p of `recv` <- rank p, offsets from a2a_plan.
void Layer::exchange(const void* send, void* recv, int chunk, int phase) {
  const ncclDataType_t dt = cfg_.dtype == MOE_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32;
  std::vector<int64_t> so(W_), ro(W_);
  int64_t elems = 0;
  a2a_plan(W_, E_, cc_, M_, chunk, phase, so.data(), ro.data(), &elems);
  const int m = static_cast<int>(cfg_.gpus_per_node);
  if (strategy_.algo == MOE_A2A_2DH && m < W_) {
    // the W blocks of either side are contiguous in rank order (a2a_plan's offsets)
    exchange_2dh(static_cast<const char*>(send) + so[0] * esz_, static_cast<char*>(recv) + ro[0] * esz_,
                 static_cast<size_t>(elems) * esz_, dt, elems);
    return;
  }
  ckn(ncclGroupStart(), "ncclGroupStart");
  for (int p = 0; p < W_; ++p) {
    ckn(ncclSend(static_cast<const char*>(send) + so[p] * esz_, elems, dt, p, comm_, comm_stream_),
        "ncclSend");
    ckn(ncclRecv(static_cast<char*>(recv) + ro[p] * esz_, elems, dt, p, comm_, comm_stream_),
        "ncclRecv");
  }
  ckn(ncclGroupEnd(), "ncclGroupEnd");
  comm_bytes_ += static_cast<double>(elems) * esz_ * (W_ - 1);
}

// all2all_2dh (collectives.cpp:58-88) on the comm stream: block p of `send` goes to rank p and
// block p of `recv` comes from rank p, as the linear exchange, but in two NCCL phases over
// n = W/m nodes of m GPUs. (1) Reorder the blocks so those for local GPU g are contiguous
// ([g][node]); (2) intra-node exchange of n blocks with each local GPU; (3) reorder to
// [node][source local]; (4) inter-node exchange of m blocks with the same-local GPU of every
// node, landing in source-rank order. The reorders are strided 2-D copies of whole blocks.
void Layer::exchange_2dh(const char* send, char* recv, size_t B, ncclDataType_t dt, int64_t elems) {
  const int m = static_cast<int>(cfg_.gpus_per_node), n = W_ / m;
  const int node = rank_ / m, local = rank_ % m;
  a2a_tmp_.alloc(2 * static_cast<size_t>(W_) * B);
  char* ta = static_cast<char*>(a2a_tmp_.p);
  char* tb = ta + static_cast<size_t>(W_) * B;
  for (int g = 0; g < m; ++g)  // ta[g][nd] = send[nd * m + g]
    ck(cudaMemcpy2DAsync(ta + static_cast<size_t>(g) * n * B, B, send + static_cast<size_t>(g) * B,
                         static_cast<size_t>(m) * B, B, n, cudaMemcpyDeviceToDevice, comm_stream_),
       "2dh align");
  ckn(ncclGroupStart(), "ncclGroupStart");
  for (int g = 0; g < m; ++g) {
    const int peer = node * m + g;
    ckn(ncclSend(ta + static_cast<size_t>(g) * n * B, n * elems, dt, peer, comm_, comm_stream_), "ncclSend");
    ckn(ncclRecv(tb + static_cast<size_t>(g) * n * B, n * elems, dt, peer, comm_, comm_stream_), "ncclRecv");
  }
  ckn(ncclGroupEnd(), "ncclGroupEnd");
  for (int nd = 0; nd < n; ++nd)  // ta[nd][g] = tb[g][nd]
    ck(cudaMemcpy2DAsync(ta + static_cast<size_t>(nd) * m * B, B, tb + static_cast<size_t>(nd) * B,
                         static_cast<size_t>(n) * B, B, m, cudaMemcpyDeviceToDevice, comm_stream_),
       "2dh align");
  ckn(ncclGroupStart(), "ncclGroupStart");
  for (int nd = 0; nd < n; ++nd) {
    const int peer = local + nd * m;
    ckn(ncclSend(ta + static_cast<size_t>(nd) * m * B, m * elems, dt, peer, comm_, comm_stream_), "ncclSend");
    ckn(ncclRecv(recv + static_cast<size_t>(nd) * m * B, m * elems, dt, peer, comm_, comm_stream_), "ncclRecv");
  }
  ckn(ncclGroupEnd(), "ncclGroupEnd");
  comm_bytes_ += static_cast<double>(B) * (static_cast<double>(n) * (m - 1) + static_cast<double>(m) * (n - 1));
}

// Copy-engine version of exchange(): push chunk `chunk` of `src` into every peer's channel
// buffer (same plan), then publish the chunk's ready flag.
// Row parts of the first chunk (pipelined in pieces so its first rows land while the own
// segment is computed): the chunk's 256-row tiles in three near-equal parts, larger first
// (MOE_PARTS: an explicit comma list of tile counts). With the peers' transfer about as long as
// their GEMM (C4 at N = 4), equal parts let every part's GEMM start as its rows land; the
// earlier 1/4, 1/4, 1/2 split left the last half's transfer exposed. Parts except the last
// publish kPartSlot0 + i, the last the chunk's slot 0.
static std::vector<uint32_t> first_chunk_parts(int64_t cc, bool enable) {
  if (!enable || cc % 256 != 0 || cc < 512) return {static_cast<uint32_t>(cc)};
  const int64_t tiles = cc / 256;
  std::vector<uint32_t> parts;
  if (const char* e = std::getenv("MOE_PARTS")) {
    int64_t sum = 0;
    for (const char* q = e; *q;) {
      char* end = nullptr;
      const long v = std::strtol(q, &end, 10);
      if (end == q) {  // not a number: skip one separator character
        ++q;
        continue;
      }
      q = end;
      if (v <= 0) {  // a zero or negative part: malformed
        sum = -1;
        break;
      }
      parts.push_back(static_cast<uint32_t>(v * 256));
      sum += v;
    }
    if (sum == tiles && !parts.empty() &&
        parts.size() <= static_cast<size_t>(PeerExchange::kPartSlots) + 1)
      return parts;
    parts.clear();  // malformed or not covering the chunk: the default
  }
  const int64_t k = std::min<int64_t>(3, tiles);
  for (int64_t i = 0; i < k; ++i)
    parts.push_back(static_cast<uint32_t>((tiles / k + (i < tiles % k ? 1 : 0)) * 256));
  return parts;
}

// Rows [row0, row0 + nrows) of every segment of chunk `chunk` to every peer (slot: ready flag).
void Layer::peer_push_rows(int ch, const void* src, int chunk, int phase, int slot, uint32_t row0,
                           uint32_t nrows, uint32_t epoch) {
  std::vector<int64_t> so(W_), ro(W_);
  int64_t elems = 0;
  a2a_plan(W_, E_, cc_, M_, chunk, phase, so.data(), ro.data(), &elems);
  for (int p = 0; p < W_; ++p) {
    so[p] *= esz_;
    ro[p] *= esz_;
  }
  const size_t row_bytes = static_cast<size_t>(M_) * esz_;
  const float* norms = (ch == 0 && sender_norms_) ? static_cast<const float*>(znorm_.p) : nullptr;
  peer_->push_rows(comm_stream_, ch, slot, src, so.data(), ro.data(), static_cast<size_t>(dE_),
                   cc_ * row_bytes, row0 * row_bytes, nrows * row_bytes, epoch, norms, row_bytes);
  comm_bytes_ += static_cast<double>(dE_) * nrows * row_bytes * (W_ - 1);
}

// Fused-combine GEMM arguments: segment (chunk, src, g) goes to rank src's channel-ch buffer.
GemmArgs Layer::peer_args(const GemmArgs& a, int ch) const {
  GemmArgs d = a;
  d.idx_mode = kIdxPeerD;
  d.peer_world = static_cast<uint32_t>(W_);
  d.peer_rank = static_cast<uint32_t>(rank_);
  d.peer_out_segs = static_cast<uint32_t>(degree_ * E_);
  for (int p = 0; p < W_; ++p) d.peer_d[p] = peer_->buffer(ch, p);
  return d;
}

void Layer::peer_push(int ch, const void* src, int chunk, int phase, uint32_t epoch,
                      cudaEvent_t local_done) {
  std::vector<int64_t> so(W_), ro(W_);
  int64_t elems = 0;
  a2a_plan(W_, E_, cc_, M_, chunk, phase, so.data(), ro.data(), &elems);
  const float* norms = (ch == 0 && sender_norms_) ? static_cast<const float*>(znorm_.p) : nullptr;
  peer_->push_chunk(comm_stream_, ch, chunk, src, so.data(), ro.data(),
                    static_cast<size_t>(elems) * esz_, esz_, epoch, local_done, norms, M_);
  comm_bytes_ += static_cast<double>(elems) * esz_ * (W_ - 1);
}

// P2's W1 slice (columns [q*h, (q+1)*h) of the computed expert's (M, V) W1) as a contiguous
// (M, h) operand; W2's slice rows and W1^T's slice rows (certificate) are contiguous in place.
void Layer::refresh_slices(cudaStream_t st) {
  const int h = V_ / s_, q = rank_ % s_;
  ck(cudaMemcpy2DAsync(w1s_.p, static_cast<size_t>(h) * esz_,
                       static_cast<const char*>(w1_.p) + static_cast<size_t>(q) * h * esz_,
                       static_cast<size_t>(V_) * esz_, static_cast<size_t>(h) * esz_, M_,
                       cudaMemcpyDeviceToDevice, st),
     "W1 slice");
}

// Sharded-placement exchanges (moe_layer.cpp:17-108) as grouped send/recv on the comm stream.
// Slabs are (cc, M) blocks: z order [chunk][E][cc], receive order [chunk][nsrc][cc] (P1: the E
// sources [q*E, (q+1)*E) this replica serves, q = rank % s; P2: all W sources), P2 partials
// [chunk][E][s][cc].
void Layer::shard_exchange(const void* send, void* recv, int chunk, int dir, bool p2) {
  const ncclDataType_t dt = cfg_.dtype == MOE_DTYPE_BF16 ? ncclBfloat16 : ncclFloat32;
  const int64_t blk = static_cast<int64_t>(cc_) * M_;
  const int nsrc = p2 ? W_ : E_;
  const int q_src = rank_ / E_;  // P1: the replica index serving my tokens
  const int q_mine = rank_ % s_;
  const char* sb = static_cast<const char*>(send);
  char* rb = static_cast<char*>(recv);
  auto zslab = [&](int e) { return (static_cast<int64_t>(chunk) * E_ + e) * blk * esz_; };
  auto rslab = [&](int j) { return (static_cast<int64_t>(chunk) * nsrc + j) * blk * esz_; };
  auto pslab = [&](int e, int q) { return ((static_cast<int64_t>(chunk) * E_ + e) * s_ + q) * blk * esz_; };
  int sent = 0;
  auto snd = [&](const char* p, int peer) {
    ckn(ncclSend(p, blk, dt, peer, comm_, comm_stream_), "ncclSend");
    sent += peer != rank_;
  };
  auto rcv = [&](char* p, int peer) { ckn(ncclRecv(p, blk, dt, peer, comm_, comm_stream_), "ncclRecv"); };
  ckn(ncclGroupStart(), "ncclGroupStart");
  if (dir == 0) {
    // dispatch_sharded_p1 (:20-39): slab e -> the replica e*s + r/E; p2 (:61-78): -> all s shards
    for (int e = 0; e < E_; ++e) {
      if (!p2) {
        snd(sb + zslab(e), e * s_ + q_src);
      } else {
        for (int q = 0; q < s_; ++q) snd(sb + zslab(e), e * s_ + q);
      }
    }
    for (int j = 0; j < nsrc; ++j) rcv(rb + rslab(j), p2 ? j : q_mine * E_ + j);
  } else {
    // combine_sharded_p1 (:42-57): source slabs back; p2 (:82-108): every shard's partials
    for (int j = 0; j < nsrc; ++j) snd(sb + rslab(j), p2 ? j : q_mine * E_ + j);
    for (int e = 0; e < E_; ++e) {
      if (!p2) {
        rcv(rb + zslab(e), e * s_ + q_src);
      } else {
        for (int q = 0; q < s_; ++q) rcv(rb + pslab(e, q), e * s_ + q);
      }
    }
  }
  ckn(ncclGroupEnd(), "ncclGroupEnd");
  comm_bytes_ += static_cast<double>(sent) * blk * esz_;
}

// Forward expert section under sharded placement: the computed expert is the full expert
// rank/s (P1) or its slice rank%s (P2, hidden width h = V/s; partial outputs summed at the
// source). Comm stream: all dispatches, then all combines; compute stream: per chunk up + down.
void Layer::sharded_forward(GemmArgs up, GemmArgs down, bool cert, cudaStream_t st) {
  const bool p2 = parallel_ == MOE_PARALLEL_P2;
  const int nsrc = p2 ? W_ : E_;
  const int h = p2 ? V_ / s_ : V_;
  const size_t qoff = p2 ? static_cast<size_t>(rank_ % s_) * h : 0;  // first hidden column held
  const void* w1 = p2 ? w1s_.p : w1_.p;
  const void* w2 = static_cast<const char*>(w2_.p) + qoff * M_ * esz_;
  const int nseg = degree_ * nsrc;
  up.G = 1;
  up.S = nsrc;
  up.seg_rows = cc_;
  up.N = h;
  up.K = M_;
  down.G = 1;
  down.S = nsrc;
  down.seg_rows = cc_;
  down.N = M_;
  down.K = h;
  if (cert) {
    up.colnorm += qoff;
    up.colnorm_blk += qoff / 64;
  }
  ck(cudaEventRecord(ev_sync_, st), "event");
  ck(cudaStreamWaitEvent(comm_stream_, ev_sync_, 0), "wait");
  prof_mark(kPhA2aFwd, true, comm_stream_);
  for (int i = 0; i < degree_; ++i) {
    shard_exchange(z_.p, recv_.p, i, 0, p2);
    ck(cudaEventRecord(ev_a_[i], comm_stream_), "event");
  }
  for (int i = 0; i < degree_; ++i) {
    ck(cudaStreamWaitEvent(st, ev_a_[i], 0), "wait");
    up.seg_base = down.seg_base = static_cast<uint32_t>(i * nsrc);
    if (cert) {
      RowSet rs;
      rs.seg_begin = static_cast<int64_t>(i) * nsrc;
      rs.nsegs = nsrc;
      rs.seg_rows = rs.nrows = cc_;
      ckr(rownorm_device(recv_.p, M_, static_cast<float*>(rownorm_.p), rs, st), "rownorm");
      ++launches_;
      ck(cudaMemsetAsync(fix_count_.p, 0, sizeof(unsigned int), st), "memset");
    }
    prof_mark(kPhUp, true, st);
    gemm(kGemmUp, recv_.p, w1, act_.p, up, nseg, st);
    prof_mark(kPhUp, false, st);
    if (cert) {
      prof_mark(kPhReluFix, true, st);
      ckr(relu_fixup_device(recv_.p, static_cast<const char*>(w1t_.p) + qoff * M_ * esz_, 1, cc_, M_, h,
                            static_cast<const unsigned long long*>(fix_list_.p),
                            static_cast<const unsigned int*>(fix_count_.p), fix_cap_, act_.p,
                            static_cast<unsigned long long*>(relu_mask_.p), st),
          "relu_fixup");
      prof_mark(kPhReluFix, false, st);
      ++launches_;
    }
    prof_mark(kPhDown, true, st);
    gemm(kGemmDown, act_.p, w2, yexp_.p, down, nseg, st);
    prof_mark(kPhDown, false, st);
    ck(cudaEventRecord(ev_b_[i], st), "event");
  }
  for (int i = 0; i < degree_; ++i) {
    ck(cudaStreamWaitEvent(comm_stream_, ev_b_[i], 0), "wait");
    shard_exchange(yexp_.p, p2 ? ypart_.p : ycomb_.p, i, 1, p2);
  }
  prof_mark(kPhA2aFwd, false, comm_stream_);
  ck(cudaEventRecord(ev_comm_done_, comm_stream_), "event");
  ck(cudaStreamWaitEvent(st, ev_comm_done_, 0), "wait");
  if (p2) {
    ckr(shard_sum_device(ypart_.p, ycomb_.p, static_cast<int64_t>(degree_) * E_, s_,
                         static_cast<int64_t>(cc_) * M_, cfg_.dtype, st),
        "shard_sum");
    ++launches_;
  }
}

// Backward expert section under sharded placement (moe_layer.cpp:246-319 with make_exchange's
// sharded ops): dY rows go out with the dispatch op, dX comes back with the combine op. The
// weight gradient of the computed expert is summed over its s replicas (P1,
// reduce_scatter_grads_p1 :247-262) or assembled from the s complete slice gradients (P2), so
// every member of the group returns the full expert gradient.
void Layer::sharded_backward(GemmArgs dgm, GemmArgs dg, GemmArgs wg1, GemmArgs wg2, float* gw1,
                             float* gw2, cudaStream_t st) {
  const bool p2 = parallel_ == MOE_PARALLEL_P2;
  const int nsrc = p2 ? W_ : E_;
  const int h = p2 ? V_ / s_ : V_;
  const size_t qoff = p2 ? static_cast<size_t>(rank_ % s_) * h : 0;
  const void* w1 = p2 ? w1s_.p : w1_.p;
  const void* w2 = static_cast<const char*>(w2_.p) + qoff * M_ * esz_;
  const int nseg = degree_ * nsrc;
  dgm.G = dg.G = wg1.G = wg2.G = 1;
  dgm.S = dg.S = nsrc;
  dgm.N = h;
  dgm.K = M_;
  dg.N = M_;
  dg.K = h;
  wg1.S = wg2.S = degree_ * nsrc;
  wg1.N = h;
  wg1.Mo = M_;
  wg2.N = M_;
  wg2.Mo = h;
  float* o1 = p2 ? static_cast<float*>(dws1_.p) : gw1;
  float* o2 = p2 ? static_cast<float*>(dws2_.p) : gw2;
  ck(cudaEventRecord(ev_sync_, st), "event");
  ck(cudaStreamWaitEvent(comm_stream_, ev_sync_, 0), "wait");
  prof_mark(kPhA2aBwd, true, comm_stream_);
  for (int i = 0; i < degree_; ++i) {  // adjoint of combine
    shard_exchange(dz_.p, drecv_.p, i, 0, p2);
    ck(cudaEventRecord(ev_a_[i], comm_stream_), "event");
  }
  for (int i = 0; i < degree_; ++i) {
    ck(cudaStreamWaitEvent(st, ev_a_[i], 0), "wait");
    dgm.seg_base = dg.seg_base = static_cast<uint32_t>(i * nsrc);
    prof_mark(kPhDgradMask, true, st);
    gemm(kGemmDgradMask, drecv_.p, w2, dh_.p, dgm, nseg, st);
    prof_mark(kPhDgradMask, false, st);
    prof_mark(kPhDgrad, true, st);
    gemm(kGemmDgrad, dh_.p, w1, dxe_.p, dg, nseg, st);
    prof_mark(kPhDgrad, false, st);
    ck(cudaEventRecord(ev_b_[i], st), "event");
  }
  for (int i = 0; i < degree_; ++i) {  // adjoint of dispatch
    ck(cudaStreamWaitEvent(comm_stream_, ev_b_[i], 0), "wait");
    shard_exchange(dxe_.p, p2 ? ypart_.p : dxcomb_.p, i, 1, p2);
  }
  prof_mark(kPhA2aBwd, false, comm_stream_);
  ck(cudaEventRecord(ev_comm_done_, comm_stream_), "event");
  prof_mark(kPhWgrad1, true, st);
  gemm(kGemmWgrad, recv_.p, dh_.p, o1, wg1, nseg, st);
  prof_mark(kPhWgrad1, false, st);
  prof_mark(kPhWgrad2, true, st);
  gemm(kGemmWgrad, act_.p, drecv_.p, o2, wg2, nseg, st);
  prof_mark(kPhWgrad2, false, st);
  // group collectives after the data exchanges (two communicators never interleave)
  ck(cudaStreamWaitEvent(st, ev_comm_done_, 0), "wait");
  const size_t mv = static_cast<size_t>(M_) * V_;
  if (p2) {
    const size_t mh = static_cast<size_t>(M_) * h;
    float* g1 = static_cast<float*>(dws1_.p) + mh;  // [q][M][h]
    ckn(ncclAllGather(o1, g1, mh, ncclFloat32, group_comm_, st), "allgather dW1");
    ckn(ncclAllGather(o2, gw2, mh, ncclFloat32, group_comm_, st), "allgather dW2");  // [q][h][M] = (V, M)
    for (int q = 0; q < s_; ++q)
      ck(cudaMemcpy2DAsync(gw1 + static_cast<size_t>(q) * h, sizeof(float) * V_, g1 + q * mh,
                           sizeof(float) * h, sizeof(float) * h, M_, cudaMemcpyDeviceToDevice, st),
         "assemble dW1");
    ckr(shard_sum_device(ypart_.p, dxcomb_.p, static_cast<int64_t>(degree_) * E_, s_,
                         static_cast<int64_t>(cc_) * M_, cfg_.dtype, st),
        "shard_sum");
    ++launches_;
  } else {
    ckn(ncclAllReduce(gw1, gw1, mv, ncclFloat32, ncclSum, group_comm_, st), "allreduce dW1");
    ckn(ncclAllReduce(gw2, gw2, mv, ncclFloat32, ncclSum, group_comm_, st), "allreduce dW2");
  }
}

void Layer::forward(const void* x, void* y, cudaStream_t st) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  if (W_ > 1 && comm_ == nullptr) throw MoeError(MOE_ECOMM, "forward: communicator aborted after an earlier failure");
  check_comm("forward");
  simt_gemms_ = 0;
  launches_ = 0;
  comm_bytes_ = 0.0;
  ck(cudaEventRecord(ev_fwd_start_, st), "event");
  tl_mark("forward start", st);

  // --- gating: router GEMM + softmax + top-k + capacity + slots (per source block)
  GatingArgs ga = gating_args(x);
  GatingBuffers gb = gating_buffers();
  if (gate_tc_ && wg_dirty_) {  // router weights changed: refresh the bf16 split + norm bound
    ckr(gate_tc_prepare_device(wg_.p == nullptr ? nullptr : static_cast<const double*>(wg_.p), M_, E_,
                               wg_pieces_.p, static_cast<float*>(wg_nmax_.p), st),
        "gate split");
    ++launches_;
    wg_dirty_ = false;
  }
  prof_mark(kPhGate, true, st);
  ckr(run_gating_device(ga, gb, st), "gating");
  if (cfg_.capacity_kind != MOE_CAP_FIXED) {
    // resolve_capacity over the max demand of all source blocks (run_gating_blocked,
    // gating.cpp:141-148): one all-reduce(max) of E counts, then the host needs the value to
    // size this step's buffers.
    const int32_t* dmax = gb.demand;
    if (W_ > 1) {
      ckn(ncclAllReduce(gb.demand, demand_max_.p, E_, ncclInt32, ncclMax, comm_, st), "allreduce(max)");
      dmax = static_cast<const int32_t*>(demand_max_.p);
    }
    ckr(resolve_capacity_device(dmax, E_, cfg_.capacity_kind, cap_formula_, gb.cap, st), "capacity");
    ck(cudaMemcpyAsync(cap_host_, gb.cap, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "copy");
    sync_comm(st, "sync");
    cap_ = *cap_host_;
    alloc_capacity(cap_);  // collective growth when needed
    gb = gating_buffers();
  }
  prof_mark(kPhGate, false, st);
  f_ = static_cast<double>(cap_) * E_ / (static_cast<double>(k_) * T_);  // capacity_to_factor
  strategy_ = cfg_.adaptive ? strategy_at(search_.choose(f_)) : Strategy{cfg_.a2a_algo, cfg_.degree};
  // 2DH degenerates to the linear algorithm inside one NVSwitch domain (collectives.cpp:58-88
  // with m == W); it is executed as linear and reported as chosen.
  degree_ = W_ == 1 ? 1 : strategy_.degree;
  cc_ = (cap_ + degree_ - 1) / degree_;
  prof_mark(kPhAssign, true, st);
  ckr(run_assign_device(ga, gb, cap_, st), "assign_locations");
  prof_mark(kPhAssign, false, st);
  // gate + column scan + capacity finalize, assign (+ BPR rank), (+ resolve_capacity)
  // gate (+ certified fix-up), capacity scan (+ resolve in its last CTA), assign (+ BPR rank)
  launches_ += 3 + (gate_tc_ ? 1 : 0) + (cfg_.bpr ? 2 : 0) + (cfg_.capacity_kind != MOE_CAP_FIXED ? 1 : 0);

  const bool cert = cfg_.dtype == MOE_DTYPE_BF16;
  if (stats_dirty_) {
    prof_mark(kPhWeightStats, true, st);
    if (cert)
      ckr(weight_stats_device(w1_.p, dE_, M_, V_, static_cast<float*>(colnorm_.p),
                              static_cast<float*>(colnorm_blk_.p), w1t_.p, st),
          "weight stats");
    if (sharded_) refresh_slices(st);
    prof_mark(kPhWeightStats, false, st);
    stats_dirty_ = false;
  }
  // ParallelControl (moe_layer.cpp:184-186): adaptive picks P1 / P2 by the cost model over the
  // gathered capacity W * dC under sharded placement and P1 otherwise; a fixed choice is
  // reported as configured (per-rank placement runs the flex exchange either way, :112-118).
  if (cfg_.parallel != MOE_PARALLEL_ADAPTIVE)
    parallel_ = cfg_.parallel;
  else if (sharded_)
    parallel_ = select_parallelism(1.0 / static_cast<double>(s_), static_cast<int64_t>(W_) * cap_, M_,
                                   8.0 * 2.0 * M_ * V_, s_);
  else
    parallel_ = MOE_PARALLEL_P1;
  const SlotGeom g = geom();
  DropZero yzero;  // fused decode: the encode pass also zeroes the dropped tokens' y rows
  if (fused_) {
    yzero.locations = gb.locations;
    yzero.T = T_;
    yzero.k = k_;
    yzero.out = y;
    yzero.row_bytes = static_cast<size_t>(M_) * esz_;
  }
  LocalDest own;  // peer backend: this rank's experts' rows go straight into its receive buffer
  uint32_t fd_epoch = 0;  // fused dispatch: this forward's channel-0 epoch
  if (peer_) {
    own.recv = recv_.p;
    own.W = W_;
    own.rank = rank_;
    own.dE = dE_;
    if (sender_norms_) own.recv_norm = static_cast<float*>(rownorm_.p);
    if (fused_dispatch_) {
      if (bwd_pending_) {  // inference-style forward: release the previous epoch's buffer first
        peer_->signal_freed(st, 0, epoch_[0]);
        ck(cudaEventRecord(ev_freed_[0], st), "event");
        bwd_pending_ = false;
      }
      fd_epoch = ++epoch_[0];
      own.all_peers = true;
      for (int p = 0; p < W_; ++p) {
        own.peer_recv[p] = peer_->buffer(0, p);
        own.peer_norm[p] = sender_norms_ ? peer_->norms(p) : nullptr;
      }
      own.freed = peer_->freed_wait(0, fd_epoch - 1);
    }
  }
  float* enc_norm = nullptr;  // row norms computed by the encode pass
  if (cert && W_ == 1) enc_norm = static_cast<float*>(rownorm_.p);
  if (peer_ && sender_norms_) enc_norm = static_cast<float*>(znorm_.p);
  prof_mark(kPhEncode, true, st);
  ckr(encode_device(g, cfg_.dtype, x, gb.slot_token, z_.p, st, enc_norm, yzero,
                    (cert && W_ == 1) ? static_cast<unsigned int*>(fix_count_.p) : nullptr, own),
      "encode");
  prof_mark(kPhEncode, false, st);
  ++launches_;
  if (fused_dispatch_)  // every chunk's rows have landed at their owners: publish the flags
    for (int i = 0; i < degree_; ++i) peer_->signal_ready(st, 0, i, fd_epoch);

  const int nseg = degree_ * W_ * dE_;
  GemmArgs up{};
  up.G = dE_;
  up.S = W_;
  up.seg_rows = cc_;
  up.N = V_;
  up.K = M_;
  GemmArgs down = up;
  down.N = M_;
  down.K = V_;
  prepare_up(up);
  auto fixup = [&](void* xin) {
    if (!cert) return;
    prof_mark(kPhReluFix, true, st);
    ckr(relu_fixup_device(xin, w1t_.p, dE_, cc_, M_, V_,
                          static_cast<const unsigned long long*>(fix_list_.p),
                          static_cast<const unsigned int*>(fix_count_.p), fix_cap_, act_.p,
                          static_cast<unsigned long long*>(relu_mask_.p), st),
        "relu_fixup");
    prof_mark(kPhReluFix, false, st);
    ++launches_;
  };

  void* recv = W_ > 1 ? recv_.p : z_.p;
  void* ycomb = W_ > 1 ? ycomb_.p : yexp_.p;
  FlagWait combine_wait;  // peer backend: the combined rows' ready flags, polled by decode
  if (fused_) {
    // decode fused into the down GEMM: y[token] = g * (act . W2)[slot], rows scattered by TMA;
    // tokens without a slot get zero rows (the decode's dropped-token case).
    up.seg_base = 0;
    down.seg_base = 0;
    down.idx_mode = kIdxScatterD | kIdxScaleRow;
    down.gather_rows = static_cast<uint32_t>(T_);
    down.row_token = gb.slot_token;
    down.row_scale = gb.slot_gate;
    prof_mark(kPhUp, true, st);
    gemm(kGemmUp, recv, w1_.p, act_.p, up, nseg, st);
    prof_mark(kPhUp, false, st);
    fixup(recv);
    prof_mark(kPhDown, true, st);
    gemm(kGemmDown, act_.p, w2_.p, y, down, nseg, st);
    prof_mark(kPhDown, false, st);
  } else if (W_ == 1) {
    up.seg_base = 0;
    down.seg_base = 0;
    prof_mark(kPhUp, true, st);
    gemm(kGemmUp, recv, w1_.p, act_.p, up, nseg, st);
    prof_mark(kPhUp, false, st);
    fixup(recv);
    prof_mark(kPhDown, true, st);
    gemm(kGemmDown, act_.p, w2_.p, yexp_.p, down, nseg, st);
    prof_mark(kPhDown, false, st);
  } else if (sharded_) {
    sharded_forward(up, down, cert, st);
  } else if (peer_) {
    if (bwd_pending_ && !fused_dispatch_) {
      // The previous forward was not followed by a backward (inference): its saved expert
      // inputs are dead, so release the receive buffer to the peers now (stream-ordered after
      // that forward's GEMMs).
      peer_->signal_freed(st, 0, epoch_[0]);
      ck(cudaEventRecord(ev_freed_[0], st), "event");
    }
    // Copy engines over NVLink: all dispatches, then all combines (the reference's FIFO order,
    // pipeline.cpp:180-190); each chunk's GEMMs start when its blocks have landed. (Fused
    // dispatch: encode already stored every row at its owner and published the flags.)
    const uint32_t e0 = fused_dispatch_ ? fd_epoch : ++epoch_[0], e1 = ++epoch_[1];
    ck(cudaEventRecord(ev_sync_, st), "event");
    ck(cudaStreamWaitEvent(comm_stream_, ev_sync_, 0), "wait");
    if (!fused_dispatch_) {
      ck(cudaStreamWaitEvent(comm_stream_, ev_freed_[0], 0), "wait");  // my recv buffer consumed
      peer_->wait_peers_freed(comm_stream_, 0, e0);
    }
    prof_mark(kPhA2aFwd, true, comm_stream_);
    // first chunk in row parts when the tile shape allows (tcgen05 path): its first rows land
    // while this rank computes its own segment
    const std::vector<uint32_t> parts0 =
        first_chunk_parts(cc_, local_first_ && fused_combine_ && !fused_dispatch_);
    const bool split0 = parts0.size() > 1;
    for (int i = 0; i < degree_ && !fused_dispatch_; ++i) {
      if (i == 0 && split0) {
        uint32_t r = 0;
        for (size_t p = 0; p < parts0.size(); ++p) {
          const int slot = p + 1 < parts0.size() ? PeerExchange::kPartSlot0 + static_cast<int>(p) : 0;
          peer_push_rows(0, z_.p, 0, 0, slot, r, parts0[p], e0);
          r += parts0[p];
        }
        tl_mark("dispatch pushed 0 (parts) [comm]", comm_stream_);
        continue;
      }
      peer_push(0, z_.p, i, 0, e0, nullptr);  // my own block: written into recv by encode
      tl_mark("dispatch pushed " + std::to_string(i) + " [comm]", comm_stream_);
    }
    // up GEMM over sources [s0, s1) of chunk i except `skip` (-1: none), rows [row0, row0 + nrows)
    // of each segment (nrows 0: to the end); the range's first kernel (the certificate's row
    // norms, or a bare wait) polls the peers' ready flags when `fw` is given
    auto up_range = [&](int i, int s0, int s1, int skip, uint32_t row0, uint32_t nrows,
                        const FlagWait* fw, bool reset) {
      const int nsrc = (s1 - s0) - (skip >= 0 ? 1 : 0);
      if (nsrc <= 0) return;
      GemmArgs u = up;
      u.seg_base = static_cast<uint32_t>(i * W_ + s0);
      u.S = static_cast<uint32_t>(nsrc);
      u.skip_seg = skip >= 0 ? skip - s0 : -1;
      u.row0 = row0;
      u.nrows = nrows;
      if (sender_norms_) {
        // norms arrived with the rows; the GEMM polls the flags itself (fixup resets the count)
        if (fw) u.wait = *fw;
      } else if (cert) {
        RowSet rs;
        rs.seg_begin = static_cast<int64_t>(i * W_ + s0) * dE_;
        rs.nsegs = static_cast<int64_t>(nsrc) * dE_;
        rs.seg_rows = cc_;
        rs.row0 = row0;
        rs.nrows = nrows ? nrows : cc_ - row0;
        if (skip >= 0) {
          rs.skip_begin = static_cast<int64_t>(i * W_ + skip) * dE_;
          rs.skip_count = dE_;
        }
        ckr(rownorm_device(recv, M_, static_cast<float*>(rownorm_.p), rs, st, fw,
                           reset ? static_cast<unsigned int*>(fix_count_.p) : nullptr),
            "rownorm");
        ++launches_;
      } else if (fw) {
        ckr(wait_flags_device(*fw, st), "wait");
        ++launches_;
      }
      if (fw) tl_mark("dispatch landed " + std::to_string(i), st);
      prof_mark(kPhUp, true, st);
      gemm(kGemmUp, recv, w1_.p, act_.p, u, nseg, st);
      prof_mark(kPhUp, false, st);
    };
    for (int i = 0; i < degree_; ++i) {
      const FlagWait fw = peer_->ready_wait(0, i, e0);
      down.seg_base = i * W_;
      if (i == 0 && split0) {
        // own rows first, then the peers' row parts in arrival order (each under its own flag):
        // every transfer hides behind the previous GEMM
        up_range(0, rank_, rank_ + 1, -1, 0, 0, nullptr, true);
        uint32_t r = 0;
        for (size_t p = 0; p < parts0.size(); ++p) {
          const FlagWait fp = p + 1 < parts0.size()
                                  ? peer_->ready_wait(0, PeerExchange::kPartSlot0 + static_cast<int>(p), e0)
                                  : fw;
          up_range(0, 0, W_, rank_, r, p + 1 < parts0.size() ? parts0[p] : 0, &fp, false);
          r += parts0[p];
        }
      } else if (i == 0 && local_first_ && fused_combine_) {
        up_range(0, rank_, rank_ + 1, -1, 0, 0, nullptr, true);
        up_range(0, 0, W_, rank_, 0, 0, &fw, false);
      } else if (i == 0 && local_first_) {  // SIMT GEMM path: contiguous source ranges only
        up_range(0, rank_, rank_ + 1, -1, 0, 0, nullptr, true);
        up_range(0, 0, rank_, -1, 0, 0, &fw, false);
        up_range(0, rank_ + 1, W_, -1, 0, 0, rank_ > 0 ? nullptr : &fw, false);
      } else {
        up_range(i, 0, W_, -1, 0, 0, &fw, true);
      }
      fixup(recv);
      prof_mark(kPhDown, true, st);
      if (fused_combine_) {
        // combine fused into the down GEMM: tiles are stored into the source ranks' ycomb over
        // NVLink as they complete; the chunk's ready flags follow the kernel
        GemmArgs dn = peer_args(down, 1);
        // before its first store into a peer's ycomb, every peer has consumed it (polled inside
        // the GEMM by the epilogue warps)
        if (i == 0) dn.wait = peer_->freed_wait(1, e1 - 1);
        gemm(kGemmDown, act_.p, w2_.p, ycomb, dn, nseg, st);
        peer_->signal_ready(st, 1, i, e1);
        comm_bytes_ += static_cast<double>(dE_) * cc_ * M_ * esz_ * (W_ - 1);
      } else {
        gemm(kGemmDown, act_.p, w2_.p, yexp_.p, down, nseg, st);
      }
      prof_mark(kPhDown, false, st);
      ck(cudaEventRecord(ev_b_[i], st), "event");
    }
    if (!fused_combine_) {
      ck(cudaStreamWaitEvent(comm_stream_, ev_freed_[1], 0), "wait");  // my ycomb consumed
      peer_->wait_peers_freed(comm_stream_, 1, e1);
      for (int i = 0; i < degree_; ++i) {
        ck(cudaStreamWaitEvent(comm_stream_, ev_b_[i], 0), "wait");
        peer_push(1, yexp_.p, i, 1, e1, ev_c_[i]);
        tl_mark("combine pushed " + std::to_string(i) + " [comm]", comm_stream_);
      }
      ck(cudaStreamWaitEvent(st, ev_c_[degree_ - 1], 0), "wait");
    }
    prof_mark(kPhA2aFwd, false, comm_stream_);
    // blocks of one source land in chunk order: the last chunk's flags cover all -- polled by
    // the decode kernel itself
    combine_wait = peer_->ready_wait(1, degree_ - 1, e1);
  } else {
    // Comm stream: all dispatches (chunk order), then all combines (reference FIFO order,
    // pipeline.cpp:180-190); compute stream: per chunk up+down GEMMs.
    ck(cudaEventRecord(ev_sync_, st), "event");
    ck(cudaStreamWaitEvent(comm_stream_, ev_sync_, 0), "wait");
    prof_mark(kPhA2aFwd, true, comm_stream_);
    for (int i = 0; i < degree_; ++i) {
      // chunk i of z: [E][cc][M] at i*E*seg; peer p gets experts [p*dE, (p+1)*dE)
      exchange(z_.p, recv, i, 0);
      ck(cudaEventRecord(ev_a_[i], comm_stream_), "event");
    }
    for (int i = 0; i < degree_; ++i) {
      ck(cudaStreamWaitEvent(st, ev_a_[i], 0), "wait");
      up.seg_base = i * W_;
      down.seg_base = i * W_;
      if (cert) {
        RowSet rs;  // every source segment of chunk i
        rs.seg_begin = static_cast<int64_t>(i) * W_ * dE_;
        rs.nsegs = static_cast<int64_t>(W_) * dE_;
        rs.seg_rows = rs.nrows = cc_;
        ckr(rownorm_device(recv, M_, static_cast<float*>(rownorm_.p), rs, st), "rownorm");
        ++launches_;
        ck(cudaMemsetAsync(fix_count_.p, 0, sizeof(unsigned int), st), "memset");
      }
      prof_mark(kPhUp, true, st);
      gemm(kGemmUp, recv, w1_.p, act_.p, up, nseg, st);
      prof_mark(kPhUp, false, st);
      fixup(recv);
      prof_mark(kPhDown, true, st);
      gemm(kGemmDown, act_.p, w2_.p, yexp_.p, down, nseg, st);
      prof_mark(kPhDown, false, st);
      ck(cudaEventRecord(ev_b_[i], st), "event");
    }
    for (int i = 0; i < degree_; ++i) {
      ck(cudaStreamWaitEvent(comm_stream_, ev_b_[i], 0), "wait");
      exchange(yexp_.p, ycomb, i, 1);
    }
    prof_mark(kPhA2aFwd, false, comm_stream_);
    ck(cudaEventRecord(ev_comm_done_, comm_stream_), "event");
    ck(cudaStreamWaitEvent(st, ev_comm_done_, 0), "wait");
  }
  if (!fused_) {
    prof_mark(kPhDecode, true, st);
    if (k_ == 1 && (static_cast<size_t>(M_) * esz_) % 16 == 0) {
      // slot-major: sequential reads of the combined rows, one row store per kept token
      DropZero dz;
      dz.locations = gb.locations;
      dz.T = T_;
      dz.k = k_;
      dz.out = y;
      dz.row_bytes = static_cast<size_t>(M_) * esz_;
      ckr(slot_scatter_device(g, cfg_.dtype, ycomb, gb.slot_token, gb.slot_gate, y, dz, st,
                              combine_wait.base ? &combine_wait : nullptr),
          "decode");
    } else {
      ckr(decode_device(g, cfg_.dtype, ycomb, gb.idxs, gb.locations, gb.gates, y, st,
                        combine_wait.base ? &combine_wait : nullptr),
          "decode");
    }
    prof_mark(kPhDecode, false, st);
    ++launches_;
  }
  if (peer_) {
    peer_->signal_freed(st, 1, epoch_[1]);
    ck(cudaEventRecord(ev_freed_[1], st), "event");
    bwd_pending_ = true;
  }
  ck(cudaEventRecord(ev_fwd_end_, st), "event");
  fwd_done_ = true;
  metrics_valid_ = false;
  // Alg. 1 feedback (pipeline.cpp:227-237). Measuring needs a host sync (and, for W > 1, an
  // all-reduce so every rank records the same time and picks the same strategy), so it runs
  // while the f bucket is still exploring; once every strategy has a time the controller
  // exploits the argmin without stalling the stream.
  // The first execution of a (f, strategy) pair is not timed: it pays one-off costs (lazy
  // loading of the kernel instantiations only that degree uses, first touches) that the
  // reference's simulated seconds never see. The search then gets one time per candidate, as in
  // the reference, but that time is the fastest of MOE_ADAPT_SAMPLES (default 3) executions:
  // measured at N = 4, single samples of forwards ~4 % apart picked the slower degree about
  // half the time.
  if (cfg_.adaptive && !search_.settled(f_)) {
    static const int samples = [] {
      const char* e = std::getenv("MOE_ADAPT_SAMPLES");
      return e ? std::max(1, std::atoi(e)) : 3;
    }();
    const auto key = std::make_pair(f_, strategy_id(strategy_));
    auto& tr = trials_[key];
    if (tr.first++ == 0) {
      tr.second = std::numeric_limits<double>::infinity();
    } else {
      ck(cudaEventSynchronize(ev_fwd_end_), "event sync");
      float ms = 0.0f;
      ck(cudaEventElapsedTime(&ms, ev_fwd_start_, ev_fwd_end_), "elapsed");
      double sec = ms * 1e-3;
      if (W_ > 1) sec = allreduce_max_host(sec);
      tr.second = std::min(tr.second, sec);
      if (tr.first > samples) search_.record(f_, strategy_id(strategy_), tr.second);
    }
  }
}

// Host wait on a stream whose work includes collectives or peer-flag waits (W > 1). Instead of
// blocking in cudaStreamSynchronize -- which never returns if a peer died mid-exchange -- poll
// the stream and the communicator's asynchronous error state (the analogue of the reference
// fabric's rank-id failure reporting, fabric.cpp:142-160), with a timeout (MOE_COMM_TIMEOUT_S,
// default 300 s). On an NCCL error or the timeout the communicator is aborted and MOE_ECOMM
// names this rank.
void Layer::sync_comm(cudaStream_t s, const char* what) {
  if (W_ == 1 || comm_ == nullptr) {
    ck(cudaStreamSynchronize(s), what);
    return;
  }
  static const double limit_s = [] {
    const char* e = std::getenv("MOE_COMM_TIMEOUT_S");
    return e ? std::atof(e) : 300.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) ck(q, what);
    check_comm(what);
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit_s) {
      ncclCommAbort(comm_);
      comm_ = nullptr;
      throw MoeError(MOE_ECOMM, "rank " + std::to_string(rank_) + ": " + what + ": timed out after " +
                                    std::to_string(static_cast<int>(limit_s)) + " s waiting for peers");
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

void Layer::check_comm(const char* what) {
  if (comm_ == nullptr) return;
  for (ncclComm_t c : {comm_, group_comm_}) {
    if (c == nullptr) continue;
    ncclResult_t r = ncclSuccess;
    ncclCommGetAsyncError(c, &r);
    if (r != ncclSuccess && r != ncclInProgress) {
      if (group_comm_) ncclCommAbort(group_comm_);
      ncclCommAbort(comm_);
      comm_ = nullptr;
      group_comm_ = nullptr;
      throw MoeError(MOE_ECOMM, "rank " + std::to_string(rank_) + ": " + what +
                                    ": NCCL asynchronous error: " + ncclGetErrorString(r));
    }
  }
}

double Layer::allreduce_max_host(double v) {
  DevMem d;
  d.alloc(sizeof(double));
  ck(cudaMemcpy(d.p, &v, sizeof(double), cudaMemcpyHostToDevice), "copy");
  ckn(ncclAllReduce(d.p, d.p, 1, ncclFloat64, ncclMax, comm_, comm_stream_), "allreduce");
  sync_comm(comm_stream_, "sync");
  ck(cudaMemcpy(&v, d.p, sizeof(double), cudaMemcpyDeviceToHost), "copy");
  return v;
}

void Layer::backward(const void* dy, void* dx, float* dw1, float* dw2, cudaStream_t st) {
  if (!fwd_done_) throw MoeError(MOE_ESTATE, "backward: no saved forward");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  if (W_ > 1 && comm_ == nullptr) throw MoeError(MOE_ECOMM, "backward: communicator aborted after an earlier failure");
  check_comm("backward");
  const SlotGeom g = geom();
  GatingBuffers gb = gating_buffers();
  float* gw1 = dw1 ? dw1 : static_cast<float*>(dw1_.p);
  float* gw2 = dw2 ? dw2 : static_cast<float*>(dw2_.p);
  const int64_t l0 = launches_;

  // dZ = decode^T(dy): slot-major gather of g * dy (fast_decode_backward_range)
  DropZero dxzero;  // fused encode-backward: this pass also zeroes the dropped tokens' dx rows
  if (fused_) {
    dxzero.locations = gb.locations;
    dxzero.T = T_;
    dxzero.k = k_;
    dxzero.out = dx;
    dxzero.row_bytes = static_cast<size_t>(M_) * esz_;
  }
  prof_mark(kPhDecodeBwd, true, st);
  LocalDest own;  // peer backend: this rank's experts' dZ rows go straight into drecv
  uint32_t fd_epoch = 0;
  if (peer_) {
    own.recv = drecv_.p;
    own.W = W_;
    own.rank = rank_;
    own.dE = dE_;
    if (fused_dispatch_) {
      fd_epoch = ++epoch_[2];
      own.all_peers = true;
      for (int p = 0; p < W_; ++p) own.peer_recv[p] = peer_->buffer(2, p);
      own.freed = peer_->freed_wait(2, fd_epoch - 1);
    }
  }
  ckr(decode_backward_device(g, cfg_.dtype, dy, gb.slot_token, gb.slot_gate, dz_.p, st, dxzero, own),
      "decode_bwd");
  prof_mark(kPhDecodeBwd, false, st);
  ++launches_;
  if (fused_dispatch_)
    for (int i = 0; i < degree_; ++i) peer_->signal_ready(st, 2, i, fd_epoch);

  const int nseg = degree_ * W_ * dE_;
  GemmArgs dgm{};  // dh = (dY . W2^T) * [a > 0]
  dgm.G = dE_;
  dgm.S = W_;
  dgm.seg_rows = cc_;
  dgm.N = V_;
  dgm.K = M_;
  dgm.aux = act_.p;  // SIMT / fp32 paths read the activation's sign
  dgm.relu_mask = static_cast<unsigned long long*>(relu_mask_.p);  // tcgen05 path: bitmask
  GemmArgs dg = dgm;  // dX = dh . W1^T
  dg.N = M_;
  dg.K = V_;
  dg.aux = nullptr;
  dg.relu_mask = nullptr;
  GemmArgs wg1{};  // dW1 = X^T dh over every (chunk, source) segment
  wg1.G = dE_;
  wg1.S = degree_ * W_;
  wg1.seg_rows = cc_;
  wg1.seg_base = 0;
  wg1.N = V_;
  wg1.Mo = M_;
  GemmArgs wg2 = wg1;  // dW2 = a^T dY
  wg2.N = M_;
  wg2.Mo = V_;

  void* recv = W_ > 1 ? recv_.p : z_.p;
  void* drecv = W_ > 1 ? drecv_.p : dz_.p;
  void* dxcomb = W_ > 1 ? dxcomb_.p : dxe_.p;
  FlagWait combine_wait;  // peer backend: polled by encode_bwd
  if (fused_) {
    // encode-backward fused into the dgrad GEMM: dx[token] = (dh . W1^T)[slot], rows scattered
    // by TMA; dropped tokens get zero rows.
    dg.idx_mode = kIdxScatterD;
    dg.gather_rows = static_cast<uint32_t>(T_);
    dg.row_token = gb.slot_token;
    prof_mark(kPhDgradMask, true, st);
    gemm(kGemmDgradMask, drecv, w2_.p, dh_.p, dgm, nseg, st);
    prof_mark(kPhDgradMask, false, st);
    prof_mark(kPhDgrad, true, st);
    gemm(kGemmDgrad, dh_.p, w1_.p, dx, dg, nseg, st);
    prof_mark(kPhDgrad, false, st);
    prof_mark(kPhWgrad1, true, st);
    gemm(kGemmWgrad, recv, dh_.p, gw1, wg1, nseg, st);
    prof_mark(kPhWgrad1, false, st);
    prof_mark(kPhWgrad2, true, st);
    gemm(kGemmWgrad, act_.p, drecv, gw2, wg2, nseg, st);
    prof_mark(kPhWgrad2, false, st);
  } else if (W_ == 1) {
    prof_mark(kPhDgradMask, true, st);
    gemm(kGemmDgradMask, drecv, w2_.p, dh_.p, dgm, nseg, st);
    prof_mark(kPhDgradMask, false, st);
    prof_mark(kPhDgrad, true, st);
    gemm(kGemmDgrad, dh_.p, w1_.p, dxe_.p, dg, nseg, st);
    prof_mark(kPhDgrad, false, st);
    prof_mark(kPhWgrad1, true, st);
    gemm(kGemmWgrad, recv, dh_.p, gw1, wg1, nseg, st);
    prof_mark(kPhWgrad1, false, st);
    prof_mark(kPhWgrad2, true, st);
    gemm(kGemmWgrad, act_.p, drecv, gw2, wg2, nseg, st);
    prof_mark(kPhWgrad2, false, st);
  } else if (sharded_) {
    sharded_backward(dgm, dg, wg1, wg2, gw1, gw2, st);
  } else if (peer_) {
    const uint32_t e2 = fused_dispatch_ ? fd_epoch : ++epoch_[2], e3 = ++epoch_[3];
    ck(cudaEventRecord(ev_sync_, st), "event");
    ck(cudaStreamWaitEvent(comm_stream_, ev_sync_, 0), "wait");
    if (!fused_dispatch_) {
      ck(cudaStreamWaitEvent(comm_stream_, ev_freed_[2], 0), "wait");
      peer_->wait_peers_freed(comm_stream_, 2, e2);
    }
    prof_mark(kPhA2aBwd, true, comm_stream_);
    const std::vector<uint32_t> parts0 =
        first_chunk_parts(cc_, local_first_ && fused_combine_ && !fused_dispatch_);
    const bool split0 = parts0.size() > 1;  // as in forward
    for (int i = 0; i < degree_ && !fused_dispatch_; ++i) {  // adjoint of combine
      if (i == 0 && split0) {
        uint32_t r = 0;
        for (size_t p = 0; p < parts0.size(); ++p) {
          const int slot = p + 1 < parts0.size() ? PeerExchange::kPartSlot0 + static_cast<int>(p) : 0;
          peer_push_rows(2, dz_.p, 0, 0, slot, r, parts0[p], e2);
          r += parts0[p];
        }
        tl_mark("bwd dispatch pushed 0 (parts) [comm]", comm_stream_);
        continue;
      }
      peer_push(2, dz_.p, i, 0, e2, nullptr);  // my own block: written into drecv by decode_bwd
      tl_mark("bwd dispatch pushed " + std::to_string(i) + " [comm]", comm_stream_);
    }
    for (int i = 0; i < degree_; ++i) {
      const FlagWait fw = peer_->ready_wait(2, i, e2);
      dg.seg_base = i * W_;
      // dgrad-mask over sources [s0, s1) except `skip`, rows [row0, row0 + nrows) of each segment
      auto dgm_range = [&](int s0, int s1, int skip, uint32_t row0, uint32_t nrows, const FlagWait* w) {
        const int nsrc = (s1 - s0) - (skip >= 0 ? 1 : 0);
        if (nsrc <= 0) return;
        GemmArgs a = dgm;
        if (w && fused_combine_) {
          a.wait = *w;  // tcgen05 path: the receive wait runs inside the GEMM
        } else if (w) {
          ckr(wait_flags_device(*w, st), "wait");
          ++launches_;
          tl_mark("bwd dispatch landed " + std::to_string(i), st);
        }
        a.seg_base = static_cast<uint32_t>(i * W_ + s0);
        a.S = static_cast<uint32_t>(nsrc);
        a.skip_seg = skip >= 0 ? skip - s0 : -1;
        a.row0 = row0;
        a.nrows = nrows;
        prof_mark(kPhDgradMask, true, st);
        gemm(kGemmDgradMask, drecv, w2_.p, dh_.p, a, nseg, st);
        prof_mark(kPhDgradMask, false, st);
      };
      if (i == 0 && split0) {
        dgm_range(rank_, rank_ + 1, -1, 0, 0, nullptr);
        uint32_t r = 0;
        for (size_t p = 0; p < parts0.size(); ++p) {
          const FlagWait fp = p + 1 < parts0.size()
                                  ? peer_->ready_wait(2, PeerExchange::kPartSlot0 + static_cast<int>(p), e2)
                                  : fw;
          dgm_range(0, W_, rank_, r, p + 1 < parts0.size() ? parts0[p] : 0, &fp);
          r += parts0[p];
        }
      } else if (i == 0 && local_first_ && fused_combine_) {
        dgm_range(rank_, rank_ + 1, -1, 0, 0, nullptr);
        dgm_range(0, W_, rank_, 0, 0, &fw);
      } else if (i == 0 && local_first_) {  // SIMT GEMM path: contiguous source ranges only
        dgm_range(rank_, rank_ + 1, -1, 0, 0, nullptr);
        dgm_range(0, rank_, -1, 0, 0, &fw);
        dgm_range(rank_ + 1, W_, -1, 0, 0, rank_ == 0 ? &fw : nullptr);
      } else {
        dgm_range(0, W_, -1, 0, 0, &fw);
      }
      prof_mark(kPhDgrad, true, st);
      if (fused_combine_) {
        // backward combine fused into the dgrad GEMM (dx blocks straight to the source ranks)
        GemmArgs d2 = peer_args(dg, 3);
        if (i == 0) d2.wait = peer_->freed_wait(3, e3 - 1);
        gemm(kGemmDgrad, dh_.p, w1_.p, dxcomb, d2, nseg, st);
        peer_->signal_ready(st, 3, i, e3);
        comm_bytes_ += static_cast<double>(dE_) * cc_ * M_ * esz_ * (W_ - 1);
      } else {
        gemm(kGemmDgrad, dh_.p, w1_.p, dxe_.p, dg, nseg, st);
      }
      prof_mark(kPhDgrad, false, st);
      ck(cudaEventRecord(ev_b_[i], st), "event");
    }
    if (!fused_combine_) {
      ck(cudaStreamWaitEvent(comm_stream_, ev_freed_[3], 0), "wait");
      peer_->wait_peers_freed(comm_stream_, 3, e3);
      for (int i = 0; i < degree_; ++i) {  // adjoint of dispatch
        ck(cudaStreamWaitEvent(comm_stream_, ev_b_[i], 0), "wait");
        peer_push(3, dxe_.p, i, 1, e3, ev_c_[i]);
        tl_mark("bwd combine pushed " + std::to_string(i) + " [comm]", comm_stream_);
      }
    }
    prof_mark(kPhA2aBwd, false, comm_stream_);
    // Weight gradients overlap the return transfers; then the receive buffers are released.
    prof_mark(kPhWgrad1, true, st);
    gemm(kGemmWgrad, recv, dh_.p, gw1, wg1, nseg, st);
    prof_mark(kPhWgrad1, false, st);
    peer_->signal_freed(st, 0, epoch_[0]);
    ck(cudaEventRecord(ev_freed_[0], st), "event");
    bwd_pending_ = false;
    prof_mark(kPhWgrad2, true, st);
    gemm(kGemmWgrad, act_.p, drecv, gw2, wg2, nseg, st);
    prof_mark(kPhWgrad2, false, st);
    peer_->signal_freed(st, 2, e2);
    ck(cudaEventRecord(ev_freed_[2], st), "event");
    if (!fused_combine_) ck(cudaStreamWaitEvent(st, ev_c_[degree_ - 1], 0), "wait");
    combine_wait = peer_->ready_wait(3, degree_ - 1, e3);  // polled by the encode_bwd kernel
  } else {
    ck(cudaEventRecord(ev_sync_, st), "event");
    ck(cudaStreamWaitEvent(comm_stream_, ev_sync_, 0), "wait");
    prof_mark(kPhA2aBwd, true, comm_stream_);
    for (int i = 0; i < degree_; ++i) {  // adjoint of combine
      exchange(dz_.p, drecv, i, 0);
      ck(cudaEventRecord(ev_a_[i], comm_stream_), "event");
    }
    for (int i = 0; i < degree_; ++i) {
      ck(cudaStreamWaitEvent(st, ev_a_[i], 0), "wait");
      dgm.seg_base = i * W_;
      dg.seg_base = i * W_;
      prof_mark(kPhDgradMask, true, st);
      gemm(kGemmDgradMask, drecv, w2_.p, dh_.p, dgm, nseg, st);
      prof_mark(kPhDgradMask, false, st);
      prof_mark(kPhDgrad, true, st);
      gemm(kGemmDgrad, dh_.p, w1_.p, dxe_.p, dg, nseg, st);
      prof_mark(kPhDgrad, false, st);
      ck(cudaEventRecord(ev_b_[i], st), "event");
    }
    for (int i = 0; i < degree_; ++i) {  // adjoint of dispatch
      ck(cudaStreamWaitEvent(comm_stream_, ev_b_[i], 0), "wait");
      exchange(dxe_.p, dxcomb, i, 1);
    }
    prof_mark(kPhA2aBwd, false, comm_stream_);
    ck(cudaEventRecord(ev_comm_done_, comm_stream_), "event");
    // Weight gradients overlap the last return exchanges.
    prof_mark(kPhWgrad1, true, st);
    gemm(kGemmWgrad, recv, dh_.p, gw1, wg1, nseg, st);
    prof_mark(kPhWgrad1, false, st);
    prof_mark(kPhWgrad2, true, st);
    gemm(kGemmWgrad, act_.p, drecv, gw2, wg2, nseg, st);
    prof_mark(kPhWgrad2, false, st);
    ck(cudaStreamWaitEvent(st, ev_comm_done_, 0), "wait");
  }
  if (!fused_) {
    prof_mark(kPhEncodeBwd, true, st);
    if (k_ == 1 && (static_cast<size_t>(M_) * esz_) % 16 == 0) {
      DropZero dz;
      dz.locations = gb.locations;
      dz.T = T_;
      dz.k = k_;
      dz.out = dx;
      dz.row_bytes = static_cast<size_t>(M_) * esz_;
      ckr(slot_scatter_device(g, cfg_.dtype, dxcomb, gb.slot_token, nullptr, dx, dz, st,
                              combine_wait.base ? &combine_wait : nullptr),
          "encode_bwd");
    } else {
      ckr(encode_backward_device(g, cfg_.dtype, dxcomb, gb.idxs, gb.locations, dx, st,
                                 combine_wait.base ? &combine_wait : nullptr),
          "encode_bwd");
    }
    prof_mark(kPhEncodeBwd, false, st);
    ++launches_;
  }
  if (peer_) {
    peer_->signal_freed(st, 3, epoch_[3]);
    ck(cudaEventRecord(ev_freed_[3], st), "event");
  }
  bwd_launches_ = launches_ - l0;
  tl_mark("backward end", st);
  tl_flush();
  last_dw1_ = gw1;
  last_dw2_ = gw2;
}

// reduce_scatter_grads_p1 (parallelism.cpp:235-286), per-rank placement: rank q receives slice
// q (dW1 columns / dW2 rows [q*h, (q+1)*h), h = V/W) of every expert's gradient from the rank that
// computed it -- pure routing, no sums. Output (device fp32): w1s [E][M][h], w2s [E][h][M].
void Layer::grad_slices(float* w1s, float* w2s, cudaStream_t st) {
  if (!last_dw1_) throw MoeError(MOE_ESTATE, "grad_slices: no backward yet");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  if (sharded_) {
    // reduce_scatter_grads_p1, sharded (parallelism.cpp:247-262): the summed gradient of slice
    // rank%s of expert rank/s -- already reduced over the group by backward.
    const int h = V_ / s_, q = rank_ % s_;
    ck(cudaMemcpy2DAsync(w1s, sizeof(float) * h, last_dw1_ + static_cast<size_t>(q) * h,
                         sizeof(float) * V_, sizeof(float) * h, M_, cudaMemcpyDeviceToDevice, st),
       "dW1 slice");
    ck(cudaMemcpyAsync(w2s, last_dw2_ + static_cast<size_t>(q) * h * M_, sizeof(float) * h * M_,
                       cudaMemcpyDeviceToDevice, st),
       "dW2 slice");
    sync_comm(st, "sync");
    return;
  }
  const int h = V_ / W_;
  const size_t blk1 = static_cast<size_t>(dE_) * M_ * h;  // floats per (dst) block, each of w1/w2
  DevMem pack;
  pack.alloc(sizeof(float) * blk1 * 2 * W_);
  float* p1 = static_cast<float*>(pack.p);
  float* p2 = p1 + blk1 * W_;
  for (int q = 0; q < W_; ++q)
    for (int i = 0; i < dE_; ++i) {
      // dW1[i][:, q*h:(q+1)*h] -> p1[q][i] (M x h): strided 2-D copy
      ck(cudaMemcpy2DAsync(p1 + (static_cast<size_t>(q) * dE_ + i) * M_ * h, sizeof(float) * h,
                           last_dw1_ + static_cast<size_t>(i) * M_ * V_ + static_cast<size_t>(q) * h,
                           sizeof(float) * V_, sizeof(float) * h, M_, cudaMemcpyDeviceToDevice, st),
         "pack dW1 slice");
      // dW2[i][q*h:(q+1)*h, :] -> p2[q][i] (h x M): contiguous rows
      ck(cudaMemcpyAsync(p2 + (static_cast<size_t>(q) * dE_ + i) * h * M_,
                         last_dw2_ + static_cast<size_t>(i) * V_ * M_ + static_cast<size_t>(q) * h * M_,
                         sizeof(float) * h * M_, cudaMemcpyDeviceToDevice, st),
         "pack dW2 slice");
    }
  if (W_ == 1) {
    ck(cudaMemcpyAsync(w1s, p1, sizeof(float) * blk1, cudaMemcpyDeviceToDevice, st), "copy");
    ck(cudaMemcpyAsync(w2s, p2, sizeof(float) * blk1, cudaMemcpyDeviceToDevice, st), "copy");
  } else {
    // block from rank p holds experts [p*dE, (p+1)*dE): contiguous in the [E][..] outputs
    ckn(ncclGroupStart(), "group");
    for (int p = 0; p < W_; ++p) {
      ckn(ncclSend(p1 + static_cast<size_t>(p) * blk1, blk1, ncclFloat32, p, comm_, st), "send");
      ckn(ncclRecv(w1s + static_cast<size_t>(p) * blk1, blk1, ncclFloat32, p, comm_, st), "recv");
      ckn(ncclSend(p2 + static_cast<size_t>(p) * blk1, blk1, ncclFloat32, p, comm_, st), "send");
      ckn(ncclRecv(w2s + static_cast<size_t>(p) * blk1, blk1, ncclFloat32, p, comm_, st), "recv");
    }
    ckn(ncclGroupEnd(), "group");
  }
  sync_comm(st, "sync");  // the pack buffer is freed on return
}

void Layer::ensure_io() {
  const size_t n = static_cast<size_t>(T_) * M_ * esz_;
  io_x_.alloc(n);
  io_y_.alloc(n);
  io_dy_.alloc(n);
  io_dx_.alloc(n);
}

void Layer::forward_host(const void* xh, void* yh, cudaStream_t st) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  ensure_io();
  const size_t n = static_cast<size_t>(T_) * M_ * esz_;
  ck(cudaMemcpyAsync(io_x_.p, xh, n, cudaMemcpyHostToDevice, st), "h2d x");
  forward(io_x_.p, io_y_.p, st);
  ck(cudaMemcpyAsync(yh, io_y_.p, n, cudaMemcpyDeviceToHost, st), "d2h y");
  sync_comm(st, "sync");
}

void Layer::backward_host(const void* dyh, void* dxh, cudaStream_t st) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  ensure_io();
  const size_t n = static_cast<size_t>(T_) * M_ * esz_;
  ck(cudaMemcpyAsync(io_dy_.p, dyh, n, cudaMemcpyHostToDevice, st), "h2d dy");
  backward(io_dy_.p, io_dx_.p, nullptr, nullptr, st);
  ck(cudaMemcpyAsync(dxh, io_dx_.p, n, cudaMemcpyDeviceToHost, st), "d2h dx");
  sync_comm(st, "sync");
}

// Host <-> device staging copy, issued in pieces of host_chunk_ bytes (MOE_HOST_CHUNK_MB; 0 =
// one copy) so that latency-critical peer pushes sharing a copy engine wait for one piece at
// most, not for a whole multi-MiB step input.
void Layer::host_copy(void* dst, const void* src, size_t n, cudaMemcpyKind kind, cudaStream_t st) {
  const size_t piece = host_chunk_ ? host_chunk_ : n;
  for (size_t o = 0; o < n; o += piece)
    ck(cudaMemcpyAsync(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o,
                       std::min(piece, n - o), kind, st),
       "host copy");
}

void Layer::pipe_call(int dir, const void* inh, void* outh, cudaStream_t st) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  const size_t n = static_cast<size_t>(T_) * M_ * esz_;
  HostPipe& p = pipe_[dir];
  if (!h2d_) {
    ck(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking), "stream");
  }
  if (!p.in_ready[0]) {
    for (int i = 0; i < 2; ++i) {
      p.in[i].alloc(n);
      p.out[i].alloc(n);
      for (cudaEvent_t* e : {&p.in_ready[i], &p.in_free[i], &p.out_ready[i], &p.out_free[i]})
        ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    }
  }
  const int s = p.slot;
  p.slot ^= 1;
  // upload once the call that last read this staging buffer is done with it
  ck(cudaStreamWaitEvent(h2d_, p.in_free[s], 0), "wait");
  const char* tag = dir == 0 ? "fwd" : "bwd";
  pipe_mark(std::string(tag) + " h2d >", h2d_);
  host_copy(p.in[s].p, inh, n, cudaMemcpyHostToDevice, h2d_);
  pipe_mark(std::string(tag) + " h2d <", h2d_);
  ck(cudaEventRecord(p.in_ready[s], h2d_), "event");
  ck(cudaStreamWaitEvent(st, p.in_ready[s], 0), "wait");
  ck(cudaStreamWaitEvent(st, p.out_free[s], 0), "wait");
  pipe_mark(std::string(tag) + " compute >", st);
  if (dir == 0)
    forward(p.in[s].p, p.out[s].p, st);
  else
    backward(p.in[s].p, p.out[s].p, nullptr, nullptr, st);
  pipe_mark(std::string(tag) + " compute <", st);
  ck(cudaEventRecord(p.in_free[s], st), "event");
  ck(cudaEventRecord(p.out_ready[s], st), "event");
  ck(cudaStreamWaitEvent(d2h_, p.out_ready[s], 0), "wait");
  pipe_mark(std::string(tag) + " d2h >", d2h_);
  host_copy(outh, p.out[s].p, n, cudaMemcpyDeviceToHost, d2h_);
  pipe_mark(std::string(tag) + " d2h <", d2h_);
  ck(cudaEventRecord(p.out_free[s], d2h_), "event");
}

// MOE_PIPE_TIMELINE=1 (debug): events on the staging-copy and compute streams of the pipelined
// host calls, printed (ms from the first) by host_sync -- no synchronisation in between.
void Layer::pipe_mark(const std::string& name, cudaStream_t st) {
  if (!pipe_tl_on_) return;
  cudaEvent_t e;
  ck(cudaEventCreateWithFlags(&e, cudaEventDefault), "event");
  ck(cudaEventRecord(e, st), "event");
  pipe_tl_.emplace_back(name, e);
}

void Layer::forward_host_async(const void* xh, void* yh, cudaStream_t st) { pipe_call(0, xh, yh, st); }
void Layer::backward_host_async(const void* dyh, void* dxh, cudaStream_t st) { pipe_call(1, dyh, dxh, st); }

void Layer::host_sync() {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  if (d2h_) ck(cudaStreamSynchronize(d2h_), "sync");
  if (h2d_) ck(cudaStreamSynchronize(h2d_), "sync");
  if (!pipe_tl_.empty()) {
    ck(cudaDeviceSynchronize(), "sync");
    for (auto& [nm, e] : pipe_tl_) {
      float t = 0.0f;
      ck(cudaEventElapsedTime(&t, pipe_tl_.front().second, e), "elapsed");
      std::fprintf(stderr, "[pipe r%d] %9.3f ms  %s\n", rank_, t, nm.c_str());
    }
    for (auto& pe : pipe_tl_) cudaEventDestroy(pe.second);
    pipe_tl_.clear();
  }
}

void Layer::get_routing(int32_t* idxs, int32_t* locs, double* gates, int64_t* capacity) {
  if (!fwd_done_) throw MoeError(MOE_ESTATE, "get_routing: no forward yet");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  ck(cudaDeviceSynchronize(), "sync");
  check_gate_error();
  const size_t Tk = static_cast<size_t>(T_) * k_;
  if (idxs) ck(cudaMemcpy(idxs, idxs_.p, 4 * Tk, cudaMemcpyDeviceToHost), "copy");
  if (locs) ck(cudaMemcpy(locs, locs_.p, 4 * Tk, cudaMemcpyDeviceToHost), "copy");
  if (gates) ck(cudaMemcpy(gates, gates_.p, 8 * Tk, cudaMemcpyDeviceToHost), "copy");
  if (capacity) *capacity = cap_;
}

void Layer::get_metrics(moe_step_metrics* m) {
  if (!fwd_done_) throw MoeError(MOE_ESTATE, "get_metrics: no forward yet");
  ck(cudaSetDevice(device_), "cudaSetDevice");
  ck(cudaEventSynchronize(ev_fwd_end_), "sync");
  check_gate_error();
  float ms = 0.0f;
  ck(cudaEventElapsedTime(&ms, ev_fwd_start_, ev_fwd_end_), "elapsed");
  int32_t drops = 0;
  ck(cudaMemcpy(&drops, drops_.p, 4, cudaMemcpyDeviceToHost), "copy");
  m->f = f_;
  m->capacity = cap_;
  m->a2a_algo = strategy_.algo;
  m->degree = strategy_.degree;
  m->seconds = ms * 1e-3;
  m->comm_bytes = comm_bytes_;
  m->drop_count = drops;
  m->relu_fixups = 0;
  m->fused = (fused_ ? MOE_FUSED_DECODE : 0) | (peer_ && fused_combine_ ? MOE_FUSED_COMBINE : 0);
  m->parallel = parallel_;
  m->gate_fixups = 0;
  m->simt_gemms = simt_gemms_;  // since the last forward began: that forward + its backward
  if (gate_tc_) {
    int32_t nf = 0;
    ck(cudaMemcpy(&nf, gate_fix_.p, 4, cudaMemcpyDeviceToHost), "copy");
    ck(cudaMemset(gate_fix_.p, 0, 4), "memset");
    m->gate_fixups = nf;
  }
  if (cfg_.dtype == MOE_DTYPE_BF16) {
    // [2]: the last fixup's list size; [3]: the largest list of any fixup since the last read
    // (an overflow in an earlier chunk or source range must not be masked by a later one)
    unsigned int c[2] = {0u, 0u};
    ck(cudaMemcpy(c, static_cast<unsigned int*>(fix_count_.p) + 2, 8, cudaMemcpyDeviceToHost), "copy");
    ck(cudaMemset(static_cast<unsigned int*>(fix_count_.p) + 3, 0, 4), "memset");
    m->relu_fixups = c[0];
    if (c[1] > fix_cap_) throw MoeError(MOE_ESTATE, "ReLU-mask certificate list overflowed");
  }
}

void Layer::get_grads(float* dw1, float* dw2) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  if (!last_dw1_ || !last_dw2_) throw MoeError(MOE_ESTATE, "expert grads: no backward yet");
  ck(cudaDeviceSynchronize(), "sync");
  const size_t n = static_cast<size_t>(dE_) * M_ * V_;
  // the last backward's gradients, wherever they went (internal or caller-supplied buffers)
  if (dw1) ck(cudaMemcpy(dw1, last_dw1_, 4 * n, cudaMemcpyDeviceToHost), "copy");
  if (dw2) ck(cudaMemcpy(dw2, last_dw2_, 4 * n, cudaMemcpyDeviceToHost), "copy");
}

void Layer::set_kernel_spans(bool on) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  constexpr size_t kMaxSpans = 4096;
  if (on && kspan_.p == nullptr) kspan_.alloc(sizeof(unsigned long long) * 4 * kMaxSpans);
  if (on) {
    ck(cudaDeviceSynchronize(), "sync");
    std::vector<unsigned long long> init(4 * kMaxSpans, 0ull);
    for (size_t i = 0; i < kMaxSpans; ++i) init[4 * i] = ~0ull;
    ck(cudaMemcpy(kspan_.p, init.data(), init.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice),
       "span init");
  }
  kspan_phase_.clear();
  kspan_on_ = on;
}

void Layer::take_kernel_spans(double* ms, int64_t* counts, int n) {
  ck(cudaSetDevice(device_), "cudaSetDevice");
  for (int i = 0; i < n; ++i) {
    ms[i] = 0.0;
    counts[i] = 0;
  }
  if (kspan_phase_.empty()) return;
  ck(cudaDeviceSynchronize(), "sync");
  std::vector<unsigned long long> h(4 * kspan_phase_.size());
  ck(cudaMemcpy(h.data(), kspan_.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "copy");
  double cyc = 0.0, nsec = 0.0;
  for (size_t i = 0; i < kspan_phase_.size(); ++i) {
    const int ph = kspan_phase_[i];
    if (ph < 0 || ph >= n || h[4 * i + 1] < h[4 * i]) continue;
    ms[ph] += static_cast<double>(h[4 * i + 1] - h[4 * i]) * 1e-6;
    counts[ph] += 1;
    cyc += static_cast<double>(h[4 * i + 2]);
    nsec += static_cast<double>(h[4 * i + 3]);
  }
  span_mhz_ = nsec > 0.0 ? cyc / nsec * 1e3 : 0.0;
  set_kernel_spans(kspan_on_);  // re-arm (clears the records)
}

}  // namespace moe
