// extern "C" boundary (include/moe_b200.h). Exceptions never cross it: every entry point maps
// MoeError codes / std exceptions onto MOE_* status codes and keeps the message.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "layer.h"

struct moe_handle {
  std::unique_ptr<moe::Layer> layer;
  std::string err;
};

struct moe_memo {
  moe::StrategySearch search;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guard(std::string* err, F&& f) {
  try {
    f();
    return MOE_OK;
  } catch (const moe::MoeError& e) {
    if (err) *err = e.what();
    g_err = e.what();
    return e.code;
  } catch (const std::invalid_argument& e) {
    if (err) *err = e.what();
    g_err = e.what();
    return MOE_EINVAL;
  } catch (const std::logic_error& e) {
    if (err) *err = e.what();
    g_err = e.what();
    return MOE_ESTATE;
  } catch (const std::bad_alloc& e) {
    if (err) *err = "out of memory";
    g_err = "out of memory";
    return MOE_ENOMEM;
  } catch (const std::exception& e) {
    if (err) *err = e.what();
    g_err = e.what();
    return MOE_ECUDA;
  }
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw moe::MoeError(MOE_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void ckr(int rc, const char* what) {
  if (rc == -1) throw moe::MoeError(MOE_EINVAL, std::string(what) + ": invalid arguments");
  if (rc != 0) {
    cudaError_t e = moe::last_launch_error();
    moe::last_launch_error() = cudaSuccess;
    throw moe::MoeError(MOE_ECUDA, std::string(what) + ": launch failed (" +
                                       cudaGetErrorString(e) + ")");
  }
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1)
    throw moe::MoeError(MOE_ECUDA, "no CUDA device (the MoE kernels have no CPU fallback)");
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// Stream-ordered scratch allocation for the stateless ops.
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <typename T>
  T* get(size_t n) {
    void* p = nullptr;
    ck(cudaMallocAsync(&p, n * sizeof(T) + 16, st), "cudaMallocAsync");
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

bool tc_shape_ok(int kind, const moe::GemmArgs& a) {
  if (a.N % 256 != 0) return false;
  if (kind == moe::kGemmWgrad) return a.Mo % 128 == 0;
  return a.K % 64 == 0;
}

int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

void expert_gemm(int kind, int dtype, int use_tc, const void* A, const void* B, void* D,
                 const moe::GemmArgs& a, int nseg, cudaStream_t st) {
  int rc;
  if (dtype == MOE_DTYPE_F32) {
    if (use_tc == 1) throw moe::MoeError(MOE_EINVAL, "tcgen05 GEMM is bf16-only");
    rc = moe::gemm_f32(kind, static_cast<const float*>(A), static_cast<const float*>(B),
                       static_cast<float*>(D), a, st);
  } else if (use_tc == 1 || (use_tc < 0 && tc_shape_ok(kind, a))) {
    if (!tc_shape_ok(kind, a)) throw moe::MoeError(MOE_EINVAL, "shape not tcgen05-tileable");
    rc = moe::gemm_fwd(static_cast<moe::GemmKind>(kind), A, B, D, a, nseg, num_sms(), st);
  } else {
    rc = moe::gemm_bf16_simt(kind, A, B, D, a, st);
  }
  ckr(rc, "gemm");
}

// Up-projection with the ReLU-mask certificate on the bf16 path (see relu_fix.cu).
// Returns the ReLU bitmask (bf16 path) for a following kGemmDgradMask.
unsigned long long* certified_up(int dtype, const void* x, const void* w1, void* act,
                                 moe::GemmArgs up, int64_t n, int64_t rows, int64_t M, int64_t V,
                                 cudaStream_t st, Scratch& sc) {
  if (dtype != MOE_DTYPE_BF16) {
    expert_gemm(moe::kGemmUp, dtype, -1, x, w1, act, up, static_cast<int>(n), st);
    return nullptr;
  }
  float* colnorm = sc.get<float>(static_cast<size_t>(n) * V);
  float* colnorm_blk = sc.get<float>(static_cast<size_t>(n) * (V / 64 + 1));
  auto* mask = sc.get<unsigned long long>(moe::relu_mask_words(static_cast<size_t>(n) * rows, (V + 63) / 64));
  void* w1t = sc.get<char>(static_cast<size_t>(n) * M * V * 2);
  float* rownorm = sc.get<float>(static_cast<size_t>(n) * rows);
  const unsigned int cap =
      static_cast<unsigned int>(std::max<int64_t>(1 << 16, n * rows * V / 256));
  auto* list = sc.get<unsigned long long>(cap);
  auto* count = sc.get<unsigned int>(4);  // list size, fixup CTAs done, last / largest list size
  ckr(moe::weight_stats_device(w1, static_cast<int>(n), static_cast<int>(M), static_cast<int>(V),
                               colnorm, colnorm_blk, w1t, st),
      "weight stats");
  moe::RowSet all;
  all.nsegs = 1;
  all.seg_rows = all.nrows = n * rows;
  ckr(moe::rownorm_device(x, static_cast<int>(M), rownorm, all, st), "rownorm");
  ck(cudaMemsetAsync(count, 0, 4 * sizeof(unsigned int), st), "memset");
  up.rownorm = rownorm;
  up.colnorm = colnorm;
  up.colnorm_blk = colnorm_blk;
  up.relu_mask = mask;
  up.fix_list = list;
  up.fix_count = count;
  up.fix_cap = cap;
  expert_gemm(moe::kGemmUp, dtype, -1, x, w1, act, up, static_cast<int>(n), st);
  ckr(moe::relu_fixup_device(x, w1t, static_cast<int>(n), static_cast<int>(rows),
                             static_cast<int>(M), static_cast<int>(V), list, count, cap, act, mask,
                             st),
      "relu_fixup");
  return mask;
}

moe::SlotGeom make_geom(int64_t blocks, int64_t T, int64_t M, int64_t E, int64_t k, int64_t cap,
                        int64_t degree) {
  if (blocks < 1 || T < 1 || M < 1 || E < 1 || k < 1 || k > E || cap < 1 || degree < 1)
    throw moe::MoeError(MOE_EINVAL, "dispatch: invalid geometry");
  moe::SlotGeom g{};
  g.blocks = static_cast<int>(blocks);
  g.T = static_cast<int>(T);
  g.M = static_cast<int>(M);
  g.E = static_cast<int>(E);
  g.k = static_cast<int>(k);
  g.cap = static_cast<int>(cap);
  g.degree = static_cast<int>(degree);
  g.cc = static_cast<int>((cap + degree - 1) / degree);
  return g;
}

void check_dtype(int32_t d) {
  if (d != MOE_DTYPE_BF16 && d != MOE_DTYPE_F32) throw moe::MoeError(MOE_EINVAL, "dtype");
}

}  // namespace

extern "C" {

int moe_expert_capacity(int64_t k, double f, int64_t tokens, int64_t experts, int64_t* out) {
  return guard(nullptr, [&] { *out = moe::expert_capacity(k, f, tokens, experts); });
}

int moe_resolve_capacity(int32_t kind, double factor, const int64_t* demand, int64_t experts,
                         int64_t top_k, int64_t tokens, int64_t* out) {
  return guard(nullptr, [&] {
    if (!demand || experts < 1) throw moe::MoeError(MOE_EINVAL, "resolve_capacity: demand must have E entries");
    int64_t mx = 1;
    for (int64_t e = 0; e < experts; ++e) mx = std::max(mx, demand[e]);
    if (kind == MOE_CAP_FIXED)
      *out = moe::expert_capacity(top_k, factor, tokens, experts);
    else if (kind == MOE_CAP_AUTO)
      *out = mx;
    else if (kind == MOE_CAP_BOUNDED)
      *out = std::min(mx, moe::expert_capacity(top_k, factor, tokens, experts));
    else
      throw moe::MoeError(MOE_EINVAL, "capacity kind");
  });
}

int moe_capacity_to_factor(int64_t capacity, int64_t experts, int64_t top_k, int64_t tokens,
                           double* out) {
  return guard(nullptr, [&] {
    if (top_k < 1 || tokens < 1) throw moe::MoeError(MOE_EINVAL, "capacity_to_factor");
    *out = static_cast<double>(capacity) * static_cast<double>(experts) /
           (static_cast<double>(top_k) * static_cast<double>(tokens));
  });
}

int moe_a2a_plan(int64_t W, int64_t E, int64_t cc, int64_t M, int64_t chunk, int32_t phase,
                 int64_t* send_off, int64_t* recv_off, int64_t* elems) {
  return guard(nullptr, [&] {
    if (W < 1 || E < 1 || E % W != 0 || cc < 1 || M < 1 || chunk < 0 || (phase != 0 && phase != 1))
      throw moe::MoeError(MOE_EINVAL, "flex_all2all: expert axis not divisible by W");
    moe::a2a_plan(W, E, cc, M, chunk, phase, send_off, recv_off, elems);
  });
}

int moe_validate_config(const moe_config* cfg) {
  return guard(nullptr, [&] {
    if (!cfg) throw moe::MoeError(MOE_EINVAL, "null config");
    moe::validate(*cfg);
  });
}

int moe_select_parallelism(double local_experts, int64_t gathered_capacity, int64_t model_dim,
                           double param_bytes, int64_t n_sharded, int32_t* out) {
  return guard(nullptr, [&] {
    if (!out) throw moe::MoeError(MOE_EINVAL, "null output");
    *out = moe::select_parallelism(local_experts, gathered_capacity, model_dim, param_bytes, n_sharded);
  });
}

int moe_get_unique_id(uint8_t* id128) {
  return guard(nullptr, [&] {
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) throw moe::MoeError(MOE_ECOMM, "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "nccl id size");
    std::memcpy(id128, &id, sizeof(id));
  });
}

// A handle's calls run on its device; the caller's current device is restored on return (the
// layer switches devices internally, a multi-GPU caller must not find its own device changed).
struct DeviceRestore {
  int prev = -1;
  DeviceRestore() {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  }
  ~DeviceRestore() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int moe_create(const moe_config* cfg, int32_t rank, const uint8_t* nccl_id128, int32_t device,
               moe_handle** out) {
  DeviceRestore restore;
  return guard(nullptr, [&] {
    if (!cfg || !out) throw moe::MoeError(MOE_EINVAL, "null argument");
    require_device();
    auto h = std::make_unique<moe_handle>();
    h->layer = std::make_unique<moe::Layer>(*cfg, rank, nccl_id128, device);
    *out = h.release();
  });
}

int moe_destroy(moe_handle* h) {
  DeviceRestore restore;
  delete h;
  return MOE_OK;
}

const char* moe_last_error(const moe_handle* h) { return h ? h->err.c_str() : g_err.c_str(); }
const char* moe_last_error_global(void) { return g_err.c_str(); }

#define LAYER_CALL(h, body)                                                 \
  do {                                                                      \
    if (!(h)) return MOE_EINVAL;                                            \
    DeviceRestore restore_;                                                 \
    return guard(&(h)->err, [&] { body; });                                 \
  } while (0)

int moe_init_params(moe_handle* h, uint64_t seed) { LAYER_CALL(h, h->layer->init_params(seed)); }
int moe_set_router(moe_handle* h, const double* wg) { LAYER_CALL(h, h->layer->set_router(wg)); }
int moe_set_capacity_factor(moe_handle* h, double f) { LAYER_CALL(h, h->layer->set_capacity_factor(f)); }
int moe_set_cosine_router(moe_handle* h, const double* proj, const double* experts, double temperature) {
  LAYER_CALL(h, h->layer->set_cosine_router(proj, experts, temperature));
}
int moe_set_expert(moe_handle* h, int64_t le, const double* w1, const double* w2) {
  LAYER_CALL(h, h->layer->set_expert(le, w1, w2));
}
int moe_set_expert_slices(moe_handle* h, const double* w1s, const double* w2s) {
  LAYER_CALL(h, h->layer->set_expert_slices(w1s, w2s));
}
int moe_forward(moe_handle* h, const void* x, void* y, void* stream) {
  LAYER_CALL(h, h->layer->forward(x, y, S(stream)));
}
int moe_backward(moe_handle* h, const void* dy, void* dx, float* dw1, float* dw2, void* stream) {
  LAYER_CALL(h, h->layer->backward(dy, dx, dw1, dw2, S(stream)));
}
int moe_forward_host(moe_handle* h, const void* xh, void* yh, void* stream) {
  LAYER_CALL(h, h->layer->forward_host(xh, yh, S(stream)));
}
int moe_backward_host(moe_handle* h, const void* dyh, void* dxh, void* stream) {
  LAYER_CALL(h, h->layer->backward_host(dyh, dxh, S(stream)));
}
int moe_forward_host_async(moe_handle* h, const void* xh, void* yh, void* stream) {
  LAYER_CALL(h, h->layer->forward_host_async(xh, yh, S(stream)));
}
int moe_backward_host_async(moe_handle* h, const void* dyh, void* dxh, void* stream) {
  LAYER_CALL(h, h->layer->backward_host_async(dyh, dxh, S(stream)));
}
int moe_host_sync(moe_handle* h) { LAYER_CALL(h, h->layer->host_sync()); }
int moe_get_routing(moe_handle* h, int32_t* idxs, int32_t* locs, double* gates, int64_t* cap) {
  LAYER_CALL(h, h->layer->get_routing(idxs, locs, gates, cap));
}
int moe_get_metrics(moe_handle* h, moe_step_metrics* out) { LAYER_CALL(h, h->layer->get_metrics(out)); }
int moe_get_expert_grads(moe_handle* h, float* dw1, float* dw2) {
  LAYER_CALL(h, h->layer->get_grads(dw1, dw2));
}
int moe_get_expert_grad_slices(moe_handle* h, float* w1_slices, float* w2_slices, void* stream) {
  LAYER_CALL(h, h->layer->grad_slices(w1_slices, w2_slices, S(stream)));
}
int moe_get_weights_device(moe_handle* h, int32_t which, void** ptr) {
  LAYER_CALL(h, {
    if (which == 1) *ptr = h->layer->w1();
    else if (which == 2) *ptr = h->layer->w2();
    else throw moe::MoeError(MOE_EINVAL, "which must be 1 or 2");
    h->layer->weights_updated();  // the caller may write through it
  });
}
int moe_weights_updated(moe_handle* h) { LAYER_CALL(h, h->layer->weights_updated()); }
int64_t moe_kernel_launches(const moe_handle* h) { return h ? h->layer->launches() : 0; }
int moe_set_profiling(moe_handle* h, int32_t on) { LAYER_CALL(h, h->layer->set_profiling(on != 0)); }
int moe_set_kernel_spans(moe_handle* h, int32_t on) { LAYER_CALL(h, h->layer->set_kernel_spans(on != 0)); }
int moe_take_kernel_spans(moe_handle* h, double* ms, int64_t* counts, int32_t n, double* sm_mhz) {
  LAYER_CALL(h, {
    h->layer->take_kernel_spans(ms, counts, n);
    if (sm_mhz) *sm_mhz = h->layer->span_mhz();
  });
}
int moe_take_profile(moe_handle* h, double* ms, int64_t* counts, int32_t n) {
  LAYER_CALL(h, h->layer->take_profile(ms, counts, n));
}

// ------------------------------------------------------------------ stateless ops
namespace {
struct CosineOp {
  const double* proj = nullptr;
  const double* experts = nullptr;
  int64_t D = 0;
  double temperature = 1.0;
};
int op_gating(const void* x, int32_t x_dtype, const double* wg, const CosineOp* cos, int64_t blocks,
              int64_t T, int64_t M, int64_t E, int64_t k, int32_t capacity_kind,
              double capacity_factor, int32_t bpr, int32_t* idxs, double* gates, int32_t* locations,
              double* probs, int64_t* capacity, int64_t* drops, void* stream) {
  return guard(nullptr, [&] {
    require_device();
    check_dtype(x_dtype);
    if (blocks < 1 || T < 1 || M < 1 || E < 1 || k < 1 || k > E)
      throw moe::MoeError(MOE_EINVAL, "gating: invalid shape");
    if (k > 32 || E > 256) throw moe::MoeError(MOE_EINVAL, "gating: k <= 32 and E <= 256 supported");
    if (capacity_kind < 0 || capacity_kind > 2) throw moe::MoeError(MOE_EINVAL, "capacity kind");
    cudaStream_t st = S(stream);
    Scratch sc(st);
    moe::GatingArgs a{};
    a.x = x;
    a.x_is_f32 = x_dtype == MOE_DTYPE_F32;
    a.wg = wg;
    a.blocks = static_cast<int>(blocks);
    a.T = static_cast<int>(T);
    a.M = static_cast<int>(M);
    a.E = static_cast<int>(E);
    a.k = static_cast<int>(k);
    a.cap_kind = capacity_kind;
    a.cap_formula = capacity_kind == MOE_CAP_AUTO
                        ? 0
                        : static_cast<int>(moe::expert_capacity(k, capacity_factor, T, E));
    a.bpr = bpr;
    const size_t n_cta = static_cast<size_t>(blocks) * moe::gate_cta_per_block(a.T);
    const size_t Tk = static_cast<size_t>(blocks) * T * k;
    moe::GatingBuffers g{};
    g.idxs = idxs;
    g.gates = gates;
    g.locations = locations;
    g.probs = probs;
    g.hist = sc.get<int32_t>(n_cta * E);
    g.offs = sc.get<int32_t>(n_cta * E);
    g.demand = sc.get<int32_t>(blocks * E);
    g.list_base = sc.get<int32_t>(blocks * E);
    g.fill = sc.get<int32_t>(blocks * E);
    g.list = sc.get<int32_t>(Tk);
    if (bpr) {
      g.bpr_keys = sc.get<unsigned long long>(Tk);
      g.bpr_pos = sc.get<int32_t>(Tk);
    }
    g.cap = sc.get<int32_t>(1);
    g.drops = sc.get<int32_t>(1);
    int32_t* err = nullptr;
    if (cos) {
      if (E > 64 || E % 2 || cos->D < 2 || cos->D % 2) throw moe::MoeError(MOE_EINVAL, "cosine gating: E <= 64 (even), even D");
      a.router = 1;
      a.cos_proj = cos->proj;
      a.cos_dim = static_cast<int>(cos->D);
      a.cos_tau = std::max(cos->temperature, 0.01);
      double* ct = sc.get<double>(static_cast<size_t>(E) * cos->D);
      double* en = sc.get<double>(static_cast<size_t>(E));
      err = sc.get<int32_t>(1);
      ck(cudaMemsetAsync(err, 0, 4, st), "memset");
      ckr(moe::cosine_prep_device(cos->experts, static_cast<int>(E), static_cast<int>(cos->D), ct, en, err, st),
          "cosine prep");
      a.cos_ct = ct;
      a.cos_en = en;
      a.cos_buf = sc.get<double>(static_cast<size_t>(blocks) * T * cos->D);
      a.err = err;
    }
    ckr(moe::run_gating_device(a, g, st), "gating");
    if (err) {
      int32_t e = 0;
      ck(cudaMemcpyAsync(&e, err, 4, cudaMemcpyDeviceToHost, st), "copy");
      ck(cudaStreamSynchronize(st), "sync");
      if (e == 2) throw moe::MoeError(MOE_EINVAL, "gate_cosine: zero-norm expert row");
      if (e) throw moe::MoeError(MOE_EINVAL, "gate_cosine: zero-norm projected token");
    }
    int32_t cap = a.cap_formula;
    if (capacity_kind != MOE_CAP_FIXED) {
      ck(cudaMemcpyAsync(&cap, g.cap, 4, cudaMemcpyDeviceToHost, st), "copy");
      ck(cudaStreamSynchronize(st), "sync");
    }
    g.slot_token = sc.get<int32_t>(static_cast<size_t>(blocks) * E * cap);
    g.slot_gate = sc.get<float>(static_cast<size_t>(blocks) * E * cap);
    ckr(moe::run_assign_device(a, g, cap, st), "assign");
    int32_t nd = 0;
    ck(cudaMemcpyAsync(&nd, g.drops, 4, cudaMemcpyDeviceToHost, st), "copy");
    ck(cudaStreamSynchronize(st), "sync");
    if (capacity) *capacity = cap;
    if (drops) *drops = nd;
  });
}
}  // namespace

int moe_op_gating(const void* x, int32_t x_dtype, const double* wg, int64_t blocks, int64_t T,
                  int64_t M, int64_t E, int64_t k, int32_t capacity_kind, double capacity_factor,
                  int32_t bpr, int32_t* idxs, double* gates, int32_t* locations, double* probs,
                  int64_t* capacity, int64_t* drops, void* stream) {
  return op_gating(x, x_dtype, wg, nullptr, blocks, T, M, E, k, capacity_kind, capacity_factor, bpr,
                   idxs, gates, locations, probs, capacity, drops, stream);
}

int moe_op_gating_cosine(const void* x, int32_t x_dtype, const double* proj, const double* experts,
                         int64_t D, double temperature, int64_t blocks, int64_t T, int64_t M,
                         int64_t E, int64_t k, int32_t capacity_kind, double capacity_factor,
                         int32_t bpr, int32_t* idxs, double* gates, int32_t* locations,
                         double* probs, int64_t* capacity, int64_t* drops, void* stream) {
  CosineOp c;
  c.proj = proj;
  c.experts = experts;
  c.D = D;
  c.temperature = temperature;
  return op_gating(x, x_dtype, nullptr, &c, blocks, T, M, E, k, capacity_kind, capacity_factor, bpr,
                   idxs, gates, locations, probs, capacity, drops, stream);
}

int moe_op_encode(const void* x, int32_t dtype, int64_t blocks, int64_t T, int64_t M, int64_t E,
                  int64_t k, int64_t capacity, int64_t degree, const int32_t* idxs,
                  const int32_t* locations, void* z, void* stream) {
  return guard(nullptr, [&] {
    require_device();
    check_dtype(dtype);
    const moe::SlotGeom g = make_geom(blocks, T, M, E, k, capacity, degree);
    cudaStream_t st = S(stream);
    Scratch sc(st);
    int32_t* stok = sc.get<int32_t>(static_cast<size_t>(blocks) * E * capacity);
    float* sg = sc.get<float>(static_cast<size_t>(blocks) * E * capacity);
    ckr(moe::build_slots_device(g.blocks, g.T, g.k, g.E, g.cap, idxs, locations, nullptr, stok, sg, st),
        "slots");
    ckr(moe::encode_device(g, dtype, x, stok, z, st), "encode");
  });
}

int moe_op_decode(const void* z, int32_t dtype, int64_t blocks, int64_t T, int64_t M, int64_t E,
                  int64_t k, int64_t capacity, int64_t degree, const int32_t* idxs,
                  const int32_t* locations, const double* gates, void* y, void* stream) {
  return guard(nullptr, [&] {
    require_device();
    check_dtype(dtype);
    const moe::SlotGeom g = make_geom(blocks, T, M, E, k, capacity, degree);
    ckr(moe::decode_device(g, dtype, z, idxs, locations, gates, y, S(stream)), "decode");
  });
}

int moe_op_decode_backward(const void* dy, const void* z, int32_t dtype, int64_t blocks,
                           int64_t T, int64_t M, int64_t E, int64_t k, int64_t capacity,
                           int64_t degree, const int32_t* idxs, const int32_t* locations,
                           const double* gates, void* dz, double* dgates, void* stream) {
  return guard(nullptr, [&] {
    require_device();
    check_dtype(dtype);
    const moe::SlotGeom g = make_geom(blocks, T, M, E, k, capacity, degree);
    cudaStream_t st = S(stream);
    Scratch sc(st);
    int32_t* stok = sc.get<int32_t>(static_cast<size_t>(blocks) * E * capacity);
    float* sg = sc.get<float>(static_cast<size_t>(blocks) * E * capacity);
    ckr(moe::build_slots_device(g.blocks, g.T, g.k, g.E, g.cap, idxs, locations, gates, stok, sg, st),
        "slots");
    ckr(moe::decode_backward_device(g, dtype, dy, stok, sg, dz, st), "decode_backward");
    if (dgates) {
      if (!z) throw moe::MoeError(MOE_EINVAL, "d_gates needs the expert output");
      ckr(moe::decode_backward_gates_device(g, dtype, z, dy, idxs, locations, dgates, st), "dgates");
    }
  });
}

int moe_op_encode_backward(const void* dz, int32_t dtype, int64_t blocks, int64_t T, int64_t M,
                           int64_t E, int64_t k, int64_t capacity, int64_t degree,
                           const int32_t* idxs, const int32_t* locations, void* dx, void* stream) {
  return guard(nullptr, [&] {
    require_device();
    check_dtype(dtype);
    const moe::SlotGeom g = make_geom(blocks, T, M, E, k, capacity, degree);
    ckr(moe::encode_backward_device(g, dtype, dz, idxs, locations, dx, S(stream)), "encode_backward");
  });
}

int moe_op_expert_ffn(const void* x, const void* w1, const void* w2, void* y, void* act,
                      int32_t dtype, int64_t n, int64_t rows, int64_t M, int64_t V, void* stream) {
  return guard(nullptr, [&] {
    require_device();
    check_dtype(dtype);
    if (n < 1 || rows < 1 || M < 1 || V < 1) throw moe::MoeError(MOE_EINVAL, "expert_ffn: shape");
    cudaStream_t st = S(stream);
    Scratch sc(st);
    const size_t esz = dtype == MOE_DTYPE_BF16 ? 2 : 4;
    void* a = act ? act : sc.get<char>(static_cast<size_t>(n) * rows * V * esz);
    moe::GemmArgs up{};
    up.G = n;
    up.S = 1;
    up.seg_rows = rows;
    up.N = V;
    up.K = M;
    moe::GemmArgs down = up;
    down.N = M;
    down.K = V;
    certified_up(dtype, x, w1, a, up, n, rows, M, V, st, sc);
    expert_gemm(moe::kGemmDown, dtype, -1, a, w2, y, down, static_cast<int>(n), st);
  });
}

int moe_op_expert_ffn_backward(const void* x, const void* w1, const void* w2, const void* dy,
                               void* dx, float* dw1, float* dw2, int32_t dtype, int64_t n,
                               int64_t rows, int64_t M, int64_t V, void* stream) {
  return guard(nullptr, [&] {
    require_device();
    check_dtype(dtype);
    if (n < 1 || rows < 1 || M < 1 || V < 1) throw moe::MoeError(MOE_EINVAL, "expert_ffn_backward: shape");
    cudaStream_t st = S(stream);
    Scratch sc(st);
    const size_t esz = dtype == MOE_DTYPE_BF16 ? 2 : 4;
    void* a = sc.get<char>(static_cast<size_t>(n) * rows * V * esz);
    void* dh = sc.get<char>(static_cast<size_t>(n) * rows * V * esz);
    moe::GemmArgs up{};
    up.G = n;
    up.S = 1;
    up.seg_rows = rows;
    up.N = V;
    up.K = M;
    const int nseg = static_cast<int>(n);
    // recompute a = relu(x W1) (parallelism.cpp:135-136)
    unsigned long long* mask = certified_up(dtype, x, w1, a, up, n, rows, M, V, st, sc);
    moe::GemmArgs dgm = up;
    dgm.aux = a;
    dgm.relu_mask = mask;
    expert_gemm(moe::kGemmDgradMask, dtype, -1, dy, w2, dh, dgm, nseg, st);
    moe::GemmArgs dg = up;
    dg.N = M;
    dg.K = V;
    expert_gemm(moe::kGemmDgrad, dtype, -1, dh, w1, dx, dg, nseg, st);
    moe::GemmArgs wg{};
    wg.G = n;
    wg.S = 1;
    wg.seg_rows = rows;
    wg.N = V;
    wg.Mo = M;
    expert_gemm(moe::kGemmWgrad, dtype, -1, x, dh, dw1, wg, nseg, st);
    wg.N = M;
    wg.Mo = V;
    expert_gemm(moe::kGemmWgrad, dtype, -1, a, dy, dw2, wg, nseg, st);
  });
}

int moe_op_weight_stats(const void* w1, int64_t n, int64_t M, int64_t V, float* colnorm,
                        float* colnorm_blk, void* w1t, void* stream) {
  return guard(nullptr, [&] {
    require_device();
    if (n < 1 || M < 1 || V < 1) throw moe::MoeError(MOE_EINVAL, "weight_stats: empty shape");
    ckr(moe::weight_stats_device(w1, static_cast<int>(n), static_cast<int>(M), static_cast<int>(V),
                                 colnorm, colnorm_blk, w1t, S(stream)),
        "weight stats");
  });
}

int moe_op_gemm(int32_t kind, int32_t dtype, int32_t use_tc, const void* A, const void* B,
                void* D, const void* aux, int64_t G, int64_t S_, int64_t seg_rows,
                int64_t seg_base, int64_t N, int64_t K, int64_t Mo, int64_t nseg_total,
                void* stream) {
  return guard(nullptr, [&] {
    require_device();
    check_dtype(dtype);
    if (kind < 0 || kind > 4) throw moe::MoeError(MOE_EINVAL, "gemm kind");
    moe::GemmArgs a{};
    a.G = static_cast<uint32_t>(G);
    a.S = static_cast<uint32_t>(S_);
    a.seg_rows = static_cast<uint32_t>(seg_rows);
    a.seg_base = static_cast<uint32_t>(seg_base);
    a.N = static_cast<uint32_t>(N);
    a.K = static_cast<uint32_t>(K);
    a.Mo = static_cast<uint32_t>(Mo);
    a.aux = aux;
    Scratch sc(S(stream));
    if (kind == moe::kGemmDgradMask && dtype == MOE_DTYPE_BF16 && use_tc != 0 && tc_shape_ok(kind, a)) {
      if (!aux) throw moe::MoeError(MOE_EINVAL, "dgrad-mask needs the activation (aux)");
      const int64_t rows = nseg_total * seg_rows;
      a.relu_mask = sc.get<unsigned long long>(moe::relu_mask_words(rows, N / 64));
      ckr(moe::relu_mask_from_act_device(aux, rows, static_cast<int>(N), a.relu_mask, S(stream)),
          "relu mask");
    }
    expert_gemm(kind, dtype, use_tc, A, B, D, a, static_cast<int>(nseg_total), S(stream));
  });
}

int moe_op_fill_uniform(void* dst, int32_t dtype, int64_t n, uint64_t seed, uint64_t offset,
                        double lo, double hi, void* stream) {
  return guard(nullptr, [&] {
    require_device();
    if (dtype < 0 || dtype > 2) throw moe::MoeError(MOE_EINVAL, "dtype");
    ckr(moe::fill_uniform_device(dst, dtype, n, seed, offset, lo, hi, S(stream)), "fill_uniform");
  });
}

// ------------------------------------------------------------------ Alg. 1 memo
int moe_memo_create(double bucket_length, moe_memo** out) {
  return guard(nullptr, [&] {
    auto m = std::make_unique<moe_memo>();
    m->search = moe::StrategySearch(bucket_length);
    *out = m.release();
  });
}
int moe_memo_destroy(moe_memo* m) {
  delete m;
  return MOE_OK;
}
int moe_memo_get_strategy(moe_memo* m, double f, int32_t* s) {
  return guard(nullptr, [&] { *s = m->search.choose(f); });
}
int moe_memo_optimize_strategy(moe_memo* m, double f, int32_t s, double seconds) {
  return guard(nullptr, [&] { m->search.record(f, s, seconds); });
}
int moe_memo_recompute_buckets(moe_memo* m, double f) {
  return guard(nullptr, [&] { m->search.rebucket(f); });
}
int moe_memo_num_buckets(moe_memo* m, int64_t* n) {
  return guard(nullptr, [&] { *n = m->search.num_buckets(); });
}
int moe_memo_bucket(moe_memo* m, int64_t i, double* start, int64_t* n_members, double* members,
                    int64_t max_members, double* table8) {
  return guard(nullptr, [&] {
    if (i < 0 || i >= m->search.num_buckets()) throw moe::MoeError(MOE_EINVAL, "bucket index");
    const int b = static_cast<int>(i);
    *start = m->search.bucket_start(b);
    const auto mem = m->search.bucket_members(b);
    *n_members = static_cast<int64_t>(mem.size());
    for (int64_t j = 0; j < *n_members && j < max_members; ++j) members[j] = mem[j];
    const double* t = m->search.bucket_times(b);
    for (int s = 0; s < moe::kNumStrategies; ++s) table8[s] = t[s];
  });
}
int moe_memo_lookup(moe_memo* m, double f, int32_t s, double* seconds, int32_t* present) {
  return guard(nullptr, [&] { *present = m->search.lookup(f, s, seconds) ? 1 : 0; });
}

}  // extern "C"
