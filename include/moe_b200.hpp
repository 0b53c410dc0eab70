// moe_b200.hpp -- header-only C++17 facade over the C ABI (moe_b200.h) with the reference's
// layer API shape (/root/reference/proj/include/moesim/moe_layer.hpp):
//
//   auto state = moeb200::LayerState::init(cfg, seed);            // LayerState::init
//   moeb200::ForwardResult r = moeb200::forward(state, x);        // forward(state, x)
//   moeb200::LayerGrads g = moeb200::backward(state, r.saved, dy); // backward(state, saved, dy)
//
// Tensors are host-side, row-major fp64 with explicit shapes (like moesim::Tensor); x / dy are
// this rank's (T, M) token block. Values are rounded to the layer dtype on the way in (the
// reference is fed the same rounded values in parity tests). Errors are rethrown as the
// reference's exception types: std::invalid_argument, std::runtime_error, std::logic_error.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "moe_b200.h"

namespace moeb200 {

using Index = std::int64_t;

struct Tensor {
  std::vector<Index> shape;
  std::vector<double> data;
  Index size() const { return static_cast<Index>(data.size()); }
  static Tensor zeros(std::vector<Index> s) {
    Index n = 1;
    for (Index e : s) n *= e;
    return Tensor{std::move(s), std::vector<double>(static_cast<size_t>(n), 0.0)};
  }
};

enum class CapacityKind { Fixed = MOE_CAP_FIXED, Auto = MOE_CAP_AUTO, Bounded = MOE_CAP_BOUNDED };
enum class DType { BF16 = MOE_DTYPE_BF16, F32 = MOE_DTYPE_F32 };

struct Dims {  // core.hpp:32-56 (E >= W: ExpertsPerRank{E/W}; E < W: RanksPerExpert{W/E})
  Index world_size = 1, gpus_per_node = 1, global_experts = 1, model_dim = 1, hidden_dim = 1,
        tokens_per_step = 1, top_k = 1;
};

struct StrategyControl {  // moe_layer.hpp:17-20
  bool adaptive = false;
  int algo = MOE_A2A_LINEAR;  // fixed.algo
  int degree = 1;
  int a2a_backend = MOE_A2A_BACKEND_PEER;
};

enum class RouterKind { Linear = MOE_ROUTER_LINEAR, Cosine = MOE_ROUTER_COSINE };  // moe_layer.hpp:10
enum class ParallelChoice { P1 = MOE_PARALLEL_P1, P2 = MOE_PARALLEL_P2 };  // parallelism.hpp

struct ParallelControl {  // moe_layer.hpp:17-20
  bool adaptive = false;
  ParallelChoice fixed = ParallelChoice::P1;
};

struct MoELayerConfig {  // moe_layer.hpp:22-29
  Dims dims;
  CapacityKind capacity = CapacityKind::Fixed;
  RouterKind router = RouterKind::Linear;
  double capacity_factor = 1.0;
  bool bpr = false;
  DType dtype = DType::BF16;
  StrategyControl strategy;
  ParallelControl parallel;

  moe_config to_c() const {
    moe_config c{};
    c.world_size = dims.world_size;
    c.gpus_per_node = dims.gpus_per_node;
    c.global_experts = dims.global_experts;
    c.model_dim = dims.model_dim;
    c.hidden_dim = dims.hidden_dim;
    c.tokens_per_step = dims.tokens_per_step;
    c.top_k = dims.top_k;
    c.capacity_kind = static_cast<int32_t>(capacity);
    c.capacity_factor = capacity_factor;
    c.bpr = bpr ? 1 : 0;
    c.dtype = static_cast<int32_t>(dtype);
    c.adaptive = strategy.adaptive ? 1 : 0;
    c.degree = strategy.degree;
    c.a2a_backend = strategy.a2a_backend;
    c.router = static_cast<int32_t>(router);
    c.parallel = parallel.adaptive ? MOE_PARALLEL_ADAPTIVE : static_cast<int32_t>(parallel.fixed);
    c.a2a_algo = strategy.algo;
    return c;
  }
};

inline void throw_status(int rc, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (rc) {
    case MOE_OK: return;
    case MOE_EINVAL: throw std::invalid_argument(m);
    case MOE_ESTATE: throw std::logic_error(m);
    default: throw std::runtime_error(m);
  }
}

struct StepMetrics {  // moe_layer.hpp:46-54 (seconds are measured, not simulated)
  double f = 1.0;
  Index capacity = 1;
  int degree = 1;
  double seconds = 0.0;
  double comm_bytes = 0.0;
  Index drop_count = 0;
  ParallelChoice parallel = ParallelChoice::P1;
};

struct SavedForward {  // handle-owned tensors of the last forward
  std::uint64_t step = 0;
};

class LayerState {
 public:
  static LayerState init(const MoELayerConfig& cfg, std::uint64_t seed, int rank = 0,
                         int device = 0, const std::uint8_t* nccl_id = nullptr) {
    LayerState s(cfg, rank, device, nccl_id);
    throw_status(moe_init_params(s.h_, seed), moe_last_error(s.h_));
    return s;
  }
  LayerState(const MoELayerConfig& cfg, int rank = 0, int device = 0,
             const std::uint8_t* nccl_id = nullptr)
      : config(cfg) {
    const moe_config c = cfg.to_c();
    throw_status(moe_create(&c, rank, nccl_id, device, &h_), moe_last_error_global());
  }
  LayerState(LayerState&& o) noexcept : config(o.config), step(o.step), h_(o.h_) { o.h_ = nullptr; }
  LayerState(const LayerState&) = delete;
  LayerState& operator=(const LayerState&) = delete;
  ~LayerState() {
    if (h_) moe_destroy(h_);
  }
  moe_handle* handle() const { return h_; }

  MoELayerConfig config;
  std::uint64_t step = 0;

 private:
  moe_handle* h_ = nullptr;
};

struct ForwardResult {
  Tensor y;
  StepMetrics metrics;
  SavedForward saved;
};

struct ExpertGrad {
  Tensor dw1;  // (M, V)
  Tensor dw2;  // (V, M)
};

struct LayerGrads {
  Tensor dx;                         // (T, M)
  std::vector<ExpertGrad> d_experts; // this rank's local experts
};

namespace detail {
inline std::uint16_t bf16_rne(double x) {  // direct fp64 -> bf16, round to nearest even
  std::uint64_t u;
  std::memcpy(&u, &x, 8);
  if ((u & 0x7FF0000000000000ULL) != 0x7FF0000000000000ULL) {
    u += (1ULL << 44) - 1 + ((u >> 45) & 1);
    u &= ~((1ULL << 45) - 1);
  }
  double r;
  std::memcpy(&r, &u, 8);
  const float f = static_cast<float>(r);
  std::uint32_t b;
  std::memcpy(&b, &f, 4);
  return static_cast<std::uint16_t>(b >> 16);
}
inline std::vector<unsigned char> pack(const Tensor& t, DType dt) {
  std::vector<unsigned char> out;
  if (dt == DType::BF16) {
    out.resize(t.data.size() * 2);
    auto* p = reinterpret_cast<std::uint16_t*>(out.data());
    for (size_t i = 0; i < t.data.size(); ++i) p[i] = bf16_rne(t.data[i]);
  } else {
    out.resize(t.data.size() * 4);
    auto* p = reinterpret_cast<float*>(out.data());
    for (size_t i = 0; i < t.data.size(); ++i) p[i] = static_cast<float>(t.data[i]);
  }
  return out;
}
inline Tensor unpack(const std::vector<unsigned char>& b, DType dt, std::vector<Index> shape) {
  Tensor t = Tensor::zeros(std::move(shape));
  if (dt == DType::BF16) {
    auto* p = reinterpret_cast<const std::uint16_t*>(b.data());
    for (size_t i = 0; i < t.data.size(); ++i) {
      const std::uint32_t u = static_cast<std::uint32_t>(p[i]) << 16;
      float f;
      std::memcpy(&f, &u, 4);
      t.data[i] = f;
    }
  } else {
    auto* p = reinterpret_cast<const float*>(b.data());
    for (size_t i = 0; i < t.data.size(); ++i) t.data[i] = p[i];
  }
  return t;
}
}  // namespace detail

inline ForwardResult forward(LayerState& state, const Tensor& x) {
  const auto& d = state.config.dims;
  if (x.shape != std::vector<Index>{d.tokens_per_step, d.model_dim})
    throw std::invalid_argument("forward: expected (T, M) input");
  auto xin = detail::pack(x, state.config.dtype);
  std::vector<unsigned char> yout(xin.size());
  throw_status(moe_forward_host(state.handle(), xin.data(), yout.data(), nullptr),
               moe_last_error(state.handle()));
  ForwardResult r;
  r.y = detail::unpack(yout, state.config.dtype, x.shape);
  moe_step_metrics m{};
  throw_status(moe_get_metrics(state.handle(), &m), moe_last_error(state.handle()));
  r.metrics = StepMetrics{m.f, m.capacity, m.degree, m.seconds, m.comm_bytes, m.drop_count,
                          static_cast<ParallelChoice>(m.parallel)};
  r.saved.step = ++state.step;
  return r;
}

inline LayerGrads backward(LayerState& state, const SavedForward& saved, const Tensor& dy) {
  const auto& d = state.config.dims;
  if (saved.step != state.step) throw std::logic_error("backward: saved forward is stale");
  if (dy.shape != std::vector<Index>{d.tokens_per_step, d.model_dim})
    throw std::invalid_argument("backward: expected (T, M) gradient");
  auto din = detail::pack(dy, state.config.dtype);
  std::vector<unsigned char> dxout(din.size());
  throw_status(moe_backward_host(state.handle(), din.data(), dxout.data(), nullptr),
               moe_last_error(state.handle()));
  LayerGrads g;
  g.dx = detail::unpack(dxout, state.config.dtype, dy.shape);
  // computed experts: E/W, or the one expert rank/s under sharded placement (E < W)
  const Index nE = d.global_experts < d.world_size ? 1 : d.global_experts / d.world_size;
  const Index M = d.model_dim, V = d.hidden_dim;
  std::vector<float> w1(static_cast<size_t>(nE * M * V)), w2(static_cast<size_t>(nE * V * M));
  throw_status(moe_get_expert_grads(state.handle(), w1.data(), w2.data()),
               moe_last_error(state.handle()));
  for (Index e = 0; e < nE; ++e) {
    ExpertGrad eg{Tensor::zeros({M, V}), Tensor::zeros({V, M})};
    for (Index i = 0; i < M * V; ++i) {
      eg.dw1.data[static_cast<size_t>(i)] = w1[static_cast<size_t>(e * M * V + i)];
      eg.dw2.data[static_cast<size_t>(i)] = w2[static_cast<size_t>(e * M * V + i)];
    }
    g.d_experts.push_back(std::move(eg));
  }
  return g;
}

}  // namespace moeb200
