// C++ caller of the drop-in facade (include/moe_b200.hpp), checked against the fp64 oracle
// (oracle/moe_oracle.h -- test infrastructure). Built and run by tests/test_gpu_cpp_facade.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "../../include/moe_b200.hpp"
#include "../../oracle/moe_oracle.h"

int main() {
  using namespace moeb200;
  MoELayerConfig cfg;
  cfg.dims.global_experts = 8;
  cfg.dims.model_dim = 256;
  cfg.dims.hidden_dim = 512;
  cfg.dims.tokens_per_step = 512;
  cfg.dims.top_k = 2;
  cfg.capacity_factor = 1.25;
  cfg.bpr = true;
  cfg.dtype = DType::F32;
  const Index E = 8, M = 256, V = 512, T = 512, k = 2;
  const std::uint64_t seed = 402;
  LayerState st = LayerState::init(cfg, seed);
  // reference draw order (moe_layer.cpp:144-163): Wg, cosine (M+E)*256, experts, then x, dy
  const std::uint64_t o_exp = M * E + 256 * (M + E), o_x = o_exp + E * 2 * M * V;
  std::vector<double> wg(M * E), w1(E * M * V), w2(E * V * M);
  orc_fill_uniform(seed, 0, M * E, -1, 1, wg.data());
  for (Index e = 0; e < E; ++e) {
    orc_fill_uniform(seed, o_exp + e * 2 * M * V, M * V, -0.5, 0.5, w1.data() + e * M * V);
    orc_fill_uniform(seed, o_exp + e * 2 * M * V + M * V, M * V, -0.5, 0.5, w2.data() + e * M * V);
  }
  for (auto& v : w1) v = static_cast<float>(v);  // fp32 layer: the oracle sees the rounded values
  for (auto& v : w2) v = static_cast<float>(v);
  Tensor x = Tensor::zeros({T, M}), dy = Tensor::zeros({T, M});
  orc_fill_uniform(seed, o_x, T * M, -1, 1, x.data.data());
  orc_fill_uniform(seed, o_x + T * M, T * M, -1, 1, dy.data.data());
  for (auto& v : x.data) v = static_cast<float>(v);
  for (auto& v : dy.data) v = static_cast<float>(v);

  ForwardResult r = forward(st, x);
  LayerGrads g = backward(st, r.saved, dy);

  std::vector<double> y(T * M), dx(T * M), dw1(E * M * V), dw2(E * V * M), gates(T * k);
  std::vector<std::int64_t> idxs(T * k), loc(T * k);
  orc_layer_step(x.data.data(), wg.data(), w1.data(), w2.data(), dy.data.data(), 1, T, M, V, E, k,
                 0, 1.25, 1, y.data(), idxs.data(), loc.data(), gates.data(), dx.data(), dw1.data(),
                 dw2.data());
  auto rel = [](const std::vector<double>& a, const std::vector<double>& b) {
    double mx = 1e-300, d = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      mx = std::fmax(mx, std::fmax(std::fabs(a[i]), std::fabs(b[i])));
      d = std::fmax(d, std::fabs(a[i] - b[i]));
    }
    return d / mx;
  };
  std::vector<double> gdw1, gdw2;
  for (auto& eg : g.d_experts) {
    gdw1.insert(gdw1.end(), eg.dw1.data.begin(), eg.dw1.data.end());
    gdw2.insert(gdw2.end(), eg.dw2.data.begin(), eg.dw2.data.end());
  }
  const double ey = rel(r.y.data, y), edx = rel(g.dx.data, dx), e1 = rel(gdw1, dw1), e2 = rel(gdw2, dw2);
  std::printf("facade: y %.2e dx %.2e dw1 %.2e dw2 %.2e drops %lld\n", ey, edx, e1, e2,
              static_cast<long long>(r.metrics.drop_count));
  bool threw = false;
  try {
    forward(st, Tensor::zeros({T, M + 1}));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  const bool ok = ey < 1e-5 && edx < 1e-5 && e1 < 1e-5 && e2 < 1e-5 && threw;
  std::printf("%s\n", ok ? "FACADE PASS" : "FACADE FAIL");
  return ok ? 0 : 1;
}
