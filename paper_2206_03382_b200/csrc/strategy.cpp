// Alg. 1 of the Tutel paper: online search of the all-to-all algorithm x pipelining degree,
// keyed by capacity factor f with greedy L-wide buckets that share exploration progress.
// Restates /root/reference/proj/src/pipeline.cpp:100-121 (strategy order) and :180-237
// (recompute_buckets, get_strategy, optimize_strategy) as host C++; the layer feeds it measured
// CUDA-event seconds instead of simulated seconds.
#include "strategy.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>

namespace moe {

const std::vector<Strategy>& strategy_space() {
  static const std::vector<Strategy> space = [] {
    std::vector<Strategy> v;
    for (int algo : {0, 1})
      for (int d : {1, 2, 4, 8}) v.push_back({algo, d});
    return v;
  }();
  return space;
}

int strategy_index(const Strategy& s) {
  const auto& sp = strategy_space();
  for (size_t i = 0; i < sp.size(); ++i)
    if (sp[i] == s) return static_cast<int>(i);
  return -1;
}

namespace {

StrategyMemo::Bucket* find_bucket(StrategyMemo& memo, double f) {
  for (auto& b : memo.buckets)
    if (std::find(b.members.begin(), b.members.end(), f) != b.members.end()) return &b;
  return nullptr;
}

}  // namespace

void recompute_buckets(StrategyMemo& memo, double f) {
  if (!(f > 0.0)) throw std::invalid_argument("recompute_buckets: f must be positive");
  memo.per_f.try_emplace(f);
  memo.buckets.clear();
  StrategyMemo::Bucket* cur = nullptr;
  for (const auto& [fv, table] : memo.per_f) {
    if (!cur || fv - cur->start > memo.bucket_length) {
      memo.buckets.push_back({fv, {}, {}});
      cur = &memo.buckets.back();
    }
    cur->members.push_back(fv);
    for (const auto& [s, t] : table) cur->table[s] = t * cur->start / fv;
  }
}

Strategy get_strategy(StrategyMemo& memo, double f) {
  if (memo.per_f.find(f) == memo.per_f.end()) recompute_buckets(memo, f);
  const auto& space = strategy_space();
  auto argmin = [&](const std::map<int, double>& table) {
    Strategy best = space.front();
    double best_t = std::numeric_limits<double>::infinity();
    for (size_t i = 0; i < space.size(); ++i) {
      auto it = table.find(static_cast<int>(i));
      if (it != table.end() && it->second < best_t) {
        best = space[i];
        best_t = it->second;
      }
    }
    return best;
  };
  const auto& own = memo.per_f[f];
  if (own.size() == space.size()) return argmin(own);
  StrategyMemo::Bucket* b = find_bucket(memo, f);
  if (!b) throw std::logic_error("get_strategy: f missing from every bucket");
  if (b->table.size() == space.size()) return argmin(b->table);
  for (size_t i = 0; i < space.size(); ++i)
    if (b->table.find(static_cast<int>(i)) == b->table.end()) return space[i];
  return argmin(b->table);
}

void optimize_strategy(StrategyMemo& memo, double f, const Strategy& s, double seconds) {
  if (memo.per_f.find(f) == memo.per_f.end()) recompute_buckets(memo, f);
  const int idx = strategy_index(s);
  if (idx < 0) throw std::invalid_argument("optimize_strategy: unknown strategy");
  memo.per_f[f][idx] = seconds;
  StrategyMemo::Bucket* b = find_bucket(memo, f);
  if (!b) throw std::logic_error("optimize_strategy: f missing from every bucket");
  b->table[idx] = seconds * b->start / f;
}

}  // namespace moe
