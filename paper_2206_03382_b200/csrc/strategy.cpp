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

namespace {

std::vector<int> allowed_of(const StrategyMemo& memo) {
  if (!memo.allowed.empty()) return memo.allowed;
  std::vector<int> all(strategy_space().size());
  for (size_t i = 0; i < all.size(); ++i) all[i] = static_cast<int>(i);
  return all;
}

bool complete(const std::map<int, double>& table, const std::vector<int>& allowed) {
  for (int i : allowed)
    if (table.find(i) == table.end()) return false;
  return true;
}

}  // namespace

Strategy get_strategy(StrategyMemo& memo, double f) {
  if (memo.per_f.find(f) == memo.per_f.end()) recompute_buckets(memo, f);
  const auto& space = strategy_space();
  const std::vector<int> allowed = allowed_of(memo);
  auto argmin = [&](const std::map<int, double>& table) {
    Strategy best = space[allowed.front()];
    double best_t = std::numeric_limits<double>::infinity();
    for (int i : allowed) {  // exploration order breaks ties
      auto it = table.find(i);
      if (it != table.end() && it->second < best_t) {
        best = space[i];
        best_t = it->second;
      }
    }
    return best;
  };
  const auto& own = memo.per_f[f];
  if (complete(own, allowed)) return argmin(own);
  StrategyMemo::Bucket* b = find_bucket(memo, f);
  if (!b) throw std::logic_error("get_strategy: f missing from every bucket");
  if (complete(b->table, allowed)) return argmin(b->table);
  for (int i : allowed)
    if (b->table.find(i) == b->table.end()) return space[i];
  return argmin(b->table);
}

bool strategy_settled(StrategyMemo& memo, double f) {
  auto it = memo.per_f.find(f);
  if (it == memo.per_f.end()) return false;
  const std::vector<int> allowed = allowed_of(memo);
  if (complete(it->second, allowed)) return true;
  StrategyMemo::Bucket* b = find_bucket(memo, f);
  return b && complete(b->table, allowed);
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
