// Alg. 1 (adaptive pipelining search). Behaviour pinned by the reference's KATs
// (test_pipeline.cpp:99-160): greedy L-wide buckets from the lowest f, times normalised by
// f_low / f, exploration in candidate order, ties to the earlier candidate. The layer feeds it
// CUDA-event seconds (layer.cpp, adaptive forward).
#include "strategy.h"

#include <algorithm>
#include <cmath>
#include <limits>

#include "layer.h"

namespace moe {

namespace {
constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();
}

int strategy_id(const Strategy& s) {
  if (s.algo < 0 || s.algo > 1) return -1;
  for (int j = 0; j < 4; ++j)
    if (s.degree == (1 << j)) return s.algo * 4 + j;
  return -1;
}

int StrategySearch::find(double f) const {
  auto it = std::lower_bound(recs_.begin(), recs_.end(), f,
                             [](const Record& r, double v) { return r.f < v; });
  return (it != recs_.end() && it->f == f) ? static_cast<int>(it - recs_.begin()) : -1;
}

int StrategySearch::bucket_of(int rec) const {
  for (int b = 0; b < num_buckets(); ++b)
    if (buckets_[b].first <= rec && rec <= buckets_[b].last) return b;
  throw MoeError(MOE_ESTATE, "strategy search: f record outside every bucket");
}

void StrategySearch::rebucket(double f) {
  if (!(f > 0.0)) throw MoeError(MOE_EINVAL, "strategy search: capacity factor must be > 0");
  if (find(f) < 0) {
    Record r;
    r.f = f;
    std::fill(std::begin(r.times), std::end(r.times), kNaN);
    auto it = std::lower_bound(recs_.begin(), recs_.end(), f,
                               [](const Record& a, double v) { return a.f < v; });
    recs_.insert(it, r);
  }
  // Greedy partition of the sorted f list: a record opens a new bucket when it lies more than
  // width_ above the current bucket's first f. The bucket's table takes every member's times
  // scaled by f_low / f, walking f upwards (a later member's time replaces an earlier one's).
  buckets_.clear();
  for (int i = 0; i < static_cast<int>(recs_.size()); ++i) {
    if (buckets_.empty() || recs_[i].f - recs_[buckets_.back().first].f > width_) {
      Bucket b;
      b.first = b.last = i;
      std::fill(std::begin(b.times), std::end(b.times), kNaN);
      buckets_.push_back(b);
    }
    Bucket& b = buckets_.back();
    b.last = i;
    for (int s = 0; s < kNumStrategies; ++s)
      if (!std::isnan(recs_[i].times[s]))
        b.times[s] = recs_[i].times[s] * recs_[b.first].f / recs_[i].f;
  }
}

int StrategySearch::ensure(double f) {
  int i = find(f);
  if (i < 0) {
    rebucket(f);
    i = find(f);
  }
  return i;
}

bool StrategySearch::full(const double* t) const {
  if (only_.empty())
    return std::none_of(t, t + kNumStrategies, [](double v) { return std::isnan(v); });
  return std::none_of(only_.begin(), only_.end(), [&](int s) { return std::isnan(t[s]); });
}

int StrategySearch::fastest(const double* t) const {
  int best = only_.empty() ? 0 : only_.front();
  double bt = std::numeric_limits<double>::infinity();
  for (int s = 0; s < kNumStrategies; ++s) {
    if (!only_.empty() && std::find(only_.begin(), only_.end(), s) == only_.end()) continue;
    if (!std::isnan(t[s]) && t[s] < bt) {  // strict: ties keep the earlier candidate
      bt = t[s];
      best = s;
    }
  }
  return best;
}

int StrategySearch::choose(double f) {
  const int i = ensure(f);
  if (full(recs_[i].times)) return fastest(recs_[i].times);
  const Bucket& b = buckets_[bucket_of(i)];
  if (full(b.times)) return fastest(b.times);
  for (int s = 0; s < kNumStrategies; ++s) {
    if (!only_.empty() && std::find(only_.begin(), only_.end(), s) == only_.end()) continue;
    if (std::isnan(b.times[s])) return s;
  }
  return fastest(b.times);
}

bool StrategySearch::settled(double f) {
  const int i = find(f);
  if (i < 0) return false;
  return full(recs_[i].times) || full(buckets_[bucket_of(i)].times);
}

void StrategySearch::record(double f, int id, double seconds) {
  if (id < 0 || id >= kNumStrategies) throw MoeError(MOE_EINVAL, "strategy search: no such strategy");
  const int i = ensure(f);
  recs_[i].times[id] = seconds;
  Bucket& b = buckets_[bucket_of(i)];
  b.times[id] = seconds * recs_[b.first].f / f;
}

std::vector<double> StrategySearch::bucket_members(int b) const {
  std::vector<double> out;
  for (int i = buckets_[b].first; i <= buckets_[b].last; ++i) out.push_back(recs_[i].f);
  return out;
}

bool StrategySearch::lookup(double f, int id, double* seconds) const {
  const int i = find(f);
  if (i < 0 || id < 0 || id >= kNumStrategies || std::isnan(recs_[i].times[id])) return false;
  *seconds = recs_[i].times[id];
  return true;
}

}  // namespace moe
