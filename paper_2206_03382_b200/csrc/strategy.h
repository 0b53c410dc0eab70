// Online search of (all-to-all algorithm, pipelining degree) keyed by the capacity factor f —
// Alg. 1 of the Tutel paper. Semantics follow the reference's StrategyMemo
// (/root/reference/proj/include/moesim/pipeline.hpp:67-88, src/pipeline.cpp:180-237); the data
// structure is this repo's own: one sorted array of f records with a fixed 8-slot time table
// each, and buckets as index ranges over that array.
#pragma once

#include <cstdint>
#include <vector>

namespace moe {

// The eight candidates, in exploration order: linear x {1,2,4,8}, then 2DH x {1,2,4,8}
// (pipeline.cpp:113-121). A strategy is identified by its slot in that order.
constexpr int kNumStrategies = 8;

struct Strategy {
  int algo = 0;    // 0 linear, 1 2DH (MOE_A2A_LINEAR / MOE_A2A_2DH)
  int degree = 1;  // capacity chunks
};

inline Strategy strategy_at(int id) { return Strategy{id / 4, 1 << (id % 4)}; }
// -1 for an (algo, degree) pair outside the search space.
int strategy_id(const Strategy& s);

class StrategySearch {
 public:
  explicit StrategySearch(double bucket_width = 0.5) : width_(bucket_width) {}

  // Limit the candidates (ascending ids; empty = all eight). Inside one NVSwitch domain the
  // layer searches only the linear degrees: 2DH there is linear plus two local reorders.
  void restrict_to(std::vector<int> ids) { only_ = std::move(ids); }

  // Register f if unseen and rebuild the buckets (recompute_buckets, pipeline.cpp:180-196).
  void rebucket(double f);
  // The next strategy for f: exploit f's own complete table, else its bucket's complete
  // table, else the first candidate the bucket has not timed (get_strategy, :198-221).
  int choose(double f);
  // Store a measurement; the bucket copy is scaled to the bucket's lowest f
  // (optimize_strategy, :223-229).
  void record(double f, int id, double seconds);
  // True once choose(f) would exploit rather than explore.
  bool settled(double f);

  // Introspection for the C ABI / tests.
  int num_buckets() const { return static_cast<int>(buckets_.size()); }
  double bucket_start(int b) const { return recs_[buckets_[b].first].f; }
  std::vector<double> bucket_members(int b) const;
  const double* bucket_times(int b) const { return buckets_[b].times; }  // NaN = never timed
  bool lookup(double f, int id, double* seconds) const;

 private:
  struct Record {
    double f;
    double times[kNumStrategies];  // measured seconds, NaN = never timed
  };
  struct Bucket {
    int first, last;               // record index range [first, last]
    double times[kNumStrategies];  // normalised to the bucket's lowest f
  };
  int find(double f) const;        // record index of f, or -1
  int bucket_of(int rec) const;    // bucket holding record rec
  int ensure(double f);            // find, registering + rebucketing an unseen f
  bool full(const double* t) const;
  int fastest(const double* t) const;

  double width_;
  std::vector<int> only_;
  std::vector<Record> recs_;       // ascending f
  std::vector<Bucket> buckets_;
};

}  // namespace moe
