// Adaptive pipelining memo (Alg. 1). See strategy.cpp.
#pragma once

#include <map>
#include <vector>

namespace moe {

struct Strategy {
  int algo = 0;    // 0 linear, 1 2DH
  int degree = 1;  // capacity chunks
  bool operator==(const Strategy& o) const { return algo == o.algo && degree == o.degree; }
};

// {Linear, TwoDH} x {1, 2, 4, 8}, linear first, ascending degree (pipeline.cpp:113-121).
const std::vector<Strategy>& strategy_space();
int strategy_index(const Strategy& s);

struct StrategyMemo {
  double bucket_length = 0.5;
  // Strategy indices the search may use (empty = the reference's full space). Inside a single
  // NVSwitch domain (gpus_per_node == W) 2DH is linear plus two local copies, so the layer
  // restricts the search to the linear degrees.
  std::vector<int> allowed;
  struct Bucket {
    double start = 0.0;
    std::vector<double> members;
    std::map<int, double> table;  // strategy index -> normalized seconds
  };
  std::map<double, std::map<int, double>> per_f;
  std::vector<Bucket> buckets;
};

void recompute_buckets(StrategyMemo& memo, double f);
Strategy get_strategy(StrategyMemo& memo, double f);
void optimize_strategy(StrategyMemo& memo, double f, const Strategy& s, double seconds);
// True once f's own table or its bucket has a time for every strategy (get_strategy exploits).
bool strategy_settled(StrategyMemo& memo, double f);

}  // namespace moe
