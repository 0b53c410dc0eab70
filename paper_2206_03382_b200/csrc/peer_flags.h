// Ready-flag wait descriptor of the copy-engine all-to-all (host and device side).
#pragma once

#include <cstdint>

namespace moe {

// Flags of one (channel, chunk) are ready[ch][src][chunk] = base + src * stride, src != rank.
struct FlagWait {
  const uint32_t* base = nullptr;  // &ready[ch][0][chunk] in this rank's flag block; null: no wait
  int stride = 0;                  // words between sources
  int world = 0, rank = 0;
  uint32_t epoch = 0;
};

}  // namespace moe
