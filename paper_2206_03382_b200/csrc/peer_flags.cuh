// Device-side wait on the copy-engine all-to-all's ready flags (peer_a2a.h): flags of one
// (channel, chunk) are ready[ch][src][chunk], i.e. base + src * stride for src != rank.
#pragma once

#include <cstdint>

#include "peer_flags.h"

namespace moe {



__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Called by one warp: lane s polls source s until its flag reaches the epoch (the data the copy
// engine wrote before the flag is then visible). A peer that never publishes (dead rank) traps
// after 20 s instead of hanging the stream.
__device__ __forceinline__ void wait_flags_warp(const FlagWait& w) {
  const int lane = threadIdx.x % 32;
  for (int s = lane; s < w.world; s += 32) {
    if (s == w.rank) continue;
    const uint32_t* f = w.base + static_cast<size_t>(s) * w.stride;
    const uint64_t t0 = globaltimer_ns();
    while (static_cast<int32_t>(ld_acquire_sys(f) - w.epoch) < 0) {
      if (globaltimer_ns() - t0 > 20000000000ull) __trap();
      __nanosleep(200);
    }
  }
  __syncwarp();
}

}  // namespace moe
