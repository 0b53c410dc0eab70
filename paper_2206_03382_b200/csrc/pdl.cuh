// Programmatic dependent launch (sm_90+): consecutive kernels of the layer overlap the next
// kernel's launch and prologue with the previous kernel's tail. Every kernel launched through
// launch_k() must call pdl_entry() (or pdl_wait() before touching its predecessor's outputs):
// griddepcontrol.wait blocks until the preceding grid has completed and its memory is visible,
// and is a no-op for kernels launched without the attribute. MOE_PDL=0 disables the attribute.
#pragma once

#include <cuda_runtime.h>

#include <cstdlib>

namespace moe {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// the common case: wait for the predecessor, then let the successor's CTAs launch as SMs free up
__device__ __forceinline__ void pdl_entry() {
  pdl_wait();
  pdl_trigger();
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MOE_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace moe
