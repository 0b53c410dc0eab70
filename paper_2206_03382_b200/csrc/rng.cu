// Counter-based splitmix64 draws, identical to the reference generator (core.cpp:66-83):
// the n-th call (1-based) of Rng(seed).next_u64() is mix(seed + n * 0x9e3779b97f4a7c15), and
// uniform(lo, hi) = lo + (hi - lo) * ((u64 >> 11) * 2^-53). Because the stream is counter-based,
// any element of the LayerState::init draw sequence (moe_layer.cpp:144-163) can be generated in
// parallel on the device by its index.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace moe {

namespace {

__device__ __forceinline__ double draw(uint64_t seed, uint64_t n1, double lo, double hi) {
  uint64_t z = seed + n1 * 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z = z ^ (z >> 31);
  const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
  return lo + (hi - lo) * u;
}

template <typename T>
__device__ __forceinline__ void store(T* p, double v);
template <>
__device__ __forceinline__ void store<__nv_bfloat16>(__nv_bfloat16* p, double v) {
  // double -> bf16 round-to-nearest-even directly (no double rounding through fp32)
  *p = __double2bfloat16(v);
}
template <>
__device__ __forceinline__ void store<float>(float* p, double v) {
  *p = __double2float_rn(v);
}
template <>
__device__ __forceinline__ void store<double>(double* p, double v) {
  *p = v;
}

template <typename T>
__global__ void fill_kernel(T* dst, int64_t rows, int64_t cols, int64_t src_stride, uint64_t seed,
                            uint64_t offset, double lo, double hi) {
  const int64_t n = rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const uint64_t idx = offset + static_cast<uint64_t>(r * src_stride + c);
    store<T>(dst + i, draw(seed, idx + 1, lo, hi));
  }
}

}  // namespace

int fill_uniform_2d_device(void* dst, int dtype, int64_t rows, int64_t cols, int64_t src_stride,
                           uint64_t seed, uint64_t offset, double lo, double hi, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return 0;
  const int64_t n = rows * cols;
  const int grid = static_cast<int>(n / 256 + 1 < 148 * 16 ? n / 256 + 1 : 148 * 16);
  if (dtype == 0)
    fill_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(dst), rows, cols,
                                                     src_stride, seed, offset, lo, hi);
  else if (dtype == 1)
    fill_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(dst), rows, cols, src_stride, seed,
                                             offset, lo, hi);
  else
    fill_kernel<double><<<grid, 256, 0, st>>>(static_cast<double*>(dst), rows, cols, src_stride,
                                              seed, offset, lo, hi);
  return launch_status();
}

int fill_uniform_device(void* dst, int dtype, int64_t n, uint64_t seed, uint64_t offset, double lo,
                        double hi, cudaStream_t st) {
  return fill_uniform_2d_device(dst, dtype, 1, n, n, seed, offset, lo, hi, st);
}

}  // namespace moe
