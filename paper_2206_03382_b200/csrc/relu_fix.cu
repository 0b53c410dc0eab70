// ReLU-mask certificate for the bf16 tensor-core path.
//
// The backward mask [h > 0] of expert_ffn_backward (parallelism.cpp:135-138) is discontinuous:
// one element whose sign differs from the fp64 reference moves a whole column of dW1 = X^T dh
// by |X| * |dA|. The tcgen05 GEMM accumulates in fp32 (measured error <= 2^-21.6 * sum|x w| on
// B200), so the up-GEMM epilogue lists every output with |h| < 2^-18 * |x_row|_2 * |w_col|_2
// (Cauchy-Schwarz: >= 2^-18 * sum|x w|, i.e. >= 12x the measured error bound; tighter than
// max|x| * sum|w| by ~1/3 at these shapes) and relu_fixup re-decides those in fp64 -- exact
// products of the bf16 inputs, so the mask equals the fp64 reference's except for |h| < ~1e-13.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gemm_sm100.h"
#include "checks.cuh"
#include "kernels.h"
#include "pdl.cuh"
#include "peer_flags.cuh"
#include "relu_mask.cuh"

namespace moe {

namespace {

// colnorm[g][v] = |W1[g][:, v]|_2 (fp64 sum of squares, rounded up)
__global__ void colnorm_kernel(const __nv_bfloat16* __restrict__ w1, int G, int M, int V,
                              float* __restrict__ colnorm) {
  pdl_entry();
  const int n = G * V;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int g = i / V, v = i % V;
    const __nv_bfloat16* col = w1 + static_cast<size_t>(g) * M * V + v;
    double s = 0.0;
    for (int m = 0; m < M; ++m) {
      const double w = __bfloat162float(col[static_cast<size_t>(m) * V]);
      s = fma(w, w, s);
    }
    colnorm[i] = static_cast<float>(sqrt(s)) * 1.0001f;  // |W1[:, col]|_2, rounded up
  }
}

// blk[g][b] = max over the 64 columns of block b of colnorm[g][:]
__global__ void colnorm_blk_kernel(const float* __restrict__ colnorm, int G, int V,
                                  float* __restrict__ blk) {
  pdl_entry();
  const int nb = V / 64;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < G * nb; i += gridDim.x * blockDim.x) {
    const float* c = colnorm + static_cast<size_t>(i / nb) * V + (i % nb) * 64;
    float m = 0.0f;
    for (int j = 0; j < 64; ++j) m = fmaxf(m, c[j]);
    blk[i] = m;
  }
}

// out[g][c][r] = in[g][r][c] (bf16, 32x32 smem tiles)
__global__ void transpose_kernel(const __nv_bfloat16* __restrict__ in, int R, int Cc,
                                 __nv_bfloat16* __restrict__ out) {
  pdl_entry();
  __shared__ __nv_bfloat16 tile[32][33];
  const size_t g = blockIdx.z;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const __nv_bfloat16* src = in + g * R * Cc;
  __nv_bfloat16* dst = out + g * R * Cc;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < Cc) tile[i][threadIdx.x] = src[static_cast<size_t>(r) * Cc + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < Cc) dst[static_cast<size_t>(c) * R + r] = tile[threadIdx.x][i];
  }
}

// One pass over W1 for the certificate's weight statistics (M % 64 == 0, V % 64 == 0): a CTA owns
// the 64-column strip [64 b, 64 b + 64) of expert g, walks M in 64-row tiles (16-byte loads, two
// per thread), writes the transposed tile to w1t with 16-byte stores, and accumulates the
// columns' sums of squares in fp64. It then writes colnorm for its 64 columns and their max
// (colnorm_blk). Algorithmic traffic: read G*M*V*2 B + write G*M*V*2 B.
__global__ void __launch_bounds__(256) weight_stats_kernel(const __nv_bfloat16* __restrict__ w1,
                                                           int M, int V, float* __restrict__ colnorm,
                                                           float* __restrict__ blk,
                                                           __nv_bfloat16* __restrict__ w1t) {
  pdl_entry();
  __shared__ __align__(16) __nv_bfloat16 tile[64][64 + 8];
  __shared__ double part[8][64];
  __shared__ float wmax[2];
  const int nb = V / 64;
  const int g = blockIdx.x / nb, b = blockIdx.x % nb;
  const int t = threadIdx.x;
  const __nv_bfloat16* src = w1 + static_cast<size_t>(g) * M * V + 64 * b;
  __nv_bfloat16* dst = w1t + (static_cast<size_t>(g) * V + 64 * b) * M;
  const int lr = t / 8, lc = (t % 8) * 8;  // load: rows lr, lr + 32; 8 columns at lc
  const int cp = t % 32, rg = t / 32;      // transpose: columns 2cp, 2cp + 1; rows [8 rg, 8 rg + 8)
  double acc0 = 0.0, acc1 = 0.0;
  uint4 v0 = __ldcs(reinterpret_cast<const uint4*>(src + static_cast<size_t>(lr) * V + lc));
  uint4 v1 = __ldcs(reinterpret_cast<const uint4*>(src + static_cast<size_t>(lr + 32) * V + lc));
  for (int m0 = 0; m0 < M; m0 += 64) {
    *reinterpret_cast<uint4*>(&tile[lr][lc]) = v0;
    *reinterpret_cast<uint4*>(&tile[lr + 32][lc]) = v1;
    __syncthreads();
    if (m0 + 64 < M) {  // the next tile's loads fly while this one is transposed
      v0 = __ldcs(reinterpret_cast<const uint4*>(src + static_cast<size_t>(m0 + 64 + lr) * V + lc));
      v1 = __ldcs(reinterpret_cast<const uint4*>(src + static_cast<size_t>(m0 + 96 + lr) * V + lc));
    }
    // 8 rows x the column pair as 32-bit words; low halves -> column 2cp, high -> 2cp + 1
    uint32_t wv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) wv[j] = *reinterpret_cast<const uint32_t*>(&tile[8 * rg + j][2 * cp]);
    uint4 o0, o1;
    o0.x = __byte_perm(wv[0], wv[1], 0x5410); o1.x = __byte_perm(wv[0], wv[1], 0x7632);
    o0.y = __byte_perm(wv[2], wv[3], 0x5410); o1.y = __byte_perm(wv[2], wv[3], 0x7632);
    o0.z = __byte_perm(wv[4], wv[5], 0x5410); o1.z = __byte_perm(wv[4], wv[5], 0x7632);
    o0.w = __byte_perm(wv[6], wv[7], 0x5410); o1.w = __byte_perm(wv[6], wv[7], 0x7632);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double lo = __uint_as_float(wv[j] << 16), hi = __uint_as_float(wv[j] & 0xffff0000u);
      acc0 = fma(lo, lo, acc0);
      acc1 = fma(hi, hi, acc1);
    }
    __stcs(reinterpret_cast<uint4*>(dst + static_cast<size_t>(2 * cp) * M + m0 + 8 * rg), o0);
    __stcs(reinterpret_cast<uint4*>(dst + static_cast<size_t>(2 * cp + 1) * M + m0 + 8 * rg), o1);
    __syncthreads();
  }
  part[rg][2 * cp] = acc0;
  part[rg][2 * cp + 1] = acc1;
  __syncthreads();
  if (t < 64) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += part[q][t];
    float n = static_cast<float>(sqrt(s)) * 1.0001f;  // |W1[:, col]|_2, rounded up
    colnorm[static_cast<size_t>(g) * V + 64 * b + t] = n;
    for (int o = 16; o > 0; o >>= 1) n = fmaxf(n, __shfl_xor_sync(0xffffffffu, n, o));
    if (t % 32 == 0) wmax[t / 32] = n;
  }
  __syncthreads();
  if (t == 0 && blk) blk[static_cast<size_t>(g) * nb + b] = fmaxf(wmax[0], wmax[1]);
}

// rownorm[i] = |x[i]|_2 (one warp per row)
// |x[r]|_2 per row (rounded up). Optionally first waits for the chunk's peer flags (fused
// receive wait) and resets the fixup counter.
__global__ void rownorm_kernel(const __nv_bfloat16* __restrict__ x, int M, float* __restrict__ rownorm,
                               RowSet rs, FlagWait fw, unsigned int* reset) {
  pdl_entry();
  if (fw.base != nullptr) {
    if (threadIdx.x < 32) wait_flags_warp(fw);
    __syncthreads();
  }
  if (reset != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *reset = 0u;
  const int lane = threadIdx.x % 32;
  const bool vec = (M % 8) == 0;
  const int64_t total = static_cast<int64_t>(rs.nsegs) * rs.nrows;
  for (int64_t id = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; id < total;
       id += static_cast<int64_t>(gridDim.x) * blockDim.x / 32) {
    int64_t seg = rs.seg_begin + id / rs.nrows;
    if (rs.skip_count > 0 && seg >= rs.skip_begin) seg += rs.skip_count;
    const int64_t r = seg * rs.seg_rows + rs.row0 + id % rs.nrows;
    const __nv_bfloat16* p = x + r * M;
    float s = 0.0f;
    if (vec) {
      const uint4* v = reinterpret_cast<const uint4*>(p);
      for (int i = lane; i < M / 8; i += 32) {
        const uint4 a = __ldg(v + i);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(h[q]);
          s = fmaf(f.x, f.x, fmaf(f.y, f.y, s));
        }
      }
    } else {
      for (int i = lane; i < M; i += 32) {
        const float f = __bfloat162float(p[i]);
        s = fmaf(f, f, s);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) rownorm[r] = sqrtf(s) * 1.001f;  // |x_row|_2, rounded up
  }
}

__global__ void wait_flags_kernel(FlagWait fw) {
  pdl_entry(); wait_flags_warp(fw); }

// For each listed (seg, row, col): h = sum_m X[seg][row][m] * W1T[g][col][m] in fp64, then
// act[seg][row][col] = bf16(max(h, 0)) and the ReLU bit. One warp per entry, two entries in
// flight per warp (the kernel is load-latency bound: two rows of x / W1^T per entry).
__device__ __forceinline__ double fixup_dot(const __nv_bfloat16* xr, const __nv_bfloat16* wr, int M,
                                            int lane) {
  double s = 0.0;
  if ((M & 7) == 0) {
    const uint4* xv = reinterpret_cast<const uint4*>(xr);
    const uint4* wv = reinterpret_cast<const uint4*>(wr);
    for (int v = lane; v < M / 8; v += 32) {
      const uint4 a = __ldg(xv + v), w = __ldg(wv + v);
      const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* wh = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 af = __bfloat1622float2(ah[q]), wf = __bfloat1622float2(wh[q]);
        s = fma(static_cast<double>(af.x), static_cast<double>(wf.x), s);
        s = fma(static_cast<double>(af.y), static_cast<double>(wf.y), s);
      }
    }
  } else {
    for (int m = lane; m < M; m += 32)
      s = fma(static_cast<double>(__bfloat162float(xr[m])), static_cast<double>(__bfloat162float(wr[m])), s);
  }
  return s;
}

#ifndef MOE_FIXUP_F32_PRODUCTS
#define MOE_FIXUP_F32_PRODUCTS 1
#endif

__global__ void __launch_bounds__(256, 2) relu_fixup_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w1t, int G, int seg_rows,
    int M, int V, const unsigned long long* __restrict__ list, const unsigned int* __restrict__ count,
    unsigned int cap, __nv_bfloat16* __restrict__ act, unsigned long long* __restrict__ relu_mask) {
  pdl_entry();
  // count[0]: entries listed by the up GEMM; count[1]: CTAs done; count[2]: the last list's size
  // (metrics); count[3]: the largest list since the host last read it (overflow check). The last CTA to finish resets [0] and [1], so the next chunk's up GEMM starts from
  // an empty list without a memset or reset kernel.
  const unsigned int n = min(__ldcg(count), cap);
  const int lane = threadIdx.x % 32;
  const unsigned int nw = gridDim.x * blockDim.x / 32;
  for (unsigned int i = (blockIdx.x * blockDim.x + threadIdx.x) / 32; i < n; i += 2 * nw) {
    const bool two = i + nw < n;
    const unsigned long long e[2] = {list[i], two ? list[i + nw] : list[i]};
    size_t r[2];
    uint32_t col[2];
    double s[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t seg = static_cast<uint32_t>(e[j] >> 44);
      const uint32_t row = static_cast<uint32_t>((e[j] >> 24) & 0xFFFFF);
      col[j] = static_cast<uint32_t>(e[j] & 0xFFFFFF);
      r[j] = static_cast<size_t>(seg) * seg_rows + row;
      MOE_CHECK(row < static_cast<uint32_t>(seg_rows) && col[j] < static_cast<uint32_t>(V), "relu fixup: entry out of range");
    }
    const __nv_bfloat16* xr[2];
    const __nv_bfloat16* wr[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      xr[j] = x + r[j] * M;
      wr[j] = w1t + (static_cast<size_t>(static_cast<uint32_t>(e[j] >> 44) % G) * V + col[j]) * M;
    }
    if ((M & 255) == 0) {
      // both entries' rows in flight 4 vectors per lane at a time before the fp64 math (the loop
      // is latency-bound on these gathers)
      constexpr int kV = 4;
      const int nv = M / 256;  // 16-byte vectors per lane per row
      double acc[2] = {0.0, 0.0};
      for (int v0 = 0; v0 < nv; v0 += kV) {
        uint4 av[2][kV], bv[2][kV];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int v = 0; v < kV; ++v)
            if (v0 + v < nv) {
              av[j][v] = __ldg(reinterpret_cast<const uint4*>(xr[j]) + (v0 + v) * 32 + lane);
              bv[j][v] = __ldg(reinterpret_cast<const uint4*>(wr[j]) + (v0 + v) * 32 + lane);
            }
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int v = 0; v < kV; ++v)
            if (v0 + v < nv) {
              const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&av[j][v]);
              const __nv_bfloat162* wh = reinterpret_cast<const __nv_bfloat162*>(&bv[j][v]);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float2 af = __bfloat1622float2(ah[q]), wf = __bfloat1622float2(wh[q]);
#if MOE_FIXUP_F32_PRODUCTS
                // bf16 x bf16 products are exact in fp32 (8 + 8 significand bits; down to
                // |product| ~ 2^-134, where a whole 1024-term row stays below 1e-37): one fp64
                // conversion per term instead of two, the sum still in fp64 (ncu: 17.8 -> 15.7 us)
                acc[j] += static_cast<double>(__fmul_rn(af.x, wf.x));
                acc[j] += static_cast<double>(__fmul_rn(af.y, wf.y));
#else
                acc[j] = fma(static_cast<double>(af.x), static_cast<double>(wf.x), acc[j]);
                acc[j] = fma(static_cast<double>(af.y), static_cast<double>(wf.y), acc[j]);
#endif
              }
            }
      }
      s[0] = acc[0];
      s[1] = acc[1];
    } else {
#pragma unroll
      for (int j = 0; j < 2; ++j) s[j] = fixup_dot(xr[j], wr[j], M, lane);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s[0] += __shfl_xor_sync(0xffffffffu, s[0], o);
      s[1] += __shfl_xor_sync(0xffffffffu, s[1], o);
    }
    if (lane < (two ? 2 : 1)) {
      const int j = lane;
      act[r[j] * V + col[j]] = __double2bfloat16(s[j] > 0.0 ? s[j] : 0.0);
      if (relu_mask) {
        unsigned long long* w = relu_mask + relu_mask_word(r[j], col[j] / 64, (V + 63) / 64);
        const unsigned long long bit = 1ull << relu_mask_bit(col[j] % 64);
        if (s[j] > 0.0) atomicOr(w, bit);
        else atomicAnd(w, ~bit);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int* c = const_cast<unsigned int*>(count);
    __threadfence();
    if (atomicAdd(c + 1, 1u) == gridDim.x - 1) {
      c[2] = c[0];
      c[3] = max(c[3], c[0]);  // sticky: the largest list since the last metrics read
      c[0] = 0u;
      c[1] = 0u;
    }
  }
}

// word (r, w) bit relu_mask_bit(i) = act[r][64 w + i] > 0 (one thread per 64-column word)
__global__ void mask_from_act_kernel(const __nv_bfloat16* __restrict__ act, int64_t rows, int V,
                                     unsigned long long* __restrict__ mask) {
  pdl_entry();
  const int nw = V / 64;
  const int64_t n = rows * nw;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const __nv_bfloat16* a = act + (i / nw) * V + (i % nw) * 64;
    unsigned long long b = 0ull;
    for (int j = 0; j < 64; ++j)
      b |= static_cast<unsigned long long>(__bfloat162float(a[j]) > 0.0f) << relu_mask_bit(j);
    mask[relu_mask_word(i / nw, static_cast<uint32_t>(i % nw), nw)] = b;
  }
}

}  // namespace

int relu_mask_from_act_device(const void* act, int64_t rows, int V, unsigned long long* mask,
                              cudaStream_t st) {
  const int64_t n = rows * (V / 64);
  const int grid = static_cast<int>(n / 256 + 1 < 148 * 16 ? n / 256 + 1 : 148 * 16);
  launch_k(mask_from_act_kernel, grid, 256, 0, st, static_cast<const __nv_bfloat16*>(act), rows, V, mask);
  return launch_status();
}

int weight_stats_device(const void* w1, int G, int M, int V, float* colnorm, float* colnorm_blk,
                        void* w1t, cudaStream_t st) {
  if (M % 64 == 0 && V % 64 == 0) {
    launch_k(weight_stats_kernel, G * (V / 64), 256, 0, st, static_cast<const __nv_bfloat16*>(w1), M,
             V, colnorm, colnorm_blk, static_cast<__nv_bfloat16*>(w1t));
    return launch_status();
  }
  const int n = G * V;
  launch_k(colnorm_kernel, (n + 255) / 256, 256, 0, st, static_cast<const __nv_bfloat16*>(w1), G, M, V,
                                                 colnorm);
  if (colnorm_blk && V % 64 == 0)
    launch_k(colnorm_blk_kernel, (G * V / 64 + 255) / 256, 256, 0, st, colnorm, G, V, colnorm_blk);
  dim3 grid((V + 31) / 32, (M + 31) / 32, G);
  launch_k(transpose_kernel, grid, dim3(32, 8), 0, st, static_cast<const __nv_bfloat16*>(w1), M, V,
                                                 static_cast<__nv_bfloat16*>(w1t));
  return launch_status();
}

int rownorm_device(const void* x, int M, float* rownorm, const RowSet& rs, cudaStream_t st,
                   const FlagWait* wait, unsigned int* reset) {
  const int64_t rows = static_cast<int64_t>(rs.nsegs) * rs.nrows;
  if (rows <= 0) return 0;
  const int64_t blocks = (rows + 7) / 8;
  const int grid = static_cast<int>(blocks < 148 * 4 ? blocks : 148 * 4);
  launch_k(rownorm_kernel, grid, 256, 0, st, static_cast<const __nv_bfloat16*>(x), M, rownorm, rs,
           wait ? *wait : FlagWait{}, reset);
  return launch_status();
}

int wait_flags_device(const FlagWait& w, cudaStream_t st) {
  launch_k(wait_flags_kernel, 1, 32, 0, st, w);
  return launch_status();
}

int relu_fixup_device(const void* x, const void* w1t, int G, int seg_rows, int M, int V,
                      const unsigned long long* list, const unsigned int* count, unsigned int cap,
                      void* act, unsigned long long* relu_mask, cudaStream_t st) {
  // one wave: the CTAs resident at once (2 per SM at this kernel's 128 registers) grid-stride
  // over the list, instead of 4 waves of mostly latency-bound CTAs
#ifndef MOE_FIXUP_CTAS_PER_SM
#define MOE_FIXUP_CTAS_PER_SM 2
#endif
  launch_k(relu_fixup_kernel, 148 * MOE_FIXUP_CTAS_PER_SM, 256, 0, st, static_cast<const __nv_bfloat16*>(x),
                                             static_cast<const __nv_bfloat16*>(w1t), G, seg_rows,
                                             M, V, list, count, cap,
                                             static_cast<__nv_bfloat16*>(act), relu_mask);
  return launch_status();
}

}  // namespace moe
