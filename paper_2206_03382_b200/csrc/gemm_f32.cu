// SIMT expert GEMMs. Same five GEMM kinds and segment addressing as the bf16 tcgen05 kernel
// (gemm_sm100.cu). The fp32 layer accumulates in fp64 (DFMA; fp32 x fp32 products are exact in
// fp64), so the ReLU mask [h > 0] agrees with the fp64 reference except for |h| < ~1e-13 and the
// 1e-5 bound holds for gradients too; the bf16 SIMT fallback accumulates in fp32. Used for (a) the fp32 layer path (1e-5 tolerance,
// config C1): the tensor cores have no fp32-exact mode (TF32 keeps 10 mantissa bits); and
// (b) bf16 shapes the tcgen05 tiling cannot take (N % 256, K % 64 or Mo % 128 != 0, e.g. the
// reference's tiny unit-test layers).
// Reference: expert_ffn / expert_ffn_backward, /root/reference/proj/src/parallelism.cpp:103-147.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <type_traits>

#include "gemm_sm100.h"
#include "kernels.h"

namespace moe {

namespace {

constexpr int TM = 64, TN = 64, TK = 16;

__device__ __forceinline__ float ldf(const float* p) { return *p; }
__device__ __forceinline__ float ldf(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ void stf(float* p, float v) { *p = v; }
__device__ __forceinline__ void stf(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

template <int kKind, typename T, typename TD>
__global__ void __launch_bounds__(256)
    gemm_simt_kernel(const T* __restrict__ A, const T* __restrict__ B, TD* __restrict__ D,
                     GemmArgs a) {
  __shared__ float As[TK][TM + 1];
  __shared__ float Bs[TK][TN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const bool rowk = kKind == kGemmWgrad;
  // Tile decode: z = group*S + segment (row-M) or group (row-K)
  const int n0 = blockIdx.x * TN;
  const int m0 = blockIdx.y * TM;
  int g, seg, rows;
  if (!rowk) {
    g = blockIdx.z / a.S;
    const int s = blockIdx.z % a.S;
    seg = (a.seg_base + s) * a.G + g;
    rows = a.seg_rows;
  } else {
    g = blockIdx.z;
    seg = 0;
    rows = a.Mo;
  }
  if (m0 >= rows) return;
  const int K = rowk ? a.S * a.seg_rows : a.K;
  using Acc = typename std::conditional<std::is_same<T, float>::value, double, float>::type;
  Acc acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int i = threadIdx.x; i < TK * TM; i += 256) {
      const int kk = i / TM, mm = i % TM;
      const int k = k0 + kk, m = m0 + mm;
      float v = 0.0f;
      if (k < K && m < rows) {
        if (!rowk) {
          v = ldf(&A[(static_cast<size_t>(seg) * a.seg_rows + m) * a.K + k]);
        } else {
          const int s = k / a.seg_rows, r = k % a.seg_rows;
          const size_t sg = static_cast<size_t>(a.seg_base + s) * a.G + g;
          v = ldf(&A[(sg * a.seg_rows + r) * a.Mo + m]);
        }
      }
      As[kk][mm] = v;
    }
    for (int i = threadIdx.x; i < TK * TN; i += 256) {
      const int kk = i / TN, nn = i % TN;
      const int k = k0 + kk, n = n0 + nn;
      float v = 0.0f;
      if (k < K && n < static_cast<int>(a.N)) {
        if (kKind == kGemmUp || kKind == kGemmDown) {
          v = ldf(&B[(static_cast<size_t>(g) * a.K + k) * a.N + n]);
        } else if (kKind == kGemmDgradMask || kKind == kGemmDgrad) {
          v = ldf(&B[(static_cast<size_t>(g) * a.N + n) * a.K + k]);
        } else {
          const int s = k / a.seg_rows, r = k % a.seg_rows;
          const size_t sg = static_cast<size_t>(a.seg_base + s) * a.G + g;
          v = ldf(&B[(sg * a.seg_rows + r) * a.N + n]);
        }
      }
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      Acc av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= static_cast<int>(a.N)) continue;
      float v = static_cast<float>(acc[i][j]);
      size_t off;
      if (!rowk)
        off = (static_cast<size_t>(seg) * a.seg_rows + m) * a.N + n;
      else
        off = (static_cast<size_t>(g) * a.Mo + m) * a.N + n;
      if (kKind == kGemmUp) {
        if (std::is_same<T, __nv_bfloat16>::value && a.fix_list != nullptr) {
          const float tau = a.rownorm[static_cast<size_t>(seg) * a.seg_rows + m] * kReluTauScale *
                            a.colnorm[static_cast<size_t>(g) * a.N + n];
          if (fabsf(v) < tau) {
            const unsigned int slot = atomicAdd(a.fix_count, 1u);
            if (slot < a.fix_cap) a.fix_list[slot] = fix_pack(seg, m, n);
          }
        }
        v = fmaxf(v, 0.0f);
      }
      if (kKind == kGemmDgradMask) v = ldf(static_cast<const T*>(a.aux) + off) > 0.0f ? v : 0.0f;
      stf(&D[off], v);
    }
  }
}

// fp32 layer (C1): the same five kinds on the FP64 tensor cores. fp32 operands are widened to
// fp64 once, when staged in shared memory, and mma.sync.m8n8k4.f64 (DMMA) accumulates in fp64:
// products are exact and the sums are fp64, as in gemm_simt_kernel<float>, at the DMMA rate
// instead of DFMA + per-use F2F conversions. CTA tile 64 x 64 x 16, 8 warps of 32 x 16 (4 m8 x
// 2 n8 tiles). Global loads run along each operand's contiguous dimension (K for row-major A and
// K-major B, M / N otherwise). Fragment layout (m8n8k4 .f64): A[r][c] r = lane/4, c = lane%4;
// B[r][c] r = lane%4, c = lane/4; D[r][2*(lane%4) + i] r = lane/4. Shared rows are padded to
// 68 doubles: a half-warp's 16 8-byte fragment loads then hit 16 distinct bank pairs.
// Tile sweep at C1 (ms/step): 64x64x16, 3 CTAs/SM 2.43; 64x64x32, 2/SM 2.52-2.55; 64x64x32 3/SM
// 2.52; 32x64x32 4/SM 2.67; 64x128x16 1/SM 2.95; 128x128x16 1/SM 2.73 -- occupancy hides the
// DMMA / shared-memory latencies better than per-warp operand reuse.
#ifndef MOE_F32_WMT
#define MOE_F32_WMT 4  // m8 tiles per warp (warps are 2 along M x 4 along N)
#endif
#ifndef MOE_F32_WNT
#define MOE_F32_WNT 2  // n8 tiles per warp
#endif
#ifndef MOE_F32_TK
#define MOE_F32_TK 16
#endif
#ifndef MOE_F32_MINB
#define MOE_F32_MINB 3
#endif
constexpr int DM_WMT = MOE_F32_WMT, DM_WNT = MOE_F32_WNT;
constexpr int DM_TM = 2 * 8 * DM_WMT, DM_TN = 4 * 8 * DM_WNT, DM_TK = MOE_F32_TK;
constexpr int DM_SA = DM_TM + 4, DM_SB = DM_TN + 4;  // padded rows: == 4 (mod 16) doubles
static_assert(DM_TK * DM_TM % 256 == 0 && DM_TK * DM_TN % 256 == 0, "stage / thread split");

__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int kKind>
__global__ void __launch_bounds__(256, MOE_F32_MINB)
    gemm_dmma_f32_kernel(const float* __restrict__ A, const float* __restrict__ B,
                         float* __restrict__ D, GemmArgs a) {
  __shared__ double As[DM_TK][DM_SA];
  __shared__ double Bs[DM_TK][DM_SB];
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const int wm = warp % 2, wn = warp / 2;  // warp tile rows [wm*8*WMT, +8*WMT), cols [wn*8*WNT, ...)
  const bool rowk = kKind == kGemmWgrad;
  const int n0 = blockIdx.x * DM_TN;
  const int m0 = blockIdx.y * DM_TM;
  int g, seg, rows;
  if (!rowk) {
    g = blockIdx.z / a.S;
    const int s = blockIdx.z % a.S;
    seg = (a.seg_base + s) * a.G + g;
    rows = a.seg_rows;
  } else {
    g = blockIdx.z;
    seg = 0;
    rows = a.Mo;
  }
  if (m0 >= rows) return;
  const int K = rowk ? a.S * a.seg_rows : a.K;
  const int N = static_cast<int>(a.N);
  constexpr bool kBk = kKind == kGemmDgradMask || kKind == kGemmDgrad;  // B is [N][K]
  double acc[DM_WMT][DM_WNT][2] = {};
  // register prefetch: stage k0 + DM_TK is loaded from global while stage k0 runs its DMMAs
  constexpr int kPer = DM_TK * DM_TM / 256, kPerB = DM_TK * DM_TN / 256;  // per thread per stage
  float ra[kPer], rb[kPerB];
  auto load_stage = [&](int k0) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int i = threadIdx.x + u * 256;
      int kk, mm;
      if (!rowk) { kk = i % DM_TK; mm = i / DM_TK; }  // A [rows][K]: K contiguous
      else { kk = i / DM_TM; mm = i % DM_TM; }        // A [K][Mo]: M contiguous
      const int k = k0 + kk, m = m0 + mm;
      float v = 0.0f;
      if (k < K && m < rows) {
        if (!rowk) {
          v = __ldg(A + (static_cast<size_t>(seg) * a.seg_rows + m) * a.K + k);
        } else {
          const int s = k / a.seg_rows, r = k % a.seg_rows;
          const size_t sg = static_cast<size_t>(a.seg_base + s) * a.G + g;
          v = __ldg(A + (sg * a.seg_rows + r) * a.Mo + m);
        }
      }
      ra[u] = v;
    }
#pragma unroll
    for (int u = 0; u < kPerB; ++u) {
      const int i = threadIdx.x + u * 256;
      int kk, nn;
      if (kBk) { kk = i % DM_TK; nn = i / DM_TK; }
      else { kk = i / DM_TN; nn = i % DM_TN; }
      const int k = k0 + kk, n = n0 + nn;
      float v = 0.0f;
      if (k < K && n < N) {
        if (kKind == kGemmUp || kKind == kGemmDown) {
          v = __ldg(B + (static_cast<size_t>(g) * a.K + k) * a.N + n);
        } else if (kBk) {
          v = __ldg(B + (static_cast<size_t>(g) * a.N + n) * a.K + k);
        } else {
          const int s = k / a.seg_rows, r = k % a.seg_rows;
          const size_t sg = static_cast<size_t>(a.seg_base + s) * a.G + g;
          v = __ldg(B + (sg * a.seg_rows + r) * a.N + n);
        }
      }
      rb[u] = v;
    }
  };
  load_stage(0);
  for (int k0 = 0; k0 < K; k0 += DM_TK) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int i = threadIdx.x + u * 256;
      if (!rowk) As[i % DM_TK][i / DM_TK] = static_cast<double>(ra[u]);
      else As[i / DM_TM][i % DM_TM] = static_cast<double>(ra[u]);
    }
#pragma unroll
    for (int u = 0; u < kPerB; ++u) {
      const int i = threadIdx.x + u * 256;
      if (kBk) Bs[i % DM_TK][i / DM_TK] = static_cast<double>(rb[u]);
      else Bs[i / DM_TN][i % DM_TN] = static_cast<double>(rb[u]);
    }
    __syncthreads();
    if (k0 + DM_TK < K) load_stage(k0 + DM_TK);
#pragma unroll
    for (int k4 = 0; k4 < DM_TK; k4 += 4) {
      double af[DM_WMT], bf[DM_WNT];
#pragma unroll
      for (int i = 0; i < DM_WMT; ++i) af[i] = As[k4 + lane % 4][wm * 8 * DM_WMT + i * 8 + lane / 4];
#pragma unroll
      for (int j = 0; j < DM_WNT; ++j) bf[j] = Bs[k4 + lane % 4][wn * 8 * DM_WNT + j * 8 + lane / 4];
#pragma unroll
      for (int i = 0; i < DM_WMT; ++i)
#pragma unroll
        for (int j = 0; j < DM_WNT; ++j) dmma_f64(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < DM_WMT; ++i) {
    const int m = m0 + wm * 8 * DM_WMT + i * 8 + lane / 4;
    if (m >= rows) continue;
#pragma unroll
    for (int j = 0; j < DM_WNT; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wn * 8 * DM_WNT + j * 8 + 2 * (lane % 4) + h;
        if (n >= N) continue;
        float v = static_cast<float>(acc[i][j][h]);
        size_t off;
        if (!rowk)
          off = (static_cast<size_t>(seg) * a.seg_rows + m) * a.N + n;
        else
          off = (static_cast<size_t>(g) * a.Mo + m) * a.N + n;
        if (kKind == kGemmUp) v = fmaxf(v, 0.0f);
        if (kKind == kGemmDgradMask) v = static_cast<const float*>(a.aux)[off] > 0.0f ? v : 0.0f;
        D[off] = v;
      }
    }
  }
}

int launch_dmma_f32(int kind, const float* A, const float* B, float* D, const GemmArgs& a,
                    cudaStream_t st) {
  if (a.row0 || a.nrows || a.skip_seg >= 0 || a.idx_mode) return -1;  // tcgen05-only features
  const bool rowk = kind == kGemmWgrad;
  const int rows = rowk ? a.Mo : a.seg_rows;
  dim3 grid((a.N + DM_TN - 1) / DM_TN, (rows + DM_TM - 1) / DM_TM, rowk ? a.G : a.G * a.S);
  switch (kind) {
    case kGemmUp: gemm_dmma_f32_kernel<kGemmUp><<<grid, 256, 0, st>>>(A, B, D, a); break;
    case kGemmDown: gemm_dmma_f32_kernel<kGemmDown><<<grid, 256, 0, st>>>(A, B, D, a); break;
    case kGemmDgradMask: gemm_dmma_f32_kernel<kGemmDgradMask><<<grid, 256, 0, st>>>(A, B, D, a); break;
    case kGemmDgrad: gemm_dmma_f32_kernel<kGemmDgrad><<<grid, 256, 0, st>>>(A, B, D, a); break;
    case kGemmWgrad: gemm_dmma_f32_kernel<kGemmWgrad><<<grid, 256, 0, st>>>(A, B, D, a); break;
    default: return -1;
  }
  return launch_status();
}

template <typename T, typename TD>
int launch_simt(int kind, const T* A, const T* B, TD* D, const GemmArgs& a, cudaStream_t st) {
  if (a.row0 || a.nrows || a.skip_seg >= 0 || a.idx_mode) return -1;  // tcgen05-only features
  const bool rowk = kind == kGemmWgrad;
  const int rows = rowk ? a.Mo : a.seg_rows;
  dim3 grid((a.N + TN - 1) / TN, (rows + TM - 1) / TM, rowk ? a.G : a.G * a.S);
  switch (kind) {
    case kGemmUp: gemm_simt_kernel<kGemmUp><<<grid, 256, 0, st>>>(A, B, D, a); break;
    case kGemmDown: gemm_simt_kernel<kGemmDown><<<grid, 256, 0, st>>>(A, B, D, a); break;
    case kGemmDgradMask: gemm_simt_kernel<kGemmDgradMask><<<grid, 256, 0, st>>>(A, B, D, a); break;
    case kGemmDgrad: gemm_simt_kernel<kGemmDgrad><<<grid, 256, 0, st>>>(A, B, D, a); break;
    case kGemmWgrad: gemm_simt_kernel<kGemmWgrad><<<grid, 256, 0, st>>>(A, B, D, a); break;
    default: return -1;
  }
  return launch_status();
}

}  // namespace

int gemm_f32(int kind, const float* A, const float* B, float* D, const GemmArgs& a,
             cudaStream_t st) {
  static const bool simt = [] {
    const char* e = std::getenv("MOE_F32_SIMT");  // A/B: the DFMA SIMT kernel
    return e != nullptr && e[0] == '1';
  }();
  if (simt) return launch_simt<float, float>(kind, A, B, D, a, st);
  return launch_dmma_f32(kind, A, B, D, a, st);
}

// bf16 operands, fp32 accumulation; bf16 output except wgrad (fp32).
int gemm_bf16_simt(int kind, const void* A, const void* B, void* D, const GemmArgs& a,
                   cudaStream_t st) {
  using Bf = __nv_bfloat16;
  if (kind == kGemmWgrad)
    return launch_simt<Bf, float>(kind, static_cast<const Bf*>(A), static_cast<const Bf*>(B),
                                  static_cast<float*>(D), a, st);
  return launch_simt<Bf, Bf>(kind, static_cast<const Bf*>(A), static_cast<const Bf*>(B),
                             static_cast<Bf*>(D), a, st);
}

}  // namespace moe
