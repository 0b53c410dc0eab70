// Gating on sm_100a: fp64 router GEMM + row softmax + top-k (one warp per token), then the
// capacity-slot assignment as a per-expert rank computation.
//
// Reference semantics (all bit-exact in idxs / locations / drop mask):
//   gate_linear + softmax_rows   /root/reference/proj/src/gating.cpp:19-35
//   topk_select (desc prob, asc index tie-break)       gating.cpp:58-78
//   assign_locations FIFO / BPR                        gating.cpp:80-112
//   expert_demand, run_gating_blocked                  gating.cpp:114-162
//   resolve_capacity / expert_capacity                 core.cpp:28-59
//
// Slot assignment restated: processing tokens in an order O (token order for FIFO; BPR: max gate
// descending, ties by token index) and giving each (t, j) the next free slot of expert e gives
//   loc(t, j) = r  if r < capacity else -1,   r = #{t' before t in O : e in idxs(t')}
// because experts are distinct within a row. FIFO r is a per-expert exclusive prefix count over
// the flattened (t, j) grid (block histogram + scan + warp match ranks); BPR r is the rank of t's
// key inside expert e's member list (counted against every other member, exact fp64 compares).
#include <cuda_runtime.h>
#include <cstdlib>

#include <cfloat>
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "checks.cuh"
#include "kernels.h"
#include "pdl.cuh"

namespace moe {

namespace {

#ifndef MOE_GATE_WARPS
#define MOE_GATE_WARPS 8  // token block of the gate / assign partition = 8 tokens per warp
#endif
// DMMA gate CTA: MOE_DM_WARPS warps x MOE_DM_MT 8-token m-tiles = the 64-token block. Measured
// at TGT: 8 warps x 1 m-tile 113 us, 4 x 2 123 us, 32-token blocks (2 x 2 / 4 x 1) 122-148 us,
// K split over two warp groups 120 us -- warps in flight beat operand reuse here. sm_100a has
// only the DMMA.8x8x4 unit (mma.m16n8k16.f64 compiles to 8 of them), so m8n8k4 loses nothing.
#ifndef MOE_DM_WARPS
#define MOE_DM_WARPS 8
#endif
#ifndef MOE_DM_MT
#define MOE_DM_MT 1
#endif
constexpr int kGateWarps = MOE_GATE_WARPS;
constexpr int kGateTokPerWarp = 8;
constexpr int kGateTok = kGateWarps * kGateTokPerWarp;  // 64 tokens per CTA

template <typename T>
__device__ __forceinline__ double to_f64(T v);
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) {
  return static_cast<double>(__bfloat162float(v));
}
template <>
__device__ __forceinline__ double to_f64<float>(float v) {
  return static_cast<double>(v);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// x: [blocks*T, M] (bf16 or f32), wg: [M, E] fp64 row-major.
// Outputs idxs/gates [blocks*T, k], hist [n_cta, E] (per-CTA expert counts), optional probs.
// Each warp owns 8 tokens; lane l owns experts l + 32j (j < EPL) and keeps the current Wg chunk in
// registers, while the token values come from shared memory as warp broadcasts. The next chunk
// of x / Wg is prefetched into registers during the current chunk's DFMAs (double-buffered smem,
// one barrier per chunk). Summation per (token, expert) is a single sequential fma chain over m.
template <typename TX, int EPL>
__global__ void __launch_bounds__(kGateWarps * 32)
    gate_topk_kernel(const TX* __restrict__ x, const double* __restrict__ wg, int T, int M, int E,
                     int k, int cta_per_block, int32_t* __restrict__ idxs,
                     double* __restrict__ gates, int32_t* __restrict__ hist,
                     double* __restrict__ probs_out) {
  pdl_entry();
  constexpr int KC = 16 / EPL;  // k-chunk staged through smem (2 x 24 KiB static smem at EPL=1)
  constexpr int NT = kGateWarps * 32;
  constexpr int XPT = (kGateTok * KC + NT - 1) / NT;  // x elements per thread per chunk
  constexpr int WPT = (KC * 32 * EPL + NT - 1) / NT;  // Wg elements per thread per chunk
  __shared__ __align__(16) double xs[2][kGateTok][KC];
  __shared__ __align__(16) double ws[2][KC][32 * EPL];
  extern __shared__ int32_t sh_hist[];  // [E]

  const int b = blockIdx.x / cta_per_block;
  const int c = blockIdx.x % cta_per_block;
  const int t_begin = b * T + c * kGateTok;
  const int t_end = min(b * T + T, t_begin + kGateTok);
  const int ntok = t_end - t_begin;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  for (int e = threadIdx.x; e < E; e += blockDim.x) sh_hist[e] = 0;

  double acc[kGateTokPerWarp][EPL];
#pragma unroll
  for (int i = 0; i < kGateTokPerWarp; ++i)
#pragma unroll
    for (int j = 0; j < EPL; ++j) acc[i][j] = 0.0;

  double xr[XPT], wrg[WPT];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int q = 0; q < XPT; ++q) {
      const int i = threadIdx.x + q * NT;
      const int tt = i / KC, kk = i % KC;
      xr[q] = (i < kGateTok * KC && tt < ntok && k0 + kk < M)
                  ? to_f64(x[static_cast<size_t>(t_begin + tt) * M + k0 + kk])
                  : 0.0;
    }
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      const int i = threadIdx.x + q * NT;
      const int kk = i / (32 * EPL), e = i % (32 * EPL);
      wrg[q] = (i < KC * 32 * EPL && k0 + kk < M && e < E)
                   ? __ldg(wg + static_cast<size_t>(k0 + kk) * E + e)
                   : 0.0;
    }
  };
  auto store_chunk = [&](int buf) {
#pragma unroll
    for (int q = 0; q < XPT; ++q) {
      const int i = threadIdx.x + q * NT;
      if (i < kGateTok * KC) xs[buf][i / KC][i % KC] = xr[q];
    }
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      const int i = threadIdx.x + q * NT;
      if (i < KC * 32 * EPL) ws[buf][i / (32 * EPL)][i % (32 * EPL)] = wrg[q];
    }
  };

  const int nchunks = (M + KC - 1) / KC;
  load_chunk(0);
  store_chunk(0);
  __syncthreads();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) load_chunk((ch + 1) * KC);  // global loads in flight during DFMAs
    double wr[KC][EPL];
#pragma unroll
    for (int kk = 0; kk < KC; ++kk)
#pragma unroll
      for (int j = 0; j < EPL; ++j) wr[kk][j] = ws[buf][kk][lane + 32 * j];
#pragma unroll
    for (int i = 0; i < kGateTokPerWarp; ++i) {
      const int tt = warp * kGateTokPerWarp + i;
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        const double xv = xs[buf][tt][kk];  // warp broadcast
#pragma unroll
        for (int j = 0; j < EPL; ++j) acc[i][j] = fma(xv, wr[kk][j], acc[i][j]);
      }
    }
    if (ch + 1 < nchunks) store_chunk(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < kGateTokPerWarp; ++i) {
    const int tt = warp * kGateTokPerWarp + i;
    if (tt >= ntok) break;  // warp-uniform
    const int t = t_begin + tt;
    double mx = -DBL_MAX;
#pragma unroll
    for (int j = 0; j < EPL; ++j)
      if (lane + 32 * j < E) mx = fmax(mx, acc[i][j]);
    mx = warp_max(mx);
    double ex[EPL];
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      ex[j] = (lane + 32 * j < E) ? exp(acc[i][j] - mx) : 0.0;
      s += ex[j];
    }
    s = warp_sum(s);
    double p[EPL];
#pragma unroll
    for (int j = 0; j < EPL; ++j) p[j] = ex[j] / s;
    if (probs_out) {
#pragma unroll
      for (int j = 0; j < EPL; ++j)
        if (lane + 32 * j < E) probs_out[static_cast<size_t>(t) * E + lane + 32 * j] = p[j];
    }
    unsigned taken = 0;  // bit j: this lane's expert lane+32j already selected
    for (int r = 0; r < k; ++r) {
      double bv = -1.0;
      int bi = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < EPL; ++j) {
        const int e = lane + 32 * j;
        if (e < E && !(taken & (1u << j)) && (p[j] > bv || (p[j] == bv && e < bi))) {
          bv = p[j];
          bi = e;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
      if (lane == 0) {
        idxs[static_cast<size_t>(t) * k + r] = bi;
        gates[static_cast<size_t>(t) * k + r] = bv;
        atomicAdd(&sh_hist[bi], 1);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    hist[static_cast<size_t>(blockIdx.x) * E + e] = sh_hist[e];
}

// FP64 tensor-core variant (E <= 64): mma.sync.m8n8k4.f64 (DMMA). A warp owns MT m8-tiles of
// tokens x NT n8-tiles of experts; per 4-deep k step it loads MT A-fragments (x) and NT
// B-fragments (Wg) from padded, conflict-free shared memory and issues MT*NT DMMAs (256 fp64
// FMAs each). Products of the bf16/fp32 inputs with fp64 Wg are exact in fp64; only the
// accumulation order differs from the reference's Eigen GEMM (ulp-level, below any routing tie).
// Fragment layout (m8n8k4 .f64): A[r][c] with r = lane/4, c = lane%4; B[r][c] with r = lane%4,
// c = lane/4; D[r][2*(lane%4) + i] with r = lane/4.
constexpr int kDmWarps = MOE_DM_WARPS, kDmMT = MOE_DM_MT, kDmTok = kDmWarps * kDmMT * 8, kDmKC = 16;
static_assert(kDmTok == kGateTok, "gate kernels must share the token-block partition of assign");

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <typename TX, int NT>
__global__ void __launch_bounds__(kDmWarps * 32)
    gate_dmma_kernel(const TX* __restrict__ x, const double* __restrict__ wg, int T, int M, int E,
                     int k, int cta_per_block, int32_t* __restrict__ idxs,
                     double* __restrict__ gates, int32_t* __restrict__ hist,
                     double* __restrict__ probs_out) {
  pdl_entry();
  constexpr int NTH = kDmWarps * 32;
  constexpr int XS = kDmKC + 4;       // x row stride (doubles): conflict-free A fragments
  constexpr int EP = 8 * NT + 4;      // Wg row stride: conflict-free B fragments
  constexpr int XPT = kDmTok * kDmKC / NTH;
  constexpr int WPT = (kDmKC * 8 * NT + NTH - 1) / NTH;
  __shared__ __align__(16) double xs[2][kDmTok][XS];
  __shared__ __align__(16) double ws[2][kDmKC][EP];
  __shared__ int32_t sh_hist[8 * NT];

  const int b = blockIdx.x / cta_per_block;
  const int c = blockIdx.x % cta_per_block;
  const int t_begin = b * T + c * kDmTok;
  const int ntok = min(b * T + T, t_begin + kDmTok) - t_begin;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int e = threadIdx.x; e < 8 * NT; e += NTH) sh_hist[e] = 0;

  double acc[kDmMT][NT][2];
#pragma unroll
  for (int i = 0; i < kDmMT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double xr[XPT], wr[WPT];
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int q = 0; q < XPT; ++q) {
      const int i = threadIdx.x + q * NTH;
      const int tt = i / kDmKC, kk = i % kDmKC;
      xr[q] = (tt < ntok && k0 + kk < M) ? to_f64(x[static_cast<size_t>(t_begin + tt) * M + k0 + kk])
                                         : 0.0;
    }
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      const int i = threadIdx.x + q * NTH;
      const int kk = i / (8 * NT), e = i % (8 * NT);
      wr[q] = (i < kDmKC * 8 * NT && k0 + kk < M && e < E)
                  ? __ldg(wg + static_cast<size_t>(k0 + kk) * E + e)
                  : 0.0;
    }
  };
  auto store_chunk = [&](int buf) {
#pragma unroll
    for (int q = 0; q < XPT; ++q) {
      const int i = threadIdx.x + q * NTH;
      xs[buf][i / kDmKC][i % kDmKC] = xr[q];
    }
#pragma unroll
    for (int q = 0; q < WPT; ++q) {
      const int i = threadIdx.x + q * NTH;
      if (i < kDmKC * 8 * NT) ws[buf][i / (8 * NT)][i % (8 * NT)] = wr[q];
    }
  };

  const int nchunks = (M + kDmKC - 1) / kDmKC;
  load_chunk(0);
  store_chunk(0);
  __syncthreads();
  const int ar = lane >> 2, ac = lane & 3;
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) load_chunk((ch + 1) * kDmKC);
#pragma unroll
    for (int ks = 0; ks < kDmKC; ks += 4) {
      double a[kDmMT], bb[NT];
#pragma unroll
      for (int i = 0; i < kDmMT; ++i) a[i] = xs[buf][(warp * kDmMT + i) * 8 + ar][ks + ac];
#pragma unroll
      for (int j = 0; j < NT; ++j) bb[j] = ws[buf][ks + ac][j * 8 + ar];
#pragma unroll
      for (int i = 0; i < kDmMT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], bb[j]);
    }
    if (ch + 1 < nchunks) store_chunk(buf ^ 1);
    __syncthreads();
  }

  // softmax + top-k: the 4 lanes of a quad (same lane/4) hold one token's 8*NT logits.
#pragma unroll
  for (int i = 0; i < kDmMT; ++i) {
    const int tt = (warp * kDmMT + i) * 8 + ar;
    const bool tok_ok = tt < ntok;
    const int t = t_begin + tt;
    double mx = -DBL_MAX;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (j * 8 + ac * 2 + h < E) mx = fmax(mx, acc[i][j][h]);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    double p[NT][2];
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        p[j][h] = (j * 8 + ac * 2 + h < E) ? exp(acc[i][j][h] - mx) : 0.0;
        s += p[j][h];
      }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        p[j][h] /= s;
        const int e = j * 8 + ac * 2 + h;
        if (probs_out && tok_ok && e < E) probs_out[static_cast<size_t>(t) * E + e] = p[j][h];
      }
    unsigned taken = 0;
    for (int r = 0; r < k; ++r) {
      double bv = -1.0;
      int bi = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = j * 8 + ac * 2 + h;
          if (e < E && !(taken & (1u << (j * 2 + h))) && (p[j][h] > bv || (p[j][h] == bv && e < bi))) {
            bv = p[j][h];
            bi = e;
          }
        }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (((bi & 7) >> 1) == ac) taken |= 1u << ((bi >> 3) * 2 + (bi & 1));
      if (ac == 0 && tok_ok) {
        idxs[static_cast<size_t>(t) * k + r] = bi;
        gates[static_cast<size_t>(t) * k + r] = bv;
        atomicAdd(&sh_hist[bi], 1);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += NTH) hist[static_cast<size_t>(blockIdx.x) * E + e] = sh_hist[e];
}

// Pipelined DMMA gate (E <= 64, 16-byte aligned rows): raw x / Wg tiles stream into a 3-stage
// shared-memory ring with cp.async (no register staging; two chunks in flight while the DMMAs
// of the current one run); x is converted bf16/f32 -> fp64 when the A fragment is loaded.
constexpr int kD2KC = 32, kD2Stages = 3;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool pred) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  const int sz = pred ? 16 : 0;  // src-size 0: zero-fill (token / k / expert tail)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename TX>
__device__ __forceinline__ double ld_x(const TX* p);
template <>
__device__ __forceinline__ double ld_x<__nv_bfloat16>(const __nv_bfloat16* p) {
  return static_cast<double>(__bfloat162float(*p));
}
template <>
__device__ __forceinline__ double ld_x<float>(const float* p) {
  return static_cast<double>(*p);
}

template <>
__device__ __forceinline__ double ld_x<double>(const double* p) {
  return *p;
}

template <typename TX, int NT>
struct D2Cfg {
  static constexpr int XROW = kD2KC * sizeof(TX) + 16;       // bytes per staged token row (padded)
  static constexpr int EP = 8 * NT + 4;                       // W row stride in smem (doubles)
  static constexpr int XBYTES = kDmTok * XROW;
  static constexpr int WBYTES = kD2KC * EP * 8;
  static constexpr int STAGE = XBYTES + WBYTES;
  static constexpr int SMEM = kD2Stages * STAGE + 8 * NT * 4 + 16;
};

// Epilogue of the pipelined DMMA x . W kernel.
enum DmmaMode : int {
  kDmGate = 0,    // logits -> softmax -> top-k + per-CTA histogram (gate_linear, gating.cpp:29-35)
  kDmRaw = 1,     // fp64 rows out (the cosine router's projection x . P, gating.cpp:43)
  kDmCosine = 2,  // logits / (|a_t| |C_e| tau) -> softmax -> top-k (gate_cosine, gating.cpp:50-55)
};

struct DmmaArgs {
  const void* x;        // A: [rows][K] (bf16 / f32 / f64), rows of the 64-token blocks
  const double* w;      // W: [K][ldw] fp64, columns [0, ncols)
  int ldw, ncols, T, K, k, cpb;
  int32_t* idxs;        // gate modes
  double* gates;
  int32_t* hist;
  double* probs_out;
  double* out;          // kDmRaw: [rows][ldo]
  int ldo;
  const double* en;     // kDmCosine: |C_e|
  double tau;           // kDmCosine: max(temperature, 0.01)
  int32_t* err;         // kDmCosine: set to 1 on a zero-norm projected token
};

template <typename TX, int NT, int kMode>
__global__ void __launch_bounds__(kDmWarps * 32) gate_dmma2_kernel(DmmaArgs a) {
  pdl_entry();
  using Cf = D2Cfg<TX, NT>;
  constexpr int NTH = kDmWarps * 32;
  constexpr int XCH = kD2KC * sizeof(TX) / 16;  // 16-byte chunks per token row
  constexpr int WCH = 8 * NT * 8 / 16;          // 16-byte chunks per W row (8*NT doubles)
  extern __shared__ __align__(16) uint8_t sm[];
  int32_t* sh_hist = reinterpret_cast<int32_t*>(sm + kD2Stages * Cf::STAGE);
  const TX* __restrict__ x = static_cast<const TX*>(a.x);
  const int M = a.K, E = a.ncols;
  const int n0 = kMode == kDmRaw ? blockIdx.y * 8 * NT : 0;

  const int b = blockIdx.x / a.cpb;
  const int c = blockIdx.x % a.cpb;
  const int t_begin = b * a.T + c * kDmTok;
  const int ntok = min(b * a.T + a.T, t_begin + kDmTok) - t_begin;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int e = threadIdx.x; e < 8 * NT; e += NTH) sh_hist[e] = 0;

  auto issue = [&](int ch) {
    const int k0 = ch * kD2KC;
    uint8_t* st = sm + (ch % kD2Stages) * Cf::STAGE;
    for (int i = threadIdx.x; i < kDmTok * XCH; i += NTH) {
      const int tt = i / XCH, q = i % XCH;
      const int kk = q * (16 / static_cast<int>(sizeof(TX)));
      const bool ok = tt < ntok && k0 + kk < M;
      const TX* src = ok ? x + static_cast<size_t>(t_begin + tt) * M + k0 + kk : x;
      cp_async16(st + tt * Cf::XROW + q * 16, src, ok);
    }
    double* ws = reinterpret_cast<double*>(st + Cf::XBYTES);
    for (int i = threadIdx.x; i < kD2KC * WCH; i += NTH) {
      const int kk = i / WCH, q = i % WCH;
      const int e = q * 2;
      const bool ok = k0 + kk < M && n0 + e < E;
      const double* src = ok ? a.w + static_cast<size_t>(k0 + kk) * a.ldw + n0 + e : a.w;
      cp_async16(ws + kk * Cf::EP + e, src, ok);
    }
  };

  double acc[kDmMT][NT][2];
  double ss[kDmMT];  // kDmCosine: sum of squares of this lane's A elements (token norm)
#pragma unroll
  for (int i = 0; i < kDmMT; ++i) {
    ss[i] = 0.0;
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }

  const int nch = (M + kD2KC - 1) / kD2KC;
  issue(0);
  cp_async_commit();
  if (nch > 1) issue(1);
  cp_async_commit();
  const int ar = lane >> 2, ac = lane & 3;
  for (int ch = 0; ch < nch; ++ch) {
    cp_async_wait<1>();  // chunk ch has landed (this thread's copies)
    __syncthreads();     // ... and everyone's; buffer (ch+2)%3 is free
    if (ch + 2 < nch) issue(ch + 2);
    cp_async_commit();
    const uint8_t* st = sm + (ch % kD2Stages) * Cf::STAGE;
    const double* ws = reinterpret_cast<const double*>(st + Cf::XBYTES);
#pragma unroll
    for (int ks = 0; ks < kD2KC; ks += 4) {
      double av[kDmMT], bb[NT];
#pragma unroll
      for (int i = 0; i < kDmMT; ++i) {
        av[i] = ld_x<TX>(reinterpret_cast<const TX*>(st + ((warp * kDmMT + i) * 8 + ar) * Cf::XROW) + ks + ac);
        if constexpr (kMode == kDmCosine) ss[i] = fma(av[i], av[i], ss[i]);
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) bb[j] = ws[(ks + ac) * Cf::EP + j * 8 + ar];
#pragma unroll
      for (int i = 0; i < kDmMT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], av[i], bb[j]);
    }
  }
  if constexpr (kMode == kDmRaw) {
    // fragment (i, j, h) = row (warp * MT + i) * 8 + ar, column j * 8 + ac * 2 + h
#pragma unroll
    for (int i = 0; i < kDmMT; ++i) {
      const int tt = (warp * kDmMT + i) * 8 + ar;
      if (tt >= ntok) continue;
      double* orow = a.out + static_cast<size_t>(t_begin + tt) * a.ldo;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = n0 + j * 8 + ac * 2 + h;
          if (e < E) orow[e] = acc[i][j][h];
        }
    }
    return;
  }
  if constexpr (kMode == kDmCosine) {
    // logits[t][e] = <a_t, C_e> / (|a_t| |C_e| tau) (gating.cpp:50-54)
#pragma unroll
    for (int i = 0; i < kDmMT; ++i) {
      double q = ss[i];
      q += __shfl_xor_sync(0xffffffffu, q, 1);
      q += __shfl_xor_sync(0xffffffffu, q, 2);
      const double tn = sqrt(q);
      const int tt = (warp * kDmMT + i) * 8 + ar;
      if (tn == 0.0 && tt < ntok && ac == 0) atomicExch(a.err, 1);
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = j * 8 + ac * 2 + h;
          if (e < E) acc[i][j][h] = acc[i][j][h] / (tn * __ldg(a.en + e) * a.tau);
        }
    }
  }
  const int T = a.T, k = a.k;
  int32_t* __restrict__ idxs = a.idxs;
  double* __restrict__ gates = a.gates;
  int32_t* __restrict__ hist = a.hist;
  double* __restrict__ probs_out = a.probs_out;
  (void)T;
  // softmax + top-k: the 4 lanes of a quad (same lane/4) hold one token's 8*NT logits.
#pragma unroll
  for (int i = 0; i < kDmMT; ++i) {
    const int tt = (warp * kDmMT + i) * 8 + ar;
    const bool tok_ok = tt < ntok;
    const int t = t_begin + tt;
    double mx = -DBL_MAX;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (j * 8 + ac * 2 + h < E) mx = fmax(mx, acc[i][j][h]);
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    double p[NT][2];
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        p[j][h] = (j * 8 + ac * 2 + h < E) ? exp(acc[i][j][h] - mx) : 0.0;
        s += p[j][h];
      }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        p[j][h] /= s;
        const int e = j * 8 + ac * 2 + h;
        if (probs_out && tok_ok && e < E) probs_out[static_cast<size_t>(t) * E + e] = p[j][h];
      }
    unsigned taken = 0;
    for (int r = 0; r < k; ++r) {
      double bv = -1.0;
      int bi = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = j * 8 + ac * 2 + h;
          if (e < E && !(taken & (1u << (j * 2 + h))) && (p[j][h] > bv || (p[j][h] == bv && e < bi))) {
            bv = p[j][h];
            bi = e;
          }
        }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (((bi & 7) >> 1) == ac) taken |= 1u << ((bi >> 3) * 2 + (bi & 1));
      if (ac == 0 && tok_ok) {
        idxs[static_cast<size_t>(t) * k + r] = bi;
        gates[static_cast<size_t>(t) * k + r] = bv;
        atomicAdd(&sh_hist[bi], 1);
      }
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += NTH) hist[static_cast<size_t>(blockIdx.x) * E + e] = sh_hist[e];
}

__device__ void finalize_capacity_cta(int blocks, int E, int T, int k, int cap_kind, int cap_formula,
                                      const int32_t* __restrict__ demand, int32_t* __restrict__ list_base,
                                      int32_t* __restrict__ fill, int32_t* __restrict__ cap_out,
                                      int32_t* __restrict__ drops);

struct FinalizeArgs {
  int32_t* done;  // null: the separate finalize kernel runs
  int blocks, T, k, cap_kind, cap_formula;
  int32_t *list_base, *fill, *cap, *drops;
};

// Per (block, expert) column: exclusive scan of the CTA histograms -> offs, demand.
// One CTA per column; each thread scans a contiguous run of CTA counts, then a block scan.
__global__ void __launch_bounds__(256)
    scan_cols_kernel(const int32_t* __restrict__ hist, int cta_per_block, int E,
                     int32_t* __restrict__ offs, int32_t* __restrict__ demand, FinalizeArgs fa) {
  pdl_entry();
  __shared__ int32_t wsum[8];
  const int p = blockIdx.x, b = p / E, e = p % E;
  const int per = (cta_per_block + blockDim.x - 1) / blockDim.x;
  const int c0 = threadIdx.x * per;
  int local[16];  // cta_per_block <= 4096 (T <= 256K tokens per block)
  int sum = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = c0 + i;
    local[i] = (i < per && c < cta_per_block) ? hist[static_cast<size_t>(b * cta_per_block + c) * E + e] : 0;
    sum += local[i];
  }
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  int inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < warp; ++w) base += wsum[w];
  int run = base + inc - sum;  // exclusive prefix of this thread's run
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int c = c0 + i;
    if (i < per && c < cta_per_block) offs[static_cast<size_t>(b * cta_per_block + c) * E + e] = run;
    run += local[i];
  }
  if (threadIdx.x == blockDim.x - 1) demand[p] = run;
  if (fa.done == nullptr) return;
  // the last column CTA to finish resolves the capacity (finalize_capacity_kernel's work)
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(fa.done, 1) == static_cast<int>(gridDim.x) - 1;
    if (last) *fa.done = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  finalize_capacity_cta(fa.blocks, E, fa.T, fa.k, fa.cap_kind, fa.cap_formula, demand, fa.list_base,
                        fa.fill, fa.cap, fa.drops);
}

// resolve_capacity (core.cpp:47-59) over the per-block max demand, fill counts and the BPR
// member-list bases. One small CTA.
// resolve_capacity body (one CTA of 256 threads): shared by the standalone kernel and the scan's
// last CTA. Every demand is loaded once, in parallel; member-list bases are a block-wide
// exclusive scan over the experts of each source block.
__device__ void finalize_capacity_cta(int blocks, int E, int T, int k, int cap_kind, int cap_formula,
                                      const int32_t* __restrict__ demand, int32_t* __restrict__ list_base,
                                      int32_t* __restrict__ fill, int32_t* __restrict__ cap_out,
                                      int32_t* __restrict__ drops) {
  __shared__ int32_t cap_sh;
  __shared__ int32_t mx_sh;
  __shared__ int32_t wsum[8];
  if (threadIdx.x == 0) {
    *drops = 0;  // the assign pass accumulates this step's drops
    mx_sh = 1;   // max demand floors at 1
  }
  __syncthreads();
  for (int p = threadIdx.x; p < blocks * E; p += blockDim.x) atomicMax(&mx_sh, __ldcg(demand + p));
  __syncthreads();
  if (threadIdx.x == 0) {
    int cap = cap_formula;
    if (cap_kind == 1) cap = mx_sh;                      // Auto
    if (cap_kind == 2) cap = min(mx_sh, cap_formula);    // Bounded (formula at max_factor)
    cap_sh = cap;
    *cap_out = cap;
  }
  __syncthreads();
  const int cap = cap_sh;
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nw = blockDim.x / 32;
  for (int b = 0; b < blocks; ++b) {
    int run = b * T * k;  // running base across chunks of blockDim.x experts
    for (int e0 = 0; e0 < E; e0 += blockDim.x) {
      const int e = e0 + threadIdx.x;
      const int d = e < E ? __ldcg(demand + b * E + e) : 0;
      int inc = d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      if (lane == 31) wsum[warp] = inc;
      __syncthreads();
      int base = run;
      for (int w = 0; w < warp; ++w) base += wsum[w];
      if (e < E) {
        list_base[b * E + e] = base + inc - d;
        fill[b * E + e] = min(d, cap);
      }
      int tot = 0;
      for (int w = 0; w < nw; ++w) tot += wsum[w];
      run += tot;
      __syncthreads();
    }
  }
}

__global__ void finalize_capacity_kernel(int blocks, int E, int T, int k, int cap_kind,
                                         int cap_formula, const int32_t* __restrict__ demand,
                                         int32_t* __restrict__ list_base,
                                         int32_t* __restrict__ fill, int32_t* __restrict__ cap_out,
                                         int32_t* __restrict__ drops) {
  pdl_entry();
  finalize_capacity_cta(blocks, E, T, k, cap_kind, cap_formula, demand, list_base, fill, cap_out, drops);
}

// FIFO ranks over the flattened (t, j) grid of each gate CTA. bpr==0: write locations + slots.
// bpr==1: write the member list (FIFO order) for the BPR rank kernel.
__global__ void __launch_bounds__(256)
    assign_kernel(const int32_t* __restrict__ idxs, const double* __restrict__ gates, int T, int k,
                  int E, int cta_per_block, const int32_t* __restrict__ offs,
                  const int32_t* __restrict__ list_base, const int32_t* __restrict__ cap_ptr,
                  int bpr, int32_t* __restrict__ locations, int32_t* __restrict__ slot_token,
                  float* __restrict__ slot_gate, int32_t* __restrict__ list,
                  int32_t* __restrict__ drops, const int32_t* __restrict__ demand) {
  pdl_entry();
  extern __shared__ int32_t sh[];  // cnt[E] + wcnt[8][E]
  int32_t* cnt = sh;
  int32_t* wcnt = sh + E;
  const int b = blockIdx.x / cta_per_block;
  const int c = blockIdx.x % cta_per_block;
  const int t_begin = b * T + c * kGateTok;
  const int t_end = min(b * T + T, t_begin + kGateTok);
  const int f_begin = t_begin * k, f_end = t_end * k;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int cap = *cap_ptr;
  if (c == 0) {
    // slots [min(demand, cap), cap) of this block's experts stay empty (FIFO and BPR both fill
    // 0 .. min(demand, cap) - 1): token -1, gate 0 -- encode zero-fills those rows
    for (int e = 0; e < E; ++e) {
      const int d0 = min(demand[static_cast<size_t>(b) * E + e], cap);
      for (int s = d0 + threadIdx.x; s < cap; s += blockDim.x) {
        const size_t slot = static_cast<size_t>(b * E + e) * cap + s;
        slot_token[slot] = -1;
        slot_gate[slot] = 0.0f;
      }
    }
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    cnt[e] = offs[static_cast<size_t>(blockIdx.x) * E + e];
  int my_drops = 0;
  for (int base = f_begin; base < f_end; base += 256) {
    for (int i = threadIdx.x; i < 8 * E; i += blockDim.x) wcnt[i] = 0;
    __syncthreads();
    const int f = base + threadIdx.x;
    const bool active = f < f_end;
    const int e = active ? idxs[f] : -1;
    const unsigned grp = __match_any_sync(0xffffffffu, e);
    const int in_warp = __popc(grp & ((1u << lane) - 1u));
    if (active && in_warp == 0) wcnt[warp * E + e] = __popc(grp);
    __syncthreads();
    if (active) {
      MOE_CHECK(e >= 0 && e < E, "assign: expert id out of range");
      int r = cnt[e] + in_warp;
      for (int w = 0; w < warp; ++w) r += wcnt[w * E + e];
      MOE_CHECK(r >= 0 && r < demand[b * E + e], "assign: FIFO rank outside the expert's demand");
      if (!bpr) {
        const int loc = r < cap ? r : -1;
        locations[f] = loc;
        if (loc >= 0) {
          const size_t slot = static_cast<size_t>(b * E + e) * cap + loc;
          slot_token[slot] = f / k;
          slot_gate[slot] = static_cast<float>(gates[f]);
        } else {
          ++my_drops;
        }
      } else {
        list[list_base[b * E + e] + r] = f;
      }
    }
    __syncthreads();
    for (int ee = threadIdx.x; ee < E; ee += blockDim.x) {
      int add = 0;
      for (int w = 0; w < 8; ++w) add += wcnt[w * E + ee];
      cnt[ee] += add;
    }
    __syncthreads();
  }
  if (!bpr && my_drops) atomicAdd(drops, my_drops);
}

// BPR by sorting: one CTA per (block, expert) list. The (max gate desc, list position asc) order
// is a bitonic sort of (key, position) pairs in shared memory -- positive fp64 gates order like
// their bit patterns, so the keys compare as u64 and ties stay exact. A member's rank is its
// sorted position: the same ranks as bpr_rank_kernel's pairwise count (O(n log^2 n) instead of
// O(n^2) fp64 compares; C3: 60 vs 76 us, ncu). Lists longer than kBprSortMax (T*k/E far above the
// configs' 2-5 K) use the pairwise count inside the same CTA.
constexpr int kBprSortMax = 8192, kBprSortThreads = 1024;
constexpr int kBprSortSmem = kBprSortMax * (8 + 4);

__device__ __forceinline__ void bpr_write(int f, int rank, int k, int b, int E, int e, int cap,
                                          const double* __restrict__ gates,
                                          int32_t* __restrict__ locations,
                                          int32_t* __restrict__ slot_token,
                                          float* __restrict__ slot_gate, int32_t* __restrict__ drops) {
  const int loc = rank < cap ? rank : -1;
  locations[f] = loc;
  if (loc >= 0) {
    const size_t slot = static_cast<size_t>(b * E + e) * cap + loc;
    slot_token[slot] = f / k;
    slot_gate[slot] = static_cast<float>(gates[f]);
  } else {
    atomicAdd(drops, 1);
  }
}

__global__ void __launch_bounds__(kBprSortThreads)
    bpr_sort_kernel(const double* __restrict__ gates, int k, int E,
                    const int32_t* __restrict__ demand, const int32_t* __restrict__ list_base,
                    const int32_t* __restrict__ list, const int32_t* __restrict__ cap_ptr,
                    int32_t* __restrict__ locations, int32_t* __restrict__ slot_token,
                    float* __restrict__ slot_gate, int32_t* __restrict__ drops) {
  pdl_entry();
  extern __shared__ __align__(16) uint8_t bsm[];
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(bsm);
  int32_t* pos = reinterpret_cast<int32_t*>(bsm + kBprSortMax * 8);
  const int be = blockIdx.x;
  const int b = be / E, e = be % E;
  const int n = demand[be];
  if (n == 0) return;
  const int32_t* lst = list + list_base[be];
  const int cap = *cap_ptr;
  auto key_of = [&](int j) {
    return static_cast<unsigned long long>(__double_as_longlong(gates[static_cast<size_t>(lst[j] / k) * k]));
  };
  if (n > kBprSortMax) {  // pairwise count (as bpr_rank_kernel), keys from global / L2
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long ki = key_of(i);
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const unsigned long long kj = key_of(j);
        rank += (kj > ki) || (kj == ki && j < i);
      }
      bpr_write(lst[i], rank, k, b, E, e, cap, gates, locations, slot_token, slot_gate, drops);
    }
    return;
  }
  int P = 1;
  while (P < n) P <<= 1;
  for (int j = threadIdx.x; j < P; j += blockDim.x) {
    keys[j] = j < n ? key_of(j) : 0ull;  // padding sorts last: key 0, position >= n
    pos[j] = j;
  }
  __syncthreads();
  // bitonic sort into (key desc, position asc)
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < P / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;  // this run sorts "first" order ascending
        const unsigned long long kl = keys[lo], kh = keys[hi];
        const int pl = pos[lo], ph = pos[hi];
        const bool h_first = kh > kl || (kh == kl && ph < pl);
        if (h_first == up) {
          keys[lo] = kh; keys[hi] = kl;
          pos[lo] = ph; pos[hi] = pl;
        }
      }
      __syncthreads();
    }
  }
  for (int r = threadIdx.x; r < n; r += blockDim.x)
    bpr_write(lst[pos[r]], r, k, b, E, e, cap, gates, locations, slot_token, slot_gate, drops);
}

// BPR ranking in chunks (C3: one 2-5 K list per expert). Phase 1: CTA (list, chunk) bitonic-sorts
// kBprChunk members of one list by (key desc, list position asc) -- key = the member token's max
// gate as u64 bits (positive fp64 orders like its bit pattern, ties stay exact) -- and writes
// the sorted chunk to scratch. Phase 2: each member's rank = its position in its own sorted
// chunk + for every other chunk the number of members ordered before it (binary search).
// Same ranks as bpr_sort_kernel / bpr_rank_kernel; ~100 CTAs instead of E, no O(n^2) work.
constexpr int kBprChunk = 512;

__device__ __forceinline__ bool bpr_before(unsigned long long ka, int pa, unsigned long long kb, int pb) {
  return ka > kb || (ka == kb && pa < pb);
}

__global__ void __launch_bounds__(256)
    bpr_chunk_sort_kernel(const double* __restrict__ gates, int k,
                          const int32_t* __restrict__ demand, const int32_t* __restrict__ list_base,
                          const int32_t* __restrict__ list, unsigned long long* __restrict__ skeys,
                          int32_t* __restrict__ spos) {
  pdl_entry();
  __shared__ unsigned long long keys[kBprChunk];
  __shared__ int32_t pos[kBprChunk];
  const int be = blockIdx.x;
  const int n = demand[be];
  const int32_t* lst = list + list_base[be];
  const size_t lb = static_cast<size_t>(list_base[be]);
  for (int c0 = blockIdx.y * kBprChunk; c0 < n; c0 += gridDim.y * kBprChunk) {  // CTA-uniform
    const int cn = min(kBprChunk, n - c0);
    for (int j = threadIdx.x; j < kBprChunk; j += blockDim.x) {
      keys[j] = j < cn ? static_cast<unsigned long long>(
                             __double_as_longlong(gates[static_cast<size_t>(lst[c0 + j] / k) * k]))
                       : 0ull;                        // padding: key 0 sorts last
      pos[j] = j < cn ? c0 + j : 0x7fffffff;
    }
    __syncthreads();
    for (int size = 2; size <= kBprChunk; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const int t = threadIdx.x;  // kBprChunk / 2 == blockDim.x
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const unsigned long long kl = keys[lo], kh = keys[hi];
        const int pl = pos[lo], ph = pos[hi];
        if (bpr_before(kh, ph, kl, pl) == up) {
          keys[lo] = kh; keys[hi] = kl;
          pos[lo] = ph; pos[hi] = pl;
        }
        __syncthreads();
      }
    }
    for (int j = threadIdx.x; j < cn; j += blockDim.x) {
      skeys[lb + c0 + j] = keys[j];
      spos[lb + c0 + j] = pos[j];
    }
    __syncthreads();
  }
}

// Phase 2 stages the whole sorted list (all chunks, kBprRankMax members max) in shared memory;
// longer lists search the chunks in global memory.
constexpr int kBprRankMax = 8192;
constexpr int kBprRankSmem = kBprRankMax * (8 + 4);

__global__ void __launch_bounds__(256)
    bpr_chunk_rank_kernel(const double* __restrict__ gates, int k, int E,
                          const int32_t* __restrict__ demand, const int32_t* __restrict__ list_base,
                          const int32_t* __restrict__ list, const unsigned long long* __restrict__ skeys,
                          const int32_t* __restrict__ spos, const int32_t* __restrict__ cap_ptr,
                          int32_t* __restrict__ locations, int32_t* __restrict__ slot_token,
                          float* __restrict__ slot_gate, int32_t* __restrict__ drops) {
  pdl_entry();
  extern __shared__ __align__(16) uint8_t rsm[];
  const int be = blockIdx.x;
  const int b = be / E, e = be % E;
  const int n = demand[be];
  if (n == 0) return;
  const int nch = (n + kBprChunk - 1) / kBprChunk;
  const size_t lb = static_cast<size_t>(list_base[be]);
  const bool staged = n <= kBprRankMax;
  const unsigned long long* K = skeys + lb;
  const int32_t* P = spos + lb;
  if (staged) {
    unsigned long long* ks = reinterpret_cast<unsigned long long*>(rsm);
    int32_t* ps = reinterpret_cast<int32_t*>(rsm + static_cast<size_t>(kBprRankMax) * 8);
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      ks[j] = skeys[lb + j];
      ps[j] = spos[lb + j];
    }
    __syncthreads();
    K = ks;
    P = ps;
  }
  const int cap = *cap_ptr;
  const int32_t* lst = list + lb;
  const int lane = threadIdx.x % 32;
  // this CTA ranks members [blockIdx.y * 256 + i * gridDim.y * 256 ...) of the sorted chunks
  for (int j0 = blockIdx.y * blockDim.x; j0 < n; j0 += gridDim.y * blockDim.x) {  // warp-uniform
    const int jj = j0 + threadIdx.x;
    const bool active = jj < n;
    int loc = 0;
    if (active) {
      const int ch = jj / kBprChunk, j = jj % kBprChunk;
      const unsigned long long kj = K[jj];
      const int pj = P[jj];
      int rank = j;  // members of its own chunk ordered before it
      for (int oc = 0; oc < nch; ++oc) {
        if (oc == ch) continue;
        const int o0 = oc * kBprChunk, on = min(kBprChunk, n - o0);
        int lo = 0, hi = on;  // first index of chunk oc NOT ordered before (kj, pj)
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (bpr_before(K[o0 + mid], P[o0 + mid], kj, pj)) lo = mid + 1;
          else hi = mid;
        }
        rank += lo;
      }
      MOE_CHECK(rank >= 0 && rank < n && pj >= 0 && pj < n, "bpr rank: rank / position out of range");
      const int f = lst[pj];
      loc = rank < cap ? rank : -1;
      locations[f] = loc;
      if (loc >= 0) {
        const size_t slot = static_cast<size_t>(b * E + e) * cap + loc;
        slot_token[slot] = f / k;
        slot_gate[slot] = static_cast<float>(gates[f]);
      }
    }
    const unsigned dropped = __ballot_sync(0xffffffffu, active && loc < 0);
    if (lane == 0 && dropped) atomicAdd(drops, __popc(dropped));
  }
}

// BPR: rank of each member of expert e's list by (max gate desc, token asc).
// gridDim.x = blocks * E, gridDim.y = ceil(max list length / 256).
__global__ void __launch_bounds__(256)
    bpr_rank_kernel(const double* __restrict__ gates, int k, int E,
                    const int32_t* __restrict__ demand, const int32_t* __restrict__ list_base,
                    const int32_t* __restrict__ list, const int32_t* __restrict__ cap_ptr,
                    int32_t* __restrict__ locations, int32_t* __restrict__ slot_token,
                    float* __restrict__ slot_gate, int32_t* __restrict__ drops) {
  pdl_entry();
  constexpr int kTile = 1024;
  __shared__ double keys[kTile];
  const int be = blockIdx.x;
  const int b = be / E, e = be % E;
  const int n = demand[be];
  const int i = blockIdx.y * 256 + threadIdx.x;
  if (blockIdx.y * 256 >= n) return;  // CTA-uniform
  const int32_t* lst = list + list_base[be];
  const int cap = *cap_ptr;
  const bool active = i < n;
  int f = 0;
  double key = 0.0;
  if (active) {
    f = lst[i];
    key = gates[static_cast<size_t>(f / k) * k];  // row max == first top-k gate
  }
  int rank = 0;
  for (int j0 = 0; j0 < n; j0 += kTile) {
    __syncthreads();
    for (int j = threadIdx.x; j < kTile; j += blockDim.x)
      keys[j] = (j0 + j < n) ? gates[static_cast<size_t>(lst[j0 + j] / k) * k] : -1.0;
    __syncthreads();
    if (active) {
      const int lim = min(kTile, n - j0);
      for (int j = 0; j < lim; ++j) {
        const double kj = keys[j];
        rank += (kj > key) || (kj == key && j0 + j < i);
      }
    }
  }
  if (!active) return;
  const int loc = rank < cap ? rank : -1;
  locations[f] = loc;
  if (loc >= 0) {
    const size_t slot = static_cast<size_t>(b * E + e) * cap + loc;
    slot_token[slot] = f / k;
    slot_gate[slot] = static_cast<float>(gates[f]);
  } else {
    atomicAdd(drops, 1);
  }
}

// Pipelined DMMA x . W launch: NT = 4 (<= 32 columns per CTA) or 8 (<= 64).
template <typename TX, int kMode>
int launch_dmma(const DmmaArgs& da, int gx, int gy, cudaStream_t st) {
  const int cols = kMode == kDmRaw ? 64 : da.ncols;
  auto go = [&](auto nt_tag) -> int {
    constexpr int NT = decltype(nt_tag)::value;
    using Cf = D2Cfg<TX, NT>;
    auto kern = gate_dmma2_kernel<TX, NT, kMode>;
    if (!smem_optin(kern, Cf::SMEM)) return -2;
    launch_k(kern, dim3(gx, gy), dim3(kDmWarps * 32), Cf::SMEM, st, da);
    return launch_status();
  };
  if (cols <= 32) return go(std::integral_constant<int, 4>{});
  return go(std::integral_constant<int, 8>{});
}

template <typename TX>
int launch_gate(const void* x, const double* wg, int blocks, int T, int M, int E, int k,
                int32_t* idxs, double* gates, int32_t* hist, double* probs, cudaStream_t st) {
  const TX* xp = static_cast<const TX*>(x);
  if (E <= 64 && E % 2 == 0 && (M * static_cast<int>(sizeof(TX))) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(x) % 16) == 0) {
    const int cpb = (T + kDmTok - 1) / kDmTok;
    DmmaArgs da{};
    da.x = xp;
    da.w = wg;
    da.ldw = E;
    da.ncols = E;
    da.T = T;
    da.K = M;
    da.k = k;
    da.cpb = cpb;
    da.idxs = idxs;
    da.gates = gates;
    da.hist = hist;
    da.probs_out = probs;
    return launch_dmma<TX, kDmGate>(da, blocks * cpb, 1, st);
  }
  if (E <= 64) {
    const int cpb = (T + kDmTok - 1) / kDmTok;
    const dim3 grid(blocks * cpb);
    if (E <= 32)
      launch_k(gate_dmma_kernel<TX, 4>, grid, kDmWarps * 32, 0, st, xp, wg, T, M, E, k, cpb, idxs, gates,
                                                              hist, probs);
    else
      launch_k(gate_dmma_kernel<TX, 8>, grid, kDmWarps * 32, 0, st, xp, wg, T, M, E, k, cpb, idxs, gates,
                                                              hist, probs);
    return launch_status();
  }
  const int cpb = (T + kGateTok - 1) / kGateTok;
  const dim3 grid(blocks * cpb);
  const size_t sh = static_cast<size_t>(E) * sizeof(int32_t);
  if (E <= 32)
    launch_k(gate_topk_kernel<TX, 1>, grid, kGateWarps * 32, sh, st, xp, wg, T, M, E, k, cpb, idxs,
                                                                gates, hist, probs);
  else if (E <= 64)
    launch_k(gate_topk_kernel<TX, 2>, grid, kGateWarps * 32, sh, st, xp, wg, T, M, E, k, cpb, idxs,
                                                                gates, hist, probs);
  else if (E <= 128)
    launch_k(gate_topk_kernel<TX, 4>, grid, kGateWarps * 32, sh, st, xp, wg, T, M, E, k, cpb, idxs,
                                                                gates, hist, probs);
  else if (E <= 256)
    launch_k(gate_topk_kernel<TX, 8>, grid, kGateWarps * 32, sh, st, xp, wg, T, M, E, k, cpb, idxs,
                                                                gates, hist, probs);
  else
    return -1;
  return launch_status();
}

// resolve_capacity (core.cpp:47-59) from an (all-reduced) demand vector.
__global__ void resolve_capacity_kernel(const int32_t* __restrict__ demand, int E, int cap_kind,
                                        int cap_formula, int32_t* __restrict__ cap_out) {
  pdl_entry();
  __shared__ int32_t mx;
  if (threadIdx.x == 0) mx = 1;
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) atomicMax(&mx, demand[e]);
  __syncthreads();
  if (threadIdx.x == 0) {
    int cap = cap_formula;
    if (cap_kind == 1) cap = mx;
    if (cap_kind == 2) cap = min(mx, cap_formula);
    *cap_out = cap;
  }
}

}  // namespace

int resolve_capacity_device(const int32_t* demand, int E, int cap_kind, int cap_formula,
                            int32_t* cap_out, cudaStream_t st) {
  launch_k(resolve_capacity_kernel, 1, 256, 0, st, demand, E, cap_kind, cap_formula, cap_out);
  return launch_status();
}

int gate_cta_per_block(int T) { return (T + kGateTok - 1) / kGateTok; }

namespace {

__global__ void cosine_prep_kernel(const double* __restrict__ ce, int E, int D,
                                   double* __restrict__ ct, double* __restrict__ en,
                                   int32_t* __restrict__ err) {
  pdl_entry();
  const int lane = threadIdx.x % 32;
  for (int e = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32; e < E;
       e += gridDim.x * (blockDim.x / 32)) {
    double s = 0.0;
    for (int d = lane; d < D; d += 32) {
      const double v = ce[static_cast<size_t>(e) * D + d];
      ct[static_cast<size_t>(d) * E + e] = v;
      s = fma(v, v, s);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      en[e] = sqrt(s);
      if (s == 0.0) atomicExch(err, 2);
    }
  }
}

// x . P for token rows that are not 16-byte aligned (tiny M): one fp64 output per thread.
template <typename TX>
__global__ void proj_simt_kernel(const TX* __restrict__ x, const double* __restrict__ P, int64_t n,
                                 int M, int D, double* __restrict__ out) {
  pdl_entry();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n * D;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / D;
    const int d = static_cast<int>(i % D);
    double s = 0.0;
    for (int m = 0; m < M; ++m) s = fma(ld_x<TX>(x + t * M + m), P[static_cast<size_t>(m) * D + d], s);
    out[i] = s;
  }
}

// RouterKind::Cosine: proj = x . P (DMMA, fp64 rows), then cos(proj_t, C_e) / tau -> softmax
// -> top-k with the same 64-token CTA partition / histograms as the linear gate.
template <typename TX>
int launch_cosine_gate(const GatingArgs& a, const GatingBuffers& g, cudaStream_t st) {
  const int D = a.cos_dim;
  if (a.E > 64 || a.E % 2 || D % 2 || !a.cos_proj || !a.cos_ct || !a.cos_en || !a.cos_buf)
    return -1;
  const int cpb = gate_cta_per_block(a.T);
  int rc;
  if ((a.M * static_cast<int>(sizeof(TX))) % 16 == 0 && reinterpret_cast<uintptr_t>(a.x) % 16 == 0) {
    DmmaArgs p{};
    p.x = a.x;
    p.w = a.cos_proj;
    p.ldw = D;
    p.ncols = D;
    p.T = a.T;
    p.K = a.M;
    p.k = a.k;
    p.cpb = cpb;
    p.out = a.cos_buf;
    p.ldo = D;
    rc = launch_dmma<TX, kDmRaw>(p, a.blocks * cpb, (D + 63) / 64, st);
  } else {
    const int64_t n = static_cast<int64_t>(a.blocks) * a.T;
    const int64_t tot = n * D;
    const int grid = static_cast<int>(std::min<int64_t>((tot + 255) / 256, 148 * 16));
    launch_k(proj_simt_kernel<TX>, dim3(grid), dim3(256), 0, st, static_cast<const TX*>(a.x),
             a.cos_proj, n, a.M, D, a.cos_buf);
    rc = launch_status();
  }
  if (rc) return rc;
  DmmaArgs q{};
  q.x = a.cos_buf;
  q.w = a.cos_ct;
  q.ldw = a.E;
  q.ncols = a.E;
  q.T = a.T;
  q.K = D;
  q.k = a.k;
  q.cpb = cpb;
  q.idxs = g.idxs;
  q.gates = g.gates;
  q.hist = g.hist;
  q.probs_out = g.probs;
  q.en = a.cos_en;
  q.tau = a.cos_tau;
  q.err = a.err;
  return launch_dmma<double, kDmCosine>(q, a.blocks * cpb, 1, st);
}

}  // namespace

int cosine_prep_device(const double* ce, int E, int D, double* ct, double* en, int32_t* err,
                       cudaStream_t st) {
  launch_k(cosine_prep_kernel, dim3((E + 7) / 8), dim3(256), 0, st, ce, E, D, ct, en, err);
  return launch_status();
}

int run_gating_device(const GatingArgs& a, const GatingBuffers& g, cudaStream_t st) {
  if (a.E < 1 || a.k < 1 || a.k > a.E || a.k > 32 || a.T < 1 || a.M < 1 || a.blocks < 1) return -1;
  const int cpb = gate_cta_per_block(a.T);
  int rc;
  if (a.router == 1)
    rc = a.x_is_f32 ? launch_cosine_gate<float>(a, g, st) : launch_cosine_gate<__nv_bfloat16>(a, g, st);
  else if (!a.x_is_f32 && a.wg_pieces != nullptr && a.gate_flags != nullptr && g.probs == nullptr &&
           gate_tc_supported(a.M, a.E, a.k) && (reinterpret_cast<uintptr_t>(a.x) % 16) == 0)
    rc = gate_tc_device(a.x, a.wg_pieces, a.wg, a.wg_norm_max, a.blocks, a.T, a.M, a.E, a.k, g.idxs,
                        g.gates, g.hist, a.gate_fixups, a.gate_flags, a.gate_flag_count, st);
  else
    rc = a.x_is_f32 ? launch_gate<float>(a.x, a.wg, a.blocks, a.T, a.M, a.E, a.k, g.idxs, g.gates,
                                         g.hist, g.probs, st)
                    : launch_gate<__nv_bfloat16>(a.x, a.wg, a.blocks, a.T, a.M, a.E, a.k, g.idxs,
                                                 g.gates, g.hist, g.probs, st);
  if (rc) return rc;
  if (cpb > 16 * 256) return -1;
  FinalizeArgs fa{g.scan_done, a.blocks, a.T, a.k, a.cap_kind, a.cap_formula, g.list_base, g.fill,
                  g.cap, g.drops};
  launch_k(scan_cols_kernel, a.blocks * a.E, 256, 0, st, g.hist, cpb, a.E, g.offs, g.demand, fa);
  if (launch_status() != 0) return -2;
  if (g.scan_done != nullptr) return 0;  // the scan's last CTA resolved the capacity
  launch_k(finalize_capacity_kernel, 1, 256, 0, st, a.blocks, a.E, a.T, a.k, a.cap_kind, a.cap_formula,
                                             g.demand, g.list_base, g.fill, g.cap, g.drops);
  if (launch_status() != 0) return -2;
  return 0;
}

int run_assign_device(const GatingArgs& a, const GatingBuffers& g, int cap_bound,
                      cudaStream_t st) {
  const int cpb = gate_cta_per_block(a.T);
  // Slots not claimed by a token are set to -1 by the assign pass itself (no memsets: they
  // would break the programmatic-dependent-launch chain); empty rows are zero-filled by encode.
  const size_t sh = static_cast<size_t>(9) * a.E * sizeof(int32_t);
  launch_k(assign_kernel, a.blocks * cpb, 256, sh, st, g.idxs, g.gates, a.T, a.k, a.E, cpb, g.offs,
                                                 g.list_base, g.cap, a.bpr, g.locations,
                                                 g.slot_token, g.slot_gate, g.list, g.drops, g.demand);
  if (launch_status() != 0) return -2;
  if (a.bpr) {
    static const bool pairwise = [] {
      const char* e = std::getenv("MOE_BPR_PAIRWISE");  // A/B: the O(n^2) pairwise-count kernel
      return e != nullptr && e[0] == '1';
    }();
    if (!pairwise && g.bpr_keys != nullptr && g.bpr_pos != nullptr &&
        smem_optin(bpr_chunk_rank_kernel, kBprRankSmem)) {
      // y: CTAs per list; the lists average T*k/E members (C3: 2048 = 4 chunks)
      const int per = std::max(1, std::min(8, (a.T * a.k / a.E + kBprChunk - 1) / kBprChunk));
      launch_k(bpr_chunk_sort_kernel, dim3(a.blocks * a.E, per), kBprChunk / 2, 0, st, g.gates, a.k,
               g.demand, g.list_base, g.list, g.bpr_keys, g.bpr_pos);
      if (launch_status() != 0) return -2;
      launch_k(bpr_chunk_rank_kernel, dim3(a.blocks * a.E, per * 2), 256, kBprRankSmem, st, g.gates,
               a.k, a.E, g.demand, g.list_base, g.list, g.bpr_keys, g.bpr_pos, g.cap, g.locations,
               g.slot_token, g.slot_gate, g.drops);
    } else if (!pairwise && smem_optin(bpr_sort_kernel, kBprSortSmem)) {
      launch_k(bpr_sort_kernel, dim3(a.blocks * a.E), kBprSortThreads, kBprSortSmem, st, g.gates, a.k,
               a.E, g.demand, g.list_base, g.list, g.cap, g.locations, g.slot_token, g.slot_gate,
               g.drops);
    } else {
      const dim3 grid(a.blocks * a.E, (a.T + 255) / 256);
      launch_k(bpr_rank_kernel, grid, 256, 0, st, g.gates, a.k, a.E, g.demand, g.list_base, g.list,
               g.cap, g.locations, g.slot_token, g.slot_gate, g.drops);
    }
    if (launch_status() != 0) return -2;
  }
  return 0;
}

}  // namespace moe
