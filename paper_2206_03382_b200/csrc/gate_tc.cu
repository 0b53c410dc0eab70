// Certified tensor-core router GEMM for the bf16 layer (linear router, FIFO routing).
//
// The reference routes in fp64 (gate_linear + softmax_rows + topk_select, gating.cpp:19-78).
// Its expert choice depends only on the ORDER of a token's logits, so the logits need fp64
// accuracy only where two of the top-(k+1) are close. This kernel computes them on the tensor
// cores and proves each token's top-k order from an error bound; tokens it cannot prove are
// re-decided from fp64 logits inside the same CTA:
//
//   Wg = hi + lo with hi = bf16(Wg), lo = bf16(Wg - hi)   (|Wg - hi - lo| <= 2^-18 |Wg|)
//   L~[t][e] = fp32 sum of fp32 partials HMMA(x, hi) + HMMA(x, lo) over 32-wide K pieces
//   |L~ - L| <= eps_t = 2^-15 * |x_t|_2 * max_e |Wg[:, e]|_2
// x is bf16, so every product is exact. Error model of one m16n8k16 step: each of its 17
// addends (16 products + the accumulator) truncated to the largest one's 24-bit grid, <= 18 *
// 2^-23 * (sum|products| + |C|), and within one accumulator window that is <= 18 * 2^-23 times
// the window's sum|x (|hi| + |lo|)|. The accumulator restarts from zero every 2 K16 steps (4 mma:
// hi and lo pieces) and is added into an fp32 running sum, so products are never aligned to the
// whole row's sum: <= 4 * 18 * 2^-23 = 2^-16.8 of each window's sum, 2^-16.8 sum|x w| in all.
// Adding the 32 partials in fp32 errs by <= 32 * 2^-24 sum|x w| = 2^-19; with the
// split residual 2^-18 the total is <= 2^-16.05 sum|x w| <= 2^-16.05 |x|_2 |w|_2
// (Cauchy-Schwarz); eps_t keeps a 2.1x margin on that
// pessimistic model (measured errors are ~100x smaller). A token is certified when each of its
// first k sorted logits beats the next by more than 2 eps_t; then its idxs are the fp64
// reference's (exactly equal logits never certify). Uncertified tokens go to a list that
// gate_fixup_kernel re-decides from fp64 logits (products of bf16 x with fp64 Wg are exact; only
// the summation order differs from Eigen) with the fp64 softmax / top-k of the DMMA gate,
// patching idxs / gates / the CTA histograms before the capacity scan reads them.
// Gate VALUES of certified tokens come from the softmax of L~ (relative error ~1e-6 typical,
// bounded by ~4 eps_t); they scale expert outputs, which the north star holds to 2e-2 (bf16).
// BPR needs fp64-accurate cross-token keys, so BPR layers keep the DMMA gate.
//
// Work: 2*T*M*(2E) bf16 MACs on mma.sync.m16n8k16 (HMMA) -- the kernel is HBM-bound on reading
// x once (T*M*2 bytes; 64 MiB at TGT ~ 10 us at 6.5 TB/s), so the tensor pipe stays mostly idle.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdlib>
#include <cstdint>

#include "checks.cuh"
#include "gemm_sm100.h"
#include "kernels.h"
#include "pdl.cuh"
#include "ptx.cuh"

namespace moe {

namespace {

constexpr int kTcWarps = 4;              // 4 warps x 16 tokens = the 64-token gate block
constexpr int kTcTok = kTcWarps * 16;
constexpr int kTcKC = 64;                // K per stage (one 128-byte row chunk)
#ifndef MOE_TC_STAGES
#define MOE_TC_STAGES 3
#endif
constexpr int kTcStages = MOE_TC_STAGES;  // 3: 48 KiB (E = 32), 4 CTAs per SM, the 512 TGT blocks in one wave
constexpr double kTcEpsScale = 1.0 / 32768.0;  // 2^-15
constexpr int kTcFold = 2;                      // hi-piece mma steps per fp32 accumulator
#ifndef MOE_FIX_WARPS
#define MOE_FIX_WARPS 32
#endif
#ifndef MOE_FIX_CTAS
#define MOE_FIX_CTAS 148
#endif
constexpr int kFixWarps = MOE_FIX_WARPS;       // fixup CTA: warps split M
constexpr int kFixCtas = MOE_FIX_CTAS;
#ifndef MOE_FIX_TOK
#define MOE_FIX_TOK 1  // measured: one token per CTA beats sharing Wg reads across 4 (shorter critical path)
#endif
constexpr int kFixTok = MOE_FIX_TOK;           // fixup CTA: tokens re-decided together
constexpr int kTcMaxK = 8;

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(pred ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];"
               : "=r"(r0), "=r"(r1)
               : "r"(addr));
}
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float bf_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// 128-byte smem rows, 16-byte chunks XOR-swizzled by row % 8 (conflict-free cp.async / ldmatrix)
__device__ __forceinline__ uint32_t sw(uint32_t base, int row, int chunk) {
  return base + row * 128 + ((chunk ^ (row & 7)) << 4);
}

template <int NT>
struct TcCfg {
  static constexpr int E = 8 * NT;
  static constexpr int XB = kTcTok * 128;     // x stage bytes
  static constexpr int WB = 2 * E * 128;      // hi + lo pieces, E rows each
  static constexpr int STAGE = XB + WB;
  static constexpr int SMEM = kTcStages * STAGE;
};

struct TcArgs {
  const __nv_bfloat16* x;       // [blocks*T][M]
  const __nv_bfloat16* pieces;  // [2][E][M]: hi, lo
  const double* wg;             // [M][E] fp64 (re-decision)
  const float* wn_max;          // max_e |Wg[:, e]|_2, rounded up
  int T, M, E, k, cpb;
  int32_t* idxs;
  double* gates;
  int32_t* hist;
  int32_t* fixups;              // += tokens re-decided in fp64 (metrics; may be null)
  int32_t* flag_list;           // [blocks*T] uncertified token indices
  int32_t* flag_count;          // [0] list size, [1] fixup CTAs done (reset by the fixup kernel)
};

template <int NT>
#ifndef MOE_GATE_MINB
#define MOE_GATE_MINB 4
#endif
__global__ void __launch_bounds__(kTcWarps * 32, NT <= 4 ? MOE_GATE_MINB : 2) gate_tc_kernel(TcArgs a) {
  using Cf = TcCfg<NT>;
  constexpr int E = Cf::E;
  constexpr int NTH = kTcWarps * 32;
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ int32_t sh_hist[E];
  pdl_entry();
  const int M = a.M;
  const int b = blockIdx.x / a.cpb, c = blockIdx.x % a.cpb;
  const int t_begin = b * a.T + c * kTcTok;
  const int ntok = min(b * a.T + a.T, t_begin + kTcTok) - t_begin;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int e = threadIdx.x; e < E; e += NTH) sh_hist[e] = 0;
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm));

  auto issue = [&](int ch) {
    const int k0 = ch * kTcKC;
    const uint32_t st = sbase + (ch % kTcStages) * Cf::STAGE;
    for (int i = threadIdx.x; i < kTcTok * 8; i += NTH) {
      const int r = i / 8, q = i % 8;
      const bool ok = r < ntok;
      const __nv_bfloat16* src = a.x + (ok ? static_cast<size_t>(t_begin + r) * M + k0 + q * 8 : 0);
      cp16(sw(st, r, q), src, ok);
    }
    for (int i = threadIdx.x; i < 2 * E * 8; i += NTH) {
      const int r = i / 8, q = i % 8;  // r = piece * E + e
      cp16(sw(st + Cf::XB, r, q), a.pieces + static_cast<size_t>(r) * M + k0 + q * 8, true);
    }
  };

  // fp32 accumulators of x.hi + x.lo restarted every kTcFold mma steps and added into fp32
  // running sums
  float run[NT][4], hacc[NT][4];
#ifdef MOE_GATE_SPLIT_ACC  // experiment: x.lo in its own whole-K accumulator (shorter mma chains)
  float lacc[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) lacc[j][i] = 0.0f;
#endif
#pragma unroll
  for (int j = 0; j < NT; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) run[j][i] = hacc[j][i] = 0.0f;
  // |x_t|^2 on the tensor pipe: the A fragment's row halves are exactly the B fragments of
  // X_rows^T, so HMMA(A, A^T) accumulates X X^T blocks whose diagonals are the row norms
  float nacc[2][4] = {{0.0f, 0.0f, 0.0f, 0.0f}, {0.0f, 0.0f, 0.0f, 0.0f}};

  const int nch = M / kTcKC;
#pragma unroll
  for (int s = 0; s < kTcStages - 1; ++s) {
    if (s < nch) issue(s);
    cp_commit();
  }
  // ldmatrix lane roles: A x4 = (rows 0-7 | 8-15) x (k 0-7 | 8-15); B x2 = 8 experts x (k 0-7 | 8-15)
  const int a_row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int a_kc = lane >> 4;
  const int b_row = lane & 7;
  const int b_kc = (lane >> 3) & 1;
  for (int ch = 0; ch < nch; ++ch) {
    cp_wait<kTcStages - 2>();
    __syncthreads();
    if (ch + kTcStages - 1 < nch) issue(ch + kTcStages - 1);
    cp_commit();
    const uint32_t st = sbase + (ch % kTcStages) * Cf::STAGE;
#pragma unroll
    for (int ks = 0; ks < kTcKC / 16; ++ks) {
      uint32_t af[4];
      ldsm_x4(sw(st, a_row, ks * 2 + a_kc), af[0], af[1], af[2], af[3]);
      hmma(nacc[0], af, af[0], af[2]);  // X . X[rows 0-7]^T
      hmma(nacc[1], af, af[1], af[3]);  // X . X[rows 8-15]^T
      // B row groups q = piece * NT + j (8 experts each), two per ldmatrix.x4
#pragma unroll
      for (int q = 0; q < 2 * NT; q += 2) {
        uint32_t b[4];
        ldsm_x4(sw(st + Cf::XB, (q + (lane >> 4)) * 8 + b_row, ks * 2 + b_kc), b[0], b[1], b[2], b[3]);
#ifdef MOE_GATE_SPLIT_ACC
        if (q < NT) hmma(hacc[q], af, b[0], b[1]);
        else hmma(lacc[q - NT], af, b[0], b[1]);
        if (q + 1 < NT) hmma(hacc[q + 1], af, b[2], b[3]);
        else hmma(lacc[q + 1 - NT], af, b[2], b[3]);
#else
        hmma(hacc[q % NT], af, b[0], b[1]);
        hmma(hacc[(q + 1) % NT], af, b[2], b[3]);
#endif
      }
      if (ks % kTcFold == kTcFold - 1) {
        // fold the hi accumulator (kTcFold steps, K = 16 * kTcFold) into the running sum
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            run[j][i] += hacc[j][i];
            hacc[j][i] = 0.0f;
          }
      }
    }
  }
  cp_wait<0>();

  // ---- epilogue: lane (g = lane / 4, c = lane % 4) holds rows g and g + 8, columns 8j + 2c + i
  const int g = lane >> 2, cq = lane & 3;
  // row norms: the diagonal of nacc[0] (row g) / nacc[1] (row g + 8) sits in lane (g, g / 2),
  // element g % 2 (rows 0-7) / 2 + g % 2 (rows 8-15); positive-term HMMA sums err by at most
  // 64 * 18 * 2^-23 relative at K = 1024, so |x|^2 * (1 + 2^-8) bounds it from above
  const int src_lane = g * 4 + g / 2;
  float d0 = (g & 1) ? nacc[0][1] : nacc[0][0];
  float d1 = (g & 1) ? nacc[1][3] : nacc[1][2];
  d0 = __shfl_sync(0xffffffffu, d0, src_lane);
  d1 = __shfl_sync(0xffffffffu, d1, src_lane);
  const float wn = __ldg(a.wn_max);
  const int k = a.k;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int tt = warp * 16 + g + 8 * h;
    const bool tok_ok = tt < ntok;
    const int t = t_begin + tt;
    float L[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        L[j][i] = run[j][2 * h + i];
#ifdef MOE_GATE_SPLIT_ACC
        L[j][i] += lacc[j][2 * h + i];
#endif
      }
    const float eps = static_cast<float>(kTcEpsScale) * sqrtf((h ? d1 : d0) * (1.0f + 1.0f / 256.0f)) * wn;
    float mx = -FLT_MAX;
#pragma unroll
    for (int j = 0; j < NT; ++j) mx = fmaxf(mx, fmaxf(L[j][0], L[j][1]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    // softmax denominator in fp32 (terms below e^-87 vanish; they are < 2^-125 of the sum)
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) s += __expf(L[j][i] - mx);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    // top-(k + 1) by (logit desc, expert asc); the (k + 1)-th only bounds the k-th's margin
    unsigned taken = 0;
    bool certified = true;
    float prev = 0.0f;
    int sel[kTcMaxK];
    float selv[kTcMaxK];
    const int kk = k < E ? k + 1 : k;
    for (int r = 0; r < kk; ++r) {
      float bv = -FLT_MAX;
      int bi = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int e = j * 8 + cq * 2 + i;
          if (!(taken & (1u << (j * 2 + i))) && (L[j][i] > bv || (L[j][i] == bv && e < bi))) {
            bv = L[j][i];
            bi = e;
          }
        }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (((bi & 7) >> 1) == cq) taken |= 1u << ((bi >> 3) * 2 + (bi & 1));
      if (r > 0 && !(prev - bv > 2.0f * eps)) certified = false;
      // the reference orders fp64 PROBABILITIES (ties -> lower id): below exp's normal range
      // distinct logits can give equal (denormal / zero) probabilities, so a selected expert
      // that deep under the max is never certified from logits
      if (r < k && bv - mx < -690.0f) certified = false;
      prev = bv;
      if (r < k) {
        sel[r] = bi;
        selv[r] = bv;
      }
    }
    if (cq == 0 && tok_ok) {
      if (certified) {
        for (int r = 0; r < k; ++r) {
          a.idxs[static_cast<size_t>(t) * k + r] = sel[r];
          a.gates[static_cast<size_t>(t) * k + r] =
              exp(static_cast<double>(selv[r] - mx)) / static_cast<double>(s);
          atomicAdd(&sh_hist[sel[r]], 1);
        }
      } else {
        const int slot = atomicAdd(a.flag_count, 1);
        MOE_CHECK(slot < static_cast<int>(gridDim.x / a.cpb) * a.T, "gate: uncertified-token list overflow");
        a.flag_list[slot] = t;
      }
    }
  }
  __syncthreads();

  for (int e = threadIdx.x; e < E; e += NTH) a.hist[static_cast<size_t>(blockIdx.x) * E + e] = sh_hist[e];
}

// ---------------------------------------------------------------- tcgen05 variant
// Same certificate, on the 5th-gen tensor cores: one CTA = 128 tokens (M = 128, TMEM lane =
// token), N = 2E columns (hi | lo pieces of Wg), K streamed by TMA in 64-wide k-blocks (SW128).
// Each k-block's 4 MMAs write a fresh accumulator (double-buffered in TMEM); the 4 epilogue
// warps drain it with tcgen05.ld and add it into per-thread fp32 running logits -- the same
// fold schedule as the HMMA kernel (hi piece: 4 mma steps per window, 2^-16.8 of the window's
// sum|x w|), so the same eps_t. The epilogue warps also read their row of each A stage from
// shared memory for |x_t|^2 (fp32, exact products), and after the last k-block finish softmax
// / top-(k+1) / certificate per thread (one token per thread: no shuffles).
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM alloc), 2..5 epilogue (TMEM lane quadrant = warp % 4).
constexpr int kT5Tok = 128;
constexpr int kT5KB = 64;       // K per stage (one 128-byte swizzle atom of bf16)
constexpr int kT5Stages = 4;
constexpr int kT5Threads = 192;

template <int E>
struct T5Cfg {
  static_assert(E % 16 == 0, "hi | lo accumulators are drained 32 columns at a time");
  static constexpr int N = 2 * E;
  static constexpr uint32_t A_BYTES = kT5Tok * kT5KB * 2;  // 16 KiB
  static constexpr uint32_t B_BYTES = N * kT5KB * 2;       // 8 KiB at E = 32
  static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  static constexpr uint32_t BAR_OFF = kT5Stages * STAGE;
  static constexpr uint32_t SMEM = BAR_OFF + 256 + 1024;   // + barriers + alignment slack
  static constexpr uint32_t TMEM_COLS = 2 * N <= 32 ? 32 : 2 * N <= 64 ? 64 : 2 * N <= 128 ? 128 : 256;
};

struct T5Args {
  TcArgs a;
  int rows_total;  // blocks * T
};

template <int E>
__global__ void __launch_bounds__(kT5Threads, 1)
    gate_tc5_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                    const T5Args args) {
  using C = T5Cfg<E>;
  constexpr int N = C::N;
  const TcArgs& a = args.a;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + kT5Stages;
  uint64_t* accf = empty + kT5Stages;
  uint64_t* acce = accf + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
  __shared__ int32_t sh_hist[2][E];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // this CTA: tokens [t0, t0 + ntok) of block b (tiles never cross a block)
  const int tiles = (a.T + kT5Tok - 1) / kT5Tok;
  const int b = blockIdx.x / tiles, c = blockIdx.x % tiles;
  const int t0 = b * a.T + c * kT5Tok;
  const int ntok = min(kT5Tok, a.T - c * kT5Tok);
  for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) (&sh_hist[0][0])[i] = 0;
  if (threadIdx.x == 0) {
    ptx::prefetch_tmap(&tmX);
    ptx::prefetch_tmap(&tmW);
    for (int i = 0; i < kT5Stages; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1 + 4);  // the MMA commit + the 4 epilogue warps (A rows read)
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&accf[i], 1);
      ptx::mbar_init(&acce[i], 4);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_entry();
  const int nkb = a.M / kT5KB;

  if (warp == 0 && lane == 0) {
    // ---------------------------------------------------------------- TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kT5Stages;
      ptx::mbar_wait(&empty[s], ((kb / kT5Stages) & 1) ^ 1);
      uint8_t* st = smem + s * C::STAGE;
      ptx::mbar_arrive_expect_tx(&full[s], C::STAGE);
      ptx::tma_load_3d(&tmX, &full[s], st, kb * kT5KB, t0, 0);
      ptx::tma_load_3d(&tmW, &full[s], st + C::A_BYTES, kb * kT5KB, 0, 0);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = ptx::make_idesc_bf16(128, N, false, false);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kT5Stages;
      const int buf = kb & 1;
      ptx::mbar_wait(&acce[buf], ((kb >> 1) & 1) ^ 1);  // the epilogue drained this buffer
      ptx::mbar_wait(&full[s], (kb / kT5Stages) & 1);
      ptx::tc_fence_after();
      const uint32_t sa = ptx::smem_u32(smem + s * C::STAGE);
      const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
      for (int k = 0; k < kT5KB / 16; ++k)
        ptx::umma_bf16(tmem + buf * N, ptx::make_sw128_desc(sa + k * 32, 16, 1024),
                       ptx::make_sw128_desc(sb + k * 32, 16, 1024), idesc, k > 0 ? 1u : 0u);
      ptx::umma_commit(&empty[s]);
      ptx::umma_commit(&accf[buf]);
    }
  } else if (warp >= 2) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp % 4;            // TMEM lane quadrant
    const int row = q * 32 + lane;     // token row within the tile
    const uint32_t taddr = tmem + ((q * 32) << 16);
    float L[E];
#pragma unroll
    for (int e = 0; e < E; ++e) L[e] = 0.0f;
    float ss = 0.0f;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kT5Stages;
      const int buf = kb & 1;
      // |x_row|^2 from this stage's A tile (SW128: chunk j of row r at ((j ^ (r % 8)) << 4))
      ptx::mbar_wait(&full[s], (kb / kT5Stages) & 1);
      const uint8_t* ar = smem + s * C::STAGE + row * 128;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint4 v = *reinterpret_cast<const uint4*>(ar + ((j ^ (row & 7)) << 4));
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float lo = __uint_as_float(w4[u] << 16), hi = __uint_as_float(w4[u] & 0xffff0000u);
          ss = fmaf(lo, lo, ss);
          ss = fmaf(hi, hi, ss);
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
      // this k-block's accumulator: hi | lo columns
      ptx::mbar_wait(&accf[buf], (kb >> 1) & 1);
      ptx::tc_fence_after();
#pragma unroll
      for (int h = 0; h < N / 32; ++h) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(taddr + buf * N + h * 32, v);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) L[(h * 32 + i) % E] += __uint_as_float(v[i]);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&acce[buf]);
    }
    // ---- certificate, softmax, top-(k + 1) of this thread's token
    const int k = a.k;
    const bool tok_ok = row < ntok;
    const int t = t0 + row;
    const float wn = __ldg(a.wn_max);
    // fp32 sum of M squares: relative error <= M * 2^-24; (1 + 2^-8) covers M up to 65 K
    const float eps = static_cast<float>(kTcEpsScale) * sqrtf(ss * (1.0f + 1.0f / 256.0f)) * wn;
    float mx = -FLT_MAX;
#pragma unroll
    for (int e = 0; e < E; ++e) mx = fmaxf(mx, L[e]);
    float sden = 0.0f;
#pragma unroll
    for (int e = 0; e < E; ++e) sden += __expf(L[e] - mx);
    unsigned long long taken = 0ull;
    bool certified = true;
    float prev = 0.0f;
    int sel[kTcMaxK];
    float selv[kTcMaxK];
    const int kk = k < E ? k + 1 : k;
    for (int r = 0; r < kk; ++r) {
      float bv = -FLT_MAX;
      int bi = 0;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (!((taken >> e) & 1ull) && L[e] > bv) {  // strict: ties keep the lower expert id
          bv = L[e];
          bi = e;
        }
      taken |= 1ull << bi;
      if (r > 0 && !(prev - bv > 2.0f * eps)) certified = false;
      if (r < k && bv - mx < -690.0f) certified = false;  // see gate_tc_kernel
      prev = bv;
      if (r < k) {
        sel[r] = bi;
        selv[r] = bv;
      }
    }
    if (tok_ok) {
      if (certified) {
        for (int r = 0; r < k; ++r) {
          a.idxs[static_cast<size_t>(t) * k + r] = sel[r];
          a.gates[static_cast<size_t>(t) * k + r] =
              exp(static_cast<double>(selv[r] - mx)) / static_cast<double>(sden);
          atomicAdd(&sh_hist[row / kTcTok][sel[r]], 1);
        }
      } else {
        const int slot = atomicAdd(a.flag_count, 1);
        MOE_CHECK(slot < args.rows_total, "gate: uncertified-token list overflow");
        a.flag_list[slot] = t;
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // histogram rows of the (up to) two 64-token gate blocks this tile covers
  for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) {
    const int hb = i / E, e = i % E;
    const int blk64 = c * 2 + hb;
    if (blk64 * kTcTok < a.T) a.hist[(static_cast<size_t>(b) * a.cpb + blk64) * E + e] = sh_hist[hb][e];
  }
  if (warp == 1) ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
}

// fp64 re-decision of the tokens gate_tc_kernel could not certify. A CTA takes up to kFixTok
// listed tokens at once (their x rows staged in shared memory) so each fp64 Wg element it streams
// from L2 serves all of them; warps split M, lanes own experts (lane, lane + 32). Then warp j
// runs the fp64 softmax + top-k (prob desc, expert asc; gating.cpp:19-78) of token j and patches
// idxs / gates / the token's CTA histogram row. The last CTA to finish resets the list and adds
// its size to the metrics counter.
__global__ void __launch_bounds__(kFixWarps * 32, kFixWarps <= 16 ? 2 : 1) gate_fixup_kernel(TcArgs a, int max_m) {
  static_assert(kFixTok <= kFixWarps, "one finalising warp per token");
  extern __shared__ __align__(16) uint8_t fsm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(fsm);                         // [kFixTok][M]
  double* red = reinterpret_cast<double*>(fsm + static_cast<size_t>(kFixTok) * max_m * 2);  // [kFixTok][warps][64]
  pdl_entry();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n = *reinterpret_cast<volatile int32_t*>(a.flag_count);
  const int M = a.M, E = a.E, k = a.k;
  const int mlen = (M + kFixWarps - 1) / kFixWarps;
  const double* __restrict__ wg = a.wg;
  for (int f0 = blockIdx.x * kFixTok; f0 < n; f0 += gridDim.x * kFixTok) {
    const int nt = min(kFixTok, n - f0);
    for (int i = threadIdx.x; i < nt * (M / 8); i += blockDim.x) {
      const int j = i / (M / 8), q = i % (M / 8);
      const int t = a.flag_list[f0 + j];
      reinterpret_cast<uint4*>(xs + static_cast<size_t>(j) * M)[q] =
          __ldg(reinterpret_cast<const uint4*>(a.x + static_cast<size_t>(t) * M) + q);
    }
    __syncthreads();
    const int m0 = warp * mlen, m1 = min(M, m0 + mlen);
#pragma unroll
    for (int i2 = 0; i2 < 2; ++i2) {
      const int e = lane + 32 * i2;
      if (e >= E) continue;
      double p[kFixTok];
#pragma unroll
      for (int j = 0; j < kFixTok; ++j) p[j] = 0.0;
      for (int mb = m0; mb < m1; mb += 16) {
        double wv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) wv[u] = mb + u < m1 ? __ldg(wg + static_cast<size_t>(mb + u) * E + e) : 0.0;
#pragma unroll
        for (int j = 0; j < kFixTok; ++j) {
          if (j >= nt) break;
          const __nv_bfloat16* xr = xs + static_cast<size_t>(j) * M;
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (mb + u < m1) p[j] = fma(static_cast<double>(__bfloat162float(xr[mb + u])), wv[u], p[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < kFixTok; ++j)
        if (j < nt) red[(static_cast<size_t>(j) * kFixWarps + warp) * 64 + e] = p[j];
    }
    __syncthreads();
    if (warp < nt) {
      const int j = warp;
      const int t = a.flag_list[f0 + j];
      double l[2], pv[2];
      double mx = -DBL_MAX;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int e = lane + 32 * i;
        l[i] = -DBL_MAX;
        if (e < E) {
          double v = 0.0;
          for (int q = 0; q < kFixWarps; ++q) v += red[(static_cast<size_t>(j) * kFixWarps + q) * 64 + e];
          l[i] = v;
          mx = fmax(mx, v);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        pv[i] = (lane + 32 * i < E) ? exp(l[i] - mx) : 0.0;
        s += pv[i];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
#pragma unroll
      for (int i = 0; i < 2; ++i) pv[i] = (lane + 32 * i < E) ? pv[i] / s : -1.0;
      const int cta = (t / a.T) * a.cpb + (t % a.T) / kTcTok;
      unsigned taken = 0;
      for (int r = 0; r < k; ++r) {
        double bv = -1.0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int e = lane + 32 * i;
          if (e < E && !(taken & (1u << i)) && (pv[i] > bv || (pv[i] == bv && e < bi))) {
            bv = pv[i];
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
          a.idxs[static_cast<size_t>(t) * k + r] = bi;
          a.gates[static_cast<size_t>(t) * k + r] = bv;
          atomicAdd(a.hist + static_cast<size_t>(cta) * E + bi, 1);
        }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.flag_count + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      if (a.fixups) atomicAdd(a.fixups, n);
      a.flag_count[0] = 0;
      a.flag_count[1] = 0;
    }
  }
}

// hi / lo bf16 split of Wg ([M][E] fp64 -> [2][E][M]) and max_e |Wg[:, e]|_2 (rounded up).
// One CTA of 32 warps; warp w handles experts w, w + 32.
__global__ void __launch_bounds__(1024) wg_split_kernel(const double* __restrict__ wg, int M, int E,
                                                        __nv_bfloat16* __restrict__ pieces,
                                                        float* __restrict__ wn_max) {
  pdl_entry();
  __shared__ float wmax[32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float nmax = 0.0f;
  for (int e = warp; e < E; e += 32) {
    double ss = 0.0;
    for (int m = lane; m < M; m += 32) {
      const double w = wg[static_cast<size_t>(m) * E + e];
      const __nv_bfloat16 hi = __double2bfloat16(w);
      const __nv_bfloat16 lo = __double2bfloat16(w - static_cast<double>(__bfloat162float(hi)));
      pieces[static_cast<size_t>(e) * M + m] = hi;
      pieces[static_cast<size_t>(E + e) * M + m] = lo;
      ss = fma(w, w, ss);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    nmax = fmaxf(nmax, static_cast<float>(sqrt(ss)) * 1.0001f);
  }
  if (lane == 0) wmax[warp] = nmax;
  __syncthreads();
  if (warp == 0) {
    float v = wmax[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) *wn_max = v;
  }
}

}  // namespace

bool gate_tc_supported(int M, int E, int k) {
  return E % 8 == 0 && E >= 8 && E <= 64 && M % kTcKC == 0 && M > 0 && k <= E && k <= kTcMaxK;
}

int gate_tc_prepare_device(const double* wg, int M, int E, void* pieces, float* wn_max,
                           cudaStream_t st) {
  launch_k(wg_split_kernel, 1, 1024, 0, st, wg, M, E,
           static_cast<__nv_bfloat16*>(pieces), wn_max);
  return launch_status();
}

int gate_tc_device(const void* x, const void* pieces, const double* wg, const float* wn_max,
                   int blocks, int T, int M, int E, int k, int32_t* idxs, double* gates,
                   int32_t* hist, int32_t* fixups, int32_t* flag_list, int32_t* flag_count,
                   cudaStream_t st) {
  if (!gate_tc_supported(M, E, k) || (reinterpret_cast<uintptr_t>(x) % 16) != 0) return -1;
  TcArgs a{};
  a.x = static_cast<const __nv_bfloat16*>(x);
  a.pieces = static_cast<const __nv_bfloat16*>(pieces);
  a.wg = wg;
  a.wn_max = wn_max;
  a.T = T;
  a.M = M;
  a.E = E;
  a.k = k;
  a.cpb = (T + kTcTok - 1) / kTcTok;
  a.idxs = idxs;
  a.gates = gates;
  a.hist = hist;
  a.fixups = fixups;
  a.flag_list = flag_list;
  a.flag_count = flag_count;

  static const bool hmma = [] {
    const char* e = std::getenv("MOE_GATE_HMMA");  // =1: the mma.sync kernel (A/B runs)
    return e != nullptr && e[0] == '1';
  }();
  if (!hmma && E <= 64 && E % 16 == 0) {  // N = 2E columns drained 32 at a time
    CUtensorMap mx{}, mw{};
    const int rows = blocks * T;
    if (tensor_map_3d(&mx, x, false, M, rows, 1, kT5KB, kT5Tok) == 0 &&
        tensor_map_3d(&mw, pieces, false, M, 2 * E, 1, kT5KB, 2 * E) == 0) {
      T5Args ta{a, rows};
      const int tiles = (T + kT5Tok - 1) / kT5Tok;
      auto go5 = [&](auto e_tag) -> int {
        constexpr int EE = decltype(e_tag)::value;
        auto kern = gate_tc5_kernel<EE>;
        if (!smem_optin(kern, T5Cfg<EE>::SMEM)) return -2;
        launch_k(kern, dim3(blocks * tiles), dim3(kT5Threads), T5Cfg<EE>::SMEM, st, mx, mw, ta);
        if (launch_status() != 0) return -2;
        const int fsmem = kFixTok * M * 2 + kFixTok * kFixWarps * 64 * 8;
        if (!smem_optin(gate_fixup_kernel, fsmem)) return -2;
        launch_k(gate_fixup_kernel, dim3(kFixCtas), dim3(kFixWarps * 32), fsmem, st, a, M);
        return launch_status();
      };
      switch (E / 16) {
        case 1: return go5(std::integral_constant<int, 16>{});
        case 2: return go5(std::integral_constant<int, 32>{});
        case 3: return go5(std::integral_constant<int, 48>{});
        default: return go5(std::integral_constant<int, 64>{});
      }
    }
  }
  auto go = [&](auto nt_tag) -> int {
    constexpr int NT = decltype(nt_tag)::value;
    auto kern = gate_tc_kernel<NT>;
    if (!smem_optin(kern, TcCfg<NT>::SMEM)) return -2;
    launch_k(kern, dim3(blocks * a.cpb), dim3(kTcWarps * 32), TcCfg<NT>::SMEM, st, a);
    if (launch_status() != 0) return -2;
    const int fsmem = kFixTok * M * 2 + kFixTok * kFixWarps * 64 * 8;
    if (!smem_optin(gate_fixup_kernel, fsmem)) return -2;
    launch_k(gate_fixup_kernel, dim3(kFixCtas), dim3(kFixWarps * 32), fsmem, st, a, M);
    return launch_status();
  };
  switch (E / 8) {
    case 1: return go(std::integral_constant<int, 1>{});
    case 2: return go(std::integral_constant<int, 2>{});
    case 3: return go(std::integral_constant<int, 3>{});
    case 4: return go(std::integral_constant<int, 4>{});
    case 5: return go(std::integral_constant<int, 5>{});
    case 6: return go(std::integral_constant<int, 6>{});
    case 7: return go(std::integral_constant<int, 7>{});
    default: return go(std::integral_constant<int, 8>{});
  }
}

}  // namespace moe
