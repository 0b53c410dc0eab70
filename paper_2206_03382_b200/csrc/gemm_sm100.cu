// Expert-FFN grouped GEMM for sm_100a: TMA -> smem (4-stage ring) -> tcgen05.mma (TMEM fp32
// accumulator, double buffered) -> epilogue warps (tcgen05.ld -> fused op -> swizzled smem ->
// TMA store). Persistent: one CTA per SM walks a static tile schedule.
//
// Replaces the Eigen GEMMs of the reference expert FFN:
//   expert_ffn          /root/reference/proj/src/parallelism.cpp:103-121  (relu(X.W1).W2)
//   expert_ffn_backward /root/reference/proj/src/parallelism.cpp:123-147  (dh, dX, dW1, dW2)
//
// Two addressing modes cover all six GEMMs of one expert FFN step:
//   row-M (fwd, dgrad): D[g,(s,r),n] = sum_k A[g,(s,r),k] * B[g,k,n]
//   row-K (wgrad)     : D[g,mo,n]    = sum_(s,r) A[g,(s,r),mo] * B[g,(s,r),n]
// "(s, r)" is a token row r of capacity segment s; segments hold `seg_rows` rows and segment
// (s, g) lives at index (seg_base + s) * G + g of a 3-D [nseg][seg_rows][cols] buffer. This is the
// (chunk, source rank, local expert, capacity slot) receive layout of the flexible all-to-all
// (collectives.cpp:123-141), addressed directly by TMA so no interleave copy is ever made.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "gemm_sm100.h"
#include "checks.cuh"
#include "kernels.h"
#include "pdl.cuh"
#include "peer_flags.cuh"
#include "ptx.cuh"
#include "relu_mask.cuh"

#ifndef MOE_GEMM_STAGES
#define MOE_GEMM_STAGES 4
#endif
#ifndef MOE_GEMM_STAGES_PAIR
#define MOE_GEMM_STAGES_PAIR 6
#endif
#ifndef MOE_GEMM_EPI_BUFS
#define MOE_GEMM_EPI_BUFS 1
#endif
#ifndef MOE_TMA_4D  // MN-major operands loaded as one 4-D box per stage instead of one per atom
#define MOE_TMA_4D 1
#endif
#ifndef MOE_GEMM_EPI_BUFS4  // staging buffers per warp with 4 epilogue warps (fits 6 stages at 2)
#define MOE_GEMM_EPI_BUFS4 MOE_GEMM_EPI_BUFS
#endif

// MOE_GEMM_TRACE (debug builds only): per-role barrier wait cycles, printed by CTAs 0 and 1.
#ifdef MOE_GEMM_TRACE
#define TRACE_WAIT(acc, call)          \
  do {                                 \
    const long long t0_ = clock64();   \
    call;                              \
    acc += clock64() - t0_;            \
  } while (0)
#else
#define TRACE_WAIT(acc, call) call
#endif

namespace moe {

namespace {

constexpr uint32_t BM = 128;  // accumulator rows per CTA (TMEM lanes)
constexpr uint32_t BN = 256;  // UMMA N
constexpr uint32_t BK = 64;   // one 128-byte swizzle atom of bf16 along K
constexpr uint32_t UK = 16;   // K per tcgen05.mma (bf16)
constexpr uint32_t kAccStages = 2;
constexpr uint32_t kTmemCols = kAccStages * BN;  // 512
constexpr uint32_t EPI_WARP_BYTES = 32 * 128;    // 32 rows x 128 B staging per epilogue warp

// kCG = 1: one CTA computes a 128 x 256 tile. kCG = 2: a CTA pair (cluster of 2, cta_group::2)
// computes 256 x 256: each CTA holds its 128 A rows and half (128 columns) of B, so B smem per
// CTA halves and the pipeline gets deeper (6 stages instead of 4).
// kPeer: the fused-combine kernels store over NVLink, where a bulk store holds its staging
// buffer longer -- two staging buffers per epilogue warp.
// Epilogue warps per CTA: 4 (one per TMEM lane quadrant, draining all 256 columns) or 8 (two
// column halves). Measured at TGT before the issuers ran on whole warps: the up GEMM's
// certificate epilogue needed 8 to keep pace with its K = 1024 mainloop; every other kind is
// faster with 4 (wgrad -8 %: fewer warps contending with the MMA / TMA issuers). Since then the
// up GEMM measures the same with 4 or 8 (179 / 180 us isolated); it stays at 8.
template <int kGemmEpiWarps>
struct EpiCfg {
  static constexpr uint32_t kEpiWarps = kGemmEpiWarps;
  static constexpr uint32_t kEpiThreads = kEpiWarps * 32;
  static constexpr uint32_t kThreads = 128 + kEpiThreads;  // warp0 TMA, warp1 MMA, warp2 TMEM, 4.. epilogue
  static constexpr uint32_t kEpiCols = BN / (kEpiWarps / 4);  // accumulator columns per epilogue warp
};

template <int kCG, bool kPeer = false, int kEW = 8>
struct Cfg : EpiCfg<kEW> {
  using EpiCfg<kEW>::kEpiWarps;
  static constexpr uint32_t kEpiBufs =  // staging buffers per warp
      kPeer ? 2 : (kEW == 4 ? MOE_GEMM_EPI_BUFS4 : MOE_GEMM_EPI_BUFS);
  // peer stores double the staging: with 8 epilogue warps that costs one pipeline stage
  static constexpr uint32_t kStages =
      (kCG == 1 ? MOE_GEMM_STAGES : MOE_GEMM_STAGES_PAIR) -
      (kPeer && MOE_GEMM_EPI_BUFS == 1 && kEW == 8 ? 1 : 0);
  static constexpr uint32_t TM = BM * kCG;   // tile rows per work unit
  static constexpr uint32_t BNL = BN / kCG;  // B columns loaded per CTA
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BNL * BK * 2;
  static constexpr uint32_t SMEM_A_OFF = 0;
  static constexpr uint32_t SMEM_B_OFF = SMEM_A_OFF + kStages * A_BYTES;
  static constexpr uint32_t SMEM_EPI_OFF = SMEM_B_OFF + kStages * B_BYTES;
  static constexpr uint32_t SMEM_BAR_OFF = SMEM_EPI_OFF + kEpiWarps * EPI_WARP_BYTES * kEpiBufs;
  static constexpr uint32_t SMEM_BYTES = SMEM_BAR_OFF + 256 + 1024;  // + barriers + alignment
};

struct PeerMaps {
  CUtensorMap m[kMaxPeers];
};

struct TileCoord {
  uint32_t g, s, m0, n0;  // row-M: m0 = row within segment; row-K: m0 = output row
};

template <bool kRowK, uint32_t TM>
__device__ __forceinline__ TileCoord tile_coord(const GemmArgs& a, uint32_t tile) {
  const uint32_t n_tiles = a.N / BN;
  TileCoord c;
  c.n0 = (tile % n_tiles) * BN;
  uint32_t rest = tile / n_tiles;
  if constexpr (!kRowK) {
    const uint32_t nr = a.nrows ? a.nrows : a.seg_rows - a.row0;
    const uint32_t mts = (nr + TM - 1) / TM;
    c.m0 = a.row0 + (rest % mts) * TM;
    rest /= mts;
    c.s = rest % a.S;
    if (a.skip_seg >= 0 && c.s >= static_cast<uint32_t>(a.skip_seg)) ++c.s;
    c.g = rest / a.S;
  } else {
    const uint32_t mts = (a.Mo + TM - 1) / TM;
    c.m0 = (rest % mts) * TM;
    c.g = rest / mts;
    c.s = 0;
  }
  return c;
}

template <bool kRowK, uint32_t TM>
__host__ __device__ __forceinline__ uint32_t num_tiles(const GemmArgs& a) {
  if constexpr (!kRowK)
    return a.G * a.S * (((a.nrows ? a.nrows : a.seg_rows - a.row0) + TM - 1) / TM) * (a.N / BN);
  else
    return a.G * ((a.Mo + TM - 1) / TM) * (a.N / BN);
}

template <bool kRowK>
__device__ __forceinline__ uint32_t num_kblocks(const GemmArgs& a) {
  if constexpr (!kRowK)
    return a.K / BK;
  else
    return a.S * ((a.seg_rows + BK - 1) / BK);
}

template <bool kAMN, bool kBMN, int kEpi, bool kRowK, int kCG, uint32_t kIdx, int kEW>
__global__ void __launch_bounds__(EpiCfg<kEW>::kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmD, const GemmArgs args,
                     const __grid_constant__ PeerMaps pm) {
  using C = Cfg<kCG, (kIdx & kIdxPeerD) != 0, kEW>;
  constexpr uint32_t kStages = C::kStages;
  constexpr uint32_t kEpiWarps = C::kEpiWarps;
  constexpr uint32_t kEpiCols = C::kEpiCols;
  constexpr uint32_t kEpiBufs = C::kEpiBufs;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::SMEM_BAR_OFF);
  uint64_t* empty_bar = full_bar + kStages;
  uint64_t* tfull_bar = empty_bar + kStages;
  uint64_t* tempty_bar = tfull_bar + kAccStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + kAccStages);

  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = threadIdx.x % 32;
  const uint32_t rank = kCG == 2 ? ptx::cluster_ctarank() : 0;  // CTA within the pair
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    ptx::prefetch_tmap(&tmD);
    for (uint32_t i = 0; i < kStages; ++i) {
      // pair: the leader's full barrier collects both CTAs' producer arrivals and TMA bytes
      ptx::mbar_init(&full_bar[i], kCG == 2 && leader ? 2 : 1);
      ptx::mbar_init(&empty_bar[i], 1);
    }
    for (uint32_t i = 0; i < kAccStages; ++i) {
      ptx::mbar_init(&tfull_bar[i], 1);
      ptx::mbar_init(&tempty_bar[i], kEpiWarps * kCG);  // one arrival per epilogue warp (of the pair)
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<kTmemCols, kCG>(tmem_slot);
  ptx::tc_fence_before();
  if constexpr (kCG == 2)
    ptx::cluster_sync();
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch: the prologue above overlapped the previous kernel's tail;
  // operands produced by it are read only after this wait
  pdl_entry();
  long long clk0 = 0;
  uint64_t ns0 = 0;
  if (args.span != nullptr && threadIdx.x == 0) {
    ns0 = globaltimer_ns();
    clk0 = clock64();
    atomicMin(args.span, ns0);
  }
  if (args.wait.base != nullptr && (warp == 0 || warp >= 4)) {
    // fused receive wait: the producer warp polls the peers' flags (ld.acquire.sys) before its
    // first TMA load -- the async proxy must then see what the copy engines wrote before the
    // flags -- and each epilogue warp acquires them itself before reading peer-written row
    // norms or storing into peer buffers
    wait_flags_warp(args.wait);
    if (warp == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
  }

  const uint32_t ntiles = num_tiles<kRowK, C::TM>(args);
  const uint32_t nkb = num_kblocks<kRowK>(args);
  const uint32_t unit0 = blockIdx.x / kCG, unit_step = gridDim.x / kCG;
  long long w_prod = 0, w_full = 0, w_tempty = 0, w_tfull = 0;
#ifdef MOE_GEMM_TRACE
  const long long t_start = clock64();
#endif

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // Like the MMA issuer: the whole warp walks the loop (warp-uniform coordinates), one elected
    // lane issues the loads and the barrier arrival.
    uint32_t stage = 0, phase = 0;
    const uint32_t kb_per_seg = (args.seg_rows + BK - 1) / BK;
    auto load = [&](const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1, int c2) {
      if constexpr (kCG == 2)
        ptx::tma_load_3d_pair(m, bar, dst, c0, c1, c2);
      else
        ptx::tma_load_3d(m, bar, dst, c0, c1, c2);
    };
#if MOE_TMA_4D
    // MN-major operand: all 64-column atoms of the box in one 4-D load ([seg][atom][row][64])
    auto load4 = [&](const CUtensorMap* m, uint64_t* bar, void* dst, int row, int atom, int seg) {
      if constexpr (kCG == 2)
        ptx::tma_load_4d_pair(m, bar, dst, 0, row, atom, seg);
      else
        ptx::tma_load_4d(m, bar, dst, 0, row, atom, seg);
    };
#endif
    // the (A, B) boxes of k-block kb of a tile into one smem stage
    // row-K: k-block kb is block kr of segment ks (kept as counters, no division)
    auto issue = [&](const TileCoord& tc, uint32_t kb, uint32_t ks, uint32_t kr, uint8_t* sa,
                     uint8_t* sb, uint64_t* bar) {
      const uint32_t m0 = tc.m0 + rank * BM;       // this CTA's A rows
      const uint32_t nb = tc.n0 + rank * C::BNL;   // this CTA's B columns
      auto go = [&](const CUtensorMap* m, void* dst, int c0, int c1, int c2) {
        load(m, bar, dst, c0, c1, c2);
      };
      if constexpr (!kRowK) {
        const int seg = static_cast<int>((args.seg_base + tc.s) * args.G + tc.g);
        const int k0 = static_cast<int>(kb * BK);
        // A: K-major [seg][seg_rows][K]
        go(&tmA, sa, k0, static_cast<int>(m0), seg);
        if constexpr (!kBMN) {
          // B: K-major [G][N][K]
          go(&tmB, sb, k0, static_cast<int>(nb), static_cast<int>(tc.g));
        } else {
          // B: N-major [G][K][N], 64-column atoms
#if MOE_TMA_4D
          load4(&tmB, bar, sb, k0, static_cast<int>(nb / 64), static_cast<int>(tc.g));
#else
#pragma unroll
          for (uint32_t a = 0; a < C::BNL / 64; ++a)
            go(&tmB, sb + a * (BK * 128), static_cast<int>(nb + a * 64), k0, static_cast<int>(tc.g));
#endif
        }
      } else {
        const int r0 = static_cast<int>(kr * BK);
        const int seg = static_cast<int>((args.seg_base + ks) * args.G + tc.g);
        // A^T: rows are K, MN-major [seg][seg_rows][Mo]; B: N-major [seg][seg_rows][N]
#if MOE_TMA_4D
        load4(&tmA, bar, sa, r0, static_cast<int>(m0 / 64), seg);
        load4(&tmB, bar, sb, r0, static_cast<int>(nb / 64), seg);
#else
#pragma unroll
        for (uint32_t a = 0; a < BM / 64; ++a)
          go(&tmA, sa + a * (BK * 128), static_cast<int>(m0 + a * 64), r0, seg);
#pragma unroll
        for (uint32_t a = 0; a < C::BNL / 64; ++a)
          go(&tmB, sb + a * (BK * 128), static_cast<int>(nb + a * 64), r0, seg);
#endif
      }
    };
    for (uint32_t tile = unit0; tile < ntiles; tile += unit_step) {
      const TileCoord tc = tile_coord<kRowK, C::TM>(args, tile);
      uint32_t ks = 0, kr = 0;
      for (uint32_t kb = 0; kb < nkb; ++kb) {
        ptx::mbar_wait(&empty_bar[stage], phase ^ 1);
        uint8_t* sa = smem + C::SMEM_A_OFF + stage * C::A_BYTES;
        uint8_t* sb = smem + C::SMEM_B_OFF + stage * C::B_BYTES;
        if (ptx::elect_one()) {
          issue(tc, kb, ks, kr, sa, sb, &full_bar[stage]);
          if (leader)
            ptx::mbar_arrive_expect_tx(&full_bar[stage], (C::A_BYTES + C::B_BYTES) * kCG);
          else
            ptx::mbar_arrive_cluster(&full_bar[stage], 0);
        }
        __syncwarp();
        if (++kr == kb_per_seg) {
          kr = 0;
          ++ks;
        }
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && leader) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    // The whole warp walks the loop so descriptors stay warp-uniform (uniform datapath, no
    // per-MMA register-to-uniform broadcast); one elected lane issues. The issue path shares its
    // SM sub-partition with two epilogue warps, so its instruction count is on the critical path
    // of the K = 1024 GEMMs.
    constexpr uint32_t idesc = ptx::make_idesc_bf16(C::TM, BN, kAMN, kBMN);
    // descriptor of stage 0, k-step 0; stage s / k-step k add (s * bytes + k * step) >> 4
    constexpr uint32_t kAStep = kAMN ? 2048 : 32, kBStep = kBMN ? 2048 : 32;
    const uint64_t adesc0 = kAMN ? ptx::make_sw128_desc(ptx::smem_u32(smem + C::SMEM_A_OFF), BK * 128, 1024)
                                 : ptx::make_sw128_desc(ptx::smem_u32(smem + C::SMEM_A_OFF), 16, 1024);
    const uint64_t bdesc0 = kBMN ? ptx::make_sw128_desc(ptx::smem_u32(smem + C::SMEM_B_OFF), BK * 128, 1024)
                                 : ptx::make_sw128_desc(ptx::smem_u32(smem + C::SMEM_B_OFF), 16, 1024);
    uint32_t stage = 0, phase = 0;
    uint32_t iter = 0;
    for (uint32_t tile = unit0; tile < ntiles; tile += unit_step, ++iter) {
      const uint32_t acc = iter % kAccStages;
      const uint32_t acc_phase = (iter / kAccStages) & 1;
      TRACE_WAIT(w_tempty, ptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1));
      ptx::tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (uint32_t kb = 0; kb < nkb; ++kb) {
        TRACE_WAIT(w_full, ptx::mbar_wait(&full_bar[stage], phase));
        ptx::tc_fence_after();
        const uint64_t ad = adesc0 + ((stage * C::A_BYTES) >> 4);
        const uint64_t bd = bdesc0 + ((stage * C::B_BYTES) >> 4);
        if (ptx::elect_one()) {
#pragma unroll
          for (uint32_t k = 0; k < BK / UK; ++k) {
            const uint64_t adesc = ad + ((k * kAStep) >> 4);
            const uint64_t bdesc = bd + ((k * kBStep) >> 4);
            if constexpr (kCG == 2)
              ptx::umma_bf16_pair(tmem_d, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
            else
              ptx::umma_bf16(tmem_d, adesc, bdesc, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          if constexpr (kCG == 2) {
            ptx::umma_commit_pair(&empty_bar[stage]);
            if (kb == nkb - 1) ptx::umma_commit_pair(&tfull_bar[acc]);
          } else {
            ptx::umma_commit(&empty_bar[stage]);
            if (kb == nkb - 1) ptx::umma_commit(&tfull_bar[acc]);
          }
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    // 8 warps: warp w reads TMEM lane quadrant w % 4 (32 rows) and column half (w - 4) / 4 of
    // the 128 x 256 accumulator; each 128-byte-wide sub-chunk (64 bf16 / 32 fp32 columns) goes
    // registers -> warp-private 128B-swizzled smem -> one TMA bulk store by lane 0.
    const uint32_t q = warp % 4;
    const uint32_t half = (warp - 4) / 4;  // column slice of this warp
    const uint32_t row = q * 32 + lane;
    constexpr uint32_t kSub = (kEpi == kEpiF32) ? 32 : 64;  // columns per 128-byte sub-chunk
    constexpr uint32_t kSubs = kEpiCols / kSub;
    constexpr uint32_t kStoreLanes = (kIdx & kIdxScatterD) ? 8 : 1;  // lanes issuing bulk stores
    uint8_t* stage_base = smem + C::SMEM_EPI_OFF + (warp - 4) * EPI_WARP_BYTES * kEpiBufs;
    uint32_t ebuf = 0;
    uint32_t iter = 0;
    for (uint32_t tile = unit0; tile < ntiles; tile += unit_step, ++iter) {
      TileCoord tc = tile_coord<kRowK, C::TM>(args, tile);
      tc.m0 += rank * BM;  // this CTA's rows of the pair tile
      const uint32_t acc = iter % kAccStages;
      const uint32_t acc_phase = (iter / kAccStages) & 1;
      const uint32_t tmem_row = tmem_base + acc * BN + ((q * 32) << 16) + half * kEpiCols;
      const uint32_t seg = kRowK ? tc.g : (args.seg_base + tc.s) * args.G + tc.g;
      const uint32_t row_in = tc.m0 + row;
      const bool row_ok =
          kRowK || row_in < (args.nrows ? min(args.seg_rows, args.row0 + args.nrows) : args.seg_rows);
      const uint32_t col0 = tc.n0 + half * kEpiCols;
      const size_t orow = static_cast<size_t>(seg) * args.seg_rows + row_in;  // row-M kinds
      const size_t mrow = relu_mask_word(orow, col0 / 64, args.N / 64);  // + 32 per 64 columns
      // token-indexed epilogue: the row's token (scatter) and gate scale
      int tok = -1;
      float scale = 1.0f;
      if constexpr ((kIdx & kIdxScatterD) != 0)
        tok = row_ok ? __ldg(args.row_token + orow) : -1;
      if constexpr ((kIdx & kIdxScaleRow) != 0)
        scale = row_ok ? __ldg(args.row_scale + orow) : 0.0f;
      int st_tok[4];
      if constexpr ((kIdx & kIdxScatterD) != 0) {
        // lane j < 8 stores rows 4j .. 4j + 3 of this warp's 32 with one scatter4
        const int t = tok < 0 ? static_cast<int>(args.gather_rows) : tok;
#pragma unroll
        for (int i = 0; i < 4; ++i) st_tok[i] = __shfl_sync(0xffffffffu, t, 4 * (lane & 7) + i);
      }
      // ReLU certificate inputs of this tile (row bound, 64-column block bounds), loaded before the
      // accumulator wait like the mask words
      float rmax = 0.0f, tblk[kSubs];
      const bool cert = kEpi == kEpiReluBf16 && args.fix_list != nullptr && row_ok;
      if constexpr (kEpi == kEpiReluBf16) {
        if (cert) {
          // coherent load: peers' row norms may have landed after this kernel started
          rmax = __ldcg(args.rownorm + orow) * kReluTauScale;
#pragma unroll
          for (uint32_t c = 0; c < kSubs; ++c)
            tblk[c] = rmax * __ldg(args.colnorm_blk + static_cast<size_t>(tc.g) * (args.N / 64) + col0 / 64 + c);
        }
      }
      unsigned long long mw[kSubs];
      if constexpr (kEpi == kEpiMaskBf16) {
        // issued before the accumulator wait so their latency hides under the MMAs
#pragma unroll
        for (uint32_t c = 0; c < kSubs; ++c)
          mw[c] = row_ok ? __ldg(args.relu_mask + mrow + 32 * c) : 0ull;
      }
      TRACE_WAIT(w_tfull, ptx::mbar_wait(&tfull_bar[acc], acc_phase));
      ptx::tc_fence_after();
#pragma unroll 1
      for (uint32_t c = 0; c < kSubs; ++c) {
        uint32_t v[kSub];
        if constexpr (kSub == 32) {
          ptx::tmem_ld_32x32b_x32(tmem_row + c * kSub, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        } else {
          ptx::tmem_ld_32x32b_x32(tmem_row + c * kSub, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
          ptx::tmem_ld_32x32b_x32(tmem_row + c * kSub + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        }
        ptx::tmem_ld_wait();
        if (c == kSubs - 1) {
          // accumulator drained into registers: hand TMEM back to the (leader's) MMA warp
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (kCG == 2)
              ptx::mbar_arrive_cluster(&tempty_bar[acc], 0);
            else
              ptx::mbar_arrive(&tempty_bar[acc]);
          }
        }
#ifdef MOE_EXP_DRAIN_ONLY  // timing experiments only: the up epilogue drains TMEM, nothing else
        if constexpr (kEpi == kEpiReluBf16) {
          uint32_t acc_or = 0u;
#pragma unroll
          for (uint32_t i = 0; i < kSub; ++i) acc_or |= v[i];
          if (acc_or == 0x7fc00001u) args.fix_count[1] = acc_or;  // keeps the loads live
          continue;
        }
#endif
        const uint32_t cols = col0 + c * kSub;
        uint8_t* stage = stage_base + ebuf * EPI_WARP_BYTES;
        const uint32_t stage_row = ptx::smem_u32(stage) + lane * 128;
        ebuf = (ebuf + 1) % kEpiBufs;
        // the TMA store that last used this staging buffer must have finished reading it
        if (lane < kStoreLanes) ptx::tma_store_wait_read<kEpiBufs - 1>();
        __syncwarp();
        if constexpr (kEpi == kEpiF32) {
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j)
            ptx::st_shared_v4(stage_row + ((j ^ (lane & 7)) << 4), v[4 * j], v[4 * j + 1],
                              v[4 * j + 2], v[4 * j + 3]);
        } else {
          float f[64];
#pragma unroll
          for (uint32_t i = 0; i < 64; ++i) f[i] = __uint_as_float(v[i]);
          if constexpr ((kIdx & kIdxScaleRow) != 0) {
            // fused decode: y[token] = g * (act . W2)[slot]
#pragma unroll
            for (uint32_t i = 0; i < 64; ++i) f[i] *= scale;
          }
          uint32_t w[32];  // the 64 outputs as bf16 pairs (round to nearest even)
#pragma unroll
          for (uint32_t j = 0; j < 32; ++j) w[j] = ptx::pack_bf16x2(f[2 * j], f[2 * j + 1]);
          if constexpr (kEpi == kEpiReluBf16) {
            // mn = min |bf16(h)| over the 64 columns (magnitude order == unsigned order of the 15
            // low bits): the certificate prefilter, and mn > 0 (no zero) lets the mask come from
            // the sign bits alone
            bool signs = false;
#ifndef MOE_EXP_NO_CERT  // timing experiments only (tools/gemm_exp.sh): drops the certificate
            if (cert) {
              // ReLU-mask certificate: |h| below the accumulation-error bound -> fp64
              // re-decision. Prefilter: mn against the block bound widened by 2^-7 for the
              // rounding; on a hit, the exact per-element test on the fp32 values.
              float tmax = 0.0f;
#pragma unroll
              for (uint32_t c2 = 0; c2 < kSubs; ++c2)
                if (c2 == c) tmax = tblk[c2];
              // (a reduction tree: the epilogue is latency-bound, a 32-deep chain is not free)
              uint32_t m16[16];
#pragma unroll
              for (uint32_t j = 0; j < 16; ++j)
                m16[j] = __vminu2(w[2 * j] & 0x7fff7fffu, w[2 * j + 1] & 0x7fff7fffu);
#pragma unroll
              for (uint32_t h = 8; h > 0; h /= 2)
#pragma unroll
                for (uint32_t j = 0; j < h; ++j) m16[j] = __vminu2(m16[j], m16[j + h]);
              const float mn = __uint_as_float(min(m16[0] & 0xffffu, m16[0] >> 16) << 16);
              signs = mn > 0.0f;
              if (mn < tmax * (1.0f + 1.0f / 128.0f)) {
                // exact test of all 64 columns first (loads free to run ahead), then one
                // atomic reservation for this row's entries
                const float* ca = args.colnorm + static_cast<size_t>(tc.g) * args.N + cols;
                unsigned long long hits = 0ull;
#pragma unroll
                for (uint32_t i = 0; i < 64; ++i)
                  hits |= static_cast<unsigned long long>(fabsf(f[i]) < rmax * __ldg(ca + i)) << i;
                if (hits != 0ull) {
                  unsigned int slot = atomicAdd(args.fix_count, static_cast<unsigned int>(__popcll(hits)));
                  while (hits != 0ull) {
                    const uint32_t i = static_cast<uint32_t>(__ffsll(static_cast<long long>(hits)) - 1);
                    hits &= hits - 1;
                    MOE_CHECK(seg < (1u << 20) && row_in < (1u << 20) && cols + i < (1u << 24),
                              "up epilogue: certificate entry does not fit its packing");
                    if (slot < args.fix_cap) args.fix_list[slot] = fix_pack(seg, row_in, cols + i);
                    ++slot;
                  }
                }
              }
            }
#endif
#ifndef MOE_EXP_NO_MASK  // timing experiments only: drops the ReLU bitmask
            // [h > 0] bits in the relu_mask.cuh order. No zero among the 64 values: [h > 0] is
            // the inverted sign bit, gathered by one funnel shift per column; else compares.
            uint32_t lo = 0u, hi = 0u;
            if (signs) {
              // four independent 8-deep chains per half instead of one 32-deep chain
              uint32_t g[8];
#pragma unroll
              for (uint32_t q = 0; q < 8; ++q) {
                g[q] = 0u;  // bits 8 (q % 4) .. + 7 of half q / 4
#pragma unroll
                for (int b = 7; b >= 0; --b)
                  g[q] = __funnelshift_l(v[32 * (q / 4) + relu_mask_col(8 * (q % 4) + b)], g[q], 1);
              }
              lo = ~(g[0] | (g[1] << 8) | (g[2] << 16) | (g[3] << 24));
              hi = ~(g[4] | (g[5] << 8) | (g[6] << 16) | (g[7] << 24));
            } else {
#pragma unroll
              for (uint32_t b = 0; b < 32; ++b) {
                lo |= static_cast<uint32_t>(f[relu_mask_col(b)] > 0.0f) << b;
                hi |= static_cast<uint32_t>(f[32 + relu_mask_col(b)] > 0.0f) << b;
              }
            }
            if (args.relu_mask != nullptr && row_ok)
              args.relu_mask[mrow + 32 * c] = (static_cast<unsigned long long>(hi) << 32) | lo;
#endif
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) w[j] = __vmaxs2(w[j], 0u);  // int16 max == bf16 relu
          }
          if constexpr (kEpi == kEpiMaskBf16) {
            // dh = (dY . W2^T) * [h > 0]; the up-GEMM's ReLU bitmask carries [h > 0]
            unsigned long long mk = 0ull;
#pragma unroll
            for (uint32_t c2 = 0; c2 < kSubs; ++c2)
              if (c2 == c) mk = mw[c2];
            uint32_t pm[32];
            relu_mask_pairs(mk, pm);
#pragma unroll
            for (uint32_t j = 0; j < 32; ++j) w[j] &= pm[j];
          }
#pragma unroll
          for (uint32_t j = 0; j < 8; ++j)
            ptx::st_shared_v4(stage_row + ((j ^ (lane & 7)) << 4), w[4 * j], w[4 * j + 1],
                              w[4 * j + 2], w[4 * j + 3]);
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if constexpr ((kIdx & kIdxScatterD) != 0) {
          if (lane < 8) {
            // rows to token positions; empty slots / rows past the segment end are out of bounds
            ptx::tma_scatter4(&tmD, stage + lane * 512, static_cast<int>(cols), st_tok[0],
                              st_tok[1], st_tok[2], st_tok[3]);
            ptx::tma_store_commit();
          }
        } else if constexpr ((kIdx & kIdxPeerD) != 0) {
          if (lane == 0) {
            // fused combine: this tile's rows go straight to the source rank's combine buffer
            const uint32_t sidx = args.seg_base + tc.s;  // chunk * W + src
            const uint32_t src = sidx % args.peer_world;
            const uint32_t oseg = (sidx / args.peer_world) * args.peer_world * args.G +
                                  args.peer_rank * args.G + tc.g;
            ptx::tma_store_3d(&pm.m[src], stage, static_cast<int>(cols),
                              static_cast<int>(tc.m0 + q * 32), static_cast<int>(oseg));
            ptx::tma_store_commit();
          }
        } else if (lane == 0) {
          // rows past the segment end are clipped by the tensor map bounds
          ptx::tma_store_3d(&tmD, stage, static_cast<int>(cols), static_cast<int>(tc.m0 + q * 32),
                            static_cast<int>(seg));
          ptx::tma_store_commit();
        }
      }
    }
    if (lane < kStoreLanes) {
      ptx::tma_store_wait_all<0>();
      // peer stores: performed system-wide before the stream publishes the ready flags
      if constexpr ((kIdx & kIdxPeerD) != 0) __threadfence_system();
    }
  }

#ifdef MOE_GEMM_TRACE
  if (blockIdx.x < 2 && lane == 0 && (warp <= 1 || warp == 4 || warp == 11))
    printf("trace cta %d warp %d: total %lld prod_empty %lld mma_full %lld mma_tempty %lld epi_tfull %lld\n",
           blockIdx.x, warp, clock64() - t_start, w_prod, w_full, w_tempty, w_tfull);
#endif
  (void)w_prod; (void)w_full; (void)w_tempty; (void)w_tfull;
  __syncwarp();
  ptx::tc_fence_before();
  if constexpr (kCG == 2)
    ptx::cluster_sync();  // the peer's remote arrivals / MMA reads must be done before exit
  else
    __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc<kTmemCols, kCG>(tmem_base);
  if (args.span != nullptr && threadIdx.x == 0) {
    const uint64_t ns1 = globaltimer_ns();
    atomicMax(args.span + 1, ns1);
    if (blockIdx.x == 0) {  // CTA 0's own SM clock over its lifetime: cycles, ns
      args.span[2] = static_cast<unsigned long long>(clock64() - clk0);
      args.span[3] = ns1 - ns0;
    }
  }
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int make_map_3d(CUtensorMap* m, const void* base, bool f32, uint64_t d0, uint64_t d1, uint64_t d2,
                uint32_t b0, uint32_t b1) {
  auto fn = encode_fn();
  if (!fn) return -1;
  const uint64_t esz = f32 ? 4 : 2;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * esz, d0 * d1 * esz};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                  const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

// 4-D view [d2][d0 / 64][d1][64] of a 3-D bf16 [d2][d1][d0] tensor: box {64, b1, atoms, 1}
// lands `atoms` 64-column swizzle atoms of b1 rows back to back (one TMA op per MN-major stage).
int make_map_mn4(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b1,
                 uint32_t atoms) {
  auto fn = encode_fn();
  if (!fn) return -1;
  if (d0 % 64 != 0) return -3;
  cuuint64_t dims[4] = {64, d1, d0 / 64, d2};
  cuuint64_t strides[3] = {d0 * 2, 128, d0 * d1 * 2};
  cuuint32_t box[4] = {64, b1, atoms, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

// 2-D [rows][cols] bf16 map with a one-row box: the row-scatter (tile::scatter4) target.
int make_map_rows(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows) {
  auto fn = encode_fn();
  if (!fn) return -1;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : -2;
}

template <bool kAMN, bool kBMN, int kEpi, bool kRowK, int kCG, uint32_t kIdx, int kEW>
int launch_cg(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& d, const GemmArgs& args,
              const PeerMaps& pm, int num_sms, cudaStream_t stream) {
  using C = Cfg<kCG, (kIdx & kIdxPeerD) != 0, kEW>;
  auto kern = gemm_bf16_kernel<kAMN, kBMN, kEpi, kRowK, kCG, kIdx, kEW>;
  if (!smem_optin(kern, C::SMEM_BYTES)) return -3;
  const uint32_t units = num_tiles<kRowK, C::TM>(args);
  if (units == 0) return 0;
  // persistent: one CTA (pair) per SM (pair of SMs)
  const uint32_t max_units = static_cast<uint32_t>(num_sms) / kCG;
  const uint32_t grid = (units < max_units ? units : max_units) * kCG;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  if (cudaLaunchKernelEx(&cfg, kern, a, b, d, args, pm) != cudaSuccess) return launch_status() ? -2 : -2;
  return launch_status();
}

// CTA-pair (cta_group::2) kernel by default; MOE_GEMM_CG=1 selects the single-CTA kernel.
int gemm_cta_group() {
  static int cg = [] {
    const char* e = std::getenv("MOE_GEMM_CG");
    return (e && e[0] == '1') ? 1 : 2;
  }();
  return cg;
}

template <bool kAMN, bool kBMN, int kEpi, bool kRowK, uint32_t kIdx = 0>
int launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& d, const GemmArgs& args,
           int num_sms, cudaStream_t stream, const PeerMaps* pm = nullptr) {
  static const PeerMaps none{};
  const PeerMaps& p = pm ? *pm : none;
#ifndef MOE_UP_EPI_WARPS
#define MOE_UP_EPI_WARPS 8
#endif
#ifndef MOE_WGRAD_EPI_WARPS
#define MOE_WGRAD_EPI_WARPS 4
#endif
#ifndef MOE_EPI_WARPS
#define MOE_EPI_WARPS 4
#endif
  constexpr int kEW = kEpi == kEpiReluBf16 ? MOE_UP_EPI_WARPS
                      : kEpi == kEpiF32    ? MOE_WGRAD_EPI_WARPS
                                           : MOE_EPI_WARPS;  // see EpiCfg
  if (gemm_cta_group() == 2)
    return launch_cg<kAMN, kBMN, kEpi, kRowK, 2, kIdx, kEW>(a, b, d, args, p, num_sms, stream);
  return launch_cg<kAMN, kBMN, kEpi, kRowK, 1, kIdx, kEW>(a, b, d, args, p, num_sms, stream);
}

}  // namespace

// Public wrapper (gate_tc.cu): a 3-D bf16 / fp32 tensor map with a {b0, b1, 1} box, 128-byte swizzle.
int tensor_map_3d(CUtensorMap* m, const void* base, bool f32, uint64_t d0, uint64_t d1, uint64_t d2,
                  uint32_t b0, uint32_t b1) {
  return make_map_3d(m, base, f32, d0, d1, d2, b0, b1);
}

int gemm_validate(const GemmArgs& a, int kind) {
  if (a.G < 1 || a.S < 1 || a.seg_rows < 1 || a.N < 1) return -1;
  if (kind != kGemmWgrad) {
    if (a.row0 >= a.seg_rows || a.row0 % 256 || a.row0 + a.nrows > a.seg_rows) return -1;
    if (a.nrows && a.nrows % 256 && a.row0 + a.nrows != a.seg_rows) return -1;
  } else if (a.row0 || a.nrows || a.skip_seg >= 0) {
    return -1;
  }
  if (a.N % BN != 0) return -1;
  if (kind == kGemmWgrad) {
    if (a.Mo % BM != 0) return -1;
  } else {
    if (a.K % BK != 0 || a.K < BK) return -1;
  }
  return 0;
}

// X:[nseg][seg_rows][K] bf16, W:[G][K][N] bf16 (row-major, N-major), D:[nseg][seg_rows][N]
int gemm_fwd(GemmKind kind, const void* A, const void* B, void* D, const GemmArgs& args_in,
             int nseg_total, int num_sms, cudaStream_t stream) {
  if (gemm_validate(args_in, kind) != 0) return -1;
  GemmArgs args = args_in;
  args.d_ptr = D;
  CUtensorMap ma, mb, md;
  const uint64_t nseg = static_cast<uint64_t>(nseg_total);
  int rc = 0;
  const uint32_t im = args.idx_mode;
  if ((im & kIdxScatterD) && (args.row_token == nullptr || args.gather_rows == 0)) return -1;
  if ((im & kIdxScaleRow) && args.row_scale == nullptr) return -1;
  PeerMaps pm{};
  if (im & kIdxPeerD) {
    if (kind != kGemmDown && kind != kGemmDgrad) return -1;
    if (args.peer_world < 2 || args.peer_world > kMaxPeers || args.peer_rank >= args.peer_world ||
        args.S != args.peer_world || args.peer_out_segs == 0)
      return -1;
    for (uint32_t p = 0; p < args.peer_world; ++p) {
      if (args.peer_d[p] == nullptr) return -1;
      if (make_map_3d(&pm.m[p], args.peer_d[p], false, args.N, args.seg_rows, args.peer_out_segs, 64, 32))
        return -2;
    }
  }
  auto map_d = [&](CUtensorMap* m) {
    return (im & kIdxScatterD) ? make_map_rows(m, D, args.N, args.gather_rows)
                               : make_map_3d(m, D, false, args.N, args.seg_rows, nseg, 64, 32);
  };
  switch (kind) {
    case kGemmUp:      // act = relu(X . W1)      A K-major, W1 [G][K=M][N=V] N-major
    case kGemmDown: {  // Y   = act . W2          A K-major, W2 [G][K=V][N=M] N-major
      rc |= make_map_3d(&ma, A, false, args.K, args.seg_rows, nseg, 64, BM);
#if MOE_TMA_4D
      rc |= make_map_mn4(&mb, B, args.N, args.K, args.G, 64, BN / gemm_cta_group() / 64);
#else
      rc |= make_map_3d(&mb, B, false, args.N, args.K, args.G, 64, 64);
#endif
      rc |= map_d(&md);
      if (rc) return -2;
      if (kind == kGemmUp)
        return im == 0 ? launch<false, true, kEpiReluBf16, false>(ma, mb, md, args, num_sms, stream) : -1;
      if (im == 0) return launch<false, true, kEpiBf16, false>(ma, mb, md, args, num_sms, stream);
      if (im == (kIdxScatterD | kIdxScaleRow))  // fused decode
        return launch<false, true, kEpiBf16, false, kIdxScatterD | kIdxScaleRow>(ma, mb, md, args,
                                                                                 num_sms, stream);
      if (im == kIdxPeerD)  // fused combine
        return launch<false, true, kEpiBf16, false, kIdxPeerD>(ma, mb, md, args, num_sms, stream, &pm);
      return -1;
    }
    case kGemmDgradMask:  // dh = (dY . W2^T) * [a > 0]; W2 [G][V][M] == B K-major [G][N=V][K=M]
      if (args.relu_mask == nullptr) return -1;
      [[fallthrough]];
    case kGemmDgrad: {    // dX = dh . W1^T;             W1 [G][M][V] == B K-major [G][N=M][K=V]
      rc |= make_map_3d(&ma, A, false, args.K, args.seg_rows, nseg, 64, BM);
      rc |= make_map_3d(&mb, B, false, args.K, args.N, args.G, 64, BN / gemm_cta_group());
      rc |= map_d(&md);
      if (rc) return -2;
      if (kind == kGemmDgradMask)
        return im == 0 ? launch<false, false, kEpiMaskBf16, false>(ma, mb, md, args, num_sms, stream) : -1;
      if (im == 0) return launch<false, false, kEpiBf16, false>(ma, mb, md, args, num_sms, stream);
      if (im == kIdxScatterD)  // fused encode-backward
        return launch<false, false, kEpiBf16, false, kIdxScatterD>(ma, mb, md, args, num_sms, stream);
      if (im == kIdxPeerD)  // fused backward combine
        return launch<false, false, kEpiBf16, false, kIdxPeerD>(ma, mb, md, args, num_sms, stream, &pm);
      return -1;
    }
    case kGemmWgrad: {  // dW[g] = A[g]^T . B[g] over all (segment, row); fp32 out [G][Mo][N]
      if (im != 0) return -1;
#if MOE_TMA_4D
      rc |= make_map_mn4(&ma, A, args.Mo, args.seg_rows, nseg, 64, BM / 64);
      rc |= make_map_mn4(&mb, B, args.N, args.seg_rows, nseg, 64, BN / gemm_cta_group() / 64);
#else
      rc |= make_map_3d(&ma, A, false, args.Mo, args.seg_rows, nseg, 64, 64);
      rc |= make_map_3d(&mb, B, false, args.N, args.seg_rows, nseg, 64, 64);
#endif
      rc |= make_map_3d(&md, D, true, args.N, args.Mo, args.G, 32, 32);
      if (rc) return -2;
      return launch<true, true, kEpiF32, true>(ma, mb, md, args, num_sms, stream);
    }
  }
  return -1;
}

}  // namespace moe
