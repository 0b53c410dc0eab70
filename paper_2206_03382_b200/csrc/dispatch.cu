// Sparse dispatch / combine kernels (HBM-bound, 128-bit vectorised, one warp per row).
//
// Reference semantics (dispatch.cpp):
//   fast_encode_range            :51-62   Z <- 0; Z[idx, loc, :] = x[t, :] for kept (t, j)
//   fast_decode_range            :75-87   y[t, :] += g * Z[idx, loc, :], j ascending
//   fast_decode_backward_range   :136-157 dZ[idx, loc] += g * dy[t];  d_gates = <Z, dy>
//   fast_encode_backward_range   :117-128 dx[t] += dZ[idx, loc]
// Encode and decode-backward are written slot-major (a gather per capacity row, driven by the
// slot -> token table built during location assignment), so the zero fill of empty and padded
// capacity rows is fused into the same coalesced pass and no scatter/atomics are needed. Decode
// and encode-backward are token-major gathers. Slot rows use the pipelined-chunk layout
// [block][chunk][expert][cc][M] (partition_capacity, pipeline.cpp:33-51), which is exactly the
// send layout of the flexible all-to-all, so chunking costs no copy.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "checks.cuh"
#include "kernels.h"
#include "pdl.cuh"
#include "peer_flags.cuh"

namespace moe {

namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kUnroll = 4;

__device__ __forceinline__ size_t slot_row(const SlotGeom& g, int b, int e, int c) {
  return static_cast<size_t>(b) * g.degree * g.E * g.cc +
         static_cast<size_t>((c / g.cc) * g.E + e) * g.cc + (c % g.cc);
}

template <typename T>
struct Vec;  // 16-byte vector of T
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static void to_f32(const uint4& v, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 p = __bfloat1622float2(h[i]);
      f[2 * i] = p.x;
      f[2 * i + 1] = p.y;
    }
  }
  __device__ static uint4 from_f32(const float (&f)[8]) {
    uint4 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return v;
  }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static void to_f32(const uint4& v, float (&f)[4]) {
    f[0] = __uint_as_float(v.x);
    f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z);
    f[3] = __uint_as_float(v.w);
  }
  __device__ static uint4 from_f32(const float (&f)[4]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
};

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
__device__ __forceinline__ float to_f(float v) { return v; }
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <>
__device__ __forceinline__ float from_f<float>(float v) {
  return v;
}

// Zero the rows of fully dropped tokens (one thread checks one token, the warp writes its
// dropped tokens' rows together). Warp-uniform loop: every lane takes part in the ballot.
__device__ __forceinline__ void zero_dropped_rows(const DropZero& d) {
  if (d.out == nullptr) return;
  const int lane = threadIdx.x % 32;
  const int vecs = static_cast<int>(d.row_bytes / 16);
  for (int base = blockIdx.x * blockDim.x + threadIdx.x - lane; base < d.T;
       base += gridDim.x * blockDim.x) {
    const int t = base + lane;
    bool dropped = t < d.T;
    for (int j = 0; j < d.k && dropped; ++j) dropped = __ldg(d.locations + static_cast<size_t>(t) * d.k + j) < 0;
    unsigned m = __ballot_sync(0xffffffffu, dropped);
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      uint4* r = static_cast<uint4*>(d.out) + static_cast<size_t>(base + src) * vecs;
      for (int v = lane; v < vecs; v += 32) r[v] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
}

// Destination row of slot-major row `row` = (block b, chunk i, expert e, slot c % cc): the send
// buffer, or (this rank's experts, LocalDest) the receive buffer's own-source segment.
__device__ __forceinline__ bool is_own(const LocalDest& ld, int e) {
  return ld.all_peers || (ld.recv != nullptr && e / ld.dE == ld.rank);
}
__device__ __forceinline__ size_t own_row(const LocalDest& ld, const SlotGeom& g, int i, int e, int rem) {
  return (static_cast<size_t>(i * ld.W + ld.rank) * ld.dE + (e - ld.rank * ld.dE)) * g.cc + rem % g.cc;
}
// fused dispatch: expert e's owner p receives this rank's rows at source segment `rank`
__device__ __forceinline__ size_t peer_row(const LocalDest& ld, const SlotGeom& g, int i, int e, int rem) {
  const int p = e / ld.dE;
  return (static_cast<size_t>(i * ld.W + ld.rank) * ld.dE + (e - p * ld.dE)) * g.cc + rem % g.cc;
}
template <typename T>
__device__ __forceinline__ T* gather_dst(T* z, const LocalDest& ld, const SlotGeom& g, size_t row,
                                         int i, int e, int rem) {
  if (ld.all_peers) return static_cast<T*>(ld.peer_recv[e / ld.dE]) + peer_row(ld, g, i, e, rem) * g.M;
  if (is_own(ld, e)) return static_cast<T*>(ld.recv) + own_row(ld, g, i, e, rem) * g.M;
  return z + row * g.M;
}
__device__ __forceinline__ bool want_norm(const float* rownorm, const LocalDest& ld, int e) {
  if (ld.all_peers) return ld.peer_norm[e / ld.dE] != nullptr;
  return rownorm != nullptr || (ld.recv_norm != nullptr && is_own(ld, e));
}
// fused dispatch: before the first store into a peer's receive buffer every peer must have
// released it (freed flags of the previous epoch); CTA-uniform
__device__ __forceinline__ void wait_peers_released(const LocalDest& ld) {
  if (!ld.all_peers || ld.freed.base == nullptr) return;
  if (threadIdx.x < 32) wait_flags_warp(ld.freed);
  __syncthreads();
}
// where the row's norm goes: the receive-side array for own rows (if given), else z order
__device__ __forceinline__ float* norm_dst(float* rownorm, const LocalDest& ld, const SlotGeom& g,
                                           size_t row, int i, int e, int rem) {
  if (ld.all_peers) {
    float* pn = ld.peer_norm[e / ld.dE];
    return pn ? pn + peer_row(ld, g, i, e, rem) : nullptr;
  }
  if (is_own(ld, e) && ld.recv_norm != nullptr) return ld.recv_norm + own_row(ld, g, i, e, rem);
  return rownorm ? rownorm + row : nullptr;
}

// ------------------------------------------------------------------ encode
// Z[row] = x[slot_token[row]] or 0. Rows enumerate [block][chunk][expert][cc].
template <typename T, bool kVec>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    encode_kernel(SlotGeom g, const T* __restrict__ x, const int32_t* __restrict__ slot_token,
                  T* __restrict__ z, float* __restrict__ rownorm, DropZero dzero,
                  unsigned int* __restrict__ reset, LocalDest ld) {
  pdl_entry();
  if (reset != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *reset = 0u;
  zero_dropped_rows(dzero);
  wait_peers_released(ld);
  const int lane = threadIdx.x % 32;
  const size_t rows = static_cast<size_t>(g.blocks) * g.degree * g.E * g.cc;
  const size_t per_block = static_cast<size_t>(g.degree) * g.E * g.cc;
  for (size_t row = static_cast<size_t>(blockIdx.x) * kWarpsPerCta + threadIdx.x / 32; row < rows;
       row += static_cast<size_t>(gridDim.x) * kWarpsPerCta) {
    const int b = static_cast<int>(row / per_block);
    const int rem = static_cast<int>(row % per_block);
    const int i = rem / (g.E * g.cc);
    const int e = (rem / g.cc) % g.E;
    const int c = i * g.cc + rem % g.cc;
    const int t = c < g.cap ? slot_token[static_cast<size_t>(b * g.E + e) * g.cap + c] : -1;
    MOE_CHECK(t == -1 || (t >= b * g.T && t < (b + 1) * g.T), "encode: slot token outside its block");
    if constexpr (kVec) {
      constexpr int VN = Vec<T>::N;
      const int nv = g.M / VN;
      uint4* dst = reinterpret_cast<uint4*>(gather_dst(z, ld, g, row, i, e, rem));
      float ssq = 0.0f;
      if (t < 0) {
        for (int v = lane; v < nv; v += 32) dst[v] = make_uint4(0, 0, 0, 0);
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * g.M);
        for (int v0 = 0; v0 < nv; v0 += 32 * kUnroll) {
          uint4 buf[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nv) buf[u] = ld_stream(src + v);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nv) {
              dst[v] = buf[u];
              if (want_norm(rownorm, ld, e)) {
                float f[VN];
                Vec<T>::to_f32(buf[u], f);
#pragma unroll
                for (int q = 0; q < VN; ++q) ssq = fmaf(f[q], f[q], ssq);
              }
            }
          }
        }
      }
      if (want_norm(rownorm, ld, e)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
        if (lane == 0) {
          float* nd = norm_dst(rownorm, ld, g, row, i, e, rem);
          if (nd) *nd = sqrtf(ssq) * 1.001f;  // |x_row|_2, rounded up
        }
      }
    } else {
      T* dst = gather_dst(z, ld, g, row, i, e, rem);
      float ssq = 0.0f;
      for (int m = lane; m < g.M; m += 32) {
        const T v = t < 0 ? from_f<T>(0.0f) : x[static_cast<size_t>(t) * g.M + m];
        dst[m] = v;
        ssq = fmaf(to_f(v), to_f(v), ssq);
      }
      if (want_norm(rownorm, ld, e)) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
        if (lane == 0) {
          float* nd = norm_dst(rownorm, ld, g, row, i, e, rem);
          if (nd) *nd = sqrtf(ssq) * 1.001f;  // |x_row|_2, rounded up
        }
      }
    }
  }
  if (ld.all_peers) __threadfence_system();  // NVLink stores performed before the ready flags
}

// ------------------------------------------------------------------ decode
// y[t] = sum_j g[t,j] * Z[row(t,j)] (fp32 accumulate, j ascending); 0 when all dropped.
template <typename T, bool kVec>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    decode_kernel(SlotGeom g, const T* __restrict__ z, const int32_t* __restrict__ idxs,
                  const int32_t* __restrict__ locations, const double* __restrict__ gates,
                  T* __restrict__ y, FlagWait fw) {
  pdl_entry();
  if (fw.base != nullptr) {  // fused receive wait (the peers' combined rows)
    if (threadIdx.x < 32) wait_flags_warp(fw);
    __syncthreads();
  }
  const int lane = threadIdx.x % 32;
  const int ntok = g.blocks * g.T;
  if constexpr (kVec) {
    if (g.k == 1 && g.M / Vec<T>::N <= 32 * kUnroll) {
      // top-1 (W > 1 combine, NCCL transport): two tokens per warp with all their row loads in
      // flight before any math (the gather is latency-bound); y = g * row, dropped -> 0
      constexpr int VN = Vec<T>::N;
      const int nv = g.M / VN;
      const int S = gridDim.x * kWarpsPerCta;
      for (int t0 = blockIdx.x * kWarpsPerCta + threadIdx.x / 32; t0 < ntok; t0 += 2 * S) {
        const int tt[2] = {t0, t0 + S};
        const uint4* src[2];
        float gv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          src[h] = nullptr;
          gv[h] = 0.0f;
          if (tt[h] < ntok) {
            const int loc = locations[tt[h]];
            if (loc >= 0) {
              const int e = idxs[tt[h]];
              MOE_CHECK(loc < g.cap && e >= 0 && e < g.E, "decode: location / expert out of range");
              src[h] = reinterpret_cast<const uint4*>(z + slot_row(g, tt[h] / g.T, e, loc) * g.M);
              gv[h] = static_cast<float>(gates[tt[h]]);
            }
          }
        }
        uint4 buf[2][kUnroll];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = u * 32 + lane;
            if (src[h] && v < nv) buf[h][u] = ld_stream(src[h] + v);
          }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (tt[h] >= ntok) continue;
          uint4* dst = reinterpret_cast<uint4*>(y + static_cast<size_t>(tt[h]) * g.M);
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = u * 32 + lane;
            if (v >= nv) continue;
            float f[VN], acc[VN];
#pragma unroll
            for (int q = 0; q < VN; ++q) acc[q] = 0.0f;
            if (src[h]) {
              Vec<T>::to_f32(buf[h][u], f);
#pragma unroll
              for (int q = 0; q < VN; ++q) acc[q] = fmaf(gv[h], f[q], acc[q]);
            }
            dst[v] = Vec<T>::from_f32(acc);
          }
        }
      }
      return;
    }
  }
  for (int t = blockIdx.x * kWarpsPerCta + threadIdx.x / 32; t < ntok;
       t += gridDim.x * kWarpsPerCta) {
    const int b = t / g.T;
    if constexpr (kVec) {
      constexpr int VN = Vec<T>::N;
      const int nv = g.M / VN;
      uint4* dst = reinterpret_cast<uint4*>(y + static_cast<size_t>(t) * g.M);
      if (g.k == 2) {
        // top-2: both rows' loads in flight before any math; same j-ascending fma order
        const int2 loc = *reinterpret_cast<const int2*>(locations + static_cast<size_t>(t) * 2);
        const int2 ex = *reinterpret_cast<const int2*>(idxs + static_cast<size_t>(t) * 2);
        MOE_CHECK(loc.x < g.cap && loc.y < g.cap && (loc.x < 0 || (ex.x >= 0 && ex.x < g.E)) &&
                      (loc.y < 0 || (ex.y >= 0 && ex.y < g.E)), "decode: location / expert out of range");
        const double2 gt = *reinterpret_cast<const double2*>(gates + static_cast<size_t>(t) * 2);
        const uint4* s0 = loc.x >= 0 ? reinterpret_cast<const uint4*>(z + slot_row(g, b, ex.x, loc.x) * g.M) : nullptr;
        const uint4* s1 = loc.y >= 0 ? reinterpret_cast<const uint4*>(z + slot_row(g, b, ex.y, loc.y) * g.M) : nullptr;
        const float g0 = static_cast<float>(gt.x), g1 = static_cast<float>(gt.y);
        for (int v0 = 0; v0 < nv; v0 += 32 * kUnroll) {
          uint4 b0[kUnroll], b1[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nv && s0) b0[u] = ld_stream(s0 + v);
            if (v < nv && s1) b1[u] = ld_stream(s1 + v);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            float acc[VN], f[VN];
#pragma unroll
            for (int q = 0; q < VN; ++q) acc[q] = 0.0f;
            if (s0) {
              Vec<T>::to_f32(b0[u], f);
#pragma unroll
              for (int q = 0; q < VN; ++q) acc[q] = fmaf(g0, f[q], acc[q]);
            }
            if (s1) {
              Vec<T>::to_f32(b1[u], f);
#pragma unroll
              for (int q = 0; q < VN; ++q) acc[q] = fmaf(g1, f[q], acc[q]);
            }
            if (v < nv) dst[v] = Vec<T>::from_f32(acc);
          }
        }
        continue;
      }
      for (int v0 = 0; v0 < nv; v0 += 32 * kUnroll) {
        float acc[kUnroll][VN];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
          for (int q = 0; q < VN; ++q) acc[u][q] = 0.0f;
        for (int j = 0; j < g.k; ++j) {
          const int loc = locations[static_cast<size_t>(t) * g.k + j];
          if (loc < 0) continue;
          const int e = idxs[static_cast<size_t>(t) * g.k + j];
          const float gv = static_cast<float>(gates[static_cast<size_t>(t) * g.k + j]);
          const uint4* src = reinterpret_cast<const uint4*>(z + slot_row(g, b, e, loc) * g.M);
          uint4 buf[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nv) buf[u] = ld_stream(src + v);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            float f[VN];
            Vec<T>::to_f32(buf[u], f);
#pragma unroll
            for (int q = 0; q < VN; ++q) acc[u][q] = fmaf(gv, f[q], acc[u][q]);
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int v = v0 + u * 32 + lane;
          if (v < nv) dst[v] = Vec<T>::from_f32(acc[u]);
        }
      }
    } else {
      for (int m = lane; m < g.M; m += 32) {
        float acc = 0.0f;
        for (int j = 0; j < g.k; ++j) {
          const int loc = locations[static_cast<size_t>(t) * g.k + j];
          if (loc < 0) continue;
          const int e = idxs[static_cast<size_t>(t) * g.k + j];
          const float gv = static_cast<float>(gates[static_cast<size_t>(t) * g.k + j]);
          acc = fmaf(gv, to_f(z[slot_row(g, b, e, loc) * g.M + m]), acc);
        }
        y[static_cast<size_t>(t) * g.M + m] = from_f<T>(acc);
      }
    }
  }
}

// ------------------------------------------------------------------ top-1 combine, slot-major
// k = 1 (W > 1 after the combine, or unfused): walk the combined rows in slot order -- sequential
// reads -- and store each kept slot's row at its token (y = g * row; encode-backward: dx = row).
// Every token has at most one slot, so each output row is written exactly once: the same values
// as the token-major gather, whose random 2 KiB reads it replaces by fire-and-forget row stores.
// Dropped tokens' rows are zeroed by the same pass.
template <typename T, bool kScale>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    slot_scatter_kernel(SlotGeom g, const T* __restrict__ src, const int32_t* __restrict__ slot_token,
                        const float* __restrict__ slot_gate, T* __restrict__ out, FlagWait fw,
                        DropZero dzero) {
  pdl_entry();
  if (fw.base != nullptr) {  // fused receive wait (the peers' combined rows)
    if (threadIdx.x < 32) wait_flags_warp(fw);
    __syncthreads();
  }
  zero_dropped_rows(dzero);
  constexpr int VN = Vec<T>::N;
  const int nv = g.M / VN;
  const int lane = threadIdx.x % 32;
  const size_t rows = static_cast<size_t>(g.blocks) * g.degree * g.E * g.cc;
  const size_t per_block = static_cast<size_t>(g.degree) * g.E * g.cc;
  for (size_t row = static_cast<size_t>(blockIdx.x) * kWarpsPerCta + threadIdx.x / 32; row < rows;
       row += static_cast<size_t>(gridDim.x) * kWarpsPerCta) {
    const int b = static_cast<int>(row / per_block);
    const int rem = static_cast<int>(row % per_block);
    const int i = rem / (g.E * g.cc);
    const int e = (rem / g.cc) % g.E;
    const int c = i * g.cc + rem % g.cc;
    if (c >= g.cap) continue;
    const size_t sl = static_cast<size_t>(b * g.E + e) * g.cap + c;
    const int t = slot_token[sl];
    if (t < 0) continue;
    MOE_CHECK(t >= b * g.T && t < (b + 1) * g.T, "slot scatter: slot token outside its block");
    const float gv = kScale ? slot_gate[sl] : 1.0f;
    const uint4* s4 = reinterpret_cast<const uint4*>(src + row * g.M);
    uint4* d4 = reinterpret_cast<uint4*>(out + static_cast<size_t>(t) * g.M);
    for (int v0 = 0; v0 < nv; v0 += 32 * kUnroll) {
      uint4 buf[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v < nv) buf[u] = ld_stream(s4 + v);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int v = v0 + u * 32 + lane;
        if (v >= nv) continue;
        if constexpr (kScale) {
          float f[VN], acc[VN];
          Vec<T>::to_f32(buf[u], f);
#pragma unroll
          for (int q = 0; q < VN; ++q) acc[q] = fmaf(gv, f[q], 0.0f);
          d4[v] = Vec<T>::from_f32(acc);
        } else {
          d4[v] = buf[u];
        }
      }
    }
  }
}

// ------------------------------------------------------------------ decode backward
// dZ[row] = g_slot * dy[t_slot] or 0 (slot-major; each kept slot has exactly one (t, j)).
template <typename T, bool kVec>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    decode_bwd_kernel(SlotGeom g, const T* __restrict__ dy, const int32_t* __restrict__ slot_token,
                      const float* __restrict__ slot_gate, T* __restrict__ dz, DropZero dzero,
                      LocalDest ld) {
  pdl_entry();
  zero_dropped_rows(dzero);
  wait_peers_released(ld);
  const int lane = threadIdx.x % 32;
  const size_t rows = static_cast<size_t>(g.blocks) * g.degree * g.E * g.cc;
  const size_t per_block = static_cast<size_t>(g.degree) * g.E * g.cc;
  for (size_t row = static_cast<size_t>(blockIdx.x) * kWarpsPerCta + threadIdx.x / 32; row < rows;
       row += static_cast<size_t>(gridDim.x) * kWarpsPerCta) {
    const int b = static_cast<int>(row / per_block);
    const int rem = static_cast<int>(row % per_block);
    const int i = rem / (g.E * g.cc);
    const int e = (rem / g.cc) % g.E;
    const int c = i * g.cc + rem % g.cc;
    int t = -1;
    float gv = 0.0f;
    if (c < g.cap) {
      const size_t s = static_cast<size_t>(b * g.E + e) * g.cap + c;
      t = slot_token[s];
      gv = slot_gate[s];
    }
    MOE_CHECK(t == -1 || (t >= b * g.T && t < (b + 1) * g.T), "decode_bwd: slot token outside its block");
    if constexpr (kVec) {
      constexpr int VN = Vec<T>::N;
      const int nv = g.M / VN;
      uint4* dst = reinterpret_cast<uint4*>(gather_dst(dz, ld, g, row, i, e, rem));
      if (t < 0) {
        for (int v = lane; v < nv; v += 32) dst[v] = make_uint4(0, 0, 0, 0);
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(dy + static_cast<size_t>(t) * g.M);
        for (int v0 = 0; v0 < nv; v0 += 32 * kUnroll) {
          uint4 buf[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nv) buf[u] = ld_stream(src + v);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nv) {
              float f[VN];
              Vec<T>::to_f32(buf[u], f);
#pragma unroll
              for (int q = 0; q < VN; ++q) f[q] *= gv;
              dst[v] = Vec<T>::from_f32(f);
            }
          }
        }
      }
    } else {
      T* dst = gather_dst(dz, ld, g, row, i, e, rem);
      for (int m = lane; m < g.M; m += 32)
        dst[m] = t < 0 ? from_f<T>(0.0f) : from_f<T>(gv * to_f(dy[static_cast<size_t>(t) * g.M + m]));
    }
  }
  if (ld.all_peers) __threadfence_system();  // NVLink stores performed before the ready flags
}

// d_gates[t, j] = <Z[row], dy[t]> in fp64 (the layer itself discards it, moe_layer.cpp:268-270).
template <typename T>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    decode_bwd_gates_kernel(SlotGeom g, const T* __restrict__ z, const T* __restrict__ dy,
                            const int32_t* __restrict__ idxs, const int32_t* __restrict__ locations,
                            double* __restrict__ dgates) {
  pdl_entry();
  const int lane = threadIdx.x % 32;
  const int n = g.blocks * g.T * g.k;
  for (int f = blockIdx.x * kWarpsPerCta + threadIdx.x / 32; f < n; f += gridDim.x * kWarpsPerCta) {
    const int t = f / g.k;
    const int loc = locations[f];
    double s = 0.0;
    if (loc >= 0) {
      const T* zr = z + slot_row(g, t / g.T, idxs[f], loc) * g.M;
      const T* dr = dy + static_cast<size_t>(t) * g.M;
      for (int m = lane; m < g.M; m += 32)
        s += static_cast<double>(to_f(zr[m])) * static_cast<double>(to_f(dr[m]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    }
    if (lane == 0) dgates[f] = s;
  }
}

// ------------------------------------------------------------------ encode backward
// dx[t] = sum_j dZ[row(t,j)] over kept j (fp32 accumulate, j ascending).
template <typename T, bool kVec>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
    encode_bwd_kernel(SlotGeom g, const T* __restrict__ dz, const int32_t* __restrict__ idxs,
                      const int32_t* __restrict__ locations, T* __restrict__ dx, FlagWait fw) {
  pdl_entry();
  if (fw.base != nullptr) {  // fused receive wait (the peers' combined dX rows)
    if (threadIdx.x < 32) wait_flags_warp(fw);
    __syncthreads();
  }
  const int lane = threadIdx.x % 32;
  const int ntok = g.blocks * g.T;
  if constexpr (kVec) {
    if (g.k == 1 && g.M / Vec<T>::N <= 32 * kUnroll) {
      // top-1: two tokens per warp, all row loads in flight; dx = row, dropped -> 0
      const int nv = g.M / Vec<T>::N;
      const int S = gridDim.x * kWarpsPerCta;
      for (int t0 = blockIdx.x * kWarpsPerCta + threadIdx.x / 32; t0 < ntok; t0 += 2 * S) {
        const int tt[2] = {t0, t0 + S};
        const uint4* src[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          src[h] = nullptr;
          if (tt[h] < ntok) {
            const int loc = locations[tt[h]];
            if (loc >= 0) {
              const int e = idxs[tt[h]];
              MOE_CHECK(loc < g.cap && e >= 0 && e < g.E, "encode_bwd: location / expert out of range");
              src[h] = reinterpret_cast<const uint4*>(dz + slot_row(g, tt[h] / g.T, e, loc) * g.M);
            }
          }
        }
        uint4 buf[2][kUnroll];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = u * 32 + lane;
            if (src[h] && v < nv) buf[h][u] = ld_stream(src[h] + v);
          }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (tt[h] >= ntok) continue;
          uint4* dst = reinterpret_cast<uint4*>(dx + static_cast<size_t>(tt[h]) * g.M);
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = u * 32 + lane;
            if (v < nv) dst[v] = src[h] ? buf[h][u] : make_uint4(0u, 0u, 0u, 0u);
          }
        }
      }
      return;
    }
  }
  for (int t = blockIdx.x * kWarpsPerCta + threadIdx.x / 32; t < ntok;
       t += gridDim.x * kWarpsPerCta) {
    const int b = t / g.T;
    if constexpr (kVec) {
      constexpr int VN = Vec<T>::N;
      const int nv = g.M / VN;
      uint4* dst = reinterpret_cast<uint4*>(dx + static_cast<size_t>(t) * g.M);
      if (g.k == 2) {
        // top-2: both rows' loads in flight before any math; same j-ascending sum order
        const int2 loc = *reinterpret_cast<const int2*>(locations + static_cast<size_t>(t) * 2);
        const int2 ex = *reinterpret_cast<const int2*>(idxs + static_cast<size_t>(t) * 2);
        MOE_CHECK(loc.x < g.cap && loc.y < g.cap && (loc.x < 0 || (ex.x >= 0 && ex.x < g.E)) &&
                      (loc.y < 0 || (ex.y >= 0 && ex.y < g.E)), "encode_bwd: location / expert out of range");
        const uint4* s0 = loc.x >= 0 ? reinterpret_cast<const uint4*>(dz + slot_row(g, b, ex.x, loc.x) * g.M) : nullptr;
        const uint4* s1 = loc.y >= 0 ? reinterpret_cast<const uint4*>(dz + slot_row(g, b, ex.y, loc.y) * g.M) : nullptr;
        for (int v0 = 0; v0 < nv; v0 += 32 * kUnroll) {
          uint4 b0[kUnroll], b1[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nv && s0) b0[u] = ld_stream(s0 + v);
            if (v < nv && s1) b1[u] = ld_stream(s1 + v);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            float acc[VN], f[VN];
#pragma unroll
            for (int q = 0; q < VN; ++q) acc[q] = 0.0f;
            if (s0) {
              Vec<T>::to_f32(b0[u], f);
#pragma unroll
              for (int q = 0; q < VN; ++q) acc[q] += f[q];
            }
            if (s1) {
              Vec<T>::to_f32(b1[u], f);
#pragma unroll
              for (int q = 0; q < VN; ++q) acc[q] += f[q];
            }
            if (v < nv) dst[v] = Vec<T>::from_f32(acc);
          }
        }
        continue;
      }
      for (int v0 = 0; v0 < nv; v0 += 32 * kUnroll) {
        float acc[kUnroll][VN];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
#pragma unroll
          for (int q = 0; q < VN; ++q) acc[u][q] = 0.0f;
        for (int j = 0; j < g.k; ++j) {
          const int loc = locations[static_cast<size_t>(t) * g.k + j];
          if (loc < 0) continue;
          const int e = idxs[static_cast<size_t>(t) * g.k + j];
          const uint4* src = reinterpret_cast<const uint4*>(dz + slot_row(g, b, e, loc) * g.M);
          uint4 buf[kUnroll];
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            const int v = v0 + u * 32 + lane;
            if (v < nv) buf[u] = ld_stream(src + v);
          }
#pragma unroll
          for (int u = 0; u < kUnroll; ++u) {
            float f[VN];
            Vec<T>::to_f32(buf[u], f);
#pragma unroll
            for (int q = 0; q < VN; ++q) acc[u][q] += f[q];
          }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int v = v0 + u * 32 + lane;
          if (v < nv) dst[v] = Vec<T>::from_f32(acc[u]);
        }
      }
    } else {
      for (int m = lane; m < g.M; m += 32) {
        float acc = 0.0f;
        for (int j = 0; j < g.k; ++j) {
          const int loc = locations[static_cast<size_t>(t) * g.k + j];
          if (loc < 0) continue;
          const int e = idxs[static_cast<size_t>(t) * g.k + j];
          acc += to_f(dz[slot_row(g, b, e, loc) * g.M + m]);
        }
        dx[static_cast<size_t>(t) * g.M + m] = from_f<T>(acc);
      }
    }
  }
}

int grid_for(size_t warps_needed) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const size_t ctas = (warps_needed + kWarpsPerCta - 1) / kWarpsPerCta;
  const size_t cap = static_cast<size_t>(sms) * 8;  // 8 resident CTAs of 8 warps per SM
  return static_cast<int>(ctas < cap ? (ctas > 0 ? ctas : 1) : cap);
}

bool vec_ok(int dtype, int M) { return (M * (dtype == 1 ? 4 : 2)) % 16 == 0; }

}  // namespace

int encode_device(const SlotGeom& g, int dtype, const void* x, const int32_t* slot_token, void* z,
                  cudaStream_t st, float* rownorm, const DropZero& dzero, unsigned int* reset,
                  const LocalDest& local) {
  if (local.recv && (g.blocks != 1 || local.dE < 1 || local.W * local.dE != g.E)) return -1;
  if (dzero.out && dzero.row_bytes % 16 != 0) return -1;
  const size_t rows = static_cast<size_t>(g.blocks) * g.degree * g.E * g.cc;
  const int grid = grid_for(rows);
  const bool v = vec_ok(dtype, g.M);
  if (dtype == 1) {
    if (v) launch_k(encode_kernel<float, true>, grid, 256, 0, st, g, static_cast<const float*>(x), slot_token, static_cast<float*>(z), rownorm, dzero, reset, local);
    else launch_k(encode_kernel<float, false>, grid, 256, 0, st, g, static_cast<const float*>(x), slot_token, static_cast<float*>(z), rownorm, dzero, reset, local);
  } else {
    using B = __nv_bfloat16;
    if (v) launch_k(encode_kernel<B, true>, grid, 256, 0, st, g, static_cast<const B*>(x), slot_token, static_cast<B*>(z), rownorm, dzero, reset, local);
    else launch_k(encode_kernel<B, false>, grid, 256, 0, st, g, static_cast<const B*>(x), slot_token, static_cast<B*>(z), rownorm, dzero, reset, local);
  }
  return launch_status();
}

int decode_device(const SlotGeom& g, int dtype, const void* z, const int32_t* idxs,
                  const int32_t* locations, const double* gates, void* y, cudaStream_t st,
                  const FlagWait* wait) {
  const FlagWait fw = wait ? *wait : FlagWait{};
  const int grid = grid_for(static_cast<size_t>(g.blocks) * g.T);
  const bool v = vec_ok(dtype, g.M);
  if (dtype == 1) {
    if (v) launch_k(decode_kernel<float, true>, grid, 256, 0, st, g, static_cast<const float*>(z), idxs, locations, gates, static_cast<float*>(y), fw);
    else launch_k(decode_kernel<float, false>, grid, 256, 0, st, g, static_cast<const float*>(z), idxs, locations, gates, static_cast<float*>(y), fw);
  } else {
    using B = __nv_bfloat16;
    if (v) launch_k(decode_kernel<B, true>, grid, 256, 0, st, g, static_cast<const B*>(z), idxs, locations, gates, static_cast<B*>(y), fw);
    else launch_k(decode_kernel<B, false>, grid, 256, 0, st, g, static_cast<const B*>(z), idxs, locations, gates, static_cast<B*>(y), fw);
  }
  return launch_status();
}

int decode_backward_device(const SlotGeom& g, int dtype, const void* dy,
                           const int32_t* slot_token, const float* slot_gate, void* dz,
                           cudaStream_t st, const DropZero& dzero, const LocalDest& local) {
  if (local.recv && (g.blocks != 1 || local.dE < 1 || local.W * local.dE != g.E)) return -1;
  if (dzero.out && dzero.row_bytes % 16 != 0) return -1;
  const size_t rows = static_cast<size_t>(g.blocks) * g.degree * g.E * g.cc;
  const int grid = grid_for(rows);
  const bool v = vec_ok(dtype, g.M);
  if (dtype == 1) {
    if (v) launch_k(decode_bwd_kernel<float, true>, grid, 256, 0, st, g, static_cast<const float*>(dy), slot_token, slot_gate, static_cast<float*>(dz), dzero, local);
    else launch_k(decode_bwd_kernel<float, false>, grid, 256, 0, st, g, static_cast<const float*>(dy), slot_token, slot_gate, static_cast<float*>(dz), dzero, local);
  } else {
    using B = __nv_bfloat16;
    if (v) launch_k(decode_bwd_kernel<B, true>, grid, 256, 0, st, g, static_cast<const B*>(dy), slot_token, slot_gate, static_cast<B*>(dz), dzero, local);
    else launch_k(decode_bwd_kernel<B, false>, grid, 256, 0, st, g, static_cast<const B*>(dy), slot_token, slot_gate, static_cast<B*>(dz), dzero, local);
  }
  return launch_status();
}

int decode_backward_gates_device(const SlotGeom& g, int dtype, const void* z, const void* dy,
                                 const int32_t* idxs, const int32_t* locations, double* dgates,
                                 cudaStream_t st) {
  const int grid = grid_for(static_cast<size_t>(g.blocks) * g.T * g.k);
  if (dtype == 1)
    launch_k(decode_bwd_gates_kernel<float>, grid, 256, 0, st, g, static_cast<const float*>(z), static_cast<const float*>(dy), idxs, locations, dgates);
  else
    launch_k(decode_bwd_gates_kernel<__nv_bfloat16>, grid, 256, 0, st, g, static_cast<const __nv_bfloat16*>(z), static_cast<const __nv_bfloat16*>(dy), idxs, locations, dgates);
  return launch_status();
}

int encode_backward_device(const SlotGeom& g, int dtype, const void* dz, const int32_t* idxs,
                           const int32_t* locations, void* dx, cudaStream_t st,
                           const FlagWait* wait) {
  const FlagWait fw = wait ? *wait : FlagWait{};
  const int grid = grid_for(static_cast<size_t>(g.blocks) * g.T);
  const bool v = vec_ok(dtype, g.M);
  if (dtype == 1) {
    if (v) launch_k(encode_bwd_kernel<float, true>, grid, 256, 0, st, g, static_cast<const float*>(dz), idxs, locations, static_cast<float*>(dx), fw);
    else launch_k(encode_bwd_kernel<float, false>, grid, 256, 0, st, g, static_cast<const float*>(dz), idxs, locations, static_cast<float*>(dx), fw);
  } else {
    using B = __nv_bfloat16;
    if (v) launch_k(encode_bwd_kernel<B, true>, grid, 256, 0, st, g, static_cast<const B*>(dz), idxs, locations, static_cast<B*>(dx), fw);
    else launch_k(encode_bwd_kernel<B, false>, grid, 256, 0, st, g, static_cast<const B*>(dz), idxs, locations, static_cast<B*>(dx), fw);
  }
  return launch_status();
}

namespace {
__global__ void build_slots_kernel(int n, int T, int k, int E, int cap,
                                   const int32_t* __restrict__ idxs,
                                   const int32_t* __restrict__ locations,
                                   const double* __restrict__ gates, int32_t* __restrict__ slot_token,
                                   float* __restrict__ slot_gate) {
  pdl_entry();
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x) {
    const int loc = locations[f];
    if (loc < 0) continue;
    const int t = f / k;
    const size_t s = static_cast<size_t>((t / T) * E + idxs[f]) * cap + loc;
    slot_token[s] = t;
    slot_gate[s] = gates ? static_cast<float>(gates[f]) : 0.0f;
  }
}
}  // namespace

// ------------------------------------------------------------------ sharded P2 combine sum
namespace {
// out[b][o] = sum_q part[b][q][o] (combine_sharded_p2, moe_layer.cpp:80-108: the source sums the
// s shards' partial rows of each expert, q ascending, fp32 accumulate). 16-byte vectors.
template <typename T>
__global__ void __launch_bounds__(256) shard_sum_kernel(const T* __restrict__ part, T* __restrict__ out,
                                                        int64_t nblk, int s, int64_t blk_vecs) {
  pdl_entry();
  constexpr int VN = Vec<T>::N;
  const int64_t n = nblk * blk_vecs;
  const uint4* p = reinterpret_cast<const uint4*>(part);
  uint4* o = reinterpret_cast<uint4*>(out);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / blk_vecs, v = i - b * blk_vecs;
    float acc[VN];
#pragma unroll
    for (int j = 0; j < VN; ++j) acc[j] = 0.0f;
    for (int q = 0; q < s; ++q) {
      float f[VN];
      Vec<T>::to_f32(ld_stream(p + (b * s + q) * blk_vecs + v), f);
#pragma unroll
      for (int j = 0; j < VN; ++j) acc[j] += f[j];
    }
    o[i] = Vec<T>::from_f32(acc);
  }
}
template <typename T>
__global__ void __launch_bounds__(256) shard_sum_scalar_kernel(const T* __restrict__ part, T* __restrict__ out,
                                                               int64_t nblk, int s, int64_t blk) {
  pdl_entry();
  const int64_t n = nblk * blk;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / blk, e = i - b * blk;
    float acc = 0.0f;
    for (int q = 0; q < s; ++q) acc += to_f(part[(b * s + q) * blk + e]);
    out[i] = from_f<T>(acc);
  }
}
}  // namespace

int shard_sum_device(const void* part, void* out, int64_t nblk, int s, int64_t blk, int dtype,
                     cudaStream_t st) {
  if (nblk < 0 || s < 1 || blk < 0) return -1;
  const int esz = dtype == 1 ? 4 : 2;
  const bool vec = (blk * esz) % 16 == 0;
  const int64_t work = vec ? nblk * (blk * esz / 16) : nblk * blk;
  const int64_t want = (work + 255) / 256;
  const int grid = static_cast<int>(want < 148 * 16 ? (want > 0 ? want : 1) : 148 * 16);
  if (dtype == 1) {
    if (vec) launch_k(shard_sum_kernel<float>, grid, 256, 0, st, static_cast<const float*>(part), static_cast<float*>(out), nblk, s, blk / 4);
    else launch_k(shard_sum_scalar_kernel<float>, grid, 256, 0, st, static_cast<const float*>(part), static_cast<float*>(out), nblk, s, blk);
  } else {
    using B = __nv_bfloat16;
    if (vec) launch_k(shard_sum_kernel<B>, grid, 256, 0, st, static_cast<const B*>(part), static_cast<B*>(out), nblk, s, blk / 8);
    else launch_k(shard_sum_scalar_kernel<B>, grid, 256, 0, st, static_cast<const B*>(part), static_cast<B*>(out), nblk, s, blk);
  }
  return launch_status();
}

// Slot tables (slot -> token, slot -> gate) from an explicit routing plan (DispatchPlan).
int build_slots_device(int blocks, int T, int k, int E, int cap, const int32_t* idxs,
                       const int32_t* locations, const double* gates, int32_t* slot_token,
                       float* slot_gate, cudaStream_t st) {
  const size_t ns = static_cast<size_t>(blocks) * E * cap;
  if (cudaMemsetAsync(slot_token, 0xFF, ns * sizeof(int32_t), st) != cudaSuccess) return -2;
  if (cudaMemsetAsync(slot_gate, 0, ns * sizeof(float), st) != cudaSuccess) return -2;
  const int n = blocks * T * k;
  const int grid = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
  launch_k(build_slots_kernel, grid > 0 ? grid : 1, 256, 0, st, n, T, k, E, cap, idxs, locations, gates,
                                                         slot_token, slot_gate);
  return launch_status();
}

int slot_scatter_device(const SlotGeom& g, int dtype, const void* src, const int32_t* slot_token,
                        const float* slot_gate, void* out, const DropZero& dzero, cudaStream_t st,
                        const FlagWait* wait) {
  if (g.k != 1 || !vec_ok(dtype, g.M)) return -1;
  const FlagWait fw = wait ? *wait : FlagWait{};
  const int grid = grid_for(static_cast<size_t>(g.blocks) * g.degree * g.E * g.cc);
  using B = __nv_bfloat16;
  const bool scale = slot_gate != nullptr;
  if (dtype == 1) {
    if (scale) launch_k(slot_scatter_kernel<float, true>, grid, 256, 0, st, g, static_cast<const float*>(src), slot_token, slot_gate, static_cast<float*>(out), fw, dzero);
    else launch_k(slot_scatter_kernel<float, false>, grid, 256, 0, st, g, static_cast<const float*>(src), slot_token, slot_gate, static_cast<float*>(out), fw, dzero);
  } else {
    if (scale) launch_k(slot_scatter_kernel<B, true>, grid, 256, 0, st, g, static_cast<const B*>(src), slot_token, slot_gate, static_cast<B*>(out), fw, dzero);
    else launch_k(slot_scatter_kernel<B, false>, grid, 256, 0, st, g, static_cast<const B*>(src), slot_token, slot_gate, static_cast<B*>(out), fw, dzero);
  }
  return launch_status();
}

}  // namespace moe
