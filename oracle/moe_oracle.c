/*
 * moe_oracle.c -- fp64 CPU restatement of the reference MoE layer (TEST INFRASTRUCTURE ONLY;
 * see moe_oracle.h). Each function cites the reference file:line it restates. Parallelised with
 * OpenMP so it doubles as the CPU baseline timed on the GPU box's host cores.
 */
#include "moe_oracle.h"

#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ core.cpp:66-91 */
uint64_t orc_next_u64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

double orc_uniform(uint64_t* state) { return (double)(orc_next_u64(state) >> 11) * 0x1.0p-53; }

void orc_fill_uniform(uint64_t seed, uint64_t offset, int64_t n, double lo, double hi, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t s = seed + (offset + (uint64_t)i) * 0x9e3779b97f4a7c15ULL;
    out[i] = lo + (hi - lo) * orc_uniform(&s);
  }
}

/* ------------------------------------------------------------------ core.cpp:28-64 */
int64_t orc_expert_capacity(int64_t k, double f, int64_t tokens, int64_t experts) {
  if (k < 1 || tokens < 1 || experts < 1 || !(f > 0.0)) return -1;
  double q = (double)k * f * (double)tokens / (double)experts;
  int64_t cap = (int64_t)ceil(q - 1e-9);
  return cap < 1 ? 1 : cap;
}

int64_t orc_resolve_capacity(int32_t kind, double factor, const int64_t* demand, int64_t E,
                             int64_t k, int64_t T) {
  int64_t mx = 1;
  for (int64_t e = 0; e < E; ++e)
    if (demand[e] > mx) mx = demand[e];
  if (kind == 0) return orc_expert_capacity(k, factor, T, E);
  if (kind == 1) return mx;
  int64_t b = orc_expert_capacity(k, factor, T, E);
  return mx < b ? mx : b;
}

double orc_capacity_to_factor(int64_t cap, int64_t E, int64_t k, int64_t T) {
  return (double)cap * (double)E / ((double)k * (double)T);
}

/* ------------------------------------------------------------------ gating.cpp:19-35 */
void orc_gate_linear(const double* x, const double* wg, int64_t T, int64_t M, int64_t E,
                     double* probs) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    double* row = probs + t * E;
    for (int64_t e = 0; e < E; ++e) row[e] = 0.0;
    for (int64_t m = 0; m < M; ++m) {
      const double xv = x[t * M + m];
      const double* w = wg + m * E;
      for (int64_t e = 0; e < E; ++e) row[e] += xv * w[e];
    }
    double mx = row[0];
    for (int64_t e = 1; e < E; ++e)
      if (row[e] > mx) mx = row[e];
    double s = 0.0;
    for (int64_t e = 0; e < E; ++e) {
      row[e] = exp(row[e] - mx);
      s += row[e];
    }
    for (int64_t e = 0; e < E; ++e) row[e] /= s;
  }
}

/* gating.cpp:37-56 (gate_cosine): proj = x . P (T, D); logits[t][e] = <proj_t, C_e> /
 * (|proj_t| |C_e| max(tau, 0.01)); row softmax. Returns -1 on a zero-norm projected token or
 * expert row (the reference's std::invalid_argument), 0 otherwise. */
int32_t orc_gate_cosine(const double* x, const double* proj_w, const double* experts,
                        double temperature, int64_t T, int64_t M, int64_t E, int64_t D,
                        double* probs) {
  const double tau = temperature > 0.01 ? temperature : 0.01;
  double* en = (double*)malloc(sizeof(double) * (size_t)E);
  for (int64_t e = 0; e < E; ++e) {
    double s = 0.0;
    for (int64_t d = 0; d < D; ++d) s += experts[e * D + d] * experts[e * D + d];
    en[e] = sqrt(s);
    if (en[e] == 0.0) {
      free(en);
      return -1;
    }
  }
  int32_t bad = 0;
#pragma omp parallel
  {
    double* pr = (double*)malloc(sizeof(double) * (size_t)D);
#pragma omp for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
      for (int64_t d = 0; d < D; ++d) pr[d] = 0.0;
      for (int64_t m = 0; m < M; ++m) {
        const double xv = x[t * M + m];
        const double* w = proj_w + m * D;
        for (int64_t d = 0; d < D; ++d) pr[d] += xv * w[d];
      }
      double s = 0.0;
      for (int64_t d = 0; d < D; ++d) s += pr[d] * pr[d];
      const double tn = sqrt(s);
      if (tn == 0.0) {
#pragma omp atomic write
        bad = 1;
        continue;
      }
      double* row = probs + t * E;
      for (int64_t e = 0; e < E; ++e) {
        double dot = 0.0;
        for (int64_t d = 0; d < D; ++d) dot += pr[d] * experts[e * D + d];
        row[e] = dot / (tn * en[e] * tau);
      }
      double mx = row[0];
      for (int64_t e = 1; e < E; ++e)
        if (row[e] > mx) mx = row[e];
      double z = 0.0;
      for (int64_t e = 0; e < E; ++e) {
        row[e] = exp(row[e] - mx);
        z += row[e];
      }
      for (int64_t e = 0; e < E; ++e) row[e] /= z;
    }
    free(pr);
  }
  free(en);
  return bad ? -1 : 0;
}

/* gating.cpp:58-78: stable sort by (prob desc, id asc) == repeated selection with that order. */
void orc_topk_select(const double* probs, int64_t T, int64_t E, int64_t k, int64_t* idxs,
                     double* gates) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    const double* p = probs + t * E;
    unsigned char taken[1024];
    memset(taken, 0, (size_t)(E < 1024 ? E : 1024));
    for (int64_t j = 0; j < k; ++j) {
      int64_t bi = -1;
      for (int64_t e = 0; e < E; ++e) {
        if (taken[e]) continue;
        if (bi < 0 || p[e] > p[bi]) bi = e; /* strict: ties keep the lower index */
      }
      taken[bi] = 1;
      idxs[t * k + j] = bi;
      gates[t * k + j] = p[bi];
    }
  }
}

/* gating.cpp:80-112 */
static const double* g_key;
static int cmp_bpr(const void* a, const void* b) {
  const int64_t ia = *(const int64_t*)a, ib = *(const int64_t*)b;
  if (g_key[ia] != g_key[ib]) return g_key[ia] > g_key[ib] ? -1 : 1;
  return ia < ib ? -1 : (ia > ib);
}

void orc_assign_locations(const int64_t* idxs, const double* gates, int64_t T, int64_t k,
                          int64_t cap, int32_t bpr, int64_t* locations) {
  int64_t experts = 0;
  for (int64_t i = 0; i < T * k; ++i)
    if (idxs[i] + 1 > experts) experts = idxs[i] + 1;
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T > 0 ? T : 1));
  for (int64_t t = 0; t < T; ++t) order[t] = t;
  if (bpr) {
    double* key = (double*)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1));
    for (int64_t t = 0; t < T; ++t) {
      double m = gates[t * k];
      for (int64_t j = 1; j < k; ++j)
        if (gates[t * k + j] > m) m = gates[t * k + j];
      key[t] = m;
    }
    g_key = key; /* (key desc, token asc) is a total order -> qsort is deterministic */
    qsort(order, (size_t)T, sizeof(int64_t), cmp_bpr);
    free(key);
  }
  int64_t* next = (int64_t*)calloc((size_t)(experts > 0 ? experts : 1), sizeof(int64_t));
  for (int64_t i = 0; i < T; ++i) {
    const int64_t t = order[i];
    for (int64_t j = 0; j < k; ++j) {
      const int64_t e = idxs[t * k + j];
      locations[t * k + j] = next[e] < cap ? next[e]++ : -1;
    }
  }
  free(next);
  free(order);
}

int64_t orc_drop_count(const int64_t* locations, int64_t n) {
  int64_t d = 0;
  for (int64_t i = 0; i < n; ++i) d += locations[i] < 0;
  return d;
}

/* gating.cpp:134-162 */
int64_t orc_run_gating_blocked(const double* probs, int64_t blocks, int64_t T, int64_t E,
                               int64_t k, int32_t cap_kind, double factor, int32_t bpr,
                               int64_t* idxs, double* gates, int64_t* locations) {
  orc_topk_select(probs, blocks * T, E, k, idxs, gates);
  int64_t* demand = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  int64_t* bd = (int64_t*)malloc(sizeof(int64_t) * (size_t)E);
  for (int64_t b = 0; b < blocks; ++b) {
    memset(bd, 0, sizeof(int64_t) * (size_t)E);
    for (int64_t i = b * T * k; i < (b + 1) * T * k; ++i) ++bd[idxs[i]];
    for (int64_t e = 0; e < E; ++e)
      if (bd[e] > demand[e]) demand[e] = bd[e];
  }
  const int64_t cap = orc_resolve_capacity(cap_kind, factor, demand, E, k, T);
  for (int64_t b = 0; b < blocks; ++b)
    orc_assign_locations(idxs + b * T * k, gates + b * T * k, T, k, cap, bpr, locations + b * T * k);
  free(bd);
  free(demand);
  return cap;
}

/* ------------------------------------------------------------------ dispatch.cpp */
void orc_encode(const double* x, int64_t blocks, int64_t T, int64_t M, int64_t E, int64_t k,
                int64_t cap, const int64_t* idxs, const int64_t* locations, double* z) {
  memset(z, 0, sizeof(double) * (size_t)(blocks * E * cap * M));
  for (int64_t t = 0; t < blocks * T; ++t) {
    const int64_t b = t / T;
    for (int64_t j = 0; j < k; ++j) {
      const int64_t loc = locations[t * k + j];
      if (loc < 0) continue;
      double* dst = z + ((b * E + idxs[t * k + j]) * cap + loc) * M;
      memcpy(dst, x + t * M, sizeof(double) * (size_t)M);
    }
  }
}

void orc_decode(const double* z, int64_t blocks, int64_t T, int64_t M, int64_t E, int64_t k,
                int64_t cap, const int64_t* idxs, const int64_t* locations, const double* gates,
                double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < blocks * T; ++t) {
    const int64_t b = t / T;
    double* yr = y + t * M;
    for (int64_t m = 0; m < M; ++m) yr[m] = 0.0;
    for (int64_t j = 0; j < k; ++j) {
      const int64_t loc = locations[t * k + j];
      if (loc < 0) continue;
      const double g = gates[t * k + j];
      const double* zr = z + ((b * E + idxs[t * k + j]) * cap + loc) * M;
      for (int64_t m = 0; m < M; ++m) yr[m] += g * zr[m];
    }
  }
}

void orc_decode_backward(const double* dy, const double* z, int64_t blocks, int64_t T, int64_t M,
                         int64_t E, int64_t k, int64_t cap, const int64_t* idxs,
                         const int64_t* locations, const double* gates, double* dz,
                         double* dgates) {
  memset(dz, 0, sizeof(double) * (size_t)(blocks * E * cap * M));
  for (int64_t t = 0; t < blocks * T; ++t) {
    const int64_t b = t / T;
    for (int64_t j = 0; j < k; ++j) {
      const int64_t loc = locations[t * k + j];
      if (dgates) dgates[t * k + j] = 0.0;
      if (loc < 0) continue;
      const double g = gates[t * k + j];
      const size_t off = (size_t)(((b * E + idxs[t * k + j]) * cap + loc) * M);
      double dot = 0.0;
      for (int64_t m = 0; m < M; ++m) {
        dz[off + m] += g * dy[t * M + m];
        if (z) dot += z[off + m] * dy[t * M + m];
      }
      if (dgates) dgates[t * k + j] = dot;
    }
  }
}

void orc_encode_backward(const double* dz, int64_t blocks, int64_t T, int64_t M, int64_t E,
                         int64_t k, int64_t cap, const int64_t* idxs, const int64_t* locations,
                         double* dx) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < blocks * T; ++t) {
    const int64_t b = t / T;
    double* xr = dx + t * M;
    for (int64_t m = 0; m < M; ++m) xr[m] = 0.0;
    for (int64_t j = 0; j < k; ++j) {
      const int64_t loc = locations[t * k + j];
      if (loc < 0) continue;
      const double* zr = dz + ((b * E + idxs[t * k + j]) * cap + loc) * M;
      for (int64_t m = 0; m < M; ++m) xr[m] += zr[m];
    }
  }
}

void orc_encode_dense(const double* x, int64_t T, int64_t M, int64_t E, int64_t k, int64_t cap,
                      const int64_t* idxs, const int64_t* locations, double* z) {
  double* mask = (double*)calloc((size_t)(T * E * cap), sizeof(double));
  for (int64_t t = 0; t < T; ++t)
    for (int64_t j = 0; j < k; ++j)
      if (locations[t * k + j] >= 0) mask[(t * E + idxs[t * k + j]) * cap + locations[t * k + j]] = 1.0;
  memset(z, 0, sizeof(double) * (size_t)(E * cap * M));
  for (int64_t e = 0; e < E; ++e)
    for (int64_t c = 0; c < cap; ++c)
      for (int64_t t = 0; t < T; ++t) {
        const double mk = mask[(t * E + e) * cap + c];
        for (int64_t d = 0; d < M; ++d) z[(e * cap + c) * M + d] += mk * x[t * M + d];
      }
  free(mask);
}

void orc_decode_dense(const double* z, int64_t T, int64_t M, int64_t E, int64_t k, int64_t cap,
                      const int64_t* idxs, const int64_t* locations, const double* gates,
                      double* y) {
  double* w = (double*)calloc((size_t)(T * E * cap), sizeof(double));
  for (int64_t t = 0; t < T; ++t)
    for (int64_t j = 0; j < k; ++j)
      if (locations[t * k + j] >= 0)
        w[(t * E + idxs[t * k + j]) * cap + locations[t * k + j]] = gates[t * k + j];
  memset(y, 0, sizeof(double) * (size_t)(T * M));
  for (int64_t t = 0; t < T; ++t)
    for (int64_t e = 0; e < E; ++e)
      for (int64_t c = 0; c < cap; ++c) {
        const double wv = w[(t * E + e) * cap + c];
        for (int64_t d = 0; d < M; ++d) y[t * M + d] += wv * z[(e * cap + c) * M + d];
      }
  free(w);
}

/* ------------------------------------------------------------------ pipeline.cpp:33-66 */
void orc_partition_capacity(const double* x, int64_t E, int64_t C, int64_t M, int64_t degree,
                            double* chunks) {
  const int64_t cc = (C + degree - 1) / degree;
  memset(chunks, 0, sizeof(double) * (size_t)(degree * E * cc * M));
  for (int64_t i = 0; i < degree; ++i)
    for (int64_t e = 0; e < E; ++e)
      for (int64_t c = 0; c < cc; ++c) {
        const int64_t src = i * cc + c;
        if (src >= C) break;
        memcpy(chunks + ((i * E + e) * cc + c) * M, x + (e * C + src) * M, sizeof(double) * (size_t)M);
      }
}

void orc_merge_chunks(const double* chunks, int64_t E, int64_t cc, int64_t M, int64_t degree,
                      int64_t C, double* x) {
  memset(x, 0, sizeof(double) * (size_t)(E * C * M));
  for (int64_t i = 0; i < degree; ++i)
    for (int64_t e = 0; e < E; ++e)
      for (int64_t c = 0; c < cc; ++c) {
        const int64_t dst = i * cc + c;
        if (dst >= C) break;
        memcpy(x + (e * C + dst) * M, chunks + ((i * E + e) * cc + c) * M, sizeof(double) * (size_t)M);
      }
}

/* ------------------------------------------------------------------ collectives.cpp:123-160 */
void orc_flex_dispatch(const double* in, int64_t W, int64_t E, int64_t dC, int64_t M,
                       double* out) {
  const int64_t dE = E / W;
  for (int64_t d = 0; d < W; ++d)
    for (int64_t e = 0; e < dE; ++e)
      for (int64_t r = 0; r < W; ++r)
        for (int64_t c = 0; c < dC; ++c)
          memcpy(out + ((d * dE + e) * (W * dC) + r * dC + c) * M,
                 in + ((r * E + d * dE + e) * dC + c) * M, sizeof(double) * (size_t)M);
}

void orc_flex_combine(const double* in, int64_t W, int64_t E, int64_t dC, int64_t M,
                      double* out) {
  const int64_t dE = E / W;
  for (int64_t d = 0; d < W; ++d)
    for (int64_t e = 0; e < dE; ++e)
      for (int64_t r = 0; r < W; ++r)
        for (int64_t c = 0; c < dC; ++c)
          memcpy(out + ((r * E + d * dE + e) * dC + c) * M,
                 in + ((d * dE + e) * (W * dC) + r * dC + c) * M, sizeof(double) * (size_t)M);
}

/* The exchanges' net effect on the layer under either placement: expert e's computed rows are
 * (source r, slot c) = z[r][e][c], whichever ranks compute them -- per-rank placement
 * (flex_all2all above), sharded P1 (one replica per source group, moe_layer.cpp:20-57) and P2
 * (slices summed back at the source, :61-108) all apply the same full expert to the same rows.
 * Identical to orc_flex_dispatch / _combine when E % W == 0. */
static void orc_expert_major(const double* in, int64_t W, int64_t E, int64_t dC, int64_t M,
                             double* out) {
  for (int64_t e = 0; e < E; ++e)
    for (int64_t r = 0; r < W; ++r)
      memcpy(out + (e * W + r) * dC * M, in + (r * E + e) * dC * M, sizeof(double) * (size_t)(dC * M));
}

static void orc_expert_major_inv(const double* in, int64_t W, int64_t E, int64_t dC, int64_t M,
                                 double* out) {
  for (int64_t e = 0; e < E; ++e)
    for (int64_t r = 0; r < W; ++r)
      memcpy(out + (r * E + e) * dC * M, in + (e * W + r) * dC * M, sizeof(double) * (size_t)(dC * M));
}

/* ------------------------------------------------------------------ dense fp64 GEMMs */
/* C (m,n) = op(A) . B, row-major; op(A) = A (m,kk) or A^T with A (kk,m). Parallel over
 * (row block, column block) tiles so small per-expert row counts still use every core. */
static void dgemm_impl(const double* A, int trans_a, const double* B, double* Cm, int64_t m,
                       int64_t n, int64_t kk) {
  const int64_t MB = 16, KB = 256, NB = 256;
  const int64_t mb = (m + MB - 1) / MB, nb = (n + NB - 1) / NB;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t tile = 0; tile < mb * nb; ++tile) {
    const int64_t i0 = (tile / nb) * MB, j0 = (tile % nb) * NB;
    const int64_t i1 = i0 + MB < m ? i0 + MB : m, j1 = j0 + NB < n ? j0 + NB : n;
    for (int64_t i = i0; i < i1; ++i)
      for (int64_t j = j0; j < j1; ++j) Cm[i * n + j] = 0.0;
    for (int64_t k0 = 0; k0 < kk; k0 += KB) {
      const int64_t k1 = k0 + KB < kk ? k0 + KB : kk;
      for (int64_t i = i0; i < i1; ++i) {
        double* c = Cm + i * n;
        for (int64_t p = k0; p < k1; ++p) {
          const double a = trans_a ? A[p * m + i] : A[i * kk + p];
          const double* b = B + p * n;
          for (int64_t j = j0; j < j1; ++j) c[j] += a * b[j];
        }
      }
    }
  }
}

static void dgemm_nn(const double* A, const double* B, double* Cm, int64_t m, int64_t n,
                     int64_t kk) {
  dgemm_impl(A, 0, B, Cm, m, n, kk);
}

/* C (m,n) = A^T . B with A (kk,m), B (kk,n). */
static void dgemm_tn(const double* A, const double* B, double* Cm, int64_t m, int64_t n,
                     int64_t kk) {
  dgemm_impl(A, 1, B, Cm, m, n, kk);
}

static double* transpose(const double* A, int64_t r, int64_t c) {
  double* T = (double*)malloc(sizeof(double) * (size_t)(r * c));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < c; ++j) T[j * r + i] = A[i * c + j];
  return T;
}

/* parallelism.cpp:103-121 */
void orc_expert_ffn(const double* x, const double* w1, const double* w2, int64_t n, int64_t rows,
                    int64_t M, int64_t V, double* y) {
  double* h = (double*)malloc(sizeof(double) * (size_t)(rows * V));
  for (int64_t e = 0; e < n; ++e) {
    dgemm_nn(x + e * rows * M, w1 + e * M * V, h, rows, V, M);
    for (int64_t i = 0; i < rows * V; ++i) h[i] = h[i] > 0.0 ? h[i] : 0.0;
    dgemm_nn(h, w2 + e * V * M, y + e * rows * M, rows, M, V);
  }
  free(h);
}

/* parallelism.cpp:123-147 */
void orc_expert_ffn_backward(const double* x, const double* w1, const double* w2,
                             const double* dy, int64_t n, int64_t rows, int64_t M, int64_t V,
                             double* dx, double* dw1, double* dw2) {
  double* h = (double*)malloc(sizeof(double) * (size_t)(rows * V));
  double* dh = (double*)malloc(sizeof(double) * (size_t)(rows * V));
  for (int64_t e = 0; e < n; ++e) {
    const double* X = x + e * rows * M;
    const double* dY = dy + e * rows * M;
    dgemm_nn(X, w1 + e * M * V, h, rows, V, M);
    double* w2t = transpose(w2 + e * V * M, V, M); /* (M, V) */
    dgemm_nn(dY, w2t, dh, rows, V, M);
    free(w2t);
    for (int64_t i = 0; i < rows * V; ++i) {
      if (!(h[i] > 0.0)) dh[i] = 0.0;
      h[i] = h[i] > 0.0 ? h[i] : 0.0; /* a = relu(h) */
    }
    double* w1t = transpose(w1 + e * M * V, M, V); /* (V, M) */
    dgemm_nn(dh, w1t, dx + e * rows * M, rows, M, V);
    free(w1t);
    dgemm_tn(X, dh, dw1 + e * M * V, M, V, rows);
    dgemm_tn(h, dY, dw2 + e * V * M, V, M, rows);
  }
  free(h);
  free(dh);
}

/* moe_layer.cpp:321-335 */
void orc_frozen_plan_forward(const double* x, int64_t Ttot, int64_t M, int64_t V, int64_t k,
                             const int64_t* idxs, const int64_t* locations, const double* gates,
                             const double* w1, const double* w2, double* y) {
#pragma omp parallel
  {
    double* hid = (double*)malloc(sizeof(double) * (size_t)V);
#pragma omp for schedule(dynamic, 4)
    for (int64_t t = 0; t < Ttot; ++t) {
      double* yr = y + t * M;
      for (int64_t m = 0; m < M; ++m) yr[m] = 0.0;
      for (int64_t j = 0; j < k; ++j) {
        if (locations[t * k + j] < 0) continue;
        const int64_t e = idxs[t * k + j];
        const double* W1 = w1 + e * M * V;
        const double* W2 = w2 + e * V * M;
        for (int64_t v = 0; v < V; ++v) hid[v] = 0.0;
        for (int64_t m = 0; m < M; ++m) {
          const double xv = x[t * M + m];
          for (int64_t v = 0; v < V; ++v) hid[v] += xv * W1[m * V + v];
        }
        const double g = gates[t * k + j];
        for (int64_t v = 0; v < V; ++v) {
          const double a = hid[v] > 0.0 ? hid[v] : 0.0;
          if (a == 0.0) continue;
          for (int64_t m = 0; m < M; ++m) yr[m] += g * a * W2[v * M + m];
        }
      }
    }
    free(hid);
  }
}

/* The backward of the frozen plan, token by token (moe_layer.cpp:246-319 restricted to the listed
 * tokens): dz = g[t,j] * dy[t] (fast_decode_backward, dispatch.cpp:136-157), the expert's
 * dX row = ((dz . W2^T) * [x W1 > 0]) . W1^T (expert_ffn_backward, parallelism.cpp:123-147),
 * summed over kept j (fast_encode_backward, dispatch.cpp:117-128). Rows are independent, so
 * a token subset of a large layer is checked exactly. */
void orc_frozen_plan_backward_rows(const double* x, const double* dy, int64_t Tsel, int64_t M,
                                   int64_t V, int64_t k, const int64_t* idxs,
                                   const int64_t* locations, const double* gates, const double* w1,
                                   const double* w2, double* dx) {
#pragma omp parallel
  {
    double* hid = (double*)malloc(sizeof(double) * (size_t)V);
    double* dh = (double*)malloc(sizeof(double) * (size_t)V);
#pragma omp for schedule(dynamic, 1)
    for (int64_t t = 0; t < Tsel; ++t) {
      double* dr = dx + t * M;
      for (int64_t m = 0; m < M; ++m) dr[m] = 0.0;
      for (int64_t j = 0; j < k; ++j) {
        if (locations[t * k + j] < 0) continue;
        const int64_t e = idxs[t * k + j];
        const double* W1 = w1 + e * M * V;
        const double* W2 = w2 + e * V * M;
        const double g = gates[t * k + j];
        for (int64_t v = 0; v < V; ++v) hid[v] = 0.0;
        for (int64_t m = 0; m < M; ++m) {
          const double xv = x[t * M + m];
          for (int64_t v = 0; v < V; ++v) hid[v] += xv * W1[m * V + v];
        }
        for (int64_t v = 0; v < V; ++v) {
          double a = 0.0;
          if (hid[v] > 0.0)
            for (int64_t m = 0; m < M; ++m) a += g * dy[t * M + m] * W2[v * M + m];
          dh[v] = a;
        }
        for (int64_t m = 0; m < M; ++m) {
          double a = 0.0;
          for (int64_t v = 0; v < V; ++v) a += dh[v] * W1[m * V + v];
          dr[m] += a;
        }
      }
    }
    free(hid);
    free(dh);
  }
}

/* Selected hidden units of one expert's weight gradient (expert_ffn_backward,
 * parallelism.cpp:123-147): with h = X W1, dh = (dZ W2^T) * [h > 0], column v of dW1 = X^T dh
 * and row v of dW2 = relu(h)^T dZ need only column v of h and dh, so a few units of a large
 * expert are exact. X, dZ: the expert's (rows, M) inputs and output gradients (gate-scaled,
 * all source ranks, empty capacity slots omitted -- they contribute zero).
 * Outputs dw1c (M, ncols) = dW1[:, cols], dw2r (ncols, M) = dW2[cols, :]. */
void orc_expert_backward_columns(const double* X, const double* dZ, int64_t rows, int64_t M,
                                 int64_t V, const double* w1, const double* w2, int64_t ncols,
                                 const int64_t* cols, double* dw1c, double* dw2r) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < ncols; ++c) {
    const int64_t v = cols[c];
    double* a1 = (double*)calloc((size_t)M, sizeof(double));
    double* a2 = (double*)calloc((size_t)M, sizeof(double));
    for (int64_t r = 0; r < rows; ++r) {
      const double* xr = X + r * M;
      const double* dr = dZ + r * M;
      double h = 0.0, da = 0.0;
      for (int64_t m = 0; m < M; ++m) h += xr[m] * w1[m * V + v];
      if (!(h > 0.0)) continue; /* a = 0 and dh = 0: the row adds nothing */
      for (int64_t m = 0; m < M; ++m) da += dr[m] * w2[v * M + m];
      for (int64_t m = 0; m < M; ++m) {
        a1[m] += xr[m] * da;
        a2[m] += h * dr[m];
      }
    }
    for (int64_t m = 0; m < M; ++m) {
      dw1c[m * ncols + c] = a1[m];
      dw2r[c * M + m] = a2[m];
    }
    free(a1);
    free(a2);
  }
}

/* ------------------------------------------------------------------ moe_layer.cpp:171-319 */
/* moe_layer.cpp:171-319 from the router's probabilities (route_probabilities, :165-169). */
int64_t orc_layer_step_probs(const double* x, const double* probs, const double* w1,
                             const double* w2, const double* dy, int64_t W, int64_t T, int64_t M,
                             int64_t V, int64_t E, int64_t k, int32_t cap_kind, double factor,
                             int32_t bpr, double* y, int64_t* idxs, int64_t* locations,
                             double* gates, double* dx, double* dw1, double* dw2) {
  const int64_t cap = orc_run_gating_blocked(probs, W, T, E, k, cap_kind, factor, bpr, idxs, gates,
                                             locations);
  const int64_t rows = W * cap; /* gathered capacity C = W * dC per expert */
  const size_t zsz = (size_t)(W * E * cap * M);
  double* z = (double*)malloc(sizeof(double) * zsz);
  double* xe = (double*)malloc(sizeof(double) * zsz);
  double* ye = (double*)malloc(sizeof(double) * zsz);
  orc_encode(x, W, T, M, E, k, cap, idxs, locations, z);
  /* flex dispatch: expert e's input rows (r, c) = z[r][e][c] (collectives.cpp:123-141) */
  if (E % W == 0) orc_flex_dispatch(z, W, E, cap, M, xe);
  else orc_expert_major(z, W, E, cap, M, xe); /* sharded placement (E < W) */
  orc_expert_ffn(xe, w1, w2, E, rows, M, V, ye);
  if (E % W == 0) orc_flex_combine(ye, W, E, cap, M, z);
  else orc_expert_major_inv(ye, W, E, cap, M, z);
  orc_decode(z, W, T, M, E, k, cap, idxs, locations, gates, y);
  if (dy) {
    double* dz = (double*)malloc(sizeof(double) * zsz);
    double* dye = (double*)malloc(sizeof(double) * zsz);
    orc_decode_backward(dy, NULL, W, T, M, E, k, cap, idxs, locations, gates, dz, NULL);
    if (E % W == 0) orc_flex_dispatch(dz, W, E, cap, M, dye);
    else orc_expert_major(dz, W, E, cap, M, dye);
    orc_expert_ffn_backward(xe, w1, w2, dye, E, rows, M, V, ye, dw1, dw2);
    if (E % W == 0) orc_flex_combine(ye, W, E, cap, M, dz);
    else orc_expert_major_inv(ye, W, E, cap, M, dz);
    orc_encode_backward(dz, W, T, M, E, k, cap, idxs, locations, dx);
    free(dz);
    free(dye);
  }
  free(z);
  free(xe);
  free(ye);
  return cap;
}

int64_t orc_layer_step(const double* x, const double* wg, const double* w1, const double* w2,
                       const double* dy, int64_t W, int64_t T, int64_t M, int64_t V, int64_t E,
                       int64_t k, int32_t cap_kind, double factor, int32_t bpr, double* y,
                       int64_t* idxs, int64_t* locations, double* gates, double* dx,
                       double* dw1, double* dw2) {
  const int64_t Ttot = W * T;
  double* probs = (double*)malloc(sizeof(double) * (size_t)(Ttot * E));
  orc_gate_linear(x, wg, Ttot, M, E, probs);
  const int64_t cap = orc_layer_step_probs(x, probs, w1, w2, dy, W, T, M, V, E, k, cap_kind,
                                           factor, bpr, y, idxs, locations, gates, dx, dw1, dw2);
  free(probs);
  return cap;
}

int32_t orc_num_threads(void) { return (int32_t)omp_get_max_threads(); }

/* bench.py's reference arm runs on rank 0 only; torchrun exports OMP_NUM_THREADS=1 to every
   rank, so the arm raises the pool back to the host's cores here. */
void orc_set_num_threads(int32_t n) { if (n > 0) omp_set_num_threads(n); }
