/*
 * moe_oracle.h -- CPU fp64 restatement of the reference MoE layer path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the sm_100a kernels and the
 * CPU baseline timed by bench.py (`cpu_baseline` leg / `--impl reference`). It is never linked
 * into, loaded by, or called from the product path (paper_2206_03382_b200/), which has no CPU
 * fallback. Only tests/, __graft_entry__.smoke() and bench.py's baseline leg may use it.
 *
 * Why a restatement: the reference (/root/reference/proj, C++20 + Eigen 3) cannot be compiled
 * here -- Eigen and the vendored doctest/CLI11 are absent. Every function
 * cites the reference file:line whose semantics it restates; Eigen GEMM/exp/sum are replaced by
 * plain loops (summation-order differences are ulp-level, far below every tolerance).
 * Pinned against the reference's own known-answer tests (tests/golden/reference_kats.json).
 */
#ifndef MOE_ORACLE_H
#define MOE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* core.cpp:66-83 splitmix64; orc_draw(seed, n) = lo + (hi-lo) * uniform of call n (0-based). */
uint64_t orc_next_u64(uint64_t* state);
double orc_uniform(uint64_t* state);
void orc_fill_uniform(uint64_t seed, uint64_t offset, int64_t n, double lo, double hi, double* out);

/* core.cpp:28-35, 47-59, 61-64 */
int64_t orc_expert_capacity(int64_t k, double f, int64_t tokens, int64_t experts);
int64_t orc_resolve_capacity(int32_t kind, double factor, const int64_t* demand, int64_t E,
                             int64_t k, int64_t T);
double orc_capacity_to_factor(int64_t cap, int64_t E, int64_t k, int64_t T);

/* gating.cpp:19-35: probs = softmax_rows(x . wg); x (T,M), wg (M,E). */
void orc_gate_linear(const double* x, const double* wg, int64_t T, int64_t M, int64_t E,
                     double* probs);
/* gating.cpp:58-78 */
int32_t orc_gate_cosine(const double* x, const double* proj_w, const double* experts,
                        double temperature, int64_t T, int64_t M, int64_t E, int64_t D,
                        double* probs);
void orc_topk_select(const double* probs, int64_t T, int64_t E, int64_t k, int64_t* idxs,
                     double* gates);
/* gating.cpp:80-112 */
void orc_assign_locations(const int64_t* idxs, const double* gates, int64_t T, int64_t k,
                          int64_t cap, int32_t bpr, int64_t* locations);
/* gating.cpp:134-162; T = rows per block; returns the resolved capacity. */
int64_t orc_run_gating_blocked(const double* probs, int64_t blocks, int64_t T, int64_t E,
                               int64_t k, int32_t cap_kind, double factor, int32_t bpr,
                               int64_t* idxs, double* gates, int64_t* locations);
int64_t orc_drop_count(const int64_t* locations, int64_t n);

/* dispatch.cpp:51-62 per block b: z[b] (E, cap, M) zero + scatter of rows [b*T, (b+1)*T). */
void orc_encode(const double* x, int64_t blocks, int64_t T, int64_t M, int64_t E, int64_t k,
                int64_t cap, const int64_t* idxs, const int64_t* locations, double* z);
/* dispatch.cpp:75-87 */
void orc_decode(const double* z, int64_t blocks, int64_t T, int64_t M, int64_t E, int64_t k,
                int64_t cap, const int64_t* idxs, const int64_t* locations, const double* gates,
                double* y);
/* dispatch.cpp:136-157 (dgates may be NULL) */
void orc_decode_backward(const double* dy, const double* z, int64_t blocks, int64_t T, int64_t M,
                         int64_t E, int64_t k, int64_t cap, const int64_t* idxs,
                         const int64_t* locations, const double* gates, double* dz,
                         double* dgates);
/* dispatch.cpp:117-128 */
void orc_encode_backward(const double* dz, int64_t blocks, int64_t T, int64_t M, int64_t E,
                         int64_t k, int64_t cap, const int64_t* idxs, const int64_t* locations,
                         double* dx);
/* dispatch.cpp:20-40 / 89-109 dense one-hot einsum oracles (single block). */
void orc_encode_dense(const double* x, int64_t T, int64_t M, int64_t E, int64_t k, int64_t cap,
                      const int64_t* idxs, const int64_t* locations, double* z);
void orc_decode_dense(const double* z, int64_t T, int64_t M, int64_t E, int64_t k, int64_t cap,
                      const int64_t* idxs, const int64_t* locations, const double* gates,
                      double* y);

/* pipeline.cpp:33-66: (E, C, M) -> degree x (E, cc, M), cc = ceil(C/degree), zero tail. */
void orc_partition_capacity(const double* x, int64_t E, int64_t C, int64_t M, int64_t degree,
                            double* chunks);
void orc_merge_chunks(const double* chunks, int64_t E, int64_t cc, int64_t M, int64_t degree,
                      int64_t C, double* x);

/* collectives.cpp:123-160 flex all-to-all on W simulated ranks (linear algorithm):
 * dispatch: in[r] (E, dC, M) -> out[d] (dE, W*dC, M), out[d][e][r*dC+c] = in[r][d*dE+e][c];
 * combine: the inverse. Buffers are rank-major concatenations. */
void orc_flex_dispatch(const double* in, int64_t W, int64_t E, int64_t dC, int64_t M,
                       double* out);
void orc_flex_combine(const double* in, int64_t W, int64_t E, int64_t dC, int64_t M,
                      double* out);

/* parallelism.cpp:103-121: y[e] = relu(x[e] . w1[e]) . w2[e]; x (n, rows, M). */
void orc_expert_ffn(const double* x, const double* w1, const double* w2, int64_t n, int64_t rows,
                    int64_t M, int64_t V, double* y);
/* parallelism.cpp:123-147 */
void orc_expert_ffn_backward(const double* x, const double* w1, const double* w2,
                             const double* dy, int64_t n, int64_t rows, int64_t M, int64_t V,
                             double* dx, double* dw1, double* dw2);

/* moe_layer.cpp:321-335: per-token oracle y[t] += g * relu(x[t] w1[e]) w2[e]. */
void orc_frozen_plan_forward(const double* x, int64_t Ttot, int64_t M, int64_t V, int64_t k,
                             const int64_t* idxs, const int64_t* locations, const double* gates,
                             const double* w1, const double* w2, double* y);

/* Frozen-plan backward of selected tokens (moe_layer.cpp:246-319): dx rows (Tsel, M). */
void orc_frozen_plan_backward_rows(const double* x, const double* dy, int64_t Tsel, int64_t M,
                                   int64_t V, int64_t k, const int64_t* idxs,
                                   const int64_t* locations, const double* gates, const double* w1,
                                   const double* w2, double* dx);
/* Selected hidden units of one expert's dW1 columns / dW2 rows (parallelism.cpp:123-147). */
void orc_expert_backward_columns(const double* X, const double* dZ, int64_t rows, int64_t M,
                                 int64_t V, const double* w1, const double* w2, int64_t ncols,
                                 const int64_t* cols, double* dw1c, double* dw2r);

/* Whole layer for W source blocks on one host (moe_layer.cpp:171-319, per-rank placement,
 * linear router): gate -> encode -> per-expert FFN over the gathered capacity rows -> decode,
 * and the reverse pass (gates frozen; d_gates discarded). w1 (E,M,V), w2 (E,V,M).
 * Outputs: y (W*T, M); routing (W*T, k); dx (W*T, M), dw1, dw2 (if dy != NULL). */
int64_t orc_layer_step_probs(const double* x, const double* probs, const double* w1,
                             const double* w2, const double* dy, int64_t W, int64_t T, int64_t M,
                             int64_t V, int64_t E, int64_t k, int32_t cap_kind, double factor,
                             int32_t bpr, double* y, int64_t* idxs, int64_t* locations,
                             double* gates, double* dx, double* dw1, double* dw2);
int64_t orc_layer_step(const double* x, const double* wg, const double* w1, const double* w2,
                       const double* dy, int64_t W, int64_t T, int64_t M, int64_t V, int64_t E,
                       int64_t k, int32_t cap_kind, double factor, int32_t bpr, double* y,
                       int64_t* idxs, int64_t* locations, double* gates, double* dx,
                       double* dw1, double* dw2);

/* Number of OpenMP threads the oracle uses (for the CPU-baseline "cores" field). */
int32_t orc_num_threads(void);
void orc_set_num_threads(int32_t n);

#ifdef __cplusplus
}
#endif

#endif
