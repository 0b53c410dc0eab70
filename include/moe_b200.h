/*
 * moe_b200.h -- C ABI of the B200-native Tutel-style MoE layer (libmoe_b200.so).
 *
 * This is the drop-in boundary for the reference's MoE layer path (the C++ library API of
 * /root/reference/proj/include/moesim/moe_layer.hpp and its sub-operators in gating.hpp /
 * dispatch.hpp / parallelism.hpp / pipeline.hpp). Every entry point names the reference
 * declaration it replaces. Conventions:
 *   - plain pointers + sizes, no C++ or torch types; streams are cudaStream_t passed as void*;
 *   - status codes instead of exceptions: MOE_EINVAL for the reference's std::invalid_argument,
 *     MOE_ECOMM for std::runtime_error raised by the fabric, MOE_ESTATE for std::logic_error;
 *   - row-major layouts exactly as the reference (x: (T, M); W1: (M, V); W2: (V, M); Wg: (M, E));
 *   - one handle per rank (one process or host thread per GPU); the handle is single-writer,
 *     like LayerState (moe_layer.hpp:33-44).
 * There is no CPU fallback: every compute entry point runs sm_100a kernels and fails with
 * MOE_ECUDA when no usable device is present.
 */
#ifndef MOE_B200_H
#define MOE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_OK 0
#define MOE_EINVAL 1 /* std::invalid_argument (core.cpp:9-25, dispatch.cpp:7-16, ...) */
#define MOE_ECUDA 2  /* CUDA launch / runtime failure, or no sm_100 device */
#define MOE_ECOMM 3  /* std::runtime_error from the fabric (fabric.cpp:144-160,233-258) */
#define MOE_ESTATE 4 /* std::logic_error (pipeline.cpp:148,216,227) / call-order misuse */
#define MOE_ENOMEM 5

#define MOE_DTYPE_BF16 0
#define MOE_DTYPE_F32 1
#define MOE_DTYPE_F64 2

#define MOE_CAP_FIXED 0   /* FixedCapacity{factor}       core.hpp:25-27 */
#define MOE_CAP_AUTO 1    /* AutoCapacity{}              core.hpp:28 */
#define MOE_CAP_BOUNDED 2 /* BoundedCapacity{max_factor} core.hpp:29-31 */

#define MOE_A2A_LINEAR 0 /* A2aAlgo::Linear (collectives.hpp:10) */
#define MOE_A2A_2DH 1    /* A2aAlgo::TwoDH (all2all_2dh, collectives.cpp:58-88): intra-node exchange
                            of node-aligned blocks, then inter-node exchange between same-local
                            GPUs. Run as two NCCL phases when gpus_per_node < W on the NCCL
                            transport; the peer transport and m == W run it as linear. */

/* MoELayerConfig (moe_layer.hpp:22-29) flattened with Dims (core.hpp:32-56). The placement
 * follows from E and W: E >= W is per-rank placement (ExpertsPerRank{E/W}, E = W*x); E < W is
 * sharded placement (RanksPerExpert{s}, W = E*s): rank r serves expert r/s, slice r%s. */
typedef struct moe_config {
  int64_t world_size;      /* W */
  int64_t gpus_per_node;   /* m */
  int64_t global_experts;  /* E (= W * local experts) */
  int64_t model_dim;       /* M */
  int64_t hidden_dim;      /* V */
  int64_t tokens_per_step; /* T, tokens per rank */
  int64_t top_k;           /* k */
  int32_t capacity_kind;   /* MOE_CAP_* */
  double capacity_factor;  /* f (Fixed) or max_factor (Bounded) */
  int32_t bpr;             /* batch-prioritized routing */
  int32_t dtype;           /* MOE_DTYPE_BF16 (tensor-core path) or MOE_DTYPE_F32 */
  int32_t adaptive;        /* StrategyControl::adaptive: Alg. 1 picks the pipelining degree */
  int32_t degree;          /* StrategyControl::fixed.degree (capacity chunks), 1..8 */
  int32_t a2a_backend;     /* MOE_A2A_BACKEND_*: how W > 1 ranks exchange tokens */
  int32_t router;          /* MOE_ROUTER_* (RouterKind, moe_layer.hpp:10) */
  int32_t parallel;        /* MOE_PARALLEL_* (ParallelControl, moe_layer.hpp:17-20); sharded only */
  int32_t a2a_algo;        /* StrategyControl::fixed.algo: MOE_A2A_LINEAR or MOE_A2A_2DH */
  int32_t gate_precision;  /* MOE_GATE_*: how the router logits are computed */
} moe_config;

/* Router GEMM precision. AUTO (0, the default): the bf16 layer with the linear router and FIFO
 * routing (E % 8 == 0, E <= 64, M % 64 == 0, k <= 8) runs the certified tensor-core gate --
 * logits from bf16 MMAs with a proven error bound, every token whose top-k order the bound
 * cannot prove re-decided from fp64 logits, so expert ids, slots and drops stay bit-exact;
 * gate values of certified tokens carry the bound's error (relative ~1e-6 typical, well inside
 * the bf16 output tolerance). Every other layer, and FP64, runs the fp64 DMMA gate (gate values
 * equal to the fp64 reference's up to summation order). */
#define MOE_GATE_AUTO 0
#define MOE_GATE_FP64 1

/* ParallelControl / ParallelChoice (parallelism.hpp): the sharded-placement exchange form.
 * P1 gathers each computed expert's weights and routes every source's tokens to one replica
 * (moe_layer.cpp:17-57); P2 keeps the weight slices in place, repeats the tokens to all s
 * shards and sums their partial outputs (moe_layer.cpp:59-108). ADAPTIVE picks the cheaper by
 * select_parallelism (parallelism.cpp:300-318) every forward. Zero is the reference default
 * (adaptive = false, fixed = P1). */
#define MOE_PARALLEL_P1 0
#define MOE_PARALLEL_P2 1
#define MOE_PARALLEL_ADAPTIVE 2

/* Router (route_probabilities, moe_layer.cpp:165-169). COSINE: softmax of
 * cos(x . P, C_e) / max(temperature, 0.01) (gate_cosine, gating.cpp:37-56), P (M, 256),
 * C (E, 256), fp64; the DMMA kernels support E <= 64 (even). */
#define MOE_ROUTER_LINEAR 0
#define MOE_ROUTER_COSINE 1
#define MOE_COSINE_DIM 256

/* All-to-all transport for W > 1. PEER: copy engines push blocks into the peers' receive
 * buffers over NVLink (CUDA IPC mappings), ordered by epoch flags -- no SMs are taken from the
 * expert GEMMs it overlaps. NCCL: grouped ncclSend/ncclRecv. Same plan (moe_a2a_plan), same
 * results bit for bit. */
#define MOE_A2A_BACKEND_PEER 0
#define MOE_A2A_BACKEND_NCCL 1

/* StepMetrics (moe_layer.hpp:46-54); sim_seconds becomes measured device seconds. */
typedef struct moe_step_metrics {
  double f;            /* capacity_to_factor(capacity) */
  int64_t capacity;    /* ΔC */
  int32_t a2a_algo;    /* MOE_A2A_* */
  int32_t degree;      /* pipelining degree used */
  double seconds;      /* forward device time (CUDA events), 0 if not measured */
  double comm_bytes;   /* bytes this rank sent in the forward all-to-alls */
  int64_t drop_count;  /* dropped (token, expert) assignments on this rank */
  int64_t relu_fixups; /* bf16 path: up-GEMM outputs re-decided in fp64 (ReLU-mask certificate,
                          last chunk of the last forward) */
  int32_t fused;       /* MOE_FUSED_* bits: which exchanges ran inside the GEMM epilogues */
  int32_t parallel;    /* MOE_PARALLEL_P1 / _P2: the exchange form used (StepMetrics::parallel) */
  int64_t gate_fixups; /* certified gate: tokens re-decided from fp64 logits since the last
                          moe_get_metrics (0 with the fp64 gate) */
  int64_t simt_gemms;  /* bf16 expert-GEMM launches of the last forward + backward that ran the
                          SIMT kernel because the shape is not tcgen05-eligible (N % 256, K % 64,
                          wgrad rows % 128): ~10x slower; 0 on every BASELINE config */
} moe_step_metrics;
#define MOE_FUSED_DECODE 1  /* W = 1, k = 1: decode / encode-backward = down / dgrad epilogue scatter */
#define MOE_FUSED_COMBINE 2 /* W > 1 peer backend: combine = down / dgrad epilogue NVLink stores */

typedef struct moe_handle moe_handle;

/* ---------------------------------------------------------------- capacity math (core.cpp) */
/* expert_capacity, core.cpp:28-35: max(1, ceil(k*f*T/E - 1e-9)). */
int moe_expert_capacity(int64_t k, double f, int64_t tokens, int64_t experts, int64_t* out);
/* resolve_capacity, core.cpp:47-59 (demand has E entries). */
int moe_resolve_capacity(int32_t capacity_kind, double factor, const int64_t* demand,
                         int64_t experts, int64_t top_k, int64_t tokens, int64_t* out);
/* capacity_to_factor, core.cpp:61-64. */
int moe_capacity_to_factor(int64_t capacity, int64_t experts, int64_t top_k, int64_t tokens,
                           double* out);
/* Dims::validate, core.cpp:8-26 (both placements) + ExpertParams' slice divisibility. */
int moe_validate_config(const moe_config* cfg);
/* select_parallelism, parallelism.cpp:288-308: P1 when comm_cost_p1 <= comm_cost_p2 (ties to
 * the weight gather). local_experts may be fractional (1/s under sharded placement). EINVAL for
 * n_sharded < 1 (comm_cost_p2's invalid_argument). *out = MOE_PARALLEL_P1 or _P2. */
int moe_select_parallelism(double local_experts, int64_t gathered_capacity, int64_t model_dim,
                           double param_bytes, int64_t n_sharded, int32_t* out);

/* Flexible all-to-all plan (flex_all2all, collectives.cpp:116-162, over all2all_linear
 * :48-56) for pipeline chunk `chunk`: element offsets of the block sent to / received from each
 * peer (arrays of W) and the block size. phase 0 = dispatch: send buffer [degree][E][cc][M],
 * peer p gets experts [p*E/W, (p+1)*E/W); receive buffer [degree][W][E/W][cc][M], i.e. expert
 * e's gathered rows (source r, slot c) -- the (dE, W*cc, M) interleave -- without a copy.
 * phase 1 = combine: the inverse. Host-only; the layer's NCCL exchanges use exactly this plan. */
int moe_a2a_plan(int64_t W, int64_t E, int64_t cc, int64_t M, int64_t chunk, int32_t phase,
                 int64_t* send_offsets, int64_t* recv_offsets, int64_t* elems);

/* ---------------------------------------------------------------- layer (moe_layer.hpp) */
/* NCCL unique id for W > 1 (128 bytes), created on rank 0 and broadcast by the caller. */
int moe_get_unique_id(uint8_t* id128);
/* LayerState construction for one rank (moe_layer.cpp:144-163 minus the weight draw):
 * allocates device state on `device`, creates the NCCL communicator when W > 1. */
int moe_create(const moe_config* cfg, int32_t rank, const uint8_t* nccl_id128, int32_t device,
               moe_handle** out);
int moe_destroy(moe_handle* h);
const char* moe_last_error(const moe_handle* h);
/* Per-thread message of the last failing stateless call (moe_op_*, moe_create). */
const char* moe_last_error_global(void);

/* LayerState::init draw (moe_layer.cpp:144-163): Rng(seed) draws Wg (M,E), the cosine router
 * (M,256)+(E,256), then w1 (M,V), w2 (V,M) per expert, all uniform; generated on the device by
 * counter index, so every rank holds exactly the reference's values for its local experts. */
int moe_init_params(moe_handle* h, uint64_t seed);
/* RouterParams::linear_weight (gating.hpp:25-30); host fp64 (M, E). */
int moe_set_router(moe_handle* h, const double* wg_host);
/* RouterParams::cosine_proj (M, 256), cosine_experts (E, 256), temperature (host fp64). A
 * zero-norm expert row is rejected (MOE_EINVAL, as gate_cosine's invalid_argument); a
 * zero-norm projected token is detected on the device and reported by the next
 * moe_get_metrics / moe_get_routing call (MOE_EINVAL). */
int moe_set_cosine_router(moe_handle* h, const double* proj_host, const double* experts_host,
                          double temperature);
/* FixedCapacity{f} from the next forward on (the scenario runner's per-step trace,
 * bench.cpp:199-201). Collective when W > 1 (buffers may grow): every rank calls it. */
int moe_set_capacity_factor(moe_handle* h, double f);
/* Full weights of local expert `local_e` (global index rank*E/W + local_e; sharded placement:
 * local_e 0 = expert rank/s); host fp64 w1 (M, V), w2 (V, M) -- ExpertParams::assemble layout
 * (parallelism.cpp:80-90). */
int moe_set_expert(moe_handle* h, int64_t local_e, const double* w1_host, const double* w2_host);
/* ZeRO-sliced parameters (ExpertParams, parallelism.hpp:22-37): this rank's slice of every
 * expert (w1 columns / w2 rows [rank*V/W, (rank+1)*V/W)), host fp64, expert-major
 * [E][M][V/W] and [E][V/W][M]. Followed by one grouped exchange that assembles the local
 * experts -- gather_computed_experts, parallelism.cpp:149-206. Sharded placement: the one slice
 * rank%s of expert rank/s, [1][M][V/s] and [1][V/s][M], all-gathered within the expert's group
 * (parallelism.cpp:155-175). */
int moe_set_expert_slices(moe_handle* h, const double* w1_slices, const double* w2_slices);

/* forward(state, x) (moe_layer.cpp:171-244) for this rank's token block: x, y are device
 * (T, M) in the layer dtype. Saves what backward needs inside the handle. */
int moe_forward(moe_handle* h, const void* x, void* y, void* stream);
/* backward(state, saved, dy) (moe_layer.cpp:246-319): dx device (T, M); dw1/dw2 device fp32
 * (E/W, M, V) and (E/W, V, M) for the local experts (may be NULL: kept in the handle). */
int moe_backward(moe_handle* h, const void* dy, void* dx, float* dw1, float* dw2, void* stream);
/* Same calls with HOST (preferably pinned) buffers: host->device copy of the input and
 * device->host copy of the result happen inside the call, as a reference caller would see. */
int moe_forward_host(moe_handle* h, const void* x_host, void* y_host, void* stream);
int moe_backward_host(moe_handle* h, const void* dy_host, void* dx_host, void* stream);
/* Pipelined variants for a stream of steps (a data loader feeding the layer): they return after
 * enqueueing; the upload of the input and the download of the result run on the handle's own
 * copy streams and overlap the neighbouring steps' compute (double-buffered device staging).
 * Host buffers must be pinned and stay untouched (inputs) / unread (outputs) until
 * moe_host_sync, which waits for every enqueued download. */
int moe_forward_host_async(moe_handle* h, const void* x_host, void* y_host, void* stream);
int moe_backward_host_async(moe_handle* h, const void* dy_host, void* dx_host, void* stream);
int moe_host_sync(moe_handle* h);

/* Routing of the last forward (GateOutput, gating.hpp:14-23): host buffers (T, k). */
int moe_get_routing(moe_handle* h, int32_t* idxs, int32_t* locations, double* gates,
                    int64_t* capacity);
int moe_get_metrics(moe_handle* h, moe_step_metrics* out);
/* Local expert gradients of the last backward, copied to host fp32 (E/W, M, V)+(E/W, V, M).
 * Sharded placement: the full gradient of expert rank/s (1, M, V)+(1, V, M), already summed over
 * the expert's s replicas (P1) or assembled from its s slices (P2). */
int moe_get_expert_grads(moe_handle* h, float* dw1_host, float* dw2_host);
/* reduce_scatter_grads_p1 (parallelism.cpp:235-286): after a backward, route slice `rank` of
 * every expert's weight gradient (dW1 columns / dW2 rows [rank*V/W, (rank+1)*V/W)) to this rank
 * -- the ZeRO slice layout of moe_set_expert_slices. Device fp32 outputs: w1_slices
 * [E][M][V/W], w2_slices [E][V/W][M]. Collective across ranks (NCCL); synchronizes `stream`.
 * Sharded placement: this rank's slice rank%s of expert rank/s, [1][M][V/s] and [1][V/s][M]. */
int moe_get_expert_grad_slices(moe_handle* h, float* w1_slices, float* w2_slices, void* stream);
/* Device pointer to local expert weights in the layer dtype: which=1 -> w1, 2 -> w2 (layouts
 * [E/W][M][V] / [E/W][V][M]). The pointer is writable (an on-device optimizer step updates the
 * weights in place): handing it out marks the layer's derived weight state (the ReLU
 * certificate's W1^T copy and column norms, the sharded W1 slice) stale, and a caller that keeps
 * the pointer and writes through it later must call moe_weights_updated before the next
 * forward. Writes must be ordered before that forward's stream work. */
int moe_get_weights_device(moe_handle* h, int32_t which, void** ptr);
/* Declare that the resident expert weights changed (in place, through moe_get_weights_device):
 * the next forward rebuilds the state derived from them. Cheap; no device work until then. */
int moe_weights_updated(moe_handle* h);
/* Number of kernels launched by the last forward + backward (benchmark bookkeeping). */
int64_t moe_kernel_launches(const moe_handle* h);
/* Measured timeline (replaces the simulated Timeline of pipeline.hpp:36-46): when on, every
 * phase is bracketed by CUDA events on the stream it runs on. Phases, in order: gate, encode,
 * gemm_up, gemm_down, decode, decode_bwd, gemm_dgrad_mask, gemm_dgrad, gemm_wgrad1,
 * gemm_wgrad2, encode_bwd, a2a_fwd, a2a_bwd, assign, relu_fixup, xfer_dispatch, xfer_combine,
 * weight_stats (MOE_NUM_PHASES; weight_stats = rebuilding the ReLU certificate's W1^T and column
 * norms after the weights changed). a2a_* span the comm stream's enqueue and waits; xfer_* span only the
 * copy-engine pushes over NVLink (peer transport), from the push's start to its last block landing. */
#define MOE_NUM_PHASES 18
int moe_set_profiling(moe_handle* h, int32_t on);
/* Kernel spans of the tcgen05 expert GEMMs, measured with the device clock (%globaltimer: first
 * CTA past its launch-dependency wait to last CTA exit) instead of CUDA events, so programmatic
 * dependent launch keeps overlapping the kernels. moe_take_kernel_spans fills, per phase of the
 * MOE_NUM_PHASES list above, the summed span in ms and the launch count since the last call;
 * sm_mhz (optional): the effective SM clock inside those kernels (clock64 / %globaltimer). */
int moe_set_kernel_spans(moe_handle* h, int32_t on);
int moe_take_kernel_spans(moe_handle* h, double* ms, int64_t* counts, int32_t n, double* sm_mhz);
/* Per-phase summed milliseconds and interval counts since the last call (synchronizes). */
int moe_take_profile(moe_handle* h, double* ms, int64_t* counts, int32_t n);

/* ---------------------------------------------------------------- stateless device ops
 * All pointers are device memory; each call is stream-ordered on `stream` and allocates its
 * own scratch. These are the reference sub-operators, for parity testing and composition. */

/* gate_linear + run_gating_blocked (gating.cpp:29-35, 134-162): x (blocks*T, M) in x_dtype,
 * wg (M, E) fp64 -> idxs/locations int32 (blocks*T, k), gates fp64 (blocks*T, k), optional
 * probs fp64 (blocks*T, E). Returns the resolved capacity and the drop count (synchronizes). */
int moe_op_gating(const void* x, int32_t x_dtype, const double* wg, int64_t blocks, int64_t T,
                  int64_t M, int64_t E, int64_t k, int32_t capacity_kind, double capacity_factor,
                  int32_t bpr, int32_t* idxs, double* gates, int32_t* locations, double* probs,
                  int64_t* capacity, int64_t* drops, void* stream);

/* gate_cosine + run_gating_blocked: as moe_op_gating with the cosine router (proj (M, D),
 * experts (E, D), device fp64). */
int moe_op_gating_cosine(const void* x, int32_t x_dtype, const double* proj, const double* experts,
                         int64_t D, double temperature, int64_t blocks, int64_t T, int64_t M,
                         int64_t E, int64_t k, int32_t capacity_kind, double capacity_factor,
                         int32_t bpr, int32_t* idxs, double* gates, int32_t* locations,
                         double* probs, int64_t* capacity, int64_t* drops, void* stream);

/* fast_encode_range per block (dispatch.cpp:51-62) + partition_capacity (pipeline.cpp:33-51):
 * z = [blocks][degree][E][cc][M], cc = ceil(capacity/degree), padded slots zero. */
int moe_op_encode(const void* x, int32_t dtype, int64_t blocks, int64_t T, int64_t M, int64_t E,
                  int64_t k, int64_t capacity, int64_t degree, const int32_t* idxs,
                  const int32_t* locations, void* z, void* stream);
/* fast_decode_range (dispatch.cpp:75-87) from the same chunked layout. */
int moe_op_decode(const void* z, int32_t dtype, int64_t blocks, int64_t T, int64_t M, int64_t E,
                  int64_t k, int64_t capacity, int64_t degree, const int32_t* idxs,
                  const int32_t* locations, const double* gates, void* y, void* stream);
/* fast_decode_backward_range (dispatch.cpp:136-157): dz chunked layout; dgates (blocks*T, k)
 * fp64 optional (needs z). */
int moe_op_decode_backward(const void* dy, const void* z, int32_t dtype, int64_t blocks,
                           int64_t T, int64_t M, int64_t E, int64_t k, int64_t capacity,
                           int64_t degree, const int32_t* idxs, const int32_t* locations,
                           const double* gates, void* dz, double* dgates, void* stream);
/* fast_encode_backward_range (dispatch.cpp:117-128). */
int moe_op_encode_backward(const void* dz, int32_t dtype, int64_t blocks, int64_t T, int64_t M,
                           int64_t E, int64_t k, int64_t capacity, int64_t degree,
                           const int32_t* idxs, const int32_t* locations, void* dx, void* stream);

/* expert_ffn (parallelism.cpp:103-121): x, y (n, rows, M); w1 (n, M, V); w2 (n, V, M);
 * act (n, rows, V) optional output (the saved relu activation). */
int moe_op_expert_ffn(const void* x, const void* w1, const void* w2, void* y, void* act,
                      int32_t dtype, int64_t n, int64_t rows, int64_t M, int64_t V, void* stream);
/* expert_ffn_backward (parallelism.cpp:123-147): dx (n, rows, M) in dtype; dw1 (n, M, V),
 * dw2 (n, V, M) fp32. */
int moe_op_expert_ffn_backward(const void* x, const void* w1, const void* w2, const void* dy,
                               void* dx, float* dw1, float* dw2, int32_t dtype, int64_t n,
                               int64_t rows, int64_t M, int64_t V, void* stream);

/* Raw grouped GEMM (kind: 0 up/relu, 1 down, 2 dgrad*mask, 3 dgrad, 4 wgrad), see
 * paper_2206_03382_b200/csrc/gemm_sm100.h for the addressing. use_tc=1 forces the tcgen05
 * kernel (bf16), 0 the SIMT kernel. */
int moe_op_gemm(int32_t kind, int32_t dtype, int32_t use_tc, const void* A, const void* B,
                void* D, const void* aux, int64_t G, int64_t S, int64_t seg_rows,
                int64_t seg_base, int64_t N, int64_t K, int64_t Mo, int64_t nseg_total,
                void* stream);

/* The ReLU certificate's weight statistics (bf16 path; no reference counterpart -- the fp64
 * reference needs no certificate): for n experts' w1 [n][M][V] bf16, colnorm [n][V] =
 * |w1[:, v]|_2 rounded up, colnorm_blk [n][V/64] = max over each 64-column block, w1t [n][V][M] =
 * w1 transposed. One pass over w1 when M % 64 == 0 and V % 64 == 0. */
int moe_op_weight_stats(const void* w1, int64_t n, int64_t M, int64_t V, float* colnorm,
                        float* colnorm_blk, void* w1t, void* stream);

/* Rng stream (core.cpp:66-83) on the device: dst[i] = lo + (hi-lo)*uniform(draw offset+i). */
int moe_op_fill_uniform(void* dst, int32_t dtype, int64_t n, uint64_t seed, uint64_t offset,
                        double lo, double hi, void* stream);

/* ---------------------------------------------------------------- Alg. 1 (pipeline.cpp:180-237)
 * Adaptive pipelining memo over the strategy space {Linear, TwoDH} x {1, 2, 4, 8} in
 * exploration order (pipeline.cpp:113-121); strategies are indices 0..7 into that order. */
typedef struct moe_memo moe_memo;
int moe_memo_create(double bucket_length, moe_memo** out);
int moe_memo_destroy(moe_memo* m);
int moe_memo_get_strategy(moe_memo* m, double f, int32_t* strategy);
int moe_memo_optimize_strategy(moe_memo* m, double f, int32_t strategy, double seconds);
int moe_memo_recompute_buckets(moe_memo* m, double f);
/* Bucket introspection: count, and (start, member count, members[...], table[8] with NaN for
 * unmeasured strategies) of bucket i. */
int moe_memo_num_buckets(moe_memo* m, int64_t* n);
int moe_memo_bucket(moe_memo* m, int64_t i, double* start, int64_t* n_members, double* members,
                    int64_t max_members, double* table8);
int moe_memo_lookup(moe_memo* m, double f, int32_t strategy, double* seconds, int32_t* present);

#ifdef __cplusplus
}
#endif

#endif /* MOE_B200_H */
