/*
 * sparsegate-b200 — C ABI of the B200-native sparse gated-FFN decode executor.
 *
 * Drop-in boundary for the reference executor API
 *   /root/reference/proj/include/sparsegate/ffn_exec.hpp (namespace sparsegate):
 *     dense_ffn              ffn_exec.hpp:103-122   -> sg_ffn_forward(..., SG_PIPELINE_DENSE, ...)
 *     predict_mask           ffn_exec.hpp:125-146   -> sg_predict_mask
 *     sparse_ffn_parallel    ffn_exec.hpp:149-178   -> sg_ffn_forward(..., SG_PIPELINE_PARALLEL, ...)
 *     sparse_ffn_sequential  ffn_exec.hpp:183-218   -> sg_ffn_forward(..., SG_PIPELINE_SEQUENTIAL, ...)
 *     op_count_model         ffn_exec.hpp:229-244   -> sg_op_count_model (pure host)
 *   with the data contract of types.hpp:21-105 (FfnWeights, Predictor, validate) and
 *   the error taxonomy of common.hpp:20-37 (IoError / DataError / PropertyViolation)
 *   mapped onto sg_status (CLI exit-code convention, tools/sparsegate_main.cpp:5).
 *
 * The reference functions are stateless and take f64 Eigen objects; a GPU
 * executor needs resident weights, so the ABI splits each call into
 *   sg_layer_create  (upload + validate ONCE; types.hpp:31-51 / :82-105 run here,
 *                     not on every call as ffn_exec.hpp:57 / :126 do)
 *   sg_ctx_create    (per-stream workspace; one per concurrently used stream/thread,
 *                     which gives the reference's reentrancy)
 *   sg_ffn_forward*  (the executor call).
 * Plain pointers and sizes only; cudaStream_t is passed as void*.
 * All functions are thread-safe for distinct sg_ctx objects.
 */
#ifndef SPARSEGATE_C_H_
#define SPARSEGATE_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sg_status {
  SG_OK = 0,
  SG_ERR_USAGE = 1,    /* bad arguments (CLI exit 1)                               */
  SG_ERR_DATA = 2,     /* DataError: shapes, non-finite x / weights (common.hpp:30) */
  SG_ERR_PROPERTY = 3, /* PropertyViolation (common.hpp:35)                        */
  SG_ERR_IO = 4,       /* IoError (common.hpp:25)                                  */
  SG_ERR_CUDA = 5,     /* CUDA runtime failure (no reference counterpart)          */
  SG_ERR_NCCL = 6      /* NCCL failure (no reference counterpart)                  */
} sg_status;

typedef enum sg_activation { SG_REGLU = 0, SG_DRELU = 1 } sg_activation; /* types.hpp:12 */

/* Same order as sparsegate::Pipeline (ffn_exec.hpp:32). */
typedef enum sg_pipeline {
  SG_PIPELINE_DENSE = 0,
  SG_PIPELINE_PARALLEL = 1,
  SG_PIPELINE_SEQUENTIAL = 2
} sg_pipeline;

typedef enum sg_dtype { SG_F64 = 0, SG_F32 = 1, SG_BF16 = 2 } sg_dtype;

/* sparsegate::ExecStats (ffn_exec.hpp:35-40), computed exactly as ffn_exec.hpp:120,
 * :173-180, :209-216 from the device-side counts; plus the counts themselves. */
typedef struct sg_exec_stats {
  double predicted_sparsity;
  double realized_sparsity;
  int64_t multiplies;
  int32_t pipeline;
  int32_t pad_;
  int64_t predicted_active; /* |P| */
  int64_t revalidated;      /* |V| (gate survivors) */
} sg_exec_stats;

/* One FFN layer (or one shard of it) plus its predictor, in the REFERENCE layouts:
 *   gate, up : inter x hidden  row-major   (types.hpp:19-24)
 *   down     : hidden x inter  row-major   (transposed to neuron-major on upload)
 *   pred_A   : inter x rank    row-major   (types.hpp:72-76)
 *   pred_B   : rank x hidden   row-major
 *   bias     : inter, f64 or f32 (+inf allowed, types.hpp:99-101)
 * Host arrays; dtype `weight_dtype` for gate/up/down/A/B (f64/f32 are rounded
 * f64->f32->bf16 RNE; bf16 arrays are uint16 bit patterns), `bias_dtype` for bias.
 * pred_A/pred_B/bias may all be NULL for a dense-only layer (rank ignored);
 * gate/up/down may all be NULL for a predictor-only layer (sg_predict_mask only).
 *
 * Sharding: the layer keeps neurons {shard_index + k*shard_count}
 * when shard_interleave != 0, else the contiguous block shard_index of
 * shard_count near-equal blocks. The arrays always describe the FULL layer. */
typedef struct sg_layer_desc {
  int64_t hidden;
  int64_t inter;
  int64_t rank;
  int32_t activation;   /* sg_activation */
  int32_t weight_dtype; /* sg_dtype */
  int32_t bias_dtype;   /* sg_dtype (SG_F64 or SG_F32) */
  int32_t device;       /* CUDA device ordinal */
  const void* gate;
  const void* up;
  const void* down;
  const void* pred_A;
  const void* pred_B;
  const void* bias;
  int32_t shard_index;
  int32_t shard_count; /* 0 or 1 = unsharded */
  int32_t shard_interleave;
  int32_t down_neuron_major; /* 1: `down` is already inter x hidden (neuron-major) */
  /* Optional device layout order of the neurons (a permutation of 0..inter-1, or
   * NULL = ascending). The executor gives CTA c the c-th contiguous block of the
   * layout, so an order built from offline activity statistics (the calibrated
   * predictor's hot / cold neurons) balances the per-CTA work. Results are the
   * same function of the data; the summation order of y follows the layout.
   * Index sets (sg_ctx_read_sets) are still reported ascending in GLOBAL indices;
   * sg_predict_mask's mask and sg_layer_global_index use the local (layout) index. */
  const int64_t* neuron_order;
} sg_layer_desc;

typedef struct sg_layer sg_layer;
typedef struct sg_ctx sg_ctx;

/* Last error message of the calling thread ("" if none). */
const char* sg_last_error(void);
/* Library version string. */
const char* sg_version(void);

sg_status sg_layer_create(const sg_layer_desc* desc, sg_layer** out);
sg_status sg_layer_destroy(sg_layer* layer);
/* Local (shard) neuron count, and the global index of local neuron k. */
int64_t sg_layer_local_inter(const sg_layer* layer);
int64_t sg_layer_global_index(const sg_layer* layer, int64_t local);
/* Device bytes held by the layer's resident weights. */
int64_t sg_layer_device_bytes(const sg_layer* layer);
/* Gate-row prefetch ahead of the predictor (sequential pipeline): the first `rows`
 * neurons of every CTA block of the layout have their gate rows fetched as soon as
 * the layer starts, overlapping stages 1a/1b; those that the mask then rejects are
 * dropped unread. Meant for a neuron_order that puts each block's most frequently
 * predicted neurons first. 0 (default) disables; capped by the free ring slots.
 * Results do not depend on it (it changes only when rows arrive and the order in
 * which a CTA's survivors are summed). */
sg_status sg_layer_set_hot_rows(sg_layer* layer, int64_t rows);

/* Workspace for one stream. max_hidden/max_inter/max_rank bound the layers it
 * will run; device = CUDA ordinal. */
sg_status sg_ctx_create(int32_t device, int64_t max_hidden, int64_t max_inter, int64_t max_rank,
                        sg_ctx** out);
sg_status sg_ctx_destroy(sg_ctx* ctx);

/* Executor, device buffers, asynchronous on `stream` (cudaStream_t; NULL = legacy
 * default). x: fp32[hidden] (device). y: fp32[hidden] (device) receives this
 * layer's (shard's) output. No host synchronisation; stats and index sets stay in
 * the ctx until sg_ctx_read_* is called. A non-finite x is flagged on device and
 * reported by sg_ctx_read_stats as SG_ERR_DATA (ffn_exec.hpp:61-63). */
sg_status sg_ffn_forward_device(sg_ctx* ctx, const sg_layer* layer, sg_pipeline pipeline,
                                const float* x, float* y, void* stream);

/* Synchronises `stream`, then copies the last call's stats (computed with the
 * reference formulas) to host. Returns SG_ERR_DATA if that call saw non-finite x. */
sg_status sg_ctx_read_stats(sg_ctx* ctx, void* stream, sg_exec_stats* stats);

/* Synchronises, then copies the last call's index sets (GLOBAL neuron indices,
 * ascending): P (predicted active, capacity >= local inter), V (gate survivors),
 * and optionally g (fp32 gate pre-activation per P entry) and z (fp32 gated value
 * per V entry). Any pointer may be NULL. */
sg_status sg_ctx_read_sets(sg_ctx* ctx, void* stream, int32_t* P, int64_t* p, int32_t* V,
                           int64_t* v, float* g, float* z);

/* Predictor only (stage 1): mask[local inter] bytes and count, host outputs.
 * ffn_exec.hpp:125-146. x: host, dtype x_dtype (SG_F64 / SG_F32), length x_len. */
sg_status sg_predict_mask(sg_ctx* ctx, const sg_layer* layer, const void* x, sg_dtype x_dtype,
                          int64_t x_len, uint8_t* mask, int64_t* count, void* stream);

/* Host-facing executor = the reference call shape: host x in, host y out
 * (x_dtype/y_dtype SG_F64 or SG_F32), stats out (may be NULL). Validates x on
 * host (length, finiteness -> SG_ERR_DATA), copies H2D through pinned staging,
 * runs sg_ffn_forward_device, copies y D2H, synchronises. */
sg_status sg_ffn_forward(sg_ctx* ctx, const sg_layer* layer, sg_pipeline pipeline, const void* x,
                         sg_dtype x_dtype, int64_t x_len, void* y, sg_dtype y_dtype,
                         sg_exec_stats* stats, void* stream);

/* Multi-layer decode step on device: runs layers[0..n) in order on `stream`,
 * layer l reading xs + l*hidden and writing ys + l*hidden (fp32, device).
 *   chain 0: layer l reads xs_l (independent layers);
 *   chain 1: layer l+1 reads layer l's output y_l (a raw decode chain);
 *   chain 2: layer l+1 reads xs_{l+1} + y_l (fp32 add: the residual-stream
 *            dependency of a decoder block, h_{l+1} + FFN_l(x_l)).
 * With chain 1 or 2, layer l+1 cannot start before every value of y_l exists. */
sg_status sg_ffn_forward_layers(sg_ctx* ctx, const sg_layer* const* layers, int32_t n,
                                sg_pipeline pipeline, const float* xs, float* ys, int32_t chain,
                                void* stream);

/* Host-buffer variant of sg_ffn_forward_layers (the end-to-end call shape):
 * copies xs_host (n*hidden fp32) H2D, runs the stack, copies ys_host back and
 * synchronises. stats (n entries, may be NULL) gets each layer's ExecStats. */
sg_status sg_ffn_forward_layers_host(sg_ctx* ctx, const sg_layer* const* layers, int32_t n,
                                     sg_pipeline pipeline, const float* xs_host, float* ys_host,
                                     int32_t chain, sg_exec_stats* stats, void* stream);

/* Synchronises, then returns per-layer stats of the last sg_ffn_forward_layers* call. */
sg_status sg_ctx_read_stack_stats(sg_ctx* ctx, void* stream, int32_t n, sg_exec_stats* stats);

/* Per-layer index sets of stack calls (diagnostics / parity): with enable != 0,
 * every later sg_ffn_forward_layers* call of at most 64 layers also records, per
 * local neuron, bit l = "predicted active in layer l" and "survivor in layer l"
 * (integer atomics; the computed outputs are unchanged). sg_ctx_read_stack_sets
 * synchronises and returns layer `layer`'s P and V of the last such call as
 * ascending GLOBAL indices (capacity >= local inter each; either may be NULL). */
sg_status sg_ctx_enable_stack_sets(sg_ctx* ctx, int32_t enable);
sg_status sg_ctx_read_stack_sets(sg_ctx* ctx, void* stream, int32_t layer, int32_t* P, int64_t* p,
                                 int32_t* V, int64_t* v);

/* Batched decode (BASELINE.json configs[4]): `batch` (1..64) tokens through one
 * layer, sequential pipeline. Each token gets exactly its own single-token
 * result (its P_b, V_b, y_b, ExecStats); the batch reads each gate row of the
 * union of the P_b and each [up | down] row of the union of the V_b once, on the
 * tensor cores. xs, ys: device fp32 [batch][hidden]. Asynchronous on `stream`. */
sg_status sg_ffn_forward_batch(sg_ctx* ctx, const sg_layer* layer, const float* xs, int32_t batch,
                               float* ys, void* stream);
/* Dense comparator of the batched path (no predictor: every gate, up and down row
 * is read once and multiplied against all tokens) on the same tensor-core kernel:
 * dense_ffn (ffn_exec.hpp:103-122) per token, batched. xs, ys: device fp32
 * [batch][hidden], batch in [1, 64]. */
sg_status sg_ffn_forward_batch_dense(sg_ctx* ctx, const sg_layer* layer, const float* xs,
                                     int32_t batch, float* ys, void* stream);
/* Batched decode of a residual stream: token b's input is xs_b + xres_b (summed in
 * fp32 inside the launch, e.g. h_{l+1} + y_l between two FFN layers); xres may be
 * NULL. dense != 0 runs the dense comparator. `next` / `next_xs` (optional): the call
 * that follows on this ctx will be on layer `next` with input next_xs + ys (next_xs
 * may be NULL: input ys) — this launch's y finishers then also write that launch's
 * bf16 hi/lo X^T, so it starts with no x split (results unchanged; a different next
 * call simply splits its x itself). Tensor-core path only (hidden <= 8192, rank <= 256). */
sg_status sg_ffn_forward_batch_res(sg_ctx* ctx, const sg_layer* layer, const float* xs, const float* xres,
                                   int32_t batch, float* ys, int32_t dense, const sg_layer* next,
                                   const float* next_xs, void* stream);
/* Diagnostics of the tensor-core batch kernel: with max_units > 0, later batched calls
 * record per work unit 8 values (%globaltimer ns: claim, inputs ready, loads issued,
 * epilogue start / end; the SM id; two epilogue-internal stamps: partial written,
 * group arrival counted); read_tc_trace copies the last call's
 * (min(max_units, its unit count)) records of 8 uint64 and the unit count. */
sg_status sg_ctx_enable_tc_trace(sg_ctx* ctx, int32_t max_units);
sg_status sg_ctx_read_tc_trace(sg_ctx* ctx, void* stream, int32_t max_units, uint64_t* out,
                               int32_t* n_units);
/* The last tensor-core call's unit claim order: type << 24 | i << 8 | j per unit. */
sg_status sg_tc_unit_codes(sg_ctx* ctx, int32_t* out, int32_t max_units);
/* Synchronises, then per-token stats (batch entries) and, optionally, per-neuron
 * bit masks (local inter entries; bit b = token b): predicted active, survivor. */
sg_status sg_ctx_read_batch(sg_ctx* ctx, void* stream, int32_t batch, sg_exec_stats* stats,
                            uint64_t* pred_bits, uint64_t* surv_bits);
/* Host-buffer variant: fp32 xs_host [batch][hidden] in, ys_host out, stats (may be NULL). */
sg_status sg_ffn_forward_batch_host(sg_ctx* ctx, const sg_layer* layer, const float* xs_host,
                                    int32_t batch, float* ys_host, sg_exec_stats* stats,
                                    void* stream);

/* Diagnostics: record per-CTA %globaltimer stamps at every phase boundary of
 * the executor (up to 32 stamps per CTA per layer) for up to
 * max_layers layers of each subsequent call; max_layers = 0 disables. */
sg_status sg_ctx_enable_phase_timing(sg_ctx* ctx, int32_t max_layers);
/* Synchronises and copies n_layers x num_ctas x 32 stamps (ns); *num_ctas = grid size. */
sg_status sg_ctx_read_phase_timing(sg_ctx* ctx, void* stream, int32_t n_layers, uint64_t* out,
                                   int32_t* num_ctas);

/* ffn_exec.hpp:229-244, pure host. */
sg_status sg_op_count_model(int64_t d, int64_t D, int64_t r, double s, double s_prime,
                            int64_t* dense, double* sparse, double* ratio);

/* Host rounding used on upload: f64 -> f32 (RNE) -> bf16 (RNE), NaN-preserving. */
void sg_round_bf16(const double* in, uint16_t* out, int64_t n);

/* ---- multi-GPU: the d_ff-sharded decode step ----
 * One process per GPU; every rank creates its shard of every layer
 * (sg_layer_desc.shard_index / shard_count) and joins one communicator. A step runs
 * each layer on the rank's shard and sums the d-sized partial outputs over ranks
 * with one NCCL all-reduce per layer, all issued from C++ on `stream` (capturable
 * in one CUDA graph). NCCL is loaded with dlopen("libnccl.so.2"). */
typedef struct sg_comm sg_comm;
/* 128-byte NCCL unique id, created on one rank and shared with the others. */
sg_status sg_comm_unique_id(void* id128);
sg_status sg_comm_create(int32_t device, int32_t nranks, int32_t rank, const void* id128, sg_comm** out);
sg_status sg_comm_destroy(sg_comm* comm);
int32_t sg_comm_size(const sg_comm* comm);
int32_t sg_comm_rank(const sg_comm* comm);
/* In-place sum of `count` fp32 values over the ranks of `comm`. */
sg_status sg_allreduce_sum(sg_comm* comm, float* buf, int64_t count, void* stream);
/* Sharded multi-layer step: same xs / ys / chain semantics as sg_ffn_forward_layers
 * (ys receives the WHOLE layer outputs on every rank); per-layer stats of the rank's
 * shard via sg_ctx_read_stack_stats (sum |P|, |V| over ranks for the whole layer). */
sg_status sg_ffn_forward_layers_sharded(sg_ctx* ctx, sg_comm* comm, const sg_layer* const* layers,
                                        int32_t n, sg_pipeline pipeline, const float* xs, float* ys,
                                        int32_t chain, void* stream);
/* Hidden size of a layer. */
int64_t sg_layer_hidden(const sg_layer* layer);

/* ---- multi-GPU sharding, pure host ----
 * The neuron set a shard holds: global index of local k = base + k*stride,
 * k in [0, count). Exactly the mapping sg_layer_create applies. */
sg_status sg_shard_range(int64_t inter, int32_t shard_index, int32_t shard_count,
                         int32_t shard_interleave, int64_t* base, int64_t* stride, int64_t* count);

/* ExecStats of the WHOLE layer from counts summed over shards (|P|, |V|), with the
 * reference formulas of ffn_exec.hpp:120, :173-180, :209-216 over the global
 * inter. (A single shard's sg_ctx_read_stats reports its local inter.) */
sg_status sg_exec_stats_from_counts(int64_t hidden, int64_t inter, int64_t rank,
                                    sg_pipeline pipeline, int64_t predicted_active,
                                    int64_t revalidated, sg_exec_stats* out);

/* ---- host-side producers of the executor's inputs (not on the device path) ---- */

/* synthetic.hpp:80-108 (make_synthetic_fixture), same mt19937_64 stream order.
 * Outputs (any NULL to skip; the stream is still drawn): gate/up inter x hidden,
 * down hidden x inter, calib hidden x calib_tokens, eval hidden x eval_tokens,
 * all f64 row-major. */
sg_status sg_synthetic_fixture(int64_t hidden, int64_t inter, int64_t calib_tokens,
                               int64_t eval_tokens, double natural_sparsity, uint64_t seed,
                               double* gate, double* up, double* down, double* calib,
                               double* eval);

/* Same stream, but weights are emitted directly as bf16 (f64->f32->bf16), down
 * already transposed to neuron-major (inter x hidden), tokens as f64. Used to
 * build multi-layer bench models without holding f64 weights. */
sg_status sg_synthetic_fixture_bf16(int64_t hidden, int64_t inter, int64_t calib_tokens,
                                    int64_t eval_tokens, double natural_sparsity, uint64_t seed,
                                    uint16_t* gate, uint16_t* up, uint16_t* down_t,
                                    double* calib, double* eval);

/* calibration.hpp:61-96 + :128-205 (build_instance + greedy_calibrate): scores and
 * weights are inter x T row-major f64; writes bias[inter] (+inf where the pointer
 * stayed at 0), and the achieved sparsity. */
sg_status sg_greedy_calibrate(const double* scores, const double* weights, int64_t inter,
                              int64_t T, int32_t eta, double target_sparsity, double* bias,
                              double* achieved_sparsity, double* total_damage);

/* ---- offline producer (csrc/sg_offline.cu): the predictor
 * factors and calibration inputs in C++ without Eigen, large products on the GPU
 * (current device). All arrays row-major f64 host buffers.
 * svd_mode: 0 = exact (one-sided Jacobi, host; small shapes), 1 = randomized
 * (range finder of width k + 8, 2 power iterations, CholeskyQR2 on the GPU). */

/* predict_mask (ffn_exec.hpp:125-146) in f64 on the GPU, bit-identical to the
 * reference: t = B x and pre = A t + bias with common.hpp's det_dot reduction order
 * (blocked 64, balanced tree, no FMA contraction); mask[i] = pre_i > 0 strictly.
 * Host arrays (A inter x rank, B rank x hidden, bias inter, x hidden; row-major f64).
 * The executors' own masks use the bf16 predictor of the layer. */
sg_status sg_predict_mask_f64(int32_t device, const double* A, const double* B, const double* bias,
                              int64_t inter, int64_t rank, int64_t hidden, const double* x,
                              uint8_t* mask, int64_t* count);

/* factorization.hpp:31-64: S = chol(X X^T + lambda I) (d x d lower) and S^-1, with the
 * damping ladder lambda = multipliers[k] * epsilon * trace(X X^T) / d tried in order;
 * X is d x T (hidden x tokens). SG_ERR_DATA when every rung fails. */
sg_status sg_cholesky_whitening(const double* X, int64_t d, int64_t T, double epsilon,
                                const double* multipliers, int32_t n_mult, double* S, double* S_inv,
                                double* lambda);
/* factorization.hpp:93-144: A (D x rank) = U_r diag(s_r), B (rank x d) = V_r^T [S^-1] from
 * the SVD of W S (whitened != 0) or W; sv receives the first n_sv singular values of
 * that target, sigma_r1 = sigma_{rank+1}(W), lambda the damping used. */
sg_status sg_build_predictor(const double* W, int64_t D, int64_t d, const double* X, int64_t T,
                             int64_t rank, int32_t whitened, int32_t svd_mode, uint64_t seed,
                             double epsilon, const double* multipliers, int32_t n_mult, double* A,
                             double* B, double* sv, int64_t n_sv, double* sigma_r1, double* lambda);
/* The k largest singular values of M (rows x cols). */
sg_status sg_singular_values(const double* M, int64_t rows, int64_t cols, int32_t svd_mode, int64_t k,
                             uint64_t seed, double* out);
/* calibration.hpp:39-46: scores (D x T) = A (B X). */
sg_status sg_proxy_scores(const double* A, const double* B, int64_t D, int64_t r, int64_t d,
                          const double* X, int64_t T, double* scores);
/* calibration.hpp:20-37: weights (D x T) = (act(gate X) * up'(X))^2 * |down column|^2. */
sg_status sg_damage_weights(const double* gate, const double* up, const double* down, int64_t D,
                            int64_t d, int32_t activation, const double* X, int64_t T, double* weights);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* SPARSEGATE_C_H_ */
