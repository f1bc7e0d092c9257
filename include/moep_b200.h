/* moep_b200.h — C ABI of the B200-native pre-attention expert predictor.
 *
 * Drop-in boundary for the hot path of the reference `moepredict` package
 * (arXiv 2511.10676). The reference has no FFI: its "operator API" is the
 * Python function surface listed in pkg/src/moepredict/__init__.py:5-118.
 * Each entry point below replaces the arithmetic behind one of those
 * functions; the Python package `paper_2511_10676_b200` binds them with
 * ctypes and keeps the reference's names, argument meaning and exceptions.
 *
 * Conventions (all entry points):
 *   - plain device pointers + explicit sizes, no torch types;
 *   - `stream` is a cudaStream_t passed as void*;
 *   - no allocation, no host synchronisation; scratch comes from the caller;
 *   - return 0 on success, a negative MOEP_E* code otherwise.
 * Layouts: row-major, bf16 = IEEE bfloat16 bit patterns (uint16).
 */
#ifndef MOEP_B200_H
#define MOEP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MOEP_OK = 0,
  MOEP_ESHAPE = -1,       /* inconsistent or unsupported dimensions       -> ConfigurationError */
  MOEP_EALIGN = -2,       /* pointer / stride alignment (TMA needs 16 B)  -> ConfigurationError */
  MOEP_EUNSUPPORTED = -3, /* configuration outside this kernel's envelope -> ValueError        */
  MOEP_ELAUNCH = -4,      /* CUDA launch / driver failure                 -> RuntimeError      */
  MOEP_EARG = -5          /* bad argument value (m out of range, ...)     -> ValueError        */
};

#define MOEP_MAX_BOUNDS 4

/* Counter block layout produced by the evaluation kernels (int64 after the
 * final reduce; int32 per-CTA partials before it):
 *   [0] n_rows  [1] top1  [2 .. 2+n_m) overprov[m]  [2+n_m .. 2+2n_m) recall[m]
 *   [2+2n_m .. +E) per_expert_hits   [2+2n_m+E .. +E) per_expert_truth
 * Replaces the integer core of metrics.evaluate_predictions (metrics.py:138-193). */
static inline int32_t moep_n_counters(int32_t n_m, int32_t n_experts) {
  return 2 + 2 * n_m + 2 * n_experts;
}

/* ------------------------------------------------------------------ K1 --
 * Fused predictor over bf16 activations: GEMM1 (tcgen05, fp32 TMEM) -> bias +
 * activation -> hi/lo bf16 split -> GEMM2 (tcgen05) -> +b2 -> per-token
 * top-m selection, near-tie margin flag, optional fused evaluation counters.
 * Replaces predictor.predict_logits / predict_topk_batch (predictor.py:330-351,
 * _forward_internal eval branch :193-240) and core.top_k_batch (core.py:42-48).
 * Tokens whose selection is not provably exact (margin < tau) are flagged and
 * appended to flag_list; moep_predict_fp64 must then be run on them. */
typedef struct {
  int64_t n_tokens;
  int32_t d, hidden, n_experts;
  int32_t arch;               /* 1: BN(eval)+GELU-tanh, 2: SiLU */
  const void* x;              /* [N, d] bf16 */
  const void* w1;             /* [hidden, d] bf16 */
  const float* b1;            /* [hidden] (arch2) */
  const float* act_alpha;     /* [hidden] arch1: folded BN scale/sqrt(var+eps) */
  const float* act_beta;      /* [hidden] arch1: folded shift - mean*alpha + b1*alpha */
  const void* w2;             /* [E, hidden] bf16 */
  const float* b2;            /* [E] */
  int32_t m_sel;              /* ids per token written to `ids` (0: none; <= 15 or == E) */
  int32_t n_bounds;           /* margin-check boundaries (positions), <= MOEP_MAX_BOUNDS */
  int32_t bounds[MOEP_MAX_BOUNDS];
  float tau_abs, tau_rel;     /* flag when gap < tau_abs + tau_rel*||h||*w2_norm; tau_rel is for the
                                 kernels with a separate lo-product accumulator (pair kernels, E <= 64
                                 in v4); the others widen it 1.5x (their measured error) */
  float w2_norm;              /* max_e ||w2[e,:]||_2 */
  int32_t* ids;               /* [N, m_sel] ascending, or NULL */
  float* logits;              /* [N, E] fp32, or NULL */
  uint8_t* flags;             /* [N], or NULL */
  int32_t* flag_list;         /* [N] compacted flagged rows */
  int32_t* flag_count;        /* [1] device counter (caller zeroes) */
  const int32_t* truth;       /* [N, k] true expert ids, or NULL (no evaluation) */
  int32_t k;
  int32_t n_m;
  int32_t m_list[MOEP_MAX_BOUNDS];
  int32_t* partials;          /* [moep_num_sms(), n_counters] int32 */
  float* a_out;               /* [N, hidden] fp32 pre-activation W1.x + b1 (training), or NULL */
  float* split_scratch;       /* hidden-split partial logits for small N (see below), or NULL */
  int64_t split_scratch_floats;
  int32_t* status;            /* [1] device word, or NULL: bit 0 is OR-ed in when a token's fp32
                                 logits are non-finite (such tokens are also flagged). The caller
                                 then checks the input for NaN/Inf, the reference's
                                 ConfigurationError (predictor.py:188-189), without a separate
                                 isfinite pass over x in the common case. */
  int32_t kernel;             /* MOEP_K1_AUTO (0) or a forced kernel (tests / measurements) */
  float* probs;               /* [N, E] fp32 softmax of the logits (core.softmax, core.py:19-24:
                                 exp(z - max) / sum, fused into the token epilogue), or NULL.
                                 From K1's fp32 logits for every row (flagged or not): each
                                 logit is within delta/2 of exact, so |p - p_ref| <= p_ref *
                                 (exp(delta) - 1) + 2^-22. */
} moep_predict_args;

enum { MOEP_K1_AUTO = 0, MOEP_K1_ONE_SM = 1, MOEP_K1_PAIR_V2 = 2, MOEP_K1_PAIR_V4 = 4, MOEP_K1_QUAD_V5 = 5 };

int moep_predict_bf16(const moep_predict_args* a, void* stream);

/* Scratch (floats) that lets moep_predict_bf16 split the hidden dimension
 * over CTA pairs when N is too small to fill the GPU with 256-token tiles
 * (partial logits per hidden group, summed in fixed order by a finish kernel
 * that runs the same selection / margin / counter epilogue). 0: no split for
 * this shape. Passing less than this in split_scratch_floats disables the split. */
int64_t moep_predict_split_floats(int64_t n_tokens, int32_t hidden, int32_t n_experts);

/* ------------------------------------------------------------------ K2 --
 * fp64 predictor on CUDA cores, mirroring the reference's float64 op order
 * per token (predictor.py:193-240, masked sigmoid :39-45). Runs on either all
 * rows (rows == NULL) or the rows listed in rows[0 .. *row_count).
 * Weights/activations may be bf16 or fp64 (dtype codes below). Writes fp64
 * logits, top-m ids, and evaluation partials for the rows it handles. */
enum { MOEP_BF16 = 1, MOEP_F64 = 2, MOEP_F32 = 3 };
typedef struct {
  int64_t n_tokens;
  int32_t d, hidden, n_experts;
  int32_t arch;
  int32_t x_dtype, w_dtype;   /* MOEP_BF16 or MOEP_F64 */
  const void* x;              /* [N, d] */
  const void* w1;             /* [hidden, d] */
  const double* b1;
  const double* bn_scale, *bn_shift, *bn_mean, *bn_var;  /* arch1 */
  double bn_eps;
  const void* w2;             /* [E, hidden] (informational; K2 reads w2t) */
  const void* w2t;            /* [hidden, E] transposed W2, same dtype as w2 */
  const double* b2;
  const int32_t* rows;        /* NULL = all rows */
  const int32_t* row_count;   /* device scalar when rows != NULL */
  int32_t m_sel;
  int32_t* ids;               /* [N, m_sel] or NULL */
  double* logits64;           /* [N, E] or NULL */
  float* logits32;            /* [N, E] or NULL (patched copy of K1 output) */
  const int32_t* truth; int32_t k; int32_t n_m; int32_t m_list[MOEP_MAX_BOUNDS];
  int32_t* partials;          /* [moep_num_sms(), n_counters] */
  double* a_out;              /* [N, hidden] fp64 pre-activation (training, exact mode), or NULL */
  int64_t row_begin;          /* first list index handled (rows mode) / first row (all rows) */
} moep_fp64_args;

int moep_predict_fp64(const moep_fp64_args* a, void* stream);

/* K2 fast path for the flagged rows (rows / row_count required): the rows in
 * rows[0 .. min(*row_count, capacity)) are recomputed in fp64 with
 * per-hidden-tile partial logits in `scratch`, by the split-hidden kernel of
 * moep_decode_fp64 when *row_count <= 256 and by a register-blocked fp64 GEMM
 * otherwise (decided on the device), then a per-token finish kernel; rows
 * beyond the capacity go through moep_predict_fp64 with their evaluation
 * partials in partials2 ([moep_num_sms(), n_counters]; written only when
 * capacity < N).
 * scratch: max(capacity * ceil(hidden/128), min(capacity, 256) * ceil(hidden/16)) * E doubles. */
int moep_fixup_fp64(const moep_fp64_args* a, double* scratch, int64_t capacity, int32_t* partials2,
                    void* stream);

/* Decode-batch predictor (serving: a few tokens per step), exact fp64 for all
 * N rows (rows must be NULL): the hidden dimension is split over
 * ceil(hidden/16) CTAs so the weight stream is spread over the whole GPU,
 * then the same finish kernel as the fix-up. Same outputs as
 * moep_predict_fp64 (predict_topk_batch, predictor.py:337-351).
 * scratch: N * ceil(hidden/16) * E doubles. No host synchronisation. */
int moep_decode_fp64(const moep_fp64_args* a, double* scratch, void* stream);

/* ------------------------------------------------------------------ K7 --
 * Evaluation / selection from given logits (fp64 or fp32), exact compares.
 * Replaces metrics.evaluate_predictions (metrics.py:138-193) and
 * core.top_k_batch (core.py:42-48) / rank_order (:51-54). */
int moep_eval_logits(const void* logits, int32_t dtype, int64_t n, int32_t n_experts,
                     const int32_t* truth, int32_t k, int32_t n_m, const int32_t* m_list,
                     int32_t* partials, void* stream);
int moep_topk_logits(const void* logits, int32_t dtype, int64_t n, int32_t n_experts, int32_t m,
                     int32_t* ids, void* stream);
/* Full stable descending order per row (core.rank_order, core.py:51-54). */
int moep_rank_order(const void* logits, int32_t dtype, int64_t n, int32_t n_experts, int32_t* order,
                    void* stream);
/* Deterministic sum of `n_blocks` int32 partial rows -> int64 counters. */
int moep_counters_reduce(const int32_t* partials, int32_t n_blocks, int32_t n_counters,
                         int64_t* out, void* stream);

/* ------------------------------------------------------------------ K0 --
 * Pre-attention input norm at the hook point (hooks.py:19,113-114; the
 * reference's norm is core.layer_norm, core.py:57-68), output rounded fp64 ->
 * bf16 RNE, bit-identical to numpy by construction: the statistics follow
 * numpy's pairwise reduction order and every element's bf16 rounding equals
 * that of numpy's (x - mean) / sqrt(var + eps) [* gamma] [+ beta] chain
 * (k0_norm.cu: a reciprocal multiply, with the exact chain for values near a
 * bf16 rounding midpoint).
 * kind: 0 none (cast), 1 rmsnorm(gamma, eps), 2 layernorm(gamma, beta, eps).
 * x dtype: MOEP_BF16, MOEP_F32 or MOEP_F64. bf16 rows with d in {512, 1024,
 * 2048, 4096} take the one-pass HBM-rate kernel; other shapes a general
 * kernel. Also reports non-finite input rows through status[0]
 * (ConfigurationError contract of predictor.py:188-189) and, for kind 0,
 * counts values that are not bf16-representable in status[1] (those inputs
 * take the fp64 path). status is int32[2], caller-zeroed. */
int moep_input_norm(const void* x, int32_t x_dtype, int64_t n, int32_t d, int32_t kind,
                    const double* gamma, const double* beta, double eps, void* xhat_bf16,
                    int32_t* status, void* stream);

/* ------------------------------------------------------------ training --
 * Every training entry point takes a dtype (MOEP_F64 or MOEP_F32) for its
 * floating-point buffers: MOEP_F64 is the exact-parity mode (reference
 * arithmetic in float64), MOEP_F32 the throughput mode (fp32 master weights,
 * bf16 tensor-core forward).
 *
 * K3: BatchLabels.from_scores (losses.py:64-74): 1-based stable ranks, top-k
 * mask, and per-token strict-pair counts among the true top-min(10,E). */
int moep_labels(const void* scores, int32_t dtype, int64_t n, int32_t n_experts, int32_t k,
                int32_t* rank_of, uint8_t* topk_mask, int32_t* pair_count, void* stream);

/* K4: loss_and_grad (losses.py:243-273). family: 0 mse, 1 wbce, 2 focal,
 * 3 ranking. Writes the per-element gradient (without the batch-global hinge
 * normaliser) to dz / dz_hinge and 3 fp64 partials per CTA {loss, hinge,
 * n_pairs}; moep_loss_finalize sums them in a fixed order (after an optional
 * cross-rank all-reduce of the partial sums) and completes dz and the loss
 * (out_loss[0] = loss, out_loss[1] = n_pairs).
 * n_global = tokens over all data-parallel ranks (the N of N*E, losses.py:129). */
typedef struct {
  int32_t family;
  double top_weight, mid_weight, rest_weight, ranking_lambda, margin, focal_gamma, focal_alpha;
  int32_t normalize_ranking;
  int64_t n, n_global;
  int32_t n_experts;
  int32_t dtype;              /* of logits / scores / dz / dz_hinge */
  const void* logits;         /* [n, E] */
  const void* scores;         /* [n, E] true affinity scores */
  const int32_t* rank_of;     /* [n, E] from moep_labels */
  const uint8_t* topk_mask;   /* [n, E] */
  void* dz;                   /* [n, E] out */
  void* dz_hinge;             /* [n, E] out (ranking) */
  double* partials;           /* [n_blocks, 3] out */
  int32_t n_blocks;
} moep_loss_args;
int moep_loss(const moep_loss_args* a, void* stream);
int moep_loss_finalize(const double* partials, int32_t n_blocks, int64_t n, int32_t n_experts,
                       int32_t family, double ranking_lambda, int32_t normalize, int32_t dtype,
                       void* dz, const void* dz_hinge, double* out_loss, void* stream);

/* K5: arch2 backward around the activation (predictor.py:261-297):
 * dA = (dZ . W2) * silu'(a); dW2 = dZ^T . silu(a); db1 = sum dA; db2 = sum dZ.
 * scratch: n_slices * (E*H + H + E) elements. dW1 = dA^T . X is a plain GEMM. */
int moep_act_backward(const void* a, const void* dz, const void* w2, int32_t dtype, int64_t n,
                      int32_t hidden, int32_t n_experts, int32_t n_slices, void* da, void* dw2,
                      void* db1, void* db2, void* scratch, void* stream);

/* K5, fp32 training mode: same as moep_act_backward (dtype fp32) but dA is
 * written as bf16: with_lo != 0: row i of da_hilo [n, 2*hidden] is
 * [hi = bf16(dA[i, :]) | lo = bf16(dA[i, :] - hi)] -- one bf16 tensor-core GEMM
 * C = da_hilo^T X ([2h, d], fp32) then gives dW1 = C[:h] + C[h:] (no fp32 dA
 * round trip through HBM, no duplicated X); with_lo == 0: da_hilo [n, hidden]
 * holds hi only (bf16 gradient operand, the "bf16" training precision). */
int moep_act_backward_bf16split(const float* a, const float* dz, const float* w2, int64_t n, int32_t hidden,
                                int32_t n_experts, int32_t n_slices, int32_t with_lo, void* da_hilo, float* dw2,
                                float* db1, float* db2, float* scratch, void* stream);

/* K6: optimizer step on a flat master buffer (trainer.py:103-122).
 * kind: 0 sgd, 1 momentum, 2 adam (bias-corrected with step t, 1-based).
 * The first n_shadow parameters are also written as bf16 (the forward copy)
 * when shadow_bf16 != NULL; *nonfinite counts CTAs that produced a non-finite
 * parameter (the NaN guard of trainer.py:125-128). */
typedef struct {
  int32_t kind;
  int32_t dtype;
  int64_t n;
  void* params;
  const void* grads;
  void* m;
  void* v;
  double lr, beta1, beta2, eps, momentum;
  int64_t t;
  void* shadow_bf16;
  int64_t n_shadow;
  int32_t* nonfinite;
} moep_optim_args;
int moep_optim_step(const moep_optim_args* a, void* stream);

/* arch1 training (fp64): batch-norm with batch statistics + running update,
 * GELU-tanh and Philox4x64-10 dropout identical to numpy's Generator.random
 * keyed (seed << 64) + step (predictor.py:70-72, 208-237); rows_dot is the
 * fp64 GEMM2 z = h . W^T + b; bn_backward is predictor.py:280-297. training = 0
 * gives the eval-mode forms (running statistics, no dropout, predictor.py:221-224, 292-296). */
int moep_bn_forward(const double* a, int64_t n, int32_t hidden, const double* scale, const double* shift,
                    double* run_mean, double* run_var, double momentum, double eps, double dropout_rate,
                    uint64_t dropout_seed, uint64_t dropout_step, const uint8_t* given_mask, double* a_hat,
                    double* bn_out, double* keep, double* h, double* inv_std, int32_t training, void* stream);
int moep_rows_dot(const double* h, const double* w, const double* b, int64_t n, int32_t hidden, int32_t n_out,
                  double* z, void* stream);
int moep_bn_backward(const double* dz, const double* w2, int64_t n, int32_t hidden, int32_t n_experts,
                     const double* h, const double* keep, const double* bn_out, const double* a_hat,
                     const double* inv_std, const double* scale, double* da, double* dw2, double* db1,
                     double* dscale, double* dshift, int32_t training, void* stream);

/* ----------------------------------------------------------------- K10 --
 * MOEPA1 trace records -> device arrays (synthgen.py:219-253 read_trace,
 * record invariants :123-145 TraceFile.validate). `records` holds n raw
 * little-endian records [d x f32 | E x f32 | k x u32] in device memory;
 * rows row0 .. row0+n-1 of acts ([*, d], fp32 or bf16 per act_dtype), scores
 * ([*, E] fp32) and topk ([*, k] int32) are written. status[6] (device,
 * caller-zeroed, accumulated across calls) counts failing records per check,
 * in the reference's order: non-finite activation, score outside [0, 1],
 * scores not summing to 1 within 1e-5, index >= E, row not strictly
 * increasing, stored top-k != top_k(scores, k). */
int moep_trace_ingest(const uint32_t* records, int64_t n, int32_t d, int32_t n_experts, int32_t k,
                      int32_t act_dtype, void* acts, float* scores, int32_t* topk, int64_t row0,
                      unsigned long long* status, void* stream);

/* ------------------------------------------------------------ prefetch --
 * K8: union of the predicted expert ids of a batch (ids[0 .. n_ids)), minus
 * experts already resident (slot_of[e] >= 0; NULL = none resident): ascending
 * need_list[0 .. *need_count), each paired with free_slots[i] (or -1 when the
 * cache is full). Replaces the per-token load set of pipesim.schedule's
 * prefetch modes (pipesim.py:272-305), which the reference only models. */
int moep_prefetch_plan(const int32_t* ids, int64_t n_ids, int32_t n_experts, const int32_t* slot_of,
                       const int32_t* free_slots, int32_t n_free, const int32_t* free_cursor, uint8_t* mask_out,
                       int32_t* need_list, int32_t* need_slot, int32_t* need_count, void* stream);
/* Residency update after a plan (device-only): slot_of[need_list[i]] =
 * need_slot[i] for every assigned entry, *free_cursor += their number (the
 * plan takes free slots from free_slots[*free_cursor ..]; NULL cursor = 0).
 * plan -> K9 gather -> commit then runs with no host round trip. */
int moep_prefetch_commit(const int32_t* need_list, const int32_t* need_slot, const int32_t* need_count,
                         int32_t* slot_of, int32_t* free_cursor, void* stream);
/* K9: GPU-driven copy of the listed experts from mapped pinned host memory
 * (expert e at host_mapped_store + e*expert_bytes) into cache slots. */
int moep_gather_experts(const void* host_mapped_store, int64_t expert_bytes, const int32_t* need_list,
                        const int32_t* need_slot, const int32_t* need_count, void* cache, int32_t n_ctas,
                        void* stream);

/* ------------------------------------------------------------------ K11 --
 * Synthetic teacher (synthgen.py:162-189). Sample first_index+i draws from
 * numpy.random.Generator(Philox(key=(seed << 64) + first_index + i))
 * (synthgen.py:44-47): d standard normals into row i of x64 (fp64) and/or x32
 * (fp32 cast), then, with with_noise, d more into noise64 (synthgen.py:170-174).
 * Normals follow numpy's ziggurat (random_standard_normal). */
int moep_teacher_normals(uint64_t seed, int64_t first_index, int64_t n, int32_t d, int32_t with_noise,
                         double* x64, float* x32, double* noise64, void* stream);
/* core.layer_norm (core.py:57-68) row-wise over [n, d] fp64 with numpy's
 * reduction order (0 + pairwise_sum) and single roundings: bit-identical to
 * numpy. out may alias x. */
/* fp64 GEMM on the fp64 tensor cores: C[M, N] = epi(A[M, K] . B[N, K]^T),
 * row-major with leading dimensions, epi 0 = identity, 1 = tanh. The
 * teacher's dense maps (synthgen.py:176-189: mix, tanh(W_in x), W_out, gate). */
int moep_dgemm_nt(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                  int64_t M, int64_t N, int64_t K, int32_t epilogue, void* stream);
/* C[M, N] = A[K, M]^T . B[K, N] in fp64 on the fp64 tensor cores (the fp64
 * training mode's dW1 = dA^T X, predictor.py:295). */
int moep_dgemm_tn(const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                  int64_t M, int64_t N, int64_t K, void* stream);
/* dW1 of the tensor-core training modes (predictor.py:295) on tcgen05:
 * dw1[h, d] = sum_n dA[n, p*h + j] X[n, i] summed over the p < passes column
 * blocks of dA (passes 2: the fp32 mode's bf16 hi | lo halves), fp32 out.
 * dA [n, passes*h] and X [n, d] bf16 row-major (token-major). workspace:
 * moep_dw1_workspace_floats(...) floats for the K-split partials (0: none
 * needed; too small a workspace disables the split). */
int64_t moep_dw1_workspace_floats(int32_t hidden, int32_t d, int64_t n_tokens, int32_t passes);
int moep_dw1_bf16(const void* da, const void* x, int64_t n_tokens, int32_t hidden, int32_t d, int32_t passes,
                  float* dw1, float* workspace, int64_t workspace_floats, void* stream);
int moep_layer_norm_np(const double* x, int64_t n, int32_t d, double eps, double* out, void* stream);
/* core.softmax (core.py:19-24) over the rows of an fp64 [n, E] array in
 * numpy's order (max, exp, 0 + pairwise_sum, divide); out may alias z. */
int moep_softmax_np(const double* z, int64_t n, int32_t E, double* out, void* stream);
/* gate softmax (core.py:19-24) of fp64 logits [n, E] in numpy order, float32
 * scores [n, E] and ascending top-k ids [n, k] of the float32 scores
 * (make_dataset, synthgen.py:148-159; core.py:42-48). E <= 256. */
int moep_teacher_finish(const double* logits, int64_t n, int32_t n_experts, int32_t k, float* scores,
                        int32_t* topk, void* stream);

/* ---------------------------------------------------------------- misc -- */
int moep_num_sms(void);
const char* moep_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MOEP_B200_H */
