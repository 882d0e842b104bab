/*
 * prorl_hotpath.h — C-ABI of the B200 (sm_100a) trainer-side scoring path for
 * ProRL Agent (arXiv 2603.18815): pack -> logprob/entropy -> GRPO advantage ->
 * DAPO clipped surrogate + per-turn metrics -> NCCL all-reduce of partials.
 *
 * The reference has no operator/FFI surface for this math; the
 * drop-in surface it does own is the C++ trainer API.  Each entry point below
 * names the reference interface it replaces or extends:
 *
 *   prorl_pack            extends  TokenTrajectory::flatten/flatten_range
 *                                  (proj/include/rollout/trajectory.hpp:76-87,
 *                                  role->mask rule at :82-83) and the id/logprob
 *                                  fields of Turn (trajectory.hpp:27-33, types.hpp:12)
 *   prorl_grpo_adv        extends  PromptGroup::usable_rewards + is_informative
 *                                  (proj/src/trainer/harness.cpp:84-102)
 *   prorl_logprob_entropy new      (absent in reference: SPEC.md:8)
 *   prorl_clipped_loss    new      (absent in reference: SPEC.md:741; DAPO PAPER.md:368)
 *   prorl_score_rows      new      K2+K4 fused (same sources as the two above)
 *   prorl_logits_grad     new      backward of the DAPO surrogate
 *                                  through the log-softmax (SURVEY §8 f rank 1)
 *   prorl_score_grad      new      score_rows + logits_grad in one kernel (K7)
 *   prorl_lmhead_logprob  new      fused LM head + logprob (SURVEY §8 f rank 2;
 *                                  the model forward is outside SPEC.md:8)
 *   prorl_ingest_responses replaces the response parse that drops the
 *                                  trajectory (proj/src/trainer/harness.cpp:
 *                                  254-273), schema of proj/src/handlers.cpp:57-91
 *   prorl_synth_rewards   restates generate_workload (proj/src/trainer/workload.cpp:62-107)
 *   prorl_allreduce       new      (the reference has no collectives)
 *   prorl_score_host      replaces the trajectory drop at
 *                                  proj/src/trainer/harness.cpp:263-273 — the
 *                                  whole per-GPU step from host SoA buffers.
 *
 * Conventions:
 *   - every function returns 0 (PRORL_OK) or a negative prorl_status; the
 *     message is in prorl_last_error() (thread-local);
 *   - negative codes map 1:1 onto rollout::Error codes (errors.hpp:10-59) plus
 *     four new ones (cuda_error, nccl_error, shape_mismatch, peer_failed);
 *   - buffers are caller-owned device memory unless a name says host_; the
 *     library only owns the workspace inside a ctx;
 *   - all device work is stream-ordered on the stream argument, no implicit
 *     device synchronisation (prorl_score_host and prorl_check_errors are the
 *     documented exceptions: they synchronise their stream);
 *   - one ctx per device; calls on distinct ctxs are thread-safe.
 */
#ifndef PRORL_HOTPATH_H
#define PRORL_HOTPATH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRORL_ABI_VERSION 2  /* 2: prorl_score_cfg.gate_tolerance; advantages fp64 */

typedef enum prorl_status {
  PRORL_OK = 0,
  PRORL_E_MALFORMED_TURN = -1,    /* rollout::MalformedTurn   "malformed_turn"   */
  PRORL_E_INCOMPLETE_GROUP = -2,  /* rollout::IncompleteGroup "incomplete_group" */
  PRORL_E_MALFORMED_REQUEST = -3, /* rollout::MalformedRequest "malformed_request" */
  PRORL_E_CUDA = -10,             /* new: "cuda_error"      */
  PRORL_E_NCCL = -11,             /* new: "nccl_error"      */
  PRORL_E_SHAPE = -12,            /* new: "shape_mismatch"  */
  PRORL_E_TOKEN_RANGE = -13,      /* new: "shape_mismatch" (token id outside [0,V)) */
  PRORL_E_PEER_FAILED = -14,      /* new: "peer_failed" — another rank's step failed (see prorl_score_host) */
} prorl_status;

typedef enum prorl_dtype { PRORL_BF16 = 0, PRORL_FP32 = 1 } prorl_dtype;

/* rollout::Role order (trajectory.hpp:11). */
enum { PRORL_ROLE_SYSTEM = 0, PRORL_ROLE_USER = 1, PRORL_ROLE_ASSISTANT = 2, PRORL_ROLE_TOOL = 3 };

/* Number of per-turn metric buckets and the partials layout. */
#define PRORL_TURN_BUCKETS 64
#define PRORL_N_GLOBAL 12
#define PRORL_N_PER_TURN 5
#define PRORL_N_PARTIALS (PRORL_N_GLOBAL + PRORL_TURN_BUCKETS * PRORL_N_PER_TURN) /* 332 */
enum {
  PRORL_P_LOSS_SUM = 0, PRORL_P_N_ACTIVE = 1, PRORL_P_ENTROPY_SUM = 2, PRORL_P_LOGP_SUM = 3,
  PRORL_P_RATIO_SUM = 4, PRORL_P_CLIP_LO = 5, PRORL_P_CLIP_HI = 6, PRORL_P_KL1_SUM = 7,
  PRORL_P_ADV_SUM = 8, PRORL_P_N_ROLLOUTS = 9, PRORL_P_KL_SUM = 10, /* sum of k3 KL vs the reference policy */
  PRORL_P_ERR_RANKS = 11 /* ranks whose step failed (0 on success); summed by the all-reduce */
};
/* per-turn bucket k starts at PRORL_N_GLOBAL + 5*k: [N_k, loss_k, H_k, logp_k, clip_k] */

typedef struct prorl_ctx prorl_ctx;

/* One turn descriptor. Turns are listed in trajectory order, trajectories in
 * ascending `traj` (the rollout index inside the shard, = seq id). `src_off`
 * indexes the flat wire arrays (ids, logprobs) passed alongside. */
typedef struct prorl_turn_desc {
  int64_t src_off;
  int32_t traj;
  int32_t len;
  uint8_t role; /* PRORL_ROLE_* */
  uint8_t pad_[7];
} prorl_turn_desc;

/* Packed outputs (device pointers, caller-owned). Sizes: N = total tokens,
 * n_seq = number of trajectories (rollout slots), A = active rows. */
typedef struct prorl_packed {
  int32_t* tokens;     /* [N]   int32 token ids (range-checked < V)           */
  uint8_t* loss_mask;  /* [N]   1 iff the token came from an ASSISTANT turn    */
  int16_t* turn_id;    /* [N]   assistant-turn ordinal, -1 for others          */
  int32_t* seq_id;     /* [N]   trajectory (rollout) index                     */
  int32_t* pos_id;     /* [N]   position inside the sequence                   */
  int32_t* cu_seqlens; /* [n_seq+1] exclusive prefix of sequence lengths        */
  float* old_lp;       /* [N]   behaviour logprob (fp64 -> fp32 RN), 0 if mask=0 */
  int32_t* act_row;    /* [A]   active rows r (token r+1 is a policy token)     */
  int32_t* act_target; /* [A]   tokens[r+1]                                     */
  float* act_old_lp;   /* [A]   old_lp[r+1]                                     */
  int32_t* act_seq;    /* [A]   seq_id[r+1]                                     */
  int16_t* act_turn;   /* [A]   turn_id[r+1]                                    */
  int64_t* n_active;   /* [1]   device scalar                                   */
} prorl_packed;

typedef struct prorl_loss_cfg {
  float eps_lo;       /* DAPO clip low  (default 0.2)  */
  float eps_hi;       /* DAPO clip high (default 0.28) */
  int32_t n_buckets;  /* per-turn buckets used (<= PRORL_TURN_BUCKETS) */
  float kl_coef;      /* k3 KL penalty vs the reference policy (PAPER.md:386 uses 1e-4); needs ref_lp */
} prorl_loss_cfg;

typedef struct prorl_score_cfg {
  prorl_loss_cfg loss;
  float inv_temperature; /* 1/SamplingParams::temperature (types.hpp:59) */
  float adv_eps;         /* GRPO epsilon (1e-6) */
  int32_t ddof;          /* GRPO std ddof (1) */
  int32_t vocab;         /* V */
  int32_t dtype;         /* prorl_dtype of logits */
  int32_t microbatch_rows; /* active rows per logits micro-batch */
  double gate_tolerance;   /* is_informative tolerance (harness.cpp:92-102; default 0 = exact).
                            * K3 gates with it; host batches must be built with the same value */
} prorl_score_cfg;

/* ---- context / errors ----------------------------------------------------- */
int prorl_abi_version(void);
/* Name of the active K2 launch configuration (warps x stages x chunk). */
const char* prorl_kernel_config(void);
const char* prorl_last_error(void);
const char* prorl_status_code(int status); /* stable rollout::Error code string */
int prorl_ctx_create(int device, prorl_ctx** out);
int prorl_ctx_destroy(prorl_ctx* ctx);
/* Synchronises `stream` and reports device-side validation failures raised by
 * earlier calls on this ctx (token out of range, unsorted turns). */
int prorl_check_errors(prorl_ctx* ctx, void* stream);

/* ---- K1: pack ------------------------------------------------------------- */
/* turns: device array [n_turns]; ids_dev/lp_dev: device flat wire arrays
 * (int64 TokenId, fp64 logprob; lp entries of non-assistant turns ignored).
 * n_tokens must equal sum(len) (host-known), n_seq = number of trajectories. */
int prorl_pack(prorl_ctx* ctx, const prorl_turn_desc* turns, int64_t n_turns,
               const int64_t* ids_dev, const double* lp_dev, int64_t n_tokens,
               int32_t n_seq, int32_t vocab, const prorl_packed* out, void* stream);

/* ---- K3: GRPO advantages -------------------------------------------------- */
/* reward: [n_rollouts] fp64, usable: [n_rollouts] (0 = FAILED), group_off:
 * [n_groups+1] int32 rollout offsets. adv [n_rollouts] fp64 (0 for
 * non-usable rollouts and non-informative groups), informative [n_groups].
 * partials (nullable): adds sum(adv) and N_rollouts (usable rollouts of
 * informative groups) into partials[8], partials[9]. */
int prorl_grpo_adv(prorl_ctx* ctx, const double* reward, const uint8_t* usable,
                   const int32_t* group_off, int32_t n_groups, int32_t ddof, float eps,
                   double tolerance, double* adv, uint8_t* informative, double* partials,
                   void* stream);

/* ---- K2: logprob + entropy over the vocabulary ------------------------------ */
/* logits: [*, row_stride] of dtype; row i of the call reads logits row
 * rows[i] (rows may be NULL = identity). targets[i] in [0,V). */
int prorl_logprob_entropy(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride,
                          int32_t vocab, const int32_t* rows, const int32_t* targets,
                          int64_t n_rows, float inv_temp, float* logp, float* entropy,
                          void* stream);

/* ---- K4: clipped surrogate + metrics -------------------------------------- */
/* Adds this call's sums into partials_dev[PRORL_N_PARTIALS] (fp64) with a
 * fixed reduction order (deterministic run to run). */
/* ref_lp (nullable): reference-policy logprob per row; with it each row adds
 * kl_coef * k3 to its loss, k3 = exp(ref - logp) - (ref - logp) - 1, and
 * sum(k3) to partials[PRORL_P_KL_SUM]. */
int prorl_clipped_loss(prorl_ctx* ctx, const float* logp, const float* entropy,
                       const float* old_lp, const double* adv, const int32_t* row_seq,
                       const int16_t* row_turn, const float* ref_lp, int64_t n_rows,
                       const prorl_loss_cfg* cfg, double* partials_dev, void* stream);

/* K2+K4 fused: one HBM pass per row and the loss epilogue in the same kernel.
 * logp/entropy outputs are optional (may be NULL). */
int prorl_score_rows(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride,
                     int32_t vocab, const int32_t* rows, const int32_t* targets,
                     const float* old_lp, const double* adv, const int32_t* row_seq,
                     const int16_t* row_turn, const float* ref_lp, int64_t n_rows, float inv_temp,
                     const prorl_loss_cfg* cfg, float* logp, float* entropy,
                     double* partials_dev, void* stream);

/* ---- K5: backward through the log-softmax (SURVEY §8 f rank 1) -------------- */
/* Writes dL/dlogits for the DAPO token-mean surrogate L = sum_i l_i / n_global:
 * grad[i][v] = g_i * inv_temp * (1[v = y_i] - softmax(x_i inv_temp)_v), with
 * g_i = -A ratio / n_global when the unclipped branch is the min, else 0, and
 * the row's lse recovered as x_y inv_temp - logp_i (logp from K2). grad rows
 * are addressed like the logits rows (rows[] indirection, same row_stride,
 * same 16-B phase); grad may alias logits (in place). dtype of grad = dtype
 * of logits. dlogp (nullable) receives g_i. With ref_lp and cfg->kl_coef the
 * k3 KL term adds kl_coef * (1 - exp(ref - logp)) / n_global to g_i. */
int prorl_logits_grad(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab,
                      const int32_t* rows, const int32_t* targets, const float* logp, const float* old_lp,
                      const double* adv, const int32_t* row_seq, const float* ref_lp, int64_t n_rows, float inv_temp,
                      const prorl_loss_cfg* cfg, double n_global, void* grad, int64_t grad_stride,
                      float* dlogp, void* stream);

/* ---- K7: the training step over the logits, one HBM read + one HBM write ---- */
/* prorl_score_rows + prorl_logits_grad in one kernel: logp / entropy
 * (optional outputs), the loss partials added into
 * partials_dev[PRORL_N_PARTIALS] (as prorl_score_rows) and grad (as
 * prorl_logits_grad, with the row's lse from this same kernel). One CTA owns a
 * row: pass A reads it from HBM (statistics), pass B re-reads it from L2 and
 * writes the gradient — 4V bytes of HBM per bf16 row instead of 2V + 4V.
 * Same layouts as prorl_logits_grad: grad_stride == row_stride, grad with
 * the logits' 16-B phase, grad may alias logits (in place). */
int prorl_score_grad(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab,
                     const int32_t* rows, const int32_t* targets, const float* old_lp, const double* adv,
                     const int32_t* row_seq, const int16_t* row_turn, const float* ref_lp, int64_t n_rows,
                     float inv_temp, const prorl_loss_cfg* cfg, double n_global, float* logp, float* entropy,
                     double* partials_dev, void* grad, int64_t grad_stride, float* dlogp, void* stream);

/* ---- K6: fused LM head + logprob / entropy (SURVEY §8 f rank 2) ------------- */
/* logits_i = W . h_i (bf16 hidden [n_rows x d], row stride h_stride; bf16
 * LM-head weight [V x d], row stride w_stride; d % 64 == 0, 16-B aligned
 * rows) computed on tcgen05 tensor cores tile by tile and reduced in place:
 * logp_i = log softmax(logits_i * inv_temp)[targets_i], entropy_i as K2.
 * The logits are never materialised in HBM. */
int prorl_lmhead_logprob(prorl_ctx* ctx, const void* hidden, int64_t h_stride, const void* weight,
                         int64_t w_stride, int32_t d, int32_t vocab, const int32_t* targets,
                         int64_t n_rows, float inv_temp, float* logp, float* entropy, void* stream);

/* ---- NCCL ------------------------------------------------------------------ */
/* 128-byte ncclUniqueId produced on rank 0, broadcast by the caller. */
int prorl_nccl_unique_id(uint8_t* id128);
int prorl_nccl_init(prorl_ctx* ctx, int nranks, int rank, const uint8_t* id128);
/* In-place sum of partials_dev[n] over the ctx's communicator (no-op if
 * nranks == 1 or no communicator). */
int prorl_allreduce(prorl_ctx* ctx, double* partials_dev, int n, void* stream);

/* ---- synthetic LM-head stand-in (bench / tests) ------------------------------ */
/* Deterministic integer-hash logits, bit-identical to oracle/oracle.c
 * (oracle_gen_logits): x[i][v] = bf16/fp32(2*sqrt(3)*sigma/2 * (u0+u1+u2+u3-2))
 * and a planted target logit. row_key0 is the global index of row 0. */
int prorl_gen_logits(prorl_ctx* ctx, void* logits, int dtype, int64_t row_stride, int32_t vocab,
                     int64_t n_rows, int64_t row_key0, const int32_t* targets,
                     const float* old_lp, uint64_t seed, float sigma, void* stream);

/* Same, with an explicit key per row (row_keys[n_rows], device). prorl_score_host
 * in fill mode keys active row r of rollout s as rollout_key[s] * 2^20 +
 * (r - cu_seqlens[s]), so a row's logits do not depend on how groups were
 * sharded over GPUs. */
int prorl_gen_logits_keyed(prorl_ctx* ctx, void* logits, int dtype, int64_t row_stride, int32_t vocab,
                           int64_t n_rows, const int64_t* row_keys, const int32_t* targets,
                           const float* old_lp, uint64_t seed, float sigma, void* stream);

/* Synthetic-logits keys of n active rows (device): keys[i] =
 * (rollout_key ? rollout_key[seq[i]] : seq[i]) * 2^20 + (rows[i] - cu_seqlens[seq[i]]). */
int prorl_row_keys(prorl_ctx* ctx, const int32_t* rows, const int32_t* seq, const int32_t* cu_seqlens,
                   const int64_t* rollout_key, int64_t n, int64_t* keys, void* stream);

/* ---- host-side helpers ------------------------------------------------------ */
/* Per-rollout rewards [num_prompts * n] with the semantics (and, under
 * libstdc++, the exact values) of the reference's generate_workload
 * (proj/src/trainer/workload.cpp:62-107), default latency options. */
int prorl_synth_rewards(int32_t num_prompts, int32_t n, uint64_t seed, double p_informative, double* out);

/* Deterministic LPT: groups sorted by load desc (tie: index asc) go to the
 * least-loaded rank (tie: lowest rank). owner[g] in [0, world). */
int prorl_shard_lpt(int32_t n_groups, const int64_t* load, int32_t world, int32_t* owner);

/* Host SoA of one shard (all host pointers; pinned memory recommended). */
typedef struct prorl_host_batch {
  const prorl_turn_desc* turns; int64_t n_turns;
  const int64_t* ids; const double* lp; int64_t n_tokens;
  const double* reward; const uint8_t* usable; int32_t n_rollouts; /* = n_seq */
  const int32_t* group_off; int32_t n_groups;
  const int64_t* rollout_key; /* nullable: global rollout identity per slot
                               * (synthetic-logits key; NULL = slot index) */
} prorl_host_batch;

/* ---- trajectory ingestion (SURVEY §8 f rank 3) ------------------------------ */
/* Parses /process responses — the reference's wire schema,
 * build_process_response (proj/src/handlers.cpp:57-91) — straight into a
 * shard's host SoA, with the reference's participation rules: turns validated
 * as TokenTrajectory::validate (MalformedTurn), FAILED rollouts not usable and
 * groups failing is_informative(tolerance) contributing empty sequences
 * (proj/src/trainer/harness.cpp:84-102). Responses are in shard order: group g
 * owns responses [group_off[g], group_off[g+1]), group_off[0] = 0; rollout
 * slot (seq id) = response index. n_threads < 1: all host threads.
 * out->batch points into library-owned memory until prorl_ingest_free. */
typedef struct prorl_ingest_result {
  prorl_host_batch batch;
  int64_t n_active;
  int32_t n_informative;
  int32_t pad_;
  void* impl;
} prorl_ingest_result;
int prorl_ingest_responses(const char* const* json, const size_t* len, const int32_t* group_off,
                           int32_t n_groups, double gate_tolerance, int32_t n_threads,
                           prorl_ingest_result* out);
int prorl_ingest_free(prorl_ingest_result* r);

/* Logits provider for prorl_score_host: micro-batch j (active rows
 * [row0, row0+n)) reads logits from pool[j % n_pool] (each buffer holds
 * >= microbatch_rows rows of row_stride elements). If `fill` is non-zero the
 * library regenerates the buffer for micro-batch j with prorl_gen_logits_keyed
 * before scoring it (parity mode; generation is then inside the call).
 * If `provide` is set, buffers/fill are ignored and the callback supplies each
 * micro-batch instead (the trainer's LM head): it receives the micro-batch's
 * device arrays (packed-stream row ids, their sequence ids and the shard's
 * cu_seqlens, targets, behaviour logprobs) and
 * returns a device pointer to n rows of `*row_stride` logits, stream-ordered
 * on `stream`; a non-zero return aborts the step with that status. */
typedef int (*prorl_logits_fn)(void* user, int64_t row0, int64_t n, const int32_t* d_rows,
                               const int32_t* d_seq, const int32_t* d_cu_seqlens,
                               const int32_t* d_targets, const float* d_old_lp,
                               const void** d_logits, int64_t* row_stride, void* stream);
/* If `provide_hidden` is set instead, the step runs the fused LM head (K6):
 * the callback returns the micro-batch's final hidden states (bf16
 * [n x d_model], row stride *h_stride) and the library computes logp /
 * entropy against `weight` (bf16 [vocab x d_model], row stride w_stride) on
 * the tensor cores, then the loss (K4); the logits are never materialised. */
typedef int (*prorl_hidden_fn)(void* user, int64_t row0, int64_t n, const int32_t* d_rows,
                               const int32_t* d_seq, const int32_t* d_cu_seqlens,
                               const void** d_hidden, int64_t* h_stride, void* stream);
/* Training mode (train != 0, logits path only): each micro-batch runs K7 —
 * loss partials AND dL/dlogits of the token-mean DAPO loss over n_global
 * active rows (n_global <= 0: this shard's own active-row count; with more
 * than one rank the caller passes the global count) — written in place into
 * the micro-batch's logits buffer, or into grad_buffers[j % n_pool] when
 * given (same row stride). consume_grad (nullable) then receives the
 * micro-batch's gradient rows, stream-ordered, before the buffer is reused
 * (the LM-head backward of the trainer); a non-zero return aborts the step. */
typedef int (*prorl_grad_fn)(void* user, int64_t row0, int64_t n, const void* d_grad, int64_t row_stride,
                             void* stream);
/* Reference-policy logprobs for the k3 KL term (cfg->loss.kl_coef,
 * PAPER.md:386): for each micro-batch, a device array of n fp32 logprobs of the
 * rows' targets under the reference policy (rows as for prorl_logits_fn),
 * stream-ordered on `stream`. prorl_score_host rejects kl_coef != 0 without
 * provide_ref (the term would silently vanish otherwise). */
typedef int (*prorl_ref_fn)(void* user, int64_t row0, int64_t n, const int32_t* d_rows, const int32_t* d_seq,
                            const int32_t* d_cu_seqlens, const int32_t* d_targets, const float** d_ref_lp,
                            void* stream);
typedef struct prorl_logits_pool {
  void* const* buffers; int32_t n_pool; int32_t fill; int64_t row_stride;
  uint64_t seed; float sigma; int32_t pad_;
  prorl_logits_fn provide; void* user;
  prorl_hidden_fn provide_hidden; const void* weight; int64_t w_stride; int32_t d_model; int32_t pad2_;
  int32_t train; int32_t pad3_; double n_global;
  void* const* grad_buffers; prorl_grad_fn consume_grad; void* grad_user;
  prorl_ref_fn provide_ref; void* ref_user;
} prorl_logits_pool;

/* Full per-GPU step from HOST buffers: H2D of the SoA, K1 pack, K3 GRPO, for
 * each micro-batch K2+K4 (fused), NCCL all-reduce (if initialised), D2H of
 * the partials into host_partials[PRORL_N_PARTIALS]. Synchronises `stream`.
 * The token SoA (ids, lp) is copied in chunks of whole sequences on an
 * internal copy stream, and each chunk is packed just before the first
 * micro-batch that needs it, so the copy overlaps the scoring launches (not
 * in training mode with consume_grad: every token is checked before the
 * first gradient leaves). Host buffers must stay valid until the call returns
 * (it does not return before the copies are done); pinned memory overlaps.
 * timings_ms (nullable, [5]): h2d (the descriptors, rewards and — when not
 * chunked — the token SoA), pack+grpo (incl. the wait for the first chunk),
 * score (K2+K4 launches + slab reduce, incl. generation when pool->fill and
 * the later chunks' packing), allreduce, d2h.
 * Collective-safe failure: with a communicator of > 1 ranks every rank takes
 * part in exactly one all-reduce per call, even when its own step fails
 * (host validation, a callback, a device-side check): it contributes zeros
 * with partials[PRORL_P_ERR_RANKS] = 1. No rank hangs; the failing rank
 * returns its own status, the others PRORL_E_PEER_FAILED. */
int prorl_score_host(prorl_ctx* ctx, const prorl_host_batch* batch, const prorl_score_cfg* cfg,
                     const prorl_logits_pool* logits, double* host_partials, float* timings_ms,
                     void* stream);

/* The collective-safe failure bookkeeping prorl_score_host applies, for callers
 * that reduce the partials themselves (e.g. over torch.distributed):
 * prorl_fail_partials turns a failed rank's host partials into its
 * contribution (zeros, partials[PRORL_P_ERR_RANKS] = 1); after the sum,
 * prorl_step_status(own status, reduced partials) is the step's outcome on
 * this rank — its own error, PRORL_E_PEER_FAILED if any other rank failed, or
 * PRORL_OK. Host-only, no ctx. */
void prorl_fail_partials(double* host_partials);
/* What the last prorl_score_host call on ctx did (diagnostics): kernels this
 * library launched (callbacks' and NCCL's work not counted), micro-batches,
 * the chunks the token SoA was copied in, and the H2D bytes. */
typedef struct prorl_step_info {
  int64_t kernel_launches; int32_t micro_batches; int32_t h2d_chunks; int64_t h2d_bytes;
} prorl_step_info;
int prorl_last_step_info(const prorl_ctx* ctx, prorl_step_info* out);
int prorl_step_status(int local_status, const double* reduced_host_partials);

#ifdef __cplusplus
}
#endif
#endif /* PRORL_HOTPATH_H */
