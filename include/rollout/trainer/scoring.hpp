// rollout/trainer/scoring.hpp — C++ façade of the B200 scoring path
// (SURVEY.md §8 b3). It starts where the reference trainer stops:
// IterationStats::informative (proj/include/rollout/trainer/harness.hpp:75)
// plus the token-level trajectories the /process responses carry
// (proj/src/handlers.cpp:57-91), which the reference harness drops
// (proj/src/trainer/harness.cpp:263-273).
//
//   auto stats  = harness.run_iteration_async(workload, plan);      // reference
//   auto shard  = rollout::train::shard_groups(stats.informative, world)[rank];
//   auto result = scorer.score_groups(shard, lm_head_logits, cfg);  // this repo
//
// Everything below calls the C-ABI in prorl_hotpath.h; errors surface as
// rollout::Error subclasses carrying the C-ABI's stable codes.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include <json.hpp>

#include "prorl_hotpath.h"
#include "rollout/errors.hpp"
#include "rollout/trainer/harness.hpp"
#include "rollout/trajectory.hpp"

namespace rollout::train {

enum class LogitsDtype { BF16 = PRORL_BF16, FP32 = PRORL_FP32 };

struct ScoreConfig {
  float eps_lo = 0.2f;           // DAPO clip-low
  float eps_hi = 0.28f;          // DAPO clip-high
  float adv_eps = 1e-6f;         // GRPO epsilon (App. B.3)
  int ddof = 1;                  // GRPO std ddof
  double gate_tolerance = 0.0;   // is_informative tolerance
  float inv_temperature = 1.0f;  // 1 / SamplingParams::temperature (types.hpp:59)
  int max_turn_buckets = PRORL_TURN_BUCKETS;
  float kl_coef = 0.0f;          // k3 KL vs a reference policy (1e-4); C-ABI ref_lp path
  int vocab = 0;
  LogitsDtype dtype = LogitsDtype::BF16;
  int microbatch_rows = 16576;   // active rows per logits micro-batch (7 waves of 148 x 16 K2 warps)
};

struct TurnMetrics {
  int turn = 0;  // assistant-turn ordinal (bucket; >= max_turn_buckets-1 folded)
  std::int64_t n = 0;
  double loss = 0, entropy = 0, logp = 0, clip_frac = 0;
};

struct ScoreResult {
  double loss = 0;  // DAPO token-mean surrogate over the global batch
  std::int64_t n_active = 0;
  double entropy = 0, logp = 0, ratio = 0, clip_lo_frac = 0, clip_hi_frac = 0, kl_k1 = 0, kl_k3 = 0;
  double adv_sum = 0;
  std::int64_t n_rollouts = 0;
  std::vector<TurnMetrics> per_turn;
  std::vector<double> partials;  // PRORL_N_PARTIALS all-reduced sums
  float timings_ms[5] = {0, 0, 0, 0, 0};  // h2d, pack+grpo, score, allreduce, d2h
};

// The LM head: produces the logits of one micro-batch of active rows.
class LogitsSource {
 public:
  virtual ~LogitsSource() = default;
  // d_rows: positions in the packed stream (row r predicts token r+1), d_seq
  // their sequence (rollout slot) ids, d_cu_seqlens the shard's sequence
  // offsets; d_targets / d_old_lp: the rows' target ids and behaviour
  // logprobs. The micro-batch covers active rows [row0, row0 + n). Returns a
  // device pointer to n rows of `row_stride` logits (cfg.dtype), valid until
  // the next call.
  virtual const void* logits(std::int64_t row0, std::int64_t n, const std::int32_t* d_rows,
                             const std::int32_t* d_seq, const std::int32_t* d_cu_seqlens,
                             const std::int32_t* d_targets, const float* d_old_lp, std::int64_t* row_stride,
                             void* stream) = 0;
  // Reference-policy logprobs of the same rows' targets (device, n floats) for
  // the k3 KL term (ScoreConfig::kl_coef). Needed only when
  // kl_coef != 0; the default has none (the step then throws MalformedRequest).
  virtual const float* ref_logprobs(std::int64_t /*row0*/, std::int64_t /*n*/, const std::int32_t* /*d_rows*/,
                                    const std::int32_t* /*d_seq*/, const std::int32_t* /*d_cu_seqlens*/,
                                    const std::int32_t* /*d_targets*/, void* /*stream*/) {
    return nullptr;
  }
};

// The LM-head backward: receives dL/dlogits of one micro-batch (active rows
// [row0, row0 + n), same dtype and row stride as the logits the source
// returned — the gradient overwrites them in place), stream-ordered, before the
// source is asked for the next micro-batch.
class GradSink {
 public:
  virtual ~GradSink() = default;
  virtual void gradient(std::int64_t row0, std::int64_t n, const void* d_grad, std::int64_t row_stride,
                        void* stream) = 0;
};

// Deterministic synthetic LM head (include/prorl_synth.h) — bench / tests.
class SyntheticLogits : public LogitsSource {
 public:
  SyntheticLogits(int device, int vocab, LogitsDtype dtype, std::int64_t max_rows, std::uint64_t seed,
                  float sigma = 2.0f);
  ~SyntheticLogits() override;
  const void* logits(std::int64_t row0, std::int64_t n, const std::int32_t* d_rows, const std::int32_t* d_seq,
                     const std::int32_t* d_cu_seqlens, const std::int32_t* d_targets, const float* d_old_lp,
                     std::int64_t* row_stride, void* stream) override;

 private:
  prorl_ctx* ctx_ = nullptr;
  void* buf_ = nullptr;
  std::int64_t* keys_ = nullptr;  // per-row synthetic keys (seq * 2^20 + position), as the oracle
  int vocab_;
  LogitsDtype dtype_;
  std::int64_t max_rows_;
  std::uint64_t seed_;
  float sigma_;
};

// Host SoA of one shard, in the C-ABI's layout. Groups are taken in the given
// order; slot i of a group is rollout (= sequence) group_off[g] + i.
struct HostBatch {
  std::vector<prorl_turn_desc> turns;
  std::vector<std::int64_t> ids;
  std::vector<double> lp;
  std::vector<double> reward;
  std::vector<std::uint8_t> usable;
  std::vector<std::int32_t> group_off{0};
  std::int64_t n_active = 0;
  prorl_host_batch view() const;
};

// Builds the SoA: FAILED rollouts (usable_rewards' exclusion, harness.cpp:87)
// and rollouts of non-informative groups contribute empty sequences; every
// other complete outcome must carry its trajectory (MalformedRequest
// otherwise). Throws IncompleteGroup for incomplete groups.
HostBatch build_host_batch(const std::vector<PromptGroup>& groups, const ScoreConfig& cfg);

// Deterministic LPT over `world` ranks by policy-token count; returns each
// rank's groups (in input order). Groups never cross ranks (App. B.3, §8 e1).
std::vector<std::vector<PromptGroup>> shard_groups(const std::vector<PromptGroup>& groups, int world);

ScoreResult finalize(const double* partials, int n_buckets = PRORL_TURN_BUCKETS);

class DeviceScorer {
 public:
  explicit DeviceScorer(int device = 0);
  ~DeviceScorer();
  DeviceScorer(const DeviceScorer&) = delete;
  DeviceScorer& operator=(const DeviceScorer&) = delete;

  static std::array<std::uint8_t, 128> nccl_unique_id();
  void init_nccl(int world, int rank, const std::array<std::uint8_t, 128>& id);

  // One trainer step over this rank's groups: H2D, pack, GRPO, fused
  // logprob/entropy + clipped loss per logits micro-batch, all-reduce, D2H.
  ScoreResult score_groups(const std::vector<PromptGroup>& groups, LogitsSource& logits, const ScoreConfig& cfg,
                           void* stream = nullptr);
  ScoreResult score_batch(const HostBatch& batch, LogitsSource& logits, const ScoreConfig& cfg,
                          void* stream = nullptr);
  // Same on a raw C-ABI batch view (e.g. from ingest_responses).
  ScoreResult score_view(const prorl_host_batch& batch, LogitsSource& logits, const ScoreConfig& cfg,
                         void* stream = nullptr);

  // Training step: the same partials plus dL/dlogits of the token-mean DAPO
  // loss over n_global active rows (<= 0: this shard's own count; pass the
  // global count when several ranks train), one HBM read and one HBM write per
  // logits row (K7). The gradient is written in place into the buffer the
  // source returned and handed to `grads` per micro-batch.
  ScoreResult train_groups(const std::vector<PromptGroup>& groups, LogitsSource& logits, GradSink& grads,
                           const ScoreConfig& cfg, double n_global = 0.0, void* stream = nullptr);
  ScoreResult train_view(const prorl_host_batch& batch, LogitsSource& logits, GradSink& grads,
                         const ScoreConfig& cfg, double n_global = 0.0, void* stream = nullptr);

  prorl_ctx* ctx() const { return ctx_; }

 private:
  prorl_ctx* ctx_ = nullptr;
};

// ---- wire ingestion (inverse of build_process_response, handlers.cpp:60-66) ----
// Each turn object: {"role", "input_ids", "output_ids", "logprobs", "text"};
// validated with TokenTrajectory::validate (MalformedTurn).
TokenTrajectory trajectory_from_json(const nlohmann::json& turns);
// The fields the reference harness records (harness.cpp:254-273) plus the trajectory.
RolloutOutcome outcome_from_response(const nlohmann::json& response);

// Wire JSON of one shard's /process responses -> host SoA (prorl_ingest_responses):
// group g owns responses [group_off[g], group_off[g+1]).
class IngestedBatch {
 public:
  IngestedBatch(const std::vector<std::string>& responses, const std::vector<std::int32_t>& group_off,
                double gate_tolerance = 0.0, int threads = 0);
  ~IngestedBatch();
  IngestedBatch(const IngestedBatch&) = delete;
  IngestedBatch& operator=(const IngestedBatch&) = delete;
  const prorl_host_batch& view() const { return r_.batch; }
  std::int64_t n_active() const { return r_.n_active; }
  int n_informative() const { return r_.n_informative; }

 private:
  prorl_ingest_result r_{};
};

// Throws the rollout::Error subclass for a C-ABI status (no-op for PRORL_OK).
void throw_status(int status);

}  // namespace rollout::train
