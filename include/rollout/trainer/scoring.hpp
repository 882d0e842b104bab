// rollout/trainer/scoring.hpp — C++ façade of the B200 scoring path
// (SURVEY.md §8 b3), header-only over the C-ABI in prorl_hotpath.h.
//
// It starts where the reference trainer stops: IterationStats::informative
// (proj/include/rollout/trainer/harness.hpp:75, filled at
// proj/src/trainer/harness.cpp:313-316) plus the token-level trajectories the
// /process responses carry (proj/src/handlers.cpp:57-91), which the reference
// harness drops when it records a response (proj/src/trainer/harness.cpp:263-273).
//
//   // the harness keeps each response's trajectory through the hook that
//   // integration/reference.patch adds at harness.cpp:273 (3 lines):
//   opts.on_response = [&](const PromptGroup& g, int slot, const nlohmann::json& r) {
//     keep_trajectory(trajectories, g, slot, r);                      // this repo
//   };
//   ...
//   auto stats  = harness.run_iteration_async(workload, plan);         // reference
//   auto shard  = shard_groups(stats.informative, trajectories, world)[rank];
//   auto result = scorer.score_groups(shard, trajectories, lm_head, cfg);
//
// The reference's types are used as they are — this header includes
// "rollout/trajectory.hpp", "rollout/errors.hpp" and
// "rollout/trainer/harness.hpp" from whichever include root the build puts
// first: the reference's own proj/include, or include/standalone/ of this repo
// for builds without the reference (same declarations). Nothing here is
// compiled into libprorl_hotpath.so: every function is inline and compiled in
// the caller's translation unit against the caller's headers, and only plain
// C types (prorl_hotpath.h) cross into the library. The trajectory travels
// beside RolloutOutcome in a TrajectoryTable keyed by (prompt_id, slot), so no
// reference type changes.
//
// Errors surface as rollout::Error subclasses carrying the C-ABI's stable
// codes: the reference's MalformedTurn / IncompleteGroup / MalformedRequest,
// plus CudaError, NcclError, ShapeMismatch and PeerFailed declared below.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include <json.hpp>

#include "prorl_hotpath.h"
#include "rollout/errors.hpp"
#include "rollout/trainer/harness.hpp"
#include "rollout/trajectory.hpp"

namespace rollout {

// Codes the device path adds to the reference's set (errors.hpp:28-59).
class CudaError : public Error {
 public:
  explicit CudaError(const std::string& msg = "cuda_error") : Error("cuda_error", msg) {}
};
class NcclError : public Error {
 public:
  explicit NcclError(const std::string& msg = "nccl_error") : Error("nccl_error", msg) {}
};
class ShapeMismatch : public Error {
 public:
  explicit ShapeMismatch(const std::string& msg = "shape_mismatch") : Error("shape_mismatch", msg) {}
};
// Another rank's step failed; this rank's all-reduced result is void.
class PeerFailed : public Error {
 public:
  explicit PeerFailed(const std::string& msg = "peer_failed") : Error("peer_failed", msg) {}
};

}  // namespace rollout

namespace rollout::train {

enum class LogitsDtype { BF16 = PRORL_BF16, FP32 = PRORL_FP32 };

struct ScoreConfig {
  float eps_lo = 0.2f;           // DAPO clip-low
  float eps_hi = 0.28f;          // DAPO clip-high
  float adv_eps = 1e-6f;         // GRPO epsilon (App. B.3)
  int ddof = 1;                  // GRPO std ddof (0 or 1)
  double gate_tolerance = 0.0;   // is_informative tolerance (host gate and the device K3 gate)
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
// source is asked for the next micro-batch. The library has already checked the
// step's token ids and descriptors on the device when the first one arrives.
class GradSink {
 public:
  virtual ~GradSink() = default;
  virtual void gradient(std::int64_t row0, std::int64_t n, const void* d_grad, std::int64_t row_stride,
                        void* stream) = 0;
};

// Throws the rollout::Error subclass for a C-ABI status (no-op for PRORL_OK).
inline void throw_status(int status) {
  if (status == PRORL_OK) return;
  const std::string msg = prorl_last_error();
  switch (status) {
    case PRORL_E_MALFORMED_TURN: throw MalformedTurn(msg);
    case PRORL_E_INCOMPLETE_GROUP: throw IncompleteGroup(msg);
    case PRORL_E_MALFORMED_REQUEST: throw MalformedRequest(msg);
    case PRORL_E_CUDA: throw CudaError(msg);
    case PRORL_E_NCCL: throw NcclError(msg);
    case PRORL_E_PEER_FAILED: throw PeerFailed(msg);
    default: throw ShapeMismatch(msg);
  }
}

// ---- trajectories beside the reference's RolloutOutcome ------------------------
// Keyed by (PromptGroup::prompt_id, slot). Written from the harness's
// per-rollout threads (one put per recorded response), read by the trainer
// step after run_iteration_* returns.
class TrajectoryTable {
 public:
  void put(const std::string& prompt_id, int slot, TokenTrajectory t) {
    std::lock_guard<std::mutex> lk(mu_);
    m_[{prompt_id, slot}] = std::move(t);
  }
  // nullptr when absent. The pointer stays valid until erase_group / clear.
  const TokenTrajectory* find(const std::string& prompt_id, int slot) const {
    std::lock_guard<std::mutex> lk(mu_);
    const auto it = m_.find({prompt_id, slot});
    return it == m_.end() ? nullptr : &it->second;
  }
  // Drop a group's trajectories (after its step, or when it is carried over).
  void erase_group(const std::string& prompt_id) {
    std::lock_guard<std::mutex> lk(mu_);
    m_.erase(m_.lower_bound({prompt_id, INT32_MIN}), m_.upper_bound({prompt_id, INT32_MAX}));
  }
  void clear() {
    std::lock_guard<std::mutex> lk(mu_);
    m_.clear();
  }
  std::size_t size() const {
    std::lock_guard<std::mutex> lk(mu_);
    return m_.size();
  }

 private:
  mutable std::mutex mu_;
  std::map<std::pair<std::string, int>, TokenTrajectory> m_;
};

namespace detail {
inline Role role_from_name(const std::string& s) {
  if (s == "system") return Role::SYSTEM;
  if (s == "user") return Role::USER;
  if (s == "assistant") return Role::ASSISTANT;
  if (s == "tool") return Role::TOOL;
  throw MalformedTurn("unknown role '" + s + "'");
}
// The ids a turn contributes to flatten() (trajectory.hpp:82-83).
inline const TokenIds& turn_tokens(const Turn& t) { return t.role == Role::ASSISTANT ? t.output_ids : t.input_ids; }
inline bool is_failed(const RolloutOutcome& o) { return o.status == "FAILED"; }
inline bool is_cancelled(const RolloutOutcome& o) { return o.status == "CANCELLED"; }

// Groups in prompt_id order: the harness hands them over in
// completion order (harness.cpp:313-316), which is not reproducible.
template <typename Groups>
std::vector<std::size_t> prompt_order(const Groups& groups) {
  std::vector<std::size_t> idx(groups.size());
  std::iota(idx.begin(), idx.end(), std::size_t{0});
  std::stable_sort(idx.begin(), idx.end(),
                   [&](std::size_t a, std::size_t b) { return groups[a].prompt_id < groups[b].prompt_id; });
  return idx;
}
}  // namespace detail

// ---- wire ingestion (inverse of build_process_response, handlers.cpp:60-66) ----
// Each turn object: {"role", "input_ids", "output_ids", "logprobs", "text"};
// validated with TokenTrajectory::validate (MalformedTurn).
inline TokenTrajectory trajectory_from_json(const nlohmann::json& turns) {
  if (!turns.is_array()) throw MalformedRequest("trajectory must be an array of turns");
  TokenTrajectory traj;
  for (const auto& tj : turns) {
    if (!tj.is_object()) throw MalformedTurn("turn must be an object");
    if (!tj.contains("role") || !tj.at("role").is_string()) throw MalformedTurn("turn without a role");
    Turn t;
    t.role = detail::role_from_name(tj.at("role").get<std::string>());
    t.input_ids = tj.value("input_ids", TokenIds{});
    t.output_ids = tj.value("output_ids", TokenIds{});
    t.logprobs = tj.value("logprobs", std::vector<double>{});
    t.text = tj.value("text", std::string{});
    traj.append(std::move(t));  // validates (MalformedTurn)
  }
  return traj;
}

// The fields the reference harness records from a response
// (harness.cpp:263-273): a missing status reads as FAILED.
inline RolloutOutcome outcome_from_response(const nlohmann::json& resp, double wall_seconds = 0.0) {
  if (!resp.is_object()) throw MalformedRequest("response must be an object");
  RolloutOutcome o;
  o.status = resp.value("status", std::string("FAILED"));
  o.reward = resp.value("reward", 0.0);
  o.address = resp.value("backend", std::string{});
  o.wall_seconds = wall_seconds;
  return o;
}

// What the harness does at harness.cpp:262-273 for a response that arrived,
// plus the trajectory it drops today: a CANCELLED response is not recorded
// (its slot is re-issued; returns false), anything else fills the slot, and a
// non-FAILED rollout's trajectory goes into `table`. Call it under the lock
// the harness already holds there.
inline bool record_response(PromptGroup& g, int slot, const nlohmann::json& resp, TrajectoryTable& table,
                            double wall_seconds = 0.0) {
  if (slot < 0 || slot >= static_cast<int>(g.outcomes.size()))
    throw MalformedRequest("record_response: slot outside the group");
  RolloutOutcome o = outcome_from_response(resp, wall_seconds);
  if (detail::is_cancelled(o)) return false;
  if (!detail::is_failed(o)) {
    if (!resp.contains("trajectory")) throw MalformedRequest("response without a trajectory");
    table.put(g.prompt_id, slot, trajectory_from_json(resp.at("trajectory")));
  }
  g.outcomes[static_cast<std::size_t>(slot)] = std::move(o);
  return true;
}

// The hook integration/reference.patch adds to the reference harness
// (TrainerOptions::on_response, called under the harness lock for every
// recorded response): keep the trajectory of a non-FAILED rollout.
//   opts.on_response = [&](const PromptGroup& g, int slot, const nlohmann::json& r) {
//     keep_trajectory(trajectories, g, slot, r);
//   };
inline void keep_trajectory(TrajectoryTable& table, const PromptGroup& g, int slot, const nlohmann::json& resp) {
  if (resp.value("status", std::string("FAILED")) == "FAILED") return;
  if (!resp.contains("trajectory")) throw MalformedRequest("response without a trajectory");
  table.put(g.prompt_id, slot, trajectory_from_json(resp.at("trajectory")));
}

// ---- host SoA of one shard ---------------------------------------------------------
// In the C-ABI's layout. Groups in prompt_id order; slot i of group g is
// rollout (= sequence) group_off[g] + i.
struct HostBatch {
  std::vector<prorl_turn_desc> turns;
  std::vector<std::int64_t> ids;
  std::vector<double> lp;
  std::vector<double> reward;
  std::vector<std::uint8_t> usable;
  std::vector<std::int32_t> group_off{0};
  std::vector<std::string> prompt_ids;  // group g's PromptGroup::prompt_id
  std::int64_t n_active = 0;
  prorl_host_batch view() const {
    prorl_host_batch b{};
    b.turns = turns.data();
    b.n_turns = static_cast<std::int64_t>(turns.size());
    b.ids = ids.data();
    b.lp = lp.data();
    b.n_tokens = static_cast<std::int64_t>(ids.size());
    b.reward = reward.data();
    b.usable = usable.data();
    b.n_rollouts = static_cast<std::int32_t>(reward.size());
    b.group_off = group_off.data();
    b.n_groups = static_cast<std::int32_t>(group_off.size()) - 1;
    return b;
  }
};

// Builds the SoA: FAILED rollouts (usable_rewards' exclusion, harness.cpp:87)
// and rollouts of non-informative groups contribute empty sequences; every
// other rollout must have its trajectory in `table` (MalformedRequest
// otherwise). Throws IncompleteGroup for an incomplete group or one holding a
// CANCELLED outcome (the reference never records those, harness.cpp:264).
template <typename Groups>
HostBatch build_host_batch(const Groups& groups, const TrajectoryTable& table, const ScoreConfig& cfg) {
  HostBatch hb;
  std::int32_t seq = 0;
  for (const std::size_t gi : detail::prompt_order(groups)) {
    const PromptGroup& g = groups[gi];
    for (const auto& slot : g.outcomes)
      if (slot && detail::is_cancelled(*slot))
        throw IncompleteGroup("group " + g.prompt_id + ": a CANCELLED rollout leaves its slot to be re-issued");
    const bool informative = is_informative(g, cfg.gate_tolerance);  // IncompleteGroup if partial
    for (std::size_t k = 0; k < g.outcomes.size(); ++k) {
      const RolloutOutcome& o = *g.outcomes[k];
      hb.reward.push_back(o.reward);
      hb.usable.push_back(detail::is_failed(o) ? 0 : 1);
      if (informative && !detail::is_failed(o)) {
        const TokenTrajectory* tr = table.find(g.prompt_id, static_cast<int>(k));
        if (!tr)
          throw MalformedRequest("group " + g.prompt_id + " slot " + std::to_string(k) +
                                 ": usable rollout without a trajectory");
        std::int64_t pos = 0;
        for (const Turn& t : tr->turns()) {
          TokenTrajectory::validate(t);
          const TokenIds& ids = detail::turn_tokens(t);
          prorl_turn_desc d{};
          d.src_off = static_cast<std::int64_t>(hb.ids.size());
          d.traj = seq;
          d.len = static_cast<std::int32_t>(ids.size());
          d.role = static_cast<std::uint8_t>(t.role);  // == PRORL_ROLE_*
          hb.turns.push_back(d);
          hb.ids.insert(hb.ids.end(), ids.begin(), ids.end());
          if (t.role == Role::ASSISTANT) {
            hb.lp.insert(hb.lp.end(), t.logprobs.begin(), t.logprobs.end());
            if (!ids.empty()) hb.n_active += static_cast<std::int64_t>(ids.size()) - (pos == 0 ? 1 : 0);
          } else {
            hb.lp.insert(hb.lp.end(), ids.size(), 0.0);
          }
          pos += static_cast<std::int64_t>(ids.size());
        }
      }
      ++seq;
    }
    hb.group_off.push_back(seq);
    hb.prompt_ids.push_back(g.prompt_id);
  }
  return hb;
}

// Deterministic LPT over `world` ranks by policy-token count (prorl_shard_lpt:
// load desc, ties by prompt_id order); returns each rank's groups in prompt_id
// order. Groups never cross ranks (App. B.3, §8 e1). Every rank computes the
// same assignment from the same set of groups, whatever order it received them in.
template <typename Groups>
std::vector<std::vector<PromptGroup>> shard_groups(const Groups& groups, const TrajectoryTable& table, int world) {
  if (world < 1) throw MalformedRequest("shard_groups: world < 1");
  const std::vector<std::size_t> order = detail::prompt_order(groups);
  std::vector<std::int64_t> load(order.size(), 0);
  for (std::size_t i = 0; i < order.size(); ++i) {
    const PromptGroup& g = groups[order[i]];
    for (std::size_t k = 0; k < g.outcomes.size(); ++k) {
      if (!g.outcomes[k] || detail::is_failed(*g.outcomes[k])) continue;
      if (const TokenTrajectory* tr = table.find(g.prompt_id, static_cast<int>(k)))
        for (const Turn& t : tr->turns())
          if (t.role == Role::ASSISTANT) load[i] += static_cast<std::int64_t>(t.output_ids.size());
    }
  }
  std::vector<std::int32_t> owner(order.size(), 0);
  throw_status(prorl_shard_lpt(static_cast<std::int32_t>(order.size()), load.data(), world, owner.data()));
  std::vector<std::vector<PromptGroup>> out(static_cast<std::size_t>(world));
  for (std::size_t i = 0; i < order.size(); ++i) out[static_cast<std::size_t>(owner[i])].push_back(groups[order[i]]);
  return out;
}

inline ScoreResult finalize(const double* p, int n_buckets = PRORL_TURN_BUCKETS) {
  ScoreResult r;
  r.partials.assign(p, p + PRORL_N_PARTIALS);
  const double n = p[PRORL_P_N_ACTIVE] > 0 ? p[PRORL_P_N_ACTIVE] : 1.0;
  r.n_active = static_cast<std::int64_t>(p[PRORL_P_N_ACTIVE]);
  r.loss = p[PRORL_P_LOSS_SUM] / n;
  r.entropy = p[PRORL_P_ENTROPY_SUM] / n;
  r.logp = p[PRORL_P_LOGP_SUM] / n;
  r.ratio = p[PRORL_P_RATIO_SUM] / n;
  r.clip_lo_frac = p[PRORL_P_CLIP_LO] / n;
  r.clip_hi_frac = p[PRORL_P_CLIP_HI] / n;
  r.kl_k1 = p[PRORL_P_KL1_SUM] / n;
  r.kl_k3 = p[PRORL_P_KL_SUM] / n;
  r.adv_sum = p[PRORL_P_ADV_SUM];
  r.n_rollouts = static_cast<std::int64_t>(p[PRORL_P_N_ROLLOUTS]);
  for (int k = 0; k < n_buckets && k < PRORL_TURN_BUCKETS; ++k) {
    const double* b = p + PRORL_N_GLOBAL + PRORL_N_PER_TURN * k;
    if (b[0] <= 0) continue;
    r.per_turn.push_back({k, static_cast<std::int64_t>(b[0]), b[1] / b[0], b[2] / b[0], b[3] / b[0], b[4] / b[0]});
  }
  return r;
}

inline prorl_score_cfg to_c(const ScoreConfig& cfg) {
  prorl_score_cfg c{};
  c.loss.eps_lo = cfg.eps_lo;
  c.loss.eps_hi = cfg.eps_hi;
  c.loss.n_buckets = cfg.max_turn_buckets;
  c.loss.kl_coef = cfg.kl_coef;
  c.inv_temperature = cfg.inv_temperature;
  c.adv_eps = cfg.adv_eps;
  c.ddof = cfg.ddof;
  c.vocab = cfg.vocab;
  c.dtype = static_cast<int>(cfg.dtype);
  c.microbatch_rows = cfg.microbatch_rows;
  c.gate_tolerance = cfg.gate_tolerance;
  return c;
}

namespace detail {
// C callbacks of prorl_logits_pool over the C++ interfaces; an exception is
// captured (it must not unwind through the C library) and rethrown as
// MalformedRequest after the step returns.
struct Trampoline {
  LogitsSource* src = nullptr;
  GradSink* sink = nullptr;
  std::string error;
  int status = PRORL_OK;
  void capture(const std::exception& e) {
    const auto* re = dynamic_cast<const Error*>(&e);
    error = re ? re->code() + ": " + e.what() : std::string(e.what());
    status = PRORL_E_MALFORMED_REQUEST;
  }
};

inline int provide_logits(void* user, std::int64_t row0, std::int64_t n, const std::int32_t* d_rows,
                          const std::int32_t* d_seq, const std::int32_t* d_cu_seqlens, const std::int32_t* d_targets,
                          const float* d_old_lp, const void** d_logits, std::int64_t* row_stride, void* stream) {
  auto* t = static_cast<Trampoline*>(user);
  try {
    *d_logits = t->src->logits(row0, n, d_rows, d_seq, d_cu_seqlens, d_targets, d_old_lp, row_stride, stream);
    return PRORL_OK;
  } catch (const std::exception& e) {
    t->capture(e);
  }
  return t->status;
}

inline int provide_ref(void* user, std::int64_t row0, std::int64_t n, const std::int32_t* d_rows,
                       const std::int32_t* d_seq, const std::int32_t* d_cu_seqlens, const std::int32_t* d_targets,
                       const float** d_ref_lp, void* stream) {
  auto* t = static_cast<Trampoline*>(user);
  try {
    *d_ref_lp = t->src->ref_logprobs(row0, n, d_rows, d_seq, d_cu_seqlens, d_targets, stream);
    if (*d_ref_lp) return PRORL_OK;
    t->error = "kl_coef != 0 but the logits source provides no reference logprobs";
    t->status = PRORL_E_MALFORMED_REQUEST;
  } catch (const std::exception& e) {
    t->capture(e);
  }
  return t->status;
}

inline int consume_grad(void* user, std::int64_t row0, std::int64_t n, const void* d_grad, std::int64_t row_stride,
                        void* stream) {
  auto* t = static_cast<Trampoline*>(user);
  try {
    t->sink->gradient(row0, n, d_grad, row_stride, stream);
    return PRORL_OK;
  } catch (const std::exception& e) {
    t->capture(e);
  }
  return t->status;
}
}  // namespace detail

class DeviceScorer {
 public:
  explicit DeviceScorer(int device = 0) {
    if (prorl_abi_version() != PRORL_ABI_VERSION)
      throw ShapeMismatch("libprorl_hotpath ABI " + std::to_string(prorl_abi_version()) + " != header " +
                          std::to_string(PRORL_ABI_VERSION));
    throw_status(prorl_ctx_create(device, &ctx_));
  }
  ~DeviceScorer() { prorl_ctx_destroy(ctx_); }
  DeviceScorer(const DeviceScorer&) = delete;
  DeviceScorer& operator=(const DeviceScorer&) = delete;

  static std::array<std::uint8_t, 128> nccl_unique_id() {
    std::array<std::uint8_t, 128> id{};
    throw_status(prorl_nccl_unique_id(id.data()));
    return id;
  }
  void init_nccl(int world, int rank, const std::array<std::uint8_t, 128>& id) {
    throw_status(prorl_nccl_init(ctx_, world, rank, id.data()));
  }

  // One trainer step over this rank's groups: H2D, pack, GRPO, fused
  // logprob/entropy + clipped loss per logits micro-batch, all-reduce, D2H.
  template <typename Groups>
  ScoreResult score_groups(const Groups& groups, const TrajectoryTable& table, LogitsSource& logits,
                           const ScoreConfig& cfg, void* stream = nullptr) {
    const HostBatch b = build_host_batch(groups, table, cfg);
    return score_view(b.view(), logits, cfg, stream);
  }
  ScoreResult score_batch(const HostBatch& batch, LogitsSource& logits, const ScoreConfig& cfg,
                          void* stream = nullptr) {
    return score_view(batch.view(), logits, cfg, stream);
  }
  // Same on a raw C-ABI batch view (e.g. from IngestedBatch).
  ScoreResult score_view(const prorl_host_batch& hb, LogitsSource& logits, const ScoreConfig& cfg,
                         void* stream = nullptr) {
    return run(hb, logits, nullptr, cfg, 0.0, stream);
  }

  // Training step: the same partials plus dL/dlogits of the token-mean DAPO
  // loss over n_global active rows (<= 0: this shard's own count, single rank
  // only; pass the global count when several ranks train), one HBM read and
  // one HBM write per logits row (K7). The gradient is written in place into
  // the buffer the source returned and handed to `grads` per micro-batch.
  template <typename Groups>
  ScoreResult train_groups(const Groups& groups, const TrajectoryTable& table, LogitsSource& logits,
                           GradSink& grads, const ScoreConfig& cfg, double n_global = 0.0, void* stream = nullptr) {
    const HostBatch b = build_host_batch(groups, table, cfg);
    return run(b.view(), logits, &grads, cfg, n_global, stream);
  }
  ScoreResult train_view(const prorl_host_batch& hb, LogitsSource& logits, GradSink& grads, const ScoreConfig& cfg,
                         double n_global = 0.0, void* stream = nullptr) {
    return run(hb, logits, &grads, cfg, n_global, stream);
  }

  prorl_ctx* ctx() const { return ctx_; }

 private:
  ScoreResult run(const prorl_host_batch& hb, LogitsSource& logits, GradSink* grads, const ScoreConfig& cfg,
                  double n_global, void* stream) {
    const prorl_score_cfg c = to_c(cfg);
    detail::Trampoline tr;
    tr.src = &logits;
    tr.sink = grads;
    prorl_logits_pool pool{};
    pool.provide = &detail::provide_logits;
    pool.user = &tr;
    if (cfg.kl_coef != 0.f) {
      pool.provide_ref = &detail::provide_ref;
      pool.ref_user = &tr;
    }
    if (grads) {
      pool.train = 1;
      pool.n_global = n_global;
      pool.consume_grad = &detail::consume_grad;
      pool.grad_user = &tr;
    }
    double partials[PRORL_N_PARTIALS];
    float tm[5];
    const int st = prorl_score_host(ctx_, &hb, &c, &pool, partials, tm, stream);
    if (st != PRORL_OK && tr.status != PRORL_OK) throw MalformedRequest("callback failed: " + tr.error);
    throw_status(st);
    ScoreResult r = finalize(partials, cfg.max_turn_buckets);
    std::memcpy(r.timings_ms, tm, sizeof tm);
    return r;
  }

  prorl_ctx* ctx_ = nullptr;
};

// Wire JSON of one shard's /process responses -> host SoA (prorl_ingest_responses):
// group g owns responses [group_off[g], group_off[g+1]); pass groups in
// prompt_id order (App. B.1).
class IngestedBatch {
 public:
  IngestedBatch(const std::vector<std::string>& responses, const std::vector<std::int32_t>& group_off,
                double gate_tolerance = 0.0, int threads = 0) {
    if (group_off.empty() || static_cast<std::size_t>(group_off.back()) != responses.size())
      throw MalformedRequest("IngestedBatch: group_off must end at the number of responses");
    std::vector<const char*> ptrs(responses.size());
    std::vector<std::size_t> lens(responses.size());
    for (std::size_t i = 0; i < responses.size(); ++i) {
      ptrs[i] = responses[i].data();
      lens[i] = responses[i].size();
    }
    throw_status(prorl_ingest_responses(ptrs.data(), lens.data(), group_off.data(),
                                        static_cast<std::int32_t>(group_off.size()) - 1, gate_tolerance, threads,
                                        &r_));
  }
  ~IngestedBatch() { prorl_ingest_free(&r_); }
  IngestedBatch(const IngestedBatch&) = delete;
  IngestedBatch& operator=(const IngestedBatch&) = delete;
  const prorl_host_batch& view() const { return r_.batch; }
  std::int64_t n_active() const { return r_.n_active; }
  int n_informative() const { return r_.n_informative; }

 private:
  prorl_ingest_result r_{};
};

}  // namespace rollout::train
