// scoring.cpp — the C++ façade (include/rollout/trainer/scoring.hpp) over the
// C-ABI. Host-only C++; everything on the device goes through prorl_*.
#include "rollout/trainer/scoring.hpp"

#include <cuda_runtime.h>

#include <cstring>
#include <numeric>

namespace rollout::train {

void throw_status(int status) {
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

static std::uint8_t role_code(Role r) { return static_cast<std::uint8_t>(r); }  // == PRORL_ROLE_*

prorl_host_batch HostBatch::view() const {
  prorl_host_batch b{};
  b.turns = turns.data();
  b.n_turns = (std::int64_t)turns.size();
  b.ids = ids.data();
  b.lp = lp.data();
  b.n_tokens = (std::int64_t)ids.size();
  b.reward = reward.data();
  b.usable = usable.data();
  b.n_rollouts = (std::int32_t)reward.size();
  b.group_off = group_off.data();
  b.n_groups = (std::int32_t)group_off.size() - 1;
  return b;
}

HostBatch build_host_batch(const std::vector<PromptGroup>& groups, const ScoreConfig& cfg) {
  HostBatch hb;
  std::int32_t seq = 0;
  for (const PromptGroup& g : groups) {
    const bool informative = is_informative(g, cfg.gate_tolerance);  // IncompleteGroup if partial
    for (const auto& slot : g.outcomes) {
      const RolloutOutcome& o = *slot;
      hb.reward.push_back(o.reward);
      hb.usable.push_back(o.failed() ? 0 : 1);
      if (informative && !o.failed()) {
        if (!o.trajectory)
          throw MalformedRequest("group " + g.prompt_id + ": usable rollout without a trajectory");
        std::int64_t pos = 0;
        for (const Turn& t : o.trajectory->turns()) {
          TokenTrajectory::validate(t);
          const TokenIds& ids = t.tokens();
          prorl_turn_desc d{};
          d.src_off = (std::int64_t)hb.ids.size();
          d.traj = seq;
          d.len = (std::int32_t)ids.size();
          d.role = role_code(t.role);
          hb.turns.push_back(d);
          hb.ids.insert(hb.ids.end(), ids.begin(), ids.end());
          if (t.role == Role::ASSISTANT) {
            hb.lp.insert(hb.lp.end(), t.logprobs.begin(), t.logprobs.end());
            if (!ids.empty()) hb.n_active += (std::int64_t)ids.size() - (pos == 0 ? 1 : 0);
          } else {
            hb.lp.insert(hb.lp.end(), ids.size(), 0.0);
          }
          pos += (std::int64_t)ids.size();
        }
      }
      ++seq;
    }
    hb.group_off.push_back(seq);
  }
  return hb;
}

std::vector<std::vector<PromptGroup>> shard_groups(const std::vector<PromptGroup>& groups, int world) {
  if (world < 1) throw MalformedRequest("shard_groups: world < 1");
  std::vector<std::int64_t> load(groups.size(), 0);
  for (std::size_t i = 0; i < groups.size(); ++i)
    for (const auto& o : groups[i].outcomes)
      if (o && !o->failed() && o->trajectory)
        for (const Turn& t : o->trajectory->turns())
          if (t.role == Role::ASSISTANT) load[i] += (std::int64_t)t.output_ids.size();
  std::vector<std::int32_t> owner(groups.size(), 0);
  throw_status(prorl_shard_lpt((std::int32_t)groups.size(), load.data(), world, owner.data()));
  std::vector<std::vector<PromptGroup>> out((std::size_t)world);
  for (std::size_t i = 0; i < groups.size(); ++i) out[(std::size_t)owner[i]].push_back(groups[i]);
  return out;
}

ScoreResult finalize(const double* p, int n_buckets) {
  ScoreResult r;
  r.partials.assign(p, p + PRORL_N_PARTIALS);
  const double n = p[PRORL_P_N_ACTIVE] > 0 ? p[PRORL_P_N_ACTIVE] : 1.0;
  r.n_active = (std::int64_t)p[PRORL_P_N_ACTIVE];
  r.loss = p[PRORL_P_LOSS_SUM] / n;
  r.entropy = p[PRORL_P_ENTROPY_SUM] / n;
  r.logp = p[PRORL_P_LOGP_SUM] / n;
  r.ratio = p[PRORL_P_RATIO_SUM] / n;
  r.clip_lo_frac = p[PRORL_P_CLIP_LO] / n;
  r.clip_hi_frac = p[PRORL_P_CLIP_HI] / n;
  r.kl_k1 = p[PRORL_P_KL1_SUM] / n;
  r.kl_k3 = p[PRORL_P_KL_SUM] / n;
  r.adv_sum = p[PRORL_P_ADV_SUM];
  r.n_rollouts = (std::int64_t)p[PRORL_P_N_ROLLOUTS];
  for (int k = 0; k < n_buckets && k < PRORL_TURN_BUCKETS; ++k) {
    const double* b = p + PRORL_N_GLOBAL + PRORL_N_PER_TURN * k;
    if (b[0] <= 0) continue;
    r.per_turn.push_back({k, (std::int64_t)b[0], b[1] / b[0], b[2] / b[0], b[3] / b[0], b[4] / b[0]});
  }
  return r;
}

// ---- synthetic LM head -------------------------------------------------------------
SyntheticLogits::SyntheticLogits(int device, int vocab, LogitsDtype dtype, std::int64_t max_rows,
                                 std::uint64_t seed, float sigma)
    : vocab_(vocab), dtype_(dtype), max_rows_(max_rows), seed_(seed), sigma_(sigma) {
  throw_status(prorl_ctx_create(device, &ctx_));
  const size_t esz = dtype == LogitsDtype::BF16 ? 2 : 4;
  if (cudaMalloc(&buf_, (size_t)max_rows * (size_t)vocab * esz) != cudaSuccess ||
      cudaMalloc(&keys_, sizeof(std::int64_t) * (size_t)max_rows) != cudaSuccess) {
    prorl_ctx_destroy(ctx_);
    throw CudaError("SyntheticLogits: cudaMalloc failed");
  }
}

SyntheticLogits::~SyntheticLogits() {
  if (buf_) cudaFree(buf_);
  if (keys_) cudaFree(keys_);
  prorl_ctx_destroy(ctx_);
}

const void* SyntheticLogits::logits(std::int64_t, std::int64_t n, const std::int32_t* d_rows,
                                    const std::int32_t* d_seq, const std::int32_t* d_cu_seqlens,
                                    const std::int32_t* d_targets, const float* d_old_lp, std::int64_t* row_stride,
                                    void* stream) {
  if (n > max_rows_) throw ShapeMismatch("SyntheticLogits: micro-batch larger than max_rows");
  throw_status(prorl_row_keys(ctx_, d_rows, d_seq, d_cu_seqlens, nullptr, n, keys_, stream));
  throw_status(prorl_gen_logits_keyed(ctx_, buf_, (int)dtype_, vocab_, vocab_, n, keys_, d_targets, d_old_lp, seed_,
                                      sigma_, stream));
  *row_stride = vocab_;
  return buf_;
}

// ---- device scorer -----------------------------------------------------------------
DeviceScorer::DeviceScorer(int device) { throw_status(prorl_ctx_create(device, &ctx_)); }

DeviceScorer::~DeviceScorer() { prorl_ctx_destroy(ctx_); }

std::array<std::uint8_t, 128> DeviceScorer::nccl_unique_id() {
  std::array<std::uint8_t, 128> id{};
  throw_status(prorl_nccl_unique_id(id.data()));
  return id;
}

void DeviceScorer::init_nccl(int world, int rank, const std::array<std::uint8_t, 128>& id) {
  throw_status(prorl_nccl_init(ctx_, world, rank, id.data()));
}

namespace {
struct Trampoline {
  LogitsSource* src;
  std::string error;  // exception text captured across the C boundary
  int status = PRORL_OK;
};

int provide_logits(void* user, std::int64_t row0, std::int64_t n, const std::int32_t* d_rows,
                   const std::int32_t* d_seq, const std::int32_t* d_cu_seqlens, const std::int32_t* d_targets,
                   const float* d_old_lp, const void** d_logits, std::int64_t* row_stride, void* stream) {
  auto* t = static_cast<Trampoline*>(user);
  try {
    *d_logits = t->src->logits(row0, n, d_rows, d_seq, d_cu_seqlens, d_targets, d_old_lp, row_stride, stream);
    return PRORL_OK;
  } catch (const Error& e) {
    t->error = e.code() + ": " + e.what();
  } catch (const std::exception& e) {
    t->error = e.what();
  }
  t->status = PRORL_E_MALFORMED_REQUEST;
  return t->status;
}
}  // namespace

namespace {
struct GradTrampoline {
  GradSink* sink;
  std::string error;
  int status = PRORL_OK;
};

int consume_grad(void* user, std::int64_t row0, std::int64_t n, const void* d_grad, std::int64_t row_stride,
                 void* stream) {
  auto* t = static_cast<GradTrampoline*>(user);
  try {
    t->sink->gradient(row0, n, d_grad, row_stride, stream);
    return PRORL_OK;
  } catch (const Error& e) {
    t->error = e.code() + ": " + e.what();
  } catch (const std::exception& e) {
    t->error = e.what();
  }
  t->status = PRORL_E_MALFORMED_REQUEST;
  return t->status;
}

prorl_score_cfg to_c(const ScoreConfig& cfg) {
  prorl_score_cfg c{};
  c.loss.eps_lo = cfg.eps_lo;
  c.loss.eps_hi = cfg.eps_hi;
  c.loss.n_buckets = cfg.max_turn_buckets;
  c.loss.kl_coef = cfg.kl_coef;
  c.inv_temperature = cfg.inv_temperature;
  c.adv_eps = cfg.adv_eps;
  c.ddof = cfg.ddof;
  c.vocab = cfg.vocab;
  c.dtype = (int)cfg.dtype;
  c.microbatch_rows = cfg.microbatch_rows;
  return c;
}
int provide_ref(void* user, std::int64_t row0, std::int64_t n, const std::int32_t* d_rows, const std::int32_t* d_seq,
                const std::int32_t* d_cu_seqlens, const std::int32_t* d_targets, const float** d_ref_lp,
                void* stream) {
  auto* t = static_cast<Trampoline*>(user);
  try {
    *d_ref_lp = t->src->ref_logprobs(row0, n, d_rows, d_seq, d_cu_seqlens, d_targets, stream);
    if (*d_ref_lp) return PRORL_OK;
    t->error = "kl_coef != 0 but the logits source provides no reference logprobs";
  } catch (const Error& e) {
    t->error = e.code() + ": " + e.what();
  } catch (const std::exception& e) {
    t->error = e.what();
  }
  t->status = PRORL_E_MALFORMED_REQUEST;
  return t->status;
}
}  // namespace

ScoreResult DeviceScorer::score_batch(const HostBatch& batch, LogitsSource& logits, const ScoreConfig& cfg,
                                      void* stream) {
  return score_view(batch.view(), logits, cfg, stream);
}

IngestedBatch::IngestedBatch(const std::vector<std::string>& responses, const std::vector<std::int32_t>& group_off,
                             double gate_tolerance, int threads) {
  std::vector<const char*> ptrs(responses.size());
  std::vector<size_t> lens(responses.size());
  for (size_t i = 0; i < responses.size(); ++i) {
    ptrs[i] = responses[i].data();
    lens[i] = responses[i].size();
  }
  if (group_off.empty() || (size_t)group_off.back() != responses.size())
    throw MalformedRequest("IngestedBatch: group_off must end at the number of responses");
  throw_status(prorl_ingest_responses(ptrs.data(), lens.data(), group_off.data(), (std::int32_t)group_off.size() - 1,
                                      gate_tolerance, threads, &r_));
}

IngestedBatch::~IngestedBatch() { prorl_ingest_free(&r_); }

ScoreResult DeviceScorer::score_view(const prorl_host_batch& hb, LogitsSource& logits, const ScoreConfig& cfg,
                                     void* stream) {
  const prorl_score_cfg c = to_c(cfg);
  Trampoline tr{&logits, {}, PRORL_OK};
  prorl_logits_pool pool{};
  pool.provide = &provide_logits;
  pool.user = &tr;
  if (cfg.kl_coef != 0.f) {
    pool.provide_ref = &provide_ref;
    pool.ref_user = &tr;
  }
  double partials[PRORL_N_PARTIALS];
  float tm[5];
  const int st = prorl_score_host(ctx_, &hb, &c, &pool, partials, tm, stream);
  if (st != PRORL_OK && tr.status != PRORL_OK) throw MalformedRequest("logits source failed: " + tr.error);
  throw_status(st);
  ScoreResult r = finalize(partials, cfg.max_turn_buckets);
  std::memcpy(r.timings_ms, tm, sizeof tm);
  return r;
}

ScoreResult DeviceScorer::score_groups(const std::vector<PromptGroup>& groups, LogitsSource& logits,
                                       const ScoreConfig& cfg, void* stream) {
  return score_batch(build_host_batch(groups, cfg), logits, cfg, stream);
}

ScoreResult DeviceScorer::train_view(const prorl_host_batch& hb, LogitsSource& logits, GradSink& grads,
                                     const ScoreConfig& cfg, double n_global, void* stream) {
  const prorl_score_cfg c = to_c(cfg);
  Trampoline tr{&logits, {}, PRORL_OK};
  GradTrampoline gt{&grads, {}, PRORL_OK};
  prorl_logits_pool pool{};
  pool.provide = &provide_logits;
  pool.user = &tr;
  if (cfg.kl_coef != 0.f) {
    pool.provide_ref = &provide_ref;
    pool.ref_user = &tr;
  }
  pool.train = 1;
  pool.n_global = n_global;
  pool.consume_grad = &consume_grad;
  pool.grad_user = &gt;
  double partials[PRORL_N_PARTIALS];
  float tm[5];
  const int st = prorl_score_host(ctx_, &hb, &c, &pool, partials, tm, stream);
  if (st != PRORL_OK && tr.status != PRORL_OK) throw MalformedRequest("logits source failed: " + tr.error);
  if (st != PRORL_OK && gt.status != PRORL_OK) throw MalformedRequest("gradient sink failed: " + gt.error);
  throw_status(st);
  ScoreResult r = finalize(partials, cfg.max_turn_buckets);
  std::memcpy(r.timings_ms, tm, sizeof tm);
  return r;
}

ScoreResult DeviceScorer::train_groups(const std::vector<PromptGroup>& groups, LogitsSource& logits,
                                       GradSink& grads, const ScoreConfig& cfg, double n_global, void* stream) {
  const HostBatch b = build_host_batch(groups, cfg);
  return train_view(b.view(), logits, grads, cfg, n_global, stream);
}

// ---- wire ingestion ---------------------------------------------------------------
static Role role_from_name(const std::string& s) {
  if (s == "system") return Role::SYSTEM;
  if (s == "user") return Role::USER;
  if (s == "assistant") return Role::ASSISTANT;
  if (s == "tool") return Role::TOOL;
  throw MalformedTurn("unknown role '" + s + "'");
}

TokenTrajectory trajectory_from_json(const nlohmann::json& turns) {
  if (!turns.is_array()) throw MalformedRequest("trajectory must be an array of turns");
  TokenTrajectory traj;
  for (const auto& tj : turns) {
    if (!tj.is_object()) throw MalformedTurn("turn must be an object");
    Turn t;
    t.role = role_from_name(tj.at("role").get<std::string>());
    t.input_ids = tj.value("input_ids", TokenIds{});
    t.output_ids = tj.value("output_ids", TokenIds{});
    t.logprobs = tj.value("logprobs", std::vector<double>{});
    t.text = tj.value("text", std::string{});
    traj.append(std::move(t));  // validates (MalformedTurn)
  }
  return traj;
}

RolloutOutcome outcome_from_response(const nlohmann::json& resp) {
  if (!resp.is_object()) throw MalformedRequest("response must be an object");
  RolloutOutcome o;
  o.status = resp.value("status", std::string{});
  o.reward = resp.value("reward", 0.0);
  o.address = resp.value("backend", std::string{});
  if (resp.contains("trajectory")) o.trajectory = trajectory_from_json(resp.at("trajectory"));
  return o;
}

}  // namespace rollout::train
