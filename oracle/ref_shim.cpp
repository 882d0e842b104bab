// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. extern "C" entry points over the
// *unmodified* reference sources compiled from /root/reference by
// oracle/build_ref.sh into oracle/_ref/libref.so. Used by tests/ to pin the
// oracle restatement (oracle/oracle.c) and the product's host logic against
// the reference itself. Never linked into the product.
//
//   ref_flatten / ref_validate_turn  -> TokenTrajectory (trajectory.hpp:135-176)
//   ref_usable_rewards / ref_is_informative -> harness.cpp:84-102
//   ref_fnv1a64 / ref_hash_token(s) / ref_token_logprob -> mock/policy.cpp:10-53
//   ref_generate_workload_rewards    -> trainer/workload.cpp:62-107
//   ref_process_response             -> handlers.cpp:57-91 (the /process wire JSON)
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "rollout/backend_pool.hpp"
#include "rollout/clock.hpp"
#include "rollout/handler.hpp"
#include "rollout/job.hpp"
#include "rollout/mock/policy.hpp"
#include "rollout/trainer/harness.hpp"
#include "rollout/trainer/workload.hpp"
#include "rollout/trajectory.hpp"

using namespace rollout;

extern "C" {

// role: 0 system, 1 user, 2 assistant, 3 tool (trajectory.hpp Role order).
// Builds a Turn with the given field sizes and runs TokenTrajectory::validate.
int ref_validate_turn(int role, int n_input, int n_output, int n_logprobs) {
  Turn t;
  t.role = static_cast<Role>(role);
  t.input_ids.assign((size_t)n_input, 1);
  t.output_ids.assign((size_t)n_output, 1);
  t.logprobs.assign((size_t)n_logprobs, -1.0);
  try {
    TokenTrajectory::validate(t);
  } catch (const MalformedTurn&) {
    return 1;
  }
  return 0;
}

// Appends n_turns well-formed turns (assistant turns take ids as output_ids
// with aligned logprobs, others as input_ids) and returns flatten_range(begin,
// end) into out (capacity cap). Returns the length, or -1 on MalformedTurn.
int64_t ref_flatten(int n_turns, const int* roles, const int64_t* lens, const int64_t* ids, const double* lps,
                    int64_t begin, int64_t end, int64_t* out, int64_t cap) {
  TokenTrajectory traj;
  int64_t off = 0;
  try {
    for (int i = 0; i < n_turns; ++i) {
      TokenIds v(ids + off, ids + off + lens[i]);
      if (roles[i] == 2) {
        std::vector<double> lp(lps + off, lps + off + lens[i]);
        traj.append(make_assistant_turn(std::move(v), std::move(lp)));
      } else {
        Turn t;
        t.role = static_cast<Role>(roles[i]);
        t.input_ids = std::move(v);
        traj.append(std::move(t));
      }
      off += lens[i];
    }
  } catch (const MalformedTurn&) {
    return -1;
  }
  TokenIds f = traj.flatten_range((size_t)begin, (size_t)end);
  if ((int64_t)f.size() <= cap) std::memcpy(out, f.data(), f.size() * sizeof(int64_t));
  return (int64_t)f.size();
}

static train::PromptGroup make_group(int n, const int* has, const int* failed, const double* rewards) {
  train::PromptGroup g;
  g.prompt_id = "p";
  g.n = n;
  g.outcomes.resize((size_t)n);
  for (int i = 0; i < n; ++i) {
    if (!has[i]) continue;
    train::RolloutOutcome o;
    o.reward = rewards[i];
    o.status = failed[i] ? "FAILED" : "DONE";
    g.outcomes[(size_t)i] = o;
  }
  return g;
}

int ref_usable_rewards(int n, const int* has, const int* failed, const double* rewards, double* out) {
  auto r = make_group(n, has, failed, rewards).usable_rewards();
  for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
  return (int)r.size();
}

// 1 / 0, or -2 when IncompleteGroup is thrown.
int ref_is_informative(int n, const int* has, const int* failed, const double* rewards, double tol) {
  try {
    return train::is_informative(make_group(n, has, failed, rewards), tol) ? 1 : 0;
  } catch (const IncompleteGroup&) {
    return -2;
  }
}

uint64_t ref_fnv1a64(const void* data, size_t len) { return mock::fnv1a64(data, len); }

int64_t ref_hash_token(uint64_t seed, const int64_t* prompt, int64_t n_prompt, uint64_t k, int64_t vocab) {
  TokenIds p(prompt, prompt + n_prompt);
  return mock::hash_token(seed, p, k, vocab);
}

double ref_token_logprob(int64_t t) { return mock::token_logprob(t); }

// Bulk forms for building whole synthetic shards from the reference's own
// generators (bench.py --impl reference): out[i] = mock::hash_token(seed,
// prompt, k0 + i, vocab) and lp_out[i] = mock::token_logprob(out[i]).
void ref_hash_tokens(uint64_t seed, const int64_t* prompt, int64_t n_prompt, uint64_t k0, int64_t n, int64_t vocab,
                     int64_t* out, double* lp_out) {
  const TokenIds p(prompt, prompt + n_prompt);
  for (int64_t i = 0; i < n; ++i) {
    out[i] = mock::hash_token(seed, p, k0 + (uint64_t)i, vocab);
    if (lp_out) lp_out[i] = mock::token_logprob(out[i]);
  }
}

uint64_t ref_prompt_digest(const int64_t* prompt, int64_t n_prompt) {
  return mock::prompt_digest(TokenIds(prompt, prompt + n_prompt));
}

int ref_generate_workload_rewards(int num_prompts, int n, uint64_t seed, double p_informative, double* out) {
  train::WorkloadGenOptions o;
  o.num_prompts = num_prompts;
  o.rollouts_per_prompt = n;
  o.seed = seed;
  o.informative_probability = p_informative;
  auto w = train::generate_workload(o);
  for (int i = 0; i < num_prompts; ++i)
    for (int j = 0; j < n; ++j) out[(size_t)i * n + j] = w.prompts[(size_t)i].rewards[(size_t)j];
  return 0;
}

// Builds a Job with the given turns (assistant turns carry ids as output_ids
// with aligned logprobs), reward and terminal status (0 DONE, 1 FAILED,
// 2 CANCELLED), and returns build_process_response(job).dump() in out.
// Returns the JSON length (or the needed capacity if cap is too small),
// -1 on MalformedTurn.
int64_t ref_process_response(const char* job_id, int n_turns, const int* roles, const int64_t* lens,
                             const int64_t* ids, const double* lps, double reward, int status, const char* backend,
                             char* out, int64_t cap) {
  auto clock = std::make_shared<ManualClock>();
  Job job(job_id, "echo", nlohmann::json::object(), SamplingParams{}, std::chrono::seconds(60), clock);
  int64_t off = 0;
  try {
    for (int i = 0; i < n_turns; ++i) {
      TokenIds v(ids + off, ids + off + lens[i]);
      if (roles[i] == 2) {
        job.append_turn(make_assistant_turn(std::move(v), std::vector<double>(lps + off, lps + off + lens[i])));
      } else {
        Turn t;
        t.role = static_cast<Role>(roles[i]);
        t.input_ids = std::move(v);
        t.text = "t" + std::to_string(i);
        job.append_turn(std::move(t));
      }
      off += lens[i];
    }
  } catch (const MalformedTurn&) {
    return -1;
  }
  job.set_reward(reward);
  if (backend && backend[0]) job.record_backend(backend);
  clock->advance(std::chrono::milliseconds(5));
  job.try_terminal(status == 1 ? JobStatus::FAILED : (status == 2 ? JobStatus::CANCELLED : JobStatus::DONE));
  const std::string js = build_process_response(job).dump();
  if ((int64_t)js.size() <= cap) std::memcpy(out, js.data(), js.size());
  return (int64_t)js.size();
}

}  // extern "C"

// ---- link stubs: httplib-backed symbols harness.cpp references but the
// oracle never calls. They throw if ever reached.
namespace rollout {
namespace backend {
std::pair<std::string, int> parse_http_address(const std::string&) { throw Error("stub", "not linked"); }
GenerateResult BackendPool::generate(const std::string&, const TokenIds&, const SamplingParams&,
                                     const std::function<bool()>&) {
  throw Error("stub", "not linked");
}
}  // namespace backend
namespace train {
RolloutClient::RolloutClient(std::string, Duration) { throw Error("stub", "not linked"); }
RolloutClient::~RolloutClient() = default;
nlohmann::json RolloutClient::process(const nlohmann::json&) { throw Error("stub", "not linked"); }
nlohmann::json RolloutClient::cancel(const std::string&) { throw Error("stub", "not linked"); }
nlohmann::json RolloutClient::add_llm_server(const std::string&) { throw Error("stub", "not linked"); }
nlohmann::json RolloutClient::clear_llm_server() { throw Error("stub", "not linked"); }
nlohmann::json RolloutClient::status() { throw Error("stub", "not linked"); }
struct RolloutClient::Impl {};
}  // namespace train
}  // namespace rollout
