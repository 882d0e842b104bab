// The drop-in seam against the UNMODIFIED reference (built and run by
// tests/test_reference_seam.py). Compiled with the reference's own include
// root first — -I/root/reference/proj/include -Iinclude — so every rollout::
// type below is the reference's, and linked against oracle/_ref/libref.so (the
// reference's handlers.cpp, trainer/harness.cpp, mock/policy.cpp, ... compiled
// from /root/reference by oracle/build_ref.sh) and libprorl_hotpath.so.
//
// Flow, one step of what the harness seam does (harness.cpp:244-279, 313-316):
//   reference Job (job.hpp) with a multi-turn trajectory whose ids and
//   logprobs come from the reference's mock policy (policy.cpp:42-53)
//   -> build_process_response (handlers.cpp:57-91) -> wire text -> parse
//   -> record_response (façade; the harness's recording rule + the trajectory)
//   -> groups handed over in completion order, one CANCELLED response re-issued
//   -> build_host_batch (façade; is_informative and usable_rewards are the
//      reference's, harness.cpp:84-102) -> JSON for the Python side, which
//      checks it against the oracle and the reference's own flatten().
//   --gpu: DeviceScorer::score_groups / train_groups on cuda:0 as well.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "rollout/clock.hpp"
#include "rollout/handler.hpp"
#include "rollout/job.hpp"
#include "rollout/mock/policy.hpp"
#include "rollout/trainer/harness.hpp"
#include "rollout/trajectory.hpp"
// this repo's façade (include/rollout/trainer/, no file shared with the reference tree)
#include "rollout/trainer/scoring.hpp"
#include "rollout/trainer/synthetic_logits.hpp"

using namespace rollout;
using namespace rollout::train;

static int g_fail = 0;
#define CHECK(cond)                                                                  \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                                      \
    }                                                                                \
  } while (0)

constexpr int kVocab = 4099;
constexpr int kGroups = 7, kN = 4;

// A reference Job holding a user prompt and alternating assistant / tool turns;
// assistant ids are mock::hash_token(seed, prompt, k) and their logprobs
// mock::token_logprob(id) — exactly what the reference's mock backend returns.
static nlohmann::json run_job(int g, int slot, JobStatus status, double reward) {
  auto clock = std::make_shared<ManualClock>();
  const std::string id = "job-" + std::to_string(g) + "-" + std::to_string(slot);
  Job job(id, "arith", nlohmann::json::object(), SamplingParams{}, std::chrono::seconds(60), clock);
  TokenIds prompt;
  for (int i = 0; i < 6 + (g + slot) % 5; ++i) prompt.push_back((TokenId)((97 * g + 31 * slot + 7 * i) % kVocab));
  Turn u;
  u.role = Role::USER;
  u.input_ids = prompt;
  u.text = "task";
  job.append_turn(std::move(u));
  std::uint64_t k = 0;
  const int n_turns = 2 + (g * 3 + slot) % 6;
  for (int t = 0; t < n_turns; ++t) {
    if (t % 2 == 0) {
      TokenIds out;
      std::vector<double> lp;
      for (int i = 0; i < 3 + (g + t + slot) % 7; ++i) {
        out.push_back(mock::hash_token(2603, prompt, k++, kVocab));
        lp.push_back(mock::token_logprob(out.back()));
      }
      job.append_turn(make_assistant_turn(std::move(out), std::move(lp), "step"));
    } else {
      Turn tool;
      tool.role = Role::TOOL;
      for (int i = 0; i < 2 + (g + t) % 4; ++i) tool.input_ids.push_back((TokenId)((13 * g + 5 * t + i) % kVocab));
      tool.text = "observation";
      job.append_turn(std::move(tool));
    }
  }
  job.set_reward(reward);
  job.record_backend("http://127.0.0.1:9000");
  clock->advance(std::chrono::milliseconds(3));
  job.try_terminal(status);
  return build_process_response(job);
}

struct Arrival {
  int g, slot;
  nlohmann::json wire;  // the response as the harness's client returns it (parsed text)
};

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "--gpu") == 0;
  // The iteration's groups as the harness builds them (harness.cpp:155-165).
  std::vector<PromptGroup> groups(kGroups);
  for (int g = 0; g < kGroups; ++g) {
    groups[g].prompt_id = "prompt-" + std::to_string(100 + 37 * g % 11);  // ids not in creation order
    groups[g].n = kN;
    groups[g].outcomes.assign(kN, std::nullopt);
  }
  // Rollout responses, in a scrambled completion order. Rewards: group 3 all
  // equal (not informative), group 5 has a FAILED rollout, group 1 slot 2 first
  // comes back CANCELLED and is re-issued (harness.cpp:264).
  std::vector<Arrival> arrivals;
  for (int g = 0; g < kGroups; ++g)
    for (int s = 0; s < kN; ++s) {
      const double reward = g == 3 ? 1.0 : (double)((g + s) % 2);
      const JobStatus st = (g == 5 && s == 1) ? JobStatus::FAILED : JobStatus::DONE;
      arrivals.push_back({g, s, nlohmann::json::parse(run_job(g, s, st, reward).dump())});
    }
  arrivals.insert(arrivals.begin() + 3, {1, 2, nlohmann::json::parse(run_job(1, 2, JobStatus::CANCELLED, 1.0).dump())});
  std::mt19937 rng(7);
  std::shuffle(arrivals.begin() + 4, arrivals.end(), rng);

  TrajectoryTable table;
  int recorded = 0;
  for (const Arrival& a : arrivals) recorded += record_response(groups[a.g], a.slot, a.wire, table, 0.003) ? 1 : 0;
  CHECK(recorded == kGroups * kN);  // the CANCELLED response did not fill its slot
  {  // the hook form (integration/reference.patch): keep_trajectory stores what record_response stored
    TrajectoryTable t2;
    for (const Arrival& a : arrivals)
      if (a.wire.value("status", std::string("FAILED")) != "CANCELLED") keep_trajectory(t2, groups[a.g], a.slot, a.wire);
    CHECK(t2.size() == table.size());
    for (int g = 0; g < kGroups; ++g)
      for (int s = 0; s < kN; ++s) {
        const TokenTrajectory* x = table.find(groups[g].prompt_id, s);
        const TokenTrajectory* y = t2.find(groups[g].prompt_id, s);
        CHECK((x == nullptr) == (y == nullptr));
        if (x && y) CHECK(x->flatten() == y->flatten());
      }
  }
  for (const auto& g : groups) CHECK(g.complete());
  CHECK(groups[5].outcomes[1]->status == "FAILED" && table.find(groups[5].prompt_id, 1) == nullptr);
  CHECK(groups[5].usable_rewards().size() == kN - 1);  // reference harness.cpp:84-90
  CHECK(!is_informative(groups[3]));                    // reference harness.cpp:92-102

  // IterationStats::informative in completion order (harness.cpp:313-316) —
  // here simply reversed; the façade packs in prompt_id order either way.
  std::vector<PromptGroup> handed(groups.rbegin(), groups.rend());
  ScoreConfig cfg;
  cfg.vocab = kVocab;
  cfg.dtype = LogitsDtype::BF16;
  cfg.microbatch_rows = 48;
  const HostBatch hb = build_host_batch(handed, table, cfg);
  const HostBatch hb2 = build_host_batch(groups, table, cfg);
  CHECK(hb.ids == hb2.ids && hb.reward == hb2.reward && hb.prompt_ids == hb2.prompt_ids);
  CHECK(std::is_sorted(hb.prompt_ids.begin(), hb.prompt_ids.end()));

  // a group still holding a CANCELLED outcome is incomplete
  auto bad = groups;
  bad[0].outcomes[0]->status = "CANCELLED";
  bool threw = false;
  try {
    build_host_batch(bad, table, cfg);
  } catch (const IncompleteGroup& e) {
    threw = e.code() == "incomplete_group";
  }
  CHECK(threw);
  if (g_fail) {
    std::fprintf(stderr, "%d checks failed\n", g_fail);
    return 1;
  }

  // JSON: the host batch, plus each usable rollout's reference flatten() and
  // its assistant mask, in the order the batch must hold them.
  std::printf("{\"turns\":[");
  for (std::size_t i = 0; i < hb.turns.size(); ++i)
    std::printf("%s[%lld,%d,%d,%d]", i ? "," : "", (long long)hb.turns[i].src_off, hb.turns[i].traj, hb.turns[i].len,
                (int)hb.turns[i].role);
  std::printf("],\"ids\":%s,\"lp\":%s,\"reward\":%s,\"usable\":%s,\"group_off\":%s,\"prompt_ids\":%s,\"n_active\":%lld",
              nlohmann::json(hb.ids).dump().c_str(), nlohmann::json(hb.lp).dump().c_str(),
              nlohmann::json(hb.reward).dump().c_str(), nlohmann::json(hb.usable).dump().c_str(),
              nlohmann::json(hb.group_off).dump().c_str(), nlohmann::json(hb.prompt_ids).dump().c_str(),
              (long long)hb.n_active);
  nlohmann::json expect = nlohmann::json::array();
  std::vector<std::size_t> order(groups.size());
  for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
  std::sort(order.begin(), order.end(), [&](auto a, auto b) { return groups[a].prompt_id < groups[b].prompt_id; });
  for (std::size_t gi : order) {
    const PromptGroup& g = groups[gi];
    const bool info = is_informative(g);
    for (int s = 0; s < kN; ++s) {
      const TokenTrajectory* t = table.find(g.prompt_id, s);
      if (!info || g.outcomes[s]->status == "FAILED" || !t) {
        expect.push_back(nullptr);
        continue;
      }
      std::vector<int> mask;
      for (const Turn& turn : t->turns()) {
        const std::size_t n = turn.role == Role::ASSISTANT ? turn.output_ids.size() : turn.input_ids.size();
        mask.insert(mask.end(), n, turn.role == Role::ASSISTANT ? 1 : 0);
      }
      expect.push_back({{"flatten", t->flatten()}, {"mask", mask}});
    }
  }
  std::printf(",\"expect\":%s", expect.dump().c_str());

  if (gpu) {
    DeviceScorer scorer(0);
    SyntheticLogits lm(0, cfg.vocab, cfg.dtype, cfg.microbatch_rows, /*seed=*/77, 2.0f);
    const ScoreResult r = scorer.score_groups(handed, table, lm, cfg);
    std::printf(",\"partials\":%s", nlohmann::json(r.partials).dump().c_str());
    struct Count : GradSink {
      long long rows = 0;
      void gradient(std::int64_t, std::int64_t n, const void*, std::int64_t, void*) override { rows += n; }
    } sink;
    SyntheticLogits lm2(0, cfg.vocab, cfg.dtype, cfg.microbatch_rows, /*seed=*/77, 2.0f);
    const ScoreResult tr = scorer.train_groups(handed, table, lm2, sink, cfg);
    std::printf(",\"train_partials\":%s,\"grad_rows\":%lld", nlohmann::json(tr.partials).dump().c_str(), sink.rows);
  }
  std::printf("}\n");
  return 0;
}
