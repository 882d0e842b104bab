// C++ drop-in surface test (built and run by tests/test_cpp_facade.py).
//   ./test_scoring          host-only checks (no GPU needed)
//   ./test_scoring --gpu    also runs DeviceScorer::score_groups on cuda:0 and
//                           prints the host batch + partials as JSON for the
//                           Python side to check against the CPU oracle.
// The host-only cases restate the reference's own tests for the types the
// path consumes: proj/tests/test_core.cpp:130-170 (flatten, malformed turns),
// proj/tests/test_trainer.cpp:148-166 (informative filter), and the response
// schema of proj/tests/test_handlers.cpp:154-173 (ids [104,105], [300,7]).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include <cuda_runtime.h>

#include "rollout/trainer/scoring.hpp"
#include "rollout/trainer/synthetic_logits.hpp"

using namespace rollout;
using namespace rollout::train;

static int g_fail = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                          \
    }                                                                    \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f, const char* code) {
  try {
    f();
  } catch (const E& e) {
    return e.code() == code;
  } catch (...) {
    return false;
  }
  return false;
}

static std::optional<RolloutOutcome> outcome(double r, const char* status = "DONE") {
  RolloutOutcome o;
  o.reward = r;
  o.status = status;
  return o;
}

static PromptGroup group_of(std::vector<std::optional<RolloutOutcome>> os, std::string id = "p") {
  PromptGroup g;
  g.prompt_id = std::move(id);
  g.n = (int)os.size();
  g.outcomes = std::move(os);
  return g;
}

static TokenTrajectory traj(std::uint64_t key, int turns, int vocab) {
  // user prompt, then alternating assistant / tool turns
  TokenTrajectory t;
  auto id = [&](int k) { return (TokenId)((key * 2654435761u + 97u * (std::uint64_t)k) % (std::uint64_t)vocab); };
  int k = 0;
  TokenIds u;
  for (int i = 0; i < 5 + (int)(key % 3); ++i) u.push_back(id(k++));
  t.append(make_user_turn(u, "prompt"));
  for (int i = 0; i < turns; ++i) {
    TokenIds ids;
    std::vector<double> lp;
    const int n = 3 + (int)((key + i) % 5);
    for (int j = 0; j < n; ++j) {
      ids.push_back(id(k++));
      lp.push_back(-(1.0 + (double)(ids.back() % 7) / 10.0));
    }
    if (i % 2 == 0) t.append(make_assistant_turn(ids, lp));
    else t.append(make_tool_turn(ids));
  }
  return t;
}

static void host_checks() {
  // test_core.cpp:130-142
  TokenTrajectory t;
  t.append(make_user_turn({1, 2, 3}, "abc"));
  t.append(make_assistant_turn({10, 11}, {-1.0, -1.1}));
  t.append(make_tool_turn({4}, "d"));
  t.append(make_assistant_turn({12}, {-1.2}));
  CHECK(t.size() == 4);
  CHECK(t.flatten() == (TokenIds{1, 2, 3, 10, 11, 4, 12}));
  CHECK(t.flatten_range(1, 3) == (TokenIds{10, 11, 4}));
  CHECK(t.flatten_range(3, 99) == (TokenIds{12}));
  CHECK(t.flatten_range(2, 2).empty());

  // test_core.cpp:144-170
  TokenTrajectory e;
  Turn bad;
  bad.role = Role::ASSISTANT;
  bad.input_ids = {1};
  CHECK(throws<MalformedTurn>([&] { e.append(bad); }, "malformed_turn"));
  Turn mis;
  mis.role = Role::ASSISTANT;
  mis.output_ids = {1, 2};
  mis.logprobs = {-1.0};
  CHECK(throws<MalformedTurn>([&] { e.append(mis); }, "malformed_turn"));
  Turn uo;
  uo.role = Role::USER;
  uo.output_ids = {5};
  CHECK(throws<MalformedTurn>([&] { e.append(uo); }, "malformed_turn"));
  Turn tl;
  tl.role = Role::TOOL;
  tl.logprobs = {-1.0};
  CHECK(throws<MalformedTurn>([&] { e.append(tl); }, "malformed_turn"));
  CHECK(e.empty());

  // test_trainer.cpp:148-166
  CHECK(!is_informative(group_of({outcome(1), outcome(1), outcome(1), outcome(1)})));
  CHECK(is_informative(group_of({outcome(1), outcome(0), outcome(1), outcome(1)})));
  CHECK(!is_informative(group_of({outcome(1), outcome(1), outcome(0, "FAILED"), outcome(1)})));
  CHECK(!is_informative(group_of({outcome(1), outcome(0, "FAILED")})));
  auto near = group_of({outcome(0.0), outcome(0.1)});
  CHECK(is_informative(near));
  CHECK(!is_informative(near, 0.1));
  CHECK(is_informative(near, 0.099));
  auto partial = group_of({outcome(1), std::nullopt});
  CHECK(throws<IncompleteGroup>([&] { is_informative(partial); }, "incomplete_group"));
  CHECK((group_of({outcome(1), outcome(0, "FAILED"), outcome(0.5)}).usable_rewards() == std::vector<double>{1, 0.5}));

  // response schema (handlers.cpp:57-91; ids as in test_handlers.cpp:154-173)
  const char* resp = R"({"job_id":"j1","status":"DONE","reward":1.0,
    "trajectory":[{"role":"user","input_ids":[104,105],"output_ids":[],"logprobs":[],"text":"hi"},
                  {"role":"assistant","input_ids":[],"output_ids":[300,7],"logprobs":[-1.0,-1.3],"text":""}],
    "timings":{"init_seconds":0.0,"run_seconds":0.1,"eval_seconds":0.0,"queue_seconds":0.0},
    "backend":"http://127.0.0.1:9000"})";
  RolloutOutcome o = outcome_from_response(nlohmann::json::parse(resp));
  CHECK(o.status == "DONE" && o.reward == 1.0 && o.address == "http://127.0.0.1:9000");
  TrajectoryTable table;
  PromptGroup rg = group_of({std::nullopt, std::nullopt}, "r");
  CHECK(record_response(rg, 1, nlohmann::json::parse(resp), table, 0.25));
  CHECK(rg.outcomes[1] && rg.outcomes[1]->status == "DONE" && rg.outcomes[1]->wall_seconds == 0.25);
  const TokenTrajectory* rt = table.find("r", 1);
  CHECK(rt && rt->flatten() == (TokenIds{104, 105, 300, 7}));
  CHECK(rt && rt->turns()[1].logprobs == (std::vector<double>{-1.0, -1.3}));
  // harness.cpp:263-265: a missing status records FAILED, CANCELLED is not recorded
  CHECK(outcome_from_response(nlohmann::json::parse(R"({"reward":1.0})")).status == "FAILED");
  CHECK(!record_response(rg, 0, nlohmann::json::parse(R"({"status":"CANCELLED","reward":1.0,"trajectory":[]})"),
                         table));
  CHECK(!rg.outcomes[0] && table.find("r", 0) == nullptr);
  CHECK(record_response(rg, 0, nlohmann::json::parse(R"({"reward":0.0})"), table));  // FAILED: no trajectory needed
  CHECK(rg.outcomes[0]->status == "FAILED" && table.find("r", 0) == nullptr);
  CHECK(throws<MalformedRequest>([&] { record_response(rg, 0, nlohmann::json::parse(R"({"status":"DONE"})"), table); },
                                 "malformed_request"));
  auto bad_json = nlohmann::json::parse(R"([{"role":"assistant","input_ids":[1],"output_ids":[],"logprobs":[]}])");
  CHECK(throws<MalformedTurn>([&] { trajectory_from_json(bad_json); }, "malformed_turn"));
  CHECK(throws<MalformedTurn>([&] { trajectory_from_json(nlohmann::json::parse(R"([{"role":"robot"}])")); },
                              "malformed_turn"));

  // build_host_batch: FAILED slot and a non-informative group contribute empty sequences
  ScoreConfig cfg;
  cfg.vocab = 50000;
  std::vector<PromptGroup> gs;
  TrajectoryTable tt;
  {
    std::vector<std::optional<RolloutOutcome>> os;
    for (int i = 0; i < 4; ++i) {
      os.push_back(outcome(i % 2 ? 1.0 : 0.0, i == 3 ? "FAILED" : "DONE"));
      tt.put("a", i, traj(10 + i, 3, 50000));
    }
    std::vector<std::optional<RolloutOutcome>> os2;
    for (int i = 0; i < 2; ++i) {
      os2.push_back(outcome(1.0));
      tt.put("b", i, traj(20 + i, 3, 50000));
    }
    // handed over in completion order "b" before "a": packed in prompt_id order (App. B.1)
    gs.push_back(group_of(os2, "b"));
    gs.push_back(group_of(os, "a"));
  }
  HostBatch hb = build_host_batch(gs, tt, cfg);
  CHECK((hb.prompt_ids == std::vector<std::string>{"a", "b"}));
  CHECK(hb.reward.size() == 6 && hb.usable.size() == 6);
  CHECK((hb.group_off == std::vector<std::int32_t>{0, 4, 6}));
  CHECK(hb.usable[3] == 0 && hb.usable[0] == 1);
  CHECK(hb.turns.size() == 3 * 4);  // 3 usable rollouts of the informative group x 4 turns
  std::int64_t toks = 0, act = 0;
  for (int s = 0; s < 3; ++s) {
    const TokenTrajectory tr = traj(10 + s, 3, 50000);
    toks += (std::int64_t)tr.flatten().size();
    for (const Turn& tt : tr.turns())
      if (tt.role == Role::ASSISTANT) act += (std::int64_t)tt.output_ids.size();
  }
  CHECK((std::int64_t)hb.ids.size() == toks && hb.lp.size() == hb.ids.size());
  CHECK(hb.n_active == act);  // first turns are user turns: every policy token has a predecessor
  for (const auto& d : hb.turns) CHECK(d.traj >= 0 && d.traj < 3);
  {
    const HostBatch again = build_host_batch(std::vector<PromptGroup>{gs[1], gs[0]}, tt, cfg);
    CHECK(again.ids == hb.ids && again.reward == hb.reward && again.group_off == hb.group_off);
  }
  TrajectoryTable partial_table;
  partial_table.put("a", 1, traj(11, 3, 50000));
  CHECK(throws<MalformedRequest>([&] { build_host_batch(gs, partial_table, cfg); }, "malformed_request"));
  auto cancelled = gs;
  cancelled[0].outcomes[1]->status = "CANCELLED";
  CHECK(throws<IncompleteGroup>([&] { build_host_batch(cancelled, tt, cfg); }, "incomplete_group"));
  // the host gate takes the tolerance (K3 gates with the same value, prorl_score_cfg.gate_tolerance)
  ScoreConfig tol_cfg = cfg;
  tol_cfg.gate_tolerance = 1.0;
  CHECK(build_host_batch(gs, tt, tol_cfg).turns.empty());
  tt.erase_group("b");
  CHECK(tt.size() == 4 && tt.find("b", 0) == nullptr && tt.find("a", 0) != nullptr);

  // deterministic LPT sharding; groups never split
  std::vector<PromptGroup> many;
  TrajectoryTable mt;
  for (int gi = 0; gi < 7; ++gi) {
    std::vector<std::optional<RolloutOutcome>> os;
    const std::string id = "g" + std::to_string(gi);
    for (int i = 0; i < 2; ++i) {
      os.push_back(outcome(i));
      mt.put(id, i, traj(100 + 7 * (gi % 4) + i, 1 + 2 * (gi % 4), 50000));  // equal loads: ties
    }
    many.push_back(group_of(os, id));
  }
  auto sh = shard_groups(many, mt, 3);
  CHECK(sh.size() == 3);
  std::size_t total = 0;
  for (auto& s : sh) {
    total += s.size();
    for (std::size_t i = 1; i < s.size(); ++i) CHECK(s[i - 1].prompt_id < s[i].prompt_id);
  }
  CHECK(total == many.size());
  // every rank computes the same assignment whatever order the groups arrived in
  auto rev = many;
  std::reverse(rev.begin(), rev.end());
  auto sh2 = shard_groups(rev, mt, 3);
  for (int r = 0; r < 3; ++r) {
    CHECK(sh[r].size() == sh2[r].size());
    for (std::size_t i = 0; i < sh[r].size() && i < sh2[r].size(); ++i) CHECK(sh[r][i].prompt_id == sh2[r][i].prompt_id);
  }

  // finalize
  std::vector<double> p(PRORL_N_PARTIALS, 0.0);
  p[PRORL_P_LOSS_SUM] = 3.0;
  p[PRORL_P_N_ACTIVE] = 6.0;
  p[PRORL_P_ENTROPY_SUM] = 12.0;
  p[PRORL_N_GLOBAL + 5 * 2 + 0] = 6.0;
  p[PRORL_N_GLOBAL + 5 * 2 + 1] = 3.0;
  ScoreResult r = finalize(p.data());
  CHECK(r.loss == 0.5 && r.entropy == 2.0 && r.n_active == 6);
  CHECK(r.per_turn.size() == 1 && r.per_turn[0].turn == 2 && r.per_turn[0].loss == 0.5);

  // C-ABI status -> exception mapping
  CHECK(throws<ShapeMismatch>([] { throw_status(PRORL_E_SHAPE); }, "shape_mismatch"));
  CHECK(throws<CudaError>([] { throw_status(PRORL_E_CUDA); }, "cuda_error"));
}

static void print_array(const char* name, const std::vector<double>& v) {
  std::printf("\"%s\":[", name);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? "," : "", v[i]);
  std::printf("]");
}

static int gpu_run() {
  const int V = 4099;  // odd vocabulary: unaligned row heads/tails
  ScoreConfig cfg;
  cfg.vocab = V;
  cfg.dtype = LogitsDtype::BF16;
  cfg.microbatch_rows = 64;
  std::vector<PromptGroup> groups;
  TrajectoryTable table;
  for (int gi = 0; gi < 6; ++gi) {
    std::vector<std::optional<RolloutOutcome>> os;
    const std::string id = "p" + std::to_string(gi);
    for (int i = 0; i < 4; ++i) {
      os.push_back(outcome((gi + i) % 3 == 0 ? 1.0 : 0.0, (gi == 2 && i == 1) ? "FAILED" : "DONE"));
      table.put(id, i, traj(1000 + 4 * gi + i, 2 + (gi % 5) * 3, V));
    }
    groups.push_back(group_of(os, id));
  }
  DeviceScorer scorer(0);
  SyntheticLogits lm(0, V, cfg.dtype, cfg.microbatch_rows, /*seed=*/4242, 2.0f);
  const HostBatch hb = build_host_batch(groups, table, cfg);
  const ScoreResult r = scorer.score_groups(groups, table, lm, cfg);
  std::printf("{\"n_active_host\":%lld,", (long long)hb.n_active);
  std::printf("\"turns\":[");
  for (std::size_t i = 0; i < hb.turns.size(); ++i)
    std::printf("%s[%lld,%d,%d,%d]", i ? "," : "", (long long)hb.turns[i].src_off, hb.turns[i].traj, hb.turns[i].len,
                (int)hb.turns[i].role);
  std::printf("],\"ids\":[");
  for (std::size_t i = 0; i < hb.ids.size(); ++i) std::printf("%s%lld", i ? "," : "", (long long)hb.ids[i]);
  std::printf("],");
  print_array("lp", hb.lp);
  std::printf(",");
  print_array("reward", hb.reward);
  std::printf(",\"usable\":[");
  for (std::size_t i = 0; i < hb.usable.size(); ++i) std::printf("%s%d", i ? "," : "", (int)hb.usable[i]);
  std::printf("],\"group_off\":[");
  for (std::size_t i = 0; i < hb.group_off.size(); ++i) std::printf("%s%d", i ? "," : "", hb.group_off[i]);
  std::printf("],");
  print_array("partials", r.partials);
  std::printf(",\"loss\":%.17g,\"n_active\":%lld,\"per_turn\":%zu,", r.loss, (long long)r.n_active,
              r.per_turn.size());

  // training step through the façade: gradient per micro-batch handed to a sink
  struct Sink : GradSink {
    int V;
    std::vector<std::pair<long long, long long>> batches;
    double max_row_sum_rel = 0.0;
    bool finite = true;
    long long nonzero_rows = 0;
    void gradient(std::int64_t row0, std::int64_t n, const void* d_grad, std::int64_t row_stride,
                  void* stream) override {
      batches.emplace_back(row0, n);
      std::vector<std::uint16_t> h((size_t)n * row_stride);
      cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
      cudaMemcpy(h.data(), d_grad, h.size() * 2, cudaMemcpyDeviceToHost);
      for (std::int64_t i = 0; i < n; ++i) {
        double sum = 0.0, mx = 0.0;
        for (int v = 0; v < V; ++v) {
          std::uint32_t b = (std::uint32_t)h[(size_t)i * row_stride + v] << 16;
          float f;
          std::memcpy(&f, &b, 4);
          if (!std::isfinite(f)) finite = false;
          sum += f;
          mx = std::max(mx, (double)std::fabs(f));
        }
        if (mx > 0) {
          ++nonzero_rows;
          max_row_sum_rel = std::max(max_row_sum_rel, std::fabs(sum) / mx);
        }
      }
    }
  } sink;
  sink.V = V;
  SyntheticLogits lm2(0, V, cfg.dtype, cfg.microbatch_rows, /*seed=*/4242, 2.0f);
  const ScoreResult tr = scorer.train_groups(groups, table, lm2, sink, cfg);
  print_array("train_partials", tr.partials);
  std::printf(",\"grad_batches\":[");
  for (std::size_t i = 0; i < sink.batches.size(); ++i)
    std::printf("%s[%lld,%lld]", i ? "," : "", sink.batches[i].first, sink.batches[i].second);
  std::printf("],\"grad_finite\":%d,\"grad_nonzero_rows\":%lld,\"grad_max_row_sum_rel\":%.6g}\n",
              sink.finite ? 1 : 0, sink.nonzero_rows, sink.max_row_sum_rel);
  return 0;
}

int main(int argc, char** argv) {
  host_checks();
  if (g_fail) {
    std::fprintf(stderr, "%d host checks failed\n", g_fail);
    return 1;
  }
  if (argc > 1 && std::strcmp(argv[1], "--gpu") == 0) return gpu_run();
  std::printf("host checks OK\n");
  return 0;
}
