// score_responses — the reference-facing flow end to end in C++:
//   /process wire JSON (one response per line, proj/src/handlers.cpp:57-91)
//   -> rollout::train::IngestedBatch (usable_rewards / is_informative applied)
//   -> DeviceScorer (pack, GRPO, logprob/entropy + DAPO loss on sm_100a,
//      NCCL all-reduce when several ranks) with the deterministic synthetic
//      LM head -> metrics as one JSON line.
//   --train: the training step instead (DeviceScorer::train_view, K7): the same
//      metrics plus dL/dlogits per micro-batch, handed to a GradSink where the
//      trainer's LM-head backward would run (here: counted).
//
//   score_responses <responses.jsonl> <group_size> <vocab> [bf16|fp32] [seed] [--train]
//
// Build (standalone: no reference tree; the façade is header-only):
//   g++ -std=c++17 -Iinclude -Iinclude/standalone -I<json.hpp dir> -I/usr/local/cuda/include \
//       tools/score_responses.cpp -Lpaper_2603_18815_b200 -lprorl_hotpath -L/usr/local/cuda/lib64 -lcudart
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "rollout/trainer/scoring.hpp"
#include "rollout/trainer/synthetic_logits.hpp"

using namespace rollout::train;

// Stand-in for the trainer's LM-head backward: records the hand-offs.
struct CountingSink : GradSink {
  long long batches = 0, rows = 0;
  void gradient(std::int64_t /*row0*/, std::int64_t n, const void* /*d_grad*/, std::int64_t /*row_stride*/,
                void* /*stream*/) override {
    ++batches;
    rows += n;
  }
};

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s responses.jsonl group_size vocab [bf16|fp32] [seed]\n", argv[0]);
    return 2;
  }
  std::ifstream in(argv[1]);
  std::vector<std::string> resp;
  for (std::string line; std::getline(in, line);)
    if (!line.empty()) resp.push_back(line);
  const int gs = std::stoi(argv[2]);
  ScoreConfig cfg;
  cfg.vocab = std::stoi(argv[3]);
  cfg.dtype = (argc > 4 && std::string(argv[4]) == "fp32") ? LogitsDtype::FP32 : LogitsDtype::BF16;
  const std::uint64_t seed = argc > 5 ? std::stoull(argv[5]) : 0;
  const bool train = argc > 6 && std::string(argv[6]) == "--train";
  cfg.microbatch_rows = 4096;
  std::vector<std::int32_t> goff;
  for (size_t i = 0; i <= resp.size(); i += (size_t)gs) goff.push_back((std::int32_t)i);
  if ((size_t)goff.back() != resp.size()) goff.push_back((std::int32_t)resp.size());
  try {
    const auto t0 = std::chrono::steady_clock::now();
    IngestedBatch batch(resp, goff);
    const auto t1 = std::chrono::steady_clock::now();
    DeviceScorer scorer(0);
    SyntheticLogits lm(0, cfg.vocab, cfg.dtype, cfg.microbatch_rows, seed);
    CountingSink sink;
    const ScoreResult r = train ? scorer.train_view(batch.view(), lm, sink, cfg) : scorer.score_view(batch.view(), lm, cfg);
    std::printf("{\"responses\":%zu,\"n_informative\":%d,\"n_active\":%lld,\"ingest_ms\":%.3f,\"loss\":%.17g,"
                "\"entropy\":%.17g,\"logp\":%.17g,\"clip_lo_frac\":%.17g,\"clip_hi_frac\":%.17g,\"partials\":[",
                resp.size(), batch.n_informative(), (long long)r.n_active,
                std::chrono::duration<double, std::milli>(t1 - t0).count(), r.loss, r.entropy, r.logp,
                r.clip_lo_frac, r.clip_hi_frac);
    for (size_t i = 0; i < r.partials.size(); ++i) std::printf("%s%.17g", i ? "," : "", r.partials[i]);
    std::printf("],\"grad_batches\":%lld,\"grad_rows\":%lld}\n", sink.batches, sink.rows);
  } catch (const rollout::Error& e) {
    std::fprintf(stderr, "%s: %s\n", e.code().c_str(), e.what());
    return 1;
  }
  return 0;
}
