// workload.cpp — synthetic per-rollout rewards with the semantics of the
// reference's trainer workload generator (proj/src/trainer/workload.cpp:62-107):
// a seeded std::mt19937_64; per prompt, with probability p_informative a
// "mixed" reward vector with k ~ U{1..n-1} successes at shuffled slots, else a
// uniform 0/1 vector; then one straggler / latency draw per rollout (kept so
// the engine state — and thus the next prompt's draws — matches the
// reference's sequence exactly). Same libstdc++ distributions as the
// reference build, so the values are identical to generate_workload's; the
// oracle test (tests/test_oracle_golden.py) checks that against the compiled
// reference. Host-only C++; used to build synthetic batches, not on the
// device path.
#include <algorithm>
#include <cstdint>
#include <random>
#include <vector>

#include "prorl_hotpath.h"

extern "C" int prorl_synth_rewards(int32_t num_prompts, int32_t n, uint64_t seed, double p_informative,
                                   double* out) {
  if (num_prompts < 1 || n < 1 || !out) return PRORL_E_MALFORMED_REQUEST;
  std::mt19937_64 rng(seed);
  std::bernoulli_distribution informative(p_informative);
  std::bernoulli_distribution straggler(0.10);                     // WorkloadGenOptions defaults
  std::uniform_real_distribution<double> base_ms(30.0, 150.0);     // (workload.hpp:37-41)
  std::uniform_real_distribution<double> tail_ms(800.0, 1500.0);
  std::bernoulli_distribution coin(0.5);
  for (int32_t i = 0; i < num_prompts; ++i) {
    double* r = out + (size_t)i * n;
    std::fill(r, r + n, 0.0);
    if (n >= 2 && informative(rng)) {
      std::uniform_int_distribution<int> k_dist(1, n - 1);
      int k = k_dist(rng);
      std::vector<std::size_t> idx((size_t)n);
      for (std::size_t j = 0; j < idx.size(); ++j) idx[j] = j;
      std::shuffle(idx.begin(), idx.end(), rng);
      for (int j = 0; j < k; ++j) r[idx[(size_t)j]] = 1.0;
    } else {
      const double u = coin(rng) ? 1.0 : 0.0;
      std::fill(r, r + n, u);
    }
    for (int32_t j = 0; j < n; ++j) (void)(straggler(rng) ? tail_ms(rng) : base_ms(rng));
  }
  return PRORL_OK;
}
