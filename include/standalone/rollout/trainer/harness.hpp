// rollout/trainer/harness.hpp — STANDALONE re-declaration of the trainer-side
// group types the scoring path consumes, for builds of this repo without the
// reference tree (a reference build never sees include/standalone/). Same
// members as the reference (proj/include/rollout/trainer/harness.hpp:35-84):
//   RolloutOutcome, PromptGroup{completed_count, complete, usable_rewards},
//   is_informative, IterationStats::informative (the hand-off point).
// RolloutOutcome is unchanged — the token trajectory travels beside it in the
// façade's TrajectoryTable (include/rollout/trainer/scoring.hpp). The
// reference defines the PromptGroup members and is_informative out of line in
// proj/src/trainer/harness.cpp:71-102; here they are inline. The scheduling
// half of the reference harness (TrainerHarness) is out of scope.
#pragma once

#include <algorithm>
#include <optional>
#include <string>
#include <vector>

#include <json.hpp>

#include "rollout/errors.hpp"

namespace rollout::train {

enum class GroupState { PENDING, IN_FLIGHT, COMPLETE, CARRIED_OVER };

struct RolloutOutcome {
  double reward = 0.0;
  std::string status;   // DONE / FAILED / CANCELLED
  std::string address;  // backend that served it, when reported
  double wall_seconds = 0.0;
};

struct PromptGroup {
  std::string prompt_id;
  nlohmann::json payload;
  int n = 0;
  std::vector<std::optional<RolloutOutcome>> outcomes;  // one slot per rollout
  GroupState state = GroupState::PENDING;

  int completed_count() const {
    return static_cast<int>(std::count_if(outcomes.begin(), outcomes.end(),
                                          [](const auto& o) { return o.has_value(); }));
  }
  bool complete() const { return n > 0 && completed_count() == n; }

  // Rewards of the non-FAILED rollouts, in slot order (reference harness.cpp:84-90).
  std::vector<double> usable_rewards() const {
    std::vector<double> r;
    r.reserve(outcomes.size());
    for (const auto& o : outcomes)
      if (o && o->status != "FAILED") r.push_back(o->reward);
    return r;
  }
};

// DAPO zero-variance gate (reference harness.cpp:92-102): false with fewer than
// two usable rewards or when max - min <= tolerance; IncompleteGroup unless
// every slot is filled.
inline bool is_informative(const PromptGroup& g, double tolerance = 0.0) {
  if (!g.complete())
    throw IncompleteGroup("group " + g.prompt_id + " has " + std::to_string(g.completed_count()) + "/" +
                          std::to_string(g.n) + " outcomes");
  const std::vector<double> r = g.usable_rewards();
  if (r.size() < 2) return false;
  const auto mm = std::minmax_element(r.begin(), r.end());
  return *mm.second - *mm.first > tolerance;
}

struct IterationStats {
  std::vector<PromptGroup> informative;   // hand-off to the trainer step
  std::vector<PromptGroup> carried_over;
  double wall_seconds = 0.0;
  int rollouts_issued = 0;
  int cancels_issued = 0;
  int waves = 0;
  double idle_fraction = 0.0;
};

}  // namespace rollout::train
