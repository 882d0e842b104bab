// rollout/trajectory.hpp — STANDALONE re-declaration of the reference type of
// the same name (proj/include/rollout/trajectory.hpp:11-103), for builds of
// this repo without the reference tree. Same members, no extras: the façade
// (include/rollout/trainer/scoring.hpp) compiles against either header. A
// reference build never sees this directory (include/standalone/).
//
// Semantics preserved exactly, because the device packer (prorl_pack) is
// defined in terms of them:
//   * Role order SYSTEM, USER, ASSISTANT, TOOL (reference :11) — the C-ABI's
//     PRORL_ROLE_* values;
//   * assistant turns carry output_ids + aligned logprobs, every other role
//     carries input_ids only; anything else is MalformedTurn (:89-99);
//   * flatten order = each turn's token field in turn order (:76-87), which is
//     the packed token stream of one sequence; assistant tokens are the policy
//     tokens (loss_mask = 1).
#pragma once

#include <algorithm>
#include <cstddef>
#include <string>
#include <vector>

#include "rollout/errors.hpp"
#include "rollout/types.hpp"

namespace rollout {

enum class Role { SYSTEM, USER, ASSISTANT, TOOL };

inline const char* role_name(Role r) {
  static const char* const kNames[] = {"system", "user", "assistant", "tool"};
  const auto i = static_cast<unsigned>(r);
  return i < 4 ? kNames[i] : "?";
}

struct Turn {
  Role role = Role::USER;
  TokenIds input_ids;          // non-assistant turns
  TokenIds output_ids;         // assistant turns
  std::vector<double> logprobs;  // aligned with output_ids (behaviour policy)
  std::string text;            // display only, never re-tokenized
};

inline Turn make_user_turn(TokenIds ids, std::string text = {}) {
  Turn t;
  t.input_ids = std::move(ids);
  t.text = std::move(text);
  return t;
}

inline Turn make_tool_turn(TokenIds ids, std::string text = {}) {
  Turn t = make_user_turn(std::move(ids), std::move(text));
  t.role = Role::TOOL;
  return t;
}

inline Turn make_assistant_turn(TokenIds output_ids, std::vector<double> logprobs, std::string text = {}) {
  Turn t;
  t.role = Role::ASSISTANT;
  t.output_ids = std::move(output_ids);
  t.logprobs = std::move(logprobs);
  t.text = std::move(text);
  return t;
}

class TokenTrajectory {
 public:
  void append(Turn turn) {
    validate(turn);
    turns_.emplace_back(std::move(turn));
  }

  const std::vector<Turn>& turns() const { return turns_; }
  std::size_t size() const { return turns_.size(); }
  bool empty() const { return turns_.empty(); }

  TokenIds flatten() const { return flatten_range(0, turns_.size()); }

  // Turns [begin, end), end clamped to size().
  TokenIds flatten_range(std::size_t begin, std::size_t end) const {
    TokenIds out;
    const std::size_t stop = std::min(end, turns_.size());
    for (std::size_t i = begin; i < stop; ++i) {
      const Turn& t = turns_[i];
      const TokenIds& ids = t.role == Role::ASSISTANT ? t.output_ids : t.input_ids;
      out.insert(out.end(), ids.begin(), ids.end());
    }
    return out;
  }

  static void validate(const Turn& t) {
    if (t.role != Role::ASSISTANT) {
      if (!t.output_ids.empty() || !t.logprobs.empty())
        throw MalformedTurn("non-assistant turn must not carry output_ids/logprobs");
      return;
    }
    if (!t.input_ids.empty()) throw MalformedTurn("assistant turn must not carry input_ids");
    if (t.output_ids.size() != t.logprobs.size())
      throw MalformedTurn("assistant turn logprobs not aligned with output_ids");
  }

 private:
  std::vector<Turn> turns_;
};

}  // namespace rollout
