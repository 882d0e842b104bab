// rollout/types.hpp — STANDALONE re-declaration (never seen by a reference
// build) of the token and sampling types the scoring path consumes, with the
// reference's names and meaning (proj/include/rollout/types.hpp:12-13
// TokenId = int64 on the wire; :58-71 SamplingParams, whose temperature is the
// logit temperature of the logprob pass).
#pragma once

#include <cstdint>
#include <vector>

#include "rollout/errors.hpp"

namespace rollout {

using TokenId = std::int64_t;
using TokenIds = std::vector<TokenId>;

struct SamplingParams {
  double temperature = 1.0;
  double top_p = 1.0;
  int max_tokens = 64;
  TokenIds stop_token_ids;

  // Same acceptance rules as the reference (types.hpp:64-70).
  void validate() const {
    const bool top_p_ok = top_p > 0.0 && top_p <= 1.0;
    if (temperature < 0.0) throw MalformedRequest("temperature must be nonnegative");
    if (!top_p_ok) throw MalformedRequest("top_p must be in (0,1]");
    if (max_tokens < 1) throw MalformedRequest("max_tokens must be >= 1");
  }
};

}  // namespace rollout
