// ingest.cpp — /process responses (JSON) -> a shard's host SoA, the trainer
// input of the device path (SURVEY.md §8 f rank 3).
//
// The wire schema is the reference's build_process_response
// (proj/src/handlers.cpp:57-91): {"job_id", "status", "reward",
// "trajectory": [{"role", "input_ids", "output_ids", "logprobs", "text"}...],
// "timings", "backend"?, "error"?}. Today the reference harness parses the
// response with nlohmann::json and keeps only status/reward/backend
// (proj/src/trainer/harness.cpp:254-273). Parsing ~10-20 bytes of decimal text
// per token through a DOM would dominate the step once the kernels run at HBM
// speed, so this is a single-pass, schema-directed scanner: integers are
// parsed by hand, doubles with std::from_chars (exact round-trip), unknown
// keys are skipped structurally, and groups are split over host threads.
//
// Semantics match the C++ façade's build_host_batch (scoring.cpp): turns are
// validated like TokenTrajectory::validate (trajectory.hpp:89-99 — MalformedTurn),
// FAILED rollouts are not usable (harness.cpp:84-90), rollouts of groups that
// fail is_informative (harness.cpp:92-102) contribute empty sequences, and
// every rollout slot keeps its reward / usable flag for the GRPO kernel.
#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "prorl_hotpath.h"

namespace {

struct ParseError {
  int status;
  std::string msg;
};

class Scanner {
 public:
  Scanner(const char* p, size_t n) : p_(p), e_(p + n) {}

  __attribute__((always_inline)) void ws() {
    while (p_ < e_ && (*p_ == ' ' || *p_ == '\n' || *p_ == '\r' || *p_ == '\t')) ++p_;
  }
  __attribute__((always_inline)) bool peek(char c) {
    ws();
    return p_ < e_ && *p_ == c;
  }
  __attribute__((always_inline)) void expect(char c) {
    ws();
    if (p_ >= e_ || *p_ != c) fail_expect(c);
    ++p_;
  }
  // String without unescaping (keys / enum values never contain escapes);
  // escapes are stepped over correctly.
  std::string_view str() {
    expect('"');
    const char* b = p_;
    while (p_ < e_ && *p_ != '"') {
      if (*p_ == '\\') ++p_;
      ++p_;
    }
    if (p_ >= e_) fail("unterminated string");
    std::string_view s(b, (size_t)(p_ - b));
    ++p_;
    return s;
  }
  __attribute__((always_inline)) double number() {
    ws();
    // Fast path (exact): [-]digits[.digits] with <= 15 significant digits and
    // no exponent is mantissa / 10^k with both operands exact doubles, so the
    // single IEEE division is the correctly rounded value from_chars returns.
    {
      const char* q = p_;
      bool neg = false;
      if (q < e_ && *q == '-') {
        neg = true;
        ++q;
      }
      uint64_t m = 0;
      int digits = 0, frac = 0;
      const char* d0 = q;
      while (q < e_ && *q >= '0' && *q <= '9' && digits < 16) m = m * 10 + (uint64_t)(*q++ - '0'), ++digits;
      if (q > d0 && q < e_ && *q == '.') {
        ++q;
        while (q < e_ && *q >= '0' && *q <= '9' && digits < 16) m = m * 10 + (uint64_t)(*q++ - '0'), ++digits, ++frac;
      }
      if (q > d0 && digits <= 15 && (q >= e_ || (*q != 'e' && *q != 'E' && (*q < '0' || *q > '9')))) {
        static constexpr double kPow10[] = {1e0, 1e1, 1e2,  1e3,  1e4,  1e5,  1e6,  1e7,
                                            1e8, 1e9, 1e10, 1e11, 1e12, 1e13, 1e14, 1e15};
        const double v = (double)m / kPow10[frac];
        p_ = q;
        return neg ? -v : v;
      }
    }
    double v = 0.0;
    auto r = std::from_chars(p_, e_, v);
    if (r.ec != std::errc()) fail("bad number");
    p_ = r.ptr;
    return v;
  }
  __attribute__((always_inline)) int64_t integer() {
    ws();
    bool neg = false;
    if (p_ < e_ && *p_ == '-') {
      neg = true;
      ++p_;
    }
    if (p_ >= e_ || *p_ < '0' || *p_ > '9') fail("bad integer");
    uint64_t v = 0;
    while (p_ < e_ && *p_ >= '0' && *p_ <= '9') v = v * 10 + (uint64_t)(*p_++ - '0');
    if (p_ < e_ && (*p_ == '.' || *p_ == 'e' || *p_ == 'E')) fail("non-integer token id");
    return neg ? -(int64_t)v : (int64_t)v;
  }
  template <typename F>
  void array(F&& item) {
    expect('[');
    if (peek(']')) {
      ++p_;
      return;
    }
    for (;;) {
      item();
      ws();
      if (p_ < e_ && *p_ == ',') {
        ++p_;
        continue;
      }
      expect(']');
      return;
    }
  }
  template <typename F>
  void object(F&& member) {
    expect('{');
    if (peek('}')) {
      ++p_;
      return;
    }
    for (;;) {
      const std::string_view k = str();
      expect(':');
      member(k);
      ws();
      if (p_ < e_ && *p_ == ',') {
        ++p_;
        continue;
      }
      expect('}');
      return;
    }
  }
  void skip(int depth = 0) {
    ws();
    if (p_ >= e_) fail("unexpected end");
    if (depth > 64) fail("nesting too deep");
    const char c = *p_;
    if (c == '"') {
      str();
    } else if (c == '{') {
      object([&](std::string_view) { skip(depth + 1); });
    } else if (c == '[') {
      array([&] { skip(depth + 1); });
    } else if (c == 't' || c == 'f' || c == 'n') {
      const char* lit = c == 't' ? "true" : (c == 'f' ? "false" : "null");
      const size_t n = std::strlen(lit);
      if ((size_t)(e_ - p_) < n || std::memcmp(p_, lit, n) != 0) fail("bad literal");
      p_ += n;
    } else {
      number();
    }
  }
  void end() {
    ws();
    if (p_ != e_) fail("trailing characters");
  }
  [[noreturn]] __attribute__((noinline, cold)) void fail(const char* what) {
    throw ParseError{PRORL_E_MALFORMED_REQUEST, what};
  }
  [[noreturn]] __attribute__((noinline, cold)) void fail_expect(char c) {
    throw ParseError{PRORL_E_MALFORMED_REQUEST, std::string("expected '") + c + "'"};
  }

 private:
  const char* p_;
  const char* e_;
};

int role_code(std::string_view r) {
  if (r == "system") return PRORL_ROLE_SYSTEM;
  if (r == "user") return PRORL_ROLE_USER;
  if (r == "assistant") return PRORL_ROLE_ASSISTANT;
  if (r == "tool") return PRORL_ROLE_TOOL;
  throw ParseError{PRORL_E_MALFORMED_TURN, "unknown role '" + std::string(r) + "'"};
}

// One thread's output for a contiguous range of groups (local offsets).
struct Part {
  std::vector<prorl_turn_desc> turns;
  std::vector<int64_t> ids;
  std::vector<double> lp;
  std::vector<double> reward;
  std::vector<uint8_t> usable;
  int64_t n_active = 0;
  int32_t n_informative = 0;
  int status = PRORL_OK;
  std::string error;
};

struct Rollout {  // one parsed response
  bool failed = false;
  double reward = 0.0;
  std::vector<prorl_turn_desc> turns;  // src_off local to ids/lp below, traj unset
  std::vector<int64_t> ids;
  std::vector<double> lp;
};

void parse_response(const char* js, size_t n, Rollout& r) {
  Scanner s(js, n);
  r.failed = false;
  r.reward = 0.0;
  r.turns.clear();
  r.ids.clear();
  r.lp.clear();
  r.ids.reserve(n / 5);
  r.lp.reserve(n / 5);
  bool have_traj = false;
  s.object([&](std::string_view key) {
    if (key == "status") {
      r.failed = s.str() == "FAILED";
    } else if (key == "reward") {
      r.reward = s.number();
    } else if (key == "trajectory") {
      have_traj = true;
      s.array([&] {
        int role = -1;
        const size_t id0 = r.ids.size(), lp0 = r.lp.size();
        size_t n_in = 0, n_out = 0;
        s.object([&](std::string_view k) {
          if (k == "role") {
            role = role_code(s.str());
          } else if (k == "input_ids") {
            s.array([&] {
              r.ids.push_back(s.integer());
              ++n_in;
            });
          } else if (k == "output_ids") {
            s.array([&] {
              r.ids.push_back(s.integer());
              ++n_out;
            });
          } else if (k == "logprobs") {
            s.array([&] { r.lp.push_back(s.number()); });
          } else {
            s.skip();
          }
        });
        const size_t n_lp = r.lp.size() - lp0;
        if (role < 0) throw ParseError{PRORL_E_MALFORMED_TURN, "turn without a role"};
        // TokenTrajectory::validate (trajectory.hpp:89-99)
        if (role == PRORL_ROLE_ASSISTANT) {
          if (n_in) throw ParseError{PRORL_E_MALFORMED_TURN, "assistant turn must not carry input_ids"};
          if (n_lp != n_out) throw ParseError{PRORL_E_MALFORMED_TURN, "assistant turn logprobs not aligned with output_ids"};
        } else {
          if (n_out || n_lp) throw ParseError{PRORL_E_MALFORMED_TURN, "non-assistant turn must not carry output_ids/logprobs"};
          r.lp.resize(lp0 + n_in, 0.0);
        }
        prorl_turn_desc d{};
        d.src_off = (int64_t)id0;
        d.len = (int32_t)(r.ids.size() - id0);
        d.role = (uint8_t)role;
        r.turns.push_back(d);
      });
    } else {
      s.skip();
    }
  });
  s.end();
  if (!have_traj) throw ParseError{PRORL_E_MALFORMED_REQUEST, "response without a trajectory"};
}

void parse_groups(const char* const* json, const size_t* len, const int32_t* group_off, int32_t g0, int32_t g1,
                  double tol, Part& out) {
  std::vector<Rollout> grp;
  size_t bytes = 0;  // capacity estimate: a token takes >= ~5 bytes of wire JSON on average
  for (int32_t i = group_off[g0]; i < group_off[g1]; ++i) bytes += len[i];
  out.ids.reserve(bytes / 5);
  out.lp.reserve(bytes / 5);
  for (int32_t g = g0; g < g1; ++g) {
    const int32_t b = group_off[g], e = group_off[g + 1];
    grp.resize((size_t)(e - b));
    for (int32_t i = b; i < e; ++i) {
      try {
        parse_response(json[i], len[i], grp[(size_t)(i - b)]);
      } catch (const ParseError& pe) {
        out.status = pe.status;
        out.error = "response " + std::to_string(i) + ": " + pe.msg;
        return;
      }
    }
    // usable_rewards + is_informative (harness.cpp:84-102)
    double mn = 0, mx = 0;
    int n_usable = 0;
    for (const Rollout& r : grp) {
      if (r.failed) continue;
      mn = n_usable ? std::min(mn, r.reward) : r.reward;
      mx = n_usable ? std::max(mx, r.reward) : r.reward;
      ++n_usable;
    }
    const bool informative = n_usable >= 2 && (mx - mn) > tol;
    out.n_informative += informative ? 1 : 0;
    for (int32_t i = b; i < e; ++i) {
      Rollout& r = grp[(size_t)(i - b)];
      out.reward.push_back(r.reward);
      out.usable.push_back(r.failed ? 0 : 1);
      if (!informative || r.failed) continue;
      const int64_t base = (int64_t)out.ids.size();
      int64_t pos = 0;
      for (prorl_turn_desc d : r.turns) {
        d.src_off += base;
        d.traj = i;  // rollout slot index in the shard
        if (d.role == PRORL_ROLE_ASSISTANT && d.len > 0) out.n_active += d.len - (pos == 0 ? 1 : 0);
        pos += d.len;
        out.turns.push_back(d);
      }
      out.ids.insert(out.ids.end(), r.ids.begin(), r.ids.end());
      out.lp.insert(out.lp.end(), r.lp.begin(), r.lp.end());
    }
  }
}

struct IngestImpl {
  std::vector<prorl_turn_desc> turns;
  std::vector<int64_t> ids;
  std::vector<double> lp;
  std::vector<double> reward;
  std::vector<uint8_t> usable;
  std::vector<int32_t> group_off;
};

}  // namespace

namespace prorl {
int fail(int status, const std::string& msg);
}

extern "C" int prorl_ingest_responses(const char* const* json, const size_t* len, const int32_t* group_off,
                                      int32_t n_groups, double gate_tolerance, int32_t n_threads,
                                      prorl_ingest_result* out) {
  if (!out || n_groups < 0 || (n_groups > 0 && (!json || !len || !group_off)))
    return prorl::fail(PRORL_E_MALFORMED_REQUEST, "prorl_ingest_responses: bad arguments");
  std::memset(out, 0, sizeof(*out));
  if (n_groups > 0 && group_off[0] != 0)
    return prorl::fail(PRORL_E_MALFORMED_REQUEST, "prorl_ingest_responses: group_off[0] must be 0");
  for (int32_t g = 0; g < n_groups; ++g)
    if (group_off[g + 1] < group_off[g])
      return prorl::fail(PRORL_E_MALFORMED_REQUEST, "prorl_ingest_responses: group_off not monotone");
  auto* impl = new IngestImpl();
  const int32_t T = std::max(1, std::min<int32_t>(n_threads < 1 ? (int32_t)std::thread::hardware_concurrency() : n_threads,
                                                  std::max(n_groups, 1)));
  std::vector<Part> parts((size_t)T);
  std::vector<std::thread> th;
  for (int32_t t = 0; t < T; ++t) {
    const int32_t g0 = (int32_t)((int64_t)n_groups * t / T), g1 = (int32_t)((int64_t)n_groups * (t + 1) / T);
    th.emplace_back(parse_groups, json, len, group_off, g0, g1, gate_tolerance, std::ref(parts[(size_t)t]));
  }
  for (auto& x : th) x.join();
  for (const Part& p : parts)
    if (p.status != PRORL_OK) {
      delete impl;
      return prorl::fail(p.status, p.error);
    }
  // offsets of each part in the merged arrays, then copy the parts in parallel
  std::vector<size_t> ot(parts.size() + 1, 0), oi(parts.size() + 1, 0), orr(parts.size() + 1, 0);
  for (size_t t = 0; t < parts.size(); ++t) {
    ot[t + 1] = ot[t] + parts[t].turns.size();
    oi[t + 1] = oi[t] + parts[t].ids.size();
    orr[t + 1] = orr[t] + parts[t].reward.size();
    out->n_active += parts[t].n_active;
    out->n_informative += parts[t].n_informative;
  }
  impl->turns.resize(ot.back());
  impl->ids.resize(oi.back());
  impl->lp.resize(oi.back());
  impl->reward.resize(orr.back());
  impl->usable.resize(orr.back());
  th.clear();
  for (size_t t = 0; t < parts.size(); ++t) {
    th.emplace_back([&, t] {
      const Part& p = parts[t];
      for (size_t k = 0; k < p.turns.size(); ++k) {
        prorl_turn_desc d = p.turns[k];
        d.src_off += (int64_t)oi[t];
        impl->turns[ot[t] + k] = d;
      }
      std::copy(p.ids.begin(), p.ids.end(), impl->ids.begin() + (ptrdiff_t)oi[t]);
      std::copy(p.lp.begin(), p.lp.end(), impl->lp.begin() + (ptrdiff_t)oi[t]);
      std::copy(p.reward.begin(), p.reward.end(), impl->reward.begin() + (ptrdiff_t)orr[t]);
      std::copy(p.usable.begin(), p.usable.end(), impl->usable.begin() + (ptrdiff_t)orr[t]);
    });
  }
  for (auto& x : th) x.join();
  impl->group_off.assign(group_off, group_off + n_groups + 1);
  prorl_host_batch& b = out->batch;
  b.turns = impl->turns.data();
  b.n_turns = (int64_t)impl->turns.size();
  b.ids = impl->ids.data();
  b.lp = impl->lp.data();
  b.n_tokens = (int64_t)impl->ids.size();
  b.reward = impl->reward.data();
  b.usable = impl->usable.data();
  b.n_rollouts = (int32_t)impl->reward.size();
  b.group_off = impl->group_off.data();
  b.n_groups = n_groups;
  b.rollout_key = nullptr;
  out->impl = impl;
  return PRORL_OK;
}

extern "C" int prorl_ingest_free(prorl_ingest_result* r) {
  if (r && r->impl) {
    delete static_cast<IngestImpl*>(r->impl);
    std::memset(r, 0, sizeof(*r));
  }
  return PRORL_OK;
}
