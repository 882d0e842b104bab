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
// keys are skipped structurally, tokens are written straight into the
// thread's output (non-participating rollouts are dropped in place once their
// group's rewards are known), and groups are split over host threads by wire
// bytes.
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
#include <memory>
#include <new>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include <sys/mman.h>

#include "prorl_hotpath.h"

namespace {

struct ParseError {
  int status;
  std::string msg;
};

[[noreturn]] __attribute__((noinline, cold)) void throw_parse(int status, const char* what) {
  throw ParseError{status, what};
}

// Uninitialised token buffer sized from the wire bytes. Large buffers are
// anonymous mappings with transparent huge pages requested: first-touch
// page faults, not parsing, otherwise dominate a fresh multi-MB batch.
template <typename T>
class TokBuf {
 public:
  TokBuf() = default;
  explicit TokBuf(size_t n) { reset(n); }
  TokBuf(TokBuf&& o) noexcept : p_(o.p_), bytes_(o.bytes_), mapped_(o.mapped_) { o.p_ = nullptr, o.bytes_ = 0; }
  TokBuf& operator=(TokBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_, bytes_ = o.bytes_, mapped_ = o.mapped_;
      o.p_ = nullptr, o.bytes_ = 0;
    }
    return *this;
  }
  TokBuf(const TokBuf&) = delete;
  TokBuf& operator=(const TokBuf&) = delete;
  ~TokBuf() { release(); }
  void reset(size_t n) {
    release();
    constexpr size_t kHuge = size_t(2) << 20;
    bytes_ = std::max<size_t>(n, 1) * sizeof(T);
    mapped_ = bytes_ >= kHuge;
    if (mapped_) {
      bytes_ = (bytes_ + kHuge - 1) / kHuge * kHuge;
      void* m = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
      if (m == MAP_FAILED) throw std::bad_alloc();
#ifdef MADV_HUGEPAGE
      madvise(m, bytes_, MADV_HUGEPAGE);
#endif
      p_ = static_cast<T*>(m);
    } else {
      p_ = static_cast<T*>(std::malloc(bytes_));
      if (!p_) throw std::bad_alloc();
    }
  }
  void reserve(size_t n) {
    if (!p_ || n * sizeof(T) > bytes_) reset(n);
  }
  T* get() const { return p_; }

 private:
  void release() {
    if (!p_) return;
    if (mapped_) munmap(p_, bytes_);
    else std::free(p_);
    p_ = nullptr;
  }
  T* p_ = nullptr;
  size_t bytes_ = 0;
  bool mapped_ = false;
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
  // escapes are stepped over correctly (a quote preceded by an odd run of
  // backslashes is escaped).
  std::string_view str() {
    expect('"');
    const char* b = p_;
    const char* q = p_;
    for (;;) {
      q = static_cast<const char*>(std::memchr(q, '"', (size_t)(e_ - q)));
      if (!q) fail("unterminated string");
      const char* r = q;
      while (r > b && r[-1] == '\\') --r;
      if (((q - r) & 1) == 0) break;
      ++q;
    }
    p_ = q + 1;
    return std::string_view(b, (size_t)(q - b));
  }
  // libstdc++'s from_chars (Eisel-Lemire) is exact and, measured here, as
  // fast as a hand-rolled pre-scan for both short and 17-digit logprobs.
  __attribute__((always_inline)) double number() {
    ws();
    if (p_ >= e_ || (*p_ != '-' && (unsigned)(*p_ - '0') > 9u)) fail("bad number");  // no inf/nan/+ (JSON)
    double v = 0.0;
    auto r = std::from_chars(p_, e_, v);
    if (r.ec != std::errc()) fail("bad number");
    p_ = r.ptr;
    return v;
  }
  // [int, int, ...] of token ids written to w (capacity guaranteed by the
  // caller: a response of n bytes holds at most n/2 numbers).
  __attribute__((always_inline)) int64_t* int_array(int64_t* w) {
    expect('[');
    if (peek(']')) {
      ++p_;
      return w;
    }
    const char* q = p_;
    for (;;) {
      if (q < e_ && (*q == ' ' || *q == '\n' || *q == '\r' || *q == '\t')) {
        p_ = q;
        ws();
        q = p_;
      }
      const bool neg = q < e_ && *q == '-';
      q += neg;
      uint64_t v = 0;
      const char* d0 = q;
      while (q < e_ && (unsigned)(*q - '0') <= 9u) v = v * 10 + (uint64_t)(*q++ - '0');
      const ptrdiff_t nd = q - d0;
      if (nd == 0 || nd > 18) {
        p_ = q;
        fail(nd == 0 ? "bad integer" : "token id out of range");
      }
      if (q < e_ && (*q == '.' || *q == 'e' || *q == 'E')) {
        p_ = q;
        fail("non-integer token id");
      }
      *w++ = neg ? -(int64_t)v : (int64_t)v;
      if (q < e_ && *q == ',') {
        ++q;
        if (q < e_ && *q == ' ') ++q;
        continue;
      }
      p_ = q;
      ws();
      if (p_ < e_ && *p_ == ',') {
        q = p_ + 1;
        continue;
      }
      expect(']');
      return w;
    }
  }
  __attribute__((always_inline)) double* num_array(double* w) {
    expect('[');
    if (peek(']')) {
      ++p_;
      return w;
    }
    for (;;) {
      *w++ = number();
      if (p_ < e_ && *p_ == ',') {
        ++p_;
        continue;
      }
      ws();
      if (p_ < e_ && *p_ == ',') {
        ++p_;
        continue;
      }
      expect(']');
      return w;
    }
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

// One thread's output for a contiguous range of groups (part-local offsets).
// Token arrays are raw (uninitialised) buffers sized from the wire bytes: a
// response of n bytes carries at most n/2 numbers, so the parser writes
// through plain pointers with no per-token capacity check.
struct Part {
  std::vector<prorl_turn_desc> turns;
  TokBuf<int64_t> ids;
  TokBuf<double> lp;
  size_t n_tok = 0;
  std::vector<double> reward;
  std::vector<uint8_t> usable;
  int64_t n_active = 0;
  int32_t n_informative = 0;
  int status = PRORL_OK;
  std::string error;
};

// Parses one response straight into the part: its turns (traj = slot) and
// tokens are appended; returns FAILED-ness and the reward.
void parse_response(const char* js, size_t n, int32_t slot, Part& out, bool& failed, double& reward) {
  Scanner s(js, n);
  failed = true;  // a response without "status" counts as FAILED (harness.cpp:263)
  reward = 0.0;
  bool have_traj = false, cancelled = false;
  int64_t* const ids = out.ids.get();
  double* const lps = out.lp.get();
  s.object([&](std::string_view key) {
    if (key == "status") {
      const std::string_view st = s.str();
      failed = st == "FAILED";
      cancelled = st == "CANCELLED";
    } else if (key == "reward") {
      reward = s.number();
    } else if (key == "trajectory") {
      have_traj = true;
      s.array([&] {
        int role = -1;
        int64_t* wid = ids + out.n_tok;
        double* const lp0 = lps + out.n_tok;
        double* wlp = lp0;
        size_t n_in = 0, n_out = 0;
        s.object([&](std::string_view k) {
          if (k == "role") {
            role = role_code(s.str());
          } else if (k == "input_ids") {
            int64_t* e = s.int_array(wid);
            n_in += (size_t)(e - wid);
            wid = e;
          } else if (k == "output_ids") {
            int64_t* e = s.int_array(wid);
            n_out += (size_t)(e - wid);
            wid = e;
          } else if (k == "logprobs") {
            wlp = s.num_array(wlp);
          } else {
            s.skip();
          }
        });
        const size_t n_lp = (size_t)(wlp - lp0);
        if (role < 0) throw_parse(PRORL_E_MALFORMED_TURN, "turn without a role");
        // TokenTrajectory::validate (trajectory.hpp:89-99)
        if (role == PRORL_ROLE_ASSISTANT) {
          if (n_in) throw_parse(PRORL_E_MALFORMED_TURN, "assistant turn must not carry input_ids");
          if (n_lp != n_out) throw_parse(PRORL_E_MALFORMED_TURN, "assistant turn logprobs not aligned with output_ids");
        } else {
          if (n_out || n_lp) throw_parse(PRORL_E_MALFORMED_TURN, "non-assistant turn must not carry output_ids/logprobs");
          std::fill(lp0, lp0 + n_in, 0.0);
        }
        prorl_turn_desc d{};
        d.src_off = (int64_t)out.n_tok;
        d.traj = slot;
        d.len = (int32_t)(n_in + n_out);
        d.role = (uint8_t)role;
        out.turns.push_back(d);
        out.n_tok += n_in + n_out;
      });
    } else {
      s.skip();
    }
  });
  s.end();
  // The reference harness never records a CANCELLED response (harness.cpp:264:
  // the slot is re-issued), so a group holding one is not complete.
  if (cancelled)
    throw_parse(PRORL_E_INCOMPLETE_GROUP, "CANCELLED rollout: its slot is re-issued, the group is incomplete");
  if (!have_traj && !failed) throw_parse(PRORL_E_MALFORMED_REQUEST, "response without a trajectory");
}

void parse_groups(const char* const* json, const size_t* len, const int32_t* group_off, int32_t g0, int32_t g1,
                  double tol, Part& out) {
  size_t cap = 16;
  for (int32_t i = group_off[g0]; i < group_off[g1]; ++i) cap += len[i] / 2 + 1;
  out.ids.reserve(cap);
  out.lp.reserve(cap);
  out.reward.reserve((size_t)(group_off[g1] - group_off[g0]));
  out.usable.reserve((size_t)(group_off[g1] - group_off[g0]));
  struct Member {
    size_t turn0, tok0;
    bool failed;
  };
  std::vector<Member> mem;
  for (int32_t g = g0; g < g1; ++g) {
    const int32_t b = group_off[g], e = group_off[g + 1];
    const size_t turn_g = out.turns.size(), tok_g = out.n_tok;
    mem.clear();
    double mn = 0, mx = 0;
    int n_usable = 0, n_failed = 0;
    for (int32_t i = b; i < e; ++i) {
      Member m{out.turns.size(), out.n_tok, false};
      double reward = 0.0;
      try {
        parse_response(json[i], len[i], i, out, m.failed, reward);
      } catch (const ParseError& pe) {
        out.status = pe.status;
        out.error = "response " + std::to_string(i) + ": " + pe.msg;
        return;
      }
      mem.push_back(m);
      out.reward.push_back(reward);
      out.usable.push_back(m.failed ? 0 : 1);
      // usable_rewards (harness.cpp:84-90)
      if (m.failed) {
        ++n_failed;
        continue;
      }
      mn = n_usable ? std::min(mn, reward) : reward;
      mx = n_usable ? std::max(mx, reward) : reward;
      ++n_usable;
    }
    // is_informative (harness.cpp:92-102); non-participants are dropped in place
    const bool informative = n_usable >= 2 && (mx - mn) > tol;
    out.n_informative += informative ? 1 : 0;
    if (!informative) {
      out.turns.resize(turn_g);
      out.n_tok = tok_g;
      continue;
    }
    if (n_failed) {
      size_t wt = turn_g, wk = tok_g;
      for (size_t j = 0; j < mem.size(); ++j) {
        const size_t t1 = j + 1 < mem.size() ? mem[j + 1].turn0 : out.turns.size();
        const size_t k1 = j + 1 < mem.size() ? mem[j + 1].tok0 : out.n_tok;
        if (mem[j].failed) continue;
        const int64_t shift = (int64_t)(mem[j].tok0 - wk);
        for (size_t t = mem[j].turn0; t < t1; ++t, ++wt) {
          prorl_turn_desc d = out.turns[t];
          d.src_off -= shift;
          out.turns[wt] = d;
        }
        std::memmove(out.ids.get() + wk, out.ids.get() + mem[j].tok0, (k1 - mem[j].tok0) * sizeof(int64_t));
        std::memmove(out.lp.get() + wk, out.lp.get() + mem[j].tok0, (k1 - mem[j].tok0) * sizeof(double));
        wk += k1 - mem[j].tok0;
      }
      out.turns.resize(wt);
      out.n_tok = wk;
    }
    // active rows: an assistant turn's tokens are targets except at position 0
    int32_t cur = -1;
    int64_t pos = 0;
    for (size_t t = turn_g; t < out.turns.size(); ++t) {
      const prorl_turn_desc& d = out.turns[t];
      if (d.traj != cur) cur = d.traj, pos = 0;
      if (d.role == PRORL_ROLE_ASSISTANT && d.len > 0) out.n_active += d.len - (pos == 0 ? 1 : 0);
      pos += d.len;
    }
  }
}

struct IngestImpl {
  std::vector<prorl_turn_desc> turns;
  TokBuf<int64_t> ids;
  TokBuf<double> lp;
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
  for (int32_t i = 0; n_groups > 0 && i < group_off[n_groups]; ++i)
    if (!json[i] && len[i]) return prorl::fail(PRORL_E_MALFORMED_REQUEST, "prorl_ingest_responses: null response");
  static const int32_t kNoGroups[1] = {0};
  if (n_groups == 0) group_off = kNoGroups;
  auto impl = std::make_unique<IngestImpl>();
  const int32_t T = std::max(1, std::min<int32_t>(n_threads < 1 ? (int32_t)std::thread::hardware_concurrency() : n_threads,
                                                  std::max(n_groups, 1)));
  // split the groups into T ranges of about equal wire bytes
  std::vector<int32_t> gsplit((size_t)T + 1, n_groups);
  {
    size_t total = 0;
    for (int32_t i = 0; n_groups > 0 && i < group_off[n_groups]; ++i) total += len[i];
    gsplit[0] = 0;
    size_t acc = 0;
    int32_t t = 1;
    for (int32_t g = 0; g < n_groups && t < T; ++g) {
      for (int32_t i = group_off[g]; i < group_off[g + 1]; ++i) acc += len[i];
      while (t < T && acc * (size_t)T >= total * (size_t)t) gsplit[(size_t)t++] = g + 1;
    }
  }
  std::vector<Part> parts((size_t)T);
  if (T == 1) {
    parse_groups(json, len, group_off, 0, n_groups, gate_tolerance, parts[0]);
  } else {
    std::vector<std::thread> th;
    for (int32_t t = 0; t < T; ++t)
      th.emplace_back(parse_groups, json, len, group_off, gsplit[(size_t)t], gsplit[(size_t)t + 1], gate_tolerance,
                      std::ref(parts[(size_t)t]));
    for (auto& x : th) x.join();
  }
  for (const Part& p : parts)
    if (p.status != PRORL_OK) return prorl::fail(p.status, p.error);
  // offsets of each part in the merged arrays, then copy the parts in parallel
  std::vector<size_t> ot(parts.size() + 1, 0), oi(parts.size() + 1, 0), orr(parts.size() + 1, 0);
  for (size_t t = 0; t < parts.size(); ++t) {
    ot[t + 1] = ot[t] + parts[t].turns.size();
    oi[t + 1] = oi[t] + parts[t].n_tok;
    orr[t + 1] = orr[t] + parts[t].reward.size();
    out->n_active += parts[t].n_active;
    out->n_informative += parts[t].n_informative;
  }
  impl->turns.resize(ot.back());
  impl->reward.resize(orr.back());
  impl->usable.resize(orr.back());
  if (parts.size() == 1) {  // single part: adopt its buffers
    impl->ids = std::move(parts[0].ids);
    impl->lp = std::move(parts[0].lp);
    impl->turns = std::move(parts[0].turns);
    impl->reward = std::move(parts[0].reward);
    impl->usable = std::move(parts[0].usable);
  } else {
    impl->ids.reset(oi.back() + 1);
    impl->lp.reset(oi.back() + 1);
    std::vector<std::thread> th;
    for (size_t t = 0; t < parts.size(); ++t) {
      th.emplace_back([&, t] {
        const Part& p = parts[t];
        for (size_t k = 0; k < p.turns.size(); ++k) {
          prorl_turn_desc d = p.turns[k];
          d.src_off += (int64_t)oi[t];
          impl->turns[ot[t] + k] = d;
        }
        std::memcpy(impl->ids.get() + oi[t], p.ids.get(), p.n_tok * sizeof(int64_t));
        std::memcpy(impl->lp.get() + oi[t], p.lp.get(), p.n_tok * sizeof(double));
        std::copy(p.reward.begin(), p.reward.end(), impl->reward.begin() + (ptrdiff_t)orr[t]);
        std::copy(p.usable.begin(), p.usable.end(), impl->usable.begin() + (ptrdiff_t)orr[t]);
      });
    }
    for (auto& x : th) x.join();
  }
  impl->group_off.assign(group_off, group_off + n_groups + 1);
  prorl_host_batch& b = out->batch;
  b.turns = impl->turns.data();
  b.n_turns = (int64_t)impl->turns.size();
  b.ids = impl->ids.get();
  b.lp = impl->lp.get();
  b.n_tokens = (int64_t)oi.back();
  b.reward = impl->reward.data();
  b.usable = impl->usable.data();
  b.n_rollouts = (int32_t)impl->reward.size();
  b.group_off = impl->group_off.data();
  b.n_groups = n_groups;
  b.rollout_key = nullptr;
  out->impl = impl.release();
  return PRORL_OK;
}

extern "C" int prorl_ingest_free(prorl_ingest_result* r) {
  if (r && r->impl) {
    delete static_cast<IngestImpl*>(r->impl);
    std::memset(r, 0, sizeof(*r));
  }
  return PRORL_OK;
}
