// pack.cu — K1: device-side trajectory packer.
//
// Semantics follow the reference's flatten order and
// role rule: a trajectory's token stream is its turns' token fields
// concatenated in turn order, assistant turns contributing output_ids and all
// others input_ids (proj/include/rollout/trajectory.hpp:76-87, rule at
// :82-83). Trajectories are concatenated in ascending `traj` (= rollout index
// in the shard = seq id). The loss mask marks assistant (policy) tokens; tool /
// user / system observation tokens are masked out (tool turns are appended at
// proj/src/handlers.cpp:292-293). Row r is *active* iff token r+1 is a policy
// token of the same sequence; its target is tokens[r+1].
//
// Work: two integer scans (turn lengths + assistant-turn counts, packed in one
// int64; active-row flags) and two scatter passes. Everything is integer or a
// single fp64->fp32 RN conversion, so the output is bit-exact vs the oracle.
#include "scan.cuh"

namespace prorl {

namespace {

constexpr int kLenBits = 40;
constexpr int64_t kLenMask = (int64_t(1) << kLenBits) - 1;

struct TurnVal {
  const prorl_turn_desc* turns;
  __device__ int64_t operator()(int64_t i) const {
    prorl_turn_desc t = turns[i];
    int64_t len = t.len < 0 ? 0 : (int64_t)t.len;
    return len | ((int64_t)(t.role == PRORL_ROLE_ASSISTANT) << kLenBits);
  }
};

struct FlagVal {
  const uint8_t* flags;
  __device__ int32_t operator()(int64_t i) const { return (int32_t)flags[i]; }
};

// One thread per turn boundary t in [0, n_turns]: fills cu_seqlens[s] and the
// assistant-turn count at sequence start for every s in (traj[t-1], traj[t]].
__global__ void k_seq_bounds(const prorl_turn_desc* turns, int64_t n_turns, const int64_t* off,
                             int32_t n_seq, int64_t n_tokens, int32_t* cu_seqlens, int64_t* asst0,
                             int* err) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > n_turns) return;
  int64_t a = (t == 0) ? -1 : (int64_t)turns[t - 1].traj;
  int64_t b = (t == n_turns) ? (int64_t)n_seq : (int64_t)turns[t].traj;
  if (t < n_turns) {
    prorl_turn_desc d = turns[t];
    if (d.traj < 0 || d.traj >= n_seq || d.len < 0 || d.role > PRORL_ROLE_TOOL) raise_flag(err, ERR_TURN_ORDER);
  } else if ((off[n_turns] & kLenMask) != n_tokens) {
    raise_flag(err, ERR_TOKEN_COUNT);
  }
  if (b < a) {
    raise_flag(err, ERR_TURN_ORDER);
    return;
  }
  if (a >= n_seq) return;
  const int64_t v = off[t];
  for (int64_t s = a + 1; s <= b && s <= n_seq; ++s) {
    cu_seqlens[s] = (int32_t)(v & kLenMask);
    if (s < n_seq) asst0[s] = v >> kLenBits;
  }
}

// One thread per token p in [p0, p1): locate its turn (binary search over turn
// offsets), convert id / logprob, emit mask, ids, and the active flag of row
// p-1 (flags[p1-1] stays 0 from the memset: p1 is a sequence start or the end).
__global__ void k_pack_tokens(const prorl_turn_desc* __restrict__ turns, int64_t n_turns,
                              const int64_t* __restrict__ off, const int64_t* __restrict__ asst0,
                              const int64_t* __restrict__ ids, const double* __restrict__ lp, int64_t p0,
                              int64_t p1, int32_t n_seq, int32_t vocab, prorl_packed out, uint8_t* flags,
                              int* err) {
  int64_t p = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= p1) return;
  // largest t in [0, n_turns) with off_len[t] <= p
  int64_t lo = 0, hi = n_turns - 1;
  while (lo < hi) {
    int64_t mid = (lo + hi + 1) >> 1;
    if ((off[mid] & kLenMask) <= p) lo = mid;
    else hi = mid - 1;
  }
  const prorl_turn_desc d = turns[lo];
  const int64_t v = off[lo];
  const int64_t k = p - (v & kLenMask);
  if (k >= d.len || d.traj < 0 || d.traj >= n_seq) {  // inconsistent descriptors (flagged)
    raise_flag(err, k >= d.len ? ERR_TOKEN_COUNT : ERR_TURN_ORDER);
    return;
  }
  const int64_t src = d.src_off + k;
  int64_t id = ids[src];
  if (id < 0 || id >= vocab) {
    raise_flag(err, ERR_TOKEN_RANGE);
    id = 0;
  }
  const bool asst = d.role == PRORL_ROLE_ASSISTANT;
  const int32_t s = d.traj;
  const int32_t pos = (int32_t)(p - out.cu_seqlens[s]);
  int16_t tid = -1;
  if (asst) {
    int64_t ord = (v >> kLenBits) - asst0[s];
    tid = (int16_t)(ord > 32767 ? 32767 : ord);
  }
  out.tokens[p] = (int32_t)id;
  out.loss_mask[p] = asst ? 1 : 0;
  out.turn_id[p] = tid;
  out.seq_id[p] = s;
  out.pos_id[p] = pos;
  out.old_lp[p] = asst ? __double2float_rn(lp[src]) : 0.0f;
  if (p > p0) flags[p - 1] = (asst && pos > 0) ? 1 : 0;
}

// Rows [p0, p1) with their chunk-local exclusive scan pos[0 .. p1-p0]; the
// chunk's active rows start at a0. The last chunk writes the total.
__global__ void k_compact(const uint8_t* __restrict__ flags, const int32_t* __restrict__ pos, int64_t p0,
                          int64_t p1, int64_t a0, bool last, prorl_packed out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, r = p0 + k;
  if (k == 0 && last) *out.n_active = a0 + (int64_t)pos[p1 - p0];
  if (r >= p1 || !flags[r]) return;
  const int32_t i = (int32_t)(a0 + pos[k]);
  out.act_row[i] = (int32_t)r;
  out.act_target[i] = out.tokens[r + 1];
  out.act_old_lp[i] = out.old_lp[r + 1];
  out.act_seq[i] = out.seq_id[r + 1];
  out.act_turn[i] = out.turn_id[r + 1];
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

namespace {
// K1 workspace: off[n_turns+1] i64 | asst0[n_seq+1] i64 | act_pos[N+1] i32 | flags[N] u8
struct PackWs {
  int64_t* off;
  int64_t* asst0;
  int32_t* pos;
  uint8_t* flags;
  size_t total;
  PackWs(uint8_t* base, int64_t n_turns, int32_t n_seq, int64_t n_tokens) {
    const size_t o_asst = sizeof(int64_t) * (size_t)(n_turns + 1);
    const size_t o_pos = o_asst + sizeof(int64_t) * (size_t)(n_seq + 1);
    const size_t o_flag = o_pos + sizeof(int32_t) * (size_t)(n_tokens + 1);
    total = o_flag + (size_t)n_tokens + 16;
    off = reinterpret_cast<int64_t*>(base);
    asst0 = reinterpret_cast<int64_t*>(base + o_asst);
    pos = reinterpret_cast<int32_t*>(base + o_pos);
    flags = base + o_flag;
  }
};
}  // namespace

int launch_pack_turns(prorl_ctx* ctx, const prorl_turn_desc* turns, int64_t n_turns, int64_t n_tokens, int32_t n_seq,
                      int32_t vocab, const prorl_packed* out, cudaStream_t st) {
  if (n_turns < 0 || n_tokens < 0 || n_seq < 0 || vocab <= 0)
    return fail(PRORL_E_SHAPE, "prorl_pack: negative size or vocab <= 0");
  if (n_tokens >= (int64_t(1) << 31) - 1)
    return fail(PRORL_E_SHAPE, "prorl_pack: more than 2^31-2 tokens per shard");
  if (n_tokens > 0 && n_turns == 0) return fail(PRORL_E_SHAPE, "prorl_pack: tokens without turns");
  PRORL_CUDA(ctx->pack_tmp.ensure(PackWs(nullptr, n_turns, n_seq, n_tokens).total));
  const size_t scan_elems = scan_tmp_elems(n_turns > n_tokens ? n_turns : n_tokens) + 1;
  PRORL_CUDA(ctx->scan_tmp.ensure(scan_elems * sizeof(int64_t)));
  const PackWs w(ctx->pack_tmp.as<uint8_t>(), n_turns, n_seq, n_tokens);
  PRORL_CUDA(exclusive_scan<int64_t>(TurnVal{turns}, n_turns, w.off, ctx->scan_tmp.as<int64_t>(), st));
  k_seq_bounds<<<blocks_for(n_turns + 1, 256), 256, 0, st>>>(turns, n_turns, w.off, n_seq, n_tokens,
                                                               out->cu_seqlens, w.asst0, ctx->d_err);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

int launch_pack_tokens(prorl_ctx* ctx, const prorl_turn_desc* turns, int64_t n_turns, const int64_t* ids,
                       const double* lp, int64_t n_tokens, int32_t n_seq, int32_t vocab, const prorl_packed* out,
                       int64_t p0, int64_t p1, int64_t a0, bool last, cudaStream_t st) {
  if (p0 < 0 || p1 < p0 || p1 > n_tokens) return fail(PRORL_E_SHAPE, "prorl_pack: token range outside [0, n_tokens]");
  if (p1 == p0 && !last) return PRORL_OK;
  const PackWs w(ctx->pack_tmp.as<uint8_t>(), n_turns, n_seq, n_tokens);
  const int64_t n = p1 - p0;
  if (n > 0) {
    PRORL_CUDA(cudaMemsetAsync(w.flags + p0, 0, (size_t)n, st));
    k_pack_tokens<<<blocks_for(n, 256), 256, 0, st>>>(turns, n_turns, w.off, w.asst0, ids, lp, p0, p1, n_seq, vocab,
                                                       *out, w.flags, ctx->d_err);
    PRORL_CUDA(cudaGetLastError());
  }
  PRORL_CUDA(exclusive_scan<int32_t>(FlagVal{w.flags + p0}, n, w.pos + p0, ctx->scan_tmp.as<int32_t>(), st));
  // (the last chunk also writes n_active, even when it holds no tokens)
  k_compact<<<n > 0 ? blocks_for(n, 256) : 1, 256, 0, st>>>(w.flags, w.pos + p0, p0, p1, a0, last, *out);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

int launch_pack(prorl_ctx* ctx, const prorl_turn_desc* turns, int64_t n_turns, const int64_t* ids,
                const double* lp, int64_t n_tokens, int32_t n_seq, int32_t vocab, const prorl_packed* out,
                cudaStream_t st) {
  PRORL_TRY_INTERNAL(launch_pack_turns(ctx, turns, n_turns, n_tokens, n_seq, vocab, out, st));
  return launch_pack_tokens(ctx, turns, n_turns, ids, lp, n_tokens, n_seq, vocab, out, 0, n_tokens, 0, true, st);
}

}  // namespace prorl
