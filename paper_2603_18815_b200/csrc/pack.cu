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

// One thread per token p: locate its turn (binary search over turn offsets),
// convert id / logprob, emit mask, ids, and the active flag of row p-1.
__global__ void k_pack_tokens(const prorl_turn_desc* __restrict__ turns, int64_t n_turns,
                              const int64_t* __restrict__ off, const int64_t* __restrict__ asst0,
                              const int64_t* __restrict__ ids, const double* __restrict__ lp,
                              int64_t n_tokens, int32_t n_seq, int32_t vocab, prorl_packed out, uint8_t* flags,
                              int* err) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_tokens) return;
  if (p == 0) flags[n_tokens - 1] = 0;
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
  if (p > 0) flags[p - 1] = (asst && pos > 0) ? 1 : 0;
}

__global__ void k_compact(const uint8_t* __restrict__ flags, const int32_t* __restrict__ pos,
                          int64_t n_tokens, prorl_packed out) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0) *out.n_active = (int64_t)pos[n_tokens];
  if (r >= n_tokens || !flags[r]) return;
  const int32_t i = pos[r];
  out.act_row[i] = (int32_t)r;
  out.act_target[i] = out.tokens[r + 1];
  out.act_old_lp[i] = out.old_lp[r + 1];
  out.act_seq[i] = out.seq_id[r + 1];
  out.act_turn[i] = out.turn_id[r + 1];
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

int launch_pack(prorl_ctx* ctx, const prorl_turn_desc* turns, int64_t n_turns, const int64_t* ids,
                const double* lp, int64_t n_tokens, int32_t n_seq, int32_t vocab, const prorl_packed* out,
                cudaStream_t st) {
  if (n_turns < 0 || n_tokens < 0 || n_seq < 0 || vocab <= 0)
    return fail(PRORL_E_SHAPE, "prorl_pack: negative size or vocab <= 0");
  if (n_tokens >= (int64_t(1) << 31) - 1)
    return fail(PRORL_E_SHAPE, "prorl_pack: more than 2^31-2 tokens per shard");
  if (n_tokens > 0 && n_turns == 0) return fail(PRORL_E_SHAPE, "prorl_pack: tokens without turns");
  // workspace: off[n_turns+1] i64 | asst0[n_seq] i64 | act_pos[N+1] i32 | flags[N] u8
  size_t o_off = 0;
  size_t o_asst = o_off + sizeof(int64_t) * (size_t)(n_turns + 1);
  size_t o_pos = o_asst + sizeof(int64_t) * (size_t)(n_seq + 1);
  size_t o_flag = o_pos + sizeof(int32_t) * (size_t)(n_tokens + 1);
  size_t total = o_flag + (size_t)n_tokens + 16;
  PRORL_CUDA(ctx->pack_tmp.ensure(total));
  size_t scan_elems = scan_tmp_elems(n_turns > n_tokens ? n_turns : n_tokens) + 1;
  PRORL_CUDA(ctx->scan_tmp.ensure(scan_elems * sizeof(int64_t)));
  uint8_t* base = ctx->pack_tmp.as<uint8_t>();
  int64_t* off = reinterpret_cast<int64_t*>(base + o_off);
  int64_t* asst0 = reinterpret_cast<int64_t*>(base + o_asst);
  int32_t* pos = reinterpret_cast<int32_t*>(base + o_pos);
  uint8_t* flags = base + o_flag;

  PRORL_CUDA(exclusive_scan<int64_t>(TurnVal{turns}, n_turns, off, ctx->scan_tmp.as<int64_t>(), st));
  k_seq_bounds<<<blocks_for(n_turns + 1, 256), 256, 0, st>>>(turns, n_turns, off, n_seq, n_tokens,
                                                               out->cu_seqlens, asst0, ctx->d_err);
  PRORL_CUDA(cudaGetLastError());
  if (n_tokens == 0) {
    PRORL_CUDA(cudaMemsetAsync(out->n_active, 0, sizeof(int64_t), st));
    return PRORL_OK;
  }
  PRORL_CUDA(cudaMemsetAsync(flags, 0, (size_t)n_tokens, st));
  k_pack_tokens<<<blocks_for(n_tokens, 256), 256, 0, st>>>(turns, n_turns, off, asst0, ids, lp, n_tokens,
                                                            n_seq, vocab, *out, flags, ctx->d_err);
  PRORL_CUDA(cudaGetLastError());
  PRORL_CUDA(exclusive_scan<int32_t>(FlagVal{flags}, n_tokens, pos, ctx->scan_tmp.as<int32_t>(), st));
  k_compact<<<blocks_for(n_tokens, 256), 256, 0, st>>>(flags, pos, n_tokens, *out);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

}  // namespace prorl
