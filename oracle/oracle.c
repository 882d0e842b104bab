/*
 * oracle.c — CPU ORACLE. TEST INFRASTRUCTURE ONLY: imported solely by tests/,
 * __graft_entry__.smoke() (as the checker) and bench.py's cpu_baseline /
 * --impl reference leg. The product path never links or calls it.
 *
 * A plain-C restatement of the trainer-side scoring path of ProRL Agent
 * (arXiv 2603.18815). Where the reference owns the semantics this file follows
 * it line by line (citations are to /root/reference):
 *   - packing order / role->mask rule: TokenTrajectory::flatten_range
 *     (proj/include/rollout/trajectory.hpp:76-87, rule :82-83), turn
 *     validation (:89-99);
 *   - FAILED exclusion + DAPO zero-variance gate: PromptGroup::usable_rewards
 *     and is_informative (proj/src/trainer/harness.cpp:84-102);
 *   - synthetic ids / behaviour logprobs: fnv1a64, hash_token, token_logprob
 *     (proj/src/mock/policy.cpp:10-53).
 * The arithmetic the reference does not have follows the
 * definitions fixed in SURVEY.md Appendix B and is computed in fp64:
 *   - logprob / entropy (B.2), GRPO advantage (B.3), DAPO clipped surrogate
 *     (B.4), metrics and the 332-double partials layout (B.5, B.6).
 * Parity status: packing / gate / generators are PINNED against the compiled
 * reference (oracle/_ref, tests/test_oracle_golden.py) and the reference's own
 * golden vectors (tests/golden/); logprob / entropy / advantage / loss are a
 * restatement with NO reference implementation: logprob and
 * entropy are pinned to the third-party prime-rl selective_log_softmax /
 * compute_entropy (tests/test_oracle_golden.py), advantage and loss to
 * hand-computed cases (no third-party GRPO/DAPO code exists in the image).
 *
 * Build: oracle/Makefile (gcc -O3 -ffp-contract=off -fPIC -shared -pthread).
 */
#define _GNU_SOURCE /* pthread_barrier_t, clock_gettime under -std=c11 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "prorl_hotpath.h"
#include "prorl_synth.h"

/* ---- reference generators (proj/src/mock/policy.cpp) ---------------------- */

/* policy.cpp:10-17 */
uint64_t oracle_fnv1a64(const void* data, size_t len, uint64_t state) {
  const unsigned char* p = (const unsigned char*)data;
  for (size_t i = 0; i < len; ++i) {
    state ^= p[i];
    state *= 1099511628211ULL;
  }
  return state;
}

/* policy.cpp:21-25: 8 little-endian bytes */
static uint64_t feed_u64(uint64_t state, uint64_t v) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = (unsigned char)((v >> (8 * i)) & 0xFF);
  return oracle_fnv1a64(b, 8, state);
}

/* policy.cpp:42-49 */
int64_t oracle_hash_token(uint64_t seed, const int64_t* prompt, int64_t n_prompt, uint64_t k, int64_t vocab) {
  uint64_t s = 14695981039346656037ULL;
  s = feed_u64(s, seed);
  for (int64_t i = 0; i < n_prompt; ++i) s = feed_u64(s, (uint64_t)prompt[i]);
  s = feed_u64(s, k);
  return (int64_t)(s % (uint64_t)vocab);
}

/* policy.cpp:51-53 */
double oracle_token_logprob(int64_t t) { return -(1.0 + (double)(t % 7) / 10.0); }

/* ---- trajectory semantics (trajectory.hpp) ---------------------------------- */

/* trajectory.hpp:89-99 — 0 ok, 1 MalformedTurn */
int oracle_validate_turn(int role, int64_t n_input, int64_t n_output, int64_t n_logprobs) {
  if (role == PRORL_ROLE_ASSISTANT) {
    if (n_input != 0) return 1;
    if (n_logprobs != n_output) return 1;
  } else {
    if (n_output != 0 || n_logprobs != 0) return 1;
  }
  return 0;
}

/* trajectory.hpp:76-87 over well-formed turns given as (role, len, ids). */
int64_t oracle_flatten(int n_turns, const int* roles, const int64_t* lens, const int64_t* ids, int64_t begin,
                       int64_t end, int64_t* out, int64_t cap) {
  int64_t off = 0, n = 0;
  (void)roles; /* the token field is chosen by role, but both carry `ids` here */
  for (int i = 0; i < n_turns; ++i) {
    if (i >= begin && i < end) {
      for (int64_t k = 0; k < lens[i]; ++k) {
        if (n < cap) out[n] = ids[off + k];
        ++n;
      }
    }
    off += lens[i];
  }
  return n;
}

/* harness.cpp:84-90 */
int oracle_usable_rewards(int n, const int* has, const int* failed, const double* rewards, double* out) {
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (has[i] && !failed[i]) out[m++] = rewards[i];
  return m;
}

/* harness.cpp:92-102 — 1/0, -2 = IncompleteGroup */
int oracle_is_informative(int n, const int* has, const int* failed, const double* rewards, double tol) {
  int complete = n > 0;
  for (int i = 0; i < n; ++i) complete &= has[i] != 0;
  if (!complete) return -2;
  double mn = INFINITY, mx = -INFINITY;
  int m = 0;
  for (int i = 0; i < n; ++i) {
    if (failed[i]) continue;
    ++m;
    if (rewards[i] < mn) mn = rewards[i];
    if (rewards[i] > mx) mx = rewards[i];
  }
  if (m < 2) return 0;
  return (mx - mn) > tol ? 1 : 0;
}

/* ---- B.1 packing ------------------------------------------------------------ */

typedef struct oracle_packed {
  int32_t* tokens; uint8_t* loss_mask; int16_t* turn_id; int32_t* seq_id; int32_t* pos_id;
  int32_t* cu_seqlens; float* old_lp;
  int32_t* act_row; int32_t* act_target; float* act_old_lp; int32_t* act_seq; int16_t* act_turn;
  int64_t n_active;
} oracle_packed;

/* 0 ok; PRORL_E_SHAPE (bad descriptors / count); PRORL_E_TOKEN_RANGE. */
int oracle_pack(const prorl_turn_desc* turns, int64_t n_turns, const int64_t* ids, const double* lp, int64_t n_tokens,
                int32_t n_seq, int32_t vocab, oracle_packed* o) {
  int64_t total = 0;
  for (int64_t t = 0; t < n_turns; ++t) {
    const prorl_turn_desc* d = &turns[t];
    if (d->traj < 0 || d->traj >= n_seq || d->len < 0 || d->role > PRORL_ROLE_TOOL) return PRORL_E_SHAPE;
    if (t > 0 && d->traj < turns[t - 1].traj) return PRORL_E_SHAPE;
    total += d->len;
  }
  if (total != n_tokens) return PRORL_E_SHAPE;
  for (int32_t s = 0; s <= n_seq; ++s) o->cu_seqlens[s] = 0;
  for (int64_t t = 0; t < n_turns; ++t) o->cu_seqlens[turns[t].traj + 1] += turns[t].len;
  for (int32_t s = 0; s < n_seq; ++s) o->cu_seqlens[s + 1] += o->cu_seqlens[s];
  int64_t p = 0, ord = 0;
  int32_t cur = -1;
  for (int64_t t = 0; t < n_turns; ++t) {
    const prorl_turn_desc* d = &turns[t];
    if (d->traj != cur) {
      cur = d->traj;
      ord = 0;
    }
    const int asst = d->role == PRORL_ROLE_ASSISTANT;
    for (int32_t k = 0; k < d->len; ++k, ++p) {
      const int64_t id = ids[d->src_off + k];
      if (id < 0 || id >= vocab) return PRORL_E_TOKEN_RANGE;
      o->tokens[p] = (int32_t)id;
      o->loss_mask[p] = (uint8_t)asst;
      o->turn_id[p] = asst ? (int16_t)(ord > 32767 ? 32767 : ord) : (int16_t)-1;
      o->seq_id[p] = d->traj;
      o->pos_id[p] = (int32_t)(p - o->cu_seqlens[d->traj]);
      o->old_lp[p] = asst ? (float)lp[d->src_off + k] : 0.0f;
    }
    if (asst) ++ord;
  }
  int64_t a = 0;
  for (int64_t r = 0; r + 1 < n_tokens; ++r) {
    if (o->loss_mask[r + 1] && o->pos_id[r + 1] > 0) {
      if (o->act_row) {
        o->act_row[a] = (int32_t)r;
        o->act_target[a] = o->tokens[r + 1];
        o->act_old_lp[a] = o->old_lp[r + 1];
        o->act_seq[a] = o->seq_id[r + 1];
        o->act_turn[a] = o->turn_id[r + 1];
      }
      ++a;
    }
  }
  o->n_active = a;
  return 0;
}

/* ---- B.3 GRPO --------------------------------------------------------------- */

/* Per group over usable rollouts; informative as harness.cpp:92-102. */
void oracle_grpo(const double* reward, const uint8_t* usable, const int32_t* goff, int32_t n_groups, int32_t ddof,
                 double eps, double tol, double* adv, uint8_t* informative, double* adv_sum, double* n_rollouts) {
  double asum = 0.0, nr = 0.0;
  for (int32_t g = 0; g < n_groups; ++g) {
    const int32_t b = goff[g], e = goff[g + 1];
    double sum = 0.0, mn = INFINITY, mx = -INFINITY;
    int32_t n = 0;
    for (int32_t i = b; i < e; ++i) {
      if (!usable[i]) continue;
      sum += reward[i];
      ++n;
      if (reward[i] < mn) mn = reward[i];
      if (reward[i] > mx) mx = reward[i];
    }
    const int info = n >= 2 && (mx - mn) > tol && n - ddof > 0;
    informative[g] = (uint8_t)info;
    const double mean = n > 0 ? sum / n : 0.0;
    double ss = 0.0;
    for (int32_t i = b; i < e; ++i)
      if (usable[i]) ss += (reward[i] - mean) * (reward[i] - mean);
    const double sd = info ? sqrt(ss / (double)(n - ddof)) : 0.0;
    for (int32_t i = b; i < e; ++i) {
      adv[i] = (info && usable[i]) ? (reward[i] - mean) / (sd + eps) : 0.0;
      if (info) asum += adv[i];
    }
    if (info) nr += n;
  }
  if (adv_sum) *adv_sum = asum;
  if (n_rollouts) *n_rollouts = nr;
}

/* ---- synthetic logits (include/prorl_synth.h) -------------------------------- */

void oracle_gen_logits(void* out, int dtype, int64_t row_stride, int32_t vocab, int64_t n_rows, int64_t row_key0,
                       const int32_t* targets, const float* old_lp, uint64_t seed, float sigma) {
  const uint32_t s0 = prorl_seed_mix(seed);
  const float scale = (float)((double)sigma * sqrt(3.0));
  const float base = prorl_plant_base(vocab, sigma);
  for (int64_t i = 0; i < n_rows; ++i) {
    const uint64_t key = (uint64_t)(row_key0 + i);
    for (int32_t c = 0; c < vocab; ++c) {
      float x;
      if (old_lp && targets[i] == c)
        x = prorl_plant_logit(key, s0, base, old_lp[i]);
      else
        x = prorl_noise_logit(key * (uint64_t)vocab + (uint64_t)c, s0, scale);
      if (dtype == PRORL_BF16)
        ((uint16_t*)out)[i * row_stride + c] = prorl_f32_to_bf16_bits(x);
      else
        ((float*)out)[i * row_stride + c] = x;
    }
  }
}

/* ---- B.2 logprob / entropy ---------------------------------------------------- */

static inline double logit_at(const void* row, int dtype, int64_t v) {
  return dtype == PRORL_BF16 ? (double)prorl_bf16_bits_to_f32(((const uint16_t*)row)[v]) : (double)((const float*)row)[v];
}

void oracle_row_logprob(const void* row, int dtype, int32_t vocab, int32_t target, float inv_temp, double* logp,
                        double* entropy) {
  const double it = (double)inv_temp;
  double m = -INFINITY;
  int32_t vmax = 0;
  for (int32_t v = 0; v < vocab; ++v) {
    double x = logit_at(row, dtype, v) * it;
    if (x > m) {
      m = x;
      vmax = v;
    }
  }
  /* S = 1 + S_rest with the (first) maximum kept out of S_rest, so that
   * ln S = log1p(S_rest) keeps full relative precision when p_max -> 1 */
  double Sr = 0.0, T = 0.0;
  for (int32_t v = 0; v < vocab; ++v) {
    double x = logit_at(row, dtype, v) * it;
    if (x == -INFINITY || v == vmax) continue;
    double e = exp(x - m);
    Sr += e;
    T += (x - m) * e;
  }
  const double lnS = log1p(Sr);
  *logp = logit_at(row, dtype, target) * it - m - lnS;
  *entropy = lnS - T / (1.0 + Sr);
}

void oracle_logprob_entropy(const void* logits, int dtype, int64_t row_stride, int32_t vocab, const int32_t* rows,
                            const int32_t* targets, int64_t n_rows, float inv_temp, double* logp, double* entropy) {
  const size_t es = dtype == PRORL_BF16 ? 2 : 4;
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t r = rows ? rows[i] : i;
    oracle_row_logprob((const char*)logits + (size_t)r * row_stride * es, dtype, vocab, targets[i], inv_temp, &logp[i],
                       &entropy[i]);
  }
}

/* ---- B.4-B.6 loss + metrics ------------------------------------------------------ */

/* Adds one row into partials / abs_partials (|term| sums, used as the
 * condition scale of the tolerance) and counts borderline clip decisions. */
static void loss_row(double logp, double ent, double old, double A, int turn, double lo, double hi, int n_buckets,
                     const double* ref, double kl_coef, double* P, double* Q, int64_t* n_border) {
  const double ratio = exp(logp - old);
  const double pg1 = ratio * A;
  const double cr = ratio < lo ? lo : (ratio > hi ? hi : ratio);
  const double pg2 = cr * A;
  /* k3 KL vs the reference policy (coefficient 1e-4) */
  const double kl = ref ? expm1(*ref - logp) - (*ref - logp) : 0.0;
  const double loss = -(pg1 < pg2 ? pg1 : pg2) + kl_coef * kl;
  const double clo = (ratio < lo && A < 0) ? 1.0 : 0.0;
  const double chi = (ratio > hi && A > 0) ? 1.0 : 0.0;
  if (n_border && (fabs(ratio - lo) <= 1e-5 * lo || fabs(ratio - hi) <= 1e-5 * hi)) ++*n_border;
  const double g[8] = {loss, 1.0, ent, logp, ratio, clo, chi, old - logp};
  for (int k = 0; k < 8; ++k) {
    P[k] += g[k];
    if (Q) Q[k] += fabs(g[k]);
  }
  P[PRORL_P_KL_SUM] += kl;
  if (Q) Q[PRORL_P_KL_SUM] += fabs(kl);
  int b = turn < 0 ? 0 : (turn >= n_buckets ? n_buckets - 1 : turn);
  const double bv[5] = {1.0, loss, ent, logp, clo + chi};
  for (int k = 0; k < 5; ++k) {
    P[PRORL_N_GLOBAL + 5 * b + k] += bv[k];
    if (Q) Q[PRORL_N_GLOBAL + 5 * b + k] += fabs(bv[k]);
  }
}

void oracle_loss(const double* logp, const double* ent, const float* old_lp, const double* adv, const int32_t* row_seq,
                 const int16_t* row_turn, const float* ref_lp, int64_t n_rows, float eps_lo, float eps_hi, float kl_coef,
                 int n_buckets, double* partials, double* abs_partials, int64_t* n_border) {
  const double lo = 1.0 - (double)eps_lo, hi = 1.0 + (double)eps_hi;
  for (int64_t i = 0; i < n_rows; ++i) {
    const double ref = ref_lp ? (double)ref_lp[i] : 0.0;
    loss_row(logp[i], ent[i], (double)old_lp[i], adv[row_seq[i]], row_turn[i], lo, hi, n_buckets,
             ref_lp ? &ref : NULL, (double)kl_coef, partials, abs_partials, n_border);
  }
}

/* ---- K5: backward through the log-softmax (SURVEY §8 f rank 1) ------------------------ */

/* grad[i][v] = g_i * invT * (1[v=y] - p_v), g_i = -A ratio / n_global if the
 * unclipped branch is the min (B.4), else 0; fp64 from the oracle's own logp.
 * border[i] = 1 when the clip decision is within 1e-5 of flipping. */
void oracle_logits_grad(const void* logits, int dtype, int64_t row_stride, int32_t vocab, const int32_t* rows,
                        const int32_t* targets, const float* old_lp, const double* adv, const int32_t* row_seq,
                        const float* ref_lp, int64_t n_rows, float inv_temp, float eps_lo, float eps_hi,
                        float kl_coef, double n_global, double* grad, double* dlogp, uint8_t* border) {
  const size_t es = dtype == PRORL_BF16 ? 2 : 4;
  const double it = (double)inv_temp, lo = 1.0 - (double)eps_lo, hi = 1.0 + (double)eps_hi;
  for (int64_t i = 0; i < n_rows; ++i) {
    const int64_t r = rows ? rows[i] : i;
    const char* row = (const char*)logits + (size_t)r * row_stride * es;
    double lp, ent;
    oracle_row_logprob(row, dtype, vocab, targets[i], inv_temp, &lp, &ent);
    const double lse = logit_at(row, dtype, targets[i]) * it - lp;
    const double A = adv[row_seq[i]];
    const double ratio = exp(lp - (double)old_lp[i]);
    const double pg1 = ratio * A, pg2 = (ratio < lo ? lo : (ratio > hi ? hi : ratio)) * A;
    double g = pg1 <= pg2 ? -A * ratio / n_global : 0.0;
    if (ref_lp) g += (double)kl_coef * (1.0 - exp((double)ref_lp[i] - lp)) / n_global;
    if (dlogp) dlogp[i] = g;
    if (border) border[i] = (fabs(ratio - lo) <= 1e-5 * lo || fabs(ratio - hi) <= 1e-5 * hi) ? 1 : 0;
    double* gr = grad + (size_t)i * vocab;
    for (int32_t v = 0; v < vocab; ++v) {
      const double x = logit_at(row, dtype, v) * it;
      const double pv = x == -INFINITY ? 0.0 : exp(x - lse);
      /* 1 - p_y = -expm1(logp): exact as p_y -> 1 */
      gr[v] = v == targets[i] ? -g * it * expm1(lp) : -g * it * pv;
    }
  }
}

/* ---- full CPU path ------------------------------------------------------------------- */

typedef struct {
  const oracle_packed* pk;
  const double* adv;
  const prorl_score_cfg* cfg;
  const int64_t* rollout_key;
  uint64_t seed;
  float sigma;
  int64_t r0, r1;
  double P[PRORL_N_PARTIALS], Q[PRORL_N_PARTIALS];
  int64_t n_border;
  double* out_logp;
  double* out_ent;
  double gen_s, score_s;
} work_t;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void* score_worker(void* arg) {
  work_t* w = (work_t*)arg;
  const prorl_score_cfg* cfg = w->cfg;
  const size_t es = cfg->dtype == PRORL_BF16 ? 2 : 4;
  void* row = malloc((size_t)cfg->vocab * es);
  const double lo = 1.0 - (double)cfg->loss.eps_lo, hi = 1.0 + (double)cfg->loss.eps_hi;
  for (int64_t i = w->r0; i < w->r1; ++i) {
    double t0 = now_s();
    /* key = rollout_key[s] * 2^20 + position in the sequence (prorl_gen_logits_keyed) */
    const int32_t s = w->pk->act_seq[i];
    const int64_t key = (w->rollout_key ? w->rollout_key[s] : (int64_t)s) * ((int64_t)1 << 20) +
                        (int64_t)(w->pk->act_row[i] - w->pk->cu_seqlens[s]);
    oracle_gen_logits(row, cfg->dtype, cfg->vocab, cfg->vocab, 1, key, &w->pk->act_target[i], &w->pk->act_old_lp[i],
                      w->seed, w->sigma);
    double t1 = now_s();
    double lp, ent;
    oracle_row_logprob(row, cfg->dtype, cfg->vocab, w->pk->act_target[i], cfg->inv_temperature, &lp, &ent);
    loss_row(lp, ent, (double)w->pk->act_old_lp[i], w->adv[w->pk->act_seq[i]], w->pk->act_turn[i], lo, hi,
             cfg->loss.n_buckets, NULL, 0.0, w->P, w->Q, &w->n_border);
    if (w->out_logp) w->out_logp[i] = lp;
    if (w->out_ent) w->out_ent[i] = ent;
    w->gen_s += t1 - t0;
    w->score_s += now_s() - t1;
  }
  free(row);
  return NULL;
}

/* The whole step on the CPU for one shard: pack (B.1) -> GRPO (B.3) -> per
 * active row: synthetic logits row (keyed as prorl_score_host with fill=1:
 * rollout_key[s] * 2^20 + position) -> logprob/entropy (B.2) -> loss/metrics (B.4-B.6). Rows
 * [row_begin, row_end) only (row_end < 0: all), split over nthreads.
 * timings[3] (s): pack+grpo, scoring (logits generation excluded, summed
 * over threads / nthreads), generation. Returns 0 or an error status. */
int oracle_score_batch(const prorl_host_batch* hb, const prorl_score_cfg* cfg, uint64_t seed, float sigma,
                       int nthreads, int64_t row_begin, int64_t row_end, double* partials, double* abs_partials,
                       int64_t* n_border, double* out_logp, double* out_ent, int64_t* n_active_out, double* timings) {
  const int64_t N = hb->n_tokens;
  const int32_t R = hb->n_rollouts;
  double t0 = now_s();
  oracle_packed pk;
  memset(&pk, 0, sizeof pk);
  size_t n1 = (size_t)(N > 0 ? N : 1);
  pk.tokens = malloc(n1 * 4); pk.loss_mask = malloc(n1); pk.turn_id = malloc(n1 * 2); pk.seq_id = malloc(n1 * 4);
  pk.pos_id = malloc(n1 * 4); pk.cu_seqlens = malloc((size_t)(R + 1) * 4); pk.old_lp = malloc(n1 * 4);
  pk.act_row = malloc(n1 * 4); pk.act_target = malloc(n1 * 4); pk.act_old_lp = malloc(n1 * 4);
  pk.act_seq = malloc(n1 * 4); pk.act_turn = malloc(n1 * 2);
  int st = oracle_pack(hb->turns, hb->n_turns, hb->ids, hb->lp, N, R, cfg->vocab, &pk);
  double* adv = malloc((size_t)(R > 0 ? R : 1) * sizeof(double));
  uint8_t* info = malloc((size_t)(hb->n_groups > 0 ? hb->n_groups : 1));
  double asum = 0.0, nr = 0.0;
  if (st == 0) oracle_grpo(hb->reward, hb->usable, hb->group_off, hb->n_groups, cfg->ddof, (double)cfg->adv_eps,
                           cfg->gate_tolerance,
                           adv, info, &asum, &nr);
  double t1 = now_s();
  if (st == 0) {
    int64_t a0 = row_begin < 0 ? 0 : row_begin, a1 = (row_end < 0 || row_end > pk.n_active) ? pk.n_active : row_end;
    if (a1 < a0) a1 = a0;
    if (nthreads < 1) nthreads = 1;
    work_t* w = calloc((size_t)nthreads, sizeof(work_t));
    pthread_t* th = calloc((size_t)nthreads, sizeof(pthread_t));
    const int64_t n = a1 - a0;
    for (int k = 0; k < nthreads; ++k) {
      w[k].pk = &pk; w[k].adv = adv; w[k].cfg = cfg; w[k].seed = seed; w[k].sigma = sigma;
      w[k].rollout_key = hb->rollout_key;
      w[k].r0 = a0 + n * k / nthreads; w[k].r1 = a0 + n * (k + 1) / nthreads;
      w[k].out_logp = out_logp; w[k].out_ent = out_ent;
      pthread_create(&th[k], NULL, score_worker, &w[k]);
    }
    double gen = 0.0, sc = 0.0;
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
    for (int k = 0; k < nthreads; ++k) {
      for (int j = 0; j < PRORL_N_PARTIALS; ++j) {
        partials[j] += w[k].P[j];
        if (abs_partials) abs_partials[j] += w[k].Q[j];
      }
      if (n_border) *n_border += w[k].n_border;
      gen += w[k].gen_s;
      sc += w[k].score_s;
    }
    partials[PRORL_P_ADV_SUM] += asum;
    partials[PRORL_P_N_ROLLOUTS] += nr;
    if (abs_partials) abs_partials[PRORL_P_N_ROLLOUTS] += nr;
    if (timings) {
      timings[0] = t1 - t0;
      timings[1] = sc / nthreads;
      timings[2] = gen / nthreads;
    }
    free(w);
    free(th);
  }
  if (n_active_out) *n_active_out = pk.n_active;
  free(pk.tokens); free(pk.loss_mask); free(pk.turn_id); free(pk.seq_id); free(pk.pos_id); free(pk.cu_seqlens);
  free(pk.old_lp); free(pk.act_row); free(pk.act_target); free(pk.act_old_lp); free(pk.act_seq); free(pk.act_turn);
  free(adv);
  free(info);
  return st;
}

/* ---- timed stratified sample (bench.py cpu_baseline / --impl reference) ----------------
 * The whole-step CPU path on a systematic (stratified) sample of a shard's
 * active rows: rows offset, offset + stride, ... (at most max_rows), so every
 * group, rollout and turn position of the shard is represented. Threads work in
 * lock-step rounds: each generates a block of its rows' synthetic logits (the
 * LM-head stand-in, outside the metric), a barrier, then all score their
 * blocks; timings[1] is the WALL-CLOCK time of the scoring phases only,
 * timings[0] the wall time of pack + GRPO over the whole shard, timings[2]
 * the wall time of the generation phases. */
typedef struct {
  const oracle_packed* pk;
  const double* adv;
  const prorl_score_cfg* cfg;
  const int64_t* rollout_key;
  uint64_t seed;
  float sigma;
  int64_t s0, s1, stride, offset; /* this thread's sample indices [s0, s1) */
  int tid, nthreads;
  pthread_barrier_t* bar;
  double P[PRORL_N_PARTIALS], Q[PRORL_N_PARTIALS];
  int64_t n_border;
  double* wall; /* [2]: scoring, generation (written by thread 0) */
  int64_t rounds;
} sample_t;

#define SAMPLE_BLOCK 16

static void* sample_worker(void* arg) {
  sample_t* w = (sample_t*)arg;
  const prorl_score_cfg* cfg = w->cfg;
  const size_t es = cfg->dtype == PRORL_BF16 ? 2 : 4;
  char* buf = malloc((size_t)SAMPLE_BLOCK * (size_t)cfg->vocab * es);
  const double lo = 1.0 - (double)cfg->loss.eps_lo, hi = 1.0 + (double)cfg->loss.eps_hi;
  for (int64_t r = 0; r < w->rounds; ++r) {
    const int64_t b0 = w->s0 + r * SAMPLE_BLOCK;
    const int64_t b1 = b0 + SAMPLE_BLOCK < w->s1 ? b0 + SAMPLE_BLOCK : w->s1;
    double t0 = 0.0;
    if (w->tid == 0) t0 = now_s();
    for (int64_t s = b0; s < b1; ++s) { /* generation phase */
      const int64_t i = w->offset + s * w->stride;
      const int32_t q = w->pk->act_seq[i];
      const int64_t key = (w->rollout_key ? w->rollout_key[q] : (int64_t)q) * ((int64_t)1 << 20) +
                          (int64_t)(w->pk->act_row[i] - w->pk->cu_seqlens[q]);
      oracle_gen_logits(buf + (size_t)(s - b0) * cfg->vocab * es, cfg->dtype, cfg->vocab, cfg->vocab, 1, key,
                        &w->pk->act_target[i], &w->pk->act_old_lp[i], w->seed, w->sigma);
    }
    pthread_barrier_wait(w->bar);
    double t1 = 0.0;
    if (w->tid == 0) {
      t1 = now_s();
      w->wall[1] += t1 - t0;
    }
    for (int64_t s = b0; s < b1; ++s) { /* scoring phase (timed) */
      const int64_t i = w->offset + s * w->stride;
      double lp, ent;
      oracle_row_logprob(buf + (size_t)(s - b0) * cfg->vocab * es, cfg->dtype, cfg->vocab, w->pk->act_target[i],
                         cfg->inv_temperature, &lp, &ent);
      loss_row(lp, ent, (double)w->pk->act_old_lp[i], w->adv[w->pk->act_seq[i]], w->pk->act_turn[i], lo, hi,
               cfg->loss.n_buckets, NULL, 0.0, w->P, w->Q, &w->n_border);
    }
    pthread_barrier_wait(w->bar);
    if (w->tid == 0) w->wall[0] += now_s() - t1;
  }
  free(buf);
  return NULL;
}

int oracle_score_sample(const prorl_host_batch* hb, const prorl_score_cfg* cfg, uint64_t seed, float sigma,
                        int nthreads, int64_t stride, int64_t offset, int64_t max_rows, double* partials,
                        double* abs_partials, int64_t* n_border, int64_t* n_scored, int64_t* n_active_out,
                        double* timings) {
  const int64_t N = hb->n_tokens;
  const int32_t R = hb->n_rollouts;
  if (stride < 1 || offset < 0 || nthreads < 1) return PRORL_E_MALFORMED_REQUEST;
  double t0 = now_s();
  oracle_packed pk;
  memset(&pk, 0, sizeof pk);
  size_t n1 = (size_t)(N > 0 ? N : 1);
  pk.tokens = malloc(n1 * 4); pk.loss_mask = malloc(n1); pk.turn_id = malloc(n1 * 2); pk.seq_id = malloc(n1 * 4);
  pk.pos_id = malloc(n1 * 4); pk.cu_seqlens = malloc((size_t)(R + 1) * 4); pk.old_lp = malloc(n1 * 4);
  pk.act_row = malloc(n1 * 4); pk.act_target = malloc(n1 * 4); pk.act_old_lp = malloc(n1 * 4);
  pk.act_seq = malloc(n1 * 4); pk.act_turn = malloc(n1 * 2);
  int st = oracle_pack(hb->turns, hb->n_turns, hb->ids, hb->lp, N, R, cfg->vocab, &pk);
  double* adv = malloc((size_t)(R > 0 ? R : 1) * sizeof(double));
  uint8_t* info = malloc((size_t)(hb->n_groups > 0 ? hb->n_groups : 1));
  double asum = 0.0, nr = 0.0;
  if (st == 0)
    oracle_grpo(hb->reward, hb->usable, hb->group_off, hb->n_groups, cfg->ddof, (double)cfg->adv_eps,
                cfg->gate_tolerance, adv, info, &asum, &nr);
  double t1 = now_s();
  int64_t n_sample = 0;
  if (st == 0 && offset < pk.n_active) {
    n_sample = (pk.n_active - offset + stride - 1) / stride;
    if (max_rows >= 0 && n_sample > max_rows) n_sample = max_rows;
    sample_t* w = calloc((size_t)nthreads, sizeof(sample_t));
    pthread_t* th = calloc((size_t)nthreads, sizeof(pthread_t));
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)nthreads);
    double wall[2] = {0.0, 0.0};
    const int64_t per = (n_sample + nthreads - 1) / nthreads;
    const int64_t rounds = (per + SAMPLE_BLOCK - 1) / SAMPLE_BLOCK;
    for (int k = 0; k < nthreads; ++k) {
      w[k].pk = &pk; w[k].adv = adv; w[k].cfg = cfg; w[k].seed = seed; w[k].sigma = sigma;
      w[k].rollout_key = hb->rollout_key;
      w[k].s0 = per * k < n_sample ? per * k : n_sample;
      w[k].s1 = per * (k + 1) < n_sample ? per * (k + 1) : n_sample;
      w[k].stride = stride; w[k].offset = offset; w[k].tid = k; w[k].nthreads = nthreads;
      w[k].bar = &bar; w[k].wall = wall; w[k].rounds = rounds;
      pthread_create(&th[k], NULL, sample_worker, &w[k]);
    }
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
    for (int k = 0; k < nthreads; ++k) {
      for (int j = 0; j < PRORL_N_PARTIALS; ++j) {
        partials[j] += w[k].P[j];
        if (abs_partials) abs_partials[j] += w[k].Q[j];
      }
      if (n_border) *n_border += w[k].n_border;
    }
    pthread_barrier_destroy(&bar);
    if (timings) {
      timings[0] = t1 - t0;
      timings[1] = wall[0];
      timings[2] = wall[1];
    }
    free(w);
    free(th);
  }
  if (n_scored) *n_scored = n_sample;
  if (n_active_out) *n_active_out = pk.n_active;
  free(pk.tokens); free(pk.loss_mask); free(pk.turn_id); free(pk.seq_id); free(pk.pos_id); free(pk.cu_seqlens);
  free(pk.old_lp); free(pk.act_row); free(pk.act_target); free(pk.act_old_lp); free(pk.act_seq); free(pk.act_turn);
  free(adv);
  free(info);
  return st;
}
