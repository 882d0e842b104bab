// score.cu — K2 (vocab-streaming logprob + entropy) with an optional fused K4
// epilogue (DAPO clipped surrogate + per-turn metrics), the standalone K4 and
// the deterministic slab reduction.
//
// No reference code exists for this arithmetic; definitions
// are SURVEY.md App. B.2 (logprob/entropy), B.4 (loss), B.5/B.6 (metrics).
//
// K2 design (HBM-bound: 2V bytes per bf16 row, read exactly once):
//   * one warp owns one row at a time (rows strided over a persistent grid of
//     one CTA per SM), so a row never needs a cross-warp reduction;
//   * each warp has a private ring of STAGES x CHUNK bytes of shared memory fed
//     by 1-D TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx, L2
//     evict_first) issued by lane 0, running ahead across row boundaries; a
//     chunk is pulled into registers with LDS.128 and its stage released at
//     once;
//   * online base-2 logsumexp with a WARP-UNIFORM running max Mc of x*c
//     (raised only when a group beats it by more than 1 in log2 units — the
//     reference point need not be the exact max, see train.cu kRaiseSlack —
//     which skips most raises: +1.2 % at C2)
//     (c = inv_temp * log2 e): per group of SUBV*8 bf16 per lane a packed
//     max (HMNMX2) and one vote decide whether the max moved; only then (a
//     handful of times per row) does the warp take the rescale path, so the
//     common path has no divergence and no per-lane rescale;
//   * the current top element (the one that set Mc) is kept OUT of the sums
//     and re-added analytically at the row end, in fp64 with the fp32 scale's
//     rounding corrected (rowmath.cuh row_stats):
//         S = 2^r (1 + q),  q = S_rest 2^-r,   r = x_top*c - Mc
//         logp = (x_y - x_top) inv_T - log1p(q)
//         H    = log1p(q) + ln2 (r q - T_rest 2^-r) / (1 + q)
//     so logp and H stay accurate even when one token takes almost all the
//     probability (p -> 1, H -> 0), where a plain fp32 sum of e^(x - max)
//     cannot resolve 1 + tiny; the loss epilogue is fp64 too (row_loss);
//   * -inf / NaN / huge-negative bf16 logits are clamped to -2^97 with one
//     packed min.u16x2 per two logits (they then contribute exactly 0);
//   * unaligned row heads/tails (V*esz not a multiple of 16 B, odd row
//     offsets) are read by lanes directly, the aligned interior goes via TMA.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "rowmath.cuh"
#include "stream.cuh"

namespace prorl {

namespace {

using namespace rowmath;

// Clamped scalar re-read of one row straight from global memory (logits
// clamped to >= -2^97, so -inf contributes exactly 0). Used only for rows whose
// fast-path sums came out NaN. Returns by value (nothing of the caller's hot
// loop state is address-taken, so it stays in registers).
struct SlowRow {
  float Mc, Mx;
  double Sr, Tr;
};
template <typename T>
__device__ __noinline__ SlowRow row_slow(const uint8_t* rp, int32_t vocab, float c, int lane) {
  Top top{-INFINITY, 0.f};
  LaneSums acc;
  acc.zero();
  const float floor_v = __uint_as_float(0xf0000000u);
  for (int32_t base = 0; base < vocab; base += 32) {
    float x = base + lane < vocab ? Elem<T>::load(rp, base + lane) : floor_v;
    if (__any_sync(kFull, x * c > top.Mc)) {
      const int L = raise_top(x, c, top, acc, lane);
      if (lane == L) x = floor_v;
    }
    const float d = fmaf(x, c, -top.Mc);
    acc.add(d, ex2_approx(d));
    if ((base & 2047) == 2016) acc.fold();
  }
  acc.fold();
  return SlowRow{top.Mc, top.Mx, warp_sum_d(acc.Sd), warp_sum_d(acc.Td)};
}

struct ScoreArgs {
  const uint8_t* logits;
  int64_t stride_bytes;
  int32_t vocab;
  const int32_t* rows;
  const int32_t* targets;
  int64_t n_rows;
  float c;  // fl(inv_temp * log2(e))
  float inv_temp;
  // fused loss
  const float* old_lp;
  const double* adv;
  const int32_t* row_seq;
  const int16_t* row_turn;
  const float* ref_lp;  // nullable
  double kl_coef;
  double lo_bound, hi_bound;  // 1 - eps_lo, 1 + eps_hi (fp64, as the oracle)
  int n_buckets;
  float* logp;
  float* entropy;
  double* slab;
  int accumulate;
  float raise_slack;  // running-max hysteresis in log2 units (PRORL_K2_SLACK; see train.cu kRaiseSlack)
};

// Block-level merge of per-warp partials (fixed warp order) into slab row b.
template <int WARPS>
__device__ __forceinline__ void merge_block_partials(const double* g_w, const double* bk_w, double* slab,
                                                     int accumulate) {
  for (int t = threadIdx.x; t < PRORL_N_PARTIALS; t += blockDim.x) {
    double v = 0.0;
    if (t < kNG) {
      for (int w = 0; w < WARPS; ++w) v += g_w[w * kNG + t];
    } else if (t >= PRORL_N_GLOBAL) {
      for (int w = 0; w < WARPS; ++w) v += bk_w[w * kBucketDoubles + (t - PRORL_N_GLOBAL)];
    }
    double* dst = slab + (size_t)blockIdx.x * PRORL_N_PARTIALS + t;
    *dst = accumulate ? *dst + v : v;
  }
}

template <int WARPS, int STAGES, int CHUNK, bool FUSED>
constexpr size_t score_smem_bytes() {
  return (size_t)WARPS * STAGES * CHUNK + (size_t)WARPS * STAGES * 8 +
         (FUSED ? (size_t)WARPS * (kNG + kBucketDoubles) * sizeof(double) : 0);
}

// 16-B vectors per lane between two fp64 folds of the fp32 accumulators
// (LaneSums): 256 bf16 / 128 fp32 logits, i.e. <= 64 terms per fp32 sum.
constexpr int kFoldVec = 32;

template <typename T, int WARPS, int STAGES, int CHUNK, int SUBV, bool FUSED>
__global__ void __launch_bounds__(WARPS * 32, 1) k_score(const ScoreArgs p) {
  static_assert(CHUNK % (512 * SUBV) == 0, "CHUNK must hold whole lane groups");
  constexpr int NV = CHUNK / 512;  // 16-B vectors per lane per chunk
  static_assert(kFoldVec % NV == 0, "fold period in whole chunks");
  constexpr int ES = Elem<T>::kSize;
  extern __shared__ __align__(128) uint8_t smem[];
  // the next scoring launch of the step (programmatic dependent launch) may
  // take SMs as this grid's CTAs finish; it waits for this grid only before
  // its slab update (pdl_allow_next / pdl_wait, common.cuh)
  pdl_allow_next();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = smem + (size_t)warp * STAGES * CHUNK;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * STAGES * CHUNK) + warp * STAGES;
  double* g_w = reinterpret_cast<double*>(smem + (size_t)WARPS * STAGES * CHUNK + WARPS * STAGES * 8);
  double* bk_w = g_w + WARPS * kNG;

  double g[kNG];
  if constexpr (FUSED) {
#pragma unroll
    for (int k = 0; k < kNG; ++k) g[k] = 0.0;
    for (int i = lane; i < kBucketDoubles; i += 32) bk_w[warp * kBucketDoubles + i] = 0.0;
  }

  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  RowRing<STAGES, CHUNK, ES> rr;
  rr.init(ring, bars, p.logits, p.stride_bytes, p.rows, p.n_rows, p.vocab, gw, nw, lane);

  const float c = p.c;
  const RoundFix rf(c);
  const uint4 fill = make_uint4(Elem<T>::kClampWord, Elem<T>::kClampWord, Elem<T>::kClampWord, Elem<T>::kClampWord);
  for (int64_t i = gw; i < p.n_rows; i += nw) {
    const uint8_t* rp = rr.row_ptr(i);
    uintptr_t a, b;
    rr.interior(rp, a, b);
    const int64_t nchunks = rr.chunks(a, b);
    const int head = (int)((a - reinterpret_cast<uintptr_t>(rp)) / ES);
    const int tail = (int)((reinterpret_cast<uintptr_t>(rp) + (uintptr_t)p.vocab * ES - b) / ES);
    const int32_t tgt = p.targets[i];
    float xy = 0.f;
    if (lane == 0) xy = Elem<T>::load(rp, tgt);

    Top top{-INFINITY, 0.f};
    LaneSums acc;
    acc.zero();
    if (head + tail > 0) {  // unaligned head / tail elements, one per lane (<= 14 of them)
      float x = __uint_as_float(0xf0000000u);  // -2^97: the clamp floor, contributes 0
      if (lane < head) x = Elem<T>::load(rp, lane);
      else if (lane < head + tail)
        x = Elem<T>::load(rp, (int64_t)((b - reinterpret_cast<uintptr_t>(rp)) / ES) + (lane - head));
      if (__any_sync(kFull, x * c > top.Mc)) {
        const int L = raise_top(x, c, top, acc, lane);
        if (lane == L) x = __uint_as_float(0xf0000000u);
      }
      const float d = fmaf(x, c, -top.Mc);
      acc.add(d, ex2_approx(d));
    }

    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const uint32_t nvec = (uint32_t)(min((uintptr_t)CHUNK, b - (a + (uintptr_t)ch * CHUNK)) >> 4);
      const uint4* sv = rr.wait();
      uint4 v[NV];
      if (nvec == (uint32_t)(CHUNK / 16)) {
#pragma unroll
        for (int j = 0; j < NV; ++j) v[j] = sv[lane + 32 * j];
      } else {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const uint32_t q = lane + 32 * j;
          v[j] = q < nvec ? sv[q] : fill;
        }
      }
      rr.release(lane);
#pragma unroll
      for (int g0 = 0; g0 < NV; g0 += SUBV) {
        uint4 u[SUBV];
#pragma unroll
        for (int j = 0; j < SUBV; ++j) u[j] = v[g0 + j];
        const float lm = Elem<T>::template group_max<SUBV>(u);
        if (__any_sync(kFull, lm * c > top.Mc + p.raise_slack)) {
          const int L = raise_top(lm, c, top, acc, lane);
          if (lane == L) Elem<T>::template mask_first<SUBV>(u, top.Mx);
        }
        const float2 nM2 = make_float2(-top.Mc, -top.Mc);
        // the RoundFix sample: the first pair of each group's first vector (1/32 of
        // the bf16 logits at the default configuration), branch-free
        Elem<T>::template accumulate<SUBV, ES == 2>(u, make_float2(c, c), nM2, acc.S, acc.T, &acc.R, &acc.Q, rf.chi2,
                                                    rf.clo2);
      }
      // fp64 fold every kFoldVec 16-B vectors per lane (warp-uniform)
      if ((ch + 1) % (kFoldVec / NV) == 0) acc.fold();
    }

    // ---- row end: merge lanes in fp64, re-add the top element analytically ----
    acc.fold();
    double Sr = warp_sum_d(acc.Sd);
    double Tr = warp_sum_d(acc.Td);
    if (!(Tr == Tr) || !(Sr == Sr)) {  // -inf / NaN / overflowing logits: clamped re-read (rare)
      const SlowRow sr = row_slow<T>(rp, p.vocab, c, lane);
      top = Top{sr.Mc, sr.Mx};
      Sr = sr.Sr;
      Tr = sr.Tr;
    } else if constexpr (ES == 2) {
      Sr = RoundFix::apply(Sr, acc.R, acc.Q);  // the FFMA rounding of d (sampled)
    }
    if (lane == 0) {
      const RowStats rs = row_stats(top.Mc, top.Mx, Sr, Tr, xy, c, (double)p.inv_temp);  // fp64 row end
      if (p.logp) p.logp[i] = (float)rs.logp;
      if (p.entropy) p.entropy[i] = (float)rs.ent;
      if constexpr (FUSED) {
        const float old = p.old_lp[i];
        const double A = p.adv[p.row_seq[i]];
        int k = p.row_turn[i];
        k = k < 0 ? 0 : (k >= p.n_buckets ? p.n_buckets - 1 : k);
        const RowLoss rl = row_loss(rs.logp, old, A, p.lo_bound, p.hi_bound, p.ref_lp, i, p.kl_coef);
        g[0] += rl.loss;
        g[1] += 1.0;
        g[2] += rs.ent;
        g[3] += rs.logp;
        g[4] += rl.ratio;
        g[5] += rl.clip_lo;
        g[6] += rl.clip_hi;
        g[7] += (double)old - rs.logp;
        g[10] += rl.kl;
        double* bk = bk_w + warp * kBucketDoubles + k * PRORL_N_PER_TURN;
        bk[0] += 1.0;
        bk[1] += rl.loss;
        bk[2] += rs.ent;
        bk[3] += rs.logp;
        bk[4] += rl.clip_lo + rl.clip_hi;
      }
    }
  }

  if constexpr (FUSED) {
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < kNG; ++k) g_w[warp * kNG + k] = g[k];
    }
    __syncthreads();
    pdl_wait();  // the previous scoring launch's slab rows are complete and visible
    merge_block_partials<WARPS>(g_w, bk_w, p.slab, p.accumulate);
  }
}

// ---- standalone K4 ------------------------------------------------------------
constexpr int kLossWarps = 8;

__global__ void __launch_bounds__(kLossWarps * 32)
    k_loss(const float* __restrict__ logp, const float* __restrict__ entropy, const float* __restrict__ old_lp,
           const double* __restrict__ adv, const int32_t* __restrict__ row_seq, const int16_t* __restrict__ row_turn,
           const float* __restrict__ ref_lp, double kl_coef, int64_t n_rows, double lo, double hi, int n_buckets,
           double* slab) {
  __shared__ double g_w[kLossWarps * kNG];
  __shared__ double bk_w[kLossWarps * kBucketDoubles];
  __shared__ int s_key[kLossWarps][32];
  __shared__ double s_val[kLossWarps][32][PRORL_N_PER_TURN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = lane; i < kBucketDoubles; i += 32) bk_w[warp * kBucketDoubles + i] = 0.0;
  double g[kNG];
#pragma unroll
  for (int k = 0; k < kNG; ++k) g[k] = 0.0;
  const int64_t gw = (int64_t)blockIdx.x * kLossWarps + warp, nw = (int64_t)gridDim.x * kLossWarps;
  const int64_t n_tiles = (n_rows + 31) / 32;
  __syncwarp();
  for (int64_t tile = gw; tile < n_tiles; tile += nw) {
    const int64_t i = tile * 32 + lane;
    int key = -1;
    if (i < n_rows) {
      const double lp = logp[i], ent = entropy[i];
      const float old = old_lp[i];
      const double A = adv[row_seq[i]];
      int k = row_turn[i];
      key = k < 0 ? 0 : (k >= n_buckets ? n_buckets - 1 : k);
      const RowLoss r = row_loss(lp, old, A, lo, hi, ref_lp, i, kl_coef);
      g[0] += r.loss;
      g[1] += 1.0;
      g[2] += ent;
      g[3] += lp;
      g[4] += r.ratio;
      g[5] += r.clip_lo;
      g[6] += r.clip_hi;
      g[7] += (double)old - lp;
      g[10] += r.kl;
      s_val[warp][lane][0] = 1.0;
      s_val[warp][lane][1] = r.loss;
      s_val[warp][lane][2] = ent;
      s_val[warp][lane][3] = lp;
      s_val[warp][lane][4] = r.clip_lo + r.clip_hi;
    }
    s_key[warp][lane] = key;
    __syncwarp();
    if (lane < PRORL_N_PER_TURN) {  // fixed-order per-turn accumulation
      for (int src = 0; src < 32; ++src) {
        const int kk = s_key[warp][src];
        if (kk >= 0) bk_w[warp * kBucketDoubles + kk * PRORL_N_PER_TURN + lane] += s_val[warp][src][lane];
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int k = 0; k < kNG; ++k) {
    const double v = warp_sum_d(g[k]);
    if (lane == 0) g_w[warp * kNG + k] = v;
  }
  __syncthreads();
  merge_block_partials<kLossWarps>(g_w, bk_w, slab, 0);
}

__global__ void k_slab_reduce(const double* __restrict__ slab, int rows, double* partials) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= PRORL_N_PARTIALS) return;
  double v = 0.0;
  for (int b = 0; b < rows; ++b) v += slab[(size_t)b * PRORL_N_PARTIALS + t];
  if (t != PRORL_P_ADV_SUM && t != PRORL_P_N_ROLLOUTS) partials[t] += v;
}

// ---- launch configurations ------------------------------------------------------------
// warps/CTA x stages x chunk bytes; one CTA per SM. The release library
// compiles only the default (chosen from ncu/bench measurements);
// a tuning build (-DPRORL_TUNING) selects the others with PRORL_K2_CONFIG.
struct K2Config {
  const char* name;
  int warps, stages, chunk, subv;  // subv: 16-B vectors per lane per max-check group (bf16: 8 logits each)
};
constexpr K2Config kConfigs[] = {{"w16s2c4096g2", 16, 2, 4096, 2}, {"w16s2c4096g4", 16, 2, 4096, 4},
                                 {"w12s3c4096g2", 12, 3, 4096, 2}, {"w8s5c4096g2", 8, 5, 4096, 2},
                                 {"w8s3c8192g4", 8, 3, 8192, 4}, {"w16s2c4096g8", 16, 2, 4096, 8}};
constexpr int kDefaultConfig = 5;

int active_config() {
  static int idx = [] {
    const char* e = tuning_env("PRORL_K2_CONFIG");
    if (e)
      for (int i = 0; i < (int)(sizeof(kConfigs) / sizeof(kConfigs[0])); ++i)
        if (std::strcmp(e, kConfigs[i].name) == 0) return i;
    return kDefaultConfig;
  }();
  return idx;
}

template <typename T, int W, int ST, int CH, int SUBV_BF16, bool FUSED>
int run_score_cfg(const ScoreArgs& a, int grid, bool pdl, cudaStream_t st) {
  constexpr int SUBV = sizeof(T) == 2 ? SUBV_BF16 : 4;
  auto kern = k_score<T, W, ST, CH, SUBV, FUSED>;
  constexpr size_t smem = score_smem_bytes<W, ST, CH, FUSED>();
  static_assert(smem <= 227 * 1024, "shared memory budget");
  PRORL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  return launch_maybe_pdl(kern, grid, W * 32, smem, pdl, st, a);
}

template <typename T, bool FUSED>
int run_score(const ScoreArgs& a, int n_sm, int64_t n_rows, int slab_rows, int* rows_used, bool pdl, cudaStream_t st) {
  const K2Config& k = kConfigs[active_config()];
  int grid = (int)std::min<int64_t>((int64_t)n_sm, (n_rows + k.warps - 1) / k.warps);
  if (FUSED && grid > slab_rows) grid = slab_rows;
  if (rows_used) *rows_used = grid;
  switch (active_config()) {
#ifdef PRORL_TUNING
    case 0: return run_score_cfg<T, 16, 2, 4096, 2, FUSED>(a, grid, pdl, st);
    case 1: return run_score_cfg<T, 16, 2, 4096, 4, FUSED>(a, grid, pdl, st);
    case 2: return run_score_cfg<T, 12, 3, 4096, 2, FUSED>(a, grid, pdl, st);
    case 3: return run_score_cfg<T, 8, 5, 4096, 2, FUSED>(a, grid, pdl, st);
    case 4: return run_score_cfg<T, 8, 3, 8192, 4, FUSED>(a, grid, pdl, st);
#endif
    default: return run_score_cfg<T, 16, 2, 4096, 8, FUSED>(a, grid, pdl, st);  // kDefaultConfig
  }
}

}  // namespace

const char* score_config_name() { return kConfigs[active_config()].name; }

int score_slab_rows(prorl_ctx* ctx) { return ctx->n_sm; }
int loss_slab_rows(prorl_ctx* ctx) { return 2 * ctx->n_sm; }

int launch_score(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab,
                 const int32_t* rows, const int32_t* targets, const float* old_lp, const double* adv,
                 const int32_t* row_seq, const int16_t* row_turn, const float* ref_lp, int64_t n_rows,
                 float inv_temp, const prorl_loss_cfg* cfg, float* logp, float* entropy, double* slab, int slab_rows,
                 bool accumulate, int* rows_used, cudaStream_t st, bool pdl) {
  if (rows_used) *rows_used = 0;
  if (dtype != PRORL_BF16 && dtype != PRORL_FP32) return fail(PRORL_E_SHAPE, "score: unknown logits dtype");
  if (vocab <= 0 || row_stride < vocab) return fail(PRORL_E_SHAPE, "score: need vocab > 0 and row_stride >= vocab");
  if (!(inv_temp > 0.f)) return fail(PRORL_E_MALFORMED_REQUEST, "score: inv_temperature must be > 0");
  const int esz = dtype == PRORL_BF16 ? 2 : 4;
  if (reinterpret_cast<uintptr_t>(logits) % esz) return fail(PRORL_E_SHAPE, "score: logits not element-aligned");
  if (n_rows <= 0) return PRORL_OK;
  if (cfg && (cfg->n_buckets < 1 || cfg->n_buckets > PRORL_TURN_BUCKETS))
    return fail(PRORL_E_SHAPE, "score: n_buckets out of [1, 64]");
  ScoreArgs a{};
  a.logits = static_cast<const uint8_t*>(logits);
  a.stride_bytes = row_stride * esz;
  a.vocab = vocab;
  a.rows = rows;
  a.targets = targets;
  a.n_rows = n_rows;
  a.c = inv_temp * kLog2e;
  a.inv_temp = inv_temp;
  a.old_lp = old_lp;
  a.adv = adv;
  a.row_seq = row_seq;
  a.row_turn = row_turn;
  a.ref_lp = ref_lp;
  a.logp = logp;
  a.entropy = entropy;
  a.slab = slab;
  a.accumulate = accumulate ? 1 : 0;
  static const float slack = [] {
    const char* e = tuning_env("PRORL_K2_SLACK");
    return e ? std::max(0.f, std::min(1.f, (float)std::atof(e))) : 1.f;  // measured +1.2 % at C2 (power-capped)
  }();
  a.raise_slack = slack;
  if (cfg) {
    a.lo_bound = 1.0 - (double)cfg->eps_lo;
    a.hi_bound = 1.0 + (double)cfg->eps_hi;
    a.n_buckets = cfg->n_buckets;
    a.kl_coef = cfg->kl_coef;
  }
  if (dtype == PRORL_BF16)
    return cfg ? run_score<__nv_bfloat16, true>(a, ctx->n_sm, n_rows, slab_rows, rows_used, pdl, st)
               : run_score<__nv_bfloat16, false>(a, ctx->n_sm, n_rows, slab_rows, rows_used, pdl, st);
  return cfg ? run_score<float, true>(a, ctx->n_sm, n_rows, slab_rows, rows_used, pdl, st)
             : run_score<float, false>(a, ctx->n_sm, n_rows, slab_rows, rows_used, pdl, st);
}

int launch_loss(prorl_ctx* ctx, const float* logp, const float* entropy, const float* old_lp, const double* adv,
                const int32_t* row_seq, const int16_t* row_turn, const float* ref_lp, int64_t n_rows,
                const prorl_loss_cfg* cfg, double* slab, int slab_rows, int* rows_used, cudaStream_t st) {
  *rows_used = 0;
  if (cfg->n_buckets < 1 || cfg->n_buckets > PRORL_TURN_BUCKETS)
    return fail(PRORL_E_SHAPE, "loss: n_buckets out of [1, 64]");
  if (n_rows <= 0) return PRORL_OK;
  const int64_t tiles = (n_rows + 31) / 32;
  int grid = (int)std::min<int64_t>((int64_t)slab_rows, (tiles + kLossWarps - 1) / kLossWarps);
  (void)ctx;
  k_loss<<<grid, kLossWarps * 32, 0, st>>>(logp, entropy, old_lp, adv, row_seq, row_turn, ref_lp, cfg->kl_coef,
                                           n_rows, 1.0 - (double)cfg->eps_lo, 1.0 + (double)cfg->eps_hi,
                                           cfg->n_buckets, slab);
  PRORL_CUDA(cudaGetLastError());
  *rows_used = grid;
  return PRORL_OK;
}

int launch_slab_reduce(const double* slab, int slab_rows, double* partials, cudaStream_t st) {
  if (slab_rows <= 0) return PRORL_OK;
  k_slab_reduce<<<1, 352, 0, st>>>(slab, slab_rows, partials);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

}  // namespace prorl
