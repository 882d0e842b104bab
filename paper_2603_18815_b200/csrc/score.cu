// score.cu — K2 (vocab-streaming logprob + entropy) with an optional fused K4
// epilogue (DAPO clipped surrogate + per-turn metrics), the standalone K4 and
// the deterministic slab reduction.
//
// No reference code exists for this arithmetic; definitions
// are SURVEY.md App. B.2 (logprob/entropy), B.4 (loss), B.5/B.6 (metrics).
//
// K2 design (HBM-bound: 2V bytes per bf16 row, one pass):
//   * one warp owns one row at a time (rows strided over a persistent grid of
//     one CTA per SM), so a row never needs a cross-warp reduction;
//   * every warp has a private ring of STAGES x CHUNK bytes of shared memory
//     fed by 1-D TMA bulk copies (cp.async.bulk ... mbarrier::complete_tx,
//     L2 evict_first) issued by lane 0, running up to STAGES chunks ahead and
//     across row boundaries; consumers read 16 B per lane per LDS.128;
//   * online base-2 logsumexp per lane: running max Mc (of x*c, c =
//     inv_temp*log2e), S = sum 2^(x*c-Mc), T = sum (x*c-Mc) 2^(x*c-Mc), with a
//     per-group max (packed bf16x2 HMNMX2) so a rescale happens at most once
//     per 64 elements and rarely after the first few chunks;
//   * row end: warp butterfly merge of (Mc, S, T);
//       logp = (x_y*c - Mc) ln2 - ln S,   H = ln S - ln2 T/S
//     (the max-relative form keeps H accurate when one logit dominates);
//   * unaligned row heads/tails (V*esz not a multiple of 16) are read by
//     lanes directly, the 16-B aligned interior goes through TMA.
#include "common.cuh"

namespace prorl {

namespace {

constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLog2e = 1.44269504088896340736f;

template <typename T> struct Elem;
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kSize = 2;
  static constexpr uint32_t kNegInfWord = 0xff80ff80u;
  __device__ static float load(const uint8_t* row, int64_t idx) {
    uint16_t b = __ldg(reinterpret_cast<const unsigned short*>(row) + idx);
    return __uint_as_float(((uint32_t)b) << 16);
  }
};
template <> struct Elem<float> {
  static constexpr int kSize = 4;
  static constexpr uint32_t kNegInfWord = 0xff800000u;
  __device__ static float load(const uint8_t* row, int64_t idx) {
    return __ldg(reinterpret_cast<const float*>(row) + idx);
  }
};

struct Acc {
  float m;     // running max of x*c (base-2 units)
  float s[4];  // sum 2^(x*c - m), four independent chains
  float t[4];  // sum (x*c - m) 2^(x*c - m)
};

__device__ __forceinline__ void acc_init(Acc& a) {
  a.m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 4; ++k) a.s[k] = a.t[k] = 0.f;
}

// Raise the running max to nm (> a.m) and rescale the sums:
//   S' = 2^(m-nm) S,  T' = 2^(m-nm) (T - (nm-m) S).
__device__ __forceinline__ void acc_rescale(Acc& a, float nm) {
  if (a.m != -INFINITY) {
    const float sc = ex2_approx(a.m - nm);
    const float dl = nm - a.m;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a.t[k] = sc * fmaf(-dl, a.s[k], a.t[k]);
      a.s[k] *= sc;
    }
  }
  a.m = nm;
}

// One element. d is clamped so -inf logits (and masked lanes) give e = 0 and
// d*e = 0 instead of NaN; 2^-200 flushes to zero anyway.
__device__ __forceinline__ void acc_elem(Acc& a, int k, float x, float c) {
  const float d = fmaxf(fmaf(x, c, -a.m), -200.f);
  const float e = ex2_approx(d);
  a.s[k] += e;
  a.t[k] = fmaf(d, e, a.t[k]);
}

template <typename T, int NV>
__device__ __forceinline__ void acc_vectors(Acc& a, const uint4 (&v)[NV], float c);

template <>
__device__ __forceinline__ void acc_vectors<__nv_bfloat16, 8>(Acc& a, const uint4 (&v)[8], float c) {
  __nv_bfloat162 mm = *reinterpret_cast<const __nv_bfloat162*>(&v[0].x);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) mm = __hmax2(mm, *reinterpret_cast<const __nv_bfloat162*>(&w[q]));
  }
  const float lmc = fmaxf(__low2float(mm), __high2float(mm)) * c;
  if (lmc > a.m) acc_rescale(a, lmc);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t w[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      acc_elem(a, (2 * q) & 3, __uint_as_float(w[q] << 16), c);
      acc_elem(a, (2 * q + 1) & 3, __uint_as_float(w[q] & 0xffff0000u), c);
    }
  }
}

template <>
__device__ __forceinline__ void acc_vectors<float, 8>(Acc& a, const uint4 (&v)[8], float c) {
  float lm = __uint_as_float(v[0].x);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    lm = fmaxf(lm, fmaxf(fmaxf(__uint_as_float(v[j].x), __uint_as_float(v[j].y)),
                         fmaxf(__uint_as_float(v[j].z), __uint_as_float(v[j].w))));
  }
  const float lmc = lm * c;
  if (lmc > a.m) acc_rescale(a, lmc);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    acc_elem(a, 0, __uint_as_float(v[j].x), c);
    acc_elem(a, 1, __uint_as_float(v[j].y), c);
    acc_elem(a, 2, __uint_as_float(v[j].z), c);
    acc_elem(a, 3, __uint_as_float(v[j].w), c);
  }
}

struct ScoreArgs {
  const uint8_t* logits;
  int64_t stride_bytes;
  int32_t vocab;
  const int32_t* rows;
  const int32_t* targets;
  int64_t n_rows;
  float c;  // inv_temp * log2(e)
  // fused loss
  const float* old_lp;
  const float* adv;
  const int32_t* row_seq;
  const int16_t* row_turn;
  float lo_bound, hi_bound;  // 1 - eps_lo, 1 + eps_hi
  int n_buckets;
  float* logp;
  float* entropy;
  double* slab;
  int accumulate;
};

// Per-row loss terms (App. B.4/B.5), fp32 math; returned through refs.
struct RowLoss {
  float loss, ratio, clip_lo, clip_hi;
};
__device__ __forceinline__ RowLoss row_loss(float logp, float old, float A, float lo, float hi) {
  RowLoss r;
  r.ratio = expf(logp - old);
  const float pg1 = r.ratio * A;
  const float pg2 = fminf(fmaxf(r.ratio, lo), hi) * A;
  r.loss = -fminf(pg1, pg2);
  r.clip_lo = (r.ratio < lo && A < 0.f) ? 1.f : 0.f;
  r.clip_hi = (r.ratio > hi && A > 0.f) ? 1.f : 0.f;
  return r;
}

constexpr int kNG = 8;  // per-row global sums kept by the loss epilogue
constexpr int kBucketDoubles = PRORL_TURN_BUCKETS * PRORL_N_PER_TURN;

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

template <typename T, int WARPS, int STAGES, int CHUNK, bool FUSED>
__global__ void __launch_bounds__(WARPS * 32, 1) k_score(const ScoreArgs p) {
  static_assert(CHUNK % 512 == 0, "CHUNK must be a multiple of 32 lanes x 16 B");
  constexpr int NV = CHUNK / 512;
  constexpr int ES = Elem<T>::kSize;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* ring = smem + (size_t)warp * STAGES * CHUNK;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * STAGES * CHUNK) + warp * STAGES;
  double* g_w = reinterpret_cast<double*>(smem + (size_t)WARPS * STAGES * CHUNK + WARPS * STAGES * 8);
  double* bk_w = g_w + WARPS * kNG;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  double g[kNG];
  if constexpr (FUSED) {
#pragma unroll
    for (int k = 0; k < kNG; ++k) g[k] = 0.0;
    for (int i = lane; i < kBucketDoubles; i += 32) bk_w[warp * kBucketDoubles + i] = 0.0;
  }
  __syncwarp();

  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  const uint64_t policy = l2_policy_evict_first();

  auto row_ptr = [&](int64_t i) -> const uint8_t* {
    const int64_t r = p.rows ? (int64_t)p.rows[i] : i;
    return p.logits + r * p.stride_bytes;
  };
  // interior [a, b) of a row: 16-B aligned, multiple of 16 bytes.
  auto interior = [&](const uint8_t* rp, uintptr_t& a, uintptr_t& b) {
    const uintptr_t st = reinterpret_cast<uintptr_t>(rp);
    const uintptr_t en = st + (uintptr_t)p.vocab * ES;
    a = (st + 15) & ~(uintptr_t)15;
    if (a > en) a = en;
    b = en & ~(uintptr_t)15;
    if (b < a) b = a;
  };

  // ---- producer state (meaningful in lane 0 only) ----
  int64_t p_row = gw;
  int64_t p_chunk = 0, p_nchunks = 0;
  uintptr_t p_a = 0, p_b = 0;
  uint32_t produced = 0;
  if (p_row < p.n_rows) {
    interior(row_ptr(p_row), p_a, p_b);
    p_nchunks = (int64_t)((p_b - p_a + CHUNK - 1) / CHUNK);
  }
  auto produce = [&]() {
    while (p_row < p.n_rows && p_chunk >= p_nchunks) {
      p_row += nw;
      p_chunk = 0;
      p_nchunks = 0;
      if (p_row < p.n_rows) {
        interior(row_ptr(p_row), p_a, p_b);
        p_nchunks = (int64_t)((p_b - p_a + CHUNK - 1) / CHUNK);
      }
    }
    if (p_row >= p.n_rows) return;
    const uintptr_t src = p_a + (uintptr_t)p_chunk * CHUNK;
    const uint32_t bytes = (uint32_t)min((uintptr_t)CHUNK, p_b - src);
    const int s = produced % STAGES;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[s], bytes);
    tma_load_1d(ring + (size_t)s * CHUNK, reinterpret_cast<const void*>(src), bytes, &bars[s], policy);
    ++produced;
    ++p_chunk;
  };
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) produce();
  }

  uint32_t consumed = 0;
  const float c = p.c;
  for (int64_t i = gw; i < p.n_rows; i += nw) {
    const uint8_t* rp = row_ptr(i);
    uintptr_t a, b;
    interior(rp, a, b);
    const int64_t nchunks = (int64_t)((b - a + CHUNK - 1) / CHUNK);
    const int head = (int)((a - reinterpret_cast<uintptr_t>(rp)) / ES);
    const int tail = (int)((reinterpret_cast<uintptr_t>(rp) + (uintptr_t)p.vocab * ES - b) / ES);
    const int32_t tgt = p.targets[i];
    float xy = 0.f;
    if (lane == 0) xy = Elem<T>::load(rp, tgt);

    Acc acc;
    acc_init(acc);
    {  // unaligned head / tail elements, one per lane (<= 14 of them)
      float x = -INFINITY;
      if (lane < head) x = Elem<T>::load(rp, lane);
      else if (lane < head + tail) x = Elem<T>::load(rp, (int64_t)((b - reinterpret_cast<uintptr_t>(rp)) / ES) + (lane - head));
      const float xc = x * c;
      if (xc > acc.m) acc_rescale(acc, xc);
      acc_elem(acc, 0, x, c);
    }

    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int s = consumed % STAGES;
      const uint32_t parity = (consumed / STAGES) & 1;
      const uint32_t nvec = (uint32_t)(min((uintptr_t)CHUNK, b - (a + (uintptr_t)ch * CHUNK)) >> 4);
      mbar_wait(&bars[s], parity);
      const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)s * CHUNK);
      uint4 v[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const uint32_t q = lane + 32 * j;
        if (q < nvec) v[j] = sv[q];
        else v[j] = make_uint4(Elem<T>::kNegInfWord, Elem<T>::kNegInfWord, Elem<T>::kNegInfWord, Elem<T>::kNegInfWord);
      }
      __syncwarp();
      ++consumed;
      if (lane == 0) produce();
      acc_vectors<T, NV>(acc, v, c);
    }

    // ---- row end: merge lanes ----
    float S = (acc.s[0] + acc.s[1]) + (acc.s[2] + acc.s[3]);
    float Tt = (acc.t[0] + acc.t[1]) + (acc.t[2] + acc.t[3]);
    const float Mw = warp_max(acc.m);
    if (S > 0.f) {
      const float sc = ex2_approx(acc.m - Mw);
      Tt = sc * fmaf(-(Mw - acc.m), S, Tt);
      S = sc * S;
    } else {
      S = 0.f;
      Tt = 0.f;
    }
    S = warp_sum(S);
    Tt = warp_sum(Tt);
    if (lane == 0) {
      const float lnS = logf(S);
      const float logp = fmaf(xy, c, -Mw) * kLn2 - lnS;
      const float ent = lnS - kLn2 * (Tt / S);
      if (p.logp) p.logp[i] = logp;
      if (p.entropy) p.entropy[i] = ent;
      if constexpr (FUSED) {
        const float old = p.old_lp[i];
        const float A = p.adv[p.row_seq[i]];
        int k = p.row_turn[i];
        k = k < 0 ? 0 : (k >= p.n_buckets ? p.n_buckets - 1 : k);
        const RowLoss r = row_loss(logp, old, A, p.lo_bound, p.hi_bound);
        g[0] += r.loss;
        g[1] += 1.0;
        g[2] += ent;
        g[3] += logp;
        g[4] += r.ratio;
        g[5] += r.clip_lo;
        g[6] += r.clip_hi;
        g[7] += (double)(old - logp);
        double* bk = bk_w + warp * kBucketDoubles + k * PRORL_N_PER_TURN;
        bk[0] += 1.0;
        bk[1] += r.loss;
        bk[2] += ent;
        bk[3] += logp;
        bk[4] += r.clip_lo + r.clip_hi;
      }
    }
  }

  if constexpr (FUSED) {
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < kNG; ++k) g_w[warp * kNG + k] = g[k];
    }
    __syncthreads();
    merge_block_partials<WARPS>(g_w, bk_w, p.slab, p.accumulate);
  }
}

// ---- standalone K4 ------------------------------------------------------------
constexpr int kLossWarps = 8;

__global__ void __launch_bounds__(kLossWarps * 32)
    k_loss(const float* __restrict__ logp, const float* __restrict__ entropy, const float* __restrict__ old_lp,
           const float* __restrict__ adv, const int32_t* __restrict__ row_seq, const int16_t* __restrict__ row_turn,
           int64_t n_rows, float lo, float hi, int n_buckets, double* slab) {
  __shared__ double g_w[kLossWarps * kNG];
  __shared__ double bk_w[kLossWarps * kBucketDoubles];
  __shared__ int s_key[kLossWarps][32];
  __shared__ float s_val[kLossWarps][32][PRORL_N_PER_TURN];
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
      const float lp = logp[i], ent = entropy[i], old = old_lp[i];
      const float A = adv[row_seq[i]];
      int k = row_turn[i];
      key = k < 0 ? 0 : (k >= n_buckets ? n_buckets - 1 : k);
      const RowLoss r = row_loss(lp, old, A, lo, hi);
      g[0] += r.loss;
      g[1] += 1.0;
      g[2] += ent;
      g[3] += lp;
      g[4] += r.ratio;
      g[5] += r.clip_lo;
      g[6] += r.clip_hi;
      g[7] += (double)(old - lp);
      s_val[warp][lane][0] = 1.f;
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
        if (kk >= 0) bk_w[warp * kBucketDoubles + kk * PRORL_N_PER_TURN + lane] += (double)s_val[warp][src][lane];
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

// ---- launch configuration ---------------------------------------------------------
constexpr int kWarps = 8;
constexpr int kStages = 5;
constexpr int kChunk = 4096;

template <typename T, bool FUSED>
size_t score_smem() {
  return (size_t)kWarps * kStages * kChunk + (size_t)kWarps * kStages * 8 +
         (FUSED ? (size_t)kWarps * (kNG + kBucketDoubles) * sizeof(double) : 0);
}

template <typename T, bool FUSED>
int run_score(const ScoreArgs& a, int grid, cudaStream_t st) {
  auto kern = k_score<T, kWarps, kStages, kChunk, FUSED>;
  const size_t smem = score_smem<T, FUSED>();
  PRORL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, kWarps * 32, smem, st>>>(a);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

}  // namespace

int score_slab_rows(prorl_ctx* ctx) { return ctx->n_sm; }
int loss_slab_rows(prorl_ctx* ctx) { return 2 * ctx->n_sm; }

int launch_score(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab,
                 const int32_t* rows, const int32_t* targets, const float* old_lp, const float* adv,
                 const int32_t* row_seq, const int16_t* row_turn, int64_t n_rows, float inv_temp,
                 const prorl_loss_cfg* cfg, float* logp, float* entropy, double* slab, int slab_rows,
                 bool accumulate, int* rows_used, cudaStream_t st) {
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
  a.old_lp = old_lp;
  a.adv = adv;
  a.row_seq = row_seq;
  a.row_turn = row_turn;
  a.logp = logp;
  a.entropy = entropy;
  a.slab = slab;
  a.accumulate = accumulate ? 1 : 0;
  if (cfg) {
    a.lo_bound = 1.0f - cfg->eps_lo;
    a.hi_bound = 1.0f + cfg->eps_hi;
    a.n_buckets = cfg->n_buckets;
  }
  int grid = (int)std::min<int64_t>((int64_t)ctx->n_sm, (n_rows + kWarps - 1) / kWarps);
  if (cfg && grid > slab_rows) grid = slab_rows;
  if (rows_used) *rows_used = grid;
  if (dtype == PRORL_BF16) {
    return cfg ? run_score<__nv_bfloat16, true>(a, grid, st) : run_score<__nv_bfloat16, false>(a, grid, st);
  }
  return cfg ? run_score<float, true>(a, grid, st) : run_score<float, false>(a, grid, st);
}

int launch_loss(prorl_ctx* ctx, const float* logp, const float* entropy, const float* old_lp, const float* adv,
                const int32_t* row_seq, const int16_t* row_turn, int64_t n_rows, const prorl_loss_cfg* cfg,
                double* slab, int slab_rows, int* rows_used, cudaStream_t st) {
  *rows_used = 0;
  if (cfg->n_buckets < 1 || cfg->n_buckets > PRORL_TURN_BUCKETS)
    return fail(PRORL_E_SHAPE, "loss: n_buckets out of [1, 64]");
  if (n_rows <= 0) return PRORL_OK;
  const int64_t tiles = (n_rows + 31) / 32;
  int grid = (int)std::min<int64_t>((int64_t)slab_rows, (tiles + kLossWarps - 1) / kLossWarps);
  (void)ctx;
  k_loss<<<grid, kLossWarps * 32, 0, st>>>(logp, entropy, old_lp, adv, row_seq, row_turn, n_rows,
                                           1.0f - cfg->eps_lo, 1.0f + cfg->eps_hi, cfg->n_buckets, slab);
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
