// train.cu — K7: the training step over the logits in ONE HBM pass per row:
// logprob / entropy (K2), the DAPO loss epilogue (K4) and dL/dlogits (K5)
// from a single read of each logits row (SURVEY.md §8 f rank 1: "fused with
// the same online pass ... or a split-row two-phase scheme"; definitions
// App. B.2-B.5; no reference code).
//
// K2 then K5 move 2V + 4V bytes per bf16 row (the backward re-reads the row
// after the forward has produced its lse). K7 moves 4V: the row stays on chip
// between the two phases.
//
//   * A thread-block CLUSTER of C CTAs (one per SM) owns one row at a time; CTA
//     r of the cluster holds slice r of the row (a contiguous, 16-B aligned
//     1/C of the row: C = 2 at V = 151 936 bf16, 152 KB per CTA) in a ring of
//     4 KB shared-memory slots filled by 1-D TMA bulk copies (L2 evict_first)
//     from a dedicated producer warp. Rows go to clusters round robin.
//   * Phase 1 (statistics): 16 consumer warps take the slice's chunks round
//     robin and run K2's online base-2 logsumexp (warp-uniform running max,
//     top element kept out of the sums) as the chunks land; the warps' partials
//     merge in fixed order, and each CTA's partial goes to every CTA of the
//     cluster through distributed shared memory (st.async with mbarrier
//     complete_tx). Every CTA merges the C partials in rank order, so all of
//     them hold bit-identical lse / logp / loss terms for the row.
//   * Phase 2 (gradient): the same warps re-read their chunks from shared
//     memory, write grad = s * (1[v = y] - p_v) as 16-B streaming stores and
//     release each slot to the producer, which is already fetching the next
//     row into the freed slots (10 spare slots prefetch ahead while the
//     exchange is in flight).
//   * CTA rank 0 keeps the loss epilogue (fp64 partials + per-turn buckets,
//     fixed order) and writes one slab row per cluster.
//
// Requirements (else the host falls back to K2 + K5): 16-B aligned logits /
// grad rows (base and row stride), a slice of <= 40 slots per CTA with C <= 8.
// grad may alias logits (in place): a row's chunks are in shared memory before
// any gradient of that row is stored.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "rowmath.cuh"

namespace prorl {

namespace {

using namespace rowmath;

constexpr int kSub = 2048;                   // bytes per warp work unit
constexpr int kNV = kSub / 512;              // 16-B vectors per lane per unit
constexpr int kSplit = 4;                    // units per TMA piece
constexpr int kPiece = kSub * kSplit;        // 8 KB per bulk copy
constexpr int kRing = 26;                    // ring pieces: 208 KB
constexpr int kMaxSlicePieces = 11;          // two rows resident + >= 4 pieces of prefetch
constexpr int kMaxCluster = 8;
constexpr int kWarps = 16;              // consumer warps (+1 producer warp)
constexpr int kThreads = (kWarps + 1) * 32;

struct TrainArgs {
  const uint8_t* logits;
  int64_t stride_bytes;
  int64_t goff;  // grad - logits (bytes; same row stride)
  int32_t vocab;
  int32_t nvec;  // 16-B vectors in a row's interior (rows are 16-B aligned)
  int32_t tail;  // elements after the interior (< 16 / esz)
  const int32_t* rows;
  const int32_t* targets;
  const float* old_lp;
  const float* adv;
  const int32_t* row_seq;
  const int16_t* row_turn;
  const float* ref_lp;  // nullable
  float kl_coef;
  int64_t n_rows;
  float c;  // inv_temp * log2 e
  float inv_temp;
  float lo, hi;  // 1 - eps_lo, 1 + eps_hi
  float inv_n;   // 1 / N_global
  int n_buckets;
  float* logp;
  float* entropy;
  float* dlogp;
  double* slab;  // [n_clusters][PRORL_N_PARTIALS]
  int accumulate;
};

// ---- cluster / DSMEM helpers ------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t n_cluster_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t smem_addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
  return r;
}
// 16 bytes into a (possibly remote) CTA's shared memory, completing 16 bytes of
// transaction count on that CTA's mbarrier.
__device__ __forceinline__ void st_async_f4(uint32_t remote_addr, float4 v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   remote_addr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
// mbarrier wait that traps after ~4 s instead of hanging the GPU on a protocol bug
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (!mbar_try_wait(bar, parity)) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) __trap();
  }
}
__device__ __forceinline__ void consumers_sync() {  // named barrier 1: the consumer warps only
  asm volatile("bar.sync 1, %0;" ::"r"(kWarps * 32) : "memory");
}

// Merge two partials (Mc, Mx, S_rest, T_rest) of the online logsumexp: the one
// with the larger max keeps its top element excluded, the other's top becomes
// an ordinary term (ties: a wins). Empty partials have Mc = -inf.
__device__ __forceinline__ float4 merge_partial(float4 a, float4 b, float c) {
  if (b.x > a.x) {
    const float4 t = a;
    a = b;
    b = t;
  }
  if (b.x == -INFINITY) return a;
  const float rk = fmaf(b.y, c, -b.x), ek = ex2_approx(rk);
  const float Sk = b.z + ek, Tk = fmaf(rk, ek, b.w);
  const float sc = ex2_approx(b.x - a.x), dl = a.x - b.x;
  a.z = fmaf(sc, Sk, a.z);
  a.w = fmaf(sc, fmaf(-dl, Sk, Tk), a.w);
  return a;
}

// Generic-address element load with the clamp of Elem<T>::load (for the rare
// NaN re-run over shared memory).
template <typename T> __device__ __forceinline__ float load_clamped(const uint8_t* base, int64_t idx);
template <> __device__ __forceinline__ float load_clamped<__nv_bfloat16>(const uint8_t* base, int64_t idx) {
  uint32_t b = reinterpret_cast<const unsigned short*>(base)[idx];
  b = b > 0xf000u ? 0xf000u : b;
  return __uint_as_float(b << 16);
}
template <> __device__ __forceinline__ float load_clamped<float>(const uint8_t* base, int64_t idx) {
  return fmaxf(reinterpret_cast<const float*>(base)[idx], -1.5845632502852868e29f);
}

// One 32-wide step of the scalar online logsumexp (element x per lane).
__device__ __forceinline__ void scalar_step(float x, float c, Top& top, float2 (&S)[2], float2 (&Tt)[2], int lane) {
  if (__any_sync(kFull, x * c > top.Mc)) {
    const int L = raise_top(x, c, top, S, Tt, lane);
    if (lane == L) x = __uint_as_float(0xf0000000u);
  }
  const float d = fmaf(x, c, -top.Mc);
  const float e = ex2_approx(d);
  S[0].x += e;
  Tt[0].x = fmaf(d, e, Tt[0].x);
}

// Per-row scalars, loaded by lane 0 and broadcast to the warp.
struct RowIn {
  const uint8_t* rp;
  int32_t y;
  float xy, old, A, ref;
};

template <typename T>
__device__ __forceinline__ RowIn load_row(const TrainArgs& p, int64_t i, int lane) {
  RowIn r;
  const int64_t row = p.rows ? (int64_t)p.rows[i] : i;
  r.rp = p.logits + row * p.stride_bytes;
  r.y = p.targets[i];
  float xy = 0.f, old = 0.f, A = 0.f, ref = 0.f;
  if (lane == 0) {
    xy = Elem<T>::load(r.rp, r.y);
    old = p.old_lp[i];
    A = p.adv[p.row_seq[i]];
    if (p.ref_lp) ref = p.ref_lp[i];
  }
  // consumed at once: with grad aliasing the logits, the CTA that owns x_y may
  // overwrite it as soon as this CTA's partial for the row has been exchanged
  r.xy = __shfl_sync(kFull, xy, 0);
  r.old = __shfl_sync(kFull, old, 0);
  r.A = __shfl_sync(kFull, A, 0);
  r.ref = __shfl_sync(kFull, ref, 0);
  return r;
}

// Slice geometry of this CTA (identical for every row: rows are 16-B aligned).
struct Slice {
  int32_t v0, v1;   // 16-B vectors [v0, v1) of the row
  uint32_t bytes;
  int npc;          // TMA pieces
  int nsub;         // warp units
  bool tail;        // this CTA also owns the < 16-B row tail
};

// Phase 1 for one row: this warp's online logsumexp partial over its units.
template <typename T, int SUBV>
__device__ __forceinline__ float4 warp_stats(const TrainArgs& p, const Slice& sl, const uint8_t* ring, uint64_t* full,
                                             uint32_t pc0, const uint8_t* rp, int warp, int lane) {
  constexpr int ES = Elem<T>::kSize;
  constexpr int E = 16 / ES;
  const float c = p.c;
  const float2 c2 = make_float2(c, c);
  const uint4 fill = make_uint4(Elem<T>::kClampWord, Elem<T>::kClampWord, Elem<T>::kClampWord, Elem<T>::kClampWord);
  Top top{-INFINITY, 0.f};
  float2 S[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  float2 Tt[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  for (int u = warp; u < sl.nsub; u += kWarps) {
    const uint32_t pc = pc0 + (uint32_t)(u / kSplit);
    const int s = (int)(pc % kRing);
    mbar_wait_t(&full[s], (pc / kRing) & 1);
    const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)s * kPiece + (size_t)(u % kSplit) * kSub);
    const uint32_t nvv = min((uint32_t)kSub, sl.bytes - (uint32_t)u * kSub) >> 4;
    uint4 v[kNV];
    if (nvv == (uint32_t)(kSub / 16)) {
#pragma unroll
      for (int jj = 0; jj < kNV; ++jj) v[jj] = sv[lane + 32 * jj];
    } else {
#pragma unroll
      for (int jj = 0; jj < kNV; ++jj) {
        const uint32_t qv = lane + 32 * jj;
        v[jj] = qv < nvv ? sv[qv] : fill;
      }
    }
#pragma unroll
    for (int g0 = 0; g0 < kNV; g0 += SUBV) {
      uint4 w[SUBV];
#pragma unroll
      for (int jj = 0; jj < SUBV; ++jj) w[jj] = v[g0 + jj];
      const float lm = Elem<T>::template group_max<SUBV>(w);
      if (__any_sync(kFull, lm * c > top.Mc)) {
        const int L = raise_top(lm, c, top, S, Tt, lane);
        if (lane == L) Elem<T>::template mask_first<SUBV>(w, top.Mx);
      }
      Elem<T>::template accumulate<SUBV>(w, c2, make_float2(-top.Mc, -top.Mc), S, Tt);
    }
  }
  if (sl.tail && warp == 0) {
    float x = __uint_as_float(0xf0000000u);
    if (lane < p.tail) x = Elem<T>::load(rp, (int64_t)p.nvec * E + lane);
    scalar_step(x, c, top, S, Tt, lane);
  }
  float Sr = warp_sum((S[0].x + S[1].x) + (S[0].y + S[1].y));
  float Tr = warp_sum((Tt[0].x + Tt[1].x) + (Tt[0].y + Tt[1].y));
  if (!(Tr == Tr) || !(Sr == Sr)) {
    // -inf / NaN / overflowing logits: clamped scalar re-run over this warp's
    // units (still in shared memory) and the tail (rare)
    top = Top{-INFINITY, 0.f};
    S[0] = S[1] = Tt[0] = Tt[1] = make_float2(0.f, 0.f);
    for (int u = warp; u < sl.nsub; u += kWarps) {
      const uint32_t pc = pc0 + (uint32_t)(u / kSplit);
      const uint8_t* sb = ring + (size_t)(pc % kRing) * kPiece + (size_t)(u % kSplit) * kSub;
      const int ne = (int)(min((uint32_t)kSub, sl.bytes - (uint32_t)u * kSub) / ES);
      for (int b = 0; b < ne; b += 32)
        scalar_step(b + lane < ne ? load_clamped<T>(sb, b + lane) : __uint_as_float(0xf0000000u), c, top, S, Tt,
                    lane);
    }
    if (sl.tail && warp == 0)
      scalar_step(lane < p.tail ? load_clamped<T>(rp, (int64_t)p.nvec * E + lane) : __uint_as_float(0xf0000000u), c,
                  top, S, Tt, lane);
    Sr = warp_sum((S[0].x + S[1].x) + (S[0].y + S[1].y));
    Tr = warp_sum((Tt[0].x + Tt[1].x) + (Tt[0].y + Tt[1].y));
  }
  return make_float4(top.Mc, top.Mx, Sr, Tr);
}

// Warp 0: fixed-shape tree over the consumer warps' partials, then the CTA
// partial goes to slot [par][crank] of every CTA of the cluster (DSMEM).
__device__ __forceinline__ void cta_send(const float4* wp, float4* xch, uint64_t* xbar, int par, uint32_t crank,
                                         uint32_t csize, float c, int lane) {
  float4 P = lane < kWarps ? wp[lane] : make_float4(-INFINITY, 0.f, 0.f, 0.f);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    float4 Q;
    Q.x = __shfl_down_sync(kFull, P.x, o);
    Q.y = __shfl_down_sync(kFull, P.y, o);
    Q.z = __shfl_down_sync(kFull, P.z, o);
    Q.w = __shfl_down_sync(kFull, P.w, o);
    const float4 M = merge_partial(P, Q, c);
    if ((lane & (2 * o - 1)) == 0) P = M;
  }
  if (lane == 0) {
    const uint32_t dst = smem_u32(&xch[par * kMaxCluster + crank]);
    const uint32_t bar = smem_u32(&xbar[par]);
    for (uint32_t r = 0; r < csize; ++r) st_async_f4(mapa(dst, r), P, mapa(bar, r));
    mbar_arrive_expect_tx(&xbar[par], csize * 16u);
  }
}

// 16-B vector of gradients with the target element replaced by gy (bf16 / fp32).
template <typename T>
__device__ __forceinline__ uint4 patch_target(uint4 o, int e, float gy) {
  uint32_t w[4] = {o.x, o.y, o.z, o.w};
  if constexpr (sizeof(T) == 2) {
    const uint32_t h = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(gy));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (e == 2 * k) w[k] = (w[k] & 0xffff0000u) | h;
      if (e == 2 * k + 1) w[k] = (w[k] & 0xffffu) | (h << 16);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (e == k) w[k] = __float_as_uint(gy);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <typename T, int SUBV>
__global__ void __launch_bounds__(kThreads, 1) k_train(const TrainArgs p) {
  constexpr int ES = Elem<T>::kSize;
  constexpr int E = 16 / ES;  // elements per 16-B vector
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)kRing * kPiece);
  uint64_t* empty = full + kRing;
  uint64_t* xbar = empty + kRing;                            // [2] exchange barriers (row parity)
  float4* xch = reinterpret_cast<float4*>(xbar + 2);         // [2][kMaxCluster] CTA partials
  float4* wpart = xch + 2 * kMaxCluster;                     // [2][kWarps] warp partials
  double* gsum = reinterpret_cast<double*>(wpart + 2 * kWarps);  // [kNG] (rank 0)
  double* bk = gsum + kNG;                                   // [kBucketDoubles] (rank 0)

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t crank = cluster_ctarank(), csize = cluster_nctarank();
  const int64_t q0 = cluster_id_x(), nq = n_cluster_x();
  Slice sl;
  sl.v0 = (int32_t)((int64_t)p.nvec * crank / csize);
  sl.v1 = (int32_t)((int64_t)p.nvec * (crank + 1) / csize);
  sl.bytes = (uint32_t)(sl.v1 - sl.v0) * 16u;
  sl.npc = (int)((sl.bytes + kPiece - 1) / kPiece);
  sl.nsub = (int)((sl.bytes + kSub - 1) / kSub);
  sl.tail = (crank == csize - 1) && p.tail > 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSplit);
    }
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_mbar_init();
  }
  if (crank == 0) {
    for (int t = threadIdx.x; t < kNG + kBucketDoubles; t += blockDim.x) gsum[t] = 0.0;
  }
  cluster_sync_all();  // peers' barriers exist before any remote complete_tx

  if (warp == kWarps) {
    // ===== producer: one lane streams this CTA's slice of each row, piece by piece =====
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      uint32_t pc = 0;
      for (int64_t i = q0; i < p.n_rows; i += nq) {
        const int64_t r = p.rows ? (int64_t)p.rows[i] : i;
        const uint8_t* src = p.logits + r * p.stride_bytes + (size_t)sl.v0 * 16;
        for (int k = 0; k < sl.npc; ++k, ++pc) {
          const int s = (int)(pc % kRing);
          mbar_wait_t(&empty[s], ((pc / kRing) & 1) ^ 1);
          const uint32_t bytes = min((uint32_t)kPiece, sl.bytes - (uint32_t)k * kPiece);
          mbar_arrive_expect_tx(&full[s], bytes);
          tma_load_1d(ring + (size_t)s * kPiece, src + (size_t)k * kPiece, bytes, &full[s], pol);
        }
      }
    }
    __syncwarp();
  } else if (q0 < p.n_rows) {
    // ===== consumers: stats(j+1) runs while the exchange of row j is in flight =====
    const float c = p.c;
    const float2 c2 = make_float2(c, c);
    RowIn cur = load_row<T>(p, q0, lane);
    {
      const float4 wp = warp_stats<T, SUBV>(p, sl, ring, full, 0u, cur.rp, warp, lane);
      if (lane == 0) wpart[warp] = wp;
    }
    consumers_sync();
    if (warp == 0) cta_send(wpart, xch, xbar, 0, crank, csize, c, lane);
    uint32_t j = 0;
    for (int64_t i = q0; i < p.n_rows; i += nq, ++j) {
      const bool has_next = i + nq < p.n_rows;
      RowIn nxt = cur;
      if (has_next) {
        nxt = load_row<T>(p, i + nq, lane);
        const float4 wp = warp_stats<T, SUBV>(p, sl, ring, full, (j + 1) * (uint32_t)sl.npc, nxt.rp, warp, lane);
        if (lane == 0) wpart[((j + 1) & 1) * kWarps + warp] = wp;
      }

      // ---- row j: merge the cluster's partials (same order everywhere) ----
      const int par = (int)(j & 1);
      mbar_wait_t(&xbar[par], (j >> 1) & 1);
      float4 G = xch[par * kMaxCluster];
      for (uint32_t r = 1; r < csize; ++r) G = merge_partial(G, xch[par * kMaxCluster + r], c);
      const float rr = fmaf(G.y, c, -G.x);
      const float ir = ex2_approx(-rr);
      const float qq = G.z * ir;
      const float l1q = log1pf(qq);
      const float logp = (fmaf(cur.xy, c, -G.x) - rr) * kLn2 - l1q;
      const float ratio = expf(logp - cur.old);
      const float pg1 = ratio * cur.A, pg2 = fminf(fmaxf(ratio, p.lo), p.hi) * cur.A;
      float dl = (pg1 <= pg2) ? -cur.A * ratio * p.inv_n : 0.f;  // dL/dlogp
      if (p.ref_lp) dl = fmaf(p.kl_coef * p.inv_n, -expm1f(cur.ref - logp), dl);
      const float sg = -dl * p.inv_temp;  // grad_v = sg p_v (v != y), grad_y = sg expm1(logp) = -sg (1 - p_y)
      const float l2 = fmaf(cur.xy, c, -logp * kLog2e);
      const float gy = sg * expm1f(logp);
      if (crank == 0 && warp == 0 && lane == 0) {
        const float ent = l1q + kLn2 * (fmaf(rr, qq, -G.w * ir) / (1.f + qq));
        if (p.logp) p.logp[i] = logp;
        if (p.entropy) p.entropy[i] = ent;
        if (p.dlogp) p.dlogp[i] = dl;
        int k = p.row_turn[i];
        k = k < 0 ? 0 : (k >= p.n_buckets ? p.n_buckets - 1 : k);
        const RowLoss rl = row_loss(logp, cur.old, cur.A, p.lo, p.hi, p.ref_lp, i, p.kl_coef);
        gsum[0] += rl.loss;
        gsum[1] += 1.0;
        gsum[2] += ent;
        gsum[3] += logp;
        gsum[4] += rl.ratio;
        gsum[5] += rl.clip_lo;
        gsum[6] += rl.clip_hi;
        gsum[7] += (double)(cur.old - logp);
        gsum[10] += rl.kl;
        double* b = bk + k * PRORL_N_PER_TURN;
        b[0] += 1.0;
        b[1] += rl.loss;
        b[2] += ent;
        b[3] += logp;
        b[4] += rl.clip_lo + rl.clip_hi;
      }

      // ---- row j, phase 2: gradient from the units in shared memory ----
      const bool zero = (sg == 0.f);
      const float2 nl2 = make_float2(-l2, -l2), s2 = make_float2(sg, sg);
      const int32_t yv = cur.y / E - sl.v0;  // target vector relative to the slice
      const bool y_here = (cur.y < p.nvec * E) && yv >= 0 && cur.y / E < sl.v1;
      const int ye = cur.y % E;
      uint8_t* gp = const_cast<uint8_t*>(cur.rp) + p.goff;
      uint4* gdst = reinterpret_cast<uint4*>(gp + (size_t)sl.v0 * 16);
      const uint32_t pc0 = j * (uint32_t)sl.npc;
      for (int u = warp; u < sl.nsub; u += kWarps) {
        const uint32_t pc = pc0 + (uint32_t)(u / kSplit);
        const int s = (int)(pc % kRing);
        const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)s * kPiece + (size_t)(u % kSplit) * kSub);
        const uint32_t nvv = min((uint32_t)kSub, sl.bytes - (uint32_t)u * kSub) >> 4;
        const int32_t tq = y_here ? yv - u * (kSub / 16) : -1;  // target vector inside this unit
        uint4* dst = gdst + (size_t)u * (kSub / 16);
#pragma unroll
        for (int jj = 0; jj < kNV; ++jj) {
          const uint32_t qv = lane + 32 * jj;
          if (qv < nvv) {
            uint4 o = make_uint4(0, 0, 0, 0);
            if (!zero) {
              o = GElem<T>::vec(sv[qv], c2, nl2, s2);
              if ((int32_t)qv == tq) o = patch_target<T>(o, ye, gy);
            }
            __stcs(dst + qv, o);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_cnt(&empty[s], u == sl.nsub - 1 ? (uint32_t)(kSplit - u % kSplit) : 1u);
      }
      if (sl.tail && warp == 0 && lane < p.tail) {
        const int64_t idx = (int64_t)p.nvec * E + lane;
        const float x = Elem<T>::load(cur.rp, idx);
        float g = 0.f;
        if (!zero) g = idx == cur.y ? gy : sg * ex2_approx(fmaf(x, c, -l2));
        if constexpr (ES == 2) reinterpret_cast<__nv_bfloat16*>(gp)[idx] = __float2bfloat16_rn(g);
        else reinterpret_cast<float*>(gp)[idx] = g;
      }
      if (!has_next) break;
      consumers_sync();  // every warp's stats(j+1) partial is in wpart[(j+1)&1]
      if (warp == 0) cta_send(wpart + ((j + 1) & 1) * kWarps, xch, xbar, (int)((j + 1) & 1), crank, csize, c, lane);
      cur = nxt;
    }
    // ---- slab row of this cluster (rank 0) ----
    if (crank == 0 && warp == 0) {
      __syncwarp();
      for (int t = lane; t < PRORL_N_PARTIALS; t += 32) {
        double v = 0.0;
        if (t < kNG) v = gsum[t];
        else if (t >= PRORL_N_GLOBAL) v = bk[t - PRORL_N_GLOBAL];
        double* d = p.slab + (size_t)q0 * PRORL_N_PARTIALS + t;
        *d = p.accumulate ? *d + v : v;
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

constexpr size_t train_smem_bytes() {
  return (size_t)kRing * kPiece + (size_t)(2 * kRing + 2) * 8 + (size_t)(2 * kMaxCluster + 2 * kWarps) * 16 +
         (size_t)(kNG + kBucketDoubles) * 8;
}
static_assert(train_smem_bytes() <= 227 * 1024, "shared memory budget");
static_assert(((size_t)kRing * kPiece + (size_t)(2 * kRing + 2) * 8) % 16 == 0, "float4 exchange alignment");

// Co-resident clusters of `cs` CTAs of k_train on the current device (cached).
int max_active_clusters(int cs) {
  static int cache[64][kMaxCluster + 1] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  int& v = cache[dev][cs];
  if (v == 0) {
    auto kern = k_train<__nv_bfloat16, 4>;  // both instantiations use the same resources
    constexpr size_t smem = train_smem_bytes();
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    int n_sm = 0;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.gridDim = dim3((unsigned)(cs * std::max(1, n_sm / cs)));
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = -1;  // not launchable: remembered as unusable
    }
    v = n;
  }
  return v < 0 ? 0 : v;
}

template <typename T>
int run_train(const TrainArgs& a, int csize, int n_sm, int* clusters_used, cudaStream_t st) {
  auto kern = k_train<T, 4>;
  constexpr size_t smem = train_smem_bytes();
  PRORL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (csize > 8) PRORL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)csize;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.gridDim = dim3((unsigned)(csize * (n_sm / csize)));
  const int max_clusters = max_active_clusters(csize);
  if (max_clusters < 1) return fail(PRORL_E_CUDA, "score_grad: no cluster of this size fits on the device");
  const int64_t nq = std::min<int64_t>((int64_t)max_clusters, a.n_rows);
  cfg.gridDim = dim3((unsigned)(nq * csize));
  *clusters_used = (int)nq;
  PRORL_CUDA(cudaLaunchKernelEx(&cfg, kern, a));
  return PRORL_OK;
}

}  // namespace

// Cluster size K7 uses for this row layout, 0 if K7 cannot run it (the caller
// then uses K2 + K5). Among the cluster sizes whose slice leaves room to
// prefetch a whole next row (<= kMaxSlicePieces pieces), take the one that
// keeps the most SMs busy (C x co-resident clusters; ties: the smaller C).
int train_cluster_size(int dtype, int32_t vocab, int64_t row_stride, const void* logits, const void* grad) {
  const int esz = dtype == PRORL_BF16 ? 2 : 4;
  if (reinterpret_cast<uintptr_t>(logits) % 16 || reinterpret_cast<uintptr_t>(grad) % 16 ||
      (row_stride * esz) % 16)
    return 0;
  const int64_t nvec = (int64_t)vocab * esz / 16;
  if (const char* e = std::getenv("PRORL_K7_CLUSTER")) {  // tuning override
    const int cs = std::atoi(e);
    const int64_t slice = (nvec + cs - 1) / std::max(cs, 1) * 16;
    if (cs >= 1 && cs <= kMaxCluster && (slice + kPiece - 1) / kPiece <= kMaxSlicePieces && max_active_clusters(cs) > 0)
      return cs;
  }
  int best = 0, best_sms = 0;
  for (int cs = 1; cs <= kMaxCluster; ++cs) {
    const int64_t slice = (nvec + cs - 1) / cs * 16;
    if ((slice + kPiece - 1) / kPiece > kMaxSlicePieces) continue;
    const int sms = cs * max_active_clusters(cs);
    if (sms > best_sms) {
      best = cs;
      best_sms = sms;
    }
  }
  return best;
}

int train_slab_rows(prorl_ctx* ctx) { return ctx->n_sm; }

int train_max_clusters(int cs) { return cs >= 1 && cs <= kMaxCluster ? max_active_clusters(cs) : 0; }

int launch_train(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab, const int32_t* rows,
                 const int32_t* targets, const float* old_lp, const float* adv, const int32_t* row_seq,
                 const int16_t* row_turn, const float* ref_lp, int64_t n_rows, float inv_temp,
                 const prorl_loss_cfg* cfg, double n_global, float* logp, float* entropy, float* dlogp, void* grad,
                 double* slab, bool accumulate, int* rows_used, cudaStream_t st) {
  *rows_used = 0;
  const int csize = train_cluster_size(dtype, vocab, row_stride, logits, grad);
  if (csize == 0) return fail(PRORL_E_SHAPE, "score_grad: layout not supported by the one-pass kernel");
  if (n_rows <= 0) return PRORL_OK;
  const int esz = dtype == PRORL_BF16 ? 2 : 4;
  TrainArgs a{};
  a.logits = static_cast<const uint8_t*>(logits);
  a.stride_bytes = row_stride * esz;
  a.goff = static_cast<const uint8_t*>(grad) - static_cast<const uint8_t*>(logits);
  a.vocab = vocab;
  a.nvec = (int32_t)((int64_t)vocab * esz / 16);
  a.tail = vocab - a.nvec * (16 / esz);
  a.rows = rows;
  a.targets = targets;
  a.old_lp = old_lp;
  a.adv = adv;
  a.row_seq = row_seq;
  a.row_turn = row_turn;
  a.ref_lp = ref_lp;
  a.kl_coef = cfg->kl_coef;
  a.n_rows = n_rows;
  a.c = inv_temp * kLog2e;
  a.inv_temp = inv_temp;
  a.lo = 1.0f - cfg->eps_lo;
  a.hi = 1.0f + cfg->eps_hi;
  a.inv_n = (float)(1.0 / n_global);
  a.n_buckets = cfg->n_buckets;
  a.logp = logp;
  a.entropy = entropy;
  a.dlogp = dlogp;
  a.slab = slab;
  a.accumulate = accumulate ? 1 : 0;
  return dtype == PRORL_BF16 ? run_train<__nv_bfloat16>(a, csize, ctx->n_sm, rows_used, st)
                             : run_train<float>(a, csize, ctx->n_sm, rows_used, st);
}

}  // namespace prorl
