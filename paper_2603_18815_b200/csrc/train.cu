// train.cu — K7: the training step over the logits with ONE HBM read and ONE
// HBM write per row: logprob / entropy (K2), the DAPO loss epilogue (K4) and
// dL/dlogits (K5) in one kernel (SURVEY.md §8 f rank 1: "fused with the same
// online pass ... or a split-row two-phase scheme"; definitions App. B.2-B.5;
// no reference code).
//
// K2 then K5 move 2V + 4V bytes of HBM per bf16 row: the backward re-reads the
// row from HBM after the forward has produced its lse. K7 moves 4V.
//
//   * One CTA per SM, persistent over rows. The CTA's consumer warps form G row
//     groups (G = 4 for rows <= 80 KB, 2 for <= 160 KB, else 1); a group owns
//     ONE row at a time, so the rows in flight (148 x G x 2V bytes: 45 MB at
//     V = 151 936 bf16) fit in the 126 MB L2 between the two passes over each
//     row, and one group's barrier and pipeline bubbles overlap the others'.
//   * Pass A (statistics): one producer warp (lane g feeds group g) streams
//     each group's row from HBM into the group's shared-memory ring of 16 KB
//     pieces (1-D TMA bulk copies; L2 evict_last on the pieces pass B
//     re-reads). Piece P goes to a fixed set of kSplit warps, one 2 or 4 KB
//     unit each (config), so every warp sees every round of its ring slots in
//     order (a parity wait never aliases a round two phases back; pieces can
//     complete out of order). Warps run K2's online base-2 logsumexp with
//     the row arithmetic of rowmath.cuh (integer running reference, fp32
//     lane sums folded into fp64 every 128 elements per lane, fp64 warp
//     sums); the warp partials meet in shared memory after one named barrier.
//     Each warp merges them with the same fixed fp32 tree (bit-identical lse
//     for the gradient); warp 0 stores the fp64 warp partials and the target
//     logit of the row for the row end.
//   * Pass B (gradient): the last ring-full of pass-A pieces is still in
//     shared memory and is consumed first, straight from there (pass A holds
//     those slots); the rest of the row is streamed again — from L2
//     (evict_first) — into the slots they free. Warps write
//     grad = s (1[v = y] - p_v) as 16-B streaming stores. The producer runs
//     ahead across passes and rows. (Rows of <= 192 KB never leave shared
//     memory between the passes.) The clip decision of s is taken in fp32
//     except within a few ulp of the clip edge, where the fp64 merge decides
//     (unclipped_f64), so gradient and loss agree on every row.
//   * Row end (k_train_rows, one lane per row, launched after K7): merges the
//     row's fp64 warp partials exactly, derives lse / logp / entropy and the
//     DAPO / KL terms in fp64 (row_stats / row_loss, as K2's epilogue) and
//     accumulates them in fixed order into one slab row per CTA
//     (deterministic). Keeping the fp64 work out of K7 keeps K7's registers
//     and issue slots on the stream (an in-kernel fp64 epilogue cost 4-18 %).
//
// Any row layout K2/K5 accept works: the 16-B aligned interior of each row goes
// through TMA, the < 16-B head/tail elements are handled by warp 0 directly;
// grad must have the logits' 16-B phase and may alias them (in place): pass B
// loads each piece before any gradient of that piece is stored.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "rowmath.cuh"

namespace prorl {

namespace {

using namespace rowmath;

constexpr int kRingBytes = 196608;           // shared-memory ring per CTA: 192 KB
constexpr int kProducerPiece = 16384;        // bytes per bulk copy (ring slot) with producer warps
constexpr int kMaxWarps = 32;                // consumer warps of any launch configuration
constexpr int kMaxGroups = 4;                // row groups of any launch configuration

struct TrainArgs {
  const uint8_t* logits;
  int64_t stride_bytes;
  int64_t goff;  // grad - logits (bytes; same row stride and 16-B phase)
  int32_t vocab;
  const int32_t* rows;
  const int32_t* targets;
  const float* old_lp;
  const double* adv;
  const int32_t* row_seq;
  const int16_t* row_turn;
  const float* ref_lp;  // nullable
  float kl_coef;
  int64_t n_rows;
  float c;  // fl(inv_temp * log2 e)
  float inv_temp;
  float lo, hi;      // 1 - eps_lo, 1 + eps_hi (fp32: the gradient's branch)
  double lo_d, hi_d;  // the same in fp64 (the loss epilogue, as the oracle)
  float inv_n;   // 1 / N_global
  int n_buckets;
  float* logp;
  float* entropy;
  float* dlogp;
  void* parts;   // [n_rows][kWarps] WPart: each row's fp64 warp partials, for k_train_rows
  float* xy;     // [n_rows] the rows' target logits (K7 may overwrite them in place)
};

__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}

// mbarrier wait that traps after ~4 s instead of hanging the GPU on a protocol
// bug (the timer is read only every 256 polls, so waiting costs few issue slots).
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t k = 1;; ++k) {
    if (mbar_try_wait(bar, parity)) return;
    if ((k & 255u) == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 4000000000ull) {
#ifdef PRORL_K7_DEBUG
        printf("k_train stuck: block %d warp %d bar %p parity %u\n", blockIdx.x, (int)(threadIdx.x >> 5), bar, parity);
#endif
        __trap();
      }
    }
  }
}

// named barrier `id` over `n` threads (the producer warps never join one)
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// One warp's partial of a row's online logsumexp: integer reference Mc, the
// excluded top logit Mx, and the fp64 sums of every other term relative to Mc.
struct WPart {
  float Mc, Mx;
  double S, T;
};

// Merge two partials: the one with the larger reference keeps its top element
// excluded, the other's top becomes an ordinary term (an ex2.approx term like
// every other, so the row-end MUFU correction applies to it), and its sums are
// rescaled by the exact 2^(Mc_b - Mc_a) (ties: a wins). fp64 throughout: 16
// warp partials merged in fp32 would put ~1e-7 of rounding noise on the row's
// sum. Empty partials have Mc = -inf.
__device__ __forceinline__ WPart merge_partial(WPart a, WPart b, float c) {
  if (b.Mc > a.Mc) {
    const WPart t = a;
    a = b;
    b = t;
  }
  if (b.Mc == -INFINITY) return a;
  const float rk = fmaf(b.Mx, c, -b.Mc), ek = ex2_approx(rk);
  const double Sk = b.S + (double)ek, Tk = fma((double)rk, (double)ek, b.T);
  const float k = b.Mc - a.Mc;
  const double sc = pow2d(k), dl = -(double)k;
  a.S = fma(sc, Sk, a.S);
  a.T = fma(sc, fma(-dl, Sk, Tk), a.T);
  return a;
}

// One row's contribution to the loss partials (k_train_rows).
__device__ __forceinline__ void add_row(const RowStats& rs, const RowLoss& rl, float old, int k, double* gsum,
                                        double* bk) {
  gsum[0] += rl.loss;
  gsum[1] += 1.0;
  gsum[2] += rs.ent;
  gsum[3] += rs.logp;
  gsum[4] += rl.ratio;
  gsum[5] += rl.clip_lo;
  gsum[6] += rl.clip_hi;
  gsum[7] += (double)old - rs.logp;
  gsum[10] += rl.kl;
  double* b = bk + k * PRORL_N_PER_TURN;
  b[0] += 1.0;
  b[1] += rl.loss;
  b[2] += rs.ent;
  b[3] += rs.logp;
  b[4] += rl.clip_lo + rl.clip_hi;
}

// The merged row state the gradient needs, fp32 (one bf16 rounding of
// tolerance): every consumer warp merges the warp partials with the same
// shuffle tree (exact 2^k rescales), so all warps hold identical values.
struct PartF {
  float Mc, Mx, S, T;
};
__device__ __forceinline__ PartF merge_partial_f(PartF a, PartF b, float c) {
  if (b.Mc > a.Mc) {
    const PartF t = a;
    a = b;
    b = t;
  }
  if (b.Mc == -INFINITY) return a;
  const float rk = fmaf(b.Mx, c, -b.Mc), ek = ex2_approx(rk);
  const float Sk = b.S + ek, Tk = fmaf(rk, ek, b.T);
  const float k = b.Mc - a.Mc;
  const float sc = pow2f(k);
  a.S = fmaf(sc, Sk, a.S);
  a.T = fmaf(sc, fmaf(k, Sk, Tk), a.T);
  return a;
}

// The fp64 merge of a row's warp partials, in warp order (the epilogue warp,
// and a consumer warp deciding a clip-bound row): deterministic.
template <int K>
__device__ __noinline__ WPart merge_parts_f64(const WPart* parts, float c) {
  WPart m = parts[0];
  for (int k = 1; k < K; ++k) m = merge_partial(m, parts[k], c);
  return m;
}

// fp64 decision of the DAPO branch for a row whose fp32 ratio sits within
// 1e-5 of a clip bound (rare): the branch the fp64 loss epilogue takes.
template <int K>
__device__ __noinline__ bool unclipped_f64(const WPart* parts, float xy, float c, double inv_t, float old, double A,
                                           double lo, double hi) {
  const WPart m = merge_parts_f64<K>(parts, c);
  const RowStats rs = row_stats(m.Mc, m.Mx, m.S, m.T, xy, c, inv_t);
  const RowLoss rl = row_loss(rs.logp, old, A, lo, hi, nullptr, 0, 0.0);
  return rl.loss == -(rl.ratio * A);
}

// Generic-address element load with the clamp of Elem<T>::load (the rare NaN
// re-run reads straight from global memory).
template <typename T> __device__ __forceinline__ float load_clamped(const uint8_t* base, int64_t idx);
template <> __device__ __forceinline__ float load_clamped<__nv_bfloat16>(const uint8_t* base, int64_t idx) {
  uint32_t b = reinterpret_cast<const unsigned short*>(base)[idx];
  b = b > 0xf000u ? 0xf000u : b;
  return __uint_as_float(b << 16);
}
template <> __device__ __forceinline__ float load_clamped<float>(const uint8_t* base, int64_t idx) {
  return fmaxf(reinterpret_cast<const float*>(base)[idx], -1.5845632502852868e29f);
}

// Hysteresis of the warp-uniform running max in pass A. The reference point Mc
// need not be the exact maximum — every formula (the excluded element's
// residual r = Mx c - Mc, q = S 2^-r, the partial merge) holds for any Mc —
// it only has to bound the terms. With a slack of 1 (log2 units) a term is at
// most 2, and a row whose peak was not excluded has p_peak <= 2/3, so
// |logp| >= 0.4 and log1p(q) <= ln 3: the fp32 error stays ~1e-7 relative,
// inside the 1e-5 contract; peaked rows (p -> 1) still raise and exclude their
// peak exactly.
constexpr float kRaiseSlack = 1.0f;

// One 32-wide step of the scalar online logsumexp (element x per lane).
__device__ __forceinline__ void scalar_step(float x, float c, Top& top, LaneSums& acc, int lane) {
  if (__any_sync(kFull, x * c > top.Mc)) {
    const int L = raise_top(x, c, top, acc, lane);
    if (lane == L) x = __uint_as_float(0xf0000000u);
  }
  const float d = fmaf(x, c, -top.Mc);
  acc.add(d, ex2_approx(d));
}

// 16-B vector of gradients with element e replaced by gy (bf16 / fp32).
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

// Row geometry: the 16-B aligned interior [a, a + nb) goes through the ring,
// `head` elements before it and `tail` after it are read directly.
struct RowGeo {
  const uint8_t* rp;
  uintptr_t a;
  uint32_t nb;
  int npc, nsub, head, tail;
};

template <int ES, int kUnit, int PB>
__device__ __forceinline__ RowGeo row_geo(const TrainArgs& p, int64_t r) {
  RowGeo g;
  g.rp = p.logits + r * p.stride_bytes;
  const uintptr_t st = reinterpret_cast<uintptr_t>(g.rp);
  const uintptr_t en = st + (uintptr_t)p.vocab * ES;
  uintptr_t a = (st + 15) & ~(uintptr_t)15;
  if (a > en) a = en;
  uintptr_t b = en & ~(uintptr_t)15;
  if (b < a) b = a;
  g.a = a;
  g.nb = (uint32_t)(b - a);
  g.npc = (int)((g.nb + PB - 1) / PB);
  g.nsub = (int)((g.nb + kUnit - 1) / kUnit);
  g.head = (int)((a - st) / ES);
  g.tail = (int)((en - b) / ES);
  return g;
}

// index (element) of head/tail lane slot l (< head + tail), -1 if none
template <int ES>
__device__ __forceinline__ int64_t edge_index(const RowGeo& g, int l) {
  if (l < g.head) return l;
  if (l < g.head + g.tail)
    return (int64_t)((g.a + g.nb - reinterpret_cast<uintptr_t>(g.rp)) / ES) + (l - g.head);
  return -1;
}

// W consumer warps + G producer warps; UNIT-byte warp work units (kPiece / UNIT
// per piece). G row groups: group g (W / G consumer warps, kRing / G ring
// pieces, producer warp W + g) takes every G-th row of the CTA, so one group's
// barrier and pipeline bubbles overlap the other's work (G = 1: one group).
//
// SELF: no producer warps — pieces are single units (PB = UNIT), every ring
// slot belongs to one consumer warp, and that warp's lane 0 refills the slot it
// has just released with the piece kRG positions later in the stream (the same
// warp's next piece there), exactly like K2's per-warp ring; no cross-warp
// mbarrier hand-off remains.
template <typename T, int SUBV, int W, int UNIT, int G, bool SELF>
__global__ void __launch_bounds__((W + (SELF ? 0 : 1)) * 32, 1) k_train(const TrainArgs p) {
  constexpr int ES = Elem<T>::kSize;
  constexpr int PB = SELF ? UNIT : kProducerPiece;  // bytes per ring slot / bulk copy
  constexpr int kRing = kRingBytes / PB;     // ring slots per CTA
  constexpr int kPiece = PB;
  constexpr int kWarps = W / G;      // consumer warps per group
  constexpr int kRG = kRing / G;     // ring pieces per group
  constexpr int kUnit = UNIT;
  constexpr int kNV = kUnit / 512;         // 16-B vectors per lane per unit
  constexpr int kSplit = kPiece / kUnit;   // units per piece
  // Piece P of a group's ring stream is consumed by the kSplit warps
  // kSplit * (P mod kPG) + (0 .. kSplit-1) (one unit each, the last piece of a
  // pass padded with empty units). kRG is a multiple of kPG, so each ring slot
  // always has the same kSplit consumers and every consumer observes every
  // round of its slots in order: a parity wait can never alias a round two
  // phases behind (pieces may complete out of order).
  constexpr int kPG = kWarps / kSplit;
  static_assert(kNV % SUBV == 0 && kPiece % kUnit == 0 && W <= kMaxWarps && G <= kMaxGroups && W % G == 0 && kRing % G == 0 &&
                    kWarps % kSplit == 0 && kRG % kPG == 0,
                "launch configuration");
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full_all = reinterpret_cast<uint64_t*>(smem + (size_t)kRing * kPiece);
  uint64_t* empty_all = full_all + kRing;
  WPart* wpart_all = reinterpret_cast<WPart*>(empty_all + kRing);  // [G][2][kWarps] warp partials (row parity)
  // warps: W consumers, then (unless SELF) one producer warp whose lane g feeds row group g
  constexpr int kProdWarp = W;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp < W ? warp / kWarps : (warp == kProdWarp && !SELF ? lane : 0);  // row group (consumers) / fed group (producer lane)
  const int wq = warp < W ? warp % kWarps : 0;          // warp index inside its group
  uint8_t* ring = smem + (size_t)grp * kRG * kPiece;
  uint64_t* full = full_all + grp * kRG;
  uint64_t* empty = empty_all + grp * kRG;
  WPart* wpart = wpart_all + grp * 2 * kWarps;
  WPart* parts_g = static_cast<WPart*>(p.parts);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&full_all[s], 1);
      mbar_init(&empty_all[s], kSplit);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (!SELF && warp == kProdWarp) {
    // ===== producer: pass A (HBM, keep in L2) then pass B (L2) of each row; lane g feeds group g =====
    // The G lanes stay converged: every iteration each polls its next ring
    // slot (non-blocking test_wait) and issues the piece when the slot is free,
    // so no group's refill waits behind another group's (a divergent blocking
    // wait per lane serialised them).
    const uint64_t pol_a = l2_policy_evict_last(), pol_b = l2_policy_evict_first();
    uint32_t pc = 0;
    int64_t i = blockIdx.x + (int64_t)lane * gridDim.x;
    RowGeo g{};
    int fh = 0, pass = 0, k = 0;
    auto settle = [&]() -> bool {  // move (row, pass, k) to the next piece to issue; false when done
      for (;;) {
        if (i >= p.n_rows) return false;
        if (k < (pass == 0 ? g.npc : fh)) return true;
        if (pass == 0) {
          pass = 1;
          k = 0;
          continue;
        }
        i += (int64_t)G * gridDim.x;
        if (i >= p.n_rows) return false;
        g = row_geo<ES, kUnit, PB>(p, p.rows ? (int64_t)p.rows[i] : i);
        fh = max(0, g.npc - kRG);  // pieces [fh, npc) stay in the ring for pass B
        pass = 0;
        k = 0;
      }
    };
    if (lane < G && i < p.n_rows) {
      g = row_geo<ES, kUnit, PB>(p, p.rows ? (int64_t)p.rows[i] : i);
      fh = max(0, g.npc - kRG);
    }
    bool live = lane < G && settle();
    uint32_t idle = 0;
    while (__any_sync(kFull, live)) {
      if (live) {
        const int s = (int)(pc % kRG);
        if (mbar_test_wait(&empty[s], ((pc / kRG) & 1) ^ 1)) {
          const uint32_t bytes = min((uint32_t)kPiece, g.nb - (uint32_t)k * kPiece);
          fence_proxy_async_smem();  // the consumers' generic reads of this slot before the async-proxy refill
          mbar_arrive_expect_tx(&full[s], bytes);
          tma_load_1d(ring + (size_t)s * kPiece, reinterpret_cast<const void*>(g.a + (uintptr_t)k * kPiece), bytes,
                      &full[s], pass == 0 && k < fh ? pol_a : pol_b);
          ++pc;
          ++k;
          live = settle();
          idle = 0;
        } else if (++idle > (1u << 26)) {
          __trap();  // a slot never freed: protocol bug (the consumers' waits trap after ~4 s too)
        }
      }
    }
    return;
  }

  // ===== consumers =====
  const float c = p.c;
  const float2 c2 = make_float2(c, c);
  const uint4 fill = make_uint4(Elem<T>::kClampWord, Elem<T>::kClampWord, Elem<T>::kClampWord, Elem<T>::kClampWord);
  uint32_t pcb = 0;  // ring piece counter at the start of the row
  uint32_t j = 0;    // rows done by this CTA
  // SELF: lane 0's feeder walks the group's piece stream (pass A pieces of a
  // row, then its re-streamed pass-B pieces, then the next row) to load piece
  // q into slot q % kRG; q only grows.
  struct Feeder {
    int64_t i;
    uint32_t pcb;
    RowGeo g;
    int fh;
  } fd;
  uint64_t pol_a = 0, pol_b = 0;
  auto feed = [&](uint32_t q) {
    while (fd.i < p.n_rows && q >= fd.pcb + (uint32_t)(fd.g.npc + fd.fh)) {
      fd.pcb += (uint32_t)(fd.g.npc + fd.fh);
      fd.i += (int64_t)G * gridDim.x;
      if (fd.i < p.n_rows) {
        fd.g = row_geo<ES, kUnit, PB>(p, p.rows ? (int64_t)p.rows[fd.i] : fd.i);
        fd.fh = max(0, fd.g.npc - kRG);
      }
    }
    if (fd.i >= p.n_rows) return;
    const int k = (int)(q - fd.pcb);
    const bool pass_a = k < fd.g.npc;
    const int kp = pass_a ? k : k - fd.g.npc;
    const int sl = (int)(q % kRG);
    const uint32_t bytes = min((uint32_t)kPiece, fd.g.nb - (uint32_t)kp * kPiece);
    fence_proxy_async_smem();  // this warp's reads of the slot before the async-proxy refill
    mbar_arrive_expect_tx(&full[sl], bytes);
    tma_load_1d(ring + (size_t)sl * kPiece, reinterpret_cast<const void*>(fd.g.a + (uintptr_t)kp * kPiece), bytes,
                &full[sl], pass_a && kp < fd.fh ? pol_a : pol_b);
  };
  // the slot of piece pc has been read by the whole warp: hand it on
  auto release = [&](int sl, uint32_t pc) {
    __syncwarp();
    if (lane != 0) return;
    if constexpr (SELF) feed(pc + (uint32_t)kRG);
    else mbar_arrive_cnt(&empty[sl], 1u);
  };
  if constexpr (SELF) {
    if (lane == 0) {
      pol_a = l2_policy_evict_last();
      pol_b = l2_policy_evict_first();
      fd.i = blockIdx.x + (int64_t)grp * gridDim.x;
      fd.pcb = 0;
      fd.fh = 0;
      if (fd.i < p.n_rows) {
        fd.g = row_geo<ES, kUnit, PB>(p, p.rows ? (int64_t)p.rows[fd.i] : fd.i);
        fd.fh = max(0, fd.g.npc - kRG);
      }
      for (uint32_t q = (uint32_t)wq; q < (uint32_t)kRG; q += kWarps) feed(q);
    }
  }
  for (int64_t i = blockIdx.x + (int64_t)grp * gridDim.x; i < p.n_rows; i += (int64_t)G * gridDim.x, ++j) {
    const RowGeo g = row_geo<ES, kUnit, PB>(p, p.rows ? (int64_t)p.rows[i] : i);
    const int32_t y = p.targets[i];
    float xy = 0.f, old = 0.f, ref = 0.f;
    double Ad = 0.0;
    if (lane == 0) {
      xy = Elem<T>::load(g.rp, y);
      old = p.old_lp[i];
      Ad = p.adv[p.row_seq[i]];
      if (p.ref_lp) ref = p.ref_lp[i];
    }
    // consumed now: in place, pass B of this row overwrites x_y
    xy = __shfl_sync(kFull, xy, 0);
    old = __shfl_sync(kFull, old, 0);
    Ad = __shfl_sync(kFull, Ad, 0);
    ref = __shfl_sync(kFull, ref, 0);
    const float A = (float)Ad;
    const int kk = wq % kSplit;  // this warp's unit inside its pieces
    // first piece (offset from pc0) of a pass that this warp consumes
    auto first_piece = [&](uint32_t pc0) { return (int)(((uint32_t)(wq / kSplit) + kPG - pc0 % kPG) % kPG); };

    // pieces [fh, npc) — the last ring-full of pass A — are held in shared
    // memory and re-read by pass B from there; only [0, fh) is streamed again
    const int fh = max(0, g.npc - kRG);

    // ---- pass A: statistics ----
    Top top{-INFINITY, 0.f};
    // fp32 sums over <= 128 elements per lane (32 per accumulator), folded into
    // fp64: a 256 K-vocabulary row (16 units per warp) summed 128 terms per
    // accumulator in fp32 and carried a -8e-9 logp bias
    constexpr int kFoldUnits = (128 / (kUnit / ES / 32)) > 0 ? 128 / (kUnit / ES / 32) : 1;
    LaneSums acc;
    acc.zero();
    int nu = 0;  // units this warp has summed in this row
    for (int k = first_piece(pcb); k < g.npc; k += kPG) {
      const uint32_t pc = pcb + (uint32_t)k;
      const int u = k * kSplit + kk;
      const int s = (int)(pc % kRG);
      mbar_wait_t(&full[s], (pc / kRG) & 1);
      if (u >= g.nsub) continue;  // padding unit of the (held) last piece: released in pass B
      const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)s * kPiece + (size_t)kk * kUnit);
      const uint32_t nvv = min((uint32_t)kUnit, g.nb - (uint32_t)u * kUnit) >> 4;
      uint4 v[kNV];
      if (nvv == (uint32_t)(kUnit / 16)) {
#pragma unroll
        for (int jj = 0; jj < kNV; ++jj) v[jj] = sv[lane + 32 * jj];
      } else {
#pragma unroll
        for (int jj = 0; jj < kNV; ++jj) {
          const uint32_t qv = lane + 32 * jj;
          v[jj] = qv < nvv ? sv[qv] : fill;
        }
      }
      if (k < fh) release(s, pc);  // streamed piece: free the slot; held pieces are released by pass B
#pragma unroll
      for (int g0 = 0; g0 < kNV; g0 += SUBV) {
        uint4 w[SUBV];
#pragma unroll
        for (int jj = 0; jj < SUBV; ++jj) w[jj] = v[g0 + jj];
        const float lm = Elem<T>::template group_max<SUBV>(w);
        // raise only when a group beats the running max by more than kRaiseSlack
        // (log2 units): later terms may then reach 2^kRaiseSlack, which keeps
        // fp32 exact enough, and most of a warp's ~5 units per row skip the
        // raise + exclusion path (see the note at kRaiseSlack)
        if (__any_sync(kFull, lm * c > top.Mc + kRaiseSlack)) {
          const int L = raise_top(lm, c, top, acc, lane);
          if (lane == L) Elem<T>::template mask_first<SUBV>(w, top.Mx);
        }
        // (no RoundFix sample here: any sampled path in pass A cost K7 4 % at
        // V = 151 936 and 11 % at 32 000, whatever the sampling rate — DESIGN §3)
        Elem<T>::template accumulate<SUBV>(w, c2, make_float2(-top.Mc, -top.Mc), acc.S, acc.T);
      }
      if (++nu % kFoldUnits == 0) acc.fold();
    }
    if (wq == 0 && g.head + g.tail > 0) {
      const int64_t idx = edge_index<ES>(g, lane);
      scalar_step(idx >= 0 ? Elem<T>::load(g.rp, idx) : __uint_as_float(0xf0000000u), c, top, acc, lane);
    }
    acc.fold();
    double Sr = warp_sum_d(acc.Sd);
    double Tr = warp_sum_d(acc.Td);
    if (!(Tr == Tr) || !(Sr == Sr)) {
      // -inf / NaN / overflowing logits: clamped scalar re-run of this warp's
      // share straight from global memory (rare)
      top = Top{-INFINITY, 0.f};
      acc.zero();
      for (int k = first_piece(pcb); k * kSplit + kk < g.nsub; k += kPG) {
        const int u = k * kSplit + kk;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(g.a + (uintptr_t)u * kUnit);
        const int ne = (int)(min((uint32_t)kUnit, g.nb - (uint32_t)u * kUnit) / ES);
        for (int b = 0; b < ne; b += 32)
          scalar_step(b + lane < ne ? load_clamped<T>(src, b + lane) : __uint_as_float(0xf0000000u), c, top, acc,
                      lane);
        acc.fold();
      }
      if (wq == 0 && g.head + g.tail > 0) {
        const int64_t idx = edge_index<ES>(g, lane);
        scalar_step(idx >= 0 ? load_clamped<T>(g.rp, idx) : __uint_as_float(0xf0000000u), c, top, acc, lane);
      }
      acc.fold();
      Sr = warp_sum_d(acc.Sd);
      Tr = warp_sum_d(acc.Td);
    }
    WPart* wp = wpart + (j & 1) * kWarps;
    if (lane == 0) wp[wq] = WPart{top.Mc, top.Mx, Sr, Tr};
    named_sync(1 + grp, kWarps * 32);
    // warp 0 hands the row's fp64 warp partials (and its target logit, which pass
    // B may overwrite in place) to k_train_rows, which finishes the row in fp64
    // off this kernel's critical path
    if (wq == 0) {
      if (lane < kWarps) parts_g[i * kWarps + lane] = wp[lane];
      if (lane == 0) p.xy[i] = xy;
    }
    // every warp merges them in fp32 with the same tree -> identical results
    PartF Gp = lane < kWarps ? PartF{wp[lane].Mc, wp[lane].Mx, (float)wp[lane].S, (float)wp[lane].T}
                             : PartF{-INFINITY, 0.f, 0.f, 0.f};
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      PartF Q;
      Q.Mc = __shfl_down_sync(kFull, Gp.Mc, o);
      Q.Mx = __shfl_down_sync(kFull, Gp.Mx, o);
      Q.S = __shfl_down_sync(kFull, Gp.S, o);
      Q.T = __shfl_down_sync(kFull, Gp.T, o);
      const PartF M = merge_partial_f(Gp, Q, c);
      if ((lane & (2 * o - 1)) == 0) Gp = M;
    }
    Gp.Mc = __shfl_sync(kFull, Gp.Mc, 0);
    Gp.Mx = __shfl_sync(kFull, Gp.Mx, 0);
    Gp.S = __shfl_sync(kFull, Gp.S, 0);

    // ---- row results ----
    // fp32 for the gradient (every warp; one bf16 rounding of tolerance); the
    // fp64 outputs and loss partials come from k_train_rows
    const float rr = fmaf(Gp.Mx, c, -Gp.Mc);
    const float ir = ex2_approx(-rr);
    const float qq = Gp.S * ir;
    const float l1q = log1pf(qq);
    const float logp = (fmaf(xy, c, -Gp.Mc) - rr) * kLn2 - l1q;
    const float ratio = expf(logp - old);
    const float pg1 = ratio * A, pg2 = fminf(fmaxf(ratio, p.lo), p.hi) * A;
    bool unclipped = pg1 <= pg2;
    if (fminf(fabsf(ratio - p.lo), fabsf(ratio - p.hi)) <= 1e-5f * ratio)
      // a ratio this close to a clip bound takes the branch the fp64 loss
      // epilogue takes (rare; warp-uniform: every warp reads the same partials)
      unclipped = unclipped_f64<kWarps>(wp, xy, c, (double)p.inv_temp, old, Ad, p.lo_d, p.hi_d);
    float dl = unclipped ? -A * ratio * p.inv_n : 0.f;  // dL/dlogp
    if (p.ref_lp) dl = fmaf(p.kl_coef * p.inv_n, -expm1f(ref - logp), dl);
    const float sg = -dl * p.inv_temp;  // grad_v = sg p_v (v != y), grad_y = sg expm1(logp) = -sg (1 - p_y)
    const float l2 = fmaf(xy, c, -logp * kLog2e);
    const float gy = sg * expm1f(logp);
    if (wq == 0 && lane == 0 && p.dlogp) p.dlogp[i] = dl;

    // ---- pass B: gradient ----
    const bool zero = (sg == 0.f);
    const float2 nl2 = make_float2(-l2, -l2), s2 = make_float2(sg, sg);
    const uintptr_t yb = reinterpret_cast<uintptr_t>(g.rp) + (uintptr_t)y * ES;  // target address
    const bool y_in = yb >= g.a && yb < g.a + g.nb;
    const int32_t yvec = y_in ? (int32_t)((yb - g.a) >> 4) : -1;
    const int ye = (int)((yb & 15) / ES);
    const uint32_t pcB = pcb + (uint32_t)g.npc;  // ring position of the first re-streamed piece
    // held pieces [fh, npc) (already in the ring, mapped by their pass-A slot),
    // then the re-streamed pieces [0, fh)
    int k = first_piece(pcb);
    if (k < fh) k += (fh - k + kPG - 1) / kPG * kPG;
    for (int held = 1; held >= 0; --held) {
      if (!held) k = first_piece(pcB);
      const int kend = held ? g.npc : fh;
      for (; k < kend; k += kPG) {
        const uint32_t pc = (held ? pcb : pcB) + (uint32_t)k;
        const int u = k * kSplit + kk;
        const int s = (int)(pc % kRG);
        if (!held) mbar_wait_t(&full[s], (pc / kRG) & 1);
        if (u >= g.nsub) {  // padding unit of the last piece
          release(s, pc);
          continue;
        }
        const uint4* sv = reinterpret_cast<const uint4*>(ring + (size_t)s * kPiece + (size_t)kk * kUnit);
        const uint32_t nvv = min((uint32_t)kUnit, g.nb - (uint32_t)u * kUnit) >> 4;
        const int32_t tq = y_in ? yvec - u * (kUnit / 16) : -1;  // target vector inside this unit
        uint4* dst = reinterpret_cast<uint4*>(g.a + (uintptr_t)u * kUnit + (uintptr_t)p.goff);
        uint4 v[kNV];
        if (nvv == (uint32_t)(kUnit / 16)) {
          // full unit: no per-vector predicates; the target element (at most
          // one per row) is re-stored by the lane that wrote its vector, after
          // that vector (same thread, same address: program order)
          if (zero) {
            release(s, pc);
#pragma unroll
            for (int jj = 0; jj < kNV; ++jj) __stcs(dst + lane + 32 * jj, make_uint4(0, 0, 0, 0));
          } else {
            // load -> exps -> store per vector (the compiler barrier keeps the
            // stores spread through the unit instead of bunched at its end)
#pragma unroll
            for (int jj = 0; jj < kNV; ++jj) {
              const uint4 vj = sv[lane + 32 * jj];
              __stcs(dst + lane + 32 * jj, GElem<T>::vec(vj, c2, nl2, s2));
              asm volatile("" ::: "memory");
            }
            release(s, pc);
            if ((uint32_t)tq < (uint32_t)(kUnit / 16) && lane == (tq & 31))
              GElem<T>::store(reinterpret_cast<uint8_t*>(dst + tq), ye, gy);
          }
          continue;
        }
#pragma unroll
        for (int jj = 0; jj < kNV; ++jj) {
          const uint32_t qv = lane + 32 * jj;
          v[jj] = qv < nvv ? sv[qv] : make_uint4(0, 0, 0, 0);
        }
        release(s, pc);
#pragma unroll
        for (int jj = 0; jj < kNV; ++jj) {
          const uint32_t qv = lane + 32 * jj;
          if (qv < nvv) {
            uint4 o = make_uint4(0, 0, 0, 0);
            if (!zero) {
              o = GElem<T>::vec(v[jj], c2, nl2, s2);
              if ((int32_t)qv == tq) o = patch_target<T>(o, ye, gy);
            }
            __stcs(dst + qv, o);
          }
        }
      }
    }
    if (wq == 0 && g.head + g.tail > 0) {
      const int64_t idx = edge_index<ES>(g, lane);
      if (idx >= 0) {
        const float x = Elem<T>::load(g.rp, idx);
        float gv = 0.f;
        if (!zero) gv = idx == y ? gy : sg * ex2_approx(fmaf(x, c, -l2));
        uint8_t* gp = const_cast<uint8_t*>(g.rp) + p.goff;
        if constexpr (ES == 2) reinterpret_cast<__nv_bfloat16*>(gp)[idx] = __float2bfloat16_rn(gv);
        else reinterpret_cast<float*>(gp)[idx] = gv;
      }
    }
    pcb += (uint32_t)(g.npc + fh);
  }
}

constexpr int kMaxSlots = kRingBytes / 4096;  // smallest piece: 4 KB
constexpr size_t train_smem_bytes() {
  return (size_t)kRingBytes + (size_t)(2 * kMaxSlots) * 8 + (size_t)(2 * kMaxWarps) * sizeof(WPart);
}
static_assert(train_smem_bytes() <= 227 * 1024, "shared memory budget");

// Launch configurations (consumer warps x unit bytes). The release library
// compiles the three defaults of k7_config; a tuning build (-DPRORL_TUNING)
// has the rest, selected with PRORL_K7_CONFIG.
constexpr const char* kK7Configs[] = {"w16u4096", "w16u2048", "w24u2048", "w12u4096", "w24u4096", "w16u4096g2",
                                     "w16u2048g2", "w8u4096", "w16u4096s", "w16u4096g2s", "w16u4096g4",
                                     "w16u4096g4s"};
constexpr int kK7Default = 1, kK7TwoGroups = 5, kK7FourGroups = 10;

// Default: row groups per CTA by row size. Short rows are dominated by the
// per-row hand-offs (pass-A barrier, row results, the ring refilled only after
// pass B), so more groups overlap more rows: four groups for rows <= 80 KB
// (V = 32 000 bf16: 6.0 vs 5.1 TB/s with two), two while two rows per SM
// still fit the L2 comfortably (row <= 160 KB: 296 rows in flight <= 48 MB;
// 1.2-1.3x over one group at V = 32 000 fp32 / 65 536 bf16, where four
// groups lose 16 %), else one group of 16 warps on 2 KB units (more rows in
// flight cost L2 hits: -15 % with two groups at V = 151 936 bf16; 2 KB units
// beat 4 KB by 0-2.5 % from V = 128 256 to 262 144).
int k7_config(int64_t row_bytes) {
  static int forced = [] {
    const char* e = tuning_env("PRORL_K7_CONFIG");
    if (e)
      for (int i = 0; i < (int)(sizeof(kK7Configs) / sizeof(kK7Configs[0])); ++i)
        if (std::strcmp(e, kK7Configs[i]) == 0) return i;
    return -1;
  }();
  if (forced >= 0) return forced;
  if (row_bytes <= 80 * 1024) return kK7FourGroups;
  return row_bytes <= 160 * 1024 ? kK7TwoGroups : kK7Default;
}

// ---- k_train_rows: the fp64 row end of K7 ---------------------------------------
// One lane per row: merges the row's K warp partials in fp64 (warp order),
// row_stats / row_loss (rowmath.cuh), writes logp / entropy, and adds the loss
// partials with the fixed-order scheme of K4 (k_loss): per-lane fp64 sums over
// a fixed tile assignment, per-turn buckets accumulated in lane order, warps
// merged in order into one slab row per CTA. Deterministic run to run. Moving
// this off K7 keeps its fp64 transcendentals (~1.2k cycles of latency per row)
// and the partial bookkeeping away from the row group's critical path.
constexpr int kRowsWarps = 8;

template <int K>
__global__ void __launch_bounds__(kRowsWarps * 32) k_train_rows(const TrainArgs p, double* slab, int accumulate) {
  __shared__ double g_w[kRowsWarps * kNG];
  __shared__ double bk_w[kRowsWarps * kBucketDoubles];
  __shared__ int s_key[kRowsWarps][32];
  __shared__ double s_val[kRowsWarps][32][PRORL_N_PER_TURN];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = lane; t < kBucketDoubles; t += 32) bk_w[warp * kBucketDoubles + t] = 0.0;
  double g[kNG];
#pragma unroll
  for (int k = 0; k < kNG; ++k) g[k] = 0.0;
  const WPart* parts = static_cast<const WPart*>(p.parts);
  const int64_t gw = (int64_t)blockIdx.x * kRowsWarps + warp, nw = (int64_t)gridDim.x * kRowsWarps;
  const int64_t n_tiles = (p.n_rows + 31) / 32;
  __syncwarp();
  for (int64_t tile = gw; tile < n_tiles; tile += nw) {
    const int64_t i = tile * 32 + lane;
    int key = -1;
    if (i < p.n_rows) {
      const WPart m = merge_parts_f64<K>(parts + i * K, p.c);
      const RowStats rs = row_stats(m.Mc, m.Mx, m.S, m.T, p.xy[i], p.c, (double)p.inv_temp);
      if (p.logp) p.logp[i] = (float)rs.logp;
      if (p.entropy) p.entropy[i] = (float)rs.ent;
      const float old = p.old_lp[i];
      int k = p.row_turn[i];
      key = k < 0 ? 0 : (k >= p.n_buckets ? p.n_buckets - 1 : k);
      const RowLoss rl = row_loss(rs.logp, old, p.adv[p.row_seq[i]], p.lo_d, p.hi_d, p.ref_lp, i, (double)p.kl_coef);
      g[0] += rl.loss;
      g[1] += 1.0;
      g[2] += rs.ent;
      g[3] += rs.logp;
      g[4] += rl.ratio;
      g[5] += rl.clip_lo;
      g[6] += rl.clip_hi;
      g[7] += (double)old - rs.logp;
      g[10] += rl.kl;
      s_val[warp][lane][0] = 1.0;
      s_val[warp][lane][1] = rl.loss;
      s_val[warp][lane][2] = rs.ent;
      s_val[warp][lane][3] = rs.logp;
      s_val[warp][lane][4] = rl.clip_lo + rl.clip_hi;
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
  for (int t = threadIdx.x; t < PRORL_N_PARTIALS; t += blockDim.x) {
    double v = 0.0;
    if (t < kNG) {
      for (int w = 0; w < kRowsWarps; ++w) v += g_w[w * kNG + t];
    } else if (t >= PRORL_N_GLOBAL) {
      for (int w = 0; w < kRowsWarps; ++w) v += bk_w[w * kBucketDoubles + (t - PRORL_N_GLOBAL)];
    }
    double* dst = slab + (size_t)blockIdx.x * PRORL_N_PARTIALS + t;
    *dst = accumulate ? *dst + v : v;
  }
}

template <typename T, int W, int UNIT, int G = 1, bool SELF = false>
int run_train_cfg(const TrainArgs& a, int n_sm, double* slab, int accumulate, int* rows_used, cudaStream_t st) {
  constexpr int SUBV_BF16 = UNIT / 512 >= 8 ? 8 : UNIT / 512;
  auto kern = k_train<T, sizeof(T) == 2 ? SUBV_BF16 : 4, W, UNIT, G, SELF>;
  constexpr size_t smem = train_smem_bytes();
  PRORL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::min<int64_t>((int64_t)n_sm, a.n_rows);
  kern<<<grid, (W + (SELF ? 0 : 1)) * 32, smem, st>>>(a);
  PRORL_CUDA(cudaGetLastError());
  // the row end: fp64 stats, outputs and the loss partials (slab rows [0, rgrid))
  const int64_t tiles = (a.n_rows + 31) / 32;
  const int rgrid = (int)std::min<int64_t>((int64_t)n_sm, (tiles + kRowsWarps - 1) / kRowsWarps);
  k_train_rows<W / G><<<rgrid, kRowsWarps * 32, 0, st>>>(a, slab, accumulate);
  PRORL_CUDA(cudaGetLastError());
  *rows_used = rgrid;
  return PRORL_OK;
}

template <typename T>
int run_train(const TrainArgs& a, int n_sm, double* slab, int accumulate, int* rows_used, cudaStream_t st) {
  switch (k7_config((int64_t)a.vocab * (int64_t)sizeof(T))) {
    case kK7TwoGroups: return run_train_cfg<T, 16, 4096, 2>(a, n_sm, slab, accumulate, rows_used, st);
    case kK7FourGroups: return run_train_cfg<T, 16, 4096, 4>(a, n_sm, slab, accumulate, rows_used, st);
#ifdef PRORL_TUNING
    case 0: return run_train_cfg<T, 16, 4096>(a, n_sm, slab, accumulate, rows_used, st);
    case 2: return run_train_cfg<T, 24, 2048>(a, n_sm, slab, accumulate, rows_used, st);
    case 3: return run_train_cfg<T, 12, 4096>(a, n_sm, slab, accumulate, rows_used, st);
    case 4: return run_train_cfg<T, 24, 4096>(a, n_sm, slab, accumulate, rows_used, st);
    case 6: return run_train_cfg<T, 16, 2048, 2>(a, n_sm, slab, accumulate, rows_used, st);
    case 7: return run_train_cfg<T, 8, 4096>(a, n_sm, slab, accumulate, rows_used, st);
    case 8: return run_train_cfg<T, 16, 4096, 1, true>(a, n_sm, slab, accumulate, rows_used, st);
    case 9: return run_train_cfg<T, 16, 4096, 2, true>(a, n_sm, slab, accumulate, rows_used, st);
    case 11: return run_train_cfg<T, 16, 4096, 4, true>(a, n_sm, slab, accumulate, rows_used, st);
#endif
    default: return run_train_cfg<T, 16, 2048>(a, n_sm, slab, accumulate, rows_used, st);  // kK7Default
  }
}

}  // namespace

int train_slab_rows(prorl_ctx* ctx) { return ctx->n_sm; }

int launch_train(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab, const int32_t* rows,
                 const int32_t* targets, const float* old_lp, const double* adv, const int32_t* row_seq,
                 const int16_t* row_turn, const float* ref_lp, int64_t n_rows, float inv_temp,
                 const prorl_loss_cfg* cfg, double n_global, float* logp, float* entropy, float* dlogp, void* grad,
                 double* slab, bool accumulate, int* rows_used, cudaStream_t st) {
  *rows_used = 0;
  // every caller (prorl_score_grad, prorl_score_host's training mode) goes
  // through these checks: the kernel indexes per-group shared-memory buckets
  // by turn and writes the gradient row by row at row_stride
  if (dtype != PRORL_BF16 && dtype != PRORL_FP32) return fail(PRORL_E_SHAPE, "train: unknown logits dtype");
  if (vocab <= 0 || row_stride < vocab) return fail(PRORL_E_SHAPE, "train: need vocab > 0 and row_stride >= vocab");
  if (!(inv_temp > 0.f)) return fail(PRORL_E_MALFORMED_REQUEST, "train: inv_temperature must be > 0");
  if (!(n_global > 0.0)) return fail(PRORL_E_MALFORMED_REQUEST, "train: n_global must be > 0");
  if (!cfg || cfg->n_buckets < 1 || cfg->n_buckets > PRORL_TURN_BUCKETS)
    return fail(PRORL_E_SHAPE, "train: n_buckets out of [1, 64]");
  const int esz = dtype == PRORL_BF16 ? 2 : 4;
  if (reinterpret_cast<uintptr_t>(logits) % esz ||
      (static_cast<const uint8_t*>(grad) - static_cast<const uint8_t*>(logits)) % 16 != 0)
    return fail(PRORL_E_SHAPE, "train: grad must share the logits' 16-byte alignment phase");
  if (n_rows <= 0) return PRORL_OK;
  TrainArgs a{};
  a.logits = static_cast<const uint8_t*>(logits);
  a.stride_bytes = row_stride * esz;
  a.goff = static_cast<const uint8_t*>(grad) - static_cast<const uint8_t*>(logits);
  a.vocab = vocab;
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
  a.lo_d = 1.0 - (double)cfg->eps_lo;
  a.hi_d = 1.0 + (double)cfg->eps_hi;
  a.inv_n = (float)(1.0 / n_global);
  a.n_buckets = cfg->n_buckets;
  a.logp = logp;
  a.entropy = entropy;
  a.dlogp = dlogp;
  // row-end workspace: each row's fp64 warp partials (<= kMaxWarps) + its target logit
  PRORL_CUDA(ctx->k7rows.ensure((size_t)n_rows * (kMaxWarps * sizeof(WPart) + sizeof(float))));
  a.parts = ctx->k7rows.p;
  a.xy = reinterpret_cast<float*>(static_cast<uint8_t*>(ctx->k7rows.p) + (size_t)n_rows * kMaxWarps * sizeof(WPart));
  const int acc = accumulate ? 1 : 0;
  return dtype == PRORL_BF16 ? run_train<__nv_bfloat16>(a, ctx->n_sm, slab, acc, rows_used, st)
                             : run_train<float>(a, ctx->n_sm, slab, acc, rows_used, st);
}

}  // namespace prorl
