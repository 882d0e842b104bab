// lmhead.cu — K6: fused LM head + logprob / entropy on the 5th-gen tensor
// cores (SURVEY.md §8 f rank 2). The model forward is outside the reference's
// scope; this kernel removes the logits round trip of K2: the
// logits tile  X[128 rows x 256 vocab] = H[128 x d] . W[256 x d]^T  is
// accumulated in TMEM by tcgen05.mma and consumed in place by an online
// logsumexp epilogue, so the [rows x V] logits never reach HBM.
//
// CTA = one 128-row tile of hidden states, persistent over all V/256 vocab
// tiles (the same order in every CTA, so the W tiles are shared through L2).
// Warp roles (192 threads):
//   warp 0      TMA producer (one elected lane): H / W tiles, 128B-swizzled
//               (cp.async.bulk.tensor.2d, K-major, BK = 64 bf16 = one swizzle
//               atom), STAGES-deep smem ring with full/empty mbarriers;
//   warp 1      TMEM owner (tcgen05.alloc 512 columns = 2 accumulators of
//               128 lanes x 256 fp32) and MMA issuer (one lane):
//               tcgen05.mma.cta_group::1.kind::f16, M128 N256 K16, bf16 in,
//               fp32 accumulate; tcgen05.commit frees smem stages and
//               signals a finished accumulator;
//   warps 2..5  epilogue: thread = one row (TMEM lane), tcgen05.ld 32 columns
//               at a time, online base-2 logsumexp with the top element kept
//               out of the sums (as K2), target-logit capture; the two TMEM
//               accumulators let MMA of tile n+1 overlap the epilogue of n.
// Output: logp / entropy per row, identical definitions to K2 (App. B.2).
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "rowmath.cuh"

namespace prorl {

namespace {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK * 2;  // 16 KB
constexpr uint32_t B_BYTES = BN * BK * 2;  // 32 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int kThreads = 192;
constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLog2e = 1.44269504088896340736f;

struct LmParams {
  int64_t n_rows;
  int32_t vocab;
  int32_t n_kb;      // d / BK
  int32_t n_ntiles;  // ceil(V / BN)
  int32_t m_tiles;   // ceil(n_rows / BM)
  int32_t n_chunks;  // vocab chunks per row tile (work unit = row tile x vocab chunk)
  int32_t tpc;       // vocab tiles per chunk
  float c;           // inv_temp * log2 e
  const int32_t* targets;
  float* part;       // [n_rows][n_chunks][6]: Mc, Mx, S, T, xy, has_y
  // Pacing (pair kernel, one chunk: every unit walks the whole vocabulary):
  // producers publish each vocab tile they have issued in pace[tile] and do
  // not issue tile n before every unit of the waves so far has issued tile
  // n - pace_window, so all pairs stream the same few W tiles through L2
  // (null: no pacing).
  int32_t* pace;
  int32_t pace_window;
};

// Work units u = chunk * m_tiles + m (chunk-major: CTAs running at the same
// time mostly share one vocab chunk of W through L2); CTA b takes b, b+G, ...
struct Unit {
  int32_t m, chunk, t0, t1;  // row tile, vocab chunk, vocab tiles [t0, t1)
};
__device__ __forceinline__ Unit unit_of(const LmParams& p, int64_t u) {
  Unit x;
  x.chunk = (int32_t)(u / p.m_tiles);
  x.m = (int32_t)(u - (int64_t)x.chunk * p.m_tiles);
  x.t0 = x.chunk * p.tpc;
  x.t1 = min(p.n_ntiles, x.t0 + p.tpc);
  return x;
}

__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t parity) {
  // bounded wait: a protocol bug traps after ~4 s instead of hanging the GPU
  if (mbar_try_wait(bar, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t k = 1;; ++k) {
    if (mbar_try_wait(bar, parity)) return;
    if ((k & 255u) == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 4000000000ull) __trap();
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(policy)
      : "memory");
}

// L2 policies: the hidden-state tile of a unit is re-streamed for every vocab
// tile of its chunk (keep it: evict_last); the W tiles are shared by all the
// units walking the same chunk at roughly the same time (normal).
__device__ __forceinline__ uint64_t policy_keep() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem) {
  const uint64_t addr = (smem_u32(smem) & 0x3FFFFu) >> 4;
  return addr | (uint64_t(1) << 16)      // leading byte offset (unused for swizzled K-major) = 1
         | (uint64_t(64) << 32)          // stride byte offset: 1024 B >> 4
         | (uint64_t(1) << 46)           // descriptor version (sm_100)
         | (uint64_t(2) << 61);          // layout: SWIZZLE_128B
}

// Instruction descriptor: kind::f16, A/B bf16 K-major, D fp32, M = 128, N = 256.
constexpr uint32_t kIdesc = (1u << 4)          // D format f32
                            | (1u << 7)        // A format bf16
                            | (1u << 10)       // B format bf16
                            | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// Online logsumexp state of one row (one epilogue thread) over a vocab chunk.
// Per row: ~V terms. Each 32-column group is summed in 4 chains, then added
// to the running (S, T) with Kahan compensation (cS, cT), so the fp32 error
// stays at a few ulps over 150K+ terms; the element that set the running max
// is kept out of the sums (re-added analytically by the merge).
struct RowAcc {
  float Mc = -INFINITY, Mx = 0.f, S = 0.f, T = 0.f, cS = 0.f, cT = 0.f, xy = 0.f;
  bool has_y = false;
};

// Consume one accumulator tile row: 256 fp32 logits at TMEM address `base`
// (this thread's lane), vocab columns [col0, col0 + ncols).
__device__ __forceinline__ void epi_tile(uint32_t base, int col0, int ncols, int32_t tgt, float c, RowAcc& a) {
  for (int c0 = 0; c0 < BN; c0 += 32) {
    float v[32];
    tmem_ld32(base + (uint32_t)c0, v);
    if (c0 >= ncols) continue;
    const int lim = min(32, ncols - c0);
    const int ty = tgt - col0 - c0;
    if (ty >= 0 && ty < lim) a.has_y = true;
#pragma unroll
    for (int j = 0; j < 32; ++j) a.xy = (j == ty) ? v[j] : a.xy;
    float lm = v[0];
#pragma unroll
    for (int j = 1; j < 32; ++j) lm = j < lim ? fmaxf(lm, v[j]) : lm;
    int excl = -1;
    if (lm * c > a.Mc) {  // new top element: fold the old one in, rescale, exclude the new one
#pragma unroll
      for (int j = 31; j >= 0; --j) excl = (j < lim && v[j] == lm) ? j : excl;
      const float nMc = lm * c;
      if (a.Mc != -INFINITY) {
        const float sc = ex2_approx(a.Mc - nMc), dl = nMc - a.Mc;
        a.T = sc * fmaf(-dl, a.S, a.T);
        a.cT = sc * fmaf(-dl, a.cS, a.cT);
        a.S *= sc;
        a.cS *= sc;
        const float d = fmaf(a.Mx, c, -nMc), e = ex2_approx(d);
        float y = e - a.cS, t = a.S + y;
        a.cS = (t - a.S) - y;
        a.S = t;
        y = d * e - a.cT;
        t = a.T + y;
        a.cT = (t - a.T) - y;
        a.T = t;
      }
      a.Mc = nMc;
      a.Mx = lm;
    }
    float gs[4] = {0.f, 0.f, 0.f, 0.f}, gt[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < lim && j != excl) {
        const float d = fmaf(v[j], c, -a.Mc), e = ex2_approx(d);
        gs[j & 3] += e;
        gt[j & 3] = fmaf(d, e, gt[j & 3]);
      }
    }
    float y = ((gs[0] + gs[1]) + (gs[2] + gs[3])) - a.cS, t = a.S + y;
    a.cS = (t - a.S) - y;
    a.S = t;
    y = ((gt[0] + gt[1]) + (gt[2] + gt[3])) - a.cT;
    t = a.T + y;
    a.cT = (t - a.T) - y;
    a.T = t;
  }
}

__device__ __forceinline__ void store_partial(const LmParams& p, int64_t grow, int32_t chunk, const RowAcc& a) {
  float* o = p.part + ((size_t)grow * p.n_chunks + chunk) * 6;
  o[0] = a.Mc;
  o[1] = a.Mx;
  o[2] = a.S;
  o[3] = a.T;
  o[4] = a.xy;
  o[5] = a.has_y ? 1.f : 0.f;
}

#ifdef PRORL_TUNING  // single-CTA variant (PRORL_K6_PAIR=0): tuning builds only
__global__ void __launch_bounds__(kThreads, 1)
    k_lmhead(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW, const LmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for the 128B-swizzle atoms
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_units = (int64_t)p.m_tiles * p.n_chunks;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmH)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
  }
  if (warp == 1) {  // whole warp: allocate 512 TMEM columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer =====
      const uint64_t pol_h = policy_keep(), pol_w = policy_normal();
      uint32_t s = 0, ph = 0;
      for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit w = unit_of(p, u);
        for (int n = w.t0; n < w.t1; ++n) {
          for (int kb = 0; kb < p.n_kb; ++kb) {
            mbar_wait_bounded(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
            tma_load_2d(sA + s * A_BYTES, &tmH, kb * BK, w.m * BM, &full[s], pol_h);
            tma_load_2d(sB + s * B_BYTES, &tmW, kb * BK, n * BN, &full[s], pol_w);
            if (++s == STAGES) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer =====
      uint32_t s = 0, ph = 0;
      int tile = 0;  // accumulator use counter across units
      for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
       const Unit w = unit_of(p, u);
       for (int n = w.t0; n < w.t1; ++n, ++tile) {
        const int acc = tile & 1;
        mbar_wait_bounded(&tempty[acc], ((tile >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d_tmem = tmem + (uint32_t)(acc * BN);
        for (int kb = 0; kb < p.n_kb; ++kb) {
          mbar_wait_bounded(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = umma_desc_sw128(sA + s * A_BYTES);
          const uint64_t bd = umma_desc_sw128(sB + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)  // K = 16 per MMA: +32 B along the swizzle atom
            umma_bf16(d_tmem, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), (kb | k) != 0);
          umma_commit(&empty[s]);  // smem stage free once these MMAs retire
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
       }
      }
    }
  } else {
    // ===== epilogue: one row per thread =====
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    const float c = p.c;
    int tile = 0;
    for (int64_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    const Unit w = unit_of(p, u);
    const int64_t grow = (int64_t)w.m * BM + row;
    const int32_t tgt = grow < p.n_rows ? p.targets[grow] : -1;
    RowAcc a;
    for (int n = w.t0; n < w.t1; ++n, ++tile) {
      const int acc = tile & 1;
      mbar_wait_bounded(&tfull[acc], (tile >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      epi_tile(base, n * BN, min(BN, p.vocab - n * BN), tgt, c, a);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[acc]);
    }
    if (grow < p.n_rows) store_partial(p, grow, w.chunk, a);  // this unit's partial for (row, chunk)
    }  // units
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}
#endif  // PRORL_TUNING

// ---- 2-CTA variant (cta_group::2): a CTA pair computes 256-row x 256-vocab
// logits tiles. Rank r of the pair holds rows [128 r, 128 r + 128) of the
// tile's hidden states and vocab rows [128 r, 128 r + 128) of the W tile in
// its shared memory; the leader (rank 0) issues tcgen05.mma.cta_group::2
// (M256 N256 K16), which reads both CTAs' operands and writes each CTA's 128
// accumulator rows into its own TMEM. Per CTA the shared-memory operand
// traffic per logit halves (each W tile is loaded once per pair instead of
// once per CTA), and one MMA instruction covers twice the work.
constexpr int STAGES2 = 6;
constexpr uint32_t A2_BYTES = BM * BK * 2;         // 16 KB: this CTA's 128 hidden rows
constexpr uint32_t B2_BYTES = (BN / 2) * BK * 2;   // 16 KB: this CTA's half of the W tile
constexpr uint32_t STAGE2_BYTES = A2_BYTES + B2_BYTES;
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)((2 * BM) >> 4) << 24);

__device__ __forceinline__ uint32_t lm_cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t lm_cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t lm_n_clusters() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void lm_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t lm_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// TMA 2-D tile into this CTA's shared memory, completing on the LEADER's mbarrier
// (cluster address `bar_cluster`).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                                 uint32_t bar_cluster, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(x), "r"(y), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(kIdesc2), "r"(accumulate)
      : "memory");
}
// one lane of the converged warp (elect.sync)
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(e));
  return e != 0;
}
// Arrive (once the MMAs issued so far retire) on barrier `bar` in BOTH CTAs of the pair.
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// Pacing counters (global memory, one int per vocab tile).
__device__ __forceinline__ void pace_post(int32_t* cnt) {
  asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(cnt) : "memory");
}
// Pacing is a hint, never a dependency: a worker waits at most ~200 us for the
// slowest one, so a launch whose pairs are not all co-resident (a GPU shared
// with other kernels) still makes progress, just without the L2 sharing.
__device__ __forceinline__ void pace_wait(const int32_t* cnt, int32_t target) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
  if (v >= target) return;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    __nanosleep(256);
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
    if (v >= target) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 200000ull) return;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_lmhead2(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmW, const LmParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES2 * A2_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE2_BYTES);  // leader's is used
  uint64_t* empty = full + STAGES2;                                              // both CTAs
  uint64_t* tfull = empty + STAGES2;                                             // both CTAs
  uint64_t* tempty = tfull + 2;                                                  // leader's is used
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = lm_cluster_ctarank();
  const int64_t q0 = lm_cluster_id(), nq = lm_n_clusters();
  const int64_t n_units = (int64_t)p.m_tiles * p.n_chunks;  // m_tiles counts 256-row pair tiles here

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmH)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
  }
  lm_cluster_sync();  // both CTAs' barriers exist before any remote arrive / complete_tx
  if (warp == 1) {    // the same warp in both CTAs: allocate 512 TMEM columns for the pair
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  lm_cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    {  // ===== TMA producer (both CTAs): the warp runs converged, one elected lane issues (as the MMA warp) =====
      const uint64_t pol_h = policy_keep(), pol_w = policy_normal();
      uint32_t s = 0, ph = 0;
      for (int64_t u = q0; u < n_units; u += nq) {
        const Unit w = unit_of(p, u);
        for (int n = w.t0; n < w.t1; ++n) {
          // every unit of the waves so far (full waves of nq pairs, then this one) has issued tile n - window
          if (p.pace && rank == 0 && n >= p.pace_window) {
            if (lane == 0) pace_wait(p.pace + (n - p.pace_window), (int32_t)min(n_units, (u / nq + 1) * nq));
            __syncwarp();
          }
          for (int kb = 0; kb < p.n_kb; ++kb) {
            mbar_wait_bounded(&empty[s], ph ^ 1);
            const uint32_t bar = lm_mapa(smem_u32(&full[s]), 0);
            if (elect_one()) {
              if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * STAGE2_BYTES);
              tma_load_2d_pair(sA + s * A2_BYTES, &tmH, kb * BK, w.m * (2 * BM) + (int)rank * BM, bar, pol_h);
              tma_load_2d_pair(sB + s * B2_BYTES, &tmW, kb * BK, n * BN + (int)rank * (BN / 2), bar, pol_w);
            }
            __syncwarp();
            if (++s == STAGES2) {
              s = 0;
              ph ^= 1;
            }
          }
          if (p.pace && rank == 0 && lane == 0) pace_post(p.pace + n);
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // ===== MMA issuer (leader only) =====
      // The whole warp runs the loop converged and one elected lane issues:
      // the descriptors stay warp-uniform, so ptxas keeps them in uniform
      // registers. (Issued from a lane-0-only branch, every tcgen05.mma came
      // with an elect / R2UR.BROADCAST waterfall: ~115 instructions per
      // 64-deep k-block against 512 cycles of tensor work, which held the
      // tensor pipe at ~88 % of the active cycles.)
      uint32_t s = 0, ph = 0;
      int tile = 0;
      for (int64_t u = q0; u < n_units; u += nq) {
        const Unit w = unit_of(p, u);
        for (int n = w.t0; n < w.t1; ++n, ++tile) {
          const int acc = tile & 1;
          mbar_wait_bounded(&tempty[acc], ((tile >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t d_tmem = tmem + (uint32_t)(acc * BN);
          for (int kb = 0; kb < p.n_kb; ++kb) {
            mbar_wait_bounded(&full[s], ph);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t ad = umma_desc_sw128(sA + s * A2_BYTES);
            const uint64_t bd = umma_desc_sw128(sB + s * B2_BYTES);
            if (elect_one()) {
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                umma_bf16_pair(d_tmem, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), (kb | k) != 0);
              umma_commit_pair(&empty[s]);  // both CTAs' stage s free once these MMAs retire
            }
            __syncwarp();
            if (++s == STAGES2) {
              s = 0;
              ph ^= 1;
            }
          }
          if (elect_one()) umma_commit_pair(&tfull[acc]);  // both CTAs' accumulators ready
          __syncwarp();
        }
      }
    }
  } else {
    // ===== epilogue (both CTAs): one row per thread =====
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const float c = p.c;
    const uint32_t tempty_leader0 = lm_mapa(smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = lm_mapa(smem_u32(&tempty[1]), 0);
    int tile = 0;
    for (int64_t u = q0; u < n_units; u += nq) {
      const Unit w = unit_of(p, u);
      const int64_t grow = (int64_t)w.m * (2 * BM) + (int64_t)rank * BM + row;
      const int32_t tgt = grow < p.n_rows ? p.targets[grow] : -1;
      RowAcc a;
      for (int n = w.t0; n < w.t1; ++n, ++tile) {
        const int acc = tile & 1;
        mbar_wait_bounded(&tfull[acc], (tile >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
        epi_tile(base, n * BN, min(BN, p.vocab - n * BN), tgt, c, a);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      }
      if (grow < p.n_rows) store_partial(p, grow, w.chunk, a);
    }
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  lm_cluster_sync();  // the peer's epilogue and the leader's MMAs are done with both TMEMs
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// Per row: merge the vocab-chunk partials (each chunk's top element is kept
// out of its sums) into logp / entropy with the same exclusion trick as K2.
__global__ void k_lmhead_merge(const float* __restrict__ part, int64_t n_rows, int32_t n_chunks, float c, float inv_t,
                               float* __restrict__ logp, float* __restrict__ entropy) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  const float* pr = part + (size_t)i * n_chunks * 6;
  int g = 0;
  float xy = 0.f;
  for (int k = 0; k < n_chunks; ++k) {
    if (pr[k * 6] > pr[g * 6]) g = k;
    if (pr[k * 6 + 5] != 0.f) xy = pr[k * 6 + 4];
  }
  const float Mc = pr[g * 6], Mx = pr[g * 6 + 1];
  float S = pr[g * 6 + 2], T = pr[g * 6 + 3];
  for (int k = 0; k < n_chunks; ++k) {
    if (k == g) continue;
    const float mk = pr[k * 6];
    if (mk == -INFINITY) continue;
    const float rk = fmaf(pr[k * 6 + 1], c, -mk), ek = exp2f(rk);
    const float Sk = pr[k * 6 + 2] + ek, Tk = fmaf(rk, ek, pr[k * 6 + 3]);  // fold the chunk's top in
    const float sc = exp2f(mk - Mc), dl = Mc - mk;
    S = fmaf(sc, Sk, S);
    T = fmaf(sc, fmaf(-dl, Sk, Tk), T);
  }
  const rowmath::RowStats rs = rowmath::row_stats(Mc, Mx, S, T, xy, c, (double)inv_t);  // fp64 row end
  logp[i] = (float)rs.logp;
  if (entropy) entropy[i] = (float)rs.ent;
}

// K6 pacing window in vocab tiles (PRORL_K6_PACE, 0 = off). Default 4: the
// pairs stay within 4 W tiles (5 MB) of each other, W streams from HBM ~twice
// instead of ~7x (ncu 1.7-2.2 GB vs 6.2 GB per 16 384-row launch), and the
// saved DRAM energy buys clock at the power cap (whole step 570 vs 587 ms).
int lmhead_pacing() {
  static int w = [] {
    const char* e = tuning_env("PRORL_K6_PACE");
    return e ? std::max(0, std::atoi(e)) : 4;
  }();
  return w;
}

// K6 launch mode: CTA pairs (cta_group::2) unless PRORL_K6_PAIR=0.
bool lmhead_pair_mode() {
  static bool pair = [] {
    const char* e = tuning_env("PRORL_K6_PAIR");
    return !(e && e[0] == '0');
  }();
  return pair;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

int make_map(CUtensorMap* m, const void* base, int64_t rows, int32_t d, int64_t stride_elems, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(PRORL_E_CUDA, "lmhead: cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)stride_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PRORL_E_SHAPE, "lmhead: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return PRORL_OK;
}

}  // namespace

int launch_lmhead(prorl_ctx* ctx, const void* hidden, int64_t h_stride, const void* weight, int64_t w_stride,
                  int32_t d, int32_t vocab, const int32_t* targets, int64_t n_rows, float inv_temp, float* logp,
                  float* entropy, cudaStream_t st) {
  if (d <= 0 || d % BK != 0) return fail(PRORL_E_SHAPE, "lmhead: hidden size must be a positive multiple of 64");
  if (vocab <= 0 || n_rows < 0) return fail(PRORL_E_SHAPE, "lmhead: bad vocab / rows");
  if (h_stride < d || w_stride < d || (h_stride * 2) % 16 || (w_stride * 2) % 16 ||
      reinterpret_cast<uintptr_t>(hidden) % 16 || reinterpret_cast<uintptr_t>(weight) % 16)
    return fail(PRORL_E_SHAPE, "lmhead: hidden/weight must be 16-B aligned with 16-B multiple row strides");
  if (!(inv_temp > 0.f)) return fail(PRORL_E_MALFORMED_REQUEST, "lmhead: inv_temperature must be > 0");
  if (n_rows == 0) return PRORL_OK;
  const bool pair = lmhead_pair_mode();
  CUtensorMap tmH, tmW;
  PRORL_TRY_INTERNAL(make_map(&tmH, hidden, n_rows, d, h_stride, BM));
  PRORL_TRY_INTERNAL(make_map(&tmW, weight, vocab, d, w_stride, pair ? BN / 2 : BN));
  LmParams p{};
  p.n_rows = n_rows;
  p.vocab = vocab;
  p.n_kb = d / BK;
  p.n_ntiles = (vocab + BN - 1) / BN;
  const int rows_per_tile = pair ? 2 * BM : BM;
  p.m_tiles = (int32_t)((n_rows + rows_per_tile - 1) / rows_per_tile);
  const int n_workers = pair ? ctx->n_sm / 2 : ctx->n_sm;  // CTA pairs or CTAs
  // Split the vocabulary into chunks only as far as needed to keep the workers
  // busy: the FEWEST chunks whose round-robin makespan ceil(units / workers) *
  // tiles_per_chunk keeps >= 85 % of the workers' time useful (else the best
  // balance; chunks of >= 16 vocab tiles). Few chunks keep every worker walking
  // the same W tiles in step, so W streams from HBM about once (ncu: 0.87 GB
  // per launch at one chunk vs 13-15 GB at 15 chunks); the kernel runs at the
  // power cap, and the saved DRAM energy buys clock (measured sustained:
  // 1 263 TFLOP/s with CTA pairs and one chunk vs 1 195 with 15 chunks).
  {
    const int64_t total = (int64_t)p.m_tiles * p.n_ntiles;
    double best = -1.0;
    for (int32_t nch = 1; nch <= p.n_ntiles; ++nch) {
      const int32_t tpc = (p.n_ntiles + nch - 1) / nch;
      if (nch > 1 && tpc < 16) break;  // keep partial-merge traffic small (<= 1/16 of the tiles)
      const int32_t chunks = (p.n_ntiles + tpc - 1) / tpc;
      const int64_t units = (int64_t)p.m_tiles * chunks;
      const int64_t g = std::min<int64_t>(units, n_workers);
      const double eff = (double)total / ((double)g * (double)((units + g - 1) / g) * tpc) * ((double)g / n_workers);
      if (eff > best + 1e-3) {
        best = eff;
        p.tpc = tpc;
        p.n_chunks = chunks;
      }
      if (eff >= 0.85) break;
    }
  }
  if (const char* e = tuning_env("PRORL_K6_CHUNKS")) {  // tuning override: vocab chunks per row tile
    const int32_t nch = std::max(1, std::min(p.n_ntiles, std::atoi(e)));
    p.tpc = (p.n_ntiles + nch - 1) / nch;
    p.n_chunks = (p.n_ntiles + p.tpc - 1) / p.tpc;
  }
  p.c = inv_temp * kLog2e;
  p.targets = targets;
  PRORL_CUDA(ctx->lm_part.ensure(sizeof(float) * 6 * (size_t)n_rows * (size_t)p.n_chunks));
  p.part = ctx->lm_part.as<float>();
  const int64_t units = (int64_t)p.m_tiles * p.n_chunks;
  p.pace = nullptr;
  // Pacing (one chunk: every unit walks every vocab tile). With more row
  // tiles than pairs the pairs take them in waves; pace[n] then counts the
  // issues of tile n over the waves so far, and a unit of wave w waits for the
  // (w + 1) * pairs (or all) units before it (without this, a second wave ran
  // at 0.85x of the unfused path: W streamed from HBM by every pair).
  if (pair && p.n_chunks == 1 && lmhead_pacing() > 0) {
    PRORL_CUDA(ctx->lm_pace.ensure(sizeof(int32_t) * (size_t)p.n_ntiles));
    PRORL_CUDA(cudaMemsetAsync(ctx->lm_pace.p, 0, sizeof(int32_t) * (size_t)p.n_ntiles, st));
    p.pace = ctx->lm_pace.as<int32_t>();
    p.pace_window = lmhead_pacing();
  }
  if (pair) {
    const size_t smem = (size_t)STAGES2 * STAGE2_BYTES + 1024 + 256;
    PRORL_CUDA(cudaFuncSetAttribute(k_lmhead2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(units, n_workers)));
    PRORL_CUDA(cudaLaunchKernelEx(&cfg, k_lmhead2, tmH, tmW, p));
  } else {
#ifdef PRORL_TUNING
    const size_t smem = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
    PRORL_CUDA(cudaFuncSetAttribute(k_lmhead, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = (unsigned)std::min<int64_t>(units, n_workers);
    k_lmhead<<<grid, kThreads, smem, st>>>(tmH, tmW, p);
#endif
  }
  PRORL_CUDA(cudaGetLastError());
  k_lmhead_merge<<<(unsigned)((n_rows + 255) / 256), 256, 0, st>>>(p.part, n_rows, p.n_chunks, p.c, inv_temp, logp,
                                                                    entropy);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

}  // namespace prorl
