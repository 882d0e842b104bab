// grad.cu — K5: backward of the DAPO token-mean surrogate through the
// log-softmax, streamed over the logits (SURVEY.md §8 f rank 1; no reference
// code: SPEC.md:741).
//
// For active row i with target y, forward logp_i (from K2), behaviour logprob
// old_i and advantage A = adv[seq_i]:
//   ratio = exp(logp - old),  l = -min(ratio A, clip(ratio, 1-eps_lo, 1+eps_hi) A)
//   dL/dlogp_i = -A ratio / N   if the unclipped branch is the min, else 0
//                (L = sum_i l_i / N, N = global active rows after the all-reduce)
//   dL/dx_iv   = dL/dlogp_i * inv_T * (1[v = y] - p_v),   p_v = exp(x_v inv_T - lse_i)
// with lse_i = x_y inv_T - logp_i recovered from the forward output. One HBM
// read + one HBM write of the row (4V bytes bf16); the same per-warp TMA ring
// as K2 feeds the reads, results leave as 16-B streaming stores (st.global.cs)
// packed to bf16 pairs (cvt.rn.bf16x2.f32). Rows whose gradient scale is 0
// (clipped branch, A = 0) skip the exp work and store zeros. The gradient
// buffer may alias the logits (in-place backward): every chunk is in shared
// memory before its region is overwritten, and the target logit is read at
// row start.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "rowmath.cuh"
#include "stream.cuh"

namespace prorl {

namespace {

using namespace rowmath;

struct GradArgs {
  const uint8_t* logits;
  int64_t stride_bytes;
  int32_t vocab;
  const int32_t* rows;
  uint8_t* grad;  // same row stride and 16-B phase as logits
  const int32_t* targets;
  const float* logp;
  const float* old_lp;
  const double* adv;
  const int32_t* row_seq;
  const float* ref_lp;  // nullable (k3 KL term)
  float kl_coef;
  int64_t n_rows;
  float c;         // inv_temp * log2 e
  float inv_temp;
  float lo, hi;    // 1 - eps_lo, 1 + eps_hi
  float inv_n;     // 1 / N_global
  float* dlogp;    // optional per-row dL/dlogp
};

template <typename T, int WARPS, int STAGES, int CHUNK>
__global__ void __launch_bounds__(WARPS * 32, 1) k_grad(const GradArgs p) {
  constexpr int NV = CHUNK / 512;
  constexpr int ES = GElem<T>::ES;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * WARPS + warp, nw = (int64_t)gridDim.x * WARPS;
  RowRing<STAGES, CHUNK, ES> rr;
  rr.init(smem + (size_t)warp * STAGES * CHUNK,
          reinterpret_cast<uint64_t*>(smem + (size_t)WARPS * STAGES * CHUNK) + warp * STAGES, p.logits,
          p.stride_bytes, p.rows, p.n_rows, p.vocab, gw, nw, lane);
  const int64_t goff = p.grad - p.logits;  // same stride and 16-B phase (checked on the host)

  for (int64_t i = gw; i < p.n_rows; i += nw) {
    const uint8_t* rp = rr.row_ptr(i);
    uint8_t* gp = const_cast<uint8_t*>(rp) + goff;
    uintptr_t a, b;
    rr.interior(rp, a, b);
    const int64_t nchunks = rr.chunks(a, b);
    const int head = (int)((a - reinterpret_cast<uintptr_t>(rp)) / ES);
    const int tail = (int)((reinterpret_cast<uintptr_t>(rp) + (uintptr_t)p.vocab * ES - b) / ES);
    const int32_t y = p.targets[i];
    // per-row scale (lane 0), broadcast
    float s = 0.f, l2 = 0.f, gy = 0.f;
    if (lane == 0) {
      const float xy = GElem<T>::load(rp, y);
      const float lp = p.logp[i], old = p.old_lp[i];
      const float A = (float)p.adv[p.row_seq[i]];
      const float ratio = expf(lp - old);
      const float pg1 = ratio * A, pg2 = fminf(fmaxf(ratio, p.lo), p.hi) * A;
      float dl = (pg1 <= pg2) ? -A * ratio * p.inv_n : 0.f;  // dL/dlogp
      if (p.ref_lp) dl = fmaf(p.kl_coef * p.inv_n, -expm1f(p.ref_lp[i] - lp), dl);  // d(k3)/dlogp = 1 - e^(ref-lp)
      if (p.dlogp) p.dlogp[i] = dl;
      s = -dl * p.inv_temp;  // grad_v = s * p_v for v != y, grad_y = -s * (1 - p_y)
      l2 = fmaf(xy, p.c, -lp * kLog2e);                            // lse in base-2 units
      gy = s * expm1f(lp);  // -s (1 - p_y), exact as p_y -> 1
    }
    s = __shfl_sync(0xffffffffu, s, 0);
    l2 = __shfl_sync(0xffffffffu, l2, 0);
    const float2 c2 = make_float2(p.c, p.c), nl2 = make_float2(-l2, -l2), s2 = make_float2(s, s);
    const bool zero = (s == 0.f);  // warp-uniform: clipped branch / A == 0 -> all-zero row

    if (head + tail > 0) {
      int64_t idx = -1;
      if (lane < head) idx = lane;
      else if (lane < head + tail) idx = (int64_t)((b - reinterpret_cast<uintptr_t>(rp)) / ES) + (lane - head);
      if (idx >= 0) {
        const float x = GElem<T>::load(rp, idx);
        GElem<T>::store(gp, idx, zero ? 0.f : s * ex2_approx(fmaf(x, p.c, -l2)));
      }
    }
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const uint32_t nvec = (uint32_t)(min((uintptr_t)CHUNK, b - (a + (uintptr_t)ch * CHUNK)) >> 4);
      const uint4* sv = rr.wait();
      uint4* dst = reinterpret_cast<uint4*>(a + (uintptr_t)ch * CHUNK + (uintptr_t)goff);
      if (!zero && nvec == (uint32_t)(CHUNK / 16)) {
        // full chunk: load -> exps -> store per vector (the compiler barrier
        // keeps the stores spread through the chunk instead of bunched)
#pragma unroll
        for (int j = 0; j < NV; ++j) {
          const uint4 vj = sv[lane + 32 * j];
          __stcs(dst + lane + 32 * j, GElem<T>::vec(vj, c2, nl2, s2));
          asm volatile("" ::: "memory");
        }
        rr.release(lane);
        continue;
      }
      uint4 v[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const uint32_t q = lane + 32 * j;
        v[j] = q < nvec ? sv[q] : make_uint4(0, 0, 0, 0);
      }
      rr.release(lane);
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        const uint32_t q = lane + 32 * j;
        if (q < nvec) __stcs(dst + q, zero ? make_uint4(0, 0, 0, 0) : GElem<T>::vec(v[j], c2, nl2, s2));
      }
    }
    __syncwarp();  // order the row's vector stores before the target fix-up
    if (lane == 0) GElem<T>::store(gp, y, gy);
  }
}

// Launch configurations (warps/CTA x stages x chunk bytes): the release library
// has the default; a tuning build (-DPRORL_TUNING) selects others with PRORL_K5_CONFIG.
template <typename T, int W, int ST, int CH>
int run_grad_cfg(const GradArgs& a, int n_sm, cudaStream_t st) {
  auto kern = k_grad<T, W, ST, CH>;
  constexpr size_t smem = (size_t)W * ST * CH + (size_t)W * ST * 8;
  static_assert(smem <= 227 * 1024, "shared memory budget");
  PRORL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::min<int64_t>((int64_t)n_sm, (a.n_rows + W - 1) / W);
  kern<<<grid, W * 32, smem, st>>>(a);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

int grad_config() {
  static int idx = [] {
    const char* e = tuning_env("PRORL_K5_CONFIG");
    if (!e) return 2;  // default: 12 warps x 4 stages (best of the sweep, scripts/k5_sweep.py)
    const char* names[] = {"w16s2c4096", "w16s3c4096", "w12s4c4096", "w8s6c4096", "w16s4c2048"};
    for (int i = 0; i < 5; ++i)
      if (std::strcmp(e, names[i]) == 0) return i;
    return 2;
  }();
  return idx;
}

template <typename T>
int run_grad(const GradArgs& a, int n_sm, cudaStream_t st) {
  switch (grad_config()) {
#ifdef PRORL_TUNING
    case 0: return run_grad_cfg<T, 16, 2, 4096>(a, n_sm, st);
    case 1: return run_grad_cfg<T, 16, 3, 4096>(a, n_sm, st);
    case 3: return run_grad_cfg<T, 8, 6, 4096>(a, n_sm, st);
    case 4: return run_grad_cfg<T, 16, 4, 2048>(a, n_sm, st);
#endif
    default: return run_grad_cfg<T, 12, 4, 4096>(a, n_sm, st);  // the default (index 2)
  }
}

}  // namespace

int launch_grad(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab, const int32_t* rows,
                const int32_t* targets, const float* logp, const float* old_lp, const double* adv,
                const int32_t* row_seq, const float* ref_lp, int64_t n_rows, float inv_temp,
                const prorl_loss_cfg* cfg, double n_global, void* grad, int64_t grad_stride, float* dlogp,
                cudaStream_t st) {
  if (dtype != PRORL_BF16 && dtype != PRORL_FP32) return fail(PRORL_E_SHAPE, "logits_grad: unknown dtype");
  if (vocab <= 0 || row_stride < vocab) return fail(PRORL_E_SHAPE, "logits_grad: need vocab > 0, row_stride >= vocab");
  if (grad_stride != row_stride)
    return fail(PRORL_E_SHAPE, "logits_grad: grad_stride must equal row_stride (in-place or same layout)");
  const int esz = dtype == PRORL_BF16 ? 2 : 4;
  const intptr_t delta = static_cast<const uint8_t*>(grad) - static_cast<const uint8_t*>(logits);
  if (reinterpret_cast<uintptr_t>(logits) % esz || (delta % 16) != 0)
    return fail(PRORL_E_SHAPE, "logits_grad: grad must have the logits' 16-byte alignment phase");
  if (!(inv_temp > 0.f) || !(n_global > 0.0)) return fail(PRORL_E_MALFORMED_REQUEST, "logits_grad: bad inv_temp/n_global");
  if (n_rows <= 0) return PRORL_OK;
  GradArgs a{};
  a.logits = static_cast<const uint8_t*>(logits);
  a.stride_bytes = row_stride * esz;
  a.vocab = vocab;
  a.rows = rows;
  a.grad = static_cast<uint8_t*>(grad);
  a.targets = targets;
  a.logp = logp;
  a.old_lp = old_lp;
  a.adv = adv;
  a.row_seq = row_seq;
  a.ref_lp = ref_lp;
  a.kl_coef = cfg->kl_coef;
  a.n_rows = n_rows;
  a.c = inv_temp * kLog2e;
  a.inv_temp = inv_temp;
  a.lo = 1.0f - cfg->eps_lo;
  a.hi = 1.0f + cfg->eps_hi;
  a.inv_n = (float)(1.0 / n_global);
  a.dlogp = dlogp;
  return dtype == PRORL_BF16 ? run_grad<__nv_bfloat16>(a, ctx->n_sm, st) : run_grad<float>(a, ctx->n_sm, st);
}

}  // namespace prorl
