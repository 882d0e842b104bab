// grpo.cu — K3: segmented GRPO group statistics.
//
// Extends the reference's group gate: PromptGroup::usable_rewards drops FAILED
// rollouts and is_informative is the DAPO zero-variance filter
// (proj/src/trainer/harness.cpp:84-102: < 2 usable -> false, else
// max - min > tolerance). On top of the gate this kernel computes the GRPO
// advantage over the usable rollouts of every informative group
// (SURVEY.md App. B.3):  A = (R - mean) / (std_ddof + eps), fp64 math and
// fp64 storage (the loss epilogue multiplies every token of a rollout by its
// A: an fp32-rounded A shifts a C2 loss sum by ~2e-6 relative). Non-usable
// rollouts and rollouts of non-informative groups get A = 0.
//
// One CTA, one warp per group (groups are small: 4..32 rollouts); the
// sum(A) / N_rollouts partials are reduced in a fixed order (deterministic).
#include "common.cuh"

namespace prorl {

namespace {

constexpr int kGrpoThreads = 1024;

__global__ void __launch_bounds__(kGrpoThreads)
    k_grpo(const double* __restrict__ reward, const uint8_t* __restrict__ usable,
           const int32_t* __restrict__ group_off, int32_t n_groups, int32_t ddof, float eps, double tol,
           double* __restrict__ adv, uint8_t* __restrict__ informative, double* partials) {
  __shared__ double s_sum[kGrpoThreads / 32];
  __shared__ double s_cnt[kGrpoThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc_a = 0.0, acc_n = 0.0;
  for (int32_t g = warp; g < n_groups; g += kGrpoThreads / 32) {
    const int32_t b = group_off[g], e = group_off[g + 1];
    double sum = 0.0, cnt = 0.0, mn = INFINITY, mx = -INFINITY;
    for (int32_t i = b + lane; i < e; i += 32) {
      if (usable[i]) {
        double r = reward[i];
        sum += r;
        cnt += 1.0;
        mn = fmin(mn, r);
        mx = fmax(mx, r);
      }
    }
    sum = warp_sum_d(sum);
    cnt = warp_sum_d(cnt);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    // exactly is_informative(tol) — the host gate (build_host_batch, ingest)
    // applies the same test, so both sides agree on which groups are packed;
    // ddof <= 1 (checked at launch) keeps cnt - ddof >= 1 for every such group
    const bool info = cnt >= 2.0 && (mx - mn) > tol;
    const double mean = cnt > 0.0 ? sum / cnt : 0.0;
    double ss = 0.0;
    for (int32_t i = b + lane; i < e; i += 32)
      if (usable[i]) {
        double d = reward[i] - mean;
        ss += d * d;
      }
    ss = warp_sum_d(ss);
    const double sd = info ? sqrt(ss / (cnt - (double)ddof)) : 0.0;
    double lsum = 0.0;
    for (int32_t i = b + lane; i < e; i += 32) {
      double a = 0.0;
      if (info && usable[i]) a = (reward[i] - mean) / (sd + (double)eps);
      adv[i] = a;
      lsum += a;
    }
    lsum = warp_sum_d(lsum);
    if (lane == 0) informative[g] = info ? 1 : 0;
    if (info) {
      acc_a += lsum;
      acc_n += cnt;
    }
  }
  if (lane == 0) {
    s_sum[warp] = acc_a;
    s_cnt[warp] = acc_n;
  }
  __syncthreads();
  if (threadIdx.x == 0 && partials != nullptr) {
    double a = 0.0, n = 0.0;
    for (int w = 0; w < kGrpoThreads / 32; ++w) {
      a += s_sum[w];
      n += s_cnt[w];
    }
    partials[PRORL_P_ADV_SUM] += a;
    partials[PRORL_P_N_ROLLOUTS] += n;
  }
}

}  // namespace

int launch_grpo(prorl_ctx* ctx, const double* reward, const uint8_t* usable, const int32_t* group_off,
                int32_t n_groups, int32_t ddof, float eps, double tol, double* adv, uint8_t* informative,
                double* partials, cudaStream_t st) {
  (void)ctx;
  if (n_groups < 0) return fail(PRORL_E_SHAPE, "prorl_grpo_adv: n_groups negative");
  // App. B.3 defines ddof 1 (torch.std) and 0; ddof >= 2 would leave an
  // informative group of ddof usable rollouts without a standard deviation
  if (ddof != 0 && ddof != 1) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_grpo_adv: ddof must be 0 or 1");
  if (!(tol >= 0.0)) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_grpo_adv: gate tolerance must be >= 0");
  if (n_groups == 0) return PRORL_OK;
  k_grpo<<<1, kGrpoThreads, 0, st>>>(reward, usable, group_off, n_groups, ddof, eps, tol, adv, informative,
                                      partials);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

}  // namespace prorl
