// synth.cu — deterministic synthetic LM-head output (stand-in for the model
// forward, out of the reference's scope: SPEC.md:8). The value of every
// element is defined in include/prorl_synth.h and is bit-identical to the CPU
// oracle's oracle_gen_logits. Not on the timed path of the benchmark.
#include "common.cuh"
#include "prorl_synth.h"

namespace prorl {

namespace {

template <bool BF16>
__global__ void k_gen_logits(uint8_t* __restrict__ out, int64_t row_stride, int32_t vocab, int64_t n_rows,
                             int64_t row_key0, const int64_t* __restrict__ row_keys,
                             const int32_t* __restrict__ targets,
                             const float* __restrict__ old_lp, uint32_t s0, float scale, float base) {
  // one CTA per row (grid-strided), threads across the vocabulary: no 64-bit division
  for (int64_t i = blockIdx.x; i < n_rows; i += gridDim.x) {
    const uint64_t row_key = row_keys ? (uint64_t)row_keys[i] : (uint64_t)(row_key0 + i);
    const int32_t tgt = old_lp != nullptr ? targets[i] : -1;
    const float plant = old_lp != nullptr ? prorl_plant_logit(row_key, s0, base, old_lp[i]) : 0.f;
    const uint64_t key0 = row_key * (uint64_t)vocab;
    for (int32_t col = threadIdx.x; col < vocab; col += blockDim.x) {
      const float x = col == tgt ? plant : prorl_noise_logit(key0 + (uint64_t)col, s0, scale);
      const int64_t o = i * row_stride + col;
      if (BF16) {
        reinterpret_cast<uint16_t*>(out)[o] = prorl_f32_to_bf16_bits(x);
      } else {
        reinterpret_cast<float*>(out)[o] = x;
      }
    }
  }
}

}  // namespace

int launch_gen_logits(void* logits, int dtype, int64_t row_stride, int32_t vocab, int64_t n_rows, int64_t row_key0,
                      const int64_t* row_keys, const int32_t* targets, const float* old_lp, uint64_t seed, float scale, float base, int n_sm,
                      cudaStream_t st) {
  if (dtype != PRORL_BF16 && dtype != PRORL_FP32) return fail(PRORL_E_SHAPE, "gen_logits: unknown dtype");
  if (vocab <= 0 || row_stride < vocab || n_rows < 0) return fail(PRORL_E_SHAPE, "gen_logits: bad shape");
  if (old_lp && !targets) return fail(PRORL_E_SHAPE, "gen_logits: old_lp given without targets");
  if (n_rows == 0) return PRORL_OK;
  const uint32_t s0 = prorl_seed_mix(seed);
  const int grid = n_sm * 8;
  if (dtype == PRORL_BF16)
    k_gen_logits<true><<<grid, 512, 0, st>>>(static_cast<uint8_t*>(logits), row_stride, vocab, n_rows, row_key0,
                                             row_keys, targets, old_lp, s0, scale, base);
  else
    k_gen_logits<false><<<grid, 512, 0, st>>>(static_cast<uint8_t*>(logits), row_stride, vocab, n_rows, row_key0,
                                              row_keys, targets, old_lp, s0, scale, base);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

// Synthetic-logits key of active row i: rollout_key[s] * 2^20 + (row - cu[s]).
__global__ void k_row_keys(const int32_t* __restrict__ act_row, const int32_t* __restrict__ act_seq,
                           const int32_t* __restrict__ cu_seqlens, const int64_t* __restrict__ rollout_key, int64_t n,
                           int64_t* __restrict__ keys) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t s = act_seq[i];
  const int64_t rk = rollout_key ? rollout_key[s] : (int64_t)s;
  keys[i] = rk * (int64_t(1) << 20) + (int64_t)(act_row[i] - cu_seqlens[s]);
}

int launch_row_keys(const int32_t* act_row, const int32_t* act_seq, const int32_t* cu_seqlens,
                    const int64_t* rollout_key, int64_t n, int64_t* keys, cudaStream_t st) {
  if (n <= 0) return PRORL_OK;
  k_row_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(act_row, act_seq, cu_seqlens, rollout_key, n, keys);
  PRORL_CUDA(cudaGetLastError());
  return PRORL_OK;
}

}  // namespace prorl
