/*
 * prorl_synth.h — definition of the deterministic synthetic LM-head output
 * (the stand-in for the model forward, which is out of the reference's scope:
 * SPEC.md:8). Shared by the sm_100a generator (prorl_gen_logits) and the CPU
 * oracle (oracle_gen_logits) so both see bit-identical logits.
 *
 * Every float operation is written out explicitly (no contraction: the CUDA
 * side uses __fmul_rn/__fadd_rn, the C side is compiled -ffp-contract=off),
 * and all values that pass through a rounding are exact or singly rounded.
 *
 *   key      = row_key * V + col                       (uint64)
 *   h1       = mix32(lo32(key) ^ mix32(hi32(key) ^ s0)) s0 = prorl_seed_mix(seed)
 *   h2       = mix32(h1 ^ 0x85ebca6b)
 *   s        = (h1>>16) + (h1&0xffff) + (h2>>16) + (h2&0xffff)   (exact int)
 *   x        = RN( (s * 2^-16 - 2) * scale )            scale = fp32(sigma*sqrt(3))
 *   logit    = RN_bf16(x)  (or x for fp32 logits)
 * Planted target: logits[row][target] =
 *   RN((base + old_lp) + (u * 0.8 - 0.4))  base = fp32(ln V + sigma^2/2),
 *   u = (mix32(lo32(row_key) ^ mix32(hi32(row_key) ^ s0 ^ 0xa5a5a5a5)) >> 8) * 2^-24
 * so logp ~ old_lp + U(-0.4, 0.4) and the clip fractions are realistic.
 */
#ifndef PRORL_SYNTH_H
#define PRORL_SYNTH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define PRORL_HD __host__ __device__ __forceinline__
#else
#define PRORL_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define PRORL_FMUL(a, b) __fmul_rn((a), (b))
#define PRORL_FADD(a, b) __fadd_rn((a), (b))
#define PRORL_FSUB(a, b) __fsub_rn((a), (b))
#else
#define PRORL_FMUL(a, b) ((a) * (b))
#define PRORL_FADD(a, b) ((a) + (b))
#define PRORL_FSUB(a, b) ((a) - (b))
#endif

PRORL_HD uint32_t prorl_mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

PRORL_HD uint32_t prorl_seed_mix(uint64_t seed) {
  return prorl_mix32((uint32_t)seed ^ 0x9e3779b9U) ^ (uint32_t)(seed >> 32);
}

/* Noise logit (fp32, before the bf16 rounding) for element `key`. */
PRORL_HD float prorl_noise_logit(uint64_t key, uint32_t s0, float scale) {
  uint32_t h1 = prorl_mix32((uint32_t)key ^ prorl_mix32((uint32_t)(key >> 32) ^ s0));
  uint32_t h2 = prorl_mix32(h1 ^ 0x85ebca6bU);
  uint32_t s = (h1 >> 16) + (h1 & 0xffffU) + (h2 >> 16) + (h2 & 0xffffU);
  float f = PRORL_FMUL((float)s, 1.52587890625e-05f); /* exact: s < 2^18, * 2^-16 */
  f = PRORL_FSUB(f, 2.0f);                            /* exact */
  return PRORL_FMUL(f, scale);                        /* single rounding */
}

/* Planted target logit for row `row_key`. */
PRORL_HD float prorl_plant_logit(uint64_t row_key, uint32_t s0, float base, float old_lp) {
  uint32_t h = prorl_mix32((uint32_t)row_key ^ prorl_mix32((uint32_t)(row_key >> 32) ^ s0 ^ 0xa5a5a5a5U));
  float u = PRORL_FMUL((float)(h >> 8), 5.9604644775390625e-08f); /* exact, [0,1) */
  float delta = PRORL_FSUB(PRORL_FMUL(u, 0.8f), 0.4f);
  return PRORL_FADD(PRORL_FADD(base, old_lp), delta);
}

/* fp32 -> bf16 bits, round to nearest even (inputs here are finite). */
PRORL_HD uint16_t prorl_f32_to_bf16_bits(float f) {
  union { float f; uint32_t u; } v;
  v.f = f;
  uint32_t lsb = (v.u >> 16) & 1U;
  uint32_t r = v.u + 0x7fffU + lsb;
  return (uint16_t)(r >> 16);
}

PRORL_HD float prorl_bf16_bits_to_f32(uint16_t b) {
  union { float f; uint32_t u; } v;
  v.u = ((uint32_t)b) << 16;
  return v.f;
}

#endif /* PRORL_SYNTH_H */
