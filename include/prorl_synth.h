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
 *   RN(RN(base + L) + g(L)),  L = min(RN(old_lp + (u * 0.5 - 0.25)), -2^-4),
 *   u = (mix32(lo32(row_key) ^ mix32(hi32(row_key) ^ s0 ^ 0xa5a5a5a5)) >> 8) * 2^-24,
 *   base = fp32(ln V + 4 ln(sinh(h)/h)), h = sigma*sqrt(3)/2 (the exact log
 *   mean of e^noise: four uniforms on [-h, h]), g(L) = -ln(1 - e^L)
 * so the noise sums to ~e^base and the target's own term to e^base e^L/(1-e^L):
 * logp ~ old_lp + U(-0.25, 0.25) with no bias (|mean| < 0.01 at V = 151936),
 * and a few per cent of the tokens clip (eps 0.2 / 0.28), as in a policy a few
 * updates from its rollout policy. g is evaluated with explicit single-rounded operations (no libm
 * exp/log), so the GPU generator and the oracle plant bit-identical logits.
 */
#ifndef PRORL_SYNTH_H
#define PRORL_SYNTH_H

#include <math.h>
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
#define PRORL_FDIV(a, b) __fdiv_rn((a), (b))
#else
#define PRORL_FMUL(a, b) ((a) * (b))
#define PRORL_FADD(a, b) ((a) + (b))
#define PRORL_FSUB(a, b) ((a) - (b))
#define PRORL_FDIV(a, b) ((a) / (b))
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

/* g(L) = -ln(1 - e^L) for L in [-16, -2^-4]: e^L = 2^k 2^f (degree-7
 * Taylor of 2^f), ln q = e ln2 + 2 atanh((m-1)/(m+1)) (q = m 2^e, m in
 * [0.5, 1), series to t^9). ~1e-6 accurate; only +, *, / and exact
 * floor / frexp / ldexp, each singly rounded. */
PRORL_HD float prorl_neg_log1mexp(float L) {
  const float y = PRORL_FMUL(L, 1.44269504f);
  const float k = floorf(y);
  const float f = PRORL_FMUL(PRORL_FSUB(y, k), 0.693147182f);
  float p = 1.98412701e-04f; /* 1/7! .. 1/0! */
  p = PRORL_FADD(PRORL_FMUL(p, f), 1.38888892e-03f);
  p = PRORL_FADD(PRORL_FMUL(p, f), 8.33333377e-03f);
  p = PRORL_FADD(PRORL_FMUL(p, f), 4.16666679e-02f);
  p = PRORL_FADD(PRORL_FMUL(p, f), 1.66666672e-01f);
  p = PRORL_FADD(PRORL_FMUL(p, f), 0.5f);
  p = PRORL_FADD(PRORL_FMUL(p, f), 1.0f);
  p = PRORL_FADD(PRORL_FMUL(p, f), 1.0f);
  const float q = PRORL_FSUB(1.0f, ldexpf(p, (int)k));
  int e;
  const float m = frexpf(q, &e);
  const float t = PRORL_FDIV(PRORL_FSUB(m, 1.0f), PRORL_FADD(m, 1.0f));
  const float t2 = PRORL_FMUL(t, t);
  float s = 1.11111112e-01f; /* 1/9, 1/7, 1/5, 1/3, 1 */
  s = PRORL_FADD(PRORL_FMUL(s, t2), 1.42857149e-01f);
  s = PRORL_FADD(PRORL_FMUL(s, t2), 0.2f);
  s = PRORL_FADD(PRORL_FMUL(s, t2), 3.33333343e-01f);
  s = PRORL_FADD(PRORL_FMUL(s, t2), 1.0f);
  const float lnq = PRORL_FADD(PRORL_FMUL((float)e, 0.693147182f), PRORL_FMUL(PRORL_FMUL(2.0f, t), s));
  return -lnq;
}

/* Planted target logit for row `row_key`. */
PRORL_HD float prorl_plant_logit(uint64_t row_key, uint32_t s0, float base, float old_lp) {
  uint32_t h = prorl_mix32((uint32_t)row_key ^ prorl_mix32((uint32_t)(row_key >> 32) ^ s0 ^ 0xa5a5a5a5U));
  float u = PRORL_FMUL((float)(h >> 8), 5.9604644775390625e-08f); /* exact, [0,1) */
  float delta = PRORL_FSUB(PRORL_FMUL(u, 0.5f), 0.25f);
  float L = PRORL_FADD(old_lp, delta);
  L = L > -0.0625f ? -0.0625f : (L < -16.0f ? -16.0f : L);
  return PRORL_FADD(PRORL_FADD(base, L), prorl_neg_log1mexp(L));
}

/* base: fp32 of ln V + the log mean of e^noise (host side). */
static inline float prorl_plant_base(int32_t vocab, float sigma) {
  const double h = (double)sigma * 0.8660254037844386; /* sigma*sqrt(3)/2 */
  const double lm = h > 0.0 ? 4.0 * log(sinh(h) / h) : 0.0;
  return (float)(log((double)vocab) + lm);
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
