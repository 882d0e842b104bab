// common.cuh — context, error plumbing and sm_100a PTX helpers shared by the
// hot-path kernels (pack / grpo / score / synth). Not part of the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cstdlib>
#include <string>

#include "prorl_hotpath.h"

namespace prorl {

// Device-side validation flags (prorl_ctx::d_err), raised by kernels and read
// by prorl_check_errors / prorl_score_host.
enum : int { ERR_TOKEN_RANGE = 0, ERR_TURN_ORDER = 1, ERR_TOKEN_COUNT = 2, ERR_N = 4 };

// Launch-configuration overrides for A/B runs. Only a tuning build
// (scripts/build_variant.sh tuning -DPRORL_TUNING, loaded through
// PRORL_HOTPATH_LIB) reads the PRORL_K*_ / PRORL_PDL variables and compiles the
// alternative kernel configurations; the release library (build.py) has one
// configuration per kernel and row-size class and ignores the environment.
inline const char* tuning_env(const char* name) {
#ifdef PRORL_TUNING
  return std::getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define PRORL_TRY_INTERNAL(call)   \
  do {                             \
    int s_ = (call);               \
    if (s_ != PRORL_OK) return s_; \
  } while (0)

#define PRORL_CUDA(call)                                      \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return ::prorl::cuda_fail(e_, #call); \
  } while (0)

// Programmatic dependent launch between consecutive streaming launches of one
// step (K2 / K7 micro-batches with no other work between them on the stream):
// a kernel calls pdl_allow_next() at entry so the next launch's CTAs may take
// SMs as its own CTAs exit (hiding the launch gap and the straggler tail), and
// pdl_wait() before it touches anything the previous launch wrote (the slab
// rows). Both are no-ops for a normally launched kernel.
__device__ __forceinline__ void pdl_allow_next() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Launch `kern` (grid x block, dynamic smem) on `st`, with the programmatic
// stream-serialization attribute when `pdl` is set.
template <typename Kern, typename... Args>
int launch_maybe_pdl(Kern kern, int grid, int block, size_t smem, bool pdl, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  PRORL_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
  return PRORL_OK;
}

// Growable device scratch owned by a ctx.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t want = n + n / 4 + 256;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// Launch geometry of the scoring kernel (K2 / K2+K4).
struct ScoreGeom {
  int blocks = 0;  // persistent grid
  int warps = 0;   // warps per CTA
};

}  // namespace prorl

struct prorl_ctx {
  int device = 0;
  int n_sm = 0;
  int* d_err = nullptr;  // [prorl::ERR_N]
  prorl::DevBuf scan_tmp, pack_tmp, slab, grpo_tmp;
  // prorl_score_host staging (device copies of the host SoA + packed outputs)
  prorl::DevBuf h_turns, h_ids, h_lp, h_reward, h_usable, h_goff;
  prorl::DevBuf p_tokens, p_mask, p_turn, p_seq, p_pos, p_cu, p_oldlp;
  prorl::DevBuf a_row, a_target, a_oldlp, a_seq, a_turn, a_nact;
  prorl::DevBuf adv, informative, partials, logp, entropy, h_rkey, row_keys, lm_part, lm_pace;
  prorl::DevBuf k7rows;  // K7 row-end handoff (per-row fp64 warp partials), see train.cu k_train_rows
  void* nccl_comm = nullptr;  // ncclComm_t
  int nranks = 1, rank = 0;
  cudaEvent_t ev[8] = {};
  // prorl_score_host's chunked H2D of the token SoA (overlaps the scoring launches)
  static constexpr int kMaxChunks = 8;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t chunk_ev[kMaxChunks + 1] = {};  // [0]: the call's start on the caller's stream
  prorl_step_info last_step{};
};

namespace prorl {

// ---- internal launchers (defined in the .cu files) --------------------------
int launch_pack(prorl_ctx* ctx, const prorl_turn_desc* turns, int64_t n_turns, const int64_t* ids,
                const double* lp, int64_t n_tokens, int32_t n_seq, int32_t vocab,
                const prorl_packed* out, cudaStream_t st);
// K1 in two phases: the turn scan (cu_seqlens; needs only the descriptors),
// then the token pass over packed tokens [p0, p1) — a whole number of
// sequences whose active rows start at a0 — so chunks can be packed as their
// host data arrives. launch_pack = turns + tokens(0, n_tokens, 0, last).
int launch_pack_turns(prorl_ctx* ctx, const prorl_turn_desc* turns, int64_t n_turns, int64_t n_tokens, int32_t n_seq,
                      int32_t vocab, const prorl_packed* out, cudaStream_t st);
int launch_pack_tokens(prorl_ctx* ctx, const prorl_turn_desc* turns, int64_t n_turns, const int64_t* ids,
                       const double* lp, int64_t n_tokens, int32_t n_seq, int32_t vocab, const prorl_packed* out,
                       int64_t p0, int64_t p1, int64_t a0, bool last, cudaStream_t st);
int launch_grpo(prorl_ctx* ctx, const double* reward, const uint8_t* usable, const int32_t* group_off,
                int32_t n_groups, int32_t ddof, float eps, double tol, double* adv, uint8_t* informative,
                double* partials, cudaStream_t st);
// Scoring: if `cfg` is null, K2 only (logp/entropy). Otherwise the fused loss
// epilogue accumulates into slab rows [blockIdx] (accumulate=true adds to the
// existing slab content). Returns the number of slab rows used via *slab_rows.
int launch_score(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab,
                 const int32_t* rows, const int32_t* targets, const float* old_lp, const double* adv,
                 const int32_t* row_seq, const int16_t* row_turn, const float* ref_lp, int64_t n_rows,
                 float inv_temp, const prorl_loss_cfg* cfg, float* logp, float* entropy, double* slab, int slab_rows,
                 bool accumulate, int* rows_used, cudaStream_t st, bool pdl = false);
int launch_loss(prorl_ctx* ctx, const float* logp, const float* entropy, const float* old_lp,
                const double* adv, const int32_t* row_seq, const int16_t* row_turn, const float* ref_lp,
                int64_t n_rows, const prorl_loss_cfg* cfg, double* slab, int slab_rows, int* rows_used,
                cudaStream_t st);
int launch_grad(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab, const int32_t* rows,
                const int32_t* targets, const float* logp, const float* old_lp, const double* adv,
                const int32_t* row_seq, const float* ref_lp, int64_t n_rows, float inv_temp,
                const prorl_loss_cfg* cfg, double n_global,
                void* grad, int64_t grad_stride, float* dlogp, cudaStream_t st);
// K7 (train.cu): one-pass logprob/entropy + loss epilogue + dL/dlogits.
int train_slab_rows(prorl_ctx* ctx);
int launch_train(prorl_ctx* ctx, const void* logits, int dtype, int64_t row_stride, int32_t vocab, const int32_t* rows,
                 const int32_t* targets, const float* old_lp, const double* adv, const int32_t* row_seq,
                 const int16_t* row_turn, const float* ref_lp, int64_t n_rows, float inv_temp,
                 const prorl_loss_cfg* cfg, double n_global, float* logp, float* entropy, float* dlogp, void* grad,
                 double* slab, bool accumulate, int* rows_used, cudaStream_t st);
int launch_lmhead(prorl_ctx* ctx, const void* hidden, int64_t h_stride, const void* weight, int64_t w_stride,
                  int32_t d, int32_t vocab, const int32_t* targets, int64_t n_rows, float inv_temp, float* logp,
                  float* entropy, cudaStream_t st);
int launch_slab_reduce(const double* slab, int slab_rows, double* partials, cudaStream_t st);
int launch_gen_logits(void* logits, int dtype, int64_t row_stride, int32_t vocab, int64_t n_rows,
                      int64_t row_key0, const int64_t* row_keys, const int32_t* targets, const float* old_lp, uint64_t seed,
                      float scale, float base, int n_sm, cudaStream_t st);
int launch_row_keys(const int32_t* act_row, const int32_t* act_seq, const int32_t* cu_seqlens,
                    const int64_t* rollout_key, int64_t n, int64_t* keys, cudaStream_t st);
const char* score_config_name();     // active K2 launch configuration
int score_slab_rows(prorl_ctx* ctx);  // slab rows the scoring kernel uses (= its grid)
int loss_slab_rows(prorl_ctx* ctx);

}  // namespace prorl

// ---- device helpers -------------------------------------------------------------
#if defined(__CUDACC__)
namespace prorl {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Non-blocking probe of the phase with `parity` (mbarrier.test_wait).
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 1-D bulk async copy global -> shared (TMA engine, UBLKCP in SASS), completing
// `bytes` of transaction count on `bar`. dst/src 16-B aligned, bytes % 16 == 0.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void raise_flag(int* err, int which) { atomicOr(err + which, 1); }

}  // namespace prorl
#endif
