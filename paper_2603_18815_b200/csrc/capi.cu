// capi.cu — the extern "C" boundary declared in include/prorl_hotpath.h:
// context/error plumbing, thin validated wrappers over the kernels, the NCCL
// partials all-reduce, deterministic LPT group sharding, and prorl_score_host
// (the whole per-GPU step from host buffers — the seam where the reference
// drops the trajectory today, proj/src/trainer/harness.cpp:263-273).
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "common.cuh"
#include "prorl_synth.h"

namespace prorl {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string("cuda_error: ") + cudaGetErrorString(e) + " in " + what;
  return PRORL_E_CUDA;
}

// NCCL is resolved at run time from whichever libnccl.so.2 the process has
// (torch brings its own); linking one at build time would clash with it.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool ok = false;
};

static const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce && a.error_string;
    return a;
  }();
  return api;
}

static int nccl_fail(ncclResult_t r, const char* what) {
  g_last_error = std::string("nccl_error: ") + (nccl().error_string ? nccl().error_string(r) : "?") + " in " + what;
  return PRORL_E_NCCL;
}

#define PRORL_NCCL_API()                                                                         \
  do {                                                                                           \
    if (!::prorl::nccl().ok) return ::prorl::fail(PRORL_E_NCCL, "nccl_error: libnccl.so.2 not loadable"); \
  } while (0)

#define PRORL_NCCL(call)                                   \
  do {                                                     \
    ncclResult_t r_ = (call);                              \
    if (r_ != ncclSuccess) return ::prorl::nccl_fail(r_, #call); \
  } while (0)

// Programmatic dependent launch between micro-batch launches: on; a tuning
// build turns it off with PRORL_PDL=0 (A/B).
static bool pdl_enabled() {
  static const bool on = [] {
    const char* e = tuning_env("PRORL_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

#define PRORL_TRY(call)            \
  do {                             \
    int s_ = (call);               \
    if (s_ != PRORL_OK) return s_; \
  } while (0)

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// NVTX range for profilers (nsys / ncu --nvtx); header-only, no-op without a tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Host-side count of active rows: a policy token at position > 0 of its
// sequence makes the previous row active.
static int64_t host_active_rows(const prorl_turn_desc* turns, int64_t n_turns) {
  int64_t n = 0;
  int32_t cur = -1;
  int64_t pos = 0;
  for (int64_t t = 0; t < n_turns; ++t) {
    if (turns[t].traj != cur) {
      cur = turns[t].traj;
      pos = 0;
    }
    if (turns[t].role == PRORL_ROLE_ASSISTANT && turns[t].len > 0) n += turns[t].len - (pos == 0 ? 1 : 0);
    pos += turns[t].len;
  }
  return n;
}

// prorl_score_host's H2D chunks: packed tokens [p0, p1) (whole sequences),
// their active rows [a0, a1), and the host SoA range [s0, s1) they read.
struct PackChunk {
  int64_t p0, p1, a0, a1, s0, s1;
};

// Split the turn list at sequence starts into at most max_chunks chunks of
// doubling size, the first holding about one micro-batch of active rows (it is
// the only copy the scoring waits for). Falls back to one chunk covering the
// whole SoA when the chunks' source ranges overlap by more than 1/8 of it
// (turns that do not read the SoA in order).
static int plan_chunks(const prorl_turn_desc* turns, int64_t n_turns, int64_t n_tokens, int64_t n_active,
                       int64_t mb_rows, int max_chunks, PackChunk* out) {
  out[0] = PackChunk{0, n_tokens, 0, n_active, 0, n_tokens};
  if (max_chunks < 2 || n_active <= mb_rows) return 1;
  int64_t target = std::max<int64_t>(
      {n_tokens / 64, 1, (int64_t)((double)mb_rows * (double)n_tokens / (double)n_active)});
  int n = 0;
  PackChunk cur{0, 0, 0, 0, INT64_MAX, 0};
  int64_t p = 0, a = 0, pos = 0, copied = 0;
  int32_t traj = -1;
  for (int64_t t = 0; t < n_turns; ++t) {
    const prorl_turn_desc& d = turns[t];
    if (d.traj != traj) {  // a sequence starts at packed token p
      if (p - cur.p0 >= target && n < max_chunks - 1) {
        cur.p1 = p;
        cur.a1 = a;
        if (cur.s0 > cur.s1) cur.s0 = cur.s1 = 0;
        copied += cur.s1 - cur.s0;
        out[n++] = cur;
        cur = PackChunk{p, p, a, a, INT64_MAX, 0};
        target *= 2;
      }
      traj = d.traj;
      pos = 0;
    }
    if (d.len > 0) {
      cur.s0 = std::min(cur.s0, d.src_off);
      cur.s1 = std::max(cur.s1, d.src_off + d.len);
      if (d.role == PRORL_ROLE_ASSISTANT) a += d.len - (pos == 0 ? 1 : 0);
    }
    pos += d.len;
    p += d.len;
  }
  cur.p1 = p;
  cur.a1 = a;
  if (cur.s0 > cur.s1) cur.s0 = cur.s1 = 0;
  copied += cur.s1 - cur.s0;
  out[n++] = cur;
  if (n < 2 || copied > n_tokens + n_tokens / 8) {
    out[0] = PackChunk{0, n_tokens, 0, n_active, 0, n_tokens};
    return 1;
  }
  return n;
}

}  // namespace prorl

using namespace prorl;

// ABI layout guards (mirrored by tests/test_abi.py against the ctypes structs)
static_assert(sizeof(prorl_turn_desc) == 24, "prorl_turn_desc layout");
static_assert(sizeof(prorl_packed) == 13 * 8, "prorl_packed layout");
static_assert(sizeof(prorl_loss_cfg) == 16, "prorl_loss_cfg layout");
static_assert(sizeof(prorl_score_cfg) == 48, "prorl_score_cfg layout");
static_assert(sizeof(prorl_host_batch) == 88, "prorl_host_batch layout");
static_assert(sizeof(prorl_logits_pool) == 144, "prorl_logits_pool layout");
static_assert(sizeof(prorl_ingest_result) == 112, "prorl_ingest_result layout");

extern "C" {

int prorl_abi_version(void) { return PRORL_ABI_VERSION; }

const char* prorl_kernel_config(void) { return score_config_name(); }

const char* prorl_last_error(void) { return g_last_error.c_str(); }

const char* prorl_status_code(int status) {
  switch (status) {
    case PRORL_OK: return "ok";
    case PRORL_E_MALFORMED_TURN: return "malformed_turn";
    case PRORL_E_INCOMPLETE_GROUP: return "incomplete_group";
    case PRORL_E_MALFORMED_REQUEST: return "malformed_request";
    case PRORL_E_CUDA: return "cuda_error";
    case PRORL_E_NCCL: return "nccl_error";
    case PRORL_E_SHAPE: return "shape_mismatch";
    case PRORL_E_TOKEN_RANGE: return "shape_mismatch";
    case PRORL_E_PEER_FAILED: return "peer_failed";
  }
  return "unknown";
}

int prorl_ctx_create(int device, prorl_ctx** out) {
  if (!out) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_ctx_create: out is null");
  *out = nullptr;
  PRORL_CUDA(cudaSetDevice(device));
  prorl_ctx* c = new prorl_ctx();
  c->device = device;
  cudaError_t e = cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_err, sizeof(int) * ERR_N);
  if (e == cudaSuccess) e = cudaMemset(c->d_err, 0, sizeof(int) * ERR_N);
  for (int i = 0; i < 8 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev[i]);
  for (int i = 0; i <= prorl_ctx::kMaxChunks && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(&c->chunk_ev[i], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    for (auto& ev : c->ev)
      if (ev) cudaEventDestroy(ev);
    for (auto& ev : c->chunk_ev)
      if (ev) cudaEventDestroy(ev);
    if (c->d_err) cudaFree(c->d_err);
    delete c;
    return cuda_fail(e, "prorl_ctx_create");
  }
  *out = c;
  return PRORL_OK;
}

int prorl_ctx_destroy(prorl_ctx* c) {
  if (!c) return PRORL_OK;
  cudaSetDevice(c->device);
  if (c->nccl_comm && nccl().ok) nccl().comm_destroy(static_cast<ncclComm_t>(c->nccl_comm));
  for (auto* b : {&c->scan_tmp, &c->pack_tmp, &c->slab, &c->grpo_tmp, &c->h_turns, &c->h_ids, &c->h_lp,
                  &c->h_reward, &c->h_usable, &c->h_goff, &c->p_tokens, &c->p_mask, &c->p_turn, &c->p_seq,
                  &c->p_pos, &c->p_cu, &c->p_oldlp, &c->a_row, &c->a_target, &c->a_oldlp, &c->a_seq, &c->a_turn,
                  &c->a_nact, &c->adv, &c->informative, &c->partials, &c->logp, &c->entropy, &c->h_rkey,
                  &c->row_keys, &c->lm_part, &c->lm_pace, &c->k7rows})
    b->release();
  for (auto& ev : c->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& ev : c->chunk_ev)
    if (ev) cudaEventDestroy(ev);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->d_err) cudaFree(c->d_err);
  delete c;
  return PRORL_OK;
}

int prorl_check_errors(prorl_ctx* c, void* stream) {
  if (!c) return fail(PRORL_E_MALFORMED_REQUEST, "null ctx");
  int h[ERR_N] = {0};
  PRORL_CUDA(cudaStreamSynchronize(S(stream)));
  PRORL_CUDA(cudaMemcpy(h, c->d_err, sizeof(h), cudaMemcpyDeviceToHost));
  PRORL_CUDA(cudaMemset(c->d_err, 0, sizeof(h)));
  if (h[ERR_TOKEN_RANGE]) return fail(PRORL_E_TOKEN_RANGE, "shape_mismatch: token id outside [0, vocab)");
  if (h[ERR_TURN_ORDER])
    return fail(PRORL_E_SHAPE, "shape_mismatch: turn descriptors not sorted by traj / traj outside [0, n_seq) / bad role");
  if (h[ERR_TOKEN_COUNT]) return fail(PRORL_E_SHAPE, "shape_mismatch: n_tokens != sum of turn lengths");
  return PRORL_OK;
}

int prorl_pack(prorl_ctx* c, const prorl_turn_desc* turns, int64_t n_turns, const int64_t* ids, const double* lp,
               int64_t n_tokens, int32_t n_seq, int32_t vocab, const prorl_packed* out, void* stream) {
  if (!c || !out) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_pack: null ctx/out");
  PRORL_CUDA(cudaSetDevice(c->device));
  return launch_pack(c, turns, n_turns, ids, lp, n_tokens, n_seq, vocab, out, S(stream));
}

int prorl_grpo_adv(prorl_ctx* c, const double* reward, const uint8_t* usable, const int32_t* group_off,
                   int32_t n_groups, int32_t ddof, float eps, double tolerance, double* adv, uint8_t* informative,
                   double* partials, void* stream) {
  if (!c) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_grpo_adv: null ctx");
  PRORL_CUDA(cudaSetDevice(c->device));
  return launch_grpo(c, reward, usable, group_off, n_groups, ddof, eps, tolerance, adv, informative, partials,
                     S(stream));
}

int prorl_logprob_entropy(prorl_ctx* c, const void* logits, int dtype, int64_t row_stride, int32_t vocab,
                          const int32_t* rows, const int32_t* targets, int64_t n_rows, float inv_temp, float* logp,
                          float* entropy, void* stream) {
  if (!c) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_logprob_entropy: null ctx");
  PRORL_CUDA(cudaSetDevice(c->device));
  return launch_score(c, logits, dtype, row_stride, vocab, rows, targets, nullptr, nullptr, nullptr, nullptr, nullptr,
                      n_rows, inv_temp, nullptr, logp, entropy, nullptr, 0, false, nullptr, S(stream));
}

int prorl_clipped_loss(prorl_ctx* c, const float* logp, const float* entropy, const float* old_lp, const double* adv,
                       const int32_t* row_seq, const int16_t* row_turn, const float* ref_lp, int64_t n_rows,
                       const prorl_loss_cfg* cfg, double* partials_dev, void* stream) {
  if (!c || !cfg) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_clipped_loss: null ctx/cfg");
  PRORL_CUDA(cudaSetDevice(c->device));
  const int rows = loss_slab_rows(c);
  PRORL_CUDA(c->slab.ensure(sizeof(double) * PRORL_N_PARTIALS * (size_t)std::max(rows, score_slab_rows(c))));
  int used = 0;
  PRORL_TRY(launch_loss(c, logp, entropy, old_lp, adv, row_seq, row_turn, ref_lp, n_rows, cfg, c->slab.as<double>(),
                        rows, &used, S(stream)));
  return launch_slab_reduce(c->slab.as<double>(), used, partials_dev, S(stream));
}

int prorl_score_rows(prorl_ctx* c, const void* logits, int dtype, int64_t row_stride, int32_t vocab,
                     const int32_t* rows, const int32_t* targets, const float* old_lp, const double* adv,
                     const int32_t* row_seq, const int16_t* row_turn, const float* ref_lp, int64_t n_rows,
                     float inv_temp, const prorl_loss_cfg* cfg, float* logp, float* entropy, double* partials_dev,
                     void* stream) {
  if (!c || !cfg) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_rows: null ctx/cfg");
  PRORL_CUDA(cudaSetDevice(c->device));
  const int srows = score_slab_rows(c);
  PRORL_CUDA(c->slab.ensure(sizeof(double) * PRORL_N_PARTIALS * (size_t)std::max(srows, loss_slab_rows(c))));
  int used = 0;
  PRORL_TRY(launch_score(c, logits, dtype, row_stride, vocab, rows, targets, old_lp, adv, row_seq, row_turn, ref_lp,
                         n_rows, inv_temp, cfg, logp, entropy, c->slab.as<double>(), srows, false, &used, S(stream)));
  return launch_slab_reduce(c->slab.as<double>(), used, partials_dev, S(stream));
}

int prorl_logits_grad(prorl_ctx* c, const void* logits, int dtype, int64_t row_stride, int32_t vocab,
                      const int32_t* rows, const int32_t* targets, const float* logp, const float* old_lp,
                      const double* adv, const int32_t* row_seq, const float* ref_lp, int64_t n_rows, float inv_temp,
                      const prorl_loss_cfg* cfg, double n_global, void* grad, int64_t grad_stride, float* dlogp,
                      void* stream) {
  if (!c || !cfg) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_logits_grad: null ctx/cfg");
  PRORL_CUDA(cudaSetDevice(c->device));
  return launch_grad(c, logits, dtype, row_stride, vocab, rows, targets, logp, old_lp, adv, row_seq, ref_lp, n_rows,
                     inv_temp, cfg, n_global, grad, grad_stride, dlogp, S(stream));
}

int prorl_score_grad(prorl_ctx* c, const void* logits, int dtype, int64_t row_stride, int32_t vocab,
                     const int32_t* rows, const int32_t* targets, const float* old_lp, const double* adv,
                     const int32_t* row_seq, const int16_t* row_turn, const float* ref_lp, int64_t n_rows,
                     float inv_temp, const prorl_loss_cfg* cfg, double n_global, float* logp, float* entropy,
                     double* partials_dev, void* grad, int64_t grad_stride, float* dlogp, void* stream) {
  if (!c || !cfg) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_grad: null ctx/cfg");
  if (dtype != PRORL_BF16 && dtype != PRORL_FP32) return fail(PRORL_E_SHAPE, "score_grad: unknown dtype");
  if (vocab <= 0 || row_stride < vocab) return fail(PRORL_E_SHAPE, "score_grad: need vocab > 0, row_stride >= vocab");
  if (grad_stride != row_stride)
    return fail(PRORL_E_SHAPE, "score_grad: grad_stride must equal row_stride (in-place or same layout)");
  if (!(inv_temp > 0.f) || !(n_global > 0.0)) return fail(PRORL_E_MALFORMED_REQUEST, "score_grad: bad inv_temp/n_global");
  if (cfg->n_buckets < 1 || cfg->n_buckets > PRORL_TURN_BUCKETS)
    return fail(PRORL_E_SHAPE, "score_grad: n_buckets out of [1, 64]");
  if (n_rows <= 0) return PRORL_OK;
  if (!logits || !grad || !targets || !old_lp || !adv || !row_seq || !row_turn)
    return fail(PRORL_E_MALFORMED_REQUEST, "score_grad: null logits/grad/targets/old_lp/adv/row_seq/row_turn");
  const int esz = dtype == PRORL_BF16 ? 2 : 4;
  const intptr_t delta = static_cast<const uint8_t*>(grad) - static_cast<const uint8_t*>(logits);
  if (reinterpret_cast<uintptr_t>(logits) % esz || (delta % 16) != 0)
    return fail(PRORL_E_SHAPE, "score_grad: grad must have the logits' 16-byte alignment phase");
  PRORL_CUDA(cudaSetDevice(c->device));
  const int slab_rows = train_slab_rows(c);
  PRORL_CUDA(c->slab.ensure(sizeof(double) * PRORL_N_PARTIALS * (size_t)std::max(slab_rows, loss_slab_rows(c))));
  int used = 0;
  PRORL_TRY(launch_train(c, logits, dtype, row_stride, vocab, rows, targets, old_lp, adv, row_seq, row_turn, ref_lp,
                         n_rows, inv_temp, cfg, n_global, logp, entropy, dlogp, grad, c->slab.as<double>(), false,
                         &used, S(stream)));
  return launch_slab_reduce(c->slab.as<double>(), used, partials_dev, S(stream));
}

int prorl_lmhead_logprob(prorl_ctx* c, const void* hidden, int64_t h_stride, const void* weight, int64_t w_stride,
                         int32_t d, int32_t vocab, const int32_t* targets, int64_t n_rows, float inv_temp,
                         float* logp, float* entropy, void* stream) {
  if (!c) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_lmhead_logprob: null ctx");
  PRORL_CUDA(cudaSetDevice(c->device));
  return launch_lmhead(c, hidden, h_stride, weight, w_stride, d, vocab, targets, n_rows, inv_temp, logp, entropy,
                       S(stream));
}

int prorl_nccl_unique_id(uint8_t* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  PRORL_NCCL_API();
  ncclUniqueId id;
  PRORL_NCCL(nccl().get_unique_id(&id));
  std::memcpy(id128, &id, sizeof(id));
  return PRORL_OK;
}

int prorl_nccl_init(prorl_ctx* c, int nranks, int rank, const uint8_t* id128) {
  if (!c || nranks < 1 || rank < 0 || rank >= nranks) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_nccl_init: bad args");
  PRORL_NCCL_API();
  PRORL_CUDA(cudaSetDevice(c->device));
  if (c->nccl_comm) {
    nccl().comm_destroy(static_cast<ncclComm_t>(c->nccl_comm));
    c->nccl_comm = nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t comm;
  PRORL_NCCL(nccl().comm_init_rank(&comm, nranks, id, rank));
  c->nccl_comm = comm;
  c->nranks = nranks;
  c->rank = rank;
  return PRORL_OK;
}

int prorl_allreduce(prorl_ctx* c, double* partials_dev, int n, void* stream) {
  if (!c) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_allreduce: null ctx");
  if (!c->nccl_comm || n <= 0) return PRORL_OK;  // a 1-rank communicator still runs (tests the NCCL plumbing)
  PRORL_CUDA(cudaSetDevice(c->device));
  PRORL_NCCL(nccl().all_reduce(partials_dev, partials_dev, (size_t)n, ncclDouble, ncclSum,
                           static_cast<ncclComm_t>(c->nccl_comm), S(stream)));
  return PRORL_OK;
}

int prorl_gen_logits(prorl_ctx* c, void* logits, int dtype, int64_t row_stride, int32_t vocab, int64_t n_rows,
                     int64_t row_key0, const int32_t* targets, const float* old_lp, uint64_t seed, float sigma,
                     void* stream) {
  if (!c) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_gen_logits: null ctx");
  PRORL_CUDA(cudaSetDevice(c->device));
  const float scale = (float)((double)sigma * std::sqrt(3.0));
  const float base = prorl_plant_base(vocab, sigma);
  return launch_gen_logits(logits, dtype, row_stride, vocab, n_rows, row_key0, nullptr, targets, old_lp, seed, scale,
                           base, c->n_sm, S(stream));
}

int prorl_gen_logits_keyed(prorl_ctx* c, void* logits, int dtype, int64_t row_stride, int32_t vocab, int64_t n_rows,
                           const int64_t* row_keys, const int32_t* targets, const float* old_lp, uint64_t seed,
                           float sigma, void* stream) {
  if (!c || !row_keys) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_gen_logits_keyed: null ctx/row_keys");
  PRORL_CUDA(cudaSetDevice(c->device));
  const float scale = (float)((double)sigma * std::sqrt(3.0));
  const float base = prorl_plant_base(vocab, sigma);
  return launch_gen_logits(logits, dtype, row_stride, vocab, n_rows, 0, row_keys, targets, old_lp, seed, scale, base,
                           c->n_sm, S(stream));
}

int prorl_row_keys(prorl_ctx* c, const int32_t* rows, const int32_t* seq, const int32_t* cu_seqlens,
                   const int64_t* rollout_key, int64_t n, int64_t* keys, void* stream) {
  if (!c) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_row_keys: null ctx");
  PRORL_CUDA(cudaSetDevice(c->device));
  return launch_row_keys(rows, seq, cu_seqlens, rollout_key, n, keys, S(stream));
}

int prorl_shard_lpt(int32_t n_groups, const int64_t* load, int32_t world, int32_t* owner) {
  if (n_groups < 0 || world < 1 || (n_groups > 0 && (!load || !owner)))
    return fail(PRORL_E_MALFORMED_REQUEST, "prorl_shard_lpt: bad args");
  std::vector<int32_t> order(n_groups);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return load[a] > load[b]; });
  std::vector<int64_t> acc(world, 0);
  for (int32_t g : order) {
    int32_t best = 0;
    for (int32_t r = 1; r < world; ++r)
      if (acc[r] < acc[best]) best = r;
    owner[g] = best;
    acc[best] += load[g];
  }
  return PRORL_OK;
}

namespace {
// Folds the device-side validation flags of this step into the partials before
// the all-reduce, so a rank whose kernels rejected their input fails every rank.
__global__ void k_fold_errors(const int* __restrict__ err, double* __restrict__ partials) {
  int any = 0;
#pragma unroll
  for (int k = 0; k < prorl::ERR_N; ++k) any |= err[k];
  if (any) partials[PRORL_P_ERR_RANKS] += 1.0;
}

int score_host_impl(prorl_ctx* c, const prorl_host_batch* hb, const prorl_score_cfg* cfg,
                    const prorl_logits_pool* pool, double* host_partials, float* timings_ms, void* stream,
                    bool& reduced);
}  // namespace

int prorl_score_host(prorl_ctx* c, const prorl_host_batch* hb, const prorl_score_cfg* cfg,
                     const prorl_logits_pool* pool, double* host_partials, float* timings_ms, void* stream) {
  if (!c) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: null ctx");
  bool reduced = false;
  const int rc = score_host_impl(c, hb, cfg, pool, host_partials, timings_ms, stream, reduced);
  if (rc == PRORL_OK || reduced || !c->nccl_comm || c->nranks < 2) return rc;
  // This rank failed before its all-reduce: still take part in it, with zeros
  // and the failure flag, so the peers return PRORL_E_PEER_FAILED instead of
  // waiting forever. The original status and message are kept.
  const std::string msg = prorl_last_error();
  cudaStream_t st = S(stream);
  if (cudaSetDevice(c->device) == cudaSuccess && c->partials.ensure(sizeof(double) * PRORL_N_PARTIALS) == cudaSuccess) {
    double* d = c->partials.as<double>();
    double h[PRORL_N_PARTIALS];
    prorl_fail_partials(h);
    if (cudaMemcpyAsync(d, h, sizeof h, cudaMemcpyHostToDevice, st) == cudaSuccess)
      nccl().all_reduce(d, d, (size_t)PRORL_N_PARTIALS, ncclDouble, ncclSum, static_cast<ncclComm_t>(c->nccl_comm), st);
    cudaStreamSynchronize(st);
  }
  return fail(rc, msg);
}

int prorl_last_step_info(const prorl_ctx* c, prorl_step_info* out) {
  if (!c || !out) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_last_step_info: null argument");
  *out = c->last_step;
  return PRORL_OK;
}

void prorl_fail_partials(double* host_partials) {
  if (!host_partials) return;
  std::memset(host_partials, 0, sizeof(double) * PRORL_N_PARTIALS);
  host_partials[PRORL_P_ERR_RANKS] = 1.0;
}

int prorl_step_status(int local_status, const double* reduced) {
  if (local_status != PRORL_OK) return local_status;  // this rank's own failure wins (message already set)
  if (!reduced) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_step_status: null partials");
  if (reduced[PRORL_P_ERR_RANKS] > 0.0)
    return fail(PRORL_E_PEER_FAILED, "peer_failed: " + std::to_string((int)reduced[PRORL_P_ERR_RANKS]) +
                                         " rank(s) failed this step; the all-reduced partials are void");
  return PRORL_OK;
}

namespace {
int score_host_impl(prorl_ctx* c, const prorl_host_batch* hb, const prorl_score_cfg* cfg,
                    const prorl_logits_pool* pool, double* host_partials, float* timings_ms, void* stream,
                    bool& reduced) {
  if (!hb || !cfg || !pool || !host_partials)
    return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: null argument");
  const bool lmhead_mode = pool->provide_hidden != nullptr;
  if (!lmhead_mode && !pool->provide && (pool->n_pool < 1 || !pool->buffers))
    return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: empty logits pool");
  if (lmhead_mode && (!pool->weight || pool->d_model <= 0))
    return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: lm-head mode needs weight and d_model");
  if (cfg->microbatch_rows < 1) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: microbatch_rows < 1");
  const bool train_mode = pool->train != 0;
  if (cfg->loss.kl_coef != 0.f && !pool->provide_ref)
    return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: kl_coef != 0 needs provide_ref (reference logprobs)");
  if (train_mode && lmhead_mode)
    return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: training mode needs the logits path (no fused LM head)");
  // the gradient is normalised by n_global while the reported loss is the
  // all-reduced token mean: with several ranks only the caller knows the global count
  if (train_mode && !(pool->n_global > 0.0) && c->nranks > 1)
    return fail(PRORL_E_MALFORMED_REQUEST,
                "prorl_score_host: training with more than one rank needs n_global (the global active-row count)");
  // configuration, checked once before any device work (the launchers re-check their own arguments)
  if (cfg->dtype != PRORL_BF16 && cfg->dtype != PRORL_FP32) return fail(PRORL_E_SHAPE, "prorl_score_host: unknown dtype");
  if (cfg->vocab <= 0) return fail(PRORL_E_SHAPE, "prorl_score_host: vocab must be > 0");
  if (!(cfg->inv_temperature > 0.f)) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: inv_temperature must be > 0");
  if (cfg->loss.n_buckets < 1 || cfg->loss.n_buckets > PRORL_TURN_BUCKETS)
    return fail(PRORL_E_SHAPE, "prorl_score_host: n_buckets out of [1, 64]");
  if (cfg->ddof != 0 && cfg->ddof != 1) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: ddof must be 0 or 1");
  if (!(cfg->gate_tolerance >= 0.0)) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: gate_tolerance must be >= 0");
  if (!lmhead_mode && !pool->provide && pool->row_stride < cfg->vocab)
    return fail(PRORL_E_SHAPE, "prorl_score_host: pool row_stride < vocab");
  if (hb->n_groups < 0 || hb->n_rollouts < 0 || hb->n_turns < 0 || hb->n_tokens < 0)
    return fail(PRORL_E_SHAPE, "prorl_score_host: negative sizes");
  if ((hb->n_turns > 0 && !hb->turns) || (hb->n_tokens > 0 && (!hb->ids || !hb->lp)) ||
      (hb->n_rollouts > 0 && (!hb->reward || !hb->usable)) || (hb->n_groups > 0 && !hb->group_off))
    return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: null host array with a non-zero size");
  if (hb->n_groups > 0 && hb->group_off[hb->n_groups] != hb->n_rollouts)
    return fail(PRORL_E_SHAPE, "prorl_score_host: group_off[n_groups] != n_rollouts");
  // host-side validation of the descriptors (the device buffers are sized from
  // them, so inconsistent input must be rejected before any kernel runs)
  int64_t tok = 0;
  for (int64_t t = 0; t < hb->n_turns; ++t) {
    const prorl_turn_desc& d = hb->turns[t];
    if (d.traj < 0 || d.traj >= hb->n_rollouts || d.len < 0 || d.role > PRORL_ROLE_TOOL ||
        (t > 0 && d.traj < hb->turns[t - 1].traj) || d.src_off < 0 || d.src_off + d.len > hb->n_tokens)
      return fail(PRORL_E_SHAPE, "prorl_score_host: turn " + std::to_string(t) +
                                     " out of order / out of range (traj, len, role or src_off)");
    tok += d.len;
  }
  if (tok != hb->n_tokens) return fail(PRORL_E_SHAPE, "prorl_score_host: n_tokens != sum of turn lengths");
  for (int32_t g = 0; g < hb->n_groups; ++g)
    if (hb->group_off[g] < 0 || hb->group_off[g] > hb->group_off[g + 1])
      return fail(PRORL_E_SHAPE, "prorl_score_host: group_off not monotone in [0, n_rollouts]");
  PRORL_CUDA(cudaSetDevice(c->device));
  cudaStream_t st = S(stream);
  const int64_t N = hb->n_tokens, A = host_active_rows(hb->turns, hb->n_turns);
  const int32_t R = hb->n_rollouts, G = hb->n_groups;
  const int srows = score_slab_rows(c);

  // device staging (grown on demand, kept across calls)
  PRORL_CUDA(c->h_turns.ensure(sizeof(prorl_turn_desc) * (size_t)std::max<int64_t>(hb->n_turns, 1)));
  PRORL_CUDA(c->h_ids.ensure(sizeof(int64_t) * (size_t)std::max<int64_t>(N, 1)));
  PRORL_CUDA(c->h_lp.ensure(sizeof(double) * (size_t)std::max<int64_t>(N, 1)));
  PRORL_CUDA(c->h_reward.ensure(sizeof(double) * (size_t)std::max(R, 1)));
  PRORL_CUDA(c->h_usable.ensure((size_t)std::max(R, 1)));
  PRORL_CUDA(c->h_goff.ensure(sizeof(int32_t) * (size_t)(G + 1)));
  PRORL_CUDA(c->p_tokens.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(N, 1)));
  PRORL_CUDA(c->p_mask.ensure((size_t)std::max<int64_t>(N, 1)));
  PRORL_CUDA(c->p_turn.ensure(sizeof(int16_t) * (size_t)std::max<int64_t>(N, 1)));
  PRORL_CUDA(c->p_seq.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(N, 1)));
  PRORL_CUDA(c->p_pos.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(N, 1)));
  PRORL_CUDA(c->p_cu.ensure(sizeof(int32_t) * (size_t)(R + 1)));
  PRORL_CUDA(c->p_oldlp.ensure(sizeof(float) * (size_t)std::max<int64_t>(N, 1)));
  PRORL_CUDA(c->a_row.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(A, 1)));
  PRORL_CUDA(c->a_target.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(A, 1)));
  PRORL_CUDA(c->a_oldlp.ensure(sizeof(float) * (size_t)std::max<int64_t>(A, 1)));
  PRORL_CUDA(c->a_seq.ensure(sizeof(int32_t) * (size_t)std::max<int64_t>(A, 1)));
  PRORL_CUDA(c->a_turn.ensure(sizeof(int16_t) * (size_t)std::max<int64_t>(A, 1)));
  PRORL_CUDA(c->a_nact.ensure(sizeof(int64_t)));
  PRORL_CUDA(c->adv.ensure(sizeof(double) * (size_t)std::max(R, 1)));
  PRORL_CUDA(c->h_rkey.ensure(sizeof(int64_t) * (size_t)std::max(R, 1)));
  PRORL_CUDA(c->row_keys.ensure(sizeof(int64_t) * (size_t)std::max<int64_t>(std::min<int64_t>(A, cfg->microbatch_rows), 1)));
  PRORL_CUDA(c->informative.ensure((size_t)std::max(G, 1)));
  PRORL_CUDA(c->partials.ensure(sizeof(double) * PRORL_N_PARTIALS));
  PRORL_CUDA(c->slab.ensure(sizeof(double) * PRORL_N_PARTIALS * (size_t)std::max(srows, loss_slab_rows(c))));
  if (lmhead_mode) {
    const size_t mbr = (size_t)std::max<int64_t>(std::min<int64_t>(A, cfg->microbatch_rows), 1);
    PRORL_CUDA(c->logp.ensure(sizeof(float) * mbr));
    PRORL_CUDA(c->entropy.ensure(sizeof(float) * mbr));
  }

  double* partials = c->partials.as<double>();
  double* slab = c->slab.as<double>();
  NvtxRange step_range("prorl_score_host");
  prorl_step_info info{};
  c->last_step = info;
  // Token SoA chunks (one chunk = copied and packed before any scoring). In
  // training mode with a gradient sink every token is checked before the first
  // gradient leaves, so there the SoA is not chunked.
  PackChunk chunks[prorl_ctx::kMaxChunks];
  const int n_chunks = plan_chunks(hb->turns, hb->n_turns, N, A, cfg->microbatch_rows,
                                   (train_mode && pool->consume_grad) ? 1 : prorl_ctx::kMaxChunks, chunks);
  // The copy stream must be idle whenever this call returns (the caller may
  // free or reuse its host buffers): joined on every exit path.
  struct CopyJoin {
    cudaStream_t s = nullptr;
    ~CopyJoin() {
      if (s) cudaStreamSynchronize(s);
    }
  } copy_join;
  PRORL_CUDA(cudaEventRecord(c->ev[0], st));
  // ---- H2D ----
  int64_t h2d = 0;
  auto h2d_copy = [&](void* dst, const void* src, size_t bytes, cudaStream_t s) -> cudaError_t {
    h2d += (int64_t)bytes;
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  };
  if (hb->n_turns) PRORL_CUDA(h2d_copy(c->h_turns.p, hb->turns, sizeof(prorl_turn_desc) * hb->n_turns, st));
  if (R) {
    PRORL_CUDA(h2d_copy(c->h_reward.p, hb->reward, sizeof(double) * R, st));
    PRORL_CUDA(h2d_copy(c->h_usable.p, hb->usable, (size_t)R, st));
    if (hb->rollout_key) PRORL_CUDA(h2d_copy(c->h_rkey.p, hb->rollout_key, sizeof(int64_t) * R, st));
  }
  if (G) PRORL_CUDA(h2d_copy(c->h_goff.p, hb->group_off, sizeof(int32_t) * (G + 1), st));
  if (N && n_chunks == 1) {
    PRORL_CUDA(h2d_copy(c->h_ids.p, hb->ids, sizeof(int64_t) * N, st));
    PRORL_CUDA(h2d_copy(c->h_lp.p, hb->lp, sizeof(double) * N, st));
  } else if (N) {
    // the staging buffers are free once the caller's earlier work on `st` is done
    PRORL_CUDA(cudaEventRecord(c->chunk_ev[0], st));
    copy_join.s = c->copy_stream;
    PRORL_CUDA(cudaStreamWaitEvent(c->copy_stream, c->chunk_ev[0], 0));
    for (int k = 0; k < n_chunks; ++k) {
      const PackChunk& ch = chunks[k];
      if (ch.s1 > ch.s0) {
        PRORL_CUDA(h2d_copy(c->h_ids.as<int64_t>() + ch.s0, hb->ids + ch.s0, sizeof(int64_t) * (ch.s1 - ch.s0),
                            c->copy_stream));
        PRORL_CUDA(h2d_copy(c->h_lp.as<double>() + ch.s0, hb->lp + ch.s0, sizeof(double) * (ch.s1 - ch.s0),
                            c->copy_stream));
      }
      PRORL_CUDA(cudaEventRecord(c->chunk_ev[k + 1], c->copy_stream));
    }
  }
  PRORL_CUDA(cudaMemsetAsync(partials, 0, sizeof(double) * PRORL_N_PARTIALS, st));
  PRORL_CUDA(cudaMemsetAsync(slab, 0, sizeof(double) * PRORL_N_PARTIALS * srows, st));
  PRORL_CUDA(cudaMemsetAsync(c->d_err, 0, sizeof(int) * ERR_N, st));  // no stale flags from an aborted call
  PRORL_CUDA(cudaEventRecord(c->ev[1], st));

  // ---- K3 grpo, K1 pack (turn scan, then the token pass chunk by chunk) ----
  prorl_packed pk{};
  pk.tokens = c->p_tokens.as<int32_t>();
  pk.loss_mask = c->p_mask.as<uint8_t>();
  pk.turn_id = c->p_turn.as<int16_t>();
  pk.seq_id = c->p_seq.as<int32_t>();
  pk.pos_id = c->p_pos.as<int32_t>();
  pk.cu_seqlens = c->p_cu.as<int32_t>();
  pk.old_lp = c->p_oldlp.as<float>();
  pk.act_row = c->a_row.as<int32_t>();
  pk.act_target = c->a_target.as<int32_t>();
  pk.act_old_lp = c->a_oldlp.as<float>();
  pk.act_seq = c->a_seq.as<int32_t>();
  pk.act_turn = c->a_turn.as<int16_t>();
  pk.n_active = c->a_nact.as<int64_t>();
  const auto scan_launches = [](int64_t n) -> int64_t { return n > 0 ? 3 : 0; };
  PRORL_TRY(launch_grpo(c, c->h_reward.as<double>(), c->h_usable.as<uint8_t>(), c->h_goff.as<int32_t>(), G, cfg->ddof,
                        cfg->adv_eps, cfg->gate_tolerance, c->adv.as<double>(), c->informative.as<uint8_t>(), partials,
                        st));
  info.kernel_launches += G > 0 ? 1 : 0;
  PRORL_TRY(launch_pack_turns(c, c->h_turns.as<prorl_turn_desc>(), hb->n_turns, N, R, cfg->vocab, &pk, st));
  info.kernel_launches += scan_launches(hb->n_turns) + 1;
  int packed = 0;             // chunks packed so far
  bool packed_since = false;  // a chunk was packed since the last scoring launch (no PDL across it)
  // pack every chunk whose active rows start below `rows` (all chunks: INT64_MAX)
  auto pack_upto = [&](int64_t rows) -> int {
    for (; packed < n_chunks && (packed == 0 || chunks[packed].a0 < rows); ++packed) {
      packed_since = true;
      const PackChunk& ch = chunks[packed];
      if (n_chunks > 1) PRORL_CUDA(cudaStreamWaitEvent(st, c->chunk_ev[packed + 1], 0));
      PRORL_TRY(launch_pack_tokens(c, c->h_turns.as<prorl_turn_desc>(), hb->n_turns, c->h_ids.as<int64_t>(),
                                   c->h_lp.as<double>(), N, R, cfg->vocab, &pk, ch.p0, ch.p1, ch.a0,
                                   packed == n_chunks - 1, st));
      const bool last = packed == n_chunks - 1;
      if (ch.p1 > ch.p0 || last) info.kernel_launches += (ch.p1 > ch.p0 ? 1 : 0) + scan_launches(ch.p1 - ch.p0) + 1;
    }
    return PRORL_OK;
  };
  PRORL_TRY(pack_upto(0));
  PRORL_CUDA(cudaEventRecord(c->ev[2], st));
  // A gradient sink may apply what it is handed at once: make sure K1 accepted
  // every token id and descriptor before the first gradient leaves the library
  // (otherwise the step would only fail after the all-reduce).
  if (train_mode && pool->consume_grad) PRORL_TRY(prorl_check_errors(c, stream));

  // ---- K2+K4 (K7 in training mode) over logits micro-batches, or K6 + K4 from hidden states ----
  const int64_t mb = cfg->microbatch_rows;
  const double n_global = pool->n_global > 0.0 ? pool->n_global : (double)std::max<int64_t>(A, 1);
  for (int64_t j = 0, row0 = 0; row0 < A; ++j, row0 += mb) {
    const int64_t n = std::min(mb, A - row0);
    PRORL_TRY(pack_upto(row0 + n));
    ++info.micro_batches;
    const float* ref_lp = nullptr;  // k3 KL reference logprobs of this micro-batch
    if (pool->provide_ref && cfg->loss.kl_coef != 0.f) {
      const int rc = pool->provide_ref(pool->ref_user, row0, n, pk.act_row + row0, pk.act_seq + row0, pk.cu_seqlens,
                                       pk.act_target + row0, &ref_lp, stream);
      if (rc != PRORL_OK)
        return fail(rc, "prorl_score_host: reference-logprob callback failed with status " + std::to_string(rc) +
                            " at micro-batch " + std::to_string(j));
      if (!ref_lp) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: reference-logprob callback returned null");
    }
    if (lmhead_mode) {
      const void* hid = nullptr;
      int64_t hs = pool->d_model;
      const int rc = pool->provide_hidden(pool->user, row0, n, pk.act_row + row0, pk.act_seq + row0, pk.cu_seqlens,
                                          &hid, &hs, stream);
      if (rc != PRORL_OK)
        return fail(rc, "prorl_score_host: hidden-state callback failed with status " + std::to_string(rc) +
                            " at micro-batch " + std::to_string(j));
      if (!hid) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: hidden-state callback returned null");
      float* lp = c->logp.as<float>();
      float* en = c->entropy.as<float>();
      PRORL_TRY(launch_lmhead(c, hid, hs, pool->weight, pool->w_stride, pool->d_model, cfg->vocab,
                              pk.act_target + row0, n, cfg->inv_temperature, lp, en, st));
      int used = 0;
      PRORL_TRY(launch_loss(c, lp, en, pk.act_old_lp + row0, c->adv.as<double>(), pk.act_seq + row0,
                            pk.act_turn + row0, ref_lp, n, &cfg->loss, slab, loss_slab_rows(c), &used, st));
      PRORL_TRY(launch_slab_reduce(slab, used, partials, st));
      info.kernel_launches += 4;  // K6, its merge, K4, slab reduce
      continue;
    }
    const void* buf = nullptr;
    int64_t stride = pool->row_stride;
    if (pool->provide) {
      const int rc = pool->provide(pool->user, row0, n, pk.act_row + row0, pk.act_seq + row0, pk.cu_seqlens,
                                   pk.act_target + row0, pk.act_old_lp + row0, &buf, &stride, stream);
      if (rc != PRORL_OK)
        return fail(rc, "prorl_score_host: logits callback failed with status " + std::to_string(rc) +
                            " at micro-batch " + std::to_string(j));
      if (!buf) return fail(PRORL_E_MALFORMED_REQUEST, "prorl_score_host: logits callback returned null");
    } else {
      void* b = pool->buffers[j % pool->n_pool];
      if (pool->fill) {
        int64_t* keys = c->row_keys.as<int64_t>();
        PRORL_TRY(launch_row_keys(pk.act_row + row0, pk.act_seq + row0, pk.cu_seqlens,
                                  hb->rollout_key ? c->h_rkey.as<int64_t>() : nullptr, n, keys, st));
        PRORL_TRY(prorl_gen_logits_keyed(c, b, cfg->dtype, pool->row_stride, cfg->vocab, n, keys,
                                         pk.act_target + row0, pk.act_old_lp + row0, pool->seed, pool->sigma, st));
        info.kernel_launches += 2;
      }
      buf = b;
    }
    if (train_mode) {
      void* grad = pool->grad_buffers ? pool->grad_buffers[j % std::max(pool->n_pool, 1)] : const_cast<void*>(buf);
      const int esz = cfg->dtype == PRORL_BF16 ? 2 : 4;
      if (!grad || reinterpret_cast<uintptr_t>(buf) % esz ||
          (static_cast<const uint8_t*>(grad) - static_cast<const uint8_t*>(buf)) % 16 != 0)
        return fail(PRORL_E_SHAPE, "prorl_score_host: gradient buffer must share the logits' 16-byte phase");
      int used = 0;
      PRORL_TRY(launch_train(c, buf, cfg->dtype, stride, cfg->vocab, nullptr, pk.act_target + row0,
                             pk.act_old_lp + row0, c->adv.as<double>(), pk.act_seq + row0, pk.act_turn + row0, ref_lp,
                             n, cfg->inv_temperature, &cfg->loss, n_global, nullptr, nullptr, nullptr, grad, slab, true,
                             &used, st));
      info.kernel_launches += 2;  // K7, its row end
      if (pool->consume_grad) {
        const int rc = pool->consume_grad(pool->grad_user, row0, n, grad, stride, stream);
        if (rc != PRORL_OK)
          return fail(rc, "prorl_score_host: gradient callback failed with status " + std::to_string(rc) +
                              " at micro-batch " + std::to_string(j));
      }
      continue;
    }
    // back-to-back scoring launches (resident pool: no callback or generator
    // work between them) overlap through programmatic dependent launch
    // (not right after a K1 chunk: PDL would let the launch read the chunk's
    // rows before K1 finished writing them)
    const bool pdl = j > 0 && pdl_enabled() && !pool->provide && !pool->fill && !ref_lp && !packed_since;
    packed_since = false;
    PRORL_TRY(launch_score(c, buf, cfg->dtype, stride, cfg->vocab, nullptr, pk.act_target + row0,
                           pk.act_old_lp + row0, c->adv.as<double>(), pk.act_seq + row0, pk.act_turn + row0, ref_lp, n,
                           cfg->inv_temperature, &cfg->loss, nullptr, nullptr, slab, srows, true, nullptr, st, pdl));
    ++info.kernel_launches;
  }
  PRORL_TRY(pack_upto(INT64_MAX));  // chunks without active rows (their packed tokens are still outputs)
  if (!lmhead_mode) PRORL_TRY(launch_slab_reduce(slab, srows, partials, st));
  k_fold_errors<<<1, 1, 0, st>>>(c->d_err, partials);
  PRORL_CUDA(cudaGetLastError());
  info.kernel_launches += (lmhead_mode ? 0 : 1) + 1;
  info.h2d_chunks = n_chunks;
  info.h2d_bytes = h2d;
  PRORL_CUDA(cudaEventRecord(c->ev[3], st));
  reduced = true;  // from here on every rank has entered (or failed inside) the collective
  PRORL_TRY(prorl_allreduce(c, partials, PRORL_N_PARTIALS, stream));
  PRORL_CUDA(cudaEventRecord(c->ev[4], st));
  PRORL_CUDA(cudaMemcpyAsync(host_partials, partials, sizeof(double) * PRORL_N_PARTIALS, cudaMemcpyDeviceToHost, st));
  PRORL_CUDA(cudaEventRecord(c->ev[5], st));
  PRORL_TRY(prorl_check_errors(c, stream));
  c->last_step = info;
  PRORL_TRY(prorl_step_status(PRORL_OK, host_partials));
  if (timings_ms) {
    for (int k = 0; k < 5; ++k) PRORL_CUDA(cudaEventElapsedTime(&timings_ms[k], c->ev[k], c->ev[k + 1]));
  }
  return PRORL_OK;
}
}  // namespace

}  // extern "C"
