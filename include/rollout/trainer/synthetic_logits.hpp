// rollout/trainer/synthetic_logits.hpp — a deterministic LogitsSource for
// benches and tests: the integer-hash logits of include/prorl_synth.h,
// generated on the device by prorl_gen_logits_keyed (bit-identical to the CPU
// oracle's oracle_gen_logits). Stands in for the trainer's LM head, which is
// outside the reference's scope. Header-only like scoring.hpp;
// needs the CUDA runtime headers for the device buffers.
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>

#include "rollout/trainer/scoring.hpp"

namespace rollout::train {

class SyntheticLogits : public LogitsSource {
 public:
  // Rows are keyed as prorl_score_host's fill mode keys them when the batch has
  // no rollout_key: slot * 2^20 + position in the sequence.
  SyntheticLogits(int device, int vocab, LogitsDtype dtype, std::int64_t max_rows, std::uint64_t seed,
                  float sigma = 2.0f)
      : vocab_(vocab), dtype_(dtype), max_rows_(max_rows), seed_(seed), sigma_(sigma) {
    throw_status(prorl_ctx_create(device, &ctx_));
    const std::size_t esz = dtype == LogitsDtype::BF16 ? 2 : 4;
    if (cudaMalloc(&buf_, static_cast<std::size_t>(max_rows) * static_cast<std::size_t>(vocab) * esz) != cudaSuccess ||
        cudaMalloc(reinterpret_cast<void**>(&keys_), sizeof(std::int64_t) * static_cast<std::size_t>(max_rows)) !=
            cudaSuccess) {
      release();
      throw CudaError("SyntheticLogits: cudaMalloc failed");
    }
  }
  ~SyntheticLogits() override { release(); }
  SyntheticLogits(const SyntheticLogits&) = delete;
  SyntheticLogits& operator=(const SyntheticLogits&) = delete;

  const void* logits(std::int64_t, std::int64_t n, const std::int32_t* d_rows, const std::int32_t* d_seq,
                     const std::int32_t* d_cu_seqlens, const std::int32_t* d_targets, const float* d_old_lp,
                     std::int64_t* row_stride, void* stream) override {
    if (n > max_rows_) throw ShapeMismatch("SyntheticLogits: micro-batch larger than max_rows");
    throw_status(prorl_row_keys(ctx_, d_rows, d_seq, d_cu_seqlens, nullptr, n, keys_, stream));
    throw_status(prorl_gen_logits_keyed(ctx_, buf_, static_cast<int>(dtype_), vocab_, vocab_, n, keys_, d_targets,
                                        d_old_lp, seed_, sigma_, stream));
    *row_stride = vocab_;
    return buf_;
  }

 private:
  void release() {
    if (buf_) cudaFree(buf_);
    if (keys_) cudaFree(keys_);
    buf_ = nullptr;
    keys_ = nullptr;
    prorl_ctx_destroy(ctx_);
    ctx_ = nullptr;
  }

  prorl_ctx* ctx_ = nullptr;
  void* buf_ = nullptr;
  std::int64_t* keys_ = nullptr;  // per-row synthetic keys (slot * 2^20 + position), as the oracle
  int vocab_;
  LogitsDtype dtype_;
  std::int64_t max_rows_;
  std::uint64_t seed_;
  float sigma_;
};

}  // namespace rollout::train
