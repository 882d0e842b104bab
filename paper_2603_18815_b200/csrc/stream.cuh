// stream.cuh — per-warp TMA ring that streams logits rows through shared
// memory, shared by the forward scorer (K2, score.cu) and the gradient kernel
// (K5, grad.cu).
//
// One warp owns one row at a time; rows i = gw, gw + nw, ... (gw = global warp
// id, nw = warps in the grid). Lane 0 is the producer: it issues 1-D bulk
// copies (cp.async.bulk ... mbarrier::complete_tx, L2 evict_first) of CHUNK-
// byte pieces of the rows' 16-B aligned interiors into STAGES ring slots,
// running ahead across row boundaries. The whole warp consumes: wait on the
// slot's mbarrier, copy the chunk to registers, release() (syncwarp + lane 0
// refills the slot). Unaligned row heads/tails (< 16 B each) are left to the
// caller to read directly.
#pragma once

#include "common.cuh"

namespace prorl {

template <int STAGES, int CHUNK, int ES>
struct RowRing {
  uint8_t* ring;   // this warp's STAGES * CHUNK bytes
  uint64_t* bars;  // this warp's STAGES mbarriers
  uint64_t policy;
  const uint8_t* base;
  int64_t stride_bytes;
  const int32_t* rows;  // nullable: identity
  int64_t n_rows;
  int32_t vocab;
  int64_t nw;
  // producer state (lane 0)
  int64_t p_row, p_chunk, p_nchunks;
  uintptr_t p_a, p_b;
  uint32_t produced;
  uint32_t consumed;

  __device__ __forceinline__ const uint8_t* row_ptr(int64_t i) const {
    const int64_t r = rows ? (int64_t)rows[i] : i;
    return base + r * stride_bytes;
  }

  // interior [a, b) of a row: 16-B aligned, a multiple of 16 bytes
  __device__ __forceinline__ void interior(const uint8_t* rp, uintptr_t& a, uintptr_t& b) const {
    const uintptr_t st = reinterpret_cast<uintptr_t>(rp);
    const uintptr_t en = st + (uintptr_t)vocab * ES;
    a = (st + 15) & ~(uintptr_t)15;
    if (a > en) a = en;
    b = en & ~(uintptr_t)15;
    if (b < a) b = a;
  }

  __device__ __forceinline__ static int64_t chunks(uintptr_t a, uintptr_t b) {
    return (int64_t)((b - a + CHUNK - 1) / CHUNK);
  }

  __device__ __forceinline__ void produce() {
    while (p_row < n_rows && p_chunk >= p_nchunks) {
      p_row += nw;
      p_chunk = 0;
      p_nchunks = 0;
      if (p_row < n_rows) {
        interior(row_ptr(p_row), p_a, p_b);
        p_nchunks = chunks(p_a, p_b);
      }
    }
    if (p_row >= n_rows) return;
    const uintptr_t src = p_a + (uintptr_t)p_chunk * CHUNK;
    const uint32_t bytes = (uint32_t)min((uintptr_t)CHUNK, p_b - src);
    const int s = produced % STAGES;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[s], bytes);
    tma_load_1d(ring + (size_t)s * CHUNK, reinterpret_cast<const void*>(src), bytes, &bars[s], policy);
    ++produced;
    ++p_chunk;
  }

  // Whole warp; smem_warp points at this warp's ring, bars_warp at its barriers.
  __device__ __forceinline__ void init(uint8_t* smem_warp, uint64_t* bars_warp, const uint8_t* base_, int64_t stride,
                                       const int32_t* rows_, int64_t n_rows_, int32_t vocab_, int64_t gw, int64_t nw_,
                                       int lane) {
    ring = smem_warp;
    bars = bars_warp;
    base = base_;
    stride_bytes = stride;
    rows = rows_;
    n_rows = n_rows_;
    vocab = vocab_;
    nw = nw_;
    policy = l2_policy_evict_first();
    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
      fence_mbar_init();
    }
    __syncwarp();
    p_row = gw;
    p_chunk = p_nchunks = 0;
    p_a = p_b = 0;
    produced = consumed = 0;
    if (p_row < n_rows) {
      interior(row_ptr(p_row), p_a, p_b);
      p_nchunks = chunks(p_a, p_b);
    }
    if (lane == 0)
      for (int s = 0; s < STAGES; ++s) produce();
  }

  // Wait for the next chunk; returns its slot (16-B vectors).
  __device__ __forceinline__ const uint4* wait() {
    const int s = consumed % STAGES;
    // bounded: a protocol bug traps after ~4 s instead of hanging the GPU
    if (!mbar_try_wait(&bars[s], (consumed / STAGES) & 1)) {
      uint64_t t0, t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (uint32_t k = 1; !mbar_try_wait(&bars[s], (consumed / STAGES) & 1); ++k)
        if ((k & 255u) == 0) {
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          if (t - t0 > 4000000000ull) __trap();
        }
    }
    return reinterpret_cast<const uint4*>(ring + (size_t)s * CHUNK);
  }

  // The warp is done reading the current slot: refill it.
  __device__ __forceinline__ void release(int lane) {
    __syncwarp();
    ++consumed;
    if (lane == 0) produce();
  }
};

}  // namespace prorl
