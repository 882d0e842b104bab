// scan.cuh — exclusive prefix sum used by the packer (K1): turn lengths ->
// token offsets, active-row flags -> compacted positions. Reduce-then-scan in
// three launches (tile reduce, single-CTA carry scan over tile sums, tile
// re-scan + offset); the input is a functor so no temporary input array is
// materialised. Integer arithmetic only: the result is exact and independent
// of the launch geometry.
#pragma once

#include "common.cuh"

namespace prorl {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // 2048 elements per CTA

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* warp_tot, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = (lane < kScanThreads / 32) ? warp_tot[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T n = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += n;
    }
    if (lane < kScanThreads / 32) warp_tot[lane] = wi - w;
    if (lane == kScanThreads / 32 - 1) *total = wi;
  }
  __syncthreads();
  T r = warp_tot[warp] + inc - v;
  __syncthreads();
  return r;
}

template <typename T, typename F>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(F f, int64_t n, T* tile_sums) {
  __shared__ T wt[kScanThreads / 32];
  __shared__ T tot;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) s += f(base + i);
  block_exclusive_scan<T>(s, wt, &tot);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// Single CTA: exclusive scan of tile_sums[0..nt) in place; tile_sums[nt] = total.
template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(T* tile_sums, int64_t nt) {
  __shared__ T wt[kScanThreads / 32];
  __shared__ T tot;
  T carry = 0;
  for (int64_t b = 0; b < nt; b += kScanThreads) {
    int64_t i = b + threadIdx.x;
    T v = (i < nt) ? tile_sums[i] : T(0);
    T ex = block_exclusive_scan<T>(v, wt, &tot);
    if (i < nt) tile_sums[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) tile_sums[nt] = carry;
}

template <typename T, typename F>
__global__ void __launch_bounds__(kScanThreads) k_scan_apply(F f, int64_t n, const T* tile_sums, T* out) {
  __shared__ T wt[kScanThreads / 32];
  __shared__ T tot;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? f(base + i) : T(0);
    s += v[i];
  }
  T ex = block_exclusive_scan<T>(s, wt, &tot) + tile_sums[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = tile_sums[gridDim.x];
}

// out[0..n] = exclusive scan of f(0..n-1), out[n] = total. tmp: >= (ntiles+1) T.
template <typename T, typename F>
cudaError_t exclusive_scan(F f, int64_t n, T* out, T* tmp, cudaStream_t st) {
  int64_t nt = (n + kScanTile - 1) / kScanTile;
  if (nt == 0) {
    return cudaMemsetAsync(out, 0, sizeof(T), st);
  }
  k_scan_reduce<T, F><<<(unsigned)nt, kScanThreads, 0, st>>>(f, n, tmp);
  k_scan_tiles<T><<<1, kScanThreads, 0, st>>>(tmp, nt);
  k_scan_apply<T, F><<<(unsigned)nt, kScanThreads, 0, st>>>(f, n, tmp, out);
  return cudaGetLastError();
}

inline size_t scan_tmp_elems(int64_t n) { return (size_t)((n + kScanTile - 1) / kScanTile) + 1; }

}  // namespace prorl
