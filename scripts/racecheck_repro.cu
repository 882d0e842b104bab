// racecheck_repro.cu — minimal repro of the only hazard class compute-sanitizer
// racecheck reports in K7 (k_train): a WAR between consumer warps' generic
// reads of a shared-memory ring slot and the producer warp's later TMA refill
// of that slot, when the hand-off is the standard warp-specialised protocol
//
//   consumer: read slot -> __syncwarp -> mbarrier.arrive(empty)      (release.cta)
//   producer: mbarrier.try_wait(empty) (acquire.cta) -> fence.proxy.async
//             -> mbarrier.arrive.expect_tx(full) -> cp.async.bulk (TMA) into the slot
//   consumer: mbarrier.try_wait(full) -> read the new contents
//
// The program checks the data it reads: every round the consumers must see
// exactly the values the producer copied for that round, so a real early
// overwrite shows up as a mismatch (printed, exit code 1). Variant "self": the
// consumer warp's lane 0 refills the slot itself after __syncwarp (K2 / K5 /
// K7-self-fed ordering). Run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/racecheck_repro scripts/racecheck_repro.cu
//   compute-sanitizer --tool racecheck build/racecheck_repro split
//   compute-sanitizer --tool racecheck build/racecheck_repro self
//   compute-sanitizer --tool racecheck build/racecheck_repro split2
// Variant "split2" is K7's two-row-group producer: two slots, one consumer warp
// per slot, ONE producer warp whose lanes 0 and 1 each feed their own slot in a
// converged polling loop (non-blocking mbarrier.test_wait, as train.cu).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>

constexpr int kSlotBytes = 4096;
constexpr int kRounds = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// blockDim = 64 (split: warp 0 consumer, warp 1 producer) or 32 (self)
__global__ void k_ring(const uint32_t* __restrict__ src, int split, int* bad) {
  __shared__ __align__(128) uint32_t slot[kSlotBytes / 4];
  __shared__ uint64_t full, empty;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&full, 1);
    mbar_init(&empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (split && warp == 1) {  // producer warp
    if (lane == 0)
      for (int r = 0; r < kRounds; ++r) {
        if (r > 0) mbar_wait(&empty, (r - 1) & 1);  // the consumers released the slot
        mbar_expect_tx(&full, kSlotBytes);
        tma_1d(slot, src + (size_t)r * (kSlotBytes / 4), kSlotBytes, &full);
      }
    __syncwarp();
    return;
  }
  // consumer warp
  if (!split && lane == 0) {
    mbar_expect_tx(&full, kSlotBytes);
    tma_1d(slot, src, kSlotBytes, &full);
  }
  for (int r = 0; r < kRounds; ++r) {
    mbar_wait(&full, r & 1);
    int err = 0;
    for (int i = lane; i < kSlotBytes / 4; i += 32) err |= slot[i] != (uint32_t)(r * 100000 + i);
    if (err) atomicAdd(bad, 1);
    __syncwarp();
    if (lane == 0) {
      if (split) mbar_arrive(&empty);
      else if (r + 1 < kRounds) {  // self: refill after the warp's reads (ordered by __syncwarp)
        mbar_expect_tx(&full, kSlotBytes);
        tma_1d(slot, src + (size_t)(r + 1) * (kSlotBytes / 4), kSlotBytes, &full);
      }
    }
  }
}

// split2: blockDim = 96 (warps 0, 1 consumers of slots 0, 1; warp 2 the producer)
__global__ void k_ring2(const uint32_t* __restrict__ src, int* bad) {
  __shared__ __align__(128) uint32_t slot[2][kSlotBytes / 4];
  __shared__ uint64_t full[2], empty[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int g = 0; g < 2; ++g) {
      mbar_init(&full[g], 1);
      mbar_init(&empty[g], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 2) {  // producer: lane g feeds slot g; the lanes stay converged and poll
    int r = 0;
    bool live = lane < 2;
    while (__any_sync(0xffffffffu, live)) {
      if (live && (r == 0 || mbar_test(&empty[lane], (r - 1) & 1))) {
        mbar_expect_tx(&full[lane], kSlotBytes);
        tma_1d(slot[lane], src + ((size_t)lane * kRounds + r) * (kSlotBytes / 4), kSlotBytes, &full[lane]);
        live = ++r < kRounds;
      }
    }
    return;
  }
  for (int r = 0; r < kRounds; ++r) {
    mbar_wait(&full[warp], r & 1);
    int err = 0;
    for (int i = lane; i < kSlotBytes / 4; i += 32)
      err |= slot[warp][i] != (uint32_t)((warp * kRounds + r) * 10000 + i);
    if (err) atomicAdd(bad, 1);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[warp]);
  }
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "split2") == 0) {
    const size_t n = (size_t)2 * kRounds * kSlotBytes / 4;
    uint32_t* h = (uint32_t*)malloc(n * 4);
    for (int g = 0; g < 2; ++g)
      for (int r = 0; r < kRounds; ++r)
        for (int i = 0; i < kSlotBytes / 4; ++i)
          h[((size_t)g * kRounds + r) * (kSlotBytes / 4) + i] = (uint32_t)((g * kRounds + r) * 10000 + i);
    uint32_t* d;
    int* bad;
    cudaMalloc(&d, n * 4);
    cudaMalloc(&bad, 4);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    cudaMemset(bad, 0, 4);
    k_ring2<<<1, 96>>>(d, bad);
    int hb = -1;
    cudaError_t e = cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    std::printf("split2 (one producer warp, lanes 0/1 feed two slots): %s, %d rounds, data mismatches: %d\n",
                cudaGetErrorString(e), kRounds, hb);
    return (e == cudaSuccess && hb == 0) ? 0 : 1;
  }
  const int split = !(argc > 1 && std::strcmp(argv[1], "self") == 0);
  const size_t n = (size_t)kRounds * kSlotBytes / 4;
  uint32_t* h = (uint32_t*)malloc(n * 4);
  for (int r = 0; r < kRounds; ++r)
    for (int i = 0; i < kSlotBytes / 4; ++i) h[(size_t)r * (kSlotBytes / 4) + i] = (uint32_t)(r * 100000 + i);
  uint32_t* d;
  int* bad;
  cudaMalloc(&d, n * 4);
  cudaMalloc(&bad, 4);
  cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
  cudaMemset(bad, 0, 4);
  k_ring<<<1, split ? 64 : 32>>>(d, split, bad);
  int hb = -1;
  cudaError_t e = cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  std::printf("%s: %s, %d rounds, data mismatches: %d\n", split ? "split (producer warp)" : "self (lane 0 refills)",
              cudaGetErrorString(e), kRounds, hb);
  return (e == cudaSuccess && hb == 0) ? 0 : 1;
}
