// ex2_shift_probe.cu — MUFU.EX2's mean relative error over a row's terms as a
// function of where the row's mass sits below the running reference. Rows of
// bf16 N(0, s^2) logits (V = 151 936), integer reference M = ceil(max x c) + k
// (k > 0: the reference set by a planted / dominant target above the bulk).
// For each (sigma, k): the term-weighted bias b = (sum MUFU(d) - sum 2^d) /
// sum 2^d averaged over rows, and the mass-weighted mean argument
// dbar = sum d 2^d / sum 2^d (what T / S gives the row end for free).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ex2_shift_probe scripts/ex2_shift_probe.cu
#include <cuda_bf16.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void k_probe(const float* x, float* y, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[i]));
    y[i] = r;
  }
}

static uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

int main() {
  const int V = 151936, R = 32;
  const float c = 1.44269504088896340736f;
  float *dx, *dy;
  cudaMalloc(&dx, (size_t)V * R * 4);
  cudaMalloc(&dy, (size_t)V * R * 4);
  std::vector<float> x((size_t)V * R), y((size_t)V * R), raw(V);
  for (int fp32 = 0; fp32 < 2; ++fp32)
    for (float sigma : {0.5f, 1.0f, 2.0f, 3.0f, 4.0f})
      for (int k : {0, 1, 2, 3, 4, 6, 8}) {
        uint64_t st = 2603 + (uint64_t)(sigma * 100) + 7919ull * k;
        for (int r = 0; r < R; ++r) {
          float mx = -1e30f;
          for (int v = 0; v < V; ++v) {
            double u = 0;
            for (int q = 0; q < 4; ++q) u += (double)(splitmix(st) >> 40) / 16777216.0;
            const float f = (float)(sigma * 1.7320508 * (u - 2.0));
            raw[v] = fp32 ? f : __bfloat162float(__float2bfloat16(f));
            mx = std::max(mx, raw[v]);
          }
          const float M = std::ceil(mx * c) + (float)k;
          for (int v = 0; v < V; ++v) x[(size_t)r * V + v] = std::fmaf(raw[v], c, -M);
        }
        cudaMemcpy(dx, x.data(), x.size() * 4, cudaMemcpyHostToDevice);
        k_probe<<<(unsigned)((x.size() + 255) / 256), 256>>>(dx, dy, (int64_t)x.size());
        cudaMemcpy(y.data(), dy, y.size() * 4, cudaMemcpyDeviceToHost);
        double bm = 0, b2 = 0, dm = 0;
        for (int r = 0; r < R; ++r) {
          double se = 0, sy = 0, sd = 0;
          for (int v = 0; v < V; ++v) {
            const size_t i = (size_t)r * V + v;
            const double e = std::exp2((double)x[i]);
            se += e;
            sy += (double)y[i];
            sd += (double)x[i] * e;
          }
          const double b = (sy - se) / se;
          bm += b;
          b2 += b * b;
          dm += sd / se;
        }
        bm /= R;
        dm /= R;
        std::printf("%s sigma=%.1f k=%d  dbar=%8.4f  bias=%.5e  sd=%.2e\n", fp32 ? "fp32" : "bf16", sigma, k, dm, bm,
                    std::sqrt(std::max(0.0, b2 / R - bm * bm)));
      }
  return 0;
}
