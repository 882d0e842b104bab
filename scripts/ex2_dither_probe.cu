// ex2_dither_probe.cu — is MUFU.EX2's bias a function of the fractional part of
// its argument only, and does a per-row fractional offset of the running
// reference (the "dithered reference" of rowmath.cuh) turn the row-dependent
// weighted bias into one constant?
//
//   1. b0: the mean relative error of ex2.approx.ftz.f32 over a uniform grid
//      of fractional parts f (2^22 points), for several integer parts;
//   2. per-row weighted bias of a bf16 N(0, 2^2) row (V = 151 936) with an
//      integer reference (what the kernels did) for many rows: its spread;
//   3. the same rows with the reference shifted by phi = j / 4096 per row:
//      the mean over rows should equal b0 and the spread is random.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ex2_dither_probe scripts/ex2_dither_probe.cu
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

static std::vector<float> run(const std::vector<float>& x) {
  const int64_t n = (int64_t)x.size();
  float *dx, *dy;
  cudaMalloc(&dx, n * 4);
  cudaMalloc(&dy, n * 4);
  cudaMemcpy(dx, x.data(), n * 4, cudaMemcpyHostToDevice);
  k_probe<<<(unsigned)((n + 255) / 256), 256>>>(dx, dy, n);
  std::vector<float> y(n);
  cudaMemcpy(y.data(), dy, n * 4, cudaMemcpyDeviceToHost);
  cudaFree(dx);
  cudaFree(dy);
  return y;
}

static uint64_t splitmix(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

int main() {
  // 1. uniform fractional parts
  for (int ip : {0, 1, 3, 7, 15}) {
    std::vector<float> x;
    const int n = 1 << 22;
    for (int j = 0; j < n; ++j) x.push_back(-(float)ip - (float)j / (float)n);
    const auto y = run(x);
    double s = 0;
    for (int j = 0; j < n; ++j) {
      const double e = std::exp2((double)x[j]);
      s += ((double)y[j] - e) / e;
    }
    std::printf("uniform f, integer part -%d: b0 = %.5e\n", ip, s / n);
  }
  // 2./3. rows of bf16 N(0, 2^2) logits, V = 151 936
  const int V = 151936, R = 256;
  const float c = 1.44269504088896340736f;
  uint64_t st = 2603;
  for (int mode = 0; mode < 3; ++mode) {
    std::vector<float> x;
    std::vector<double> w;
    x.reserve((size_t)V * R);
    for (int r = 0; r < R; ++r) {
      std::vector<float> raw(V);
      float mx = -1e30f;
      for (int v = 0; v < V; ++v) {
        double u = 0;
        for (int k = 0; k < 4; ++k) u += (double)(splitmix(st) >> 40) / 16777216.0;
        raw[v] = __bfloat162float(__float2bfloat16((float)(2.0 * 1.7320508 * (u - 2.0))));
        mx = std::max(mx, raw[v]);
      }
      const float Mi = std::ceil(mx * c);
      const float phi = mode == 0 ? 0.f : mode == 1 ? (float)(splitmix(st) & 4095) / 4096.f : (float)(r % 16) / 16.f;
      const float P = Mi + phi;  // exact for |Mi| < 2^11
      for (int v = 0; v < V; ++v) x.push_back(std::fmaf(raw[v], c, -P));
    }
    const auto y = run(x);
    double mean = 0, m2 = 0;
    for (int r = 0; r < R; ++r) {
      double se = 0, sy = 0;
      for (int v = 0; v < V; ++v) {
        const size_t i = (size_t)r * V + v;
        se += std::exp2((double)x[i]);
        sy += (double)y[i];
      }
      const double b = (sy - se) / se;
      mean += b;
      m2 += b * b;
    }
    mean /= R;
    const double sd = std::sqrt(std::max(0.0, m2 / R - mean * mean));
    std::printf("%s: per-row weighted bias mean = %.5e  sd over rows = %.3e  (sd of the mean %.2e)\n",
                mode == 0 ? "integer reference          " : mode == 1 ? "reference + j/4096 per row " : "reference + j/16 per row   ",
                mean, sd, sd / std::sqrt((double)R));
  }
  return 0;
}
