// ubench_gather.cu -- gather microbenchmark (diagnostic tool): how fast can
// 65,536 rows of 512 B be copied from random slots of a 1 GB table into a
// fresh output, and does the table span (TLB reach) matter?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ug tools/ubench_gather.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

constexpr int D = 128;

template <int P>
__global__ void __launch_bounds__(256) k_gather(const float* __restrict__ rows,
                                               const uint32_t* __restrict__ slot, int n,
                                               float* __restrict__ out) {
  int w = (blockIdx.x * 256 + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int base = w * P;
  if (base >= n) return;
  float4 v[P];
#pragma unroll
  for (int p = 0; p < P; ++p)
    v[p] = reinterpret_cast<const float4*>(rows + uint64_t(slot[base + p]) * D)[lane];
#pragma unroll
  for (int p = 0; p < P; ++p) reinterpret_cast<float4*>(out + uint64_t(base + p) * D)[lane] = v[p];
}

// persistent, many rows in flight per warp
template <int P>
__global__ void __launch_bounds__(256) k_gather_pers(const float* __restrict__ rows,
                                                    const uint32_t* __restrict__ slot, int n,
                                                    float* __restrict__ out) {
  int lane = threadIdx.x & 31;
  int w = (blockIdx.x * 256 + threadIdx.x) >> 5, nw = gridDim.x * 8;
  for (int base = w * P; base < n; base += nw * P) {
    float4 v[P];
#pragma unroll
    for (int p = 0; p < P; ++p)
      v[p] = base + p < n ? reinterpret_cast<const float4*>(rows + uint64_t(slot[base + p]) * D)[lane]
                          : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int p = 0; p < P; ++p)
      if (base + p < n) reinterpret_cast<float4*>(out + uint64_t(base + p) * D)[lane] = v[p];
  }
}

__global__ void k_write(float4* out, uint64_t n4) {
  for (uint64_t i = uint64_t(blockIdx.x) * 256 + threadIdx.x; i < n4; i += uint64_t(gridDim.x) * 256)
    out[i] = make_float4(1, 2, 3, 4);
}

int main() {
  const uint64_t slots = 2000000;
  const int n = 65536, K = 40;
  float *rows, *out;
  uint32_t* slot;
  cudaMalloc(&rows, slots * D * 4);
  cudaMalloc(&out, uint64_t(n) * D * 4 * 8);
  cudaMalloc(&slot, uint64_t(n) * 4 * K);
  cudaMemset(rows, 0, slots * D * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::mt19937_64 g(1);
  auto run = [&](const char* name, auto launch) {
    for (int it = 0; it < 5; ++it) launch(it);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int it = 0; it < K; ++it) launch(it);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1000 / K;
    printf("%-40s %7.2f us/launch  %6.0f GB/s (rd+wr of rows)\n", name, us,
           2.0 * n * D * 4 / (us * 1e3));
  };
  {
    const uint64_t n4 = uint64_t(n) * D / 4;
    run("write 33.5 MB", [&](int it) {
      k_write<<<148 * 4, 256>>>(reinterpret_cast<float4*>(out) + (it % 8) * n4, n4);
    });
  }
  // power-law (alpha 1.2) slots over the whole table: the lookup's real mix
  std::vector<double> cdf(slots);
  {
    double acc = 0;
    for (uint64_t r = 0; r < slots; ++r) cdf[r] = (acc += std::pow(double(r + 1), -1.2));
    for (auto& x : cdf) x /= acc;
  }
  std::vector<uint32_t> perm(slots);
  for (uint64_t i = 0; i < slots; ++i) perm[i] = uint32_t(i);
  std::shuffle(perm.begin(), perm.end(), g);
  for (uint64_t span : {uint64_t(0), uint64_t(32768), uint64_t(262144), slots}) {
    std::vector<uint32_t> h(uint64_t(n) * K);
    std::uniform_real_distribution<double> U(0, 1);
    for (auto& x : h) {
      if (span == 0) {
        const uint64_t r = std::lower_bound(cdf.begin(), cdf.end(), U(g)) - cdf.begin();
        x = perm[std::min<uint64_t>(r, slots - 1)];
      } else {
        x = uint32_t(g() % span);
      }
    }
    cudaMemcpy(slot, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    char buf[128];
    snprintf(buf, sizeof buf, "gather P=4 span %.0f MB (0=powerlaw)", span * 512.0 / 1e6);
    run(buf, [&](int it) {
      k_gather<4><<<n / 4 / 8, 256>>>(rows, slot + uint64_t(it) * n, n, out + uint64_t(it % 8) * n * D);
    });
    snprintf(buf, sizeof buf, "gather P=8 span %.0f MB", span * 512.0 / 1e6);
    run(buf, [&](int it) {
      k_gather<8><<<n / 8 / 8, 256>>>(rows, slot + uint64_t(it) * n, n, out + uint64_t(it % 8) * n * D);
    });
    snprintf(buf, sizeof buf, "gather pers P=8 x592 span %.0f MB", span * 512.0 / 1e6);
    run(buf, [&](int it) {
      k_gather_pers<8><<<148 * 4, 256>>>(rows, slot + uint64_t(it) * n, n, out + uint64_t(it % 8) * n * D);
    });
  }
  return 0;
}
