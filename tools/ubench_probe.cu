// ubench_probe.cu -- microbenchmark isolating the costs of the lookup
// kernel's phases on B200 (diagnostic tool, not product code).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ub tools/ubench_probe.cu
//
// Table: S slabsets x 2 slabs x 32 slots, d = 128 f32 rows (1 GB at S=31250).
// Query: 65536 positions, slot drawn uniform or power-law (alpha 1.2).
// Kernels (each timed with CUDA events, median of 20):
//   gather   warp per 4 positions: row[slot] -> out[i] (no probe)
//   probe    warp per 4 positions: load mask + 32 slab keys, ballot
//   probe+g  both
//   lane     probe with one lane per position reading its 256 B slab
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));     \
      return 1;                                                            \
    }                                                                      \
  } while (0)

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

template <int P, bool GATHER>
__global__ void __launch_bounds__(256) k_probe(const uint64_t* __restrict__ skeys,
                                              const uint32_t* __restrict__ masks,
                                              const float* __restrict__ rows,
                                              const uint64_t* __restrict__ q, int n,
                                              float* __restrict__ out, uint32_t* hits) {
  int w = (blockIdx.x * 256 + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int base = w * P;
  if (base >= n) return;
  uint64_t key[P];
  uint32_t slab[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    key[p] = q[base + p];
    slab[p] = uint32_t(key[p] >> 5);  // key = slot id; slab = slot / 32
  }
  uint64_t sk[P];
  uint32_t m[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    m[p] = masks[slab[p]];
    sk[p] = skeys[uint64_t(slab[p]) * 32 + lane];
  }
  uint32_t found[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    uint32_t b = __ballot_sync(~0u, ((m[p] >> lane) & 1) && sk[p] == key[p]);
    found[p] = b ? slab[p] * 32 + __ffs(b) - 1 : ~0u;
  }
  if (GATHER) {
    float4 v[P];
#pragma unroll
    for (int p = 0; p < P; ++p)
      v[p] = reinterpret_cast<const float4*>(rows + uint64_t(found[p]) * D)[lane];
#pragma unroll
    for (int p = 0; p < P; ++p)
      reinterpret_cast<float4*>(out + uint64_t(base + p) * D)[lane] = v[p];
  } else if (lane < P) {
    uint32_t f = 0;
#pragma unroll
    for (int p = 0; p < P; ++p)
      if (p == lane) f = found[p];
    hits[base + lane] = f;
  }
}

__global__ void __launch_bounds__(256) k_copy(const float4* __restrict__ in, float4* __restrict__ out,
                                             uint64_t n4) {
  uint64_t i = uint64_t(blockIdx.x) * 256 + threadIdx.x;
  for (; i < n4; i += uint64_t(gridDim.x) * 256) out[i] = in[i];
}
__global__ void __launch_bounds__(256) k_write(float4* __restrict__ out, uint64_t n4) {
  uint64_t i = uint64_t(blockIdx.x) * 256 + threadIdx.x;
  for (; i < n4; i += uint64_t(gridDim.x) * 256) out[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

// TMA bulk-copy gather: each warp moves its rows global->smem->global with
// cp.async.bulk (one elected lane issues, an mbarrier tracks the loads).
template <int R>
__global__ void __launch_bounds__(128) k_gather_bulk(const float* __restrict__ rows,
                                                     const uint32_t* __restrict__ slot, int n,
                                                     float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar[4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* buf = smem + warp * R * D * 4;
  const uint32_t bar_addr = uint32_t(__cvta_generic_to_shared(&bar[warp]));
  if (lane == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar_addr));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  uint32_t phase = 0;
  const int gw = blockIdx.x * 4 + warp, nw = gridDim.x * 4;
  for (int base = gw * R; base < n; base += nw * R) {
    const int cnt = min(R, n - base);
    if (lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar_addr),
                   "r"(cnt * D * 4));
    }
    __syncwarp();
    if (lane < cnt) {
      const float* src = rows + uint64_t(slot[base + lane]) * D;
      const uint32_t dst = uint32_t(__cvta_generic_to_shared(buf + lane * D * 4));
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
          "l"(src), "r"(D * 4), "r"(bar_addr)
          : "memory");
    }
    // wait for all loads of this round
    asm volatile(
        "{ .reg .pred P; WAIT_%=: mbarrier.try_wait.parity.shared.b64 P, [%0], %1; @!P bra WAIT_%=; }" ::"r"(bar_addr),
        "r"(phase)
        : "memory");
    phase ^= 1;
    if (lane < cnt) {
      const uint32_t srcs = uint32_t(__cvta_generic_to_shared(buf + lane * D * 4));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + uint64_t(base + lane) * D),
                   "r"(srcs), "r"(D * 4)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
  }
}

// one lane per position: each lane scans its own slab with 16-byte loads
__global__ void __launch_bounds__(256) k_probe_lane(const uint64_t* __restrict__ skeys,
                                                   const uint32_t* __restrict__ masks,
                                                   const uint64_t* __restrict__ q, int n,
                                                   uint32_t* hits) {
  int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= n) return;
  uint64_t key = q[i];
  uint32_t slab = uint32_t(key >> 5);
  uint32_t m = masks[slab];
  const ulonglong2* s = reinterpret_cast<const ulonglong2*>(skeys + uint64_t(slab) * 32);
  uint32_t f = ~0u;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    ulonglong2 v = s[j];
    if (((m >> (2 * j)) & 1) && v.x == key) f = slab * 32 + 2 * j;
    if (((m >> (2 * j + 1)) & 1) && v.y == key) f = slab * 32 + 2 * j + 1;
  }
  hits[i] = f;
}

int main() {
  const int S = 31250, W = 2;
  const uint64_t slots = uint64_t(S) * W * 32;
  const int n = 65536;
  std::vector<uint64_t> hk(slots);
  for (uint64_t s = 0; s < slots; ++s) hk[s] = s;
  std::vector<uint32_t> hm(S * W, 0xFFFFFFFFu);
  uint64_t *skeys, *q;
  uint32_t *masks, *slot, *hits;
  float *rows, *out;
  CK(cudaMalloc(&skeys, slots * 8));
  CK(cudaMalloc(&masks, S * W * 4));
  CK(cudaMalloc(&rows, slots * D * 4));
  CK(cudaMalloc(&out, uint64_t(n) * D * 4 * 8));
  CK(cudaMalloc(&q, n * 8 * 32));
  CK(cudaMalloc(&slot, n * 4 * 32));
  CK(cudaMalloc(&hits, n * 4));
  CK(cudaMemcpy(skeys, hk.data(), slots * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(masks, hm.data(), S * W * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(rows, 0, slots * D * 4));
  std::mt19937_64 g(1);
  // power-law CDF over slots (rank r -> slot perm[r])
  std::vector<double> cdf(slots);
  double run = 0;
  for (uint64_t r = 1; r <= slots; ++r) cdf[r - 1] = (run += std::pow(double(r), -1.2));
  for (auto& c : cdf) c /= run;
  std::vector<uint64_t> perm(slots);
  for (uint64_t i = 0; i < slots; ++i) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), g);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  {
    const uint64_t n4 = uint64_t(n) * D / 4;
    std::vector<float> ts;
    for (int it = 0; it < 30; ++it) {
      cudaEventRecord(a);
      k_copy<<<148 * 8, 256>>>(reinterpret_cast<const float4*>(rows) + (it % 8) * n4,
                               reinterpret_cast<float4*>(out) + (it % 8) * n4, n4);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ts.push_back(ms * 1000);
    }
    std::sort(ts.begin(), ts.end());
    printf("copy 33.5MB contiguous median %.2f us (%.0f GB/s rd+wr)\n", ts[15], 2 * n4 * 16 / (ts[15] * 1e3));
    ts.clear();
    for (int it = 0; it < 30; ++it) {
      cudaEventRecord(a);
      k_write<<<148 * 8, 256>>>(reinterpret_cast<float4*>(out) + (it % 8) * n4, n4);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ts.push_back(ms * 1000);
    }
    std::sort(ts.begin(), ts.end());
    printf("write 33.5MB median %.2f us (%.0f GB/s)\n", ts[15], n4 * 16 / (ts[15] * 1e3));
    ts.clear();
    for (int it = 0; it < 30; ++it) {
      cudaEventRecord(a);
      k_write<<<1, 32>>>(reinterpret_cast<float4*>(out), 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ts.push_back(ms * 1000);
    }
    std::sort(ts.begin(), ts.end());
    printf("empty-ish launch median %.2f us\n", ts[15]);
  }
  CK(cudaFuncSetAttribute(k_gather_bulk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16 * D * 4));
  CK(cudaFuncSetAttribute(k_gather_bulk<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * D * 4));
  for (int dist = 0; dist < 2; ++dist) {
    std::vector<uint64_t> hq(n * 32);
    std::vector<uint32_t> hs(n * 32);
    std::uniform_real_distribution<double> U(0, 1);
    for (int i = 0; i < n * 32; ++i) {
      uint64_t s;
      if (dist == 0) {
        s = g() % slots;
      } else {
        s = perm[std::min<uint64_t>(slots - 1,
                                    std::upper_bound(cdf.begin(), cdf.end(), U(g)) - cdf.begin())];
      }
      hq[i] = s;
      hs[i] = uint32_t(s);
    }
    CK(cudaMemcpy(q, hq.data(), n * 8 * 32, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(slot, hs.data(), n * 4 * 32, cudaMemcpyHostToDevice));
    auto timeit = [&](const char* name, auto launch) {
      std::vector<float> ts;
      for (int it = 0; it < 40; ++it) {
        int bi = it % 32;
        cudaEventRecord(a);
        launch(bi, it % 8);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (it >= 8) ts.push_back(ms * 1000);
      }
      std::sort(ts.begin(), ts.end());
      printf("%-8s %-22s median %7.2f us  min %7.2f us\n", dist ? "powerlaw" : "uniform", name,
             ts[ts.size() / 2], ts[0]);
    };
    const int blocks4 = (n / 4 * 32 + 255) / 256;
    const int blocks1 = (n * 32 + 255) / 256;
    timeit("gather P=4", [&](int bi, int o) {
      k_gather<4><<<blocks4, 256>>>(rows, slot + bi * n, n, out + uint64_t(o) * n * D);
    });
    timeit("gather bulk R=16", [&](int bi, int o) {
      k_gather_bulk<16><<<148 * 3, 128, 4 * 16 * D * 4>>>(rows, slot + bi * n, n, out + uint64_t(o) * n * D);
    });
    timeit("gather bulk R=32", [&](int bi, int o) {
      k_gather_bulk<32><<<148 * 3, 128, 4 * 32 * D * 4>>>(rows, slot + bi * n, n, out + uint64_t(o) * n * D);
    });
    timeit("gather P=8", [&](int bi, int o) {
      k_gather<8><<<(n / 8 * 32 + 255) / 256, 256>>>(rows, slot + bi * n, n, out + uint64_t(o) * n * D);
    });
    timeit("gather P=1", [&](int bi, int o) {
      k_gather<1><<<blocks1, 256>>>(rows, slot + bi * n, n, out + uint64_t(o) * n * D);
    });
    timeit("probe P=4", [&](int bi, int o) {
      k_probe<4, false><<<blocks4, 256>>>(skeys, masks, rows, q + bi * n, n, out, hits);
    });
    timeit("probe P=1", [&](int bi, int o) {
      k_probe<1, false><<<blocks1, 256>>>(skeys, masks, rows, q + bi * n, n, out, hits);
    });
    timeit("probe+gather P=4", [&](int bi, int o) {
      k_probe<4, true><<<blocks4, 256>>>(skeys, masks, rows, q + bi * n, n,
                                        out + uint64_t(o) * n * D, hits);
    });
    timeit("probe lane/pos", [&](int bi, int o) {
      k_probe_lane<<<(n + 255) / 256, 256>>>(skeys, masks, q + bi * n, n, hits);
    });
  }
  return 0;
}
