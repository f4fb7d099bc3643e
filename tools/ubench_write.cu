// ubench_write.cu -- diagnostic: what write bandwidth can a 33.5 MB output
// stream reach on B200, and what does the row gather of the lookup cost
// with each store flavour? (Outputs rotate over 8 buffers = 268 MB > L2.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_write tools/ubench_write.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

constexpr int D = 128;
static int N = 65536;  // rows per launch (argv[1] multiplies it)

__device__ __forceinline__ void st256(void* p, uint32_t v, bool cs) {
  if (cs)
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
  else
    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p), "r"(v) : "memory");
}

__global__ void k_write4(float4* out, uint64_t n4) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = make_float4(1, 2, 3, 4);
}

template <bool CS>
__global__ void k_write8(uint8_t* out, uint64_t n32) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n32;
       i += uint64_t(gridDim.x) * blockDim.x)
    st256(out + i * 32, 0x3f800000u, CS);
}

// contiguous per-block slabs (each block writes its own 16 KB chunks)
template <bool CS>
__global__ void k_write8_chunked(uint8_t* out, uint64_t chunks) {
  for (uint64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x)
    for (uint32_t j = threadIdx.x; j < 512; j += blockDim.x) st256(out + ch * 16384 + j * 32, 1u, CS);
}

// TMA bulk store: a block fills 16 KB of smem once, then streams it out
__global__ void k_write_bulk(uint8_t* out, uint64_t chunks) {
  __shared__ __align__(128) uint8_t buf[16384];
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(buf)[i] = 1u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t s = uint32_t(__cvta_generic_to_shared(buf));
    for (uint64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(
                       out + ch * 16384),
                   "r"(s)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// gather: warp copies 32 rows (slot[base+i]) into its contiguous output block
template <int U, bool CS>
__global__ void __launch_bounds__(256) k_gather8(const float* __restrict__ rows,
                                                const uint32_t* __restrict__ slot, int n,
                                                float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int base = ((blockIdx.x * 256 + threadIdx.x) >> 5) * 32;
  if (base >= n) return;
  const uint32_t my = slot[base + lane];
  const int total = 32 * (D / 8);
  for (int c0 = 0; c0 < total; c0 += 32 * U) {
    uint32_t x[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int ch = c0 + u * 32 + lane;
      const int row = ch / (D / 8), j = ch % (D / 8);
      const uint32_t s = __shfl_sync(0xFFFFFFFFu, my, row);
      const float* p = rows + uint64_t(s) * D + j * 8;
      asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(x[u][0]), "=r"(x[u][1]), "=r"(x[u][2]), "=r"(x[u][3]), "=r"(x[u][4]),
                     "=r"(x[u][5]), "=r"(x[u][6]), "=r"(x[u][7])
                   : "l"(p));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int ch = c0 + u * 32 + lane;
      float* p = out + uint64_t(base) * D + uint64_t(ch) * 8;
      if (CS)
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(x[u][0]),
                     "r"(x[u][1]), "r"(x[u][2]), "r"(x[u][3]), "r"(x[u][4]), "r"(x[u][5]),
                     "r"(x[u][6]), "r"(x[u][7])
                     : "memory");
      else
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(x[u][0]),
                     "r"(x[u][1]), "r"(x[u][2]), "r"(x[u][3]), "r"(x[u][4]), "r"(x[u][5]),
                     "r"(x[u][6]), "r"(x[u][7])
                     : "memory");
    }
  }
}

int main(int argc, char** argv) {
  if (argc > 1) N *= atoi(argv[1]);
  const uint64_t slots = 2000000, bytes = uint64_t(N) * D * 4;
  float *rows, *out;
  uint32_t* slot;
  const int K = 40;
  cudaMalloc(&rows, slots * D * 4);
  cudaMalloc(&out, bytes * (N > 65536 ? 2 : 8));
  cudaMalloc(&slot, uint64_t(N) * 4 * K);
  cudaMemset(rows, 0, slots * D * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, double moved, auto launch) {
    for (int it = 0; it < 8; ++it) launch(it);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int it = 0; it < K; ++it) launch(it);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double us = ms * 1000 / K;
    printf("%-46s %7.2f us  %6.0f GB/s\n", name, us, moved / (us * 1e3));
  };
  auto ob = [&](int it) { return reinterpret_cast<uint8_t*>(out) + (it % (N > 65536 ? 2 : 8)) * bytes; };
  for (int g : {148 * 4, 148 * 8, 148 * 16}) {
    char nm[96];
    snprintf(nm, sizeof nm, "write float4 grid %d", g);
    run(nm, bytes, [&](int it) { k_write4<<<g, 256>>>(reinterpret_cast<float4*>(ob(it)), bytes / 16); });
    snprintf(nm, sizeof nm, "write 256b grid %d", g);
    run(nm, bytes, [&](int it) { k_write8<false><<<g, 256>>>(ob(it), bytes / 32); });
    snprintf(nm, sizeof nm, "write 256b .cs grid %d", g);
    run(nm, bytes, [&](int it) { k_write8<true><<<g, 256>>>(ob(it), bytes / 32); });
    snprintf(nm, sizeof nm, "write 256b 16KB-chunked grid %d", g);
    run(nm, bytes, [&](int it) { k_write8_chunked<false><<<g, 256>>>(ob(it), bytes / 16384); });
    snprintf(nm, sizeof nm, "write TMA bulk 16KB grid %d", g);
    run(nm, bytes, [&](int it) { k_write_bulk<<<g, 128>>>(ob(it), bytes / 16384); });
  }
  run("cudaMemsetAsync", bytes, [&](int it) { cudaMemsetAsync(ob(it), 1, bytes); });
  // gather with a power-law slot stream
  std::mt19937_64 rng(1);
  std::vector<double> cdf(slots);
  double acc = 0;
  for (uint64_t r = 0; r < slots; ++r) cdf[r] = (acc += std::pow(double(r + 1), -1.2));
  for (auto& x : cdf) x /= acc;
  std::vector<uint32_t> perm(slots);
  for (uint64_t i = 0; i < slots; ++i) perm[i] = uint32_t(i);
  std::shuffle(perm.begin(), perm.end(), rng);
  std::vector<uint32_t> h(uint64_t(N) * K);
  std::uniform_real_distribution<double> U01(0, 1);
  for (auto& x : h) {
    const uint64_t r = std::lower_bound(cdf.begin(), cdf.end(), U01(rng)) - cdf.begin();
    x = perm[std::min<uint64_t>(r, slots - 1)];
  }
  cudaMemcpy(slot, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  const int grid = N / 256;  // one warp per 32 positions
  run("gather 256b U=4 st", 2.0 * bytes, [&](int it) {
    k_gather8<4, false><<<grid, 256>>>(rows, slot + uint64_t(it) * N, N, reinterpret_cast<float*>(ob(it)));
  });
  run("gather 256b U=4 st.cs", 2.0 * bytes, [&](int it) {
    k_gather8<4, true><<<grid, 256>>>(rows, slot + uint64_t(it) * N, N, reinterpret_cast<float*>(ob(it)));
  });
  run("gather 256b U=8 st.cs", 2.0 * bytes, [&](int it) {
    k_gather8<8, true><<<grid, 256>>>(rows, slot + uint64_t(it) * N, N, reinterpret_cast<float*>(ob(it)));
  });
  run("gather 256b U=16 st.cs", 2.0 * bytes, [&](int it) {
    k_gather8<16, true><<<grid, 256>>>(rows, slot + uint64_t(it) * N, N, reinterpret_cast<float*>(ob(it)));
  });
  return 0;
}
