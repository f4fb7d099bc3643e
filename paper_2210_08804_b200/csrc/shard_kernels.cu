// shard_kernels.cu -- routing kernels of the key-hash-sharded mode
// (no reference counterpart: the reference has no multi-GPU
// code, the paper deploys one replica per GPU).
//
// A key's owner is (xxh64(key, kShardSeed) >> 32) % G. kShardSeed differs
// from the slabset seed: reusing the placement hash with S a multiple of G
// would leave (G-1)/G of every shard's slabsets empty.
//   k_shard_count    owners of a batch -> per-owner counts (block-aggregated)
//   k_shard_scatter  keys into per-owner send segments (+ their original
//                    positions); order inside a segment is arbitrary, the
//                    carried position undoes it
//   k_shard_unroute  rows / flags received back from the owners -> the
//                    requester's original positions (warp per row, 128-bit)
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "common.cuh"
#include "kernels.hpp"
#include "probe.cuh"

namespace hpsb {

namespace {
inline void check_launch(const char* what, uint32_t kernels) {
  note_launches(kernels);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
constexpr int kMaxShards = 64;
}  // namespace

__host__ __device__ inline uint32_t shard_of_key(uint64_t key, uint32_t world) {
  return uint32_t((xxh64_key(key, kShardSeed) >> 32) % world);
}

uint32_t shard_of(uint64_t key, uint32_t world) { return shard_of_key(key, world); }

__global__ void __launch_bounds__(256)
    k_shard_count(const uint64_t* __restrict__ keys, uint64_t n, uint32_t world,
                  unsigned long long* __restrict__ counts) {
  __shared__ uint32_t s_cnt[kMaxShards];
  for (uint32_t i = threadIdx.x; i < world; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(&s_cnt[shard_of_key(keys[i], world)], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < world; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(counts + i, (unsigned long long)s_cnt[i]);
}

__global__ void __launch_bounds__(256)
    k_shard_scatter(const uint64_t* __restrict__ keys, uint64_t n, uint32_t world,
                    unsigned long long* __restrict__ cursor, uint64_t* __restrict__ send_keys,
                    uint32_t* __restrict__ send_pos) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  const uint32_t o = shard_of_key(k, world);
  // warp-aggregated slot claims per owner
  const uint32_t peers = __match_any_sync(__activemask(), o);
  const uint32_t leader = __ffs(peers) - 1;
  unsigned long long at = 0;
  if (lane_id() == leader) at = atomicAdd(cursor + o, (unsigned long long)__popc(peers));
  at = __shfl_sync(peers, at, leader);
  const uint64_t j = at + __popc(peers & ((1u << lane_id()) - 1u));
  send_keys[j] = k;
  send_pos[j] = uint32_t(i);
}

__global__ void __launch_bounds__(256)
    k_shard_unroute(uint64_t m, uint32_t d, const uint32_t* __restrict__ send_pos,
                    const float* __restrict__ rows, const uint8_t* __restrict__ flags_in,
                    float* __restrict__ out, uint8_t* __restrict__ flags_out) {
  const uint64_t j = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (j >= m) return;
  const uint32_t p = send_pos[j];
  warp_copy_row(rows + j * d, out + uint64_t(p) * d, d);
  if (lane_id() == 0 && flags_out != nullptr) flags_out[p] = flags_in[j];
}

void launch_shard_count(const uint64_t* keys, uint64_t n, uint32_t world,
                        unsigned long long* counts, cudaStream_t st) {
  if (world == 0 || world > kMaxShards) throw std::invalid_argument("shard count out of range");
  cudaMemsetAsync(counts, 0, world * 8, st);
  if (n == 0) return;
  const unsigned grid = unsigned(std::min<uint64_t>((n + 255) / 256, 148 * 8));
  k_shard_count<<<grid, 256, 0, st>>>(keys, n, world, counts);
  check_launch("shard_count", 1);
}

void launch_shard_scatter(const uint64_t* keys, uint64_t n, uint32_t world,
                          unsigned long long* cursor, uint64_t* send_keys, uint32_t* send_pos,
                          cudaStream_t st) {
  if (n == 0) return;
  k_shard_scatter<<<unsigned((n + 255) / 256), 256, 0, st>>>(keys, n, world, cursor, send_keys,
                                                             send_pos);
  check_launch("shard_scatter", 1);
}

void launch_shard_unroute(uint64_t m, uint32_t d, const uint32_t* send_pos, const float* rows,
                          const uint8_t* flags_in, float* out, uint8_t* flags_out,
                          cudaStream_t st) {
  if (m == 0) return;
  k_shard_unroute<<<unsigned((m * 32 + 255) / 256), 256, 0, st>>>(m, d, send_pos, rows, flags_in,
                                                                  out, flags_out);
  check_launch("shard_unroute", 1);
}

}  // namespace hpsb
