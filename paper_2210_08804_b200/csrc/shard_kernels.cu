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
#include <type_traits>
#include <string>

#include "common.cuh"
#include "kernels.hpp"
#include "peer.hpp"
#include "probe.cuh"
#include "tag_probe.cuh"

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

// ------------------------------------------------ peer-memory lookup --
// Lane per position (peer.hpp): owner = shard_of(key); the owner's slabs are
// probed through its mapped memory (fingerprints + masks in one round trip,
// key verification -- tag_probe.cuh), a hit stamps the owner's counter
// (atomicMax, one lane per distinct (owner, slot) of the warp) and the
// owner's row is read straight into the local output (a warp streams its 32
// rows, 4 rows in flight); a miss writes the default row, sets the flag and
// appends the key once per warp to the owner's inbox.
// One tick of every owner's clock for a call (slab_cache.cpp:73-74).
// The lookup is launched as its programmatic dependent: it may start at once
// and waits for the stamps only after its probe.
__global__ void k_peer_stamps(const PeerShard* __restrict__ shards, uint32_t world,
                              unsigned long long* __restrict__ stamps) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t g = threadIdx.x;
  if (g < world) stamps[g] = atomicAdd(shards[g].clock, 1ull) + 1ull;
}

__global__ void __launch_bounds__(256, 3)
    k_peer_lookup(const PeerShard* __restrict__ shards, uint32_t world,
                  const uint64_t* __restrict__ keys, uint64_t n, float* __restrict__ out,
                  uint8_t* __restrict__ flags, const float* __restrict__ default_row, uint32_t d,
                  const unsigned long long* __restrict__ stamps) {
  __shared__ PeerShard s_sh[kMaxPeers];
  for (uint32_t i = threadIdx.x; i < world; i += blockDim.x) s_sh[i] = shards[i];
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint64_t pos = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t base = pos - lane;
  if (base >= n) return;  // whole warp past the end
  const bool valid = pos < n;
  const uint64_t key = valid ? keys[pos] : 0ull;
  const uint32_t owner = valid ? shard_of_key(key, world) : 0u;
  const PeerShard& sh = s_sh[owner];
  const uint32_t res = lane_probe(sh.c, key, valid);
  const bool hit = res != kNoSlot;
  // recency: one atomic per distinct (owner, slot) of the warp, with the
  // call's tick of the owner's clock (the stamps kernel has completed and
  // its writes are visible after the grid-dependency wait)
  const uint64_t tag = hit ? ((uint64_t(owner) << 32) | res) : ~0ull;
  const uint32_t same = __match_any_sync(0xFFFFFFFFu, tag);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (hit && (__ffs(same) - 1) == lane) {
    // read first: a hot slot is hit by nearly every warp of the call, and
    // same-line atomics serialise in its L2 slice (as in the local lookup)
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(sh.c.counters) + res;
    const unsigned long long st = stamps[owner];
    if (__ldcg(ctr) < st) atomicMax(ctr, st);
  }
  // misses: one inbox entry per distinct key of the warp, reserved with one
  // add per (warp, owner) on the owner's inbox counter
  const bool miss = valid && !hit;
  // (every lane runs the warp-collective calls: no short-circuit around them)
  const uint32_t same_key = __match_any_sync(0xFFFFFFFFu, miss ? key : 0ull);
  const uint32_t missing = __ballot_sync(0xFFFFFFFFu, miss);
  const bool lead_miss = miss && (__ffs(same_key & missing) - 1) == lane;
  const uint32_t same_owner = __match_any_sync(0xFFFFFFFFu, lead_miss ? owner : ~0u);
  const uint32_t grp = same_owner & __ballot_sync(0xFFFFFFFFu, lead_miss);
  if (lead_miss) {
    const uint32_t first = __ffs(grp) - 1;
    unsigned long long at = 0;
    if (lane == first) at = atomicAdd(sh.inbox_count, (unsigned long long)__popc(grp));
    at = __shfl_sync(grp, at, first) + __popc(grp & ((1u << lane) - 1u));
    if (at < sh.inbox_cap) sh.inbox_keys[at] = key;
  }
  if (valid) flags[pos] = miss ? 1 : 0;
  // rows: the warp's 32 output rows are one contiguous block; lane i's row
  // comes from its owner's shard (or the default row). 256-bit chunks, U in
  // flight per lane (d % 8 == 0), else 128-bit / scalar.
  const float* src = hit ? sh.c.rows + uint64_t(res) * d : default_row;
  const uint32_t nrows = n - base < 32 ? uint32_t(n - base) : 32u;
  float* obase = out + base * d;
  const uintptr_t sp = reinterpret_cast<uintptr_t>(src);
  auto copy = [&](auto chunk_tag, auto u_tag) {
    using Ch = decltype(chunk_tag);
    constexpr int CH = sizeof(Ch) / 4;
    constexpr int U = decltype(u_tag)::value;
    const uint32_t cpr = d / CH;
    const uint32_t total = nrows * cpr;
    for (uint32_t c0 = 0; c0 < total; c0 += 32 * U) {
      Ch x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t ch = c0 + uint32_t(u) * 32 + lane;
        const uint32_t row = min(ch / cpr, 31u);
        const float* rs = reinterpret_cast<const float*>(__shfl_sync(0xFFFFFFFFu, sp, row));
        if (ch < total) x[u].load(rs + (ch - row * cpr) * CH);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t ch = c0 + uint32_t(u) * 32 + lane;
        if (ch < total) x[u].store(obase + uint64_t(ch) * CH);
      }
    }
  };
  const bool al32 = (d & 7u) == 0 && (reinterpret_cast<uintptr_t>(out) & 31u) == 0 &&
                    (reinterpret_cast<uintptr_t>(default_row) & 31u) == 0;
  const bool al16 = (d & 3u) == 0 && (reinterpret_cast<uintptr_t>(out) & 15u) == 0 &&
                    (reinterpret_cast<uintptr_t>(default_row) & 15u) == 0;
  if (al32)
    copy(Chunk<8>{}, std::integral_constant<int, 4>{});
  else if (al16)
    copy(Chunk<4>{}, std::integral_constant<int, 8>{});
  else
    copy(Chunk<1>{}, std::integral_constant<int, 8>{});
}

void launch_peer_lookup(const PeerShard* d_shards, uint32_t world, const uint64_t* keys,
                        uint64_t n, float* out, uint8_t* flags, const float* default_row,
                        uint32_t d, unsigned long long* d_stamps, cudaStream_t st) {
  // every call ticks the owners' clocks, even an empty one (a query bumps
  // the clock before anything else, slab_cache.cpp:73-74)
  k_peer_stamps<<<1, kMaxPeers, 0, st>>>(d_shards, world, d_stamps);
  if (n == 0) {
    check_launch("peer_lookup", 1);
    return;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned((n + 255) / 256));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_peer_lookup, static_cast<const PeerShard*>(d_shards), world, keys, n,
                     out, flags, default_row, d,
                     static_cast<const unsigned long long*>(d_stamps));
  check_launch("peer_lookup", 2);
}

}  // namespace hpsb
