// common.cuh -- shared device/host vocabulary for the B200 lookup path.
//
// * XXH64 of an 8-byte little-endian key, restated for the one-stripe case
//   of the reference (xxhash64.hpp:60-124 with length 8): one round of the
//   8-byte lane loop plus the avalanche. Pinned by tests against the
//   reference's golden vectors (test_core.cpp:26-48).
// * The device view of the slab table.
// * Decoupled look-back tile prefix (single-pass ordered compaction).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hpsb {

constexpr uint32_t kSlotsPerSlab = 32;  // slab_cache.hpp:25
constexpr uint64_t kSlabsetSeed = 0x5EED5E7ull;  // xxhash64.hpp:127
constexpr uint64_t kSlabSeed = 0x51ABull;        // xxhash64.hpp:128
constexpr uint64_t kPartitionSeed = 0ull;        // xxhash64.hpp:129
constexpr uint64_t kShardSeed = 0x5A4D5EEDull;   // sharded mode owner hash (ours)
constexpr uint32_t kFullSlab = 0xFFFFFFFFu;

constexpr uint64_t kP1 = 0x9E3779B185EBCA87ull;
constexpr uint64_t kP2 = 0xC2B2AE3D27D4EB4Full;
constexpr uint64_t kP3 = 0x165667B19E3779F9ull;
constexpr uint64_t kP4 = 0x85EBCA77C2B2AE63ull;
constexpr uint64_t kP5 = 0x27D4EB2F165667C5ull;

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int r) {
  return (x << r) | (x >> (64 - r));
}

// xxh64 over the 8 LE bytes of `key` (xxhash64.hpp:86-113 with length 8).
__host__ __device__ __forceinline__ uint64_t xxh64_key(uint64_t key, uint64_t seed) {
  uint64_t h = seed + kP5 + 8ull;
  h ^= rotl64(key * kP2, 31) * kP1;
  h = rotl64(h, 27) * kP1 + kP4;
  h ^= h >> 33;
  h *= kP2;
  h ^= h >> 29;
  h *= kP3;
  h ^= h >> 32;
  return h;
}

// Internal (non-placement) table hash: murmur3 fmix64. Only used for the
// per-call scratch hash tables, never for placement.
__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

// Device view of one cache replica. Layout in HBM (structure of arrays, one
// allocation each, slab-contiguous):
//   keys     [S][W][32] u64   256 B per slab = two 128 B lines
//   counters [S][W][32] u64   recency stamps
//   masks    [S][W]     u32   occupancy bits, grow contiguously from bit 0
//   tags     [S][W][32] u8    8-bit fingerprint of each stored key (probe
//                             filter of the lookup kernel; 64 B per W=2 set,
//                             one 256-bit load per slab)
//   rows     [S][W][32][d] f32
struct CacheDev {
  uint64_t* keys;
  uint64_t* counters;
  uint32_t* masks;
  uint8_t* tags;
  float* rows;
  unsigned long long* occupied;
  uint64_t S;
  uint32_t W;
  uint32_t d;
  uint64_t mS;  // floor((2^64 - 1) / S): Barrett reciprocal for h % S
  uint64_t mW;  // same for W
};

// h % m without a 64-bit divide: q = mulhi(h, floor((2^64-1)/m)) is at most
// two below floor(h / m), so at most two corrections.
__host__ __device__ __forceinline__ uint64_t fastmod(uint64_t h, uint64_t m, uint64_t recip) {
#ifdef __CUDA_ARCH__
  const uint64_t q = __umul64hi(h, recip);
#else
  const uint64_t q = uint64_t((unsigned __int128)h * recip >> 64);
#endif
  uint64_t r = h - q * m;
  if (r >= m) r -= m;
  if (r >= m) r -= m;
  return r;
}

__host__ __device__ __forceinline__ uint64_t slabset_of(const CacheDev& c, uint64_t key) {
  return fastmod(xxh64_key(key, kSlabsetSeed), c.S, c.mS);
}
__host__ __device__ __forceinline__ uint32_t first_slab_of(const CacheDev& c, uint64_t key) {
  return uint32_t(fastmod(xxh64_key(key, kSlabSeed), c.W, c.mW));
}

// Fingerprint of a key: the top byte of its first-slab hash (the slab
// choice uses h % W, i.e. the low bits for power-of-two W). Maintained by
// replace next to the key; never part of the reference's state.
__host__ __device__ __forceinline__ uint8_t key_tag(uint64_t first_slab_hash) {
  return uint8_t(first_slab_hash >> 56);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// ---- decoupled look-back (single pass ordered prefix across tiles) ----
// Status word per tile: [63:40] epoch (24 bits) | [39:38] flag | [37:0] value.
// flag 1 = tile aggregate available, 2 = inclusive prefix available. Words
// from an older epoch read as "not yet published", so the status array
// never needs clearing (the host re-zeroes it when the 24-bit epoch wraps).
constexpr uint64_t kLbValueMask = (1ull << 38) - 1;

__device__ __forceinline__ uint64_t lb_pack(uint32_t epoch, uint32_t flag, uint64_t v) {
  return (uint64_t(epoch & 0xFFFFFFu) << 40) | (uint64_t(flag) << 38) | (v & kLbValueMask);
}

__device__ __forceinline__ void lb_store(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t lb_load(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Called by warp 0 of the block (all 32 lanes) once the tile aggregate is
// known; returns the exclusive prefix of this tile. Warp-parallel look-back
// over 32 predecessors at a time.
__device__ __forceinline__ uint64_t lb_exclusive_prefix(uint64_t* status, uint32_t tile,
                                                        uint32_t epoch, uint64_t aggregate) {
  const uint32_t lane = lane_id();
  const uint32_t ep = epoch & 0xFFFFFFu;
  if (tile == 0) {
    if (lane == 0) lb_store(status, lb_pack(ep, 2, aggregate));
    return 0;
  }
  if (lane == 0) lb_store(status + tile, lb_pack(ep, 1, aggregate));
  uint64_t exclusive = 0;
  int32_t window_end = int32_t(tile) - 1;  // highest predecessor not yet folded
  while (true) {
    const int32_t t = window_end - int32_t(lane);
    uint64_t w = 0;
    uint32_t flag = 2;  // lanes past tile 0 act as a zero inclusive prefix
    uint64_t val = 0;
    if (t >= 0) {
      do {
        w = lb_load(status + t);
        flag = (uint32_t(w >> 40) == ep) ? uint32_t((w >> 38) & 3u) : 0u;
      } while (flag == 0);
      val = w & kLbValueMask;
    }
    // the first lane (lowest lane index = nearest predecessor) holding an
    // inclusive prefix ends the look-back
    const uint32_t incl = __ballot_sync(0xFFFFFFFFu, flag == 2);
    const uint32_t stop = __ffs(incl) - 1;  // incl != 0 guaranteed? not always
    uint64_t contrib = (incl != 0) ? ((lane <= stop) ? val : 0) : val;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xFFFFFFFFu, contrib, o);
    exclusive += contrib;
    if (incl != 0) break;
    window_end -= 32;
  }
  if (lane == 0) lb_store(status + tile, lb_pack(ep, 2, exclusive + aggregate));
  return exclusive;
}

// Block-wide exclusive scan of one u32 per thread (BLOCK threads). Returns
// the thread's exclusive prefix within the block; *total gets the block sum.
template <int BLOCK>
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* smem_warp,
                                                         uint32_t* total) {
  constexpr int NW = BLOCK / 32;
  const uint32_t lane = lane_id();
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= uint32_t(o)) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = (lane < NW) ? smem_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= uint32_t(o)) w += y;
    }
    if (lane < NW) smem_warp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t warp_base = (warp == 0) ? 0 : smem_warp[warp - 1];
  *total = smem_warp[NW - 1];
  return warp_base + x - v;
}

}  // namespace hpsb
