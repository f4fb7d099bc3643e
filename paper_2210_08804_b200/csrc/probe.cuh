// probe.cuh -- warp-cooperative slab probe shared by query / update / lookup.
//
// Restates the reference probe (slab_cache.cpp:236-256, apply_query): probe
// slabs (first + step) % W, match only occupied slots, stop at the first
// slab that is not full. One warp serves P positions at once: lane j reads
// slot j of each position's slab (one coalesced 256 B read per slab) and
// __ballot_sync / __ffs pick the matching slot. The P probes of a round are
// issued back to back so the warp keeps P slab reads in flight.
#pragma once

#include "common.cuh"
#include "kernels.hpp"

namespace hpsb {

// Per-position placement, computed by lanes 0..P-1 in parallel and
// broadcast to the warp.
// Slot indices are u32 (the cache holds < 2^32 slots, checked at creation).
constexpr uint32_t kNoSlot = 0xFFFFFFFFu;

template <int P>
struct WarpKeys {
  uint64_t key[P];
  uint32_t set[P];
  uint32_t first[P];
  bool valid[P];
};

// Lanes 0..P-1 hash their own key; the placement is broadcast.
template <int P>
__device__ __forceinline__ void warp_place_keys(const CacheDev& c, uint64_t k, uint64_t base,
                                                uint64_t n, WarpKeys<P>& wk) {
  const uint32_t lane = lane_id();
  uint32_t s = 0, f = 0;
  if (lane < uint32_t(P)) {
    s = uint32_t(slabset_of(c, k));
    f = first_slab_of(c, k);
  }
#pragma unroll
  for (int p = 0; p < P; ++p) {
    wk.key[p] = __shfl_sync(0xFFFFFFFFu, k, p);
    wk.set[p] = __shfl_sync(0xFFFFFFFFu, s, p);
    wk.first[p] = __shfl_sync(0xFFFFFFFFu, f, p);
    wk.valid[p] = (base + p) < n;
  }
}

template <int P>
__device__ __forceinline__ void warp_load_keys(const CacheDev& c, const uint64_t* __restrict__ keys,
                                               uint64_t base, uint64_t n, WarpKeys<P>& wk) {
  const uint32_t lane = lane_id();
  const uint64_t k = (lane < uint32_t(P) && base + lane < n) ? keys[base + lane] : 0ull;
  warp_place_keys<P>(c, k, base, n, wk);
}

// slot[p] = global slot index of key p, or kNoSlot. Warp-uniform results.
template <int P>
__device__ __forceinline__ void warp_probe(const CacheDev& c, const WarpKeys<P>& wk,
                                           uint32_t (&slot)[P]) {
  const uint32_t lane = lane_id();
  bool pending[P];
#pragma unroll
  for (int p = 0; p < P; ++p) {
    pending[p] = wk.valid[p];
    slot[p] = kNoSlot;
  }
  for (uint32_t step = 0; step < c.W; ++step) {
    uint64_t sk[P];
    uint32_t m[P];
    uint32_t slab[P];
    bool any = false;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (pending[p]) {
        uint32_t sl = wk.first[p] + step;
        sl = (sl >= c.W) ? sl - c.W : sl;
        slab[p] = wk.set[p] * c.W + sl;
        m[p] = c.masks[slab[p]];
        sk[p] = c.keys[uint64_t(slab[p]) * kSlotsPerSlab + lane];
        any = true;
      }
    }
    if (!any) break;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (pending[p]) {
        const uint32_t b =
            __ballot_sync(0xFFFFFFFFu, ((m[p] >> lane) & 1u) && sk[p] == wk.key[p]);
        if (b) {
          slot[p] = slab[p] * kSlotsPerSlab + (__ffs(b) - 1);
          pending[p] = false;
        } else if (m[p] != kFullSlab) {
          pending[p] = false;  // a free slot before the key: not resident
        }
      }
    }
  }
}

// Warp copy of one d-float row. Vector path when d % 4 == 0 (rows are
// 16 B aligned then); lanes stride over float4 chunks.
__device__ __forceinline__ void warp_copy_row(const float* __restrict__ src, float* __restrict__ dst,
                                              uint32_t d) {
  const uint32_t lane = lane_id();
  if ((d & 3u) == 0) {
    const uint32_t d4 = d >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* o4 = reinterpret_cast<float4*>(dst);
    for (uint32_t c = lane; c < d4; c += 32) o4[c] = s4[c];
  } else {
    for (uint32_t c = lane; c < d; c += 32) dst[c] = src[c];
  }
}

// ---------------------------------------------------- ordered selection --
// Generic single-pass stable selection: tile of kScanBlock threads x
// kScanItems consecutive items per thread (blocked arrangement keeps input
// order), block scan + decoupled look-back across tiles.
template <class Pred, class Emit>
__device__ __forceinline__ void select_tile(uint64_t n, ScanState scan, Pred pred, Emit emit,
                                            unsigned long long* total_out) {
  __shared__ uint32_t s_warp[kScanBlock / 32];
  __shared__ uint64_t s_tile;
  __shared__ uint64_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(scan.tile_ctr, 1ull) - scan.tile_base;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t first = tile * kScanTile + uint64_t(threadIdx.x) * kScanItems;
  bool sel[kScanItems];
  uint32_t cnt = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint64_t i = first + k;
    sel[k] = (i < n) && pred(i);
    cnt += sel[k] ? 1u : 0u;
  }
  uint32_t block_total;
  const uint32_t excl = block_exclusive_scan<kScanBlock>(cnt, s_warp, &block_total);
  if (threadIdx.x < 32) {
    const uint64_t pre = lb_exclusive_prefix(scan.status, uint32_t(tile), scan.epoch, block_total);
    if (threadIdx.x == 0) {
      s_prefix = pre;
      const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
      if (total_out != nullptr && tile == tiles - 1) *total_out = pre + block_total;
    }
  }
  __syncthreads();
  uint64_t r = s_prefix + excl;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (sel[k]) emit(first + k, r++);
  }
}


// Table entry = (epoch << 32) | position. Positions of equal keys converge
// on one entry (the key is read back from the immutable input through the
// stored position), and atomicMin keeps the first occurrence.
__device__ __forceinline__ uint32_t dedup_insert(uint64_t* table, uint64_t cap,
                                                 const uint64_t* __restrict__ keys, uint64_t key,
                                                 uint32_t pos, uint32_t epoch, bool* claimed) {
  const uint64_t mine = (uint64_t(epoch) << 32) | pos;
  uint64_t t = fmix64(key ^ 0x9E3779B97F4A7C15ull) & (cap - 1);
  *claimed = false;
  while (true) {
    unsigned long long* e = reinterpret_cast<unsigned long long*>(table + t);
    unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(e);
    if (uint32_t(cur >> 32) != epoch) {
      const unsigned long long old = atomicCAS(e, cur, mine);
      if (old == cur) {
        *claimed = true;
        return uint32_t(t);
      }
      cur = old;
      if (uint32_t(cur >> 32) != epoch) continue;  // raced with another stale swap
    }
    const uint32_t other = uint32_t(cur);
    if (keys[other] == key) {
      if (pos < other) atomicMin(e, mine);
      return uint32_t(t);
    }
    t = (t + 1) & (cap - 1);
  }
}

// Lookup miss table: u32 entries, 0 = empty, else first position + 1. The
// claimer of an empty entry needs one round trip (a CAS from 0); later
// positions of the same key compare through the immutable input and keep
// the minimum position with a fire-and-forget atomicMin. The ordering tail
// clears every claimed entry, so the table is all-zero between calls.
// READ_FIRST: the entry is read (L2, never a stale L1 line) before the CAS, and
// an entry already holding this key is joined without one -- a power-law
// batch's hottest missing keys sit in nearly every warp, and ~2,000 CASes per
// call on one entry serialise in its L2 slice (the recency counters had the
// same problem, §5).
#ifndef HPSB_CLAIM_READ_FIRST
#define HPSB_CLAIM_READ_FIRST 1
#endif
__device__ __forceinline__ uint32_t miss_insert(uint32_t* table, uint64_t cap,
                                                const uint64_t* __restrict__ keys, uint64_t key,
                                                uint32_t pos, bool* claimed) {
  uint64_t t = fmix64(key ^ 0x9E3779B97F4A7C15ull) & (cap - 1);
  const uint32_t mine = pos + 1;
  while (true) {
#if HPSB_CLAIM_READ_FIRST
    const uint32_t seen = __ldcg(table + t);
    if (seen != 0u) {
      if (keys[seen - 1] == key) {
        *claimed = false;
        if (mine < seen) atomicMin(table + t, mine);
        return uint32_t(t);
      }
      t = (t + 1) & (cap - 1);
      continue;
    }
#endif
    const uint32_t old = atomicCAS(table + t, 0u, mine);
    if (old == 0u) {
      *claimed = true;
      return uint32_t(t);
    }
    if (keys[old - 1] == key) {
      *claimed = false;
      if (mine < old) atomicMin(table + t, mine);
      return uint32_t(t);
    }
    t = (t + 1) & (cap - 1);
  }
}

}  // namespace hpsb
