// tag_probe.cuh -- lane-per-position fingerprint probe and vector accessors
// shared by the lookup (lookup_kernels.cu) and update (cache_kernels.cu)
// kernels.
//
// Probe rule restated (slab_cache.cpp:236-256): probe slabs (first + step)
// % W, match only occupied slots, the lowest matching slot wins, and stop at
// the first slab that is not full. Here one lane serves one position: it
// reads the set's 8-bit fingerprints (32 B per slab, 256-bit loads) and the
// occupancy masks, and verifies byte-equal candidates against the stored
// key. A key is stored at most once per set, so the first verified candidate
// in slot order is the reference's hit.
#pragma once

#include "common.cuh"
#include "probe.cuh"

namespace hpsb {

// Row loads: non-coherent path with L1 allocation (the table does not change
// during a lookup; repeated hot rows are served from the SM's L1).
__device__ __forceinline__ float4 ld_row_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
// Output rows are written once and not re-read here: evict-first.
__device__ __forceinline__ void st_cs_f4(float4* p, const float4& v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
#ifndef HPSB_ROW_LOAD
#define HPSB_ROW_LOAD ""
#endif
__device__ __forceinline__ void ld256_nc(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc" HPSB_ROW_LOAD ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
// Output rows are written once and never re-read here: no L1 allocation and
// evict-first in L2 (vs .cs: cfg 2 +2 %, profiles/r01_ab_history.txt).
__device__ __forceinline__ void st256_cs(void* p, const uint32_t (&r)[8]) {
  asm volatile(
      "st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
// Bit j set when byte j of the 32-byte fingerprint block may equal `tag`
// (zero-byte test on w ^ tag; it can over-report -- verified against the
// key -- but never misses an equal byte).
__device__ __forceinline__ uint32_t tag_candidates(const uint32_t (&w)[8], uint32_t tag4) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t x = w[i] ^ tag4;
    const uint32_t z = (x - 0x01010101u) & ~x & 0x80808080u;
    m |= ((z * 0x00204081u) >> 28) << (4 * i);
  }
  return m;
}

// Placement + fingerprint probe of one position. Returns the global slot of
// `key` or kNoSlot.
__device__ __forceinline__ uint32_t lane_probe(const CacheDev& c, uint64_t key, bool valid) {
  const uint64_t h2 = xxh64_key(key, kSlabSeed);
  const uint32_t set = uint32_t(slabset_of(c, key));
  const uint32_t first = c.W == 2 ? uint32_t(h2 & 1u) : uint32_t(fastmod(h2, c.W, c.mW));
  const uint32_t tag4 = uint32_t(key_tag(h2)) * 0x01010101u;
  if (!valid) return kNoSlot;
  const unsigned long long* ck = reinterpret_cast<const unsigned long long*>(c.keys);
  if (c.W == 2) {
    // both slabs' fingerprints and masks in one round trip
    uint32_t t0[8], t1[8];
    const uint8_t* tp = c.tags + uint64_t(set) * 64;
    ld256_nc(tp, t0);
    ld256_nc(tp + 32, t1);
    const uint2 mm = __ldg(reinterpret_cast<const uint2*>(c.masks) + set);
    const uint32_t c0 = tag_candidates(t0, tag4) & mm.x;
    const uint32_t c1 = tag_candidates(t1, tag4) & mm.y;
    // probe order: slab `first`, then the other one only if `first` is full
    const uint32_t ma = first ? mm.y : mm.x;
    const uint32_t ca = first ? c1 : c0;
    const uint32_t cb = (ma == kFullSlab) ? (first ? c0 : c1) : 0u;
    const uint32_t sa = (set * 2 + first) * kSlotsPerSlab;
    const uint32_t sb = (set * 2 + (first ^ 1u)) * kSlotsPerSlab;
    uint64_t cand = uint64_t(ca) | (uint64_t(cb) << 32);
    while (cand) {
      // two candidates per round trip
      const uint32_t b1 = __ffsll(cand) - 1;
      cand &= cand - 1;
      const uint32_t s1 = b1 < 32 ? sa + b1 : sb + (b1 - 32);
      uint32_t s2 = kNoSlot;
      if (cand) {
        const uint32_t b2 = __ffsll(cand) - 1;
        cand &= cand - 1;
        s2 = b2 < 32 ? sa + b2 : sb + (b2 - 32);
      }
      const uint64_t k1 = __ldg(ck + s1);
      const uint64_t k2 = s2 != kNoSlot ? __ldg(ck + s2) : ~key;
      if (k1 == key) return s1;
      if (k2 == key) return s2;
    }
    return kNoSlot;
  }
  // general W: slab by slab in probe order, stop at a hit or at the first
  // slab that is not full
  for (uint32_t step = 0; step < c.W; ++step) {
    uint32_t sl = first + step;
    sl = (sl >= c.W) ? sl - c.W : sl;
    const uint32_t slab = set * c.W + sl;
    uint32_t t[8];
    ld256_nc(c.tags + uint64_t(slab) * 32, t);
    const uint32_t m = __ldg(c.masks + slab);
    uint32_t cand = tag_candidates(t, tag4) & m;
    while (cand) {
      const uint32_t b = __ffs(cand) - 1;
      cand &= cand - 1;
      const uint32_t s = slab * kSlotsPerSlab + b;
      if (__ldg(ck + s) == key) return s;
    }
    if (m != kFullSlab) break;
  }
  return kNoSlot;
}


// Row chunk of CH floats: 8 = 256-bit, 4 = 128-bit, 1 = scalar accesses;
// store() is evict-first (streamed outputs), store_wb() write-back.
template <int CH>
struct Chunk;
template <>
struct Chunk<8> {
  uint32_t x[8];
  __device__ __forceinline__ void load(const float* p) { ld256_nc(p, x); }
  __device__ __forceinline__ void store(float* p) const { st256_cs(p, x); }
  __device__ __forceinline__ void store_wb(float* p) const {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(x[0]),
                 "r"(x[1]), "r"(x[2]), "r"(x[3]), "r"(x[4]), "r"(x[5]), "r"(x[6]), "r"(x[7])
                 : "memory");
  }
};
template <>
struct Chunk<4> {
  float4 x;
  __device__ __forceinline__ void load(const float* p) {
    x = ld_row_f4(reinterpret_cast<const float4*>(p));
  }
  __device__ __forceinline__ void store(float* p) const {
    st_cs_f4(reinterpret_cast<float4*>(p), x);
  }
  __device__ __forceinline__ void store_wb(float* p) const { *reinterpret_cast<float4*>(p) = x; }
};
template <>
struct Chunk<1> {
  float x;
  __device__ __forceinline__ void load(const float* p) { x = __ldg(p); }
  __device__ __forceinline__ void store(float* p) const { __stcs(p, x); }
  __device__ __forceinline__ void store_wb(float* p) const { *p = x; }
};

}  // namespace hpsb
