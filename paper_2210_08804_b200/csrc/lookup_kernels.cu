// lookup_kernels.cu -- the lookup hot path (sm_100a).
//
// Restates LookupEngine::lookup (lookup_engine.cpp:130-241) for a batch of
// |Q| query positions:
//
//   k_lookup    a warp serves 8 positions, 4 lanes per position, so each
//               position's dependent chain is short: key load, both
//               placement hashes (XXH64 + Barrett modulo), ONE round trip
//               for both probe slabs and masks (each lane compares 8 of a
//               slab's 32 keys loaded as 128-bit vectors; a 4-lane min picks
//               the lowest matching slot -- the ballot/ffs rule of
//               slab_cache.cpp:240-245, and the second slab only counts when
//               the first is full, :249-256), ONE round trip for the row
//               (each lane moves a quarter of it with 128-bit L1-cached
//               loads and evict-first stores) straight into the position's
//               output row: the expansion of lookup_engine.cpp:194-203 is
//               fused, and missing positions get the default row (the async
//               branch's answer, :185-192).
//               Recency: the exchange that first moves a slot to this call's
//               stamp counts one UNIQUE hit, so |Q*| needs no dedup of hits;
//               a per-block set of stamped slots keeps the hottest keys'
//               exchanges (power-law batches repeat their top key in ~19% of
//               positions) off a single L2 line.
//               Misses: the group leader inserts the key into a per-call
//               miss table keeping the minimum position; the position that
//               claims an empty entry appends a claim (slot, key).
//   k_finalize  per claim: first position = table entry, entry cleared for
//               the next call; per-call counts. Sorting claims by first
//               position gives the reference's miss order -- the engine does
//               it on the host, where the tiers are.
//   k_scatter   (sync branch only) copies the rows fetched from the tiers
//               into every position of their key and clears the default
//               flag (lookup_engine.cpp:165-181).
#include <cuda_runtime.h>

#include <cstdlib>
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
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
  }
}
inline uint64_t a256(uint64_t v) { return (v + 255) / 256 * 256; }
inline uint64_t table_cap(uint64_t cap) {
  uint64_t t = 16;
  while (t < 2 * cap) t <<= 1;
  return t;
}
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kSetBits = 7;       // 128-entry per-block stamped-slot set (64 positions)
constexpr uint32_t kCountLanes = 64;  // distributed (unique hit, unique miss) counter pairs
}  // namespace

size_t lookup_scratch_bytes(uint64_t cap) {
  const uint64_t tcap = table_cap(cap);
  return a256(tcap * 4) * 2 + a256(cap * 4) * 3 + a256(cap * 8) + a256(kCountLanes * 16) +
         a256(64);
}

LookupScratch lookup_scratch_carve(void* base, uint64_t cap) {
  LookupScratch ls;
  const uint64_t tcap = table_cap(cap);
  char* p = static_cast<char*>(base);
  auto take = [&](uint64_t b) {
    char* r = p;
    p += a256(b);
    return r;
  };
  ls.cap = tcap;
  ls.miss_table = reinterpret_cast<uint32_t*>(take(tcap * 4));
  ls.claim_of_slot = reinterpret_cast<uint32_t*>(take(tcap * 4));
  ls.miss_slot = reinterpret_cast<uint32_t*>(take(cap * 4));
  ls.list = reinterpret_cast<uint32_t*>(take(cap * 4));
  ls.list_firsts = reinterpret_cast<uint32_t*>(take(cap * 4));
  ls.list_keys = reinterpret_cast<uint64_t*>(take(cap * 8));
  ls.counts = reinterpret_cast<unsigned long long*>(take(kCountLanes * 16));
  unsigned long long* small = reinterpret_cast<unsigned long long*>(take(64));
  ls.counts_prev = small;  // [0..1] cumulative totals at the previous call
  ls.list_ctr = reinterpret_cast<uint32_t*>(small + 2);  // [2] u32
  return ls;
}

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

// Probe one slab for `key` with L lanes per position (this lane checks keys
// sub*K .. sub*K+K-1, K = 32/L). Returns the lowest matching slot index in
// the slab (0..31) or 32.
template <int L>
__device__ __forceinline__ uint32_t quad_match(const uint64_t (&kk)[32 / L], uint32_t m,
                                               uint64_t key, uint32_t sub) {
  constexpr int K = 32 / L;
  uint32_t h = 32;
#pragma unroll
  for (int j = K - 1; j >= 0; --j) {
    const uint32_t s = sub * K + j;
    if (((m >> s) & 1u) && kk[j] == key) h = s;
  }
#pragma unroll
  for (int o = 1; o < L; o <<= 1) h = min(h, __shfl_xor_sync(0xFFFFFFFFu, h, o));
  return h;
}

template <int L>
__device__ __forceinline__ void load_slab_part(const CacheDev& c, uint32_t slab, uint32_t sub,
                                               uint64_t (&kk)[32 / L]) {
  constexpr int K = 32 / L;
  const ulonglong2* p2 =
      reinterpret_cast<const ulonglong2*>(c.keys + uint64_t(slab) * kSlotsPerSlab) + sub * (K / 2);
#pragma unroll
  for (int j = 0; j < K / 2; ++j) {
    const ulonglong2 v = p2[j];
    kk[2 * j] = v.x;
    kk[2 * j + 1] = v.y;
  }
}

// L = lanes per position (4 or 8): a warp serves 32/L positions.
template <int L>
__global__ void __launch_bounds__(kThreads)
    k_lookup(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n, float* __restrict__ out,
             uint8_t* __restrict__ flags, const float* __restrict__ default_row, uint64_t stamp,
             LookupScratch ls, uint32_t parity) {
  constexpr int K = 32 / L;   // keys of a slab per lane
  constexpr int POS = 32 / L; // positions per warp
  constexpr int RC = 32 / L;  // float4 chunks per lane per 128-float row segment
  __shared__ uint32_t s_stamped[1u << kSetBits];
  for (uint32_t i = threadIdx.x; i < (1u << kSetBits); i += blockDim.x) s_stamped[i] = kNoSlot;
  // the other parity's claim counter belongs to the next call: reset it
  if (blockIdx.x == 0 && threadIdx.x == 0) ls.list_ctr[parity ^ 1u] = 0;
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint32_t q = lane / L, sub = lane % L;
  const uint64_t pos = ((uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5) * POS + q;
  const bool valid = pos < n;
  const uint64_t key = valid ? keys[pos] : 0ull;
  // ---- placement and probe ----
  const uint32_t set = uint32_t(slabset_of(c, key));
  const uint32_t first = first_slab_of(c, key);
  uint32_t res = kNoSlot;
  if (c.W == 2) {
    // both probe slabs and masks in one round trip
    const uint32_t sa = set * 2 + first, sb = set * 2 + (first ^ 1u);
    uint32_t ma = 0, mb = 0;
    uint64_t ka[K], kb[K];
    if (valid) {
      ma = c.masks[sa];
      mb = c.masks[sb];
      load_slab_part<L>(c, sa, sub, ka);
      load_slab_part<L>(c, sb, sub, kb);
    }
    const uint32_t ha = quad_match<L>(ka, valid ? ma : 0u, key, sub);
    const uint32_t hb = quad_match<L>(kb, valid ? mb : 0u, key, sub);
    if (ha < 32)
      res = sa * kSlotsPerSlab + ha;
    else if (ma == kFullSlab && hb < 32)
      res = sb * kSlotsPerSlab + hb;
  } else {
    // general W: slab by slab in probe order; a group stops at a hit or at
    // the first slab that is not full
    bool pending = valid;
    for (uint32_t step = 0; step < c.W; ++step) {
      if (!__any_sync(0xFFFFFFFFu, pending)) break;
      uint32_t sl = first + step;
      sl = (sl >= c.W) ? sl - c.W : sl;
      const uint32_t slab = set * c.W + sl;
      uint32_t m = 0;
      uint64_t kk[K];
      if (pending) {
        m = c.masks[slab];
        load_slab_part<L>(c, slab, sub, kk);
      }
      const uint32_t h = quad_match<L>(kk, pending ? m : 0u, key, sub);
      if (pending) {
        if (h < 32) {
          res = slab * kSlotsPerSlab + h;
          pending = false;
        } else if (m != kFullSlab) {
          pending = false;
        }
      }
    }
  }
  // ---- recency exchange by the group's lane 0, issued before the copy ----
  unsigned long long old = stamp;
  bool stamp_it = valid && sub == 0 && res != kNoSlot;
  if (stamp_it) {
    uint32_t h = (res * 0x9E3779B1u) >> (32 - kSetBits);
    for (int probe = 0; probe < 16; ++probe) {
      const uint32_t cur = atomicCAS(&s_stamped[h], kNoSlot, res);
      if (cur == kNoSlot) break;
      if (cur == res) {
        stamp_it = false;  // this block already exchanged this slot
        break;
      }
      h = (h + 1) & ((1u << kSetBits) - 1u);
    }
  }
  if (stamp_it) old = atomicExch(reinterpret_cast<unsigned long long*>(c.counters + res), stamp);
  // ---- row copy: lane `sub` moves float4 chunks sub, sub+L, sub+2L, ... ----
  if (valid) {
    const uint32_t d = c.d;
    const float* src = res != kNoSlot ? c.rows + uint64_t(res) * d : default_row;
    float* dst = out + pos * d;
    if ((d & 3u) == 0) {
      const uint32_t d4 = d >> 2;
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* o4 = reinterpret_cast<float4*>(dst);
      for (uint32_t ch0 = 0; ch0 < d4; ch0 += L * RC) {
        float4 v[RC];
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          const uint32_t ch = ch0 + uint32_t(j) * L + sub;
          if (ch < d4) v[j] = ld_row_f4(s4 + ch);
        }
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          const uint32_t ch = ch0 + uint32_t(j) * L + sub;
          if (ch < d4) st_cs_f4(o4 + ch, v[j]);
        }
      }
    } else {
      for (uint32_t ch = sub; ch < d; ch += L) dst[ch] = src[ch];
    }
  }
  // ---- misses: the group's lane 0 claims the key; bookkeeping ----
  bool claimed = false;
  uint32_t tslot = 0;
  if (valid && sub == 0 && res == kNoSlot) {
    tslot = miss_insert(ls.miss_table, ls.cap, keys, key, uint32_t(pos), &claimed);
    ls.miss_slot[pos] = tslot;
  }
  if (valid && sub == 0) flags[pos] = res == kNoSlot ? 1 : 0;
  const uint32_t cm = __ballot_sync(0xFFFFFFFFu, claimed);
  uint32_t uh = 0, um = 0;
  if (cm) {
    const uint32_t first_lane = __ffs(cm) - 1;
    uint32_t at = 0;
    if (lane == first_lane) at = atomicAdd(ls.list_ctr + parity, uint32_t(__popc(cm)));
    at = __shfl_sync(0xFFFFFFFFu, at, first_lane);
    if (claimed) {
      const uint32_t e = at + __popc(cm & ((1u << lane) - 1u));
      ls.list[e] = tslot;
      ls.list_keys[e] = key;
      ls.claim_of_slot[tslot] = e;
    }
    um = claimed ? 1u : 0u;
  }
  if (stamp_it) uh = (old != stamp) ? 1u : 0u;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uh += __shfl_xor_sync(0xFFFFFFFFu, uh, o);
    um += __shfl_xor_sync(0xFFFFFFFFu, um, o);
  }
  // fire-and-forget adds into one of kCountLanes counter pairs (no block
  // barrier at the end, no single hot counter); finalize sums them
  if (lane == 0 && (uh | um)) {
    const uint32_t w = ((blockIdx.x * kWarps) + (threadIdx.x >> 5)) & (kCountLanes - 1);
    if (uh) atomicAdd(ls.counts + 2 * w, (unsigned long long)uh);
    if (um) atomicAdd(ls.counts + 2 * w + 1, (unsigned long long)um);
  }
  // let the finalize kernel (programmatic dependent launch) get scheduled
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Runs after k_lookup (stream order): first position of every claim, miss
// table left empty for the next call, per-call counts.
__global__ void __launch_bounds__(256)
    k_finalize(LookupScratch ls, uint32_t parity) {
  // programmatic dependent launch: wait until every lookup block is done
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t m = ls.list_ctr[parity];
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint32_t s = ls.list[e];
    ls.list_firsts[e] = ls.miss_table[s] - 1u;
    ls.miss_table[s] = 0u;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    // cumulative totals of the distributed counters -> this call's counts
    const uint32_t i = threadIdx.x & 1u;
    unsigned long long v = 0;
    for (uint32_t w = threadIdx.x >> 1; w < kCountLanes; w += 16) v += ls.counts[2 * w + i];
#pragma unroll
    for (int o = 16; o >= 2; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (threadIdx.x < 2) {
      const unsigned long long prev = ls.counts_prev[i];
      ls.counts_prev[i] = v;
      if (ls.counts_out != nullptr) ls.counts_out[i] = v - prev;
    }
  }
}

unsigned launch_lookup_probe(const CacheDev& c, const uint64_t* keys, uint64_t n, float* out,
                             uint8_t* flags, const float* default_row, uint64_t stamp,
                             const LookupScratch& ls, uint32_t parity, cudaStream_t st) {
  if (n == 0) return 0;
  // lanes per position: 8 by default (shorter per-lane state, more warps in
  // flight); HPSB_LOOKUP_LANES=4 selects the 4-lane variant
  static const int lanes = (std::getenv("HPSB_LOOKUP_LANES") &&
                            std::atoi(std::getenv("HPSB_LOOKUP_LANES")) == 4)
                               ? 4
                               : 8;
  const uint64_t per_block = uint64_t(kWarps) * (32 / lanes);
  const unsigned grid = unsigned((n + per_block - 1) / per_block);
  if (lanes == 4)
    k_lookup<4><<<grid, kThreads, 0, st>>>(c, keys, n, out, flags, default_row, stamp, ls, parity);
  else
    k_lookup<8><<<grid, kThreads, 0, st>>>(c, keys, n, out, flags, default_row, stamp, ls, parity);
  check_launch("lookup", 1);
  static const bool no_finalize = std::getenv("HPSB_DIAG_NO_FINALIZE") != nullptr;  // diagnostic
  if (no_finalize) return 1;
  // claims are at most the unique keys; one wave of small blocks covers them.
  // Programmatic dependent launch: scheduled while the lookup drains.
  const unsigned fgrid = unsigned(std::min<uint64_t>((n + 255) / 256, 148 * 4));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(fgrid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_finalize, ls, parity);
  check_launch("lookup_finalize", 1);
  return 2;
}

__global__ void __launch_bounds__(256)
    k_lookup_scatter(uint64_t n, uint32_t d, uint8_t* __restrict__ flags, LookupScratch ls,
                     const int32_t* __restrict__ row_of_claim, const float* __restrict__ staged,
                     float* __restrict__ out) {
  const uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  if (flags[i] == 0) return;
  const uint32_t e = ls.claim_of_slot[ls.miss_slot[i]];
  const int32_t r = row_of_claim[e];
  if (r < 0) return;  // absent from every tier: keep default + flag
  warp_copy_row(staged + uint64_t(r) * d, out + i * d, d);
  __syncwarp();
  if (lane_id() == 0) flags[i] = 0;
}

void launch_lookup_scatter(uint64_t n, uint32_t d, const uint8_t* flags_in, uint8_t* flags,
                           const LookupScratch& ls, const int32_t* row_of_claim,
                           const float* staged, float* out, cudaStream_t st) {
  (void)flags_in;
  if (n == 0) return;
  const uint64_t threads = n * 32;
  k_lookup_scatter<<<unsigned((threads + 255) / 256), 256, 0, st>>>(n, d, flags, ls,
                                                                    row_of_claim, staged, out);
  check_launch("lookup_scatter", 1);
}

}  // namespace hpsb
