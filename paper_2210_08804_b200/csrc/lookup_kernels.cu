// lookup_kernels.cu -- the fused lookup hot path (sm_100a).
//
// Restates LookupEngine::lookup (lookup_engine.cpp:130-241) for a batch of
// |Q| query positions in ONE kernel launch, without materialising the dedup
// step for hits:
//
//   body  persistent grid (one wave), one warp per group of P positions per
//         iteration: placement hash (Barrett modulo), ballot probe of 32-key
//         slabs, 128-bit gather of the hit row straight into the position's
//         output row (the expansion of lookup_engine.cpp:194-203 is fused),
//         recency stamp via atomicExch -- the exchange that first moves a
//         slot to this call's stamp counts one UNIQUE hit, so |Q*| needs no
//         dedup of hits. Missing positions get the default row (the async
//         branch's answer) and are deduplicated in a per-call hash table
//         that keeps the first occurrence; the claiming position of every
//         missing key appends the table slot to a short list. The next
//         group's keys are prefetched and the exchange results are consumed
//         one iteration late, so neither round trip sits on the warp's
//         critical path.
//   tail  the last block to finish (threadfence + completion counter) orders
//         the unique misses by first occurrence with a position bitmap (in
//         shared memory for batches up to 2^18) and a block scan -> the
//         unique miss list in first-occurrence order (the order the
//         reference's dedup + query produce, slab_cache.cpp:84-89) and the
//         rank of every miss-table entry; it also clears the entries it used.
//   K3    lookup_scatter (sync branch only) copies the rows fetched from the
//         tiers into every position of their key, clearing the default flag
//         (lookup_engine.cpp:165-181).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
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
constexpr int kLookupWarps = 8;
constexpr int kLookupThreads = kLookupWarps * 32;
constexpr uint64_t kSmemBitmapMax = 1u << 18;  // positions ordered in shared memory
constexpr int kTailBatch = 8;
}  // namespace

size_t lookup_scratch_bytes(uint64_t cap) {
  uint64_t tcap = 16;
  while (tcap < 2 * cap) tcap <<= 1;
  const uint64_t words = (cap + 31) / 32;
  return a256(tcap * 4) + a256(tcap * 4) + a256(cap * 4) * 3 + a256(words * 4) * 2 + a256(64);
}

LookupScratch lookup_scratch_carve(void* base, uint64_t cap) {
  LookupScratch ls;
  uint64_t tcap = 16;
  while (tcap < 2 * cap) tcap <<= 1;
  const uint64_t words = (cap + 31) / 32;
  char* p = static_cast<char*>(base);
  auto take = [&](uint64_t b) {
    char* r = p;
    p += a256(b);
    return r;
  };
  ls.cap = tcap;
  ls.miss_table = reinterpret_cast<uint32_t*>(take(tcap * 4));
  ls.rank_of_slot = reinterpret_cast<uint32_t*>(take(tcap * 4));
  ls.miss_slot = reinterpret_cast<uint32_t*>(take(cap * 4));
  ls.list = reinterpret_cast<uint32_t*>(take(cap * 4));
  ls.list_firsts = reinterpret_cast<uint32_t*>(take(cap * 4));
  ls.bitmap = reinterpret_cast<uint32_t*>(take(words * 4));
  ls.word_prefix = reinterpret_cast<uint32_t*>(take(words * 4));
  unsigned long long* small = reinterpret_cast<unsigned long long*>(take(64));
  ls.counts = small;           // [0..1]
  ls.counts_prev = small + 2;  // [2..3]
  ls.blocks_done = small + 4;  // [4]
  ls.list_ctr = reinterpret_cast<uint32_t*>(small + 5);
  return ls;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float4 ld_nc_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_cs_f4(float4* p, const float4& v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// Orders the unique misses of this call by first occurrence (run by the
// last block). list[e] = miss-table slot claimed by some position of a
// missing key; the table entry holds that key's first position + 1.
__device__ __noinline__ void order_misses_tail(const uint64_t* __restrict__ keys, uint64_t n,
                                               const LookupScratch& ls, uint32_t* bm,
                                               bool smem_bm) {
  __shared__ uint32_t s_warp[kLookupWarps];
  const uint32_t tid = threadIdx.x;
  const uint32_t m = __ldcg(ls.list_ctr);
  const uint32_t words = uint32_t((n + 31) / 32);
  if (smem_bm) {
    for (uint32_t w = tid; w < words; w += kLookupThreads) bm[w] = 0;
    __syncthreads();
  }
  // 1. first positions -> bitmap (loads batched for memory-level parallelism)
  for (uint32_t e0 = tid; e0 < m; e0 += kLookupThreads * kTailBatch) {
    uint32_t s[kTailBatch], f[kTailBatch];
#pragma unroll
    for (int j = 0; j < kTailBatch; ++j) {
      const uint32_t e = e0 + j * kLookupThreads;
      s[j] = e < m ? __ldcg(ls.list + e) : 0u;
    }
#pragma unroll
    for (int j = 0; j < kTailBatch; ++j) {
      const uint32_t e = e0 + j * kLookupThreads;
      f[j] = e < m ? __ldcg(ls.miss_table + s[j]) - 1u : 0u;
    }
#pragma unroll
    for (int j = 0; j < kTailBatch; ++j) {
      const uint32_t e = e0 + j * kLookupThreads;
      if (e < m) {
        ls.list_firsts[e] = f[j];
        atomicOr(bm + (f[j] >> 5), 1u << (f[j] & 31u));
      }
    }
  }
  __syncthreads();
  // 2. exclusive popcount prefix per bitmap word
  const uint32_t per = (words + kLookupThreads - 1) / kLookupThreads;
  const uint32_t w0 = min(words, tid * per), w1 = min(words, w0 + per);
  uint32_t cnt = 0;
  for (uint32_t w = w0; w < w1; ++w) cnt += __popc(smem_bm ? bm[w] : __ldcg(bm + w));
  uint32_t total;
  uint32_t run = block_exclusive_scan<kLookupThreads>(cnt, s_warp, &total);
  for (uint32_t w = w0; w < w1; ++w) {
    ls.word_prefix[w] = run;
    run += __popc(smem_bm ? bm[w] : __ldcg(bm + w));
  }
  __syncthreads();
  // 3. rank = prefix(word) + popc(bits below) -> ordered miss keys, ranks
  for (uint32_t e0 = tid; e0 < m; e0 += kLookupThreads * kTailBatch) {
    uint32_t s[kTailBatch], f[kTailBatch], r[kTailBatch];
#pragma unroll
    for (int j = 0; j < kTailBatch; ++j) {
      const uint32_t e = e0 + j * kLookupThreads;
      s[j] = e < m ? __ldcg(ls.list + e) : 0u;
      f[j] = e < m ? __ldcg(ls.list_firsts + e) : 0u;
    }
#pragma unroll
    for (int j = 0; j < kTailBatch; ++j) {
      const uint32_t w = f[j] >> 5;
      const uint32_t word = smem_bm ? bm[w] : __ldcg(bm + w);
      r[j] = __ldcg(ls.word_prefix + w) + __popc(word & ((1u << (f[j] & 31u)) - 1u));
    }
    uint64_t k[kTailBatch];
#pragma unroll
    for (int j = 0; j < kTailBatch; ++j) {
      const uint32_t e = e0 + j * kLookupThreads;
      k[j] = e < m ? keys[f[j]] : 0ull;
    }
#pragma unroll
    for (int j = 0; j < kTailBatch; ++j) {
      const uint32_t e = e0 + j * kLookupThreads;
      if (e < m) {
        ls.miss_keys[r[j]] = k[j];
        ls.rank_of_slot[s[j]] = r[j];
        ls.miss_table[s[j]] = 0u;  // leave the table empty for the next call
      }
    }
  }
  __syncthreads();
  if (!smem_bm)
    for (uint32_t w = w0; w < w1; ++w) bm[w] = 0;
  if (tid == 0) *ls.list_ctr = 0;
  if (ls.counts_out != nullptr && tid < 2) {
    const unsigned long long cum = __ldcg(ls.counts + tid);
    ls.counts_out[tid] = cum - ls.counts_prev[tid];
    ls.counts_prev[tid] = cum;
  }
}

template <int P, int MINB>
__global__ void __launch_bounds__(kLookupThreads, MINB)
    k_lookup_probe(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                   float* __restrict__ out, uint8_t* __restrict__ flags,
                   const float* __restrict__ default_row, uint64_t stamp, LookupScratch ls,
                   int smem_bm) {
  extern __shared__ uint32_t s_bitmap[];
  __shared__ unsigned int s_counts[2];
  __shared__ bool s_last;
  if (threadIdx.x < 2) s_counts[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t lane = lane_id();
  if (ls.dbg && threadIdx.x == 0) atomicMin(ls.dbg + 0, gtimer());
  const uint64_t groups = (n + P - 1) / P;
  const uint64_t stride = uint64_t(gridDim.x) * kLookupWarps;
  uint64_t g = uint64_t(blockIdx.x) * kLookupWarps + (threadIdx.x >> 5);
  uint32_t uh = 0, um = 0;
  bool miss_work = false;
  // software pipeline state
  uint64_t next_key = 0;
  if (g < groups && lane < uint32_t(P) && g * P + lane < n) next_key = keys[g * P + lane];
  unsigned long long pend_old = 0;
  bool pend = false;
  const uint32_t d = c.d;
  while (g < groups) {
    const uint64_t base = g * P;
    const uint64_t k = next_key;
    const uint64_t gn = g + stride;
    if (gn < groups && lane < uint32_t(P) && gn * P + lane < n) next_key = keys[gn * P + lane];
    WarpKeys<P> wk;
    warp_place_keys<P>(c, k, base, n, wk);
    uint32_t slot[P];
    warp_probe<P>(c, wk, slot);
    // the previous iteration's exchange has long returned by now
    if (pend) uh += (pend_old != stamp) ? 1u : 0u;
    uint32_t my_slot = kNoSlot;
#pragma unroll
    for (int p = 0; p < P; ++p)
      if (uint32_t(p) == lane) my_slot = slot[p];
    const uint64_t i = base + lane;
    const bool mine = lane < uint32_t(P) && i < n;
    pend = mine && my_slot != kNoSlot;
    if (pend) {
      if (smem_bm & 2)
        pend_old = 0;  // diagnostic: skip the exchange
      else
        pend_old = atomicExch(reinterpret_cast<unsigned long long*>(c.counters + my_slot), stamp);
    }
    if ((d & 3u) == 0) {
      // 128-bit path: the first 32 float4 chunks of every row are loaded for
      // all P positions before any store so P row reads are in flight.
      const uint32_t d4 = d >> 2;
      float4 v[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (wk.valid[p] && lane < d4) {
          const float* src = slot[p] != kNoSlot ? c.rows + uint64_t(slot[p]) * d : default_row;
          v[p] = (smem_bm & 4) ? make_float4(0.f, 0.f, 0.f, 0.f)
                               : ld_nc_f4(reinterpret_cast<const float4*>(src) + lane);
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (wk.valid[p] && lane < d4 && !(smem_bm & 8))
          st_cs_f4(reinterpret_cast<float4*>(out + (base + p) * d) + lane, v[p]);
      }
      for (uint32_t ch = lane + 32; ch < d4; ch += 32) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          if (!wk.valid[p]) continue;
          const float* src = slot[p] != kNoSlot ? c.rows + uint64_t(slot[p]) * d : default_row;
          st_cs_f4(reinterpret_cast<float4*>(out + (base + p) * d) + ch,
                   ld_nc_f4(reinterpret_cast<const float4*>(src) + ch));
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (!wk.valid[p]) continue;
        const float* src = slot[p] != kNoSlot ? c.rows + uint64_t(slot[p]) * d : default_row;
        for (uint32_t ch = lane; ch < d; ch += 32) out[(base + p) * d + ch] = src[ch];
      }
    }
    bool claimed = false;
    uint32_t tslot = 0;
    if (mine) {
      if (my_slot != kNoSlot) {
        flags[i] = 0;
      } else {
        tslot = miss_insert(ls.miss_table, ls.cap, keys, k, uint32_t(i), &claimed);
        ls.miss_slot[i] = tslot;
        flags[i] = 1;
        miss_work = true;
      }
    }
    // claimers append their table slot (one warp-aggregated atomic)
    const uint32_t cm = __ballot_sync(0xFFFFFFFFu, claimed);
    if (cm) {
      const uint32_t leader = __ffs(cm) - 1;
      uint32_t at = 0;
      if (lane == leader) at = atomicAdd(ls.list_ctr, uint32_t(__popc(cm)));
      at = __shfl_sync(0xFFFFFFFFu, at, leader);
      if (claimed) ls.list[at + __popc(cm & ((1u << lane) - 1u))] = tslot;
      um += claimed ? 1u : 0u;
    }
    g = gn;
  }
  if (pend) uh += (pend_old != stamp) ? 1u : 0u;
  if (ls.dbg && lane == 0) atomicMax(ls.dbg + 1, gtimer());
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uh += __shfl_xor_sync(0xFFFFFFFFu, uh, o);
    um += __shfl_xor_sync(0xFFFFFFFFu, um, o);
  }
  if (lane == 0 && (uh | um)) {
    atomicAdd(&s_counts[0], uh);
    atomicAdd(&s_counts[1], um);
  }
  if (miss_work) __threadfence();  // publish table / list writes before completion
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_counts[0]) atomicAdd(ls.counts + 0, (unsigned long long)s_counts[0]);
    if (s_counts[1]) atomicAdd(ls.counts + 1, (unsigned long long)s_counts[1]);
    __threadfence();
    const unsigned long long prev = atomicAdd(ls.blocks_done, 1ull);
    s_last = (prev == ls.blocks_base + gridDim.x - 1);
    if (s_last) __threadfence();
  }
  __syncthreads();
  if (s_last) {
    if (ls.dbg && threadIdx.x == 0) ls.dbg[2] = gtimer();
    order_misses_tail(keys, n, ls, (smem_bm & 1) ? s_bitmap : ls.bitmap, (smem_bm & 1) != 0);
    __syncthreads();
    if (ls.dbg && threadIdx.x == 0) ls.dbg[3] = gtimer();
  }
}

__device__ __forceinline__ float4 ld_nc_f4_l1(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// Warp-deduplicated variant. Power-law batches repeat their hottest keys
// thousands of times (alpha 1.2: the top key is ~19% of all positions), and
// a per-position probe turns every repeat into a read of the same slab,
// mask and row and an atomic on the same counter -- L2 hot spots that
// serialise. Here a warp takes 32 consecutive positions, groups equal keys
// with __match_any_sync, and only the group leader (lowest lane = lowest
// position) probes, stamps, inserts a miss, and loads the row; the row is
// then stored from registers to every position of the group.
template <int P, int MINB>
__global__ void __launch_bounds__(kLookupThreads, MINB)
    k_lookup_dedup(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                   float* __restrict__ out, uint8_t* __restrict__ flags,
                   const float* __restrict__ default_row, uint64_t stamp, LookupScratch ls,
                   int smem_bm) {
  extern __shared__ uint32_t s_bitmap[];
  __shared__ unsigned int s_counts[2];
  __shared__ bool s_last;
  if (threadIdx.x < 2) s_counts[threadIdx.x] = 0;
  __syncthreads();
  const uint32_t lane = lane_id();
  if (ls.dbg && threadIdx.x == 0) atomicMin(ls.dbg + 0, gtimer());
  const uint64_t tiles = (n + 31) / 32;
  const uint64_t stride = uint64_t(gridDim.x) * kLookupWarps;
  uint64_t t = uint64_t(blockIdx.x) * kLookupWarps + (threadIdx.x >> 5);
  uint32_t uh = 0, um = 0;
  bool miss_work = false;
  uint64_t next_key = (t < tiles && t * 32 + lane < n) ? keys[t * 32 + lane] : 0ull;
  const uint32_t d = c.d;
  const uint32_t d4 = d >> 2;
  const bool vec = (d & 3u) == 0;
  while (t < tiles) {
    const uint64_t base = t * 32;
    const uint64_t pos = base + lane;
    const bool valid = pos < n;
    const uint64_t key = next_key;
    const uint64_t tn = t + stride;
    next_key = (tn < tiles && tn * 32 + lane < n) ? keys[tn * 32 + lane] : 0ull;
    const uint32_t vmask = __ballot_sync(0xFFFFFFFFu, valid);
    uint32_t grp = 1u << lane;
    if (valid) grp = __match_any_sync(vmask, key);
    const uint32_t my_leader = __ffs(grp) - 1;
    const bool leader = valid && my_leader == lane;
    const uint32_t my_set = uint32_t(slabset_of(c, key));
    const uint32_t my_first = first_slab_of(c, key);
    uint32_t L = __ballot_sync(0xFFFFFFFFu, leader);
    uint32_t my_res = kNoSlot;
    while (L) {
      uint32_t ld[P];
      WarpKeys<P> wk;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        wk.valid[p] = L != 0;
        ld[p] = L ? __ffs(L) - 1 : 0;
        L &= L - 1;
        wk.key[p] = __shfl_sync(0xFFFFFFFFu, key, ld[p]);
        wk.set[p] = __shfl_sync(0xFFFFFFFFu, my_set, ld[p]);
        wk.first[p] = __shfl_sync(0xFFFFFFFFu, my_first, ld[p]);
      }
      uint32_t slot[P];
      warp_probe<P>(c, wk, slot);
      bool stamp_now = false;
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (wk.valid[p] && lane == ld[p]) {
          my_res = slot[p];
          stamp_now = slot[p] != kNoSlot;
        }
      }
      unsigned long long old = stamp;
      if (stamp_now)
        old = atomicExch(reinterpret_cast<unsigned long long*>(c.counters + my_res), stamp);
      if (vec) {
        float4 v[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          if (wk.valid[p] && lane < d4) {
            const float* src = slot[p] != kNoSlot ? c.rows + uint64_t(slot[p]) * d : default_row;
            v[p] = ld_nc_f4_l1(reinterpret_cast<const float4*>(src) + lane);
          }
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
          if (!wk.valid[p]) continue;
          uint32_t g = __shfl_sync(0xFFFFFFFFu, grp, ld[p]);
          while (g) {
            const uint32_t j = __ffs(g) - 1;
            g &= g - 1;
            if (lane < d4) st_cs_f4(reinterpret_cast<float4*>(out + (base + j) * d) + lane, v[p]);
          }
        }
        for (uint32_t ch = lane + 32; ch < d4; ch += 32) {
#pragma unroll
          for (int p = 0; p < P; ++p) {
            if (!wk.valid[p]) continue;
            const float* src = slot[p] != kNoSlot ? c.rows + uint64_t(slot[p]) * d : default_row;
            const float4 x = ld_nc_f4_l1(reinterpret_cast<const float4*>(src) + ch);
            uint32_t g = __shfl_sync(0xFFFFFFFFu, grp, ld[p]);
            while (g) {
              const uint32_t j = __ffs(g) - 1;
              g &= g - 1;
              st_cs_f4(reinterpret_cast<float4*>(out + (base + j) * d) + ch, x);
            }
          }
        }
      } else {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          if (!wk.valid[p]) continue;
          const float* src = slot[p] != kNoSlot ? c.rows + uint64_t(slot[p]) * d : default_row;
          uint32_t g = __shfl_sync(0xFFFFFFFFu, grp, ld[p]);
          while (g) {
            const uint32_t j = __ffs(g) - 1;
            g &= g - 1;
            for (uint32_t ch = lane; ch < d; ch += 32) out[(base + j) * d + ch] = src[ch];
          }
        }
      }
      if (stamp_now) uh += (old != stamp) ? 1u : 0u;
    }
    // leaders of missing keys insert into the miss table; every position
    // learns its leader's outcome
    bool claimed = false;
    uint32_t tslot = 0;
    if (leader && my_res == kNoSlot) {
      tslot = miss_insert(ls.miss_table, ls.cap, keys, key, uint32_t(pos), &claimed);
      miss_work = true;
    }
    const uint32_t res = __shfl_sync(0xFFFFFFFFu, my_res, my_leader);
    const uint32_t tsl = __shfl_sync(0xFFFFFFFFu, tslot, my_leader);
    if (valid) {
      flags[pos] = res == kNoSlot ? 1 : 0;
      if (res == kNoSlot) ls.miss_slot[pos] = tsl;
    }
    const uint32_t cm = __ballot_sync(0xFFFFFFFFu, claimed);
    if (cm) {
      const uint32_t first_lane = __ffs(cm) - 1;
      uint32_t at = 0;
      if (lane == first_lane) at = atomicAdd(ls.list_ctr, uint32_t(__popc(cm)));
      at = __shfl_sync(0xFFFFFFFFu, at, first_lane);
      if (claimed) ls.list[at + __popc(cm & ((1u << lane) - 1u))] = tslot;
      um += claimed ? 1u : 0u;
    }
    t = tn;
  }
  if (ls.dbg && lane == 0) atomicMax(ls.dbg + 1, gtimer());
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uh += __shfl_xor_sync(0xFFFFFFFFu, uh, o);
    um += __shfl_xor_sync(0xFFFFFFFFu, um, o);
  }
  if (lane == 0 && (uh | um)) {
    atomicAdd(&s_counts[0], uh);
    atomicAdd(&s_counts[1], um);
  }
  if (miss_work) __threadfence();  // publish table / list writes before completion
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_counts[0]) atomicAdd(ls.counts + 0, (unsigned long long)s_counts[0]);
    if (s_counts[1]) atomicAdd(ls.counts + 1, (unsigned long long)s_counts[1]);
    __threadfence();
    const unsigned long long prev = atomicAdd(ls.blocks_done, 1ull);
    s_last = (prev == ls.blocks_base + gridDim.x - 1);
    if (s_last) __threadfence();
  }
  __syncthreads();
  if (s_last) {
    if (ls.dbg && threadIdx.x == 0) ls.dbg[2] = gtimer();
    order_misses_tail(keys, n, ls, (smem_bm & 1) ? s_bitmap : ls.bitmap, (smem_bm & 1) != 0);
    __syncthreads();
    if (ls.dbg && threadIdx.x == 0) ls.dbg[3] = gtimer();
  }
}

unsigned launch_lookup_probe(const CacheDev& c, const uint64_t* keys, uint64_t n, float* out,
                             uint8_t* flags, const float* default_row, uint64_t stamp,
                             const LookupScratch& ls, cudaStream_t st) {
  if (n == 0) return 0;
  // Variant table: (positions per warp, min resident blocks per SM). The
  // default was chosen from measurements on B200 (profiles/); HPSB_LOOKUP_VARIANT
  // selects another for experiments.
  using Kern = void (*)(CacheDev, const uint64_t*, uint64_t, float*, uint8_t*, const float*,
                        uint64_t, LookupScratch, int);
  struct Variant {
    Kern fn;
    int P;
    int per_sm;
  };
  // P = positions per group for the per-position kernels (0-2); for the
  // warp-dedup kernels (3-6) positions per warp-tile are 32 and P is the
  // number of group leaders probed concurrently.
  static Variant variants[] = {{k_lookup_dedup<4, 3>, 32, 3}, {k_lookup_probe<4, 3>, 4, 3},
                               {k_lookup_probe<4, 2>, 4, 2},  {k_lookup_probe<2, 4>, 2, 4},
                               {k_lookup_dedup<8, 2>, 32, 2}, {k_lookup_dedup<4, 2>, 32, 2},
                               {k_lookup_dedup<2, 4>, 32, 4}};
  constexpr int kVariants = sizeof(variants) / sizeof(variants[0]);
  static std::once_flag once;
  static int sms = 148;
  static int vi = 0;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (const char* e = std::getenv("HPSB_LOOKUP_VARIANT")) vi = std::atoi(e) % kVariants;
    for (auto& v : variants) {
      cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(kSmemBitmapMax / 8));
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, v.fn, kLookupThreads, 8192) ==
              cudaSuccess &&
          b > 0)
        v.per_sm = b;
    }
  });
  const Variant& v = variants[vi];
  const bool smem_bm = n <= kSmemBitmapMax;
  const size_t dyn = smem_bm ? ((n + 31) / 32) * 4 : 0;
  const uint64_t groups = (n + v.P - 1) / v.P;
  const uint64_t need = (groups + kLookupWarps - 1) / kLookupWarps;
  const unsigned grid = unsigned(std::min<uint64_t>(need, uint64_t(sms) * v.per_sm));
  // Diagnostic (HPSB_DEBUG_TIMING=1): globaltimer stamps of kernel start,
  // last warp out of the body, tail start / end, printed to stderr. Adds a
  // synchronisation per call; never set for measurements.
  static unsigned long long* dbg = nullptr;
  static const bool debug = std::getenv("HPSB_DEBUG_TIMING") != nullptr;
  LookupScratch lsd = ls;
  if (debug) {
    if (!dbg) cudaMalloc(&dbg, 64);
    const unsigned long long init[4] = {~0ull, 0, 0, 0};
    cudaMemcpyAsync(dbg, init, sizeof(init), cudaMemcpyHostToDevice, st);
    lsd.dbg = dbg;
  }
  // bit 0: order in shared memory; bits 1-3 (HPSB_LOOKUP_SKIP, diagnostic
  // only): skip the recency exchange / the row loads / the row stores
  static const int skip = std::getenv("HPSB_LOOKUP_SKIP") ? std::atoi(std::getenv("HPSB_LOOKUP_SKIP")) : 0;
  v.fn<<<grid, kLookupThreads, dyn, st>>>(c, keys, n, out, flags, default_row, stamp, lsd,
                                          (smem_bm ? 1 : 0) | (skip & 14));
  check_launch("lookup_probe", 1);
  if (debug) {
    unsigned long long h[4];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    std::fprintf(stderr, "lookup_timing n=%llu grid=%u body_us=%.2f tail_wait_us=%.2f tail_us=%.2f\n",
                 (unsigned long long)n, grid, (h[1] - h[0]) * 1e-3, (h[2] - h[1]) * 1e-3,
                 (h[3] - h[2]) * 1e-3);
  }
  return grid;
}

__global__ void __launch_bounds__(256)
    k_lookup_scatter(uint64_t n, uint32_t d, uint8_t* __restrict__ flags, LookupScratch ls,
                     const int32_t* __restrict__ row_of, const float* __restrict__ staged,
                     float* __restrict__ out) {
  const uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  if (flags[i] == 0) return;
  const uint32_t u = ls.rank_of_slot[ls.miss_slot[i]];
  const int32_t r = row_of[u];
  if (r < 0) return;  // absent from every tier: keep default + flag
  warp_copy_row(staged + uint64_t(r) * d, out + i * d, d);
  __syncwarp();
  if (lane_id() == 0) flags[i] = 0;
}

void launch_lookup_scatter(uint64_t n, uint32_t d, const uint8_t* flags_in, uint8_t* flags,
                           const LookupScratch& ls, const int32_t* row_of,
                           const float* staged, float* out, cudaStream_t st) {
  (void)flags_in;
  if (n == 0) return;
  const uint64_t threads = n * 32;
  k_lookup_scatter<<<unsigned((threads + 255) / 256), 256, 0, st>>>(n, d, flags, ls, row_of,
                                                                    staged, out);
  check_launch("lookup_scatter", 1);
}

}  // namespace hpsb
