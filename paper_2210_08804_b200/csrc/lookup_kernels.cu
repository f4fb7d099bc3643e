// lookup_kernels.cu -- the fused lookup hot path (sm_100a).
//
// Restates LookupEngine::lookup (lookup_engine.cpp:130-241) for a batch of
// |Q| query positions in ONE kernel launch:
//
//   body  persistent grid (one wave); a warp takes tiles of 32 consecutive
//         positions. Lane-parallel: key load (next tile prefetched), both
//         placement hashes (Barrett modulo), __match_any_sync grouping of
//         equal keys (power-law batches repeat their hottest key in ~19% of
//         positions -- grouping keeps probes, stamps and miss inserts off a
//         single L2 line). Group leaders are probed 8 at a time with 4 lanes
//         per leader (each lane compares 8 of the slab's 32 keys loaded as
//         128-bit vectors; a 4-lane min-reduction picks the lowest matching
//         slot, i.e. the ballot/ffs rule of slab_cache.cpp:240-245), slab
//         by slab until found or a non-full slab ends the probe. Leaders
//         issue the recency exchange (the one that first moves a slot to this
//         call's stamp counts a UNIQUE hit, so |Q*| needs no hit dedup) and,
//         on a miss, claim the key in a per-call miss table that keeps the
//         first occurrence. Then every position's row is gathered with
//         128-bit loads (L1-cached: hot rows are served by the SM) straight
//         into its output row -- the expansion of lookup_engine.cpp:194-203
//         fused -- or gets the default row (the async branch's answer).
//   tail  the last block to finish (threadfence + completion counter) orders
//         the unique misses by first occurrence with a position bitmap and a
//         block scan in shared memory -> the unique miss list in
//         first-occurrence order (the order the reference's dedup + query
//         produce, slab_cache.cpp:84-89) and the rank of every miss-table
//         entry; it also clears the entries it used.
//   K3    lookup_scatter (sync branch only) copies the rows fetched from the
//         tiers into every position of their key, clearing the default flag
//         (lookup_engine.cpp:165-181).
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <vector>
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
constexpr uint64_t kSmemTailMax = 1u << 17;  // positions ordered in shared memory
constexpr int kTailBatch = 8;
constexpr int kGatherUnroll = 8;
constexpr uint32_t kStampSetBits = 11;  // 2048-entry per-block stamped-slot set
}  // namespace

size_t lookup_scratch_bytes(uint64_t cap) {
  uint64_t tcap = 16;
  while (tcap < 2 * cap) tcap <<= 1;
  const uint64_t words = (cap + 31) / 32;
  return a256(tcap * 4) + a256(tcap * 4) + a256(cap * 4) * 4 + a256(cap * 8) +
         a256(words * 4) * 2 + a256(64);
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
  ls.list_keys = reinterpret_cast<uint64_t*>(take(cap * 8));
  ls.pos_slot = reinterpret_cast<uint32_t*>(take(cap * 4));
  ls.bitmap = reinterpret_cast<uint32_t*>(take(words * 4));
  ls.word_prefix = reinterpret_cast<uint32_t*>(take(words * 4));
  unsigned long long* small = reinterpret_cast<unsigned long long*>(take(64));
  ls.counts = small;           // [0..1]
  ls.counts_prev = small + 2;  // [2..3]
  ls.blocks_done = small + 4;  // [4]
  ls.list_ctr = reinterpret_cast<uint32_t*>(small + 5);
  ls.gather_done = small + 6;  // [6]
  ls.tail_done = reinterpret_cast<unsigned int*>(small + 7);
  return ls;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
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
// Output rows are written once and not re-read: evict-first.
__device__ __forceinline__ void st_cs_f4(float4* p, const float4& v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// Orders the unique misses of this call by first occurrence (run by the
// last block). list[e] = miss-table slot claimed by the leader position of
// a missing key; the table entry holds that key's first position + 1.
// bm / pre: bitmap and word prefix (shared memory when `smem`, else the
// global scratch arrays).
__device__ __noinline__ void order_misses_tail(const uint64_t* __restrict__ keys, uint64_t n,
                                               const LookupScratch& ls, uint32_t* bm,
                                               uint32_t* pre, bool smem) {
  __shared__ uint32_t s_warp[kLookupWarps];
  const uint32_t tid = threadIdx.x;
  const uint32_t m = __ldcg(ls.list_ctr);
  const uint32_t words = uint32_t((n + 31) / 32);
  if (smem) {
    for (uint32_t w = tid; w < words; w += kLookupThreads) bm[w] = 0;
    __syncthreads();
  }
  // 1. first positions -> bitmap (loads batched for memory-level parallelism).
  // With at most one batch per thread (m <= 2048) the entries stay in
  // registers through phase 3: two dependent global round trips in total.
  const bool one = m <= uint32_t(kLookupThreads * kTailBatch);
  uint32_t s[kTailBatch], f[kTailBatch];
  uint64_t k[kTailBatch];
  for (uint32_t e0 = tid; e0 < m; e0 += kLookupThreads * kTailBatch) {
#pragma unroll
    for (int j = 0; j < kTailBatch; ++j) {
      const uint32_t e = e0 + j * kLookupThreads;
      s[j] = e < m ? __ldcg(ls.list + e) : 0u;
      k[j] = e < m ? __ldcg(reinterpret_cast<const unsigned long long*>(ls.list_keys) + e) : 0ull;
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
        if (!one) ls.list_firsts[e] = f[j];
        atomicOr(bm + (f[j] >> 5), 1u << (f[j] & 31u));
      }
    }
  }
  __syncthreads();
  if (ls.dbg && tid == 0) ls.dbg[9] = gtimer();
  // 2. exclusive popcount prefix per bitmap word
  const uint32_t per = (words + kLookupThreads - 1) / kLookupThreads;
  const uint32_t w0 = min(words, tid * per), w1 = min(words, w0 + per);
  uint32_t cnt = 0;
  for (uint32_t w = w0; w < w1; ++w) cnt += __popc(smem ? bm[w] : __ldcg(bm + w));
  uint32_t total;
  uint32_t run = block_exclusive_scan<kLookupThreads>(cnt, s_warp, &total);
  for (uint32_t w = w0; w < w1; ++w) {
    pre[w] = run;
    run += __popc(smem ? bm[w] : __ldcg(bm + w));
  }
  __syncthreads();
  if (ls.dbg && tid == 0) ls.dbg[10] = gtimer();
  // 3. rank = prefix(word) + popc(bits below) -> ordered miss keys, ranks
  (void)keys;
  for (uint32_t e0 = tid; e0 < m; e0 += kLookupThreads * kTailBatch) {
    uint32_t r[kTailBatch];
    if (!one) {
#pragma unroll
      for (int j = 0; j < kTailBatch; ++j) {
        const uint32_t e = e0 + j * kLookupThreads;
        s[j] = e < m ? __ldcg(ls.list + e) : 0u;
        f[j] = e < m ? ls.list_firsts[e] : 0u;  // written by this thread in phase 1
        k[j] = e < m ? __ldcg(reinterpret_cast<const unsigned long long*>(ls.list_keys) + e)
                     : 0ull;
      }
    }
#pragma unroll
    for (int j = 0; j < kTailBatch; ++j) {
      const uint32_t w = f[j] >> 5;
      const uint32_t word = smem ? bm[w] : __ldcg(bm + w);
      const uint32_t pw = smem ? pre[w] : __ldcg(pre + w);
      r[j] = pw + __popc(word & ((1u << (f[j] & 31u)) - 1u));
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
  if (ls.dbg && tid == 0) ls.dbg[11] = gtimer();
  if (!smem)
    for (uint32_t w = w0; w < w1; ++w) bm[w] = 0;
  if (tid == 0) *ls.list_ctr = 0;
  if (ls.counts_out != nullptr && tid < 2) {
    const unsigned long long cum = __ldcg(ls.counts + tid);
    ls.counts_out[tid] = cum - ls.counts_prev[tid];
    ls.counts_prev[tid] = cum;
  }
}

// Block epilogue shared by the lookup kernels: counts, completion counter,
// and the ordering tail in the last block.
__device__ __forceinline__ void lookup_block_finish(const uint64_t* keys, uint64_t n,
                                                    const LookupScratch& ls, uint32_t uh,
                                                    uint32_t um, bool miss_work, int flags_mode,
                                                    unsigned int* s_counts, bool* s_last,
                                                    uint32_t* s_dyn) {
  const uint32_t lane = lane_id();
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
  // this block's slots are written: the gather kernel (programmatic
  // dependent launch) may start once every block got here
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    if (s_counts[0]) atomicAdd(ls.counts + 0, (unsigned long long)s_counts[0]);
    if (s_counts[1]) atomicAdd(ls.counts + 1, (unsigned long long)s_counts[1]);
    __threadfence();
    const unsigned long long prev = atomicAdd(ls.blocks_done, 1ull);
    *s_last = (prev == gridDim.x - 1);
    if (*s_last) {
      // every other block has arrived: reset for the next call (stream order
      // keeps calls apart; replay-safe inside CUDA graphs)
      *ls.blocks_done = 0;
      __threadfence();
    }
  }
  __syncthreads();
  if (*s_last) {
    if (ls.dbg && threadIdx.x == 0) ls.dbg[2] = gtimer();
    const bool smem = (flags_mode & 1) != 0;
    const uint32_t words = uint32_t((n + 31) / 32);
    order_misses_tail(keys, n, ls, smem ? s_dyn : ls.bitmap, smem ? s_dyn + words : ls.word_prefix,
                      smem);
    __syncthreads();
    if (ls.dbg && threadIdx.x == 0) ls.dbg[3] = gtimer();
    if (threadIdx.x == 0 && !(flags_mode & 16)) {
      // release the ordered miss list to the gather kernel's last block
      __threadfence();
      atomicExch(ls.tail_done, 1u);
    }
  }
}

// ---------------------------------------------------------------------------
// Tile kernel (default). mode bit 0: shared-memory tail; bits 1-3
// (HPSB_LOOKUP_SKIP, diagnostic only): skip exchange / row loads / stores.
template <int MINB>
__global__ void __launch_bounds__(kLookupThreads, MINB)
    k_lookup_tile(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                  float* __restrict__ out, uint8_t* __restrict__ flags,
                  const float* __restrict__ default_row, uint64_t stamp, LookupScratch ls,
                  int mode) {
  extern __shared__ uint32_t s_dyn[];
  __shared__ unsigned int s_counts[2];
  __shared__ bool s_last;
  __shared__ uint32_t s_stamped[1u << kStampSetBits];
  if (threadIdx.x < 2) s_counts[threadIdx.x] = 0;
  for (uint32_t i = threadIdx.x; i < (1u << kStampSetBits); i += blockDim.x)
    s_stamped[i] = kNoSlot;
  __syncthreads();
  const uint32_t lane = lane_id();
  if (ls.dbg && threadIdx.x == 0) atomicMin(ls.dbg + 0, gtimer());
  const uint64_t tiles = (n + 31) / 32;
  const uint64_t stride = uint64_t(gridDim.x) * kLookupWarps;
  uint64_t t = uint64_t(blockIdx.x) * kLookupWarps + (threadIdx.x >> 5);
  uint32_t uh = 0, um = 0;
  bool miss_work = false;
  const unsigned long long t_start = ls.dbg ? gtimer() : 0ull;
  uint64_t next_key = (t < tiles && t * 32 + lane < n) ? keys[t * 32 + lane] : 0ull;
  const uint32_t d = c.d;
  const uint32_t d4 = d >> 2;
  const bool vec = (d & 3u) == 0;
  long long ph[5] = {0, 0, 0, 0, 0};  // diagnostic phase cycles (ls.dbg)
  const uint32_t q = lane >> 2;    // probe group (leader) within a pass
  const uint32_t sub = lane & 3u;  // which 8 of the slab's 32 keys this lane checks
  while (t < tiles) {
    const uint64_t base = t * 32;
    const uint64_t pos = base + lane;
    const bool valid = pos < n;
    const uint64_t key = next_key;
    const uint64_t tn = t + stride;
    next_key = (tn < tiles && tn * 32 + lane < n) ? keys[tn * 32 + lane] : 0ull;
    long long tprev = ls.dbg ? clock64() : 0;
#define HPSB_PHASE(i)                  \
  if (ls.dbg) {                        \
    const long long now_ = clock64();  \
    ph[i] += now_ - tprev;             \
    tprev = now_;                      \
  }
    // ---- group equal keys, hash lane-parallel ----
    const uint32_t vmask = __ballot_sync(0xFFFFFFFFu, valid);
    uint32_t grp = 1u << lane;
    if (valid) grp = __match_any_sync(vmask, key);
    const uint32_t my_leader = __ffs(grp) - 1;
    const bool leader = valid && my_leader == lane;
    const uint32_t set = uint32_t(slabset_of(c, key));
    const uint32_t first = first_slab_of(c, key);
    HPSB_PHASE(0)
    // ---- probe leaders, slab by slab ----
    uint32_t res = kNoSlot;                        // leader's slot
    uint32_t pend = __ballot_sync(0xFFFFFFFFu, leader);
    if (c.W == 2) {
      // Two slabs per set (every configured geometry): both probe slabs and
      // masks are loaded in the same round, so one dependent round trip
      // resolves a leader (probe order first, first+1; the second slab only
      // counts if the first is full -- slab_cache.cpp:249-256).
      const uint32_t slab_a = set * 2 + first;
      const uint32_t slab_b = set * 2 + (first ^ 1u);
      const uint32_t np = __popc(pend);
      const uint32_t my_rank = __popc(pend & ((1u << lane) - 1u));
      for (uint32_t pass = 0; pass < np; pass += 8) {
        uint64_t ka[8], kb[8];
        uint32_t ma = 0, mb = 0;
        const uint32_t e = pass + q;
        const bool act = e < np;
        const uint32_t src = act ? __fns(pend, 0, int(e) + 1) : lane;
        const uint64_t qkey = __shfl_sync(0xFFFFFFFFu, key, src);
        const uint32_t sa = __shfl_sync(0xFFFFFFFFu, slab_a, src);
        const uint32_t sbb = __shfl_sync(0xFFFFFFFFu, slab_b, src);
        if (act) {
          ma = c.masks[sa];
          mb = c.masks[sbb];
          const ulonglong2* pa =
              reinterpret_cast<const ulonglong2*>(c.keys + uint64_t(sa) * kSlotsPerSlab) + sub * 4;
          const ulonglong2* pb =
              reinterpret_cast<const ulonglong2*>(c.keys + uint64_t(sbb) * kSlotsPerSlab) + sub * 4;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const ulonglong2 va = pa[j];
            const ulonglong2 vb = pb[j];
            ka[2 * j] = va.x;
            ka[2 * j + 1] = va.y;
            kb[2 * j] = vb.x;
            kb[2 * j + 1] = vb.y;
          }
        }
        uint32_t ha = 32, hb = 32;
        if (act) {
#pragma unroll
          for (int j = 7; j >= 0; --j) {
            const uint32_t s = sub * 8 + j;
            if (((ma >> s) & 1u) && ka[j] == qkey) ha = s;
            if (((mb >> s) & 1u) && kb[j] == qkey) hb = s;
          }
        }
        ha = min(ha, __shfl_xor_sync(0xFFFFFFFFu, ha, 1));
        ha = min(ha, __shfl_xor_sync(0xFFFFFFFFu, ha, 2));
        hb = min(hb, __shfl_xor_sync(0xFFFFFFFFu, hb, 1));
        hb = min(hb, __shfl_xor_sync(0xFFFFFFFFu, hb, 2));
        uint32_t found = kNoSlot;
        if (ha < 32)
          found = sa * kSlotsPerSlab + ha;
        else if (act && ma == kFullSlab && hb < 32)
          found = sbb * kSlotsPerSlab + hb;
        const uint32_t rank_in_round = my_rank - pass;
        const uint32_t from = (rank_in_round < 8u) ? rank_in_round * 4 : lane;
        const uint32_t f = __shfl_sync(0xFFFFFFFFu, found, from);
        if (((pend >> lane) & 1u) && rank_in_round < 8u) res = f;
      }
      pend = 0;
    }
    for (uint32_t step = 0; step < c.W && pend; ++step) {
      uint32_t sl = first + step;
      sl = (sl >= c.W) ? sl - c.W : sl;
      const uint32_t slab_l = set * c.W + sl;      // this lane's slab for this step
      const uint32_t np = __popc(pend);
      bool cont = false;                           // leader: not found, slab full
      const uint32_t my_rank = __popc(pend & ((1u << lane) - 1u));
      for (uint32_t pass = 0; pass < np; pass += 16) {
        // two rounds of 8 leaders issued together
        uint32_t found[2];
        bool full[2];
        uint64_t kk[2][8];
        uint32_t mk[2], sb[2];
        uint64_t qkey[2];
        bool act[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const uint32_t e = pass + r * 8 + q;
          act[r] = e < np;
          const uint32_t src = act[r] ? __fns(pend, 0, int(e) + 1) : lane;
          qkey[r] = __shfl_sync(0xFFFFFFFFu, key, src);
          sb[r] = __shfl_sync(0xFFFFFFFFu, slab_l, src);
          if (act[r]) {
            mk[r] = c.masks[sb[r]];
            const ulonglong2* p2 =
                reinterpret_cast<const ulonglong2*>(c.keys + uint64_t(sb[r]) * kSlotsPerSlab) +
                sub * 4;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const ulonglong2 v = p2[j];
              kk[r][2 * j] = v.x;
              kk[r][2 * j + 1] = v.y;
            }
          }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          uint32_t hit = 32;
          if (act[r]) {
#pragma unroll
            for (int j = 7; j >= 0; --j) {
              const uint32_t s = sub * 8 + j;
              if (((mk[r] >> s) & 1u) && kk[r][j] == qkey[r]) hit = s;
            }
          }
          hit = min(hit, __shfl_xor_sync(0xFFFFFFFFu, hit, 1));
          hit = min(hit, __shfl_xor_sync(0xFFFFFFFFu, hit, 2));
          found[r] = hit < 32 ? sb[r] * kSlotsPerSlab + hit : kNoSlot;
          full[r] = act[r] && mk[r] == kFullSlab;
        }
        // hand results back to the leader lanes (group q's result sits in lane 4q)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const uint32_t rank_in_round = my_rank - (pass + r * 8);
          const uint32_t from = (rank_in_round < 8u) ? rank_in_round * 4 : lane;
          const uint32_t f = __shfl_sync(0xFFFFFFFFu, found[r], from);
          const bool fu = __shfl_sync(0xFFFFFFFFu, full[r] ? 1u : 0u, from) != 0;
          if (((pend >> lane) & 1u) && rank_in_round < 8u) {
            res = f;
            cont = (f == kNoSlot) && fu;
          }
        }
      }
      pend = __ballot_sync(0xFFFFFFFFu, cont);
    }
    HPSB_PHASE(1)
    // ---- leaders: recency exchange / miss claim ----
    // The block-level stamped set sends each slot's exchange to L2 once per
    // block: the hottest key is a leader in every tile, and 2048 exchanges
    // on one counter would serialise in one L2 slice.
    unsigned long long old = stamp;
    bool stamp_it = leader && res != kNoSlot;
    if (stamp_it) {
      uint32_t h = (res * 0x9E3779B1u) >> (32 - kStampSetBits);
      bool first_here = true;
      for (int probe = 0; probe < 16; ++probe) {
        const uint32_t cur = atomicCAS(&s_stamped[h], kNoSlot, res);
        if (cur == kNoSlot) break;
        if (cur == res) {
          first_here = false;
          break;
        }
        h = (h + 1) & ((1u << kStampSetBits) - 1u);
      }
      stamp_it = first_here;
    }
    if (stamp_it && !(mode & 2))
      old = atomicExch(reinterpret_cast<unsigned long long*>(c.counters + res), stamp);
    bool claimed = false;
    uint32_t tslot = 0;
    if (leader && res == kNoSlot) {
      tslot = miss_insert(ls.miss_table, ls.cap, keys, key, uint32_t(pos), &claimed);
      miss_work = true;
    }
    const uint32_t my_res = __shfl_sync(0xFFFFFFFFu, res, my_leader);
    const uint32_t my_tsl = __shfl_sync(0xFFFFFFFFu, tslot, my_leader);
    HPSB_PHASE(2)
    // ---- gather every position's row (fused mode) or hand the slot to the
    // gather kernel (split mode, default) ----
    if (!(mode & 16)) {
      if (valid) ls.pos_slot[pos] = my_res;
    } else if (vec) {
      for (uint32_t j0 = 0; j0 < 32; j0 += kGatherUnroll) {
        float4 v[kGatherUnroll];
        uint32_t sj[kGatherUnroll];
#pragma unroll
        for (int u = 0; u < kGatherUnroll; ++u) {
          sj[u] = __shfl_sync(0xFFFFFFFFu, my_res, j0 + u);
          if (lane < d4 && base + j0 + u < n && !(mode & 4)) {
            const float* src = sj[u] != kNoSlot ? c.rows + uint64_t(sj[u]) * d : default_row;
            v[u] = ld_row_f4(reinterpret_cast<const float4*>(src) + lane);
          } else {
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < kGatherUnroll; ++u) {
          if (lane < d4 && base + j0 + u < n && !(mode & 8))
            st_cs_f4(reinterpret_cast<float4*>(out + (base + j0 + u) * d) + lane, v[u]);
        }
        // rows wider than 128 floats
        for (uint32_t ch = lane + 32; ch < d4; ch += 32) {
#pragma unroll
          for (int u = 0; u < kGatherUnroll; ++u) {
            if (base + j0 + u >= n) continue;
            const float* src = sj[u] != kNoSlot ? c.rows + uint64_t(sj[u]) * d : default_row;
            st_cs_f4(reinterpret_cast<float4*>(out + (base + j0 + u) * d) + ch,
                     ld_row_f4(reinterpret_cast<const float4*>(src) + ch));
          }
        }
      }
    } else {
      for (uint32_t j = 0; j < 32; ++j) {
        const uint32_t sj = __shfl_sync(0xFFFFFFFFu, my_res, j);
        if (base + j >= n) continue;
        const float* src = sj != kNoSlot ? c.rows + uint64_t(sj) * d : default_row;
        for (uint32_t ch = lane; ch < d; ch += 32) out[(base + j) * d + ch] = src[ch];
      }
    }
    HPSB_PHASE(3)
    // ---- per-position bookkeeping ----
    if (valid) {
      flags[pos] = my_res == kNoSlot ? 1 : 0;
      if (my_res == kNoSlot) ls.miss_slot[pos] = my_tsl;
    }
    const uint32_t cm = __ballot_sync(0xFFFFFFFFu, claimed);
    if (cm) {
      const uint32_t first_lane = __ffs(cm) - 1;
      uint32_t at = 0;
      if (lane == first_lane) at = atomicAdd(ls.list_ctr, uint32_t(__popc(cm)));
      at = __shfl_sync(0xFFFFFFFFu, at, first_lane);
      if (claimed) {
        const uint32_t e = at + __popc(cm & ((1u << lane) - 1u));
        ls.list[e] = tslot;
        ls.list_keys[e] = key;
      }
      um += claimed ? 1u : 0u;
    }
    if (stamp_it) uh += (mode & 2) ? 1u : ((old != stamp) ? 1u : 0u);
    HPSB_PHASE(4)
#undef HPSB_PHASE
    t = tn;
  }
  if (ls.dbg && lane == 0) {
    for (int i = 0; i < 5; ++i) atomicAdd(ls.dbg + 4 + i, (unsigned long long)ph[i]);
    // per-warp start / end / miss-work stamps (diagnostic)
    const uint64_t wid = uint64_t(blockIdx.x) * kLookupWarps + (threadIdx.x >> 5);
    ls.dbg[16 + 3 * wid + 0] = t_start;
    ls.dbg[16 + 3 * wid + 1] = gtimer();
    ls.dbg[16 + 3 * wid + 2] = (miss_work ? 1u : 0u) | (um ? 2u : 0u);
  }
  lookup_block_finish(keys, n, ls, uh, um, miss_work, mode, s_counts, &s_last, s_dyn);
}

// Gather kernel (split mode): launched as a programmatic dependent of the
// probe kernel; one warp streams P positions' rows (hit: cached row, miss:
// default row) with 128-bit L1-cached loads and evict-first stores. Its last
// block waits for the probe kernel's ordering tail, so work queued after the
// gather also sees the ordered miss list.
template <int P>
__global__ void __launch_bounds__(256)
    k_lookup_gather(CacheDev c, uint64_t n, float* __restrict__ out,
                    const float* __restrict__ default_row, LookupScratch ls, int mode) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t lane = lane_id();
  const uint64_t base = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * P;
  const uint32_t d = c.d;
  if (base < n) {
    const uint32_t mine = (lane < uint32_t(P) && base + lane < n) ? ls.pos_slot[base + lane] : 0u;
    uint32_t sj[P];
#pragma unroll
    for (int u = 0; u < P; ++u) sj[u] = __shfl_sync(0xFFFFFFFFu, mine, u);
    if ((d & 3u) == 0) {
      const uint32_t d4 = d >> 2;
      for (uint32_t ch = lane; ch < d4; ch += 32) {
        float4 v[P];
#pragma unroll
        for (int u = 0; u < P; ++u) {
          if (base + u < n && !(mode & 4)) {
            const float* src = sj[u] != kNoSlot ? c.rows + uint64_t(sj[u]) * d : default_row;
            v[u] = ld_row_f4(reinterpret_cast<const float4*>(src) + ch);
          } else {
            v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < P; ++u)
          if (base + u < n && !(mode & 8))
            st_cs_f4(reinterpret_cast<float4*>(out + (base + u) * d) + ch, v[u]);
      }
    } else {
#pragma unroll
      for (int u = 0; u < P; ++u) {
        if (base + u >= n) continue;
        const float* src = sj[u] != kNoSlot ? c.rows + uint64_t(sj[u]) * d : default_row;
        for (uint32_t ch = lane; ch < d; ch += 32) out[(base + u) * d + ch] = src[ch];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long prev = atomicAdd(ls.gather_done, 1ull);
    if (prev == gridDim.x - 1) {
      *ls.gather_done = 0;
      volatile unsigned int* td = ls.tail_done;
      while (*td == 0u) {
      }
      __threadfence();
      *ls.tail_done = 0u;
    }
  }
}

// ---------------------------------------------------------------------------
// Quad kernel (default): a warp serves 8 positions, 4 lanes per position, so
// one position's whole chain is short -- key load, both placement hashes, ONE
// round trip for both probe slabs + masks (each lane compares 8 of the 32
// keys of each slab; a 4-lane min picks the lowest matching slot), ONE round
// trip for the row (each lane moves a quarter of it with 128-bit loads and
// evict-first stores). Hot keys hit the SM's L1 for slabs and rows; a
// per-block stamped-slot set keeps their recency exchanges off one L2 line.
constexpr int kQuadPos = 8;       // positions per warp
constexpr int kQuadSetBits = 7;   // 128-entry per-block stamped set (64 positions)
constexpr int kQuadRowChunks = 8; // float4 chunks per lane held in flight (d <= 128)

__global__ void __launch_bounds__(kLookupThreads)
    k_lookup_quad(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                  float* __restrict__ out, uint8_t* __restrict__ flags,
                  const float* __restrict__ default_row, uint64_t stamp, LookupScratch ls,
                  int mode) {
  extern __shared__ uint32_t s_dyn[];
  __shared__ unsigned int s_counts[2];
  __shared__ bool s_last;
  __shared__ uint32_t s_stamped[1u << kQuadSetBits];
  if (threadIdx.x < 2) s_counts[threadIdx.x] = 0;
  for (uint32_t i = threadIdx.x; i < (1u << kQuadSetBits); i += blockDim.x) s_stamped[i] = kNoSlot;
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint32_t q = lane >> 2, sub = lane & 3u;
  const uint64_t pos = ((uint64_t(blockIdx.x) * kLookupThreads + threadIdx.x) >> 5) * kQuadPos + q;
  const bool valid = pos < n;
  uint32_t uh = 0, um = 0;
  bool miss_work = false;
  const uint64_t key = valid ? keys[pos] : 0ull;
  // ---- placement + both probe slabs in one round trip ----
  const uint32_t set = uint32_t(slabset_of(c, key));
  const uint32_t first = first_slab_of(c, key);
  uint32_t res = kNoSlot;
  if (c.W == 2) {
    const uint32_t sa = set * 2 + first, sb = set * 2 + (first ^ 1u);
    uint32_t ma = 0, mb = 0;
    uint64_t ka[8], kb[8];
    if (valid) {
      ma = c.masks[sa];
      mb = c.masks[sb];
      const ulonglong2* pa =
          reinterpret_cast<const ulonglong2*>(c.keys + uint64_t(sa) * kSlotsPerSlab) + sub * 4;
      const ulonglong2* pb =
          reinterpret_cast<const ulonglong2*>(c.keys + uint64_t(sb) * kSlotsPerSlab) + sub * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const ulonglong2 va = pa[j];
        const ulonglong2 vb = pb[j];
        ka[2 * j] = va.x;
        ka[2 * j + 1] = va.y;
        kb[2 * j] = vb.x;
        kb[2 * j + 1] = vb.y;
      }
    }
    uint32_t ha = 32, hb = 32;
    if (valid) {
#pragma unroll
      for (int j = 7; j >= 0; --j) {
        const uint32_t s = sub * 8 + j;
        if (((ma >> s) & 1u) && ka[j] == key) ha = s;
        if (((mb >> s) & 1u) && kb[j] == key) hb = s;
      }
    }
    ha = min(ha, __shfl_xor_sync(0xFFFFFFFFu, ha, 1));
    ha = min(ha, __shfl_xor_sync(0xFFFFFFFFu, ha, 2));
    hb = min(hb, __shfl_xor_sync(0xFFFFFFFFu, hb, 1));
    hb = min(hb, __shfl_xor_sync(0xFFFFFFFFu, hb, 2));
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
      uint64_t kk[8];
      if (pending) {
        m = c.masks[slab];
        const ulonglong2* p2 =
            reinterpret_cast<const ulonglong2*>(c.keys + uint64_t(slab) * kSlotsPerSlab) + sub * 4;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const ulonglong2 v = p2[j];
          kk[2 * j] = v.x;
          kk[2 * j + 1] = v.y;
        }
      }
      uint32_t h = 32;
      if (pending) {
#pragma unroll
        for (int j = 7; j >= 0; --j) {
          const uint32_t s = sub * 8 + j;
          if (((m >> s) & 1u) && kk[j] == key) h = s;
        }
      }
      h = min(h, __shfl_xor_sync(0xFFFFFFFFu, h, 1));
      h = min(h, __shfl_xor_sync(0xFFFFFFFFu, h, 2));
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
  // ---- recency exchange (leader lane of the group), issued before the copy ----
  unsigned long long old = stamp;
  bool stamp_it = valid && sub == 0 && res != kNoSlot;
  if (stamp_it) {
    uint32_t h = (res * 0x9E3779B1u) >> (32 - kQuadSetBits);
    for (int probe = 0; probe < 16; ++probe) {
      const uint32_t cur = atomicCAS(&s_stamped[h], kNoSlot, res);
      if (cur == kNoSlot) break;
      if (cur == res) {
        stamp_it = false;
        break;
      }
      h = (h + 1) & ((1u << kQuadSetBits) - 1u);
    }
  }
  if (stamp_it && !(mode & 2))
    old = atomicExch(reinterpret_cast<unsigned long long*>(c.counters + res), stamp);
  // ---- copy the row: lane `sub` moves float4 chunks sub, sub+4, ... ----
  if (valid) {
    const uint32_t d = c.d;
    const float* src = res != kNoSlot ? c.rows + uint64_t(res) * d : default_row;
    float* dst = out + pos * d;
    if ((d & 3u) == 0) {
      const uint32_t d4 = d >> 2;
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* o4 = reinterpret_cast<float4*>(dst);
      for (uint32_t ch0 = 0; ch0 < d4; ch0 += 4 * kQuadRowChunks) {
        float4 v[kQuadRowChunks];
#pragma unroll
        for (int j = 0; j < kQuadRowChunks; ++j) {
          const uint32_t ch = ch0 + uint32_t(j) * 4 + sub;
          if (ch < d4 && !(mode & 4)) v[j] = ld_row_f4(s4 + ch);
        }
#pragma unroll
        for (int j = 0; j < kQuadRowChunks; ++j) {
          const uint32_t ch = ch0 + uint32_t(j) * 4 + sub;
          if (ch < d4 && !(mode & 8)) st_cs_f4(o4 + ch, (mode & 4) ? make_float4(0, 0, 0, 0) : v[j]);
        }
      }
    } else {
      for (uint32_t ch = sub; ch < d; ch += 4) dst[ch] = src[ch];
    }
  }
  // ---- misses: leader lane claims the key; bookkeeping ----
  bool claimed = false;
  uint32_t tslot = 0;
  if (valid && sub == 0 && res == kNoSlot) {
    tslot = miss_insert(ls.miss_table, ls.cap, keys, key, uint32_t(pos), &claimed);
    ls.miss_slot[pos] = tslot;
    miss_work = true;
  }
  if (valid && sub == 0) flags[pos] = res == kNoSlot ? 1 : 0;
  const uint32_t cm = __ballot_sync(0xFFFFFFFFu, claimed);
  if (cm) {
    const uint32_t first_lane = __ffs(cm) - 1;
    uint32_t at = 0;
    if (lane == first_lane) at = atomicAdd(ls.list_ctr, uint32_t(__popc(cm)));
    at = __shfl_sync(0xFFFFFFFFu, at, first_lane);
    if (claimed) {
      const uint32_t e = at + __popc(cm & ((1u << lane) - 1u));
      ls.list[e] = tslot;
      ls.list_keys[e] = key;
    }
    um = claimed ? 1u : 0u;
  }
  if (stamp_it) uh = (mode & 2) ? 1u : ((old != stamp) ? 1u : 0u);
  lookup_block_finish(keys, n, ls, uh, um, miss_work, mode | 16, s_counts, &s_last, s_dyn);
}

unsigned launch_lookup_probe(const CacheDev& c, const uint64_t* keys, uint64_t n, float* out,
                             uint8_t* flags, const float* default_row, uint64_t stamp,
                             const LookupScratch& ls, cudaStream_t st) {
  if (n == 0) return 0;
  static const int quad_off = std::getenv("HPSB_LOOKUP_VARIANT") != nullptr;
  if (!quad_off) {
    static std::once_flag qonce;
    std::call_once(qonce, [] {
      cudaFuncSetAttribute(k_lookup_quad, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           int(kSmemTailMax / 32 * 4 * 2));
    });
    const bool smem_tail = n <= kSmemTailMax;
    const size_t dyn = smem_tail ? ((n + 31) / 32) * 4 * 2 : 0;
    const uint64_t per_block = uint64_t(kLookupWarps) * kQuadPos;
    const unsigned grid = unsigned((n + per_block - 1) / per_block);
    static const int qskip =
        std::getenv("HPSB_LOOKUP_SKIP") ? std::atoi(std::getenv("HPSB_LOOKUP_SKIP")) : 0;
    k_lookup_quad<<<grid, kLookupThreads, dyn, st>>>(c, keys, n, out, flags, default_row, stamp,
                                                     ls, (smem_tail ? 1 : 0) | (qskip & 14));
    check_launch("lookup_quad", 1);
    return grid;
  }
  // Variants: minimum resident blocks per SM (register budget). The default
  // was chosen from B200 measurements (profiles/); HPSB_LOOKUP_VARIANT
  // selects another for experiments.
  using Kern = void (*)(CacheDev, const uint64_t*, uint64_t, float*, uint8_t*, const float*,
                        uint64_t, LookupScratch, int);
  struct Variant {
    Kern fn;
    int per_sm;
  };
  static Variant variants[] = {{k_lookup_tile<2>, 2}, {k_lookup_tile<3>, 3},
                               {k_lookup_tile<4>, 4}};
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
                           int(kSmemTailMax / 32 * 4 * 2));
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, v.fn, kLookupThreads, 16384) ==
              cudaSuccess &&
          b > 0)
        v.per_sm = b;
    }
  });
  const Variant& v = variants[vi];
  const bool smem_tail = n <= kSmemTailMax;
  const size_t dyn = smem_tail ? ((n + 31) / 32) * 4 * 2 : 0;
  const uint64_t tiles = (n + 31) / 32;
  const uint64_t need = (tiles + kLookupWarps - 1) / kLookupWarps;
  const unsigned grid = unsigned(std::min<uint64_t>(need, uint64_t(sms) * v.per_sm));
  // Diagnostic (HPSB_DEBUG_TIMING=1): globaltimer stamps of kernel start,
  // last warp out of the body, tail start / end, printed to stderr. Adds a
  // synchronisation per call; never set for measurements.
  static unsigned long long* dbg = nullptr;
  static const bool debug = std::getenv("HPSB_DEBUG_TIMING") != nullptr;
  static const int skip =
      std::getenv("HPSB_LOOKUP_SKIP") ? std::atoi(std::getenv("HPSB_LOOKUP_SKIP")) : 0;
  LookupScratch lsd = ls;
  if (debug) {
    if (!dbg) cudaMalloc(&dbg, (16 + 3 * 8192) * 8);
    static unsigned long long init[16 + 3 * 8192] = {~0ull};
    cudaMemcpyAsync(dbg, init, sizeof(init), cudaMemcpyHostToDevice, st);
    lsd.dbg = dbg;
  }
  const int mode = (smem_tail ? 1 : 0) | (skip & 30);
  v.fn<<<grid, kLookupThreads, dyn, st>>>(c, keys, n, out, flags, default_row, stamp, lsd, mode);
  check_launch("lookup_probe", 1);
  if (!(mode & 16)) {
    constexpr int kGP = 8;
    const uint64_t warps = (n + kGP - 1) / kGP;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned((warps * 32 + 255) / 256));
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_lookup_gather<kGP>, c, n, out, default_row, lsd, mode);
    check_launch("lookup_gather", 1);
  }
  if (debug) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const double tot = double(h[4] + h[5] + h[6] + h[7] + h[8]) + 1e-9;
    std::fprintf(stderr,
                 "lookup_timing n=%llu grid=%u body_us=%.2f tail_wait_us=%.2f tail_us=%.2f "
                 "phases hash=%.2f probe=%.2f exch=%.2f gather=%.2f book=%.2f warp_cycles=%.0f\n",
                 (unsigned long long)n, grid, (h[1] - h[0]) * 1e-3, (h[2] - h[1]) * 1e-3,
                 (h[3] - h[2]) * 1e-3, h[4] / tot, h[5] / tot, h[6] / tot, h[7] / tot, h[8] / tot,
                 tot / double(n / 32));
    std::fprintf(stderr, "  tail phases: firsts=%.2f scan=%.2f ranks=%.2f end=%.2f us\n",
                 (h[9] - h[2]) * 1e-3, (h[10] - h[9]) * 1e-3, (h[11] - h[10]) * 1e-3,
                 (h[3] - h[11]) * 1e-3);
    const unsigned warps = grid * kLookupWarps;
    static unsigned long long w[3 * 8192];
    cudaMemcpy(w, dbg + 16, size_t(warps) * 3 * 8, cudaMemcpyDeviceToHost);
    std::vector<double> st_off, life, life_miss, life_nomiss;
    unsigned long long t0 = ~0ull;
    for (unsigned i = 0; i < warps; ++i) t0 = std::min(t0, w[3 * i]);
    for (unsigned i = 0; i < warps; ++i) {
      st_off.push_back((w[3 * i] - t0) * 1e-3);
      const double l = (w[3 * i + 1] - w[3 * i]) * 1e-3;
      life.push_back(l);
      (w[3 * i + 2] & 1 ? life_miss : life_nomiss).push_back(l);
    }
    auto pct = [](std::vector<double> v, double p) {
      if (v.empty()) return 0.0;
      std::sort(v.begin(), v.end());
      return v[size_t(p * (v.size() - 1))];
    };
    std::fprintf(stderr,
                 "  warps: start p50=%.2f p99=%.2f max=%.2f | life p10=%.2f p50=%.2f p90=%.2f "
                 "max=%.2f | life(miss) p50=%.2f (n=%zu) life(no miss) p50=%.2f\n",
                 pct(st_off, .5), pct(st_off, .99), pct(st_off, 1), pct(life, .1), pct(life, .5),
                 pct(life, .9), pct(life, 1), pct(life_miss, .5), life_miss.size(),
                 pct(life_nomiss, .5));
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
