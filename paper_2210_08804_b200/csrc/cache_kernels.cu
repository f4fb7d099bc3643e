// cache_kernels.cu -- sm_100a kernels for SlabCache query / replace /
// update / dump and for GPU dedup.
//
// Reference behaviour restated here (all under /root/reference/proj):
//   query    core/src/slab_cache.cpp:69-91, 228-259
//   replace  core/src/slab_cache.cpp:93-107, 261-326
//   update   core/src/slab_cache.cpp:109-125, 328-358
//   dump     core/src/slab_cache.cpp:360-394
//   dedup    core/src/types.cpp:20-34
#include <cuda_runtime.h>

#include <atomic>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "kernels.hpp"
#include "probe.cuh"
#include "tag_probe.cuh"

namespace hpsb {

namespace {

inline void check_launch(const char* what, uint32_t kernels) {
  note_launches(kernels);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

inline uint64_t pow2_at_least(uint64_t v) {
  uint64_t c = 16;
  while (c < v) c <<= 1;
  return c;
}

inline uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

constexpr int kWarpsPerBlock = 8;  // 256-thread blocks for warp-per-key kernels

}  // namespace

static std::atomic<uint64_t> g_launches{0};
void note_launches(uint32_t kernels) { g_launches.fetch_add(kernels, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

// ------------------------------------------------------------------ scan --
void scan_begin(ScanState& s, uint64_t tiles, cudaStream_t st) {
  (void)tiles;
  s.epoch = (s.epoch + 1) & 0xFFFFFFu;
  if (s.epoch == 0) {
    // 24-bit epoch wrapped: clear the status words once, then restart at 1
    cudaMemsetAsync(s.status, 0, s.capacity_tiles * sizeof(uint64_t), st);
    s.epoch = 1;
  }
}

// ------------------------------------------------------------------ query --
// One warp serves P keys (P = keys_per_warp): hits copy the row into out[i]
// and stamp the slot; misses leave out[i] untouched (slab_cache.cpp:248-251).
template <int P>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    k_cache_query(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                  float* __restrict__ out, uint8_t* __restrict__ hit, uint64_t stamp) {
  const uint64_t warp = (uint64_t(blockIdx.x) * kWarpsPerBlock) + (threadIdx.x >> 5);
  const uint64_t base = warp * P;
  if (base >= n) return;
  WarpKeys<P> wk;
  warp_load_keys<P>(c, keys, base, n, wk);
  uint32_t slot[P];
  warp_probe<P>(c, wk, slot);
  const uint32_t lane = lane_id();
#pragma unroll
  for (int p = 0; p < P; ++p) {
    if (!wk.valid[p]) continue;
    const uint64_t i = base + p;
    if (slot[p] != kNoSlot) {
      warp_copy_row(c.rows + uint64_t(slot[p]) * c.d, out + i * c.d, c.d);
      if (lane == 0) {
        c.counters[slot[p]] = stamp;
        hit[i] = 1;
      }
    } else if (lane == 0) {
      hit[i] = 0;
    }
  }
}

void launch_cache_query(const CacheDev& c, const uint64_t* keys, uint64_t n, float* out,
                        uint8_t* hit, uint64_t stamp, int keys_per_warp, cudaStream_t st) {
  if (n == 0) return;
  const int P = keys_per_warp >= 8 ? 8 : (keys_per_warp >= 4 ? 4 : (keys_per_warp >= 2 ? 2 : 1));
  const uint64_t warps = (n + P - 1) / P;
  const dim3 grid(unsigned((warps + kWarpsPerBlock - 1) / kWarpsPerBlock));
  const dim3 block(kWarpsPerBlock * 32);
  switch (P) {
    case 8: k_cache_query<8><<<grid, block, 0, st>>>(c, keys, n, out, hit, stamp); break;
    case 4: k_cache_query<4><<<grid, block, 0, st>>>(c, keys, n, out, hit, stamp); break;
    case 2: k_cache_query<2><<<grid, block, 0, st>>>(c, keys, n, out, hit, stamp); break;
    default: k_cache_query<1><<<grid, block, 0, st>>>(c, keys, n, out, hit, stamp); break;
  }
  check_launch("cache_query", 1);
}

__global__ void __launch_bounds__(kScanBlock)
    k_select_misses(const uint64_t* __restrict__ keys, const uint8_t* __restrict__ hit,
                    uint64_t n, uint32_t* __restrict__ miss_pos,
                    uint64_t* __restrict__ miss_keys, unsigned long long* n_miss,
                    ScanState scan) {
  select_tile(
      n, scan, [&](uint64_t i) { return hit[i] == 0; },
      [&](uint64_t i, uint64_t r) {
        miss_pos[r] = uint32_t(i);
        miss_keys[r] = keys[i];
      },
      n_miss);
}

void launch_select_misses(const uint64_t* keys, const uint8_t* hit, uint64_t n,
                          uint32_t* miss_pos, uint64_t* miss_keys,
                          unsigned long long* n_miss, ScanState& scan, cudaStream_t st) {
  if (n == 0) {
    cudaMemsetAsync(n_miss, 0, sizeof(unsigned long long), st);
    return;
  }
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  scan_begin(scan, tiles, st);
  k_select_misses<<<unsigned(tiles), kScanBlock, 0, st>>>(keys, hit, n, miss_pos, miss_keys,
                                                          n_miss, scan);
  scan.tile_base += tiles;
  check_launch("select_misses", 1);
}

// ---------------------------------------------------------------- replace --
// Deterministic parity with the reference's grouped application
// (slab_cache.cpp:131-142: keys grouped by slabset, input order inside a
// group) in two launches and no memsets (batches above kSmallReplaceMax):
//   k_replace_bin    one thread per key: slabset, the set's entry in a
//                    per-call table (one 64-bit word: set id | key count; the
//                    CAS that claims it ranks the first key, an add ranks the
//                    rest), the key's index and the key itself appended there;
//                    the rank-0 key publishes (entry, set) into a compact list
//                    of touched sets (one warp-aggregated add per warp)
//   [k_replace_dups] (validated calls) a warp per touched set compares its
//                    keys: any duplicate rejects the whole call before mutation
//   k_replace_sets   persistent warps over the compact list of TOUCHED SETS
//                    (each warp walks it with a stride, the next item's list
//                    entry in flight while the current one is applied; the
//                    walk ends on the list's sentinel): the set's masks, keys
//                    and counters loaded ONCE into registers (lane j holds slot
//                    j of every slab) together with the set's key indices and
//                    keys, the indices sorted into input order, the first rows
//                    prefetched; then every key of the set applied serially
//                    against that register state -- probe by ballot, lowest
//                    free slot of the first non-full probed slab, else the
//                    argmin counter (ties to the lowest (slab, slot)); only the
//                    changed words are stored; the set's table entry and list
//                    slot are cleared (the scratch is clean again). Dependent
//                    round trips per set: (set state, indices, keys) -> rows.
size_t replace_scratch_bytes(uint64_t n) {
  const uint64_t cap = pow2_at_least(2 * n);
  return align_up(cap * 8, 256) + align_up(cap * 4, 256) * 2 + align_up(cap * 4 * kReplaceInline, 256) * 2 +
         align_up(cap * 8 * kReplaceInline, 256) + align_up(n * 4, 256) * 4 + 256;
}

ReplaceScratch replace_scratch_carve(void* base, uint64_t n) {
  ReplaceScratch r;
  r.cap = pow2_at_least(2 * n);
  r.ncap = n;
  char* p = static_cast<char*>(base);
  auto take = [&](uint64_t bytes) {
    uint32_t* q = reinterpret_cast<uint32_t*>(p);
    p += align_up(bytes, 256);
    return q;
  };
  // zero-initialised part first, then the all-ones part (two memsets once)
  r.ent = reinterpret_cast<unsigned long long*>(take(r.cap * 8));
  r.cursor = take(256);
  r.dup_flag = r.cursor + 1;
  r.ovf = take(r.cap * 4);
  r.boff = take(r.cap * 4);
  r.lead_e = take(n * 4);
  r.idx = take(r.cap * 4 * kReplaceInline);
  r.kin = reinterpret_cast<uint64_t*>(take(r.cap * 8 * kReplaceInline));
  r.hin = take(r.cap * 4 * kReplaceInline);
  r.next = take(n * 4);
  r.lead_s = take(n * 4);
  r.bucket = take(n * 4);
  return r;
}

void replace_scratch_init(const ReplaceScratch& rs, cudaStream_t st) {
  const char* z0 = reinterpret_cast<const char*>(rs.ent);
  const char* o0 = reinterpret_cast<const char*>(rs.ovf);
  const char* o1 = reinterpret_cast<const char*>(rs.idx);
  cudaMemsetAsync(rs.ent, 0, size_t(o0 - z0), st);
  cudaMemsetAsync(rs.ovf, 0xFF, size_t(o1 - o0), st);
}

constexpr uint32_t kNone = 0xFFFFFFFFu;

// The set kernel's register cap (4 blocks of 256 per SM: 32 warps) and the
// rows it prefetches into registers per set. A/B on B200 (profiles/
// r02_ab_replace.txt): the cap is worth ~30 %; L2 prefetches of the input
// rows / set state from the bin kernel were measured and dropped (no gain).
#ifndef HPSB_REPL_MINB
#define HPSB_REPL_MINB 4
#endif
#ifndef HPSB_REPL_KPRE
#define HPSB_REPL_KPRE 2
#endif

// DIRECT: a call touching a cache of at most `cap` slabsets indexes the set
// table by the slabset itself (one atomicAdd per key, no CAS probe). FAST:
// the bin kernel hands each inline key's slab meta to the set kernel, and
// the eviction argmin uses 32-bit warp min-reductions while every counter
// and the stamp fit in 32 bits. Together 47.1-47.6 -> 40.9-42.4 us per
// 65,536-key fill (profiles/r02_ab_replace.txt, r02ay).
#ifndef HPSB_REPL_DIRECT
#define HPSB_REPL_DIRECT 1
#endif
#ifndef HPSB_REPL_FAST
#define HPSB_REPL_FAST 1
#endif
#ifndef HPSB_REPL_BINAGG
#define HPSB_REPL_BINAGG 1
#endif
// DYN: items handed out per block from a shared counter (40.3-40.9 -> 39.2-39.8 us,
// r02bb; one global counter was slower: r02q)
#ifndef HPSB_REPL_DYN
#define HPSB_REPL_DYN 1
#endif
// A key's slab-hash facts the set kernel needs (its first probed slab and
// its fingerprint), computed once per key by the bin kernel's thread rather
// than by a whole warp per set: tag << 24 | first slab.
__device__ __forceinline__ uint32_t slab_meta(const CacheDev& c, uint64_t key) {
  const uint64_t h2 = xxh64_key(key, kSlabSeed);
  const uint32_t first =
      c.W == 1 ? 0u : (c.W == 2 ? uint32_t(h2 & 1u) : uint32_t(fastmod(h2, c.W, c.mW)));
  return (uint32_t(key_tag(h2)) << 24) | first;
}

__global__ void __launch_bounds__(256)
    k_replace_bin(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n, ReplaceScratch rs) {
  // the set kernel may launch now (it waits for this grid before reading)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) {
    rs.cursor[0] = 0u;
    rs.dup_flag[0] = 0u;
  }
  bool lead = false;
  uint32_t e32 = 0;
  uint64_t set = 0;
  if (i < n) {
    const uint64_t key = keys[i];
    set = slabset_of(c, key);
    const unsigned long long tag = (set + 1ull) << 32;
    const uint64_t mask = rs.cap - 1;
    uint64_t e = fmix64(set + 1ull) & mask;
    uint32_t r;
#if HPSB_REPL_DIRECT
    // no more sets than table entries: the set IS its entry (one atomic per
    // key for its rank, no CAS probe)
    const bool direct = c.S <= rs.cap;
    if (direct) {
      e = set;
      r = uint32_t(atomicAdd(rs.ent + e, 1ull));
    }
    while (!direct) {
#else
    while (true) {
#endif
      const unsigned long long old = atomicCAS(rs.ent + e, 0ull, tag | 1ull);
      if (old == 0ull) {
        r = 0;
        break;
      }
      if ((old >> 32) == (tag >> 32)) {
        r = uint32_t(atomicAdd(rs.ent + e, 1ull));  // the low word: this key's rank
        break;
      }
      e = (e + 1) & mask;
    }
    if (r < kReplaceInline) {
      rs.idx[e * kReplaceInline + r] = uint32_t(i);
      rs.kin[e * kReplaceInline + r] = key;
#if HPSB_REPL_FAST
      rs.hin[e * kReplaceInline + r] = slab_meta(c, key);
#endif
    } else {
      rs.next[i] = atomicExch(rs.ovf + e, uint32_t(i));
    }
    lead = r == 0;
    e32 = uint32_t(e);
  }
#if HPSB_REPL_BINAGG
  // the touched-set list: one global cursor add per BLOCK (every warp adding
  // on the same word serialised ~2,000 same-address atomics in one L2 slice)
  __shared__ uint32_t s_cnt, s_base;
  if (threadIdx.x == 0) s_cnt = 0u;
  __syncthreads();
  const uint32_t lm = __ballot_sync(0xFFFFFFFFu, lead);
  const uint32_t lane = lane_id();
  uint32_t woff = 0;
  if (lane == 0 && lm) woff = atomicAdd(&s_cnt, uint32_t(__popc(lm)));
  woff = __shfl_sync(0xFFFFFFFFu, woff, 0);
  __syncthreads();
  if (threadIdx.x == 0 && s_cnt) s_base = atomicAdd(rs.cursor + 2, s_cnt);
  __syncthreads();
  if (lead) {
    const uint32_t k = s_base + woff + uint32_t(__popc(lm & ((1u << lane) - 1u)));
    rs.lead_e[k] = e32;
    rs.lead_s[k] = uint32_t(set);
  }
#else
  __syncwarp();
  const uint32_t lm = __ballot_sync(0xFFFFFFFFu, lead);
  if (lm == 0u) return;
  const uint32_t lane = lane_id();
  uint32_t base = 0;
  if (lane == 0) base = atomicAdd(rs.cursor + 2, uint32_t(__popc(lm)));
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  if (lead) {
    const uint32_t k = base + uint32_t(__popc(lm & ((1u << lane) - 1u)));
    rs.lead_e[k] = e32;
    rs.lead_s[k] = uint32_t(set);
  }
#endif
}

// Sets of more than 32 keys (tiny caches): the indices in a sorted bucket
// range, built once per call by whichever kernel needs it first.
__device__ __forceinline__ const uint32_t* big_bucket(const ReplaceScratch& rs, uint64_t e,
                                                      uint32_t cnt) {
  uint32_t off = 0;
  if (lane_id() == 0) {
    off = rs.boff[e];
    if (off == kNone) {
      off = atomicAdd(rs.cursor, cnt);
      uint32_t* b = rs.bucket + off;
      uint32_t j = 0;
      for (; j < kReplaceInline; ++j) b[j] = rs.idx[e * kReplaceInline + j];
      for (uint32_t x = rs.ovf[e]; x != kNone; x = rs.next[x]) b[j++] = x;
      rs.boff[e] = off;
    }
  }
  off = __shfl_sync(0xFFFFFFFFu, off, 0);
  __syncwarp();
  uint32_t* b = rs.bucket + off;
  // rank sort / insertion sort (already sorted on the second call: linear)
  if (lane_id() == 0) {
    for (uint32_t a = 1; a < cnt; ++a) {
      const uint32_t x = b[a];
      uint32_t j = a;
      while (j > 0 && b[j - 1] > x) {
        b[j] = b[j - 1];
        --j;
      }
      b[j] = x;
    }
  }
  __syncwarp();
  return b;
}

// Indices of a set with at most 32 keys into lanes, sorted: lane j holds the
// j-th smallest (kNone past cnt) and, in *key, that key. `sw` = 32 words and
// `sk` = 32 keys of per-warp shared memory.
__device__ __forceinline__ uint32_t small_group(const ReplaceScratch& rs, uint64_t e, uint32_t cnt,
                                                const uint64_t* __restrict__ keys, uint32_t* sw,
                                                uint64_t* sk, uint64_t* key,
                                                bool preloaded = false, uint32_t v_in = kNone,
                                                uint64_t k_in = 0, uint32_t* meta = nullptr,
                                                const CacheDev* cd = nullptr) {
  // meta != nullptr: *meta holds the lane's preloaded slab meta on entry and
  // the sorted one on return (keys past the inline ones: computed here)
  const uint32_t lane = lane_id();
  uint32_t v = kNone;
  uint64_t k = 0;
  uint32_t mt = meta ? *meta : 0u;
  if (lane < kReplaceInline && lane < cnt) {
    v = preloaded ? v_in : rs.idx[e * kReplaceInline + lane];
    k = preloaded ? k_in : rs.kin[e * kReplaceInline + lane];
  }
  if (cnt > kReplaceInline) {
    if (lane == 0) {
      uint32_t j = kReplaceInline;
      for (uint32_t x = rs.ovf[e]; x != kNone && j < 32; x = rs.next[x]) sw[j++] = x;
    }
    __syncwarp();
    if (lane >= kReplaceInline && lane < cnt) {
      v = sw[lane];
      k = keys[v];
#if HPSB_REPL_FAST
      if (meta) mt = slab_meta(*cd, k);
#endif
    }
    __syncwarp();
  }
  if (cnt > 1) {
    uint32_t rank = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
      const uint32_t o = __shfl_sync(0xFFFFFFFFu, v, j);
      rank += (o < v) ? 1u : 0u;
    }
    // the metas sorted the same way (sw reused once the indices are out)
    if (lane < cnt) {
      sw[rank] = v;
      sk[rank] = k;
    }
    __syncwarp();
    const uint32_t vs = lane < cnt ? sw[lane] : kNone;
    k = lane < cnt ? sk[lane] : 0ull;
    __syncwarp();
    if (meta) {
      if (lane < cnt) sw[rank] = mt;
      __syncwarp();
      mt = lane < cnt ? sw[lane] : 0u;
      __syncwarp();
    }
    v = vs;
  }
  if (meta) *meta = mt;
  *key = k;
  return v;
}

__global__ void __launch_bounds__(256)
    k_replace_dups(const uint64_t* __restrict__ keys, uint64_t n, ReplaceScratch rs) {
  __shared__ uint32_t s_w[8][32];
  __shared__ uint64_t s_k[8][32];
  const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  const uint32_t e = rs.lead_e[w];
  if (e == kNone) return;
  const uint32_t cnt = uint32_t(rs.ent[e]);
  if (cnt < 2) return;
  const uint32_t lane = lane_id();
  bool dup = false;
  if (cnt <= 32) {
    uint64_t k;
    (void)small_group(rs, e, cnt, keys, s_w[threadIdx.x >> 5], s_k[threadIdx.x >> 5], &k);
    for (uint32_t j = 0; j < cnt; ++j) {
      const uint64_t o = __shfl_sync(0xFFFFFFFFu, k, j);
      dup |= (lane < cnt && j != lane && o == k);
    }
  } else {
    const uint32_t* b = big_bucket(rs, e, cnt);
    for (uint32_t x = lane; x < cnt; x += 32) {
      const uint64_t kx = keys[b[x]];
      for (uint32_t y = x + 1; y < cnt; ++y) dup |= (keys[b[y]] == kx);
    }
  }
  if (__any_sync(0xFFFFFFFFu, dup) && lane == 0) atomicOr(rs.dup_flag, 1u);
}

// The set's state in registers: lane j holds slot j of each of its W slabs.
template <int W>
struct SetRegs {
  uint64_t k[W];
  uint64_t ct[W];
  uint32_t m[W];
};

// Returns the number of keys inserted into free slots (lane 0's value).
template <int W>
__device__ __forceinline__ void load_set(const CacheDev& c, uint64_t set, SetRegs<W>& st) {
  const uint32_t lane = lane_id();
  const uint64_t sbase = set * W;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    st.m[w] = c.masks[sbase + w];
    st.k[w] = c.keys[(sbase + w) * kSlotsPerSlab + lane];
    st.ct[w] = c.counters[(sbase + w) * kSlotsPerSlab + lane];
  }
}

template <int W>
__device__ __forceinline__ uint32_t replace_apply_set(const CacheDev& c, uint64_t set,
                                                  const uint64_t* __restrict__ keys,
                                                  const float* __restrict__ rows, uint64_t stamp,
                                                  uint32_t cnt, uint32_t my_idx,
                                                  uint64_t my_key_in,
                                                  const uint32_t* __restrict__ big,
                                                  const SetRegs<W>& loaded,
                                                  uint32_t my_meta_in = 0u) {
  constexpr int kPre = HPSB_REPL_KPRE;  // rows prefetched (d <= 128, 16 B aligned)
  const uint32_t lane = lane_id();
  const uint32_t d = c.d;
  const uint64_t sbase = set * W;
  SetRegs<W> st = loaded;  // loaded with the set's count and inline keys
  uint32_t m0[W];
#pragma unroll
  for (int w = 0; w < W; ++w) m0[w] = st.m[w];
  // lane j < cnt: key and first-slab hash of the j-th key (small groups)
  uint64_t my_key = 0;
#if HPSB_REPL_FAST
  // the bin kernel's per-key slab meta (tag << 24 | first slab)
  uint32_t my_meta = 0;
  if (big == nullptr && my_idx != kNone) {
    my_key = my_key_in;
    my_meta = my_meta_in;
  }
  // every counter of the set and the stamp below 2^32: the eviction argmin
  // runs on the low words with warp min-reductions
  bool lo32 = (stamp >> 32) == 0;
#pragma unroll
  for (int x = 0; x < W; ++x) lo32 = lo32 && (st.ct[x] >> 32) == 0;
  lo32 = __all_sync(0xFFFFFFFFu, lo32);
#else
  (void)my_meta_in;
  uint64_t my_h2 = 0;
  if (big == nullptr && my_idx != kNone) {
    my_key = my_key_in;
    my_h2 = xxh64_key(my_key, kSlabSeed);
  }
#endif
  const bool vec = (d & 3u) == 0 && d <= 128 && (reinterpret_cast<uintptr_t>(rows) & 15u) == 0;
  float4 pre[kPre];
  if (vec && big == nullptr) {
#pragma unroll
    for (int j = 0; j < kPre; ++j) {
      const uint32_t ij = __shfl_sync(0xFFFFFFFFu, my_idx, j);
      pre[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (uint32_t(j) < cnt && lane < (d >> 2))
        pre[j] = reinterpret_cast<const float4*>(rows + uint64_t(ij) * d)[lane];
    }
  }
  uint32_t inserted = 0;
  for (uint32_t j = 0; j < cnt; ++j) {
    uint32_t ij;
    uint64_t key;
#if HPSB_REPL_FAST
    uint32_t meta;
    if (big == nullptr) {
      ij = __shfl_sync(0xFFFFFFFFu, my_idx, j);
      key = __shfl_sync(0xFFFFFFFFu, my_key, j);
      meta = __shfl_sync(0xFFFFFFFFu, my_meta, j);
    } else {
      ij = big[j];
      key = keys[ij];
      meta = slab_meta(c, key);
    }
    const uint32_t first = meta & 0xFFFFFFu;
    const uint8_t ktag = uint8_t(meta >> 24);
#else
    uint64_t h2;
    if (big == nullptr) {
      ij = __shfl_sync(0xFFFFFFFFu, my_idx, j);
      key = __shfl_sync(0xFFFFFFFFu, my_key, j);
      h2 = __shfl_sync(0xFFFFFFFFu, my_h2, j);
    } else {
      ij = big[j];
      key = keys[ij];
      h2 = xxh64_key(key, kSlabSeed);
    }
    const uint32_t first = W == 1 ? 0u : (W == 2 ? uint32_t(h2 & 1u) : uint32_t(fastmod(h2, W, c.mW)));
    const uint8_t ktag = key_tag(h2);
#endif
    // probe in slab order from `first` (slab_cache.cpp:292-310)
    int hit_w = -1, ins_w = -1;
    uint32_t hit_j = 0;
#pragma unroll
    for (int step = 0; step < W; ++step) {
      int w = int(first) + step;
      if (w >= W) w -= W;
      if (hit_w >= 0 || ins_w >= 0) continue;
      uint64_t kw = 0;
      uint32_t mw = 0;
#pragma unroll
      for (int x = 0; x < W; ++x)
        if (x == w) {
          kw = st.k[x];
          mw = st.m[x];
        }
      const uint32_t hb = __ballot_sync(0xFFFFFFFFu, ((mw >> lane) & 1u) && kw == key);
      if (hb) {
        hit_w = w;
        hit_j = __ffs(hb) - 1;
      } else if (mw != kFullSlab) {
        ins_w = w;
      }
    }
    if (hit_w >= 0) {
      // resident: recency refresh only, the vector is kept (:283-288)
      if (lane == hit_j) {
#pragma unroll
        for (int x = 0; x < W; ++x)
          if (x == hit_w) st.ct[x] = stamp;
        c.counters[(sbase + hit_w) * kSlotsPerSlab + lane] = stamp;
      }
      continue;
    }
    int tw;
    uint32_t tj;
    if (ins_w >= 0) {
      uint32_t mw = 0;
#pragma unroll
      for (int x = 0; x < W; ++x)
        if (x == ins_w) mw = st.m[x];
      tj = __ffs(~mw) - 1;  // countr_one(mask) (:299)
#pragma unroll
      for (int x = 0; x < W; ++x)
        if (x == ins_w) st.m[x] = mw | (1u << tj);
      tw = ins_w;
      ++inserted;
    } else {
      // every probed slab full: evict the minimum counter of the set, ties
      // to the lowest (slab, slot) in slab-major order (:312-324)
      uint64_t bc = st.ct[0];
      uint32_t bi = lane;
#pragma unroll
      for (int x = 1; x < W; ++x)
        if (st.ct[x] < bc) {
          bc = st.ct[x];
          bi = uint32_t(x) * 32 + lane;
        }
#if HPSB_REPL_FAST
      if (lo32) {
        const uint32_t mn = __reduce_min_sync(0xFFFFFFFFu, uint32_t(bc));
        bi = __reduce_min_sync(0xFFFFFFFFu, uint32_t(bc) == mn ? bi : 0xFFFFFFFFu);
      } else
#endif
      {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const uint64_t oc = __shfl_xor_sync(0xFFFFFFFFu, bc, o);
          const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
          if (oc < bc || (oc == bc && oi < bi)) {
            bc = oc;
            bi = oi;
          }
        }
      }
      tw = int(bi >> 5);
      tj = bi & 31u;
    }
    const uint64_t slot = (sbase + tw) * kSlotsPerSlab + tj;
    if (lane == tj) {
#pragma unroll
      for (int x = 0; x < W; ++x)
        if (x == tw) {
          st.k[x] = key;
          st.ct[x] = stamp;
        }
      c.keys[slot] = key;
      c.counters[slot] = stamp;
      c.tags[slot] = ktag;
    }
    const float* src = rows + uint64_t(ij) * d;
    float* dst = c.rows + slot * d;
    if (vec && big == nullptr && j < uint32_t(kPre)) {
      float4 x = pre[0];
#pragma unroll
      for (int q = 1; q < kPre; ++q)
        if (uint32_t(q) == j) x = pre[q];
      if (lane < (d >> 2)) reinterpret_cast<float4*>(dst)[lane] = x;
    } else {
      warp_copy_row(src, dst, d);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int w = 0; w < W; ++w)
      if (st.m[w] != m0[w]) c.masks[sbase + w] = st.m[w];
  }
  return inserted;
}

__device__ __forceinline__ void warp_replace_key(const CacheDev& c, uint64_t set, uint64_t key,
                                                 const float* __restrict__ row, uint64_t stamp);

// W = 0: any slab count, the set re-read for every key (warp_replace_key)
template <int W>
__global__ void __launch_bounds__(256, HPSB_REPL_MINB)
    k_replace_sets(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                   const float* __restrict__ rows, uint64_t stamp, uint32_t validate,
                   ReplaceScratch rs) {
  __shared__ uint32_t s_w[8][32];
  __shared__ uint64_t s_k[8][32];
  __shared__ unsigned long long s_ins;
#if HPSB_REPL_DYN
  // the block's items are list entries blockIdx + gridDim * k; its warps
  // take k = 0..7 first, then grab the next k from a shared counter (sets
  // carry 1..10 keys: a static share leaves warps idle at the end)
  __shared__ uint32_t s_next;
  if (threadIdx.x == 0) s_next = blockDim.x >> 5;
#endif
  if (threadIdx.x == 0) s_ins = 0ull;
  __syncthreads();
  // launched as the bin kernel's programmatic dependent: everything below
  // reads what bin wrote
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if HPSB_REPL_DYN
  uint64_t w = uint64_t(blockIdx.x) + uint64_t(gridDim.x) * (threadIdx.x >> 5);
#else
  const uint64_t stride = uint64_t(gridDim.x) * (blockDim.x >> 5);
  uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
#endif
  // the list is consumed through its sentinels; its count restarts here
  if (blockIdx.x == 0 && threadIdx.x == 0) rs.cursor[2] = 0u;
  const bool rejected = validate && *reinterpret_cast<volatile uint32_t*>(rs.dup_flag) != 0u;
  uint32_t e = w < n ? rs.lead_e[w] : kNone;
  uint32_t sset = w < n ? rs.lead_s[w] : 0u;
  uint32_t inserted = 0;
  while (e != kNone) {
    // the next item's list entry is in flight while this one is applied
#if HPSB_REPL_DYN
    uint32_t kn = 0;
    if (lane_id() == 0) kn = atomicAdd(&s_next, 1u);
    const uint64_t wn =
        uint64_t(blockIdx.x) + uint64_t(gridDim.x) * __shfl_sync(0xFFFFFFFFu, kn, 0);
#else
    const uint64_t wn = w + stride;
#endif
    const uint32_t en = wn < n ? rs.lead_e[wn] : kNone;
    const uint32_t sn = wn < n ? rs.lead_s[wn] : 0u;
    const uint64_t set = sset;
    // ONE round trip: the set's key count, its inline key indices and keys
    // (read whatever the count; entries past it are ignored) and the set's
    // masks / keys / counters -- all depend only on the list entry
    const uint32_t cnt = uint32_t(rs.ent[e]);
    const uint32_t lane = lane_id();
    uint32_t v_in = kNone, m_in = 0u;
    uint64_t k_in = 0;
    if (lane < kReplaceInline) {
      v_in = rs.idx[uint64_t(e) * kReplaceInline + lane];
      k_in = rs.kin[uint64_t(e) * kReplaceInline + lane];
#if HPSB_REPL_FAST
      if constexpr (W > 0) m_in = rs.hin[uint64_t(e) * kReplaceInline + lane];
#endif
    }
    SetRegs<W == 0 ? 1 : W> pre;
    if constexpr (W > 0) {
      if (!rejected) load_set<W>(c, set, pre);
    }
    if (!rejected) {
      uint64_t k = 0;
      const uint32_t v = cnt <= 32 ? small_group(rs, e, cnt, keys, s_w[threadIdx.x >> 5],
                                                 s_k[threadIdx.x >> 5], &k, true, v_in, k_in,
                                                 (HPSB_REPL_FAST && W > 0) ? &m_in : nullptr, &c)
                                   : kNone;
      const uint32_t* b = cnt <= 32 ? nullptr : big_bucket(rs, e, cnt);
      if constexpr (W == 0) {
        for (uint32_t j = 0; j < cnt; ++j) {
          const uint32_t ij = b ? b[j] : __shfl_sync(0xFFFFFFFFu, v, j);
          warp_replace_key(c, set, keys[ij], rows + uint64_t(ij) * c.d, stamp);
        }
      } else {
        inserted += replace_apply_set<W>(c, set, keys, rows, stamp, cnt, v, k, b, pre, m_in);
      }
    }
    __syncwarp();
    if (lane_id() == 0) {
      // the scratch is clean again for the next call
      rs.ent[e] = 0ull;
      rs.ovf[e] = kNone;
      rs.boff[e] = kNone;
      rs.lead_e[w] = kNone;
    }
    w = wn;
    e = en;
    sset = sn;
  }
  // occupancy: one atomic per block (W = 0 counts per key in warp_replace_key)
  if (lane_id() == 0 && inserted) atomicAdd(&s_ins, (unsigned long long)inserted);
  __syncthreads();
  if (threadIdx.x == 0 && s_ins) atomicAdd(c.occupied, s_ins);
}

// One key of a set, applied by a whole warp (slab_cache.cpp:261-326): ballot
// probe of the set's slabs in probe order; resident -> recency refresh only;
// else insert at the lowest free slot of the first non-full probed slab; else
// evict the minimum counter of the set, ties to the lowest (slab, slot).
__device__ __forceinline__ void warp_replace_key(const CacheDev& c, uint64_t set, uint64_t key,
                                                 const float* __restrict__ row, uint64_t stamp) {
  const uint32_t lane = lane_id();
  volatile uint32_t* vmask = c.masks;
  volatile uint64_t* vkeys = c.keys;
  volatile uint64_t* vctr = c.counters;
  const uint64_t per_set = uint64_t(c.W) * kSlotsPerSlab;
  const uint32_t first = first_slab_of(c, key);
  // rows of up to 128 floats: prefetched into registers with everything else
  const bool pre = (c.d & 3u) == 0 && c.d <= 128 && (reinterpret_cast<uintptr_t>(row) & 15u) == 0;
  float4 rv = make_float4(0.f, 0.f, 0.f, 0.f);
  if (pre && lane < (c.d >> 2)) rv = reinterpret_cast<const float4*>(row)[lane];
  if (c.W == 2) {
    // both slabs' masks and keys and the set's 64 counters in ONE round trip
    const uint64_t sa = set * 2 + first, sb = set * 2 + (first ^ 1u);
    const uint32_t ma = vmask[sa], mb = vmask[sb];
    const uint64_t ka = vkeys[sa * kSlotsPerSlab + lane], kb = vkeys[sb * kSlotsPerSlab + lane];
    const uint64_t c0 = vctr[set * 64 + lane], c1 = vctr[set * 64 + 32 + lane];
    uint64_t slot;
    int64_t found = -1;
    const uint32_t ha = __ballot_sync(0xFFFFFFFFu, ((ma >> lane) & 1u) && ka == key);
    const uint32_t hb = __ballot_sync(0xFFFFFFFFu, ((mb >> lane) & 1u) && kb == key);
    if (ha) {
      found = int64_t(sa * kSlotsPerSlab + (__ffs(ha) - 1));
    } else if (ma == kFullSlab && hb) {
      found = int64_t(sb * kSlotsPerSlab + (__ffs(hb) - 1));
    }
    if (found >= 0) {
      if (lane == 0) vctr[found] = stamp;  // resident: recency refresh only
      __syncwarp();
      return;
    }
    if (ma != kFullSlab || mb != kFullSlab) {
      const uint64_t ins = ma != kFullSlab ? sa : sb;
      const uint32_t m = ma != kFullSlab ? ma : mb;
      const uint32_t j = __ffs(~m) - 1;  // countr_one(mask) (slab_cache.cpp:299)
      slot = ins * kSlotsPerSlab + j;
      if (lane == 0) {
        vmask[ins] = m | (1u << j);
        atomicAdd(c.occupied, 1ull);
      }
    } else {
      uint64_t best_c = c0;
      uint32_t best_i = lane;
      if (c1 < best_c) {
        best_c = c1;
        best_i = lane + 32;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t oc = __shfl_xor_sync(0xFFFFFFFFu, best_c, o);
        const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, best_i, o);
        if (oc < best_c || (oc == best_c && oi < best_i)) {
          best_c = oc;
          best_i = oi;
        }
      }
      slot = set * 64 + best_i;
    }
    if (lane == 0) {
      vkeys[slot] = key;
      vctr[slot] = stamp;
      c.tags[slot] = key_tag(xxh64_key(key, kSlabSeed));
    }
    if (pre) {
      if (lane < (c.d >> 2)) reinterpret_cast<float4*>(c.rows + slot * c.d)[lane] = rv;
    } else {
      warp_copy_row(row, c.rows + slot * c.d, c.d);
    }
    __threadfence_block();
    __syncwarp();
    return;
  }
  int64_t found = -1;
  int64_t ins_slab = -1;
  for (uint32_t step = 0; step < c.W; ++step) {
    uint32_t sl = first + step;
    sl = (sl >= c.W) ? sl - c.W : sl;
    const uint64_t slab = set * c.W + sl;
    const uint32_t m = vmask[slab];
    const uint64_t k = vkeys[slab * kSlotsPerSlab + lane];
    const uint32_t hitb = __ballot_sync(0xFFFFFFFFu, ((m >> lane) & 1u) && k == key);
    if (hitb) {
      found = int64_t(slab * kSlotsPerSlab + (__ffs(hitb) - 1));
      break;
    }
    if (m != kFullSlab) {
      ins_slab = int64_t(slab);
      break;
    }
  }
  if (found >= 0) {
    // resident: recency refresh only, vector kept (slab_cache.cpp:283-288)
    if (lane == 0) vctr[found] = stamp;
    __syncwarp();
    return;
  }
  uint64_t slot;
  if (ins_slab >= 0) {
    const uint32_t m = vmask[ins_slab];
    const uint32_t j = __ffs(~m) - 1;  // countr_one(mask) (slab_cache.cpp:299)
    slot = uint64_t(ins_slab) * kSlotsPerSlab + j;
    if (lane == 0) {
      vmask[ins_slab] = m | (1u << j);
      atomicAdd(c.occupied, 1ull);
    }
  } else {
    // all slabs full: evict min counter, ties to lowest (slab, slot)
    const uint64_t base = set * per_set;
    uint64_t best_c = ~0ull;
    uint32_t best_i = 0xFFFFFFFFu;
    for (uint32_t s = lane; s < per_set; s += 32) {
      const uint64_t cv = vctr[base + s];
      if (cv < best_c) {
        best_c = cv;
        best_i = s;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t oc = __shfl_xor_sync(0xFFFFFFFFu, best_c, o);
      const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, best_i, o);
      if (oc < best_c || (oc == best_c && oi < best_i)) {
        best_c = oc;
        best_i = oi;
      }
    }
    slot = base + best_i;
  }
  if (lane == 0) {
    vkeys[slot] = key;
    vctr[slot] = stamp;
    c.tags[slot] = key_tag(xxh64_key(key, kSlabSeed));
  }
  warp_copy_row(row, c.rows + slot * c.d, c.d);
  __threadfence_block();
  __syncwarp();
}

// Small batches (the engine's per-call unique misses at small batch sizes;
// n <= kSmallReplaceMax) in ONE single-block launch without scratch
// memsets -- 32 warps take the touched sets 32 at a time, so beyond a few
// hundred keys the multi-kernel path's warp per set wins: (set, index) pairs
// bitonic-sorted in shared memory (input order within each set), one warp per
// set applying its keys serially as above; the duplicate check (device-mode
// replace) runs over each set's keys before any mutation.
constexpr uint32_t kSmallReplace = 1024;   // block size (and sort capacity)
constexpr uint32_t kSmallReplaceMax = 256;  // dispatch limit

__global__ void __launch_bounds__(kSmallReplace)
    k_replace_small(CacheDev c, const uint64_t* __restrict__ keys, uint32_t n,
                    const float* __restrict__ rows, uint64_t stamp, uint32_t validate,
                    ReplaceScratch rs) {
  __shared__ unsigned long long sk[kSmallReplace];
  __shared__ uint32_t s_heads[kSmallReplace];
  __shared__ uint32_t s_nheads, s_dup;
  const uint32_t t = threadIdx.x;
  uint32_t P = 1;
  while (P < n) P <<= 1;
  if (t == 0) {
    s_nheads = 0;
    s_dup = 0;
  }
  if (t < P) sk[t] = t < n ? (slabset_of(c, keys[t]) << 10) | t : ~0ull;
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      const uint32_t x = t ^ j;
      if (t < P && x > t) {
        const unsigned long long a = sk[t], b = sk[x];
        if ((a > b) == ((t & k) == 0)) {
          sk[t] = b;
          sk[x] = a;
        }
      }
      __syncthreads();
    }
  }
  if (t < n && (t == 0 || (sk[t] >> 10) != (sk[t - 1] >> 10))) s_heads[atomicAdd(&s_nheads, 1u)] = t;
  __syncthreads();
  const uint32_t warp = t >> 5, lane = t & 31u, nh = s_nheads;
  if (validate) {
    for (uint32_t h = warp; h < nh; h += kSmallReplace / 32) {
      const uint32_t s0 = s_heads[h];
      const unsigned long long set = sk[s0] >> 10;
      uint32_t e = s0 + 1;
      while (e < n && (sk[e] >> 10) == set) ++e;
      bool dup = false;
      for (uint32_t x = s0 + lane; x < e; x += 32) {
        const uint64_t kx = keys[sk[x] & 1023u];
        for (uint32_t y = x + 1; y < e; ++y) dup |= keys[sk[y] & 1023u] == kx;
      }
      if (__any_sync(0xFFFFFFFFu, dup) && lane == 0) atomicOr(&s_dup, 1u);
    }
    __syncthreads();
  }
  if (!s_dup) {
    for (uint32_t h = warp; h < nh; h += kSmallReplace / 32) {
      const uint32_t s0 = s_heads[h];
      const unsigned long long set = sk[s0] >> 10;
      for (uint32_t g = s0; g < n && (sk[g] >> 10) == set; ++g) {
        const uint32_t i = uint32_t(sk[g] & 1023u);
        warp_replace_key(c, set, keys[i], rows + uint64_t(i) * c.d, stamp);
      }
    }
  }
  if (t == 0) {
    rs.cursor[0] = 0u;
    rs.dup_flag[0] = s_dup;
  }
}

// Small batches without the duplicate check (the engine's fills: unique
// misses): no sort at all -- one warp per key across as many blocks as
// needed; the warp owning the FIRST key of a set (in input order) applies
// every key of that set in input order, the others have nothing to do, so
// all touched sets proceed in parallel.
__global__ void __launch_bounds__(256)
    k_replace_tiny(CacheDev c, const uint64_t* __restrict__ keys, uint32_t n,
                   const float* __restrict__ rows, uint64_t stamp, ReplaceScratch rs) {
  __shared__ unsigned long long s_set[kSmallReplaceMax];
  __shared__ unsigned long long s_key[kSmallReplaceMax];
  for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
    const uint64_t k = keys[t];
    s_key[t] = k;
    s_set[t] = slabset_of(c, k);
  }
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rs.cursor[0] = 0u;
    rs.dup_flag[0] = 0u;
  }
  if (i >= n) return;
  const unsigned long long set = s_set[i];
  bool earlier = false;
  for (uint32_t j = lane; j < i; j += 32) earlier |= s_set[j] == set;
  if (__any_sync(0xFFFFFFFFu, earlier)) return;  // not the set's first key
  for (uint32_t j = i; j < n; ++j) {
    if (s_set[j] != set) continue;
    warp_replace_key(c, set, s_key[j], rows + uint64_t(j) * c.d, stamp);
  }
}

// ------------------------------------------------------- relaxed replace --
// Opt-in (SURVEY §7 "Hard parts": a relaxed atomicCAS-claim mode where the
// north star's tolerance clause applies): every key of the call is applied
// by its own warp, all keys at once -- no grouping by set, no per-set
// serialisation. Placement rules are the reference's (probe the W slabs from
// the first slab; resident -> recency refresh only; else the lowest free slot
// of the first non-full probed slab; else evict the minimum counter of the
// set, ties to the lowest (slab, slot), slab_cache.cpp:283-324), but keys of
// the same set race for slots and win them with atomics instead of being
// applied in input order. A won slot's counter holds stamp | kClaimBit until
// the call's second kernel clears the bit, so within the call
//   * no other key can claim it again (a claimed counter is never the
//     minimum, and every claim is an atomicCAS from the value observed),
//   * so every slot is written by at most one key: rows are never torn.
//   free slot  atomicOr of the slot's bit into the slab mask (the claimer
//              whose OR found the bit clear owns the mask bit; a loser
//              retries on the mask the OR returned, so masks still fill
//              from bit 0), then atomicCAS(counter, observed, stamp|claim)
//              -- an evictor that saw the slab full may have taken it first
//   eviction   argmin over the set's unclaimed counters, won by
//              atomicCAS(counter, min, stamp|claim); a lost CAS updates the
//              one observed counter (it only ever grows: a refresh raises it
//              to the stamp, a claim sets the bit) and retries
//   refresh    atomicMax(counter, stamp) (keeps a concurrent claim's bit)
// Keys of one call therefore never evict each other: a key whose set has no
// unclaimed slot left is not admitted (counted in *dropped), where the exact
// mode would evict a key this call inserted. Keys must be DISTINCT. Slots,
// and which keys of an over-subscribed set survive, can differ from the
// exact mode; invariants and every stored row's bytes are the same.
constexpr unsigned long long kClaimBit = 1ull << 63;

#ifndef HPSB_RELAX_MINB
#define HPSB_RELAX_MINB 5
#endif

// A key is applied by a GROUP of G lanes (G = 32 / keys per warp): lane l
// of the group holds slots l, l + G, ... of each slab (SPL = 32 / G slots
// per slab per lane); every collective op is masked to the group, so the
// groups of a warp proceed independently (2 keys in flight per warp at
// G = 16 -- the kernel is bound by its dependent round trips, not by issue).
template <int W, int G>
__global__ void __launch_bounds__(256, W <= 2 ? HPSB_RELAX_MINB : 4)
    k_replace_relaxed(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                      const float* __restrict__ rows, uint64_t stamp,
                      uint64_t* __restrict__ claimed, unsigned long long* __restrict__ dropped) {
  constexpr int SPL = 32 / G;
  constexpr uint32_t kGroupBits = G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u);
  constexpr int RV = (32 + G - 1) / G;  // float4 of a <= 128-float row per lane
  __shared__ unsigned long long s_ins, s_drop;
  if (threadIdx.x == 0) {
    s_ins = 0ull;
    s_drop = 0ull;
  }
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint32_t l = lane % G;             // lane within the group
  const uint32_t gb = lane - l;            // the group's first lane
  const uint32_t gm = kGroupBits << gb;    // the group's lanes
  const uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  unsigned long long* const ctr = reinterpret_cast<unsigned long long*>(c.counters);
  const unsigned long long mine = stamp | kClaimBit;
  if (i < n) {
    const uint32_t d = c.d;
    const uint64_t key = keys[i];
    const float* src = rows + i * d;
    const bool vec = (d & 3u) == 0 && d <= 128 && (reinterpret_cast<uintptr_t>(src) & 15u) == 0;
    float4 rv[RV];
#pragma unroll
    for (int r = 0; r < RV; ++r) {
      const uint32_t q = uint32_t(r) * G + l;
      rv[r] = (vec && q < (d >> 2)) ? reinterpret_cast<const float4*>(src)[q]
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const uint64_t set = slabset_of(c, key);
    const uint64_t h2 = xxh64_key(key, kSlabSeed);
    const uint32_t first = W == 1 ? 0u : (W == 2 ? uint32_t(h2 & 1u) : uint32_t(fastmod(h2, W, c.mW)));
    const uint64_t sbase = set * W;
    uint32_t m[W];
    uint64_t k[W][SPL], ct[W][SPL];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      m[w] = c.masks[sbase + w];
#pragma unroll
      for (int r = 0; r < SPL; ++r) {
        k[w][r] = c.keys[(sbase + w) * kSlotsPerSlab + r * G + l];
        ct[w][r] = c.counters[(sbase + w) * kSlotsPerSlab + r * G + l];
      }
    }
    // probe in slab order from `first` (slab_cache.cpp:292-310)
    int hit_w = -1, ins_step = -1;
    uint32_t hit_j = 0;
#pragma unroll
    for (int step = 0; step < W; ++step) {
      int w = int(first) + step;
      if (w >= W) w -= W;
      if (hit_w >= 0 || ins_step >= 0) continue;
      uint32_t mw = 0;
#pragma unroll
      for (int x = 0; x < W; ++x)
        if (x == w) mw = m[x];
      uint32_t hb = 0;
#pragma unroll
      for (int r = 0; r < SPL; ++r) {
        uint64_t kw = 0;
#pragma unroll
        for (int x = 0; x < W; ++x)
          if (x == w) kw = k[x][r];
        const uint32_t b = __ballot_sync(gm, ((mw >> (r * G + l)) & 1u) && kw == key);
        hb |= ((b >> gb) & kGroupBits) << (r * G);
      }
      if (hb) {
        hit_w = w;
        hit_j = __ffs(hb) - 1;
      } else if (mw != kFullSlab) {
        ins_step = step;
      }
    }
    uint64_t slot = ~0ull;
    if (hit_w >= 0) {
      // resident: recency refresh only, the vector is kept (:283-288)
      if (l == 0) atomicMax(ctr + (sbase + hit_w) * kSlotsPerSlab + hit_j, (unsigned long long)stamp);
    } else {
      int tw = -1;
      uint32_t tj = 0;
      // free slots: the probed slabs from the first non-full one, in order
      if (ins_step >= 0) {
#pragma unroll
        for (int step = 0; step < W; ++step) {
          if (step < ins_step || tw >= 0) continue;
          int w = int(first) + step;
          if (w >= W) w -= W;
          uint32_t mw = 0;
#pragma unroll
          for (int x = 0; x < W; ++x)
            if (x == w) mw = m[x];
          // terminates: every lost OR returns a mask with more bits set
          while (mw != kFullSlab) {
            const uint32_t j = __ffs(~mw) - 1;  // countr_one(mask) (:299)
            uint64_t cv = 0;
#pragma unroll
            for (int x = 0; x < W; ++x)
#pragma unroll
              for (int r = 0; r < SPL; ++r)
                if (x == w && uint32_t(r) == j / G) cv = ct[x][r];
            const uint64_t cj = __shfl_sync(gm, cv, gb + j % G);
            uint32_t old = 0, won = 0;
            if (l == 0) {
              old = atomicOr(c.masks + sbase + w, 1u << j);
              if (((old >> j) & 1u) == 0u) {
                // occupied from here on, by this key or by an evictor's
                atomicAdd(&s_ins, 1ull);
                won = atomicCAS(ctr + (sbase + w) * kSlotsPerSlab + j, (unsigned long long)cj,
                                mine) == cj ? 1u : 0u;
              }
            }
            old = __shfl_sync(gm, old, gb);
            won = __shfl_sync(gm, won, gb);
            if (won) {
              tw = w;
              tj = j;
              break;
            }
            mw = old | (1u << j);
          }
#pragma unroll
          for (int x = 0; x < W; ++x)
            if (x == w) m[x] = mw;
        }
      }
      // eviction: argmin over the set's unclaimed counters; terminates --
      // a lost CAS shows a strictly larger value (at most two raises a slot)
      for (uint32_t tries = 0; tw < 0 && tries <= 2u * uint32_t(W) * 32u; ++tries) {
        uint64_t bc = ~0ull;
        uint32_t bi = 0xFFFFFFFFu;
#pragma unroll
        for (int x = 0; x < W; ++x)
#pragma unroll
          for (int r = 0; r < SPL; ++r)
            if ((ct[x][r] & kClaimBit) == 0ull && ct[x][r] < bc) {
              bc = ct[x][r];
              bi = uint32_t(x) * 32 + uint32_t(r) * G + l;
            }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
          const uint64_t oc = __shfl_xor_sync(gm, bc, o);
          const uint32_t oi = __shfl_xor_sync(gm, bi, o);
          if (oc < bc || (oc == bc && oi < bi)) {
            bc = oc;
            bi = oi;
          }
        }
        if (bi == 0xFFFFFFFFu) break;  // every slot of the set claimed by this call
        const uint32_t bw = bi >> 5, bj = bi & 31u;
        unsigned long long old = 0;
        if (l == 0) old = atomicCAS(ctr + (sbase + bw) * kSlotsPerSlab + bj, (unsigned long long)bc, mine);
        old = __shfl_sync(gm, old, gb);
        if (old == bc) {
          tw = int(bw);
          tj = bj;
        } else if (l == bj % G) {
#pragma unroll
          for (int x = 0; x < W; ++x)
#pragma unroll
            for (int r = 0; r < SPL; ++r)
              if (uint32_t(x) == bw && uint32_t(r) == bj / G) ct[x][r] = old;
        }
      }
      if (tw >= 0) {
        slot = (sbase + uint64_t(tw)) * kSlotsPerSlab + tj;
        if (l == 0) {
          c.keys[slot] = key;
          c.tags[slot] = key_tag(h2);
        }
        float* dst = c.rows + slot * d;
        if (vec) {
#pragma unroll
          for (int r = 0; r < RV; ++r) {
            const uint32_t q = uint32_t(r) * G + l;
            if (q < (d >> 2)) reinterpret_cast<float4*>(dst)[q] = rv[r];
          }
        } else {
          for (uint32_t x = l; x < d; x += G) dst[x] = src[x];
        }
      } else if (l == 0) {
        atomicAdd(&s_drop, 1ull);
      }
    }
    if (l == 0) claimed[i] = slot;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_ins) atomicAdd(c.occupied, s_ins);
    if (s_drop && dropped != nullptr) atomicAdd(dropped, s_drop);
  }
}

// The call's claims become plain counters (= the stamp).
__global__ void __launch_bounds__(256)
    k_replace_relaxed_release(CacheDev c, const uint64_t* __restrict__ claimed, uint64_t n,
                              uint64_t stamp) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t slot = claimed[i];
  if (slot != ~0ull) c.counters[slot] = stamp;
}

bool launch_replace_relaxed(const CacheDev& c, const uint64_t* keys, uint64_t n, const float* rows,
                            uint64_t stamp, uint64_t* claimed, unsigned long long* dropped,
                            cudaStream_t st) {
  if (n == 0) return true;
  if (c.W == 0 || c.W > 4) return false;  // wider sets: the exact path
#ifndef HPSB_RELAX_G
#define HPSB_RELAX_G 16
#endif
  // lanes per key: HPSB_RELAX_G for W <= 2, a whole warp for wider sets
  constexpr int G2 = HPSB_RELAX_G;
  const unsigned g12 = unsigned((n * G2 + 255) / 256), g34 = unsigned((n * 32 + 255) / 256);
  switch (c.W) {
    case 1: k_replace_relaxed<1, G2><<<g12, 256, 0, st>>>(c, keys, n, rows, stamp, claimed, dropped); break;
    case 2: k_replace_relaxed<2, G2><<<g12, 256, 0, st>>>(c, keys, n, rows, stamp, claimed, dropped); break;
    case 3: k_replace_relaxed<3, 32><<<g34, 256, 0, st>>>(c, keys, n, rows, stamp, claimed, dropped); break;
    default: k_replace_relaxed<4, 32><<<g34, 256, 0, st>>>(c, keys, n, rows, stamp, claimed, dropped); break;
  }
  k_replace_relaxed_release<<<unsigned((n + 255) / 256), 256, 0, st>>>(c, claimed, n, stamp);
  check_launch("replace_relaxed", 2);
  return true;
}

void launch_replace(const CacheDev& c, const uint64_t* keys, uint64_t n, const float* rows,
                    uint64_t stamp, bool validate, const ReplaceScratch& rs, cudaStream_t st,
                    int device) {
  if (n == 0) return;
  static const bool no_small = std::getenv("HPSB_REPLACE_NO_SMALL") != nullptr;
  if (n <= kSmallReplaceMax && !no_small && !validate) {
    k_replace_tiny<<<unsigned((n + 7) / 8), 256, 0, st>>>(c, keys, uint32_t(n), rows, stamp, rs);
    check_launch("replace", 1);
    return;
  }
  if (n <= kSmallReplaceMax && !no_small) {
    k_replace_small<<<1, kSmallReplace, 0, st>>>(c, keys, uint32_t(n), rows, stamp,
                                                 validate ? 1u : 0u, rs);
    check_launch("replace", 1);
    return;
  }
  const unsigned tb = 256;
  k_replace_bin<<<unsigned((n + tb - 1) / tb), tb, 0, st>>>(c, keys, n, rs);
  const unsigned wgrid = unsigned((n * 32 + tb - 1) / tb);
  if (validate) k_replace_dups<<<wgrid, tb, 0, st>>>(keys, n, rs);
  // persistent set kernel: as many blocks as fit on the device at once
  // (fewer when the call touches fewer sets than that many warps)
  auto grid_for = [&](const void* fn) {
    static int sms = 0, per_sm[5] = {0, 0, 0, 0, 0};
    const int wi = c.W <= 4 ? int(c.W) : 0;
    if (sms == 0) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (per_sm[wi] == 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[wi], fn, tb, 0);
    const uint64_t full = uint64_t(std::max(sms, 1)) * uint64_t(std::max(per_sm[wi], 1));
    return unsigned(std::min<uint64_t>(full, wgrid));
  };
  // the set kernel as a programmatic dependent of the kernel before it (bin,
  // or the duplicate check): its launch and prologue overlap that tail
  static const bool no_pdl = std::getenv("HPSB_NO_PDL") != nullptr;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(tb);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  const uint32_t vflag = validate ? 1u : 0u;
  auto sets = [&](auto kern) {
    cfg.gridDim = dim3(grid_for((const void*)kern));
    cudaLaunchKernelEx(&cfg, kern, c, keys, n, rows, stamp, vflag, rs);
  };
  switch (c.W) {
    case 1: sets(k_replace_sets<1>); break;
    case 2: sets(k_replace_sets<2>); break;
    case 3: sets(k_replace_sets<3>); break;
    case 4: sets(k_replace_sets<4>); break;
    default: sets(k_replace_sets<0>); break;
  }
  check_launch("replace", validate ? 3 : 2);
}

// ----------------------------------------------------------------- update --
// Overwrite resident rows; the last occurrence of a key in input order wins
// (the reference applies a set's keys in input order, slab_cache.cpp:137-142,
// 328-358), counters untouched, nothing admitted.
//   k_update_probe  lane per position: fingerprint probe (tag_probe.cuh);
//                   slot recorded; max(position + 1) per hit slot into the
//                   cache's `winner` array (fire-and-forget); hits counted
//   k_update_write  warp per 8 positions: the winning position of each
//                   slot copies its row (256-bit loads from the contiguous
//                   input block, write-back stores into the table; a d = 128
//                   warp moves its 4 KB in ONE round trip, every row of the
//                   call in flight at once) and clears the winner entry (the
//                   array is all-zero between calls)
// Consecutive updates alternate between two winner arrays and two scratch
// halves (DeviceCache): the next update's probe may run while this write is
// still in flight (it launches behind the next lookup, which launches when
// this write starts).
__global__ void __launch_bounds__(256)
    k_update_probe(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                   uint32_t* __restrict__ slot_of, uint32_t* __restrict__ winner,
                   uint32_t* __restrict__ block_hits, uint32_t wait_at_end) {
  const uint64_t pos = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool valid = pos < n;
  const uint64_t key = valid ? keys[pos] : 0ull;
  const uint32_t res = lane_probe(c, key, valid);
  if (valid) slot_of[pos] = res;
  if (res != kNoSlot) atomicMax(winner + res, uint32_t(pos + 1));
  // per-block hit count (no zeroed counter needed: every block writes its own)
  __shared__ uint32_t s_hits;
  if (threadIdx.x == 0) s_hits = 0;
  __syncthreads();
  const uint32_t hits = __reduce_add_sync(0xFFFFFFFFu, res != kNoSlot ? 1u : 0u);
  if (lane_id() == 0 && hits) atomicAdd(&s_hits, hits);
  __syncthreads();
  if (threadIdx.x == 0) block_hits[blockIdx.x] = s_hits;
  // Launched as the programmatic dependent of a lookup (it only reads the
  // probe structures, which lookups do not change): complete only after that
  // lookup, so the row writes that follow never race its row reads.
  if (wait_at_end) asm volatile("griddepcontrol.wait;" ::: "memory");
}

constexpr uint32_t kUpdateRowsPerWarp = 8;

template <int CH>
__global__ void __launch_bounds__(256)
    k_update_write(CacheDev c, const float* __restrict__ rows, uint64_t n,
                   const uint32_t* __restrict__ slot_of, uint32_t* __restrict__ winner,
                   const uint32_t* __restrict__ block_hits, uint32_t probe_blocks,
                   unsigned long long* __restrict__ written) {
  // the next lookup may launch now (it waits for this grid before its copies)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr uint32_t R = kUpdateRowsPerWarp;
  constexpr int U = CH == 8 ? 4 : 8;
  const uint32_t lane = lane_id();
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    unsigned long long h = 0;
    for (uint32_t b = threadIdx.x; b < probe_blocks; b += 32) h += block_hits[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, o);
    if (threadIdx.x == 0) *written = h;
  }
  const uint64_t base = ((uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * R;
  const uint64_t pos = base + lane;
  uint32_t slot = kNoSlot;
  if (lane < R && pos < n) {
    slot = slot_of[pos];
    if (slot != kNoSlot && __ldcg(winner + slot) != uint32_t(pos + 1)) slot = kNoSlot;  // a later duplicate wins
  }
  const uint32_t nrows = n > base + R ? R : uint32_t(n > base ? n - base : 0);
  const uint32_t d = c.d;
  const uint32_t cpr = d / CH;
  const bool pow2 = (cpr & (cpr - 1)) == 0;
  const uint32_t sh = __ffs(cpr) - 1;
  const uint32_t total = nrows * cpr;
  const float* src = rows + base * d;
  for (uint32_t c0 = 0; c0 < total; c0 += 32 * U) {
    Chunk<CH> x[U];
    uint32_t dst_slot[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t ch = c0 + uint32_t(u) * 32 + lane;
      uint32_t row = pow2 ? (ch >> sh) : (ch / cpr);
      row = min(row, R - 1);
      dst_slot[u] = __shfl_sync(0xFFFFFFFFu, slot, row);
      if (ch < total && dst_slot[u] != kNoSlot) x[u].load(src + uint64_t(ch) * CH);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t ch = c0 + uint32_t(u) * 32 + lane;
      if (ch < total && dst_slot[u] != kNoSlot) {
        const uint32_t row = pow2 ? (ch >> sh) : (ch / cpr);
        x[u].store_wb(c.rows + uint64_t(dst_slot[u]) * d + (ch - row * cpr) * CH);
      }
    }
  }
  if (slot != kNoSlot) winner[slot] = 0u;
}

size_t update_scratch_bytes(uint64_t n) { return (n * 4 + 255) / 256 * 256 + ((n + 255) / 256) * 4; }

void launch_update(const CacheDev& c, const uint64_t* keys, uint64_t n, const float* rows,
                   void* scratch, uint32_t* winner, unsigned long long* written,
                   bool after_lookup, cudaStream_t st) {
  if (n == 0) {
    cudaMemsetAsync(written, 0, 8, st);
    check_launch("update", 0);
    return;
  }
  uint32_t* slot_of = static_cast<uint32_t*>(scratch);
  uint32_t* block_hits = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) +
                                                     (n * 4 + 255) / 256 * 256);
  const unsigned grid = unsigned((n + 255) / 256);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = after_lookup ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k_update_probe, c, keys, n, slot_of, winner, block_hits,
                     uint32_t(after_lookup ? 1 : 0));
  const bool a32 = (reinterpret_cast<uintptr_t>(rows) % 32) == 0;
  const bool a16 = (reinterpret_cast<uintptr_t>(rows) % 16) == 0;
  const unsigned wgrid = unsigned((n + 8 * kUpdateRowsPerWarp - 1) / (8 * kUpdateRowsPerWarp));
  if (c.d % 8 == 0 && a32)
    k_update_write<8><<<wgrid, 256, 0, st>>>(c, rows, n, slot_of, winner, block_hits, grid, written);
  else if (c.d % 4 == 0 && a16)
    k_update_write<4><<<wgrid, 256, 0, st>>>(c, rows, n, slot_of, winner, block_hits, grid, written);
  else
    k_update_write<1><<<wgrid, 256, 0, st>>>(c, rows, n, slot_of, winner, block_hits, grid, written);
  check_launch("update", 2);
}

// ------------------------------------------------------------------- dump --
// Resident keys of slabs [set_begin*W, set_end*W) in slab order, slot order
// inside a slab (slab_cache.cpp:380-392). A tile = kDumpTile slabs, one per
// thread: (1) a block scan of the masks' popcounts plus a decoupled
// look-back give every slab its output offset; (2) each warp copies its 32
// slabs' keys -- occupancy grows contiguously from bit 0, so lane j of an
// occupied slab writes out[offset + j]: coalesced 256 B loads and contiguous
// stores, 8 slabs in flight per warp. (Tiles of 1,024 slabs -- 61 blocks at
// cfg 2 -- left the copy latency-bound: 26 us for 2 M slots.)
__global__ void __launch_bounds__(kScanBlock)
    k_dump_keys(CacheDev c, uint64_t slab_begin, uint64_t n_slabs, uint64_t* __restrict__ out,
                unsigned long long* n_out, ScanState scan) {
  static_assert(kDumpTile == kScanBlock, "one slab per thread");
  __shared__ uint32_t s_warp[kScanBlock / 32];
  __shared__ uint64_t s_tile;
  __shared__ uint64_t s_prefix;
  if (threadIdx.x == 0) s_tile = atomicAdd(scan.tile_ctr, 1ull) - scan.tile_base;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t first = tile * kDumpTile;
  const uint64_t sl = first + threadIdx.x;
  const uint32_t m = (sl < n_slabs) ? c.masks[slab_begin + sl] : 0u;
  const uint32_t cnt = __popc(m);
  uint32_t block_total;
  const uint32_t excl = block_exclusive_scan<kScanBlock>(cnt, s_warp, &block_total);
  if (threadIdx.x < 32) {
    const uint64_t pre = lb_exclusive_prefix(scan.status, uint32_t(tile), scan.epoch, block_total);
    if (threadIdx.x == 0) {
      s_prefix = pre;
      const uint64_t tiles = (n_slabs + kDumpTile - 1) / kDumpTile;
      if (tile == tiles - 1) *n_out = pre + block_total;
    }
  }
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint64_t prefix = s_prefix;
  // this warp's 32 slabs: slab (warp base + i) held by lane i (count, offset)
  const uint64_t wslab = first + (threadIdx.x & ~31u);
  const uint64_t* kbase = c.keys + (slab_begin + wslab) * kSlotsPerSlab;
#pragma unroll
  for (int i0 = 0; i0 < 32; i0 += 8) {
    uint64_t k[8];
    uint32_t ci[8], oi[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      ci[u] = __shfl_sync(0xFFFFFFFFu, cnt, i0 + u);
      oi[u] = __shfl_sync(0xFFFFFFFFu, excl, i0 + u);
      k[u] = lane < ci[u] ? kbase[uint64_t(i0 + u) * kSlotsPerSlab + lane] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (lane < ci[u]) out[prefix + oi[u] + lane] = k[u];
  }
}

void launch_dump(const CacheDev& c, uint64_t set_begin, uint64_t set_end, uint64_t* out,
                 unsigned long long* n_out, ScanState& scan, cudaStream_t st) {
  const uint64_t n_slabs = (set_end - set_begin) * c.W;
  if (n_slabs == 0) {
    cudaMemsetAsync(n_out, 0, 8, st);
    return;
  }
  const uint64_t tiles = (n_slabs + kDumpTile - 1) / kDumpTile;
  scan_begin(scan, tiles, st);
  k_dump_keys<<<unsigned(tiles), kScanBlock, 0, st>>>(c, set_begin * c.W, n_slabs, out, n_out,
                                                      scan);
  scan.tile_base += tiles;
  check_launch("dump", 1);
}

// ------------------------------------------------------------------ dedup --
__global__ void k_dedup_insert(const uint64_t* __restrict__ keys, uint64_t n, DedupScratch ds,
                               uint32_t epoch) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool claimed;
  ds.slot_of[i] = dedup_insert(ds.table, ds.cap, keys, keys[i], uint32_t(i), epoch, &claimed);
}

__global__ void __launch_bounds__(kScanBlock)
    k_dedup_compact(const uint64_t* __restrict__ keys, uint64_t n, DedupScratch ds,
                    uint64_t* __restrict__ unique_out, ScanState scan) {
  select_tile(
      n, scan, [&](uint64_t i) { return uint32_t(ds.table[ds.slot_of[i]]) == uint32_t(i); },
      [&](uint64_t i, uint64_t r) {
        unique_out[r] = keys[i];
        ds.rank_of_slot[ds.slot_of[i]] = uint32_t(r);
      },
      ds.n_unique);
}

__global__ void k_dedup_inverse(uint64_t n, DedupScratch ds, uint32_t* __restrict__ inverse) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  inverse[i] = ds.rank_of_slot[ds.slot_of[i]];
}

void launch_dedup(const uint64_t* keys, uint64_t n, uint64_t* unique_out, uint32_t* inverse,
                  const DedupScratch& ds, uint32_t table_epoch, ScanState& scan,
                  cudaStream_t st) {
  if (n == 0) {
    cudaMemsetAsync(ds.n_unique, 0, 8, st);
    return;
  }
  const unsigned tb = 256;
  k_dedup_insert<<<unsigned((n + tb - 1) / tb), tb, 0, st>>>(keys, n, ds, table_epoch);
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  scan_begin(scan, tiles, st);
  k_dedup_compact<<<unsigned(tiles), kScanBlock, 0, st>>>(keys, n, ds, unique_out, scan);
  scan.tile_base += tiles;
  k_dedup_inverse<<<unsigned((n + tb - 1) / tb), tb, 0, st>>>(n, ds, inverse);
  check_launch("dedup", 3);
}

}  // namespace hpsb
