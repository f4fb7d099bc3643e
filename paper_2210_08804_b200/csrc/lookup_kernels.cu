// lookup_kernels.cu -- the lookup hot path (sm_100a).
//
// Restates LookupEngine::lookup's device half (lookup_engine.cpp:130-241:
// dedup -> query -> unique-key counts -> expansion, with the default row for
// missing positions, :185-203) for a batch of |Q| query positions, in ONE
// kernel launch per call:
//
//   k_lookup_tag  (default) lane i of a warp owns position base+i:
//       A  key (coalesced), both placement hashes (XXH64 + Barrett modulo),
//          the set's 8-bit fingerprints and occupancy masks (W = 2: 64 B in
//          two 256-bit loads + one 8 B load, one round trip), candidate
//          keys verified in slot order (the first equal key is the
//          reference's lowest-matching-slot hit, slab_cache.cpp:240-245; the
//          second slab only counts when the first is full, :249-256);
//          missing keys claimed in a per-call miss table (minimum position
//          kept), one attempt per warp-distinct key; miss flags
//       B  griddepcontrol.wait: when launched as a programmatic dependent of
//          the previous lookup on the stream, everything above overlapped
//          that lookup's row traffic; from here on the previous call is
//          complete (its stamps landed, its last block finished)
//       C  recency exchange (one per distinct slot per block; the exchange
//          that moves a slot to this call's stamp counts one UNIQUE hit, so
//          |Q*| needs no dedup of hits), row copy of the warp's 32 rows as
//          one contiguous output block with 256-bit L1-allocating loads and
//          evict-first stores, per-warp counts
//       D  the last block to finish completes the call: first position of
//          every claim (sorting claims by it gives the reference's miss
//          order -- dedup first-occurrence, types.cpp:20-34, then ascending
//          miss positions, slab_cache.cpp:84-89), miss table cleared,
//          per-call counts, per-call state reset for the call after next
//   k_lookup<L>   the warp-cooperative variant (L lanes per position probe a
//          slab's 32 keys with 128-bit loads and a min/ballot rule), kept
//          for A/B measurement (HPSB_LOOKUP_KERNEL=warp4|warp8)
//   k_lookup_scatter (sync branch only) copies the rows fetched from the
//          tiers into every position of their key and clears the default
//          flag (lookup_engine.cpp:165-181).
//
// Consecutive lookups on one stream alternate between the two halves
// (parities) of a LookupScratch, so call i+1's phase A may run while call i
// is still copying rows: nothing in phase A reads state that call i writes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <type_traits>

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
inline uint64_t a256(uint64_t v) { return (v + 255) / 256 * 256; }
inline uint64_t table_cap(uint64_t cap) {
  uint64_t t = 16;
  while (t < 2 * cap) t <<= 1;
  return t;
}
constexpr int kWarps = 8;  // warp variant: 256-thread blocks
constexpr int kThreads = kWarps * 32;
constexpr int kSetBits = 7;           // warp variant: 128-entry per-block stamped-slot set
constexpr uint32_t kCountLanes = 64;  // distributed (unique hit, unique miss) counter pairs

// Diagnostic skip bits (HPSB_DIAG_SKIP, measurement only; results are wrong
// with any bit set): 1 = recency exchange, 2 = miss claims, 4 = row copy.
constexpr uint32_t kSkipStamp = 1, kSkipMiss = 2, kSkipCopy = 4;
// not a diagnostic: set by the launcher when the lookup follows an update
constexpr uint32_t kWaitBeforeCopy = 1u << 8;

uint64_t view_bytes(uint64_t cap) {
  const uint64_t tcap = table_cap(cap);
  return a256(tcap * 4) * 2 + a256(cap * 4) * 3 + a256(cap * 8) + a256(kCountLanes * 16) +
         a256(64);
}
}  // namespace

size_t lookup_scratch_bytes(uint64_t cap, int nviews) {
  return uint64_t(nviews) * (view_bytes(cap) + a256(table_cap(cap) * 8));
}

LookupView lookup_next_view(LookupScratch& ls, bool chain) {
  const int i = ls.next;
  LookupView v = ls.v[i];
  v.gen = ls.uses[i]++;
  v.idx = uint32_t(i);
  if (chain && ls.last >= 0) {
    v.prev_completed = ls.v[ls.last].completed;
    v.prev_target = ls.uses[ls.last];  // that call's gen + 1
    v.prev_idx = uint32_t(ls.last);
  }
  ls.last = i;
  ls.next = (i + 1) % ls.nviews;
  return v;
}

LookupScratch lookup_scratch_carve(void* base, uint64_t cap, int nviews) {
  LookupScratch ls;
  ls.nviews = nviews;
  const uint64_t tcap = table_cap(cap);
  char* p = static_cast<char*>(base);
  auto take = [&](uint64_t b) {
    char* r = p;
    p += a256(b);
    return r;
  };
  uint32_t lg = 0;
  while ((1ull << lg) < tcap) ++lg;
  // every view's hit table first, contiguous
  ls.hits_base = p;
  ls.hits_bytes = uint64_t(nviews) * a256(tcap * 8);
  for (int k = 0; k < nviews; ++k) {
    ls.v[k].hits = reinterpret_cast<unsigned long long*>(take(tcap * 8));
    ls.v[k].log2cap = lg;
  }
  for (int k = 0; k < nviews; ++k) {
    LookupView& v = ls.v[k];
    v.cap = tcap;
    v.miss_table = reinterpret_cast<uint32_t*>(take(tcap * 4));
    v.claim_of_slot = reinterpret_cast<uint32_t*>(take(tcap * 4));
    v.miss_slot = reinterpret_cast<uint32_t*>(take(cap * 4));
    v.list = reinterpret_cast<uint32_t*>(take(cap * 4));
    v.list_firsts = reinterpret_cast<uint32_t*>(take(cap * 4));
    v.list_keys = reinterpret_cast<uint64_t*>(take(cap * 8));
    v.counts = reinterpret_cast<unsigned long long*>(take(kCountLanes * 16));
    unsigned long long* small = reinterpret_cast<unsigned long long*>(take(64));
    v.counts_out = small;                                 // [0..1] default destination
    v.list_ctr = reinterpret_cast<uint32_t*>(small + 2);  // claim counter
    v.done = reinterpret_cast<uint32_t*>(small + 3);      // [2] block tickets
    v.completed = small + 4;
  }
  return ls;
}

// ------------------------------------------------------------ accessors --
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Trace fields: 0 first block start, 1 last block done with A, 2 last
// block start, 3 first block done with A, 4 first block done
// copying, 5 last block done copying, 6 claims finish start, 7 claims
// finish end.
__device__ __forceinline__ void trace_min(const LookupView& v, int f, bool as_max) {
  if (v.trace != nullptr && threadIdx.x == 0) {
    const unsigned long long t = global_ns();
    atomicMin(v.trace + f, as_max ? ~t : t);
  }
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Block ticket arrival: a release (this block's writes -- ordered before it
// by the preceding barrier -- are visible to whoever sees the count) without
// the acquire half, which on sm_100 invalidates the SM's whole L1 (CCTL.IVALL)
// and with it the hot rows every resident block is reading.
__device__ __forceinline__ uint32_t atom_add_release(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Spins (one thread) until *p >= target. Calls on one stream only ever wait
// on calls launched before them, whose blocks have all started, so this
// cannot deadlock -- unless captured graphs are replayed out of capture
// order; a wait longer than 2 s traps (the launch fails) instead of hanging.
__device__ __forceinline__ void spin_ge(const unsigned long long* p, unsigned long long target) {
  if (ld_acquire(p) >= target) return;
  const unsigned long long t0 = global_ns();
  while (ld_acquire(p) < target) {
    __nanosleep(200);
    if (global_ns() - t0 > 2000000000ull) __trap();
  }
}
// The same wait at every block start of a lookup, with relaxed loads: a
// view's scratch is only ever accessed through L2 (atomics, .cg loads,
// stores), which already holds the previous use's writes when its release
// is observed, so the L1-invalidating acquire is not needed here.
__device__ __forceinline__ void spin_ge_relaxed(const unsigned long long* p,
                                                unsigned long long target) {
  if (ld_relaxed(p) >= target) return;
  const unsigned long long t0 = global_ns();
  while (ld_relaxed(p) < target) {
    __nanosleep(200);
    if (global_ns() - t0 > 2000000000ull) __trap();
  }
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------- call completion --
// A call completes in two parts, each run by the last block through a
// ticket (a release atomic per block, an acquire fence in the last one, so
// all earlier blocks' writes are visible):
//   finish_claims  once every block has made its claims (ticket taken before
//                  the row copies, run after the block's own copies): first
//                  position of each claim, miss table cleared
//   finish_counts  once every block has added its counts (after the copies):
//                  per-call counts, counters zeroed, tickets and claim
//                  counter reset for the next call on this view
// finish_claims is one block's work, written for memory-level parallelism:
// each thread issues all its loads of a round before using any.
__device__ void finish_claims(const LookupView& v) {
  constexpr int kClaimsPerThread = 8;
  const uint32_t m = __ldcg(v.list_ctr);
  for (uint32_t e0 = 0; e0 < m; e0 += kClaimsPerThread * blockDim.x) {
    uint32_t s[kClaimsPerThread], f[kClaimsPerThread];
#pragma unroll
    for (int k = 0; k < kClaimsPerThread; ++k) {
      const uint32_t e = e0 + k * blockDim.x + threadIdx.x;
      s[k] = e < m ? __ldcg(v.list + e) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kClaimsPerThread; ++k) {
      const uint32_t e = e0 + k * blockDim.x + threadIdx.x;
      f[k] = e < m ? __ldcg(v.miss_table + s[k]) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kClaimsPerThread; ++k) {
      const uint32_t e = e0 + k * blockDim.x + threadIdx.x;
      if (e < m) {
        v.list_firsts[e] = f[k] - 1u;
        v.miss_table[s[k]] = 0u;  // the table is all-zero between calls
      }
    }
  }
}

__device__ void finish_counts(const LookupView& v, unsigned long long gen,
                              unsigned long long prev_target) {
  if (threadIdx.x < 32) {
    // 128 values, 4 per lane, loaded together
    const uint32_t i = threadIdx.x & 1u;
    unsigned long long x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = __ldcg(v.counts + 2 * ((threadIdx.x >> 1) + 16 * k) + i);
    unsigned long long s = x[0] + x[1] + x[2] + x[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) v.counts[2 * ((threadIdx.x >> 1) + 16 * k) + i] = 0ull;
#pragma unroll
    for (int o = 16; o >= 2; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if (threadIdx.x < 2) v.counts_out[i] = s;
    if (threadIdx.x == 0) {
      *v.list_ctr = 0u;
      v.done[0] = 0u;
      v.done[1] = 0u;
      // completion order = launch order: this call completes after the
      // previous one, so stream work after it sees every earlier lookup done
      if (v.prev_completed != nullptr) spin_ge(v.prev_completed, prev_target);
      __threadfence();
      st_release(v.completed, gen + 1);  // the view is free for its next use
    }
  }
}

// Ticket `t` (0 = claims, 1 = counts): true in every thread of the block
// that got there last.
__device__ __forceinline__ bool last_block(const LookupView& v, int t, uint32_t nblocks) {
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    s_last = atom_add_release(v.done + t, 1u) == nblocks - 1 ? 1u : 0u;
    if (s_last) fence_acq_rel();  // acquire: every block's writes (one block per call)
  }
  __syncthreads();
  return s_last != 0;
}

// Adds a warp's (unique hit, unique miss) totals into one of kCountLanes
// counter pairs (no single hot counter).
__device__ __forceinline__ void warp_add_counts(const LookupView& v, uint32_t uh, uint32_t um,
                                                uint32_t warp_global) {
  uh = __reduce_add_sync(0xFFFFFFFFu, uh);
  um = __reduce_add_sync(0xFFFFFFFFu, um);
  if (lane_id() == 0 && (uh | um)) {
    const uint32_t w = warp_global & (kCountLanes - 1);
    if (uh) atomicAdd(v.counts + 2 * w, (unsigned long long)uh);
    if (um) atomicAdd(v.counts + 2 * w + 1, (unsigned long long)um);
  }
}

// Claims the missing keys of a warp (one lane per position; `miss` lanes):
// one miss-table attempt per warp-distinct key by its lowest position, the
// claim appended to the call's list; miss_slot recorded for the scatter
// kernel. Returns this lane's unique-miss contribution (0/1).
__device__ __forceinline__ uint32_t warp_claim_misses(const LookupView& v,
                                                      const uint64_t* __restrict__ keys,
                                                      uint64_t pos, uint64_t key, bool miss) {
  const uint32_t lane = lane_id();
  const uint32_t miss_lanes = __ballot_sync(0xFFFFFFFFu, miss);
  if (miss_lanes == 0) return 0;
  uint32_t key_leader = lane;
  bool claimed = false;
  uint32_t tslot = 0;
  if (miss) {
    key_leader = __ffs(__match_any_sync(miss_lanes, key)) - 1;
    if (key_leader == lane) tslot = miss_insert(v.miss_table, v.cap, keys, key, uint32_t(pos), &claimed);
  }
  // lanes of the same key share the table slot (the scatter kernel reads it)
  tslot = __shfl_sync(0xFFFFFFFFu, tslot, key_leader);
  if (miss) v.miss_slot[pos] = tslot;
  const uint32_t cm = __ballot_sync(0xFFFFFFFFu, claimed);
  if (cm) {
    const uint32_t first_lane = __ffs(cm) - 1;
    uint32_t at = 0;
    if (lane == first_lane) at = atomicAdd(v.list_ctr, uint32_t(__popc(cm)));
    at = __shfl_sync(0xFFFFFFFFu, at, first_lane);
    if (claimed) {
      const uint32_t e = at + __popc(cm & ((1u << lane) - 1u));
      v.list[e] = tslot;
      v.list_keys[e] = key;
      v.claim_of_slot[tslot] = e;
    }
  }
  return claimed ? 1u : 0u;
}

// Per-call sequence values: a lookup captured into a CUDA graph carries them
// relative to rebase words the library writes before every launch of the
// graph (DeviceCache capture sessions), so replays take fresh stamps and
// view generations in stream order.
struct CallSeq {
  unsigned long long stamp, gen, prev_target;
};
__device__ __forceinline__ CallSeq resolve_seq(const LookupView& v, uint64_t stamp) {
  CallSeq q{stamp, v.gen, v.prev_target};
  if (v.rebase != nullptr) {
    q.stamp += __ldg(v.rebase);
    q.gen += __ldg(v.rebase + 1 + v.idx);
    q.prev_target += __ldg(v.rebase + 1 + v.prev_idx);
  }
  return q;
}
// The pieces separately, where the multi-block kernels need them (each
// re-derived at its point of use instead of held in registers across the
// probe: the pipelined kernel runs at a 40-register cap).
__device__ __forceinline__ unsigned long long call_stamp(const LookupView& v, uint64_t stamp) {
  return v.rebase != nullptr ? stamp + __ldg(v.rebase) : stamp;
}
__device__ __forceinline__ unsigned long long call_gen(const LookupView& v) {
  return v.rebase != nullptr ? v.gen + __ldg(v.rebase + 1 + v.idx) : v.gen;
}
__device__ __forceinline__ unsigned long long call_prev_target(const LookupView& v) {
  return v.rebase != nullptr ? v.prev_target + __ldg(v.rebase + 1 + v.prev_idx) : v.prev_target;
}

// Home entry of `slot` in the call's hit table.
__device__ __forceinline__ uint64_t hit_home(const LookupView& v, uint32_t slot) {
  return (uint64_t(slot) * 0x9E3779B97F4A7C15ull) >> (64 - v.log2cap);
}
// Inserts `slot` into the call's distinct-hit table, starting at entry h whose
// current value `cur` the caller has already loaded (issued early, so the
// round trip overlaps other work). Entries tagged with another stamp are free.
// Returns 1 when this call inserted the slot (one unique hit), else 0.
__device__ __forceinline__ uint32_t hit_insert(const LookupView& v, uint32_t slot, uint32_t tag,
                                               uint64_t h, unsigned long long cur) {
  const unsigned long long mine = (uint64_t(tag) << 32) | slot;
  const uint64_t mask = v.cap - 1;
  for (uint64_t probes = 0; probes <= mask;) {
    if (uint32_t(cur >> 32) == tag) {
      if (uint32_t(cur) == slot) return 0u;
      h = (h + 1) & mask;
      ++probes;
      cur = __ldcg(v.hits + h);
      continue;
    }
    const unsigned long long old = atomicCAS(v.hits + h, cur, mine);
    if (old == cur) return 1u;
    cur = old;
  }
  return 0u;
}

// Recency exchange of a hit slot: the call's stamp becomes the slot's
// counter (max: calls may overlap, a later call's stamp wins), and inserting
// the slot into the call's hit table tells whether this is the call's first
// hit of the slot (one unique hit). Both are read first and only written
// when not already done: a power-law batch's hot slot is hit by every block
// of the call, and same-line read-modify-writes serialise in its L2 slice
// (reading first: 10.27 vs 11.25 us per cfg-2 batch).
__device__ __forceinline__ uint32_t stamp_slot(const CacheDev& c, const LookupView& v,
                                               uint32_t slot, unsigned long long stamp) {
  unsigned long long* ctr = reinterpret_cast<unsigned long long*>(c.counters) + slot;
  const unsigned long long cur_ctr = __ldcg(ctr);
  const uint64_t h = hit_home(v, slot);
  const unsigned long long cur = __ldcg(v.hits + h);
  if (cur_ctr < stamp) atomicMax(ctr, stamp);
  return hit_insert(v, slot, uint32_t(stamp), h, cur);  // low 32 bits never 0
}

// Inserts `slot` into a block-shared open-addressing set; false when the
// block already holds it (another warp of the block exchanged it).
__device__ __forceinline__ bool block_set_insert(uint32_t* set, uint32_t size_pow2, uint32_t slot) {
  uint32_t h = (slot * 0x9E3779B1u) >> 7;
  for (int probe = 0; probe < 32; ++probe) {
    h &= size_pow2 - 1;
    const uint32_t cur = atomicCAS(&set[h], kNoSlot, slot);
    if (cur == kNoSlot) return true;
    if (cur == slot) return false;
    ++h;
  }
  return true;  // set crowded: fall back to the global exchange
}

// ============================================== warp-cooperative variant --
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
    const ulonglong2 x = p2[j];
    kk[2 * j] = x.x;
    kk[2 * j + 1] = x.y;
  }
}

// L = lanes per position (4 or 8): a warp serves 32/L positions.
template <int L>
__global__ void __launch_bounds__(kThreads)
    k_lookup(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n, float* __restrict__ out,
             uint8_t* __restrict__ flags, const float* __restrict__ default_row, uint64_t stamp,
             LookupView v) {
  constexpr int K = 32 / L;    // keys of a slab per lane
  constexpr int POS = 32 / L;  // positions per warp
  constexpr int RC = 32 / L;   // float4 chunks per lane per 128-float row segment
  __shared__ uint32_t s_stamped[1u << kSetBits];
  for (uint32_t i = threadIdx.x; i < (1u << kSetBits); i += kThreads) s_stamped[i] = kNoSlot;
  const CallSeq seq = resolve_seq(v, stamp);
  stamp = seq.stamp;
  if (threadIdx.x == 0) spin_ge_relaxed(v.completed, seq.gen);
  __syncthreads();
  const uint32_t lane = lane_id();
  const uint32_t q = lane / L, sub = lane % L;
  const uint64_t pos = ((uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5) * POS + q;
  const bool valid = pos < n;
  const uint64_t key = valid ? keys[pos] : 0ull;
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
  // misses: the group's lane 0 claims the key
  bool claimed = false;
  uint32_t tslot = 0;
  if (valid && sub == 0 && res == kNoSlot) {
    tslot = miss_insert(v.miss_table, v.cap, keys, key, uint32_t(pos), &claimed);
    v.miss_slot[pos] = tslot;
  }
  if (valid && sub == 0) {
    flags[pos] = res == kNoSlot ? 1 : 0;
    if (v.flags_dev != nullptr) v.flags_dev[pos] = res == kNoSlot ? 1 : 0;
  }
  pdl_trigger();
  // recency exchange by the group's lane 0, issued before the copy
  bool stamp_it = valid && sub == 0 && res != kNoSlot;
  if (stamp_it) stamp_it = block_set_insert(s_stamped, 1u << kSetBits, res);
  const uint32_t uh = stamp_it ? stamp_slot(c, v, res, stamp) : 0u;
  // row copy (after the call's bookkeeping): lane `sub` moves float4
  // chunks sub, sub+L, sub+2L, ...
  auto copy_row = [&] {
    const uint32_t d = c.d;
    const float* src = res != kNoSlot ? c.rows + uint64_t(res) * d : default_row;
    float* dst = out + pos * d;
    if ((d & 3u) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15u) == 0 &&
        (reinterpret_cast<uintptr_t>(src) & 15u) == 0) {
      const uint32_t d4 = d >> 2;
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* o4 = reinterpret_cast<float4*>(dst);
      for (uint32_t ch0 = 0; ch0 < d4; ch0 += L * RC) {
        float4 x[RC];
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          const uint32_t ch = ch0 + uint32_t(j) * L + sub;
          if (ch < d4) x[j] = ld_row_f4(s4 + ch);
        }
#pragma unroll
        for (int j = 0; j < RC; ++j) {
          const uint32_t ch = ch0 + uint32_t(j) * L + sub;
          if (ch < d4) st_cs_f4(o4 + ch, x[j]);
        }
      }
    } else {
      for (uint32_t ch = sub; ch < d; ch += L) dst[ch] = src[ch];
    }
  };
  // claims and counts
  const uint32_t cm = __ballot_sync(0xFFFFFFFFu, claimed);
  if (cm) {
    const uint32_t first_lane = __ffs(cm) - 1;
    uint32_t at = 0;
    if (lane == first_lane) at = atomicAdd(v.list_ctr, uint32_t(__popc(cm)));
    at = __shfl_sync(0xFFFFFFFFu, at, first_lane);
    if (claimed) {
      const uint32_t e = at + __popc(cm & ((1u << lane) - 1u));
      v.list[e] = tslot;
      v.list_keys[e] = key;
      v.claim_of_slot[tslot] = e;
    }
  }
  if (last_block(v, 0, gridDim.x)) finish_claims(v);
  if (valid) copy_row();
  warp_add_counts(v, uh, claimed ? 1u : 0u, blockIdx.x * kWarps + (threadIdx.x >> 5));
  if (last_block(v, 1, gridDim.x)) finish_counts(v, seq.gen, seq.prev_target);
}

// ====================================================== lane-per-position --
// Compile-time A/B knobs (tools/build_variant.py): 256-bit chunks in flight
// per lane in the row copy, and the minimum resident blocks per SM (the
// register cap); defaults = the measured best.
#ifndef HPSB_COPY_U
#define HPSB_COPY_U 2
#endif
#ifndef HPSB_SINGLE_COPY_U
#define HPSB_SINGLE_COPY_U 4
#endif
#ifndef HPSB_SINGLE_MINB_THREADS
#define HPSB_SINGLE_MINB_THREADS 1024
#endif
#ifndef HPSB_MINB_THREADS
#define HPSB_MINB_THREADS 1536
#endif
// Copy of a warp's rows (lane i's row = slot `res` of lane i, or the
// default row) into the warp's contiguous output block: `CH` floats per
// access (8 = 256-bit, 4 = 128-bit, 1 = scalar), U accesses in flight.
template <int CH, int U>
__device__ __forceinline__ void warp_copy_rows(const CacheDev& c, uint32_t res, uint32_t nrows,
                                               const float* __restrict__ default_row,
                                               float* __restrict__ obase) {
  const uint32_t lane = lane_id();
  const uint32_t d = c.d;
  const uint32_t cpr = d / CH;  // chunks per row
  const bool pow2 = (cpr & (cpr - 1)) == 0;
  const uint32_t sh = __ffs(cpr) - 1;
  const uint32_t total = nrows * cpr;
  for (uint32_t c0 = 0; c0 < total; c0 += 32 * U) {
    Chunk<CH> x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t ch = c0 + uint32_t(u) * 32 + lane;
      uint32_t row = pow2 ? (ch >> sh) : (ch / cpr);
      row = min(row, 31u);
      const uint32_t slot = __shfl_sync(0xFFFFFFFFu, res, row);
      if (ch < total) {
        const uint32_t j = ch - row * cpr;
        const float* src = slot != kNoSlot ? c.rows + uint64_t(slot) * d : default_row;
        x[u].load(src + j * CH);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t ch = c0 + uint32_t(u) * 32 + lane;
      if (ch < total) x[u].store(obase + uint64_t(ch) * CH);
    }
  }
}

// WARPS = warps per block; the block keeps a shared set of the slots it has
// stamped, so a hot slot sees one global exchange per block (a power-law
// batch repeats its top key in ~19% of positions). The register budget is
// capped so the next lookup's blocks can be resident during this one's
// copies (2 x 1024 threads per SM).
// The body of one table's lookup for block `blk` of its `nblocks` blocks
// (the single-table kernel passes blockIdx / gridDim; the multi-table
// kernel the block's rank within its table).
template <int CH, int WARPS, bool SF>
__device__ __forceinline__ void lookup_body(const CacheDev& c, const uint64_t* __restrict__ keys,
                                            uint64_t n, float* __restrict__ out,
                                            uint8_t* __restrict__ flags,
                                            const float* __restrict__ default_row,
                                            uint64_t stamp, const LookupView& v, uint32_t skip,
                                            uint32_t blk, uint32_t nblocks) {
  constexpr int kThreadsB = WARPS * 32;
  constexpr uint32_t kSetSize = 2 * kThreadsB;  // power of two for WARPS in {2, 4, 8, 16}
  __shared__ uint32_t s_stamped[kSetSize];
  for (uint32_t i = threadIdx.x; i < kSetSize; i += kThreadsB) s_stamped[i] = kNoSlot;
  // the view's previous use must have completed (normally long ago)
  if (threadIdx.x == 0) spin_ge_relaxed(v.completed, call_gen(v));
  __syncthreads();
  trace_min(v, 0, false);
  trace_min(v, 2, true);
  // The next lookup on the stream may start now (programmatic dependent
  // launch): nothing in this call depends on the previous one past the
  // view wait above, so as many calls overlap as views and SM slots allow
  // (trigger here vs after the probe and claims: 9.4 vs 10.0 us per cfg-2
  // batch).
  pdl_trigger();
  const uint32_t lane = lane_id();
  const uint64_t base = (uint64_t(blk) * kThreadsB + threadIdx.x) & ~31ull;
  const uint64_t pos = base + lane;
  const bool valid = pos < n;
  // ---- A: probe, claims, flags (independent of the previous call) ----
  const uint64_t key = valid ? keys[pos] : 0ull;
  const uint32_t res = lane_probe(c, key, valid);
  const bool miss = valid && res == kNoSlot && !(skip & kSkipMiss);
  // SF: recency exchange before the claims -- the slot's counter and mark
  // reads go out first and their round trip overlaps the claims' atomics
  // (single-call latency 26.8 -> 25.0 us at cfg 2); a call pipelined behind
  // another lookup keeps the exchange after the claims ticket (1-2 % more
  // throughput when calls overlap)
  uint32_t uh = 0, um = 0;
  if constexpr (SF) {
    stamp = call_stamp(v, stamp);
    const uint32_t same_slot = __match_any_sync(0xFFFFFFFFu, res);
    bool stamp_it = res != kNoSlot && (__ffs(same_slot) - 1) == lane && !(skip & kSkipStamp);
    if (stamp_it) stamp_it = block_set_insert(s_stamped, kSetSize, res);
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(c.counters) + res;
    unsigned long long cur_ctr = ~0ull, cur_hit = 0ull;
    uint64_t hh = 0;
    if (stamp_it) {
      cur_ctr = __ldcg(ctr);
      hh = hit_home(v, res);
      cur_hit = __ldcg(v.hits + hh);
    }
    um = warp_claim_misses(v, keys, pos, key, miss);
    if (valid) {
      flags[pos] = res == kNoSlot ? 1 : 0;
      if (v.flags_dev != nullptr) v.flags_dev[pos] = res == kNoSlot ? 1 : 0;
    }
    if (cur_ctr < stamp) atomicMax(ctr, stamp);
    uh = stamp_it ? hit_insert(v, res, uint32_t(stamp), hh, cur_hit) : 0u;
  } else {
    um = warp_claim_misses(v, keys, pos, key, miss);
    if (valid) {
      flags[pos] = res == kNoSlot ? 1 : 0;
      if (v.flags_dev != nullptr) v.flags_dev[pos] = res == kNoSlot ? 1 : 0;
    }
  }
  if (v.trace) {
    __syncthreads();
    trace_min(v, 1, true);
    trace_min(v, 3, false);
  }
  // ---- claims ticket without stalling the block: warps 1.. arrive at a
  // named barrier and go on; warp 0 waits for them and takes the ticket; the
  // block that was last completes the claim list after its copies (a
  // block-wide barrier + ticket here: 10.33 vs 10.01 us per cfg-2 batch) ----
  __shared__ uint32_t s_last_claims;
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("bar.sync 1, %0;" ::"r"(kThreadsB) : "memory");
    if (threadIdx.x == 0) {
      const bool last = atom_add_release(v.done, 1u) == nblocks - 1;
      if (last) fence_acq_rel();
      s_last_claims = last ? 1u : 0u;
    }
  } else {
    asm volatile("bar.arrive 1, %0;" ::"r"(kThreadsB) : "memory");
  }
  // ---- C: recency exchange, row copy, counts ----
  if constexpr (!SF) {
    stamp = call_stamp(v, stamp);
    const uint32_t same_slot = __match_any_sync(0xFFFFFFFFu, res);
    bool stamp_it = res != kNoSlot && (__ffs(same_slot) - 1) == lane && !(skip & kSkipStamp);
    if (stamp_it) stamp_it = block_set_insert(s_stamped, kSetSize, res);
    uh = stamp_it ? stamp_slot(c, v, res, stamp) : 0u;
  }
  // behind an update (programmatic dependent launch): its row writes must be
  // complete before the rows are read
  if (skip & kWaitBeforeCopy) pdl_wait();
  const uint32_t nrows = n > base + 32 ? 32u : uint32_t(n > base ? n - base : 0);
  // a lone call has the SMs to itself: twice the chunks in flight per lane
  // (single-call latency -1.7 us at cfg 2); pipelined calls keep registers
  // low so several calls stay resident
  constexpr int kU = SF ? HPSB_SINGLE_COPY_U : HPSB_COPY_U;
  if (!(skip & kSkipCopy))
    warp_copy_rows<CH, CH == 8 ? kU : 2 * kU>(c, res, nrows, default_row, out + base * c.d);
  warp_add_counts(v, uh, um, blk * WARPS + (threadIdx.x >> 5));
  if (v.trace) {
    __syncthreads();
    trace_min(v, 4, false);
    trace_min(v, 5, true);
  }
  __syncthreads();
  if (s_last_claims) {
    trace_min(v, 6, false);
    finish_claims(v);
    trace_min(v, 7, false);
  }
  if (last_block(v, 1, nblocks)) finish_counts(v, call_gen(v), call_prev_target(v));
}

template <int CH, int WARPS, bool SF>
__global__ void __launch_bounds__(WARPS * 32,
                                  (SF ? HPSB_SINGLE_MINB_THREADS : HPSB_MINB_THREADS) / (WARPS * 32))
    k_lookup_tag(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                 float* __restrict__ out, uint8_t* __restrict__ flags,
                 const float* __restrict__ default_row, uint64_t stamp, LookupView v,
                 uint32_t skip) {
  lookup_body<CH, WARPS, SF>(c, keys, n, out, flags, default_row, stamp, v, skip, blockIdx.x,
                             gridDim.x);
}

// Several tables (caches) in ONE launch: block b belongs to the table whose
// [block_begin, block_begin + nblocks) range holds b; each table runs the
// single-table body on its own blocks, views and tickets.
template <int CH, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1024 / (WARPS * 32))
    k_lookup_tag_multi(const TableLookup* __restrict__ tables, uint32_t count) {
  __shared__ uint32_t s_t;
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    while (t + 1 < count && tables[t + 1].block_begin <= blockIdx.x) ++t;
    s_t = t;
  }
  __syncthreads();
  const TableLookup& tl = tables[s_t];
  lookup_body<CH, WARPS, true>(tl.c, tl.keys, tl.n, tl.out, tl.flags, tl.default_row, tl.stamp,
                               tl.v, 0u, blockIdx.x - tl.block_begin, tl.nblocks);
}

void launch_lookup_multi(const TableLookup* d_tables, uint32_t count, uint32_t total_blocks,
                         int ch, cudaStream_t st) {
  if (total_blocks == 0) return;
  constexpr int W = 8;
  if (ch == 8)
    k_lookup_tag_multi<8, W><<<total_blocks, W * 32, 0, st>>>(d_tables, count);
  else if (ch == 4)
    k_lookup_tag_multi<4, W><<<total_blocks, W * 32, 0, st>>>(d_tables, count);
  else
    k_lookup_tag_multi<1, W><<<total_blocks, W * 32, 0, st>>>(d_tables, count);
  check_launch("lookup_multi", 1);
}

// ============================================= small calls (one block) --
// A lone call of at most kSmallLookup positions in ONE block, every step in
// shared memory: the miss dedup (first position by atomicMin in a block hash
// table over the batch's keys, staged in shared memory), the distinct-slot
// set for recency stamps and unique hits, the per-call counts. No global
// miss table, no block tickets, no finish passes: a 32-key call was ~15 us
// event-bracketed through the multi-block kernel's dozen dependent global
// round trips. Claims are emitted in table order (the host sorts them by
// first position, as for the large kernel); miss_slot[pos] holds the claim
// index and claim_of_slot the identity, so the sync-branch scatter works
// unchanged. Used only when the call is not chained behind another lookup
// (stream order then covers every view-ordering rule).
constexpr uint32_t kSmallLookup = 1024;
constexpr uint32_t kSmallTab = 2 * kSmallLookup;

template <int CH>
__global__ void __launch_bounds__(kSmallLookup)
    k_lookup_small(CacheDev c, const uint64_t* __restrict__ keys, uint32_t n,
                   float* __restrict__ out, uint8_t* __restrict__ flags,
                   const float* __restrict__ default_row, uint64_t stamp, LookupView v) {
  __shared__ unsigned long long s_key[kSmallLookup];
  __shared__ uint32_t s_tab[kSmallTab];    // 0 = empty, else first position + 1
  __shared__ uint32_t s_slots[kSmallTab];  // distinct hit slots
  __shared__ uint32_t s_claim[kSmallTab];  // claim index of a table entry
  __shared__ uint32_t s_nclaims, s_uh;
  const uint32_t t = threadIdx.x;
  const uint32_t lane = lane_id();
  for (uint32_t i = t; i < kSmallTab; i += blockDim.x) {
    s_tab[i] = 0u;
    s_slots[i] = kNoSlot;
  }
  if (t == 0) {
    s_nclaims = 0u;
    s_uh = 0u;
  }
  stamp = call_stamp(v, stamp);
  const bool valid = t < n;
  const uint64_t key = valid ? keys[t] : 0ull;
  s_key[t] = key;
  const uint32_t res = lane_probe(c, key, valid);
  __syncthreads();
  // hits: one recency exchange and one unique hit per distinct slot
  uint32_t uh = 0;
  bool first_hit = false;
  if (res != kNoSlot) {
    // exact distinct-slot set (at most kSmallLookup slots in 2x entries)
    uint32_t q = (res * 0x9E3779B1u) >> 7;
    while (true) {
      q &= kSmallTab - 1;
      const uint32_t cur = atomicCAS(&s_slots[q], kNoSlot, res);
      if (cur == kNoSlot) {
        first_hit = true;
        break;
      }
      if (cur == res) break;
      ++q;
    }
  }
  if (first_hit) {
    atomicMax(reinterpret_cast<unsigned long long*>(c.counters) + res,
              (unsigned long long)stamp);
    uh = 1;
  }
  // misses: dedup in the block table, first position kept
  uint32_t h = 0;
  if (valid && res == kNoSlot) {
    h = uint32_t(fmix64(key ^ 0x9E3779B97F4A7C15ull)) & (kSmallTab - 1);
    while (true) {
      const uint32_t old = atomicCAS(&s_tab[h], 0u, t + 1);
      if (old == 0u) break;
      if (s_key[old - 1] == key) {
        if (t + 1 < old) atomicMin(&s_tab[h], t + 1);
        break;
      }
      h = (h + 1) & (kSmallTab - 1);
    }
  }
  uh = __reduce_add_sync(0xFFFFFFFFu, uh);
  if (lane == 0 && uh) atomicAdd(&s_uh, uh);
  if (valid) {
    flags[t] = res == kNoSlot ? 1 : 0;
    if (v.flags_dev != nullptr) v.flags_dev[t] = res == kNoSlot ? 1 : 0;
  }
  __syncthreads();
  // one claim per table entry (the entry's final value is the first position)
  for (uint32_t i = t; i < kSmallTab; i += blockDim.x) {
    const uint32_t f = s_tab[i];
    if (f != 0u) {
      const uint32_t e = atomicAdd(&s_nclaims, 1u);
      s_claim[i] = e;
      v.list_keys[e] = s_key[f - 1];
      v.list_firsts[e] = f - 1;
      v.claim_of_slot[e] = e;
    }
  }
  __syncthreads();
  if (valid && res == kNoSlot) v.miss_slot[t] = s_claim[h];
  // rows: the warp's 32 consecutive positions as one contiguous block
  const uint32_t base = t & ~31u;
  const uint32_t nrows = n > base + 32 ? 32u : (n > base ? n - base : 0u);
  if (nrows) warp_copy_rows<CH, CH == 8 ? 4 : 8>(c, res, nrows, default_row, out + uint64_t(base) * c.d);
  __syncthreads();
  if (t == 0) {
    v.counts_out[0] = s_uh;
    v.counts_out[1] = s_nclaims;
    // the view is free for its next use (the large kernel's completion rule)
    __threadfence();
    st_release(v.completed, call_gen(v) + 1);
  }
}

// --------------------------------------------------------------- rebase --
struct RebaseWords {
  unsigned long long w[1 + kLookupViews];
};
__global__ void k_rebase(unsigned long long* __restrict__ out, RebaseWords r) {
  if (threadIdx.x <= kLookupViews) out[threadIdx.x] = r.w[threadIdx.x];
}

void launch_rebase(unsigned long long* w, unsigned long long stamp_base,
                   const unsigned long long (&use_base)[kLookupViews], cudaStream_t st) {
  RebaseWords r;
  r.w[0] = stamp_base;
  for (int k = 0; k < kLookupViews; ++k) r.w[1 + k] = use_base[k];
  k_rebase<<<1, 32, 0, st>>>(w, r);
  check_launch("rebase", 1);
}

// --------------------------------------------------------------- launch --
unsigned launch_lookup_probe(const CacheDev& c, const uint64_t* keys, uint64_t n, float* out,
                             uint8_t* flags, const float* default_row, uint64_t stamp,
                             const LookupView& v, bool after_lookup, cudaStream_t st,
                             bool wait_before_copy) {
  if (n == 0) return 0;
  // Kernel choice (HPSB_LOOKUP_KERNEL): lane-per-position fingerprint probe
  // by default; "warp4" / "warp8" = the warp-cooperative ballot probe (4 or
  // 8 lanes per position) for A/B measurement.
  static const int variant = [] {
    const char* e = std::getenv("HPSB_LOOKUP_KERNEL");
    if (e && std::string(e) == "warp4") return 4;
    if (e && std::string(e) == "warp8") return 8;
    return 0;
  }();
  static const uint32_t diag_skip = [] {
    const char* e = std::getenv("HPSB_DIAG_SKIP");
    return e ? uint32_t(std::atoi(e)) & 7u : 0u;
  }();
  const uint32_t skip = diag_skip | ((wait_before_copy && after_lookup) ? kWaitBeforeCopy : 0u);
  static const int warps = [] {
    const char* e = std::getenv("HPSB_LOOKUP_WARPS");
    const int w = e ? std::atoi(e) : 8;
    return (w == 2 || w == 4 || w == 16) ? w : 8;
  }();
  // Programmatic dependent launch behind a preceding lookup kernel on this
  // stream (HPSB_NO_PDL=1 disables): its phase A overlaps that lookup's tail.
  static const bool no_pdl = std::getenv("HPSB_NO_PDL") != nullptr;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.stream = st;
  cfg.attrs = attr;
  // (the warp-cooperative variant has no grid wait before its copies: it
  // never chains behind an update)
  cfg.numAttrs = (after_lookup && !no_pdl && !(variant != 0 && wait_before_copy)) ? 1 : 0;
  if (variant == 0) {
    auto aligned = [](const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; };
    const int ch = (c.d % 8 == 0 && aligned(out, 32) && aligned(default_row, 32))   ? 8
                   : (c.d % 4 == 0 && aligned(out, 16) && aligned(default_row, 16)) ? 4
                                                                                     : 1;
    // The throughput-ordered variant for every call except one chained
    // behind an update (which waits before its copies): the latency-ordered
    // variant (SF, recency exchange before the claims) measured no lower
    // single-call latency on the round-2 kernel and made the first call of a
    // pipelined sequence slower (20-step cfg-2 graph: 7.62 vs 7.49 G keys/s,
    // 3 reps each, profiles/r02_ab_lookup.txt). HPSB_LOOKUP_LONE_VARIANT=1
    // restores it for unchained calls.
    static const bool lone_variant = std::getenv("HPSB_LOOKUP_LONE_VARIANT") != nullptr;
    const bool pipelined = (cfg.numAttrs == 1 || !lone_variant) && !(skip & kWaitBeforeCopy);
    static const bool no_small = std::getenv("HPSB_LOOKUP_NO_SMALL") != nullptr;
    if (cfg.numAttrs == 0 && n <= kSmallLookup && diag_skip == 0 && v.trace == nullptr &&
        !no_small) {
      if (ch == 8)
        k_lookup_small<8><<<1, kSmallLookup, 0, st>>>(c, keys, uint32_t(n), out, flags,
                                                      default_row, stamp, v);
      else if (ch == 4)
        k_lookup_small<4><<<1, kSmallLookup, 0, st>>>(c, keys, uint32_t(n), out, flags,
                                                      default_row, stamp, v);
      else
        k_lookup_small<1><<<1, kSmallLookup, 0, st>>>(c, keys, uint32_t(n), out, flags,
                                                      default_row, stamp, v);
      check_launch("lookup", 1);
      return 1;
    }
    auto go = [&](auto chc, auto wc) {
      constexpr int CH = decltype(chc)::value, WARPS = decltype(wc)::value;
      cfg.gridDim = dim3(unsigned((n + WARPS * 32 - 1) / (WARPS * 32)));
      cfg.blockDim = dim3(WARPS * 32);
      if (pipelined)
        cudaLaunchKernelEx(&cfg, k_lookup_tag<CH, WARPS, false>, c, keys, n, out, flags,
                           default_row, stamp, v, skip);
      else
        cudaLaunchKernelEx(&cfg, k_lookup_tag<CH, WARPS, true>, c, keys, n, out, flags,
                           default_row, stamp, v, skip);
    };
    auto by_warps = [&](auto chc) {
      switch (warps) {
        case 2: go(chc, std::integral_constant<int, 2>{}); break;
        case 4: go(chc, std::integral_constant<int, 4>{}); break;
        case 16: go(chc, std::integral_constant<int, 16>{}); break;
        default: go(chc, std::integral_constant<int, 8>{}); break;
      }
    };
    if (ch == 8) by_warps(std::integral_constant<int, 8>{});
    else if (ch == 4) by_warps(std::integral_constant<int, 4>{});
    else by_warps(std::integral_constant<int, 1>{});
  } else {
    const uint64_t per_block = uint64_t(kWarps) * (32 / variant);
    cfg.gridDim = dim3(unsigned((n + per_block - 1) / per_block));
    cfg.blockDim = dim3(kThreads);
    if (variant == 4)
      cudaLaunchKernelEx(&cfg, k_lookup<4>, c, keys, n, out, flags, default_row, stamp, v);
    else
      cudaLaunchKernelEx(&cfg, k_lookup<8>, c, keys, n, out, flags, default_row, stamp, v);
  }
  check_launch("lookup", 1);
  return 1;
}

// ---------------------------------------------------- sync-branch scatter --
__global__ void __launch_bounds__(256)
    k_lookup_scatter(uint64_t n, uint32_t d, uint8_t* __restrict__ flags, LookupView v,
                     const int32_t* __restrict__ row_of_claim, const float* __restrict__ staged,
                     float* __restrict__ out) {
  const uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  if ((v.flags_dev != nullptr ? v.flags_dev[i] : flags[i]) == 0) return;
  const uint32_t e = v.claim_of_slot[v.miss_slot[i]];
  const int32_t r = row_of_claim[e];
  if (r < 0) return;  // absent from every tier: keep default + flag
  warp_copy_row(staged + uint64_t(r) * d, out + i * d, d);
  __syncwarp();
  if (lane_id() == 0) flags[i] = 0;
}

void launch_lookup_scatter(uint64_t n, uint32_t d, uint8_t* flags, const LookupView& v,
                           const int32_t* row_of_claim, const float* staged, float* out,
                           cudaStream_t st) {
  if (n == 0) return;
  const uint64_t threads = n * 32;
  k_lookup_scatter<<<unsigned((threads + 255) / 256), 256, 0, st>>>(n, d, flags, v, row_of_claim,
                                                                    staged, out);
  check_launch("lookup_scatter", 1);
}

}  // namespace hpsb
