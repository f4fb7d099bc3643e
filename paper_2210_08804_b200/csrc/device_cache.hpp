// device_cache.hpp -- one HBM-resident slab-cache replica and its
// operations; the object behind the hps_cache_* C ABI.
//
// Mirrors hps::SlabCache (slab_cache.hpp:41-179): same configuration
// checks, same recency clock rules (query bumps once per call before any
// check, replace stamps with the current value, update never touches it),
// same results. Concurrency model: one CUDA stream per cache; every
// operation holds `mu_` while it enqueues, so operations are linearised in
// stream order (the reference's per-slabset gates, slab_cache.cpp:214, are
// replaced by stream ordering -- no torn reads).
#pragma once

#include <atomic>
#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.hpp"
#include "peer.hpp"
#include "runtime.hpp"

namespace hpsb {

struct CacheConfig {
  uint64_t slabset_count = 1;
  uint32_t slabs_per_set = 2;
  uint32_t dimension = 0;
  uint32_t worker_pool_size = 1;
  uint32_t tasks_per_worker = 8;
};

enum MemKind : int { kHostMem = 0, kDeviceMem = 1 };

class DeviceCache;

// One cache's lookups inside one captured CUDA graph: what every replay
// consumes (clock ticks, uses of each lookup view) and the device words the
// graph's lookups read their stamps / generations relative to.
struct GraphCacheUse {
  DeviceCache* cache = nullptr;
  uint64_t serial = 0;  // the cache's identity (pointers may be reused)
  int slot = -1;        // rebase slot of the cache
  uint64_t stamps = 0;  // clock ticks per replay
  uint64_t uses[kLookupViews] = {};
};

struct StreamHolder {
  cudaStream_t s = nullptr;
  ~StreamHolder() {
    if (s) cudaStreamDestroy(s);
  }
};

class DeviceCache {
 public:
  // share_stream_with: join another cache's stream (a cache group on one
  // device, e.g. the tables of one model); null = a stream of its own.
  DeviceCache(const CacheConfig& cfg, int device, const DeviceCache* share_stream_with = nullptr);
  ~DeviceCache();
  DeviceCache(const DeviceCache&) = delete;
  DeviceCache& operator=(const DeviceCache&) = delete;

  // slab_cache.cpp:69-91. Returns the miss count; misses ascending.
  size_t query(const uint64_t* keys, size_t n, float* out, size_t out_len, uint32_t* miss_pos,
               uint64_t* miss_keys, int mem, cudaStream_t user);
  // slab_cache.cpp:93-107
  void replace(const uint64_t* keys, size_t n, const float* vectors, size_t vectors_len,
               int mem, cudaStream_t user);
  // slab_cache.cpp:109-125
  size_t update(const uint64_t* keys, size_t n, const float* vectors, size_t vectors_len,
                int mem, cudaStream_t user);
  // Replace mode: 0 = exact (the reference's per-set input order, the
  // default), 1 = relaxed (atomicCAS slot claims, every key at once; used by
  // the calls whose keys are known distinct: host-mode replace, the device
  // fill below and the engine's fills -- a device-mode replace that must
  // reject duplicates stays exact).
  void set_replace_mode(int mode);
  int replace_mode() const { return replace_mode_.load(std::memory_order_relaxed); }
  // keys the relaxed mode did not admit so far (syncs the stream)
  uint64_t relaxed_dropped();
  // Stream-ordered replace of DISTINCT keys on device pointers (the engine's
  // fill primitive): no duplicate check, no host synchronisation.
  void replace_device_async(const uint64_t* keys, size_t n, const float* rows, cudaStream_t user);
  // Stream-ordered update on device pointers (online training path): no
  // host sync; *written (device u64, may be null) gets the count.
  void update_device(const uint64_t* keys, size_t n, const float* vectors, uint64_t* written,
                     cudaStream_t user);
  // Stream-ordered dump into device memory (refresh on the GPU): resident
  // keys of sets [set_begin, set_end) in set / slab / slot order into `out`
  // (capacity (set_end - set_begin) * W * 32), the count into *n_out.
  void dump_device(uint64_t set_begin, uint64_t set_end, uint64_t* out, uint64_t* n_out,
                   cudaStream_t user);
  // Lookup-level query on device pointers (the engine's hot path without
  // the tier logic): bumps the clock, writes every position's row (hit:
  // cached row, miss: default_row), miss flags, the unique missing keys with
  // their first-occurrence positions (claim order; ascending position = the
  // reference's order) and {unique hits, unique misses} of this call to
  // device memory. Stream-ordered, no host synchronisation.
  void lookup_device(const uint64_t* keys, size_t n, float* out, uint8_t* flags,
                     const float* default_row, uint64_t* miss_keys, uint32_t* miss_firsts,
                     uint64_t* counts, cudaStream_t user);
  // Diagnostic: events recorded around the probe kernel of the next
  // lookup_device calls (null = off).
  void set_profile_events(cudaEvent_t start, cudaEvent_t end) {
    prof_start_ = start;
    prof_end_ = end;
  }
  // DumpCursor::next over a slabset range (host output)
  size_t dump(uint64_t set_begin, uint64_t set_end, uint64_t* out, size_t cap);
  // slab_cache.cpp:407-442
  void check_invariants();
  void export_state(uint64_t* keys, uint64_t* counters, uint32_t* masks, float* rows);

  uint32_t dimension() const { return cfg_.dimension; }
  uint64_t slabset_count() const { return cfg_.slabset_count; }
  uint32_t slabs_per_set() const { return cfg_.slabs_per_set; }
  uint64_t capacity() const { return cfg_.slabset_count * cfg_.slabs_per_set * 32ull; }
  uint64_t occupied();
  uint64_t recency_clock() const { return clock_.load(std::memory_order_relaxed); }
  int device() const { return device_; }
  cudaStream_t stream() const { return stream_; }
  const CacheDev& dev() const { return dev_; }
  int keys_per_warp() const { return keys_per_warp_; }

  // Staging of the refresh loop (refresh_cache, engine.cpp), kept across
  // calls: a periodic refresh reuses its pinned / device buffers (a fresh
  // 2 x 33.5 MB cudaHostAlloc per pass cost more than the pass's host fetch).
  struct RefreshBuffers {
    std::mutex mu;  // one refresh pass of this cache at a time
    PinnedBuffer h[2];
    DeviceBuffer dv[2];
    DeviceBuffer written;
    std::vector<uint64_t> keys;
  };
  RefreshBuffers& refresh_buffers() { return refresh_; }

  // ---- peer-memory sharded mode (peer.hpp) ----
  // Exports this shard for peers: IPC handles of the probe structures, the
  // rows and a miss inbox of inbox_cap keys (allocated on the first export).
  void peer_export(uint64_t inbox_cap, PeerBlob* out);
  void peer_inbox(unsigned long long** count, uint64_t** keys, uint64_t* cap) const;
  // Takes the keys peers appended to this shard's inbox since the last
  // drain (up to cap into out; returns how many were appended, which may
  // exceed the inbox capacity -- the rest were dropped) and empties it. Call
  // only between lookup phases (no peer may be appending).
  size_t peer_drain(uint64_t* out, size_t cap);

  // ---- engine-facing primitives (caller holds mutex()) ----
  std::mutex& mutex() { return mu_; }
  // grows the replace scratch for calls of up to n keys now (engine reserve)
  void reserve_replace(uint64_t n);
  // Callers that enqueue their own work on stream() (the engine) call this
  // under mutex() so the next lookup does not chain onto a stale lookup.
  void note_stream_op() { mark_other_op(); }
  // Makes the distinct-hit tables of `ls` valid for a call with `stamp`
  // (call under mutex(); enqueues a clear on stream() when the stamps' high
  // 32 bits changed since the tables were last used).
  void prepare_hits(LookupScratch& ls, uint64_t stamp);
  uint64_t capacity_slots() const { return cfg_.slabset_count * cfg_.slabs_per_set * 32ull; }
  // Stamps never have zero low 32 bits (the tag of a free hit-table entry).
  uint64_t bump_clock() {
    uint64_t s = clock_.fetch_add(1, std::memory_order_relaxed) + 1;
    if (uint32_t(s) == 0) s = clock_.fetch_add(1, std::memory_order_relaxed) + 1;
    return s;
  }
  // Device keys / rows, distinct keys guaranteed by the caller; stamp = the
  // current clock. Enqueued on stream(); scratch is the cache's own.
  void replace_device_locked(const uint64_t* d_keys, size_t n, const float* d_rows);

  // Makes stream() wait for work already queued on `user` (no-op if null
  // or identical), and the reverse.
  void join_from(cudaStream_t user);
  void join_to(cudaStream_t user);

  // ---- CUDA graph replay (hps_stream_begin_capture / hps_graph_launch) ----
  // Lookups captured into a graph take their stamps and view generations
  // relative to device words (a rebase slot of the cache); every launch of
  // the graph first writes the current clock and view uses there and
  // advances them by what one replay consumes, so replays are exactly
  // equivalent to issuing the same lookups again (fresh stamps in stream
  // order, unique hits counted, views reused only after release).
  // The sessions of capture `capture_id`, closed (the host clock and view
  // uses restored to their values at capture start).
  static std::vector<GraphCacheUse> end_capture(unsigned long long capture_id);
  // Launch of a graph on `x`: before -- orders earlier cache work before the
  // graph and writes the rebase words; after -- orders later cache work after
  // it. Callers hold mutex() of every cache of the graph.
  void graph_before_launch_locked(const GraphCacheUse& u, cudaStream_t x);
  void graph_after_launch_locked(cudaStream_t x);
  void release_rebase_slot(int slot);
  uint64_t serial() const { return serial_; }
  // true when `c` with `serial` is a live cache
  static bool alive(const DeviceCache* c, uint64_t serial);

 private:
  void* scratch(size_t bytes) { return scratch_.ensure(bytes, stream_); }
  void* pinned(size_t bytes) { return pinned_.ensure(bytes); }
  void ensure_scan_tiles(uint64_t tiles);

  CacheConfig cfg_;
  int device_;
  int keys_per_warp_;
  CacheDev dev_{};
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev_in_ = nullptr, ev_out_ = nullptr;
  std::mutex mu_;
  std::atomic<uint64_t> clock_{0};
  std::atomic<int> replace_mode_{0};
  // exact or relaxed replace of device keys / rows (distinct keys)
  void launch_replace_mode(const uint64_t* d_keys, uint64_t n, const float* d_rows,
                           uint64_t stamp, bool validate, const ReplaceScratch& rs);
  ScanState scan_;
  DeviceBuffer scratch_;
  // replace: persistent per-call set table (kernels.hpp ReplaceScratch)
  DeviceBuffer rbuf_;
  DeviceBuffer relaxed_buf_;  // relaxed replace: each key's claimed slot
  ReplaceScratch rs_;
  uint64_t rcap_ = 0;
  const ReplaceScratch& replace_scratch_locked(uint64_t n);
  PinnedBuffer pinned_;
  // lookup_device scratch
  DeviceBuffer lbuf_;
  LookupScratch lws_;
  uint64_t lcap_ = 0;
  // true while the last operation enqueued on stream_ is a lookup kernel
  // (the next lookup may then launch as its programmatic dependent)
  bool last_op_lookup_ = false;
  // true while the last operation enqueued is an update's write kernel (the
  // next lookup may chain behind it, waiting before its row copies)
  bool last_op_update_ = false;
  void mark_other_op() {
    last_op_lookup_ = false;
    last_op_update_ = false;
  }
  std::shared_ptr<StreamHolder> stream_holder_;
  // graph capture: the open session of this cache (capture id 0 = none)
  struct CaptureSession {
    unsigned long long id = 0;
    int slot = -1;
    uint64_t clock0 = 0;
    uint64_t uses0[kLookupViews] = {};
  } cap_;
  static constexpr int kRebaseSlots = 64;
  unsigned long long* rebase_ = nullptr;  // kRebaseSlots x 16 words
  std::vector<int> free_slots_;
  uint64_t serial_ = 0;
  // update: per-slot winning position + 1 (all-zero between calls); two
  // arrays, consecutive updates alternate (the next update's probe may run
  // while this update's write kernel is in flight)
  uint32_t* winner_ = nullptr;
  void* probe_mem_ = nullptr;  // keys + fingerprints (one allocation)
  uint64_t updates_ = 0;
  uint32_t* next_winner() {
    return winner_ + ((updates_++ & 1u) ? cfg_.slabset_count * cfg_.slabs_per_set * 32ull : 0ull);
  }
  DeviceBuffer ubuf_;  // update_device scratch
  void* inbox_ = nullptr;  // peer miss inbox: [u64 count | 248 B pad | keys]
  uint64_t inbox_cap_ = 0;
  RefreshBuffers refresh_;
  PinnedBuffer qstage_;  // zero-copy host-mode query staging
  static constexpr uint64_t kZeroCopyQueryMax = 65536;
  static constexpr uint64_t kZeroCopyReplaceMax = 256;  // the one-launch replace kernels' limit
  uint64_t ucap_ = 0;
  // diagnostic lookup timeline ring (HPSB_TRACE=1): kTraceRing calls x 8
  unsigned long long* trace_ = nullptr;
  uint64_t trace_calls_ = 0;

 public:
  static constexpr uint64_t kTraceRing = 4096;
  // Copies the ring (kTraceRing x 8 u64, call k at row k % kTraceRing) and
  // returns the number of traced calls; 0 when tracing is off.
  uint64_t trace(unsigned long long* out);

 private:
  cudaEvent_t prof_start_ = nullptr, prof_end_ = nullptr;
  unsigned long long* d_small_ = nullptr;  // small device counters
  unsigned long long* h_small_ = nullptr;  // pinned mirror
};

}  // namespace hpsb
