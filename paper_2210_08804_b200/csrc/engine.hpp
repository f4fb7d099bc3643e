// engine.hpp -- B200 lookup engine (the object behind hps_engine_*).
//
// Mirrors hps::LookupEngine (lookup_engine.hpp:152-196): one lookup =
// fused device probe of every query position (dedup of hits is implicit,
// see lookup_kernels.cu), unique-key hit rate h = 1 - |misses|/|Q*|
// (h = 1 for an empty batch), strict `h < threshold` switch between the
// synchronous tier fetch + replace and the asynchronous default-rows path
// whose fetch + replace run on background workers holding the workspace
// lease, and the same statistics. Workspaces are a bounded pool of device
// + pinned buffers (the reference's WorkspacePool, lookup_engine.cpp:9-48):
// acquiring one is the admission ticket, so the pool bounds in-flight
// batches and provides backpressure.
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "device_cache.hpp"
#include "kernels.hpp"
#include "runtime.hpp"
#include "volatile_store.hpp"

namespace hpsb {

// Cold tier (stands in for PersistentStore::get, persistent_store.cpp:405-439).
using ColdFetchFn = int (*)(void* ctx, const uint64_t* keys, size_t n, uint64_t* found_keys,
                            float* found_vectors, size_t* n_found, uint64_t* missing_keys,
                            size_t* n_missing);

struct TierCounters {
  uint64_t vdb_hits = 0, cold_hits = 0, missing = 0;
};

// tier_fetch (lookup_engine.cpp:50-89) writing found rows straight into
// `rows` (n * dim) in found order (VDB hits in input order, then cold hits in
// input order); row_of[i] = found row of keys[i] or -1. found_keys holds n.
void tier_fetch_staged(VolatileStore* vdb, const std::string& table, uint32_t dim,
                       ColdFetchFn cold, void* cold_ctx, const uint64_t* keys, size_t n,
                       uint64_t* found_keys, float* rows, int32_t* row_of, size_t* n_found,
                       uint64_t* missing_keys, size_t* n_missing, TierCounters* counters);

// refresh_engine.cpp:5-22 (refresh_cache) on the B200 cache: dump, tier
// fetch, non-admitting update, pipelined over two staging buffers.
struct RefreshResult {
  uint64_t refreshed = 0;            // cache rows actually rewritten
  std::vector<uint64_t> unresolved;  // resident but absent from every tier (dump order)
};
RefreshResult refresh_cache(DeviceCache& cache, VolatileStore* vdb, const std::string& table,
                            ColdFetchFn cold, void* cold_ctx, size_t dump_batch);

struct EngineConfig {
  double hit_rate_threshold = 0.8;
  std::vector<float> default_vector;
  uint32_t workspace_pool_size = 16;
  uint32_t async_worker_count = 2;
  bool volatile_tier_enabled = true;
  uint32_t max_batch = 0;  // largest accepted batch (0 = any below 2^32)
};

struct LookupOutcome {
  bool sync_branch = false;
  double unique_hit_rate = 0.0;
  uint64_t unique_count = 0;
  uint64_t defaults_returned = 0;
};

struct EngineStats {
  uint64_t queries = 0, queried_keys = 0, unique_keys = 0, cache_hits = 0, cache_misses = 0,
           sync_batches = 0, async_batches = 0, defaults_returned = 0, vdb_hits = 0,
           pdb_hits = 0, tier_missing = 0, async_faults = 0;
};

// Device + pinned buffers of one in-flight batch.
struct Workspace {
  int device = 0;
  uint64_t capacity = 0;  // keys
  uint32_t dim = 0;
  // device
  DeviceBuffer dbuf;
  uint64_t* d_keys = nullptr;
  float* d_out = nullptr;
  uint8_t* d_flags = nullptr;
  int32_t* d_row_of = nullptr;
  float* d_staged = nullptr;
  uint64_t* d_found_keys = nullptr;
  LookupScratch ls;
  LookupView lv;  // the view of the last lookup
  // pinned host
  PinnedBuffer hbuf;
  uint64_t* h_keys = nullptr;
  unsigned long long* h_counts = nullptr;
  uint64_t* h_miss_keys = nullptr;
  int32_t* h_row_of = nullptr;
  float* h_staged = nullptr;
  uint64_t* h_found_keys = nullptr;
  uint64_t* h_missing = nullptr;
  uint8_t* h_flags = nullptr;
  float* h_out = nullptr;
  uint64_t* h_claim_keys = nullptr;    // unique misses in claim order
  uint32_t* h_claim_firsts = nullptr;  // their first positions
  int32_t* h_row_of_claim = nullptr;   // staged row per claim (sync branch)
  char* h_hdr = nullptr;               // zero-copy calls: [counts | firsts | keys | flags]
  std::vector<uint32_t> order;         // claims sorted by first position
  // sync branch of a host-mode call: found miss key -> staged row (open
  // addressing; hs_used marks occupied entries, every u64 is a legal key)
  const uint64_t* scatter_keys = nullptr;
  std::vector<uint64_t> hs_keys;
  std::vector<int32_t> hs_rows;
  std::vector<uint8_t> hs_used;
  // batch state (for the async task)
  std::vector<uint64_t> missing_keys;
  cudaEvent_t done = nullptr;
  cudaEvent_t rows_ready = nullptr;  // zero-copy sync branch: rows final (replace may run on)
  cudaEvent_t counts_ready = nullptr;  // the lookup's counts and first claims are in host memory
  cudaEvent_t uploaded = nullptr;      // async fill: staged rows copied to the device (copy stream)
  // pageable output: the rows come back in chunks into h_out, one event per
  // chunk, and are copied on to the caller's memory by several threads as
  // each chunk lands
  static constexpr int kOutChunks = 64;
  cudaEvent_t chunk_ev[kOutChunks] = {};
  int out_chunks = 0;
  bool pending = false;  // `done` recorded, not yet waited

  ~Workspace();
  void ensure(uint64_t n, uint32_t d, cudaStream_t st);
  void wait_idle();
};

class WorkspacePool {
 public:
  WorkspacePool(size_t size, int device);
  Workspace* acquire();  // blocks until one is free
  void release(Workspace* ws);
  // fn(ws) on every workspace, each taken out of the pool for the call
  template <class F>
  void for_each(F&& fn) {
    std::vector<Workspace*> held;
    for (size_t i = 0; i < slots_.size(); ++i) held.push_back(acquire());
    try {
      for (Workspace* w : held) fn(*w);
    } catch (...) {
      for (Workspace* w : held) release(w);
      throw;
    }
    for (Workspace* w : held) release(w);
  }
  size_t size() const { return slots_.size(); }
  size_t outstanding() const;
  size_t peak_outstanding() const;

 private:
  std::vector<std::unique_ptr<Workspace>> slots_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::vector<Workspace*> free_;
  size_t outstanding_ = 0, peak_ = 0;
};

class LookupEngine {
 public:
  LookupEngine(const std::string& table, uint32_t dim, DeviceCache* cache, VolatileStore* vdb,
               ColdFetchFn cold, void* cold_ctx, EngineConfig cfg);
  ~LookupEngine();

  void lookup(const uint64_t* keys, size_t n, float* out, size_t out_len, uint8_t* flags,
              LookupOutcome* outcome, int mem, cudaStream_t user);
  // Several tables at once (one engine each; the reference's caller loops
  // over tables): every table's device work is enqueued before any host
  // wait, so the lookups overlap on the GPU. Same per-table semantics.
  static void lookup_multi(LookupEngine* const* engines, size_t count,
                           const uint64_t* const* keys, const size_t* n, float* const* out,
                           uint8_t* const* flags, LookupOutcome* outcomes, int mem);
  void drain_async();
  // Allocates every workspace (device + pinned staging) and the cache's
  // replace scratch for batches of up to n keys now, so no lookup pays a
  // first-use allocation (a pinned staging set is ~100 MB at cfg 2). Also
  // run at construction when EngineConfig::max_batch is set.
  void reserve(uint64_t n);
  EngineStats stats() const;
  uint32_t dimension() const { return dim_; }
  WorkspacePool& pool() { return pool_; }
  DeviceCache* cache() const { return cache_; }
  uint32_t dim() const { return dim_; }
  const float* default_row() const { return d_default_; }

  // One table of a MultiLookup: its device part ran in the group launch and
  // the counts, the claims (sorted to the reference's miss order) and the
  // rows are already on the host (`out`/`flags`, user memory). Applies the
  // hit-rate switch, the miss path (sync: fetch, scatter into the table's
  // device rows d_out with view `v`, replace, rows copied back; async: the
  // background fill) and the stats -- exactly LookupEngine::finish's rules.
  struct GroupResult {
    size_t n = 0;
    uint64_t uh = 0, um = 0;
    const uint64_t* miss_keys = nullptr;  // um keys, reference order
    float* out = nullptr;
    uint8_t* flags = nullptr;
    const uint64_t* h_keys = nullptr;  // the table's keys (host)
  };
  void finish_group(const GroupResult& r, LookupOutcome* outcome);

 private:
  // claims copied back speculatively with the counts (one round trip when a
  // call has at most this many unique misses)
  static constexpr uint64_t kSpeculativeClaims = 4096;
  static constexpr uint64_t kPackedMax = 4096;
  static constexpr uint64_t kZeroCopyReplaceMax = 256;  // = the single-block replace limit
  // one lookup split at its first host wait (begin enqueues, finish waits)
  struct LookupCall {
    std::chrono::steady_clock::time_point t0;  // start of begin (phase trace)
    LookupEngine* engine = nullptr;
    Workspace* ws = nullptr;
    size_t n = 0;
    float* out = nullptr;
    uint8_t* flags = nullptr;
    int mem = 0;
    cudaStream_t user = nullptr;
    bool host = true, spec_rows = false, out_pinned = false, flags_pinned = false;
    uint64_t spec_claims = 0;
    // packed: zero-copy call (host mode, <= kPackedMax keys): the kernels read
    // keys and write rows, flags, counts and every claim (first positions,
    // keys) in pinned host memory; out_direct = rows go to the caller's own
    // pinned `out`
    bool packed = false, out_direct = false;
    const unsigned long long* hc = nullptr;
    const uint32_t* hcf = nullptr;
    const uint64_t* hck = nullptr;
    const uint8_t* hfl = nullptr;
    const uint64_t* d_keys = nullptr;
    const uint64_t* h_keys = nullptr;  // host mode: the caller's keys
    float* d_out = nullptr;
    uint8_t* d_flags = nullptr;
  };
  // Sync branch of a host-mode call whose rows came back with the counts:
  // the fetched rows are written straight into the host output at every
  // position of their key (and those flags cleared) by the copy threads.
  // (ws.scatter_keys: the unique misses in the order of ws.h_row_of)
  void host_scatter(Workspace& ws, size_t n, const uint64_t* keys, float* out, uint64_t um,
                    uint8_t* hflags);
  LookupCall begin(const uint64_t* keys, size_t n, float* out, size_t out_len, uint8_t* flags,
                   int mem, cudaStream_t user);
  void finish(LookupCall& c, LookupOutcome* outcome);
  void abandon(LookupCall& c);
  // the previous lookup took the async branch: speculate that this one will
  // too and bring its rows back with the counts
  std::atomic<bool> last_async_{false};

  struct AsyncTask {
    Workspace* ws;
  };
  void async_loop();
  // fetch ws->missing_keys from the tiers into ws's pinned staging, upload,
  // and (optionally) scatter into the output + replace into the cache.
  size_t fetch_and_upload(Workspace& ws, const uint64_t* miss_keys, size_t n_miss,
                          TierCounters* counters, size_t* n_found);
  // rows (n * dim floats at d_out) back to the host: straight into the
  // caller's `out` when it is pinned, else chunked into ws.h_out
  void rows_d2h(Workspace& ws, const LookupCall& c, cudaStream_t st);
  // completes rows_d2h for a pageable `out`: waits chunk by chunk and copies
  // each on to `out` over the copy threads
  void rows_to_pageable(Workspace& ws, const LookupCall& c);

  std::string table_;
  uint32_t dim_;
  DeviceCache* cache_;
  VolatileStore* vdb_;
  ColdFetchFn cold_;
  void* cold_ctx_;
  EngineConfig cfg_;
  float* d_default_ = nullptr;
  WorkspacePool pool_;
  // the miss path's side stream: background fills upload their staged rows
  // here, so the copies never sit in front of a lookup on the cache stream
  cudaStream_t copy_stream_ = nullptr;
  ThreadPool copy_threads_;  // pageable-output copies

  mutable std::mutex stats_mu_;
  EngineStats stats_;

  std::mutex q_mu_;
  std::condition_variable q_cv_, idle_cv_;
  std::deque<AsyncTask> queue_;
  size_t active_ = 0;
  bool stopping_ = false;
  std::vector<std::thread> workers_;
};

// Several tables whose caches form one cache group (one stream): a lookup
// of all of them is ONE H2D (descriptors + packed keys), ONE kernel
// (k_lookup_tag_multi), one D2H of every table's counts / flags / first
// claims, one D2H of the rows, and one host wait -- then each table's
// hit-rate switch and miss path (LookupEngine::finish_group). The small-batch
// latency of a many-table model is then one round trip, not one per table.
class MultiLookup {
 public:
  MultiLookup(std::vector<LookupEngine*> engines, uint64_t max_batch);
  ~MultiLookup();
  MultiLookup(const MultiLookup&) = delete;
  MultiLookup& operator=(const MultiLookup&) = delete;
  void lookup(const uint64_t* const* keys, const size_t* n, float* const* out,
              uint8_t* const* flags, LookupOutcome* outcomes);
  size_t tables() const { return eng_.size(); }

 private:
  static constexpr uint64_t kPackedRowBytes = 1 << 20;
  static constexpr uint64_t kDirectRowBytes = 64ull << 20;
  std::vector<LookupEngine*> eng_;
  uint64_t maxb_;
  int ch_ = 1;
  std::mutex mu_;
  std::vector<LookupScratch> ls_;  // per table, its own views
  DeviceBuffer scratch_dev_;
  DeviceBuffer dev_;
  PinnedBuffer host_;
  cudaEvent_t done_ = nullptr;
  // layout (offsets in the device / host blocks)
  uint64_t d_desc_ = 0, d_keys_ = 0, d_counts_ = 0, d_flags_ = 0, d_ckeys_ = 0, d_cfirsts_ = 0,
           d_rows_ = 0;
  std::vector<uint64_t> row_off_;  // per table, in floats from d_rows_
  uint64_t h_rows_ = 0;
  std::vector<uint32_t> order_;
  std::vector<uint64_t> miss_;
};

// The paper's concurrent deployment in ONE process: one
// cache replica per GPU, each with its own engine, all engines over the SAME
// host volatile DB (its partitions shared, host RAM not multiplied by the GPU
// count), each replica serving its own query stream. lookup() hands every
// replica its batch on its own persistent host thread and returns when all
// are done; there is no collective -- the replicas only meet in the VDB.
class ReplicaGroup {
 public:
  explicit ReplicaGroup(std::vector<LookupEngine*> engines);
  ~ReplicaGroup();
  ReplicaGroup(const ReplicaGroup&) = delete;
  ReplicaGroup& operator=(const ReplicaGroup&) = delete;
  size_t size() const { return eng_.size(); }
  // replica r looks up keys[r][0..n[r]) exactly as LookupEngine::lookup;
  // the first failure (if any) is rethrown after every replica finished
  void lookup(const uint64_t* const* keys, const size_t* n, float* const* out,
              uint8_t* const* flags, LookupOutcome* outcomes, int mem);

 private:
  struct Job {
    const uint64_t* keys = nullptr;
    size_t n = 0;
    float* out = nullptr;
    uint8_t* flags = nullptr;
    LookupOutcome* outcome = nullptr;
    int mem = 0;
  };
  void worker(size_t r);
  std::vector<LookupEngine*> eng_;
  std::vector<Job> jobs_;
  std::vector<std::exception_ptr> errs_;
  std::vector<std::thread> threads_;
  std::mutex call_mu_;  // one group call at a time
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  size_t pending_ = 0;
  bool stop_ = false;
};

}  // namespace hpsb
