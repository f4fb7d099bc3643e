// include/hps/lookup_engine.hpp -- drop-in replacement for the reference's
// core/include/hps/lookup_engine.hpp (hps::LookupEngine, tier_fetch,
// lookup_engine.hpp:29-196), backed by the B200 lookup engine of
// libhps_b200.so (hps_engine_* in include/hps_b200.h).
//
// The dedup -> cache query -> hit-rate switch -> expansion runs on the GPU
// (one kernel per lookup, lookup_kernels.cu); the misses are fetched
// in-process from the NATIVE volatile DB (include/hps/volatile_store.hpp,
// the drop-in hps::VolatileStore) straight into the engine's pinned staging,
// then from the reference's PersistentStore (kept; reached through the
// engine's cold-tier callback) for the rest, in the reference's tier order
// (lookup_engine.cpp:50-89), and admitted with the GPU replace.
//
// Use: this repo's include/ ahead of core/include, link libhps_b200.so and
// the reference's types.cpp + persistent_store.cpp instead of
// slab_cache.cpp / lookup_engine.cpp / volatile_store.cpp. The reference's
// tests/unit/test_lookup_engine.cpp compiles unchanged against it
// (oracle/Makefile target _ref/test_lookup_engine_b200).
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hps/persistent_store.hpp"
#include "hps/slab_cache.hpp"
#include "hps/types.hpp"
#include "hps/volatile_store.hpp"
#include "hps_b200.h"

#if defined(__linux__)
#include <sys/mman.h>
#endif
#if defined(__GLIBC__)
#include <malloc.h>
#endif

namespace hps {

// lookup_engine.hpp:29-37
struct EngineConfig {
  double hit_rate_threshold = 0.8;
  std::vector<float> default_vector;
  std::size_t workspace_pool_size = 16;
  std::uint32_t async_worker_count = 2;
  bool volatile_tier_enabled = true;
};

// lookup_engine.hpp:115-119
struct TierCounters {
  std::uint64_t vdb_hits = 0;
  std::uint64_t pdb_hits = 0;
  std::uint64_t missing = 0;
};

namespace b200_detail {
// A value-initialised vector of n elements, as std::vector(n) gives, but with
// its storage advised onto transparent huge pages before the zero-fill: a
// 33.5 MB result (cfg 2: 65,536 x 128 floats) then takes ~17 page faults
// instead of ~8,200 -- the fault path dominates a fresh result's cost.
template <class T>
std::vector<T> sized_vector(std::size_t n) {
  std::vector<T> v;
  v.reserve(n);
#if defined(__linux__) && defined(MADV_HUGEPAGE)
  constexpr std::uintptr_t kHuge = std::uintptr_t(2) << 20;
  const auto a = reinterpret_cast<std::uintptr_t>(v.data());
  const std::uintptr_t lo = (a + kHuge - 1) & ~(kHuge - 1);
  const std::uintptr_t hi = (a + n * sizeof(T)) & ~(kHuge - 1);
  if (hi > lo) (void)::madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);
#endif
  v.resize(n);
  return v;
}

// hps_cold_fetch_fn over the reference's PersistentStore::get
// (persistent_store.cpp:405-439): the tier below the native volatile DB.
struct PdbTier {
  PersistentStore* pdb;
  const std::string* table;
};
inline int pdb_fetch(void* ctx, const uint64_t* keys, size_t n, uint64_t* found_keys,
                     float* found_vectors, size_t* n_found, uint64_t* missing_keys,
                     size_t* n_missing) {
  auto* t = static_cast<PdbTier*>(ctx);
  try {
    FetchResult f = t->pdb->get(*t->table, std::span<const EmbeddingKey>(keys, n));
    std::copy(f.found_keys.begin(), f.found_keys.end(), found_keys);
    std::copy(f.found_vectors.begin(), f.found_vectors.end(), found_vectors);
    std::copy(f.missing_keys.begin(), f.missing_keys.end(), missing_keys);
    *n_found = f.found_keys.size();
    *n_missing = f.missing_keys.size();
    return 0;
  } catch (...) {
    return 1;  // surfaces as TierFault (sync) or an async fault
  }
}
}  // namespace b200_detail

// lookup_engine.cpp:50-89 (tier order: volatile first, persistent for the
// rest, persistent hits promoted to the volatile tier asynchronously; found
// rows in (volatile-found, persistent-found) order) -- run by the native
// hps_tier_fetch over the native volatile DB.
inline FetchResult tier_fetch(const TableId& table, std::span<const EmbeddingKey> keys,
                              VolatileStore* vdb, PersistentStore& pdb,
                              TierCounters* counters = nullptr) {
  FetchResult out;
  if (keys.empty()) return out;
  out.found_keys.resize(keys.size());
  out.found_vectors.resize(keys.size() * table.dimension);
  out.missing_keys.resize(keys.size());
  b200_detail::PdbTier tier{&pdb, &table.name};
  std::size_t nf = 0, nm = 0;
  std::uint64_t c[3] = {0, 0, 0};
  b200_detail::check(hps_tier_fetch(vdb ? vdb->handle() : nullptr, table.name.c_str(),
                                    table.dimension, &b200_detail::pdb_fetch, &tier, keys.data(),
                                    keys.size(), out.found_keys.data(), out.found_vectors.data(),
                                    &nf, out.missing_keys.data(), &nm, c));
  out.found_keys.resize(nf);
  out.found_vectors.resize(nf * table.dimension);
  out.missing_keys.resize(nm);
  if (counters) {
    counters->vdb_hits += c[0];
    counters->pdb_hits += c[1];
    counters->missing += c[2];
  }
  return out;
}

// lookup_engine.hpp:129-142
struct EngineStatsSnapshot {
  std::uint64_t queries = 0;
  std::uint64_t queried_keys = 0;
  std::uint64_t unique_keys = 0;
  std::uint64_t cache_hits = 0;
  std::uint64_t cache_misses = 0;
  std::uint64_t sync_batches = 0;
  std::uint64_t async_batches = 0;
  std::uint64_t defaults_returned = 0;
  std::uint64_t vdb_hits = 0;
  std::uint64_t pdb_hits = 0;
  std::uint64_t tier_missing = 0;
  std::uint64_t async_faults = 0;
};

// lookup_engine.hpp:145-150
struct LookupOutcome {
  bool sync_branch = false;
  double unique_hit_rate = 0.0;
  std::size_t unique_count = 0;
  std::size_t defaults_returned = 0;
};

// The engine's bounded workspace pool (lookup_engine.hpp:49-71): each
// workspace is a device + pinned staging set; acquiring one is the admission
// ticket, a background fill holds it until the fetched rows are admitted.
class WorkspacePool {
 public:
  std::size_t size() const { return info(0); }
  std::size_t outstanding() const { return info(1); }
  std::size_t peak_outstanding() const { return info(2); }

 private:
  friend class LookupEngine;
  std::size_t info(int which) const {
    std::uint64_t v[3] = {0, 0, 0};
    b200_detail::check(hps_engine_pool_info(engine_, &v[0], &v[1], &v[2]));
    return v[which];
  }
  hps_engine* engine_ = nullptr;
};

class LookupEngine {
 public:
  // lookup_engine.cpp:91-117 (same validation, std::invalid_argument)
  LookupEngine(const TableId& table, SlabCache& cache, VolatileStore* vdb, PersistentStore& pdb,
               EngineConfig config)
      : table_(table),
        cache_(cache),
        vdb_(vdb),
        pdb_(pdb),
        config_(std::move(config)),
        tier_{&pdb_, &table_.name} {
    if (config_.workspace_pool_size == 0)
      throw std::invalid_argument("workspace pool size must be positive");
    validate_table_id(table_);
    hps_engine_config c{};
    c.hit_rate_threshold = config_.hit_rate_threshold;
    c.default_vector = config_.default_vector.empty() ? nullptr : config_.default_vector.data();
    c.default_vector_len = uint32_t(config_.default_vector.size());
    c.workspace_pool_size = uint32_t(config_.workspace_pool_size);
    c.async_worker_count = config_.async_worker_count;
    c.volatile_tier_enabled = config_.volatile_tier_enabled ? 1 : 0;
    c.max_batch = 0;
    // misses: the native volatile DB in-process, then the persistent tier
    b200_detail::check(hps_engine_create(table_.name.c_str(), table_.dimension, cache_.handle(),
                                         vdb_ ? vdb_->handle() : nullptr,
                                         &b200_detail::pdb_fetch, &tier_, &c, &h_));
    pool_.engine_ = h_;
  }
  ~LookupEngine() {
    {
      std::lock_guard<std::mutex> lk(spare_mu_);
      spare_stop_ = true;
    }
    spare_cv_.notify_all();
    if (spare_thr_.joinable()) spare_thr_.join();
    hps_engine_destroy(h_);
  }

  LookupEngine(const LookupEngine&) = delete;
  LookupEngine& operator=(const LookupEngine&) = delete;

  // lookup_engine.cpp:130-241
  LookupResult lookup(std::span<const EmbeddingKey> keys, LookupOutcome* outcome = nullptr) {
    LookupResult r;
    r.dimension = table_.dimension;
    r.vectors = take_result_storage(keys.size() * table_.dimension);
    r.miss_flags.resize(keys.size());
    hps_lookup_outcome o{};
    b200_detail::check(hps_engine_lookup(h_, keys.data(), keys.size(), r.vectors.data(),
                                         r.vectors.size(), r.miss_flags.data(), &o, HPS_MEM_HOST,
                                         nullptr));
    if (outcome) {
      outcome->sync_branch = o.sync_branch != 0;
      outcome->unique_hit_rate = o.unique_hit_rate;
      outcome->unique_count = o.unique_count;
      outcome->defaults_returned = o.defaults_returned;
    }
    return r;
  }

  void drain_async() { b200_detail::check(hps_engine_drain_async(h_)); }

  // B200 extension: allocate every workspace for batches of up to max_keys
  // now (pinned staging included), so no lookup pays a first-use allocation.
  // Also keeps LookupResult storage of that size on the malloc heap: glibc
  // serves blocks above M_MMAP_THRESHOLD (at most 32 MiB by default) with a
  // fresh mmap and unmaps them on free, so every result of a large batch
  // (cfg 2: 33.5 MB) would page-fault its whole buffer again while
  // resize() zero-fills it; with the threshold raised the freed block of
  // the previous result is reused, already faulted in. Process-wide
  // allocator tuning, done only here (serving setup).
  void reserve(std::size_t max_keys) {
    b200_detail::check(hps_engine_reserve(h_, max_keys));
#if defined(__GLIBC__)
    const std::size_t bytes = max_keys * std::size_t(table_.dimension) * sizeof(float);
    if (bytes >= (std::size_t(16) << 20) && bytes < (std::size_t(256) << 20)) {
      (void)::mallopt(M_MMAP_THRESHOLD, int(bytes + bytes / 4 + (std::size_t(1) << 20)));
      (void)::mallopt(M_TRIM_THRESHOLD, int(4 * bytes));
    }
#endif
  }

  EngineStatsSnapshot stats() const {
    hps_engine_stats s{};
    b200_detail::check(hps_engine_get_stats(h_, &s));
    EngineStatsSnapshot o;
    o.queries = s.queries;
    o.queried_keys = s.queried_keys;
    o.unique_keys = s.unique_keys;
    o.cache_hits = s.cache_hits;
    o.cache_misses = s.cache_misses;
    o.sync_batches = s.sync_batches;
    o.async_batches = s.async_batches;
    o.defaults_returned = s.defaults_returned;
    o.async_faults = s.async_faults;
    o.vdb_hits = s.vdb_hits;  // sync and background fetches alike
    o.pdb_hits = s.pdb_hits;
    o.tier_missing = s.tier_missing;
    return o;
  }
  const TableId& table() const { return table_; }
  WorkspacePool& workspace_pool() { return pool_; }

 private:
  // Result storage (B200 extension, no API change): LookupResult::vectors is
  // a std::vector<float> the call hands to the caller, and sizing one
  // zero-fills it (33.5 MB per cfg-2 call, serial, before any row can land).
  // Large results are instead taken from a spare vector a background thread
  // has already sized for the previous call's shape, and the thread sizes
  // the next spare while the caller works -- the zero-fill leaves the call's
  // critical path. Other sizes, or a spare not ready yet, size in the call
  // as before. Every element is overwritten by the lookup either way.
  static constexpr std::size_t kSpareMinFloats = std::size_t(1) << 18;  // 1 MB
  std::vector<float> take_result_storage(std::size_t n) {
    if (n < kSpareMinFloats) return b200_detail::sized_vector<float>(n);
    std::vector<float> v;
    {
      std::lock_guard<std::mutex> lk(spare_mu_);
      if (spare_ready_ && spare_.size() == n) {
        v.swap(spare_);
        spare_ready_ = false;
      }
      spare_want_ = n;
      if (!spare_thr_.joinable()) spare_thr_ = std::thread([this] { spare_loop(); });
    }
    spare_cv_.notify_one();
    if (v.size() != n) v = b200_detail::sized_vector<float>(n);
    return v;
  }
  void spare_loop() {
    std::unique_lock<std::mutex> lk(spare_mu_);
    while (true) {
      spare_cv_.wait(lk, [this] { return spare_stop_ || (!spare_ready_ && spare_want_ != 0); });
      if (spare_stop_) return;
      const std::size_t n = spare_want_;
      lk.unlock();
      std::vector<float> v = b200_detail::sized_vector<float>(n);
      lk.lock();
      if (spare_want_ == n) {
        spare_ = std::move(v);
        spare_ready_ = true;
      }
    }
  }
  std::mutex spare_mu_;
  std::condition_variable spare_cv_;
  std::vector<float> spare_;
  std::size_t spare_want_ = 0;
  bool spare_ready_ = false;
  bool spare_stop_ = false;
  std::thread spare_thr_;

  TableId table_;
  SlabCache& cache_;
  VolatileStore* vdb_;
  PersistentStore& pdb_;
  EngineConfig config_;
  b200_detail::PdbTier tier_;
  hps_engine* h_ = nullptr;
  WorkspacePool pool_;
};

}  // namespace hps
