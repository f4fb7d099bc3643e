// include/hps/volatile_store.hpp -- drop-in replacement for the reference's
// core/include/hps/volatile_store.hpp (hps::VolatileStore,
// VolatileTableConfig, partition_of; volatile_store.hpp:27-89), backed by the
// native host volatile DB of libhps_b200.so (hps_vdb_* in include/hps_b200.h).
//
// Same class, same members, same semantics and error behaviour: hash
// partitions routed by xxh64(key, 0) % P, upsert + evict-oldest down to the
// overflow margin (ties toward the smaller key), one clock tick per lookup /
// insert, last-access refreshes that never move a stamp backwards. The
// storage underneath is the miss path's: open-addressing arenas, lookups
// fanned out over a thread pool, found rows copied once in found order.
//
// The point of swapping it in is the lookup path: a hps::LookupEngine
// (include/hps/lookup_engine.hpp) built over THIS VolatileStore hands the
// native store straight to the GPU engine, so cache misses are fetched
// in-process into the engine's pinned staging -- no per-key partition
// mutex, no unordered_map, no std::vector per row. The reference's
// tests/unit/test_volatile_store.cpp compiles unchanged against this header
// (oracle/Makefile target _ref/test_volatile_store_b200).
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "hps/slab_cache.hpp"  // b200_detail::check, the reference vocabulary
#include "hps/types.hpp"
#include "hps_b200.h"

namespace hps {

// volatile_store.hpp:27-29
enum class EvictionPolicy {
  EvictOldest,
};

// volatile_store.hpp:31-40
struct VolatileTableConfig {
  std::uint32_t partition_count = 16;
  // Maximum entries a partition may hold after an insert returns.
  std::size_t overflow_margin = 1u << 20;
  EvictionPolicy policy = EvictionPolicy::EvictOldest;
  // Consumed by the wiring layer (preload fraction), stored with the tier.
  double initial_cache_rate = 1.0;
};

// volatile_store.cpp:10-13 (stable across hosts and runs)
inline std::uint32_t partition_of(EmbeddingKey key, std::uint32_t partition_count) {
  return hps_partition_of(key, partition_count);
}

class VolatileStore {
 public:
  // `lookup_threads` = host threads one lookup fans out over (0 = all cores).
  explicit VolatileStore(std::uint32_t lookup_threads = 0) {
    b200_detail::check(hps_vdb_create(lookup_threads, &h_));
  }
  ~VolatileStore() { hps_vdb_destroy(h_); }

  VolatileStore(const VolatileStore&) = delete;
  VolatileStore& operator=(const VolatileStore&) = delete;

  // volatile_store.cpp:26-52 (validate_table_id + the same checks)
  void register_table(const TableId& table, const VolatileTableConfig& config) {
    b200_detail::check(hps_vdb_register_table(h_, table.name.c_str(), table.dimension,
                                              config.partition_count,
                                              config.overflow_margin));
  }
  bool has_table(const std::string& name) const {
    return hps_vdb_has_table(h_, name.c_str()) != 0;
  }
  std::uint32_t partition_count(const std::string& name) const {
    std::uint32_t v = 0;
    b200_detail::check(hps_vdb_partition_count(h_, name.c_str(), &v));
    return v;
  }

  // volatile_store.cpp:82-112: found rows in input order, one clock tick.
  FetchResult lookup(const std::string& name, std::span<const EmbeddingKey> keys) {
    const std::uint32_t dim = dimension(name);
    FetchResult r;
    r.found_keys.resize(keys.size());
    r.found_vectors.resize(keys.size() * dim);
    r.missing_keys.resize(keys.size());
    std::size_t nf = 0, nm = 0;
    b200_detail::check(hps_vdb_lookup(h_, name.c_str(), keys.data(), keys.size(),
                                      r.found_keys.data(), r.found_vectors.data(), &nf,
                                      r.missing_keys.data(), &nm));
    r.found_keys.resize(nf);
    r.found_vectors.resize(nf * dim);
    r.missing_keys.resize(nm);
    return r;
  }

  // volatile_store.cpp:114-125: upsert, prune touched partitions, evicted keys.
  std::vector<EmbeddingKey> insert(const std::string& name, std::span<const EmbeddingKey> keys,
                                   std::span<const float> vectors) {
    std::vector<EmbeddingKey> ev(keys.size() + 64);
    std::size_t n = 0;
    b200_detail::check(hps_vdb_insert(h_, name.c_str(), keys.data(), keys.size(), vectors.data(),
                                      vectors.size(), ev.data(), ev.size(), &n));
    return finish_evicted(std::move(ev), n);
  }

  // volatile_store.cpp:175-189: validated now, applied on the background worker.
  void insert_async(const std::string& name, std::vector<EmbeddingKey> keys,
                    std::vector<float> vectors) {
    b200_detail::check(hps_vdb_insert_async(h_, name.c_str(), keys.data(), keys.size(),
                                            vectors.data(), vectors.size()));
  }

  // volatile_store.cpp:191-200
  std::vector<EmbeddingKey> evict(const std::string& name, std::uint32_t partition) {
    std::vector<EmbeddingKey> ev(64);
    std::size_t n = 0;
    b200_detail::check(
        hps_vdb_evict(h_, name.c_str(), partition, ev.data(), ev.size(), &n));
    return finish_evicted(std::move(ev), n);
  }

  // volatile_store.cpp:251-254
  void drain() { b200_detail::check(hps_vdb_drain(h_)); }

  std::size_t partition_size(const std::string& name, std::uint32_t partition) const {
    std::uint64_t v = 0;
    b200_detail::check(hps_vdb_partition_size(h_, name.c_str(), partition, &v));
    return v;
  }
  std::size_t table_size(const std::string& name) const {
    std::uint64_t v = 0;
    b200_detail::check(hps_vdb_table_size(h_, name.c_str(), &v));
    return v;
  }
  std::optional<std::uint64_t> last_access(const std::string& name, EmbeddingKey key) const {
    std::uint64_t v = 0;
    int found = 0;
    b200_detail::check(hps_vdb_last_access(h_, name.c_str(), key, &v, &found));
    if (!found) return std::nullopt;
    return v;
  }
  std::uint64_t table_clock(const std::string& name) const {
    std::uint64_t v = 0;
    b200_detail::check(hps_vdb_table_clock(h_, name.c_str(), &v));
    return v;
  }
  std::vector<EmbeddingKey> keys(const std::string& name) const {
    std::size_t n = 0;
    b200_detail::check(hps_vdb_keys(h_, name.c_str(), nullptr, 0, &n));
    std::vector<EmbeddingKey> out(n + 1024);  // concurrent inserts may add keys
    b200_detail::check(hps_vdb_keys(h_, name.c_str(), out.data(), out.size(), &n));
    if (n > out.size()) {
      out.resize(n);
      b200_detail::check(hps_vdb_keys(h_, name.c_str(), out.data(), out.size(), &n));
    }
    out.resize(std::min(n, out.size()));
    return out;
  }

  // B200 extension: the native store, for hps_engine_create / hps_tier_fetch.
  hps_vdb* handle() const { return h_; }

 private:
  std::uint32_t dimension(const std::string& name) const {
    std::uint32_t d = 0;
    b200_detail::check(hps_vdb_dimension(h_, name.c_str(), &d));
    return d;
  }
  static std::vector<EmbeddingKey> finish_evicted(std::vector<EmbeddingKey> ev, std::size_t n) {
    if (n > ev.size()) {
      ev.resize(n);
      b200_detail::check(hps_vdb_last_evicted(ev.data(), ev.size(), &n));
    }
    ev.resize(n);
    return ev;
  }

  hps_vdb* h_ = nullptr;
};

}  // namespace hps
