// ref_shim.cpp -- C ABI over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY (see oracle/hps_oracle.c header). Compiled by
// oracle/Makefile together with the reference's own .cpp files straight
// from /root/reference/proj (never copied) into oracle/_ref/libhps_ref.so.
// Used (1) to pin the C restatement in oracle/hps_oracle.c, (2) to generate
// the golden fixtures under tests/golden/, and (3) as the timed CPU baseline
// (`bench.py --impl reference`, cpu_baseline kind "reference").
//
// Wrapped reference entry points:
//   hps::SlabCache            core/include/hps/slab_cache.hpp:41-116
//   hps_test::ReferenceCache  tests/oracles/reference_cache.hpp:18-180
//   hps::dedup_keys           core/src/types.cpp:20-34
//   hps::xxh64 / xxh64_key    core/include/hps/xxhash64.hpp:60-124
//   hps::PowerLawSampler      core/src/workload.cpp:24-70
//   hps::VolatileStore        core/include/hps/volatile_store.hpp:45-137
//   hps::LookupEngine         core/include/hps/lookup_engine.hpp:152-196
//   hps::PersistentStore      core/include/hps/persistent_store.hpp:39-95
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "hps/lookup_engine.hpp"
#include "hps/persistent_store.hpp"
#include "hps/slab_cache.hpp"
#include "hps/types.hpp"
#include "hps/wire.hpp"
#include "hps/volatile_store.hpp"
#include "hps/workload.hpp"
#include "hps/xxhash64.hpp"
#include "oracles/reference_cache.hpp"

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_xxh64(const void* p, size_t n, uint64_t seed) {
  return hps::xxh64(p, n, seed);
}
uint64_t ref_xxh64_key(uint64_t k, uint64_t seed) {
  return hps::xxh64_key(k, seed);
}
uint32_t ref_partition_of(uint64_t k, uint32_t p) { return hps::partition_of(k, p); }

size_t ref_dedup(const uint64_t* keys, size_t n, uint64_t* uniq, uint32_t* inv) {
  auto d = hps::dedup_keys(std::span<const uint64_t>(keys, n));
  std::memcpy(uniq, d.unique_keys.data(), d.unique_keys.size() * 8);
  std::memcpy(inv, d.inverse_indices.data(), n * 4);
  return d.unique_keys.size();
}

// ---- SlabCache ----
int ref_cache_create(uint64_t S, uint32_t W, uint32_t d, uint32_t workers,
                     uint32_t tpw, void** out) {
  return guard([&] {
    hps::SlabCacheConfig c;
    c.slabset_count = S;
    c.slabs_per_set = W;
    c.dimension = d;
    c.worker_pool_size = workers;
    c.tasks_per_worker = tpw;
    *out = new hps::SlabCache(c);
  });
}
void ref_cache_destroy(void* c) { delete static_cast<hps::SlabCache*>(c); }

int ref_cache_query(void* c, const uint64_t* keys, size_t n, float* out,
                    size_t out_len, uint64_t* miss_pos, uint64_t* miss_keys,
                    size_t* n_miss) {
  return guard([&] {
    auto m = static_cast<hps::SlabCache*>(c)->query(
        std::span<const uint64_t>(keys, n), std::span<float>(out, out_len));
    for (size_t i = 0; i < m.size(); ++i) {
      miss_pos[i] = m[i].position;
      miss_keys[i] = m[i].key;
    }
    *n_miss = m.size();
  });
}
int ref_cache_replace(void* c, const uint64_t* keys, size_t n, const float* v,
                      size_t v_len) {
  return guard([&] {
    static_cast<hps::SlabCache*>(c)->replace(std::span<const uint64_t>(keys, n),
                                             std::span<const float>(v, v_len));
  });
}
int ref_cache_update(void* c, const uint64_t* keys, size_t n, const float* v,
                     size_t v_len, size_t* written) {
  return guard([&] {
    *written = static_cast<hps::SlabCache*>(c)->update(
        std::span<const uint64_t>(keys, n), std::span<const float>(v, v_len));
  });
}
size_t ref_cache_dump_all(void* c, uint64_t* out, size_t cap) {
  auto all = static_cast<hps::SlabCache*>(c)->dump_all();
  std::memcpy(out, all.data(), std::min(cap, all.size()) * 8);
  return all.size();
}
uint64_t ref_cache_clock(void* c) {
  return static_cast<hps::SlabCache*>(c)->recency_clock();
}
size_t ref_cache_occupied(void* c) {
  return static_cast<hps::SlabCache*>(c)->occupied();
}
int ref_cache_check(void* c) {
  return guard([&] { static_cast<hps::SlabCache*>(c)->check_invariants(); });
}

// ---- ReferenceCache (the reference's own slot-exact test model) ----
void* ref_model_create(uint64_t S, uint32_t W, uint32_t d) {
  return new hps_test::ReferenceCache(S, W, d);
}
void ref_model_destroy(void* m) { delete static_cast<hps_test::ReferenceCache*>(m); }
void ref_model_query(void* m, const uint64_t* keys, size_t n, float* out,
                     size_t out_len, uint8_t* hit) {
  auto h = static_cast<hps_test::ReferenceCache*>(m)->query(
      std::span<const uint64_t>(keys, n), std::span<float>(out, out_len));
  std::memcpy(hit, h.data(), n);
}
void ref_model_replace(void* m, const uint64_t* keys, size_t n, const float* v,
                       size_t v_len) {
  static_cast<hps_test::ReferenceCache*>(m)->replace(
      std::span<const uint64_t>(keys, n), std::span<const float>(v, v_len));
}
size_t ref_model_update(void* m, const uint64_t* keys, size_t n, const float* v,
                        size_t v_len) {
  return static_cast<hps_test::ReferenceCache*>(m)->update(
      std::span<const uint64_t>(keys, n), std::span<const float>(v, v_len));
}
size_t ref_model_resident(void* m, uint64_t* out, size_t cap) {
  auto r = static_cast<hps_test::ReferenceCache*>(m)->resident_keys();
  std::memcpy(out, r.data(), std::min(cap, r.size()) * 8);
  return r.size();
}
uint64_t ref_model_clock(void* m) {
  return static_cast<hps_test::ReferenceCache*>(m)->clock();
}

// ---- PowerLawSampler ----
int ref_powerlaw_sample(double alpha, uint64_t keyspace, uint64_t permute_seed,
                        uint64_t draw_seed, size_t count, uint64_t* out) {
  return guard([&] {
    hps::PowerLawSpec spec;
    spec.alpha = alpha;
    spec.keyspace = keyspace;
    spec.permute_seed = permute_seed;
    hps::PowerLawSampler s(spec);
    auto v = s.sample(count, draw_seed);
    std::memcpy(out, v.data(), count * 8);
  });
}

// ---- LookupEngine over VDB (+ an empty PDB in a scratch dir) ----
struct RefEngine {
  std::filesystem::path dir;
  std::unique_ptr<hps::PersistentStore> pdb;
  std::unique_ptr<hps::VolatileStore> vdb;
  std::unique_ptr<hps::SlabCache> cache;
  std::unique_ptr<hps::LookupEngine> engine;
  hps::TableId table;
  ~RefEngine() {
    engine.reset();
    cache.reset();
    vdb.reset();
    pdb.reset();
    std::error_code ec;
    std::filesystem::remove_all(dir, ec);
  }
};

int ref_engine_create(uint32_t dim, uint64_t S, uint32_t W, uint32_t workers,
                      double threshold, uint32_t partitions, int use_vdb,
                      const float* default_vec, uint32_t default_len,
                      uint32_t pool, uint32_t async_workers, void** out) {
  return guard([&] {
    auto e = std::make_unique<RefEngine>();
    std::random_device rd;
    e->dir = std::filesystem::temp_directory_path() /
             ("hps-ref-" + std::to_string(rd()) + std::to_string(rd()));
    std::filesystem::create_directories(e->dir);
    e->table = hps::TableId{"t", dim};
    e->pdb = std::make_unique<hps::PersistentStore>(e->dir);
    e->pdb->create_table(e->table);
    e->vdb = std::make_unique<hps::VolatileStore>();
    hps::VolatileTableConfig vc;
    vc.partition_count = partitions;
    vc.overflow_margin = std::size_t(1) << 40;
    e->vdb->register_table(e->table, vc);
    hps::SlabCacheConfig cc;
    cc.slabset_count = S;
    cc.slabs_per_set = W;
    cc.dimension = dim;
    cc.worker_pool_size = workers;
    e->cache = std::make_unique<hps::SlabCache>(cc);
    hps::EngineConfig ec;
    ec.hit_rate_threshold = threshold;
    ec.default_vector.assign(default_vec, default_vec + default_len);
    ec.workspace_pool_size = pool;
    ec.async_worker_count = async_workers;
    ec.volatile_tier_enabled = use_vdb != 0;
    e->engine = std::make_unique<hps::LookupEngine>(
        e->table, *e->cache, e->vdb.get(), *e->pdb, ec);
    *out = e.release();
  });
}
void ref_engine_destroy(void* e) { delete static_cast<RefEngine*>(e); }

int ref_engine_vdb_insert(void* e, const uint64_t* keys, size_t n, const float* v) {
  auto* r = static_cast<RefEngine*>(e);
  return guard([&] {
    r->vdb->insert("t", std::span<const uint64_t>(keys, n),
                   std::span<const float>(v, n * r->table.dimension));
  });
}
int ref_engine_pdb_put(void* e, const uint64_t* keys, size_t n, const float* v) {
  auto* r = static_cast<RefEngine*>(e);
  return guard([&] {
    r->pdb->put("t", std::span<const uint64_t>(keys, n),
                std::span<const float>(v, n * r->table.dimension));
    r->pdb->flush("t");
  });
}
int ref_engine_cache_replace(void* e, const uint64_t* keys, size_t n, const float* v) {
  auto* r = static_cast<RefEngine*>(e);
  return guard([&] {
    r->cache->replace(std::span<const uint64_t>(keys, n),
                      std::span<const float>(v, n * r->table.dimension));
  });
}
// outcome: [sync_branch, unique_count, defaults_returned]; hit rate separate
int ref_engine_lookup(void* e, const uint64_t* keys, size_t n, float* out,
                      uint8_t* flags, uint64_t* outcome, double* hit_rate) {
  auto* r = static_cast<RefEngine*>(e);
  return guard([&] {
    hps::LookupOutcome o;
    auto res = r->engine->lookup(std::span<const uint64_t>(keys, n), &o);
    std::memcpy(out, res.vectors.data(), res.vectors.size() * 4);
    std::memcpy(flags, res.miss_flags.data(), n);
    outcome[0] = o.sync_branch;
    outcome[1] = o.unique_count;
    outcome[2] = o.defaults_returned;
    *hit_rate = o.unique_hit_rate;
  });
}
void ref_engine_drain(void* e) {
  auto* r = static_cast<RefEngine*>(e);
  r->engine->drain_async();
  r->vdb->drain();
}
// stats: 12 u64 in EngineStatsSnapshot declaration order
void ref_engine_stats(void* e, uint64_t* s) {
  auto st = static_cast<RefEngine*>(e)->engine->stats();
  uint64_t v[12] = {st.queries,        st.queried_keys,  st.unique_keys,
                    st.cache_hits,     st.cache_misses,  st.sync_batches,
                    st.async_batches,  st.defaults_returned, st.vdb_hits,
                    st.pdb_hits,       st.tier_missing,  st.async_faults};
  std::memcpy(s, v, sizeof(v));
}
void* ref_engine_cache(void* e) { return static_cast<RefEngine*>(e)->cache.get(); }

unsigned ref_hw_threads() { return std::thread::hardware_concurrency(); }

// hps::encode_response_frame(Opcode::Lookup, ...) (wire.cpp:174-188) with the
// miss bitmap built as handle_frame does (server.cpp:284-294); returns the
// frame length (copies min(len, cap) bytes).
size_t ref_wire_lookup_frame(const float* rows, const uint8_t* flags, uint32_t count, uint32_t dim,
                             uint8_t* out, size_t cap) {
  hps::WireResponse resp;
  resp.status = hps::Status::Ok;
  resp.count = count;
  resp.dim = dim;
  resp.vectors.assign(rows, rows + size_t(count) * dim);
  resp.miss_bitmap.assign((size_t(count) + 7) / 8, 0);
  for (uint32_t i = 0; i < count; ++i)
    if (flags[i]) hps::set_miss_bit(resp.miss_bitmap, i);
  const auto f = hps::encode_response_frame(hps::Opcode::Lookup, resp);
  std::memcpy(out, f.data(), std::min(cap, f.size()));
  return f.size();
}

// ---- PersistentStore (the f4 row's parity partner) ----
int ref_pdb_open(const char* root, void** out) {
  return guard([&] { *out = new hps::PersistentStore(root); });
}
void ref_pdb_destroy(void* p) { delete static_cast<hps::PersistentStore*>(p); }
int ref_pdb_create_table(void* p, const char* name, uint32_t dim) {
  return guard([&] { static_cast<hps::PersistentStore*>(p)->create_table({name, dim}); });
}
int ref_pdb_put(void* p, const char* name, const uint64_t* keys, size_t n, const float* v) {
  return guard([&] {
    auto* s = static_cast<hps::PersistentStore*>(p);
    const uint32_t d = s->table(name).dimension;
    s->put(name, std::span<const uint64_t>(keys, n), std::span<const float>(v, n * d));
  });
}
int ref_pdb_flush(void* p, const char* name) {
  return guard([&] { static_cast<hps::PersistentStore*>(p)->flush(name); });
}
int ref_pdb_compact(void* p, const char* name) {
  return guard([&] { static_cast<hps::PersistentStore*>(p)->compact(name); });
}
int ref_pdb_get(void* p, const char* name, const uint64_t* keys, size_t n, uint64_t* fk,
                float* fv, size_t* nf, uint64_t* mk, size_t* nm) {
  return guard([&] {
    auto r = static_cast<hps::PersistentStore*>(p)->get(name, std::span<const uint64_t>(keys, n));
    std::copy(r.found_keys.begin(), r.found_keys.end(), fk);
    std::copy(r.found_vectors.begin(), r.found_vectors.end(), fv);
    std::copy(r.missing_keys.begin(), r.missing_keys.end(), mk);
    *nf = r.found_keys.size();
    *nm = r.missing_keys.size();
  });
}
size_t ref_pdb_segment_count(void* p, const char* name) {
  return static_cast<hps::PersistentStore*>(p)->segment_count(name);
}
size_t ref_pdb_key_count(void* p, const char* name) {
  return static_cast<hps::PersistentStore*>(p)->key_count(name);
}

}  // extern "C"
