/*
 * hps_b200.h -- C ABI of the B200-native HPS lookup path.
 *
 * This is the drop-in boundary: plain pointers and sizes, no CUDA or torch
 * types in the signatures (streams are passed as `void*` holding a
 * cudaStream_t; NULL = the legacy default stream). Every entry point names the
 * reference interface it replaces (file:line under /root/reference/proj).
 * The C++ shim in include/hps_b200/slab_cache.hpp re-exposes the
 * reference's hps::SlabCache API on top of these calls, and
 * paper_2210_08804_b200/__init__.py binds them with ctypes.
 *
 * Status codes: 0 OK, 1 INVALID_ARGUMENT (reference:
 * std::invalid_argument), 2 INTERNAL / CUDA error, 3 OUT_OF_MEMORY,
 * 4 LOGIC_ERROR (reference: std::logic_error from check_invariants),
 * 5 TIER_FAULT (reference: hps::TierFault). hps_last_error() returns the
 * thread-local message of the last failing call on this thread.
 *
 * Memory modes: HPS_MEM_HOST -- every key / row / output pointer is host
 * memory; the call is synchronous (the reference's drop-in semantics).
 * HPS_MEM_DEVICE -- key / row / output pointers are device memory on the
 * object's GPU; work is ordered after `stream` and results are ready when
 * `stream` reaches the point of the call. Calls that must report a count
 * (query misses, update writes) synchronise before returning.
 *
 * Thread safety: every object serialises its own calls (one mutex and one
 * CUDA stream per cache), matching the reference's per-call atomicity
 * ("safe for arbitrary concurrent calls").
 */
#ifndef HPS_B200_H_
#define HPS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_OK 0
#define HPS_INVALID_ARGUMENT 1
#define HPS_INTERNAL 2
#define HPS_OUT_OF_MEMORY 3
#define HPS_LOGIC_ERROR 4
#define HPS_TIER_FAULT 5

#define HPS_MEM_HOST 0
#define HPS_MEM_DEVICE 1

typedef struct hps_cache hps_cache;
typedef struct hps_vdb hps_vdb;
typedef struct hps_engine hps_engine;
typedef struct hps_multi hps_multi;
typedef struct hps_pdb hps_pdb;
typedef struct hps_replicas hps_replicas;
typedef struct hps_peer_group hps_peer_group;

/* ---- vocabulary ------------------------------------------------------- */

/* Thread-local message of the last failing call. */
const char* hps_last_error(void);

/* Number of CUDA kernels this library has launched in this process
 * (diagnostic; bench.py reports it for the timed region). */
uint64_t hps_kernel_launch_count(void);

/* XXH64; replaces hps::xxh64 / xxh64_key (xxhash64.hpp:60-124). */
uint64_t hps_xxh64(const void* data, size_t len, uint64_t seed);
uint64_t hps_xxh64_key(uint64_t key, uint64_t seed);
/* replaces SlabCache::slabset_of / first_slab_of (slab_cache.cpp:60-67) */
uint64_t hps_slabset_of(uint64_t key, uint64_t slabset_count);
uint32_t hps_first_slab_of(uint64_t key, uint32_t slabs_per_set);
/* replaces hps::partition_of (volatile_store.cpp:10-13) */
uint32_t hps_partition_of(uint64_t key, uint32_t partition_count);

/* GPU dedup; replaces hps::dedup_keys (types.cpp:20-34). Writes the unique
 * keys in first-occurrence order and the u32 inverse index; *n_unique gets
 * the unique count. `unique_out` must hold n keys. */
int hps_dedup_keys(int device, const uint64_t* keys, size_t n, uint64_t* unique_out,
                   uint32_t* inverse_out, size_t* n_unique, int mem, void* stream);

/* ---- embedding cache (replaces hps::SlabCache, slab_cache.hpp:41-116) ---- */

/* Mirrors SlabCacheConfig (slab_cache.hpp:27-34). worker_pool_size and
 * tasks_per_worker are validated like the reference (worker_pool_size == 0
 * is an error) and map to keys-per-warp on the device. */
typedef struct {
  uint64_t slabset_count;
  uint32_t slabs_per_set;
  uint32_t dimension;
  uint32_t worker_pool_size;
  uint32_t tasks_per_worker;
} hps_cache_config;

typedef struct {
  uint32_t dimension;
  uint32_t slabs_per_set;
  uint64_t slabset_count;
  uint64_t capacity;
  uint64_t occupied;
  uint64_t recency_clock;
  int device;
  int reserved;
} hps_cache_info;

/* replaces SlabCache::SlabCache (slab_cache.cpp:17-41) */
int hps_cache_create(const hps_cache_config* config, int device, hps_cache** out);
/* A cache in the same CACHE GROUP as `share_with`: same device, one CUDA
 * stream for all members (the tables of one model), so a multi-table lookup
 * (hps_multi_*) can run every member in one launch. Otherwise identical to
 * hps_cache_create. */
int hps_cache_create_shared(const hps_cache_config* config, int device, hps_cache* share_with,
                            hps_cache** out);
/* replaces SlabCache::~SlabCache (slab_cache.cpp:43-52) */
int hps_cache_destroy(hps_cache* cache);
int hps_cache_get_info(hps_cache* cache, hps_cache_info* out);
/* Raw cudaStream_t of the cache's own stream (for event-based chaining). */
void* hps_cache_stream(hps_cache* cache);

/* replaces SlabCache::query (slab_cache.cpp:69-91). Bumps the recency clock
 * once, even for n == 0 and before the size check. Hit rows are copied into
 * out (n * dimension floats, out_len must equal that), miss rows are left
 * untouched. Misses are reported in ascending position order into
 * miss_positions / miss_keys (each must hold n entries; same memory kind as
 * keys) and their count into *n_miss (host). */
int hps_cache_query(hps_cache* cache, const uint64_t* keys, size_t n, float* out,
                    size_t out_len, uint32_t* miss_positions, uint64_t* miss_keys,
                    size_t* n_miss, int mem, void* stream);

/* Lookup-level query, device pointers only: the hot path of
 * hps_engine_lookup without the tier logic (LookupEngine::lookup's dedup ->
 * query -> expand, lookup_engine.cpp:131-153,194-203). Bumps the recency
 * clock once; out (n * dim) gets every position's row -- the cached row on
 * a hit, default_row (dim floats, device) on a miss; miss_flags[n] = 1 on a
 * miss; miss_keys / miss_firsts (capacity n each) get the unique missing
 * keys and their first-occurrence positions, one entry per key in claim
 * order -- sorting by position gives the reference's miss order;
 * counts[2] = {unique hits, unique misses} of this call (so
 * h = 1 - counts[1] / (counts[0] + counts[1]), and counts[1] entries are
 * valid). Stream-ordered: returns without synchronising. */
int hps_cache_lookup_device(hps_cache* cache, const uint64_t* keys, size_t n, float* out,
                            uint8_t* miss_flags, const float* default_row,
                            uint64_t* miss_keys, uint32_t* miss_firsts, uint64_t* counts,
                            void* stream);

/* Diagnostic: record these cudaEvent_t (as void*) on the cache stream right
 * before / after the probe kernel of subsequent hps_cache_lookup_device
 * calls; NULL disables. Used by bench.py to time the dominant kernel. */
int hps_cache_set_profile_events(hps_cache* cache, void* start_event, void* end_event);

/* CUDA graph capture through this library's runtime (device-mode calls
 * enqueued on `stream` between begin and end become graph nodes; no host
 * synchronising calls may be made in between, and a cache captured on one
 * thread must not be used by other threads until end_capture). end_capture
 * instantiates the graph into *graph_exec (an opaque handle of this
 * library). Captured lookups are REPLAYABLE: each hps_graph_launch writes
 * the caches' current recency clock and lookup-view uses into device words
 * the graph's lookups read their stamps and view generations relative to
 * (one small kernel before the graph), then advances them by what one replay
 * consumes -- a replay is exactly the same lookups issued again (fresh
 * stamps in stream order, unique hits counted). Replays
 * must go through hps_graph_launch, which also orders each cache's own
 * stream before and after the graph; destroy a graph before its caches. */
int hps_stream_begin_capture(void* stream);
int hps_stream_end_capture(void* stream, void** graph_exec);
int hps_graph_launch(void* graph_exec, void* stream);
int hps_graph_destroy(void* graph_exec);
/* Records the cudaEvent_t `event` on `stream`; inside a capture as an
 * external record node (its timestamp stays readable after each launch of
 * the graph -- bench.py's timed region is bracketed this way). */
int hps_event_record(void* event, void* stream);

/* replaces SlabCache::replace (slab_cache.cpp:93-107). Rejects a wrong
 * vector size or duplicate keys before any mutation. */
int hps_cache_replace(hps_cache* cache, const uint64_t* keys, size_t n,
                      const float* vectors, size_t vectors_len, int mem, void* stream);

/* Stream-ordered SlabCache::replace on device pointers for keys the caller
 * guarantees DISTINCT (the engine's miss fill: unique misses): no duplicate
 * check and no host synchronisation; same placement, recency and eviction
 * as hps_cache_replace. */
int hps_cache_replace_device_async(hps_cache* cache, const uint64_t* keys, size_t n,
                                   const float* vectors, size_t vectors_len, void* stream);

/* B200 extension (SURVEY §7 "Hard parts": the opt-in relaxed mode). mode
 * HPS_REPLACE_EXACT (default): every replace is slot-exact with the
 * reference -- a set's keys applied in input order (slab_cache.cpp:131-142,
 * 261-326). HPS_REPLACE_RELAXED: replaces whose keys are known distinct
 * (host-mode hps_cache_replace after its CPU duplicate check,
 * hps_cache_replace_device_async, the engine's miss fills) apply every key
 * at once, winning slots with atomicOr on the slab mask / atomicCAS on the
 * slot counter; same probe / insert / LRU rules, but same-set keys race, so
 * slots and the survivors of an over-subscribed set may differ from the
 * exact mode, and a key whose set has no slot left that this call has not
 * already stamped is not admitted (counted). A device-mode hps_cache_replace
 * (which must reject duplicates) stays exact. W > 4 stays exact. */
#define HPS_REPLACE_EXACT 0
#define HPS_REPLACE_RELAXED 1
int hps_cache_set_replace_mode(hps_cache* cache, int mode);
/* mode and the number of keys the relaxed mode has not admitted so far
 * (either may be NULL; reading `dropped` synchronises the cache stream) */
int hps_cache_get_replace_mode(hps_cache* cache, int* mode, uint64_t* dropped);

/* replaces SlabCache::update (slab_cache.cpp:109-125). *written = number of
 * positions whose key was resident (duplicates count every time; the last
 * occurrence's row wins). */
int hps_cache_update(hps_cache* cache, const uint64_t* keys, size_t n,
                     const float* vectors, size_t vectors_len, size_t* written,
                     int mem, void* stream);

/* Stream-ordered SlabCache::update on device pointers (the online-training
 * path: no host synchronisation). *written (device u64, may be NULL) gets the
 * number of positions whose key was resident once `stream` reaches the call. */
int hps_cache_update_device(hps_cache* cache, const uint64_t* keys, size_t n,
                            const float* vectors, size_t vectors_len, uint64_t* written,
                            void* stream);

/* replaces DumpCursor::next (slab_cache.cpp:367-394) over the slabset range
 * [set_begin, set_end): resident keys in set, slab, slot order into the host
 * buffer out (capacity cap). *n_out = number of resident keys in the range
 * (may exceed cap; then only cap are written). */
int hps_cache_dump(hps_cache* cache, uint64_t set_begin, uint64_t set_end,
                   uint64_t* out, size_t cap, size_t* n_out);

/* Stream-ordered DumpCursor pass into DEVICE memory (the GPU refresh path):
 * resident keys of slabsets [set_begin, set_end) in set, slab, slot order
 * into `out` (capacity (set_end - set_begin) * slabs_per_set * 32 keys) and
 * their count into *n_out (device u64). */
int hps_cache_dump_device(hps_cache* cache, uint64_t set_begin, uint64_t set_end, uint64_t* out,
                          uint64_t* n_out, void* stream);

/* replaces SlabCache::check_invariants (slab_cache.cpp:407-442); returns
 * HPS_LOGIC_ERROR with the reference's message on violation. */
int hps_cache_check_invariants(hps_cache* cache);

/* Test/diagnostic: copy the whole device table to host buffers (any may be
 * NULL): keys/counters hold capacity entries, masks S*W, rows capacity*d. */
int hps_cache_export_state(hps_cache* cache, uint64_t* keys, uint64_t* counters,
                           uint32_t* masks, float* rows);

/* Diagnostic (HPSB_TRACE=1 in the environment): per-call phase timeline of
 * the lookup kernel, 8 u64 per call (see lookup_kernels.cu) for the last
 * calls in a ring of 4096; copies up to cap values and resets the ring. */
int hps_cache_debug_trace(hps_cache* cache, uint64_t* out, size_t cap, uint64_t* n_calls);

/* ---- volatile DB (replaces hps::VolatileStore, volatile_store.hpp:45-137) ---- */

int hps_vdb_create(uint32_t lookup_threads, hps_vdb** out);
int hps_vdb_destroy(hps_vdb* vdb);
/* replaces register_table (volatile_store.cpp:25-51) */
int hps_vdb_register_table(hps_vdb* vdb, const char* name, uint32_t dimension,
                           uint32_t partition_count, uint64_t overflow_margin);
int hps_vdb_has_table(hps_vdb* vdb, const char* name);
/* replaces insert (volatile_store.cpp:113-152); evicted keys (if not NULL,
 * capacity evicted_cap) and their count. */
int hps_vdb_insert(hps_vdb* vdb, const char* name, const uint64_t* keys, size_t n,
                   const float* vectors, size_t vectors_len, uint64_t* evicted,
                   size_t evicted_cap, size_t* n_evicted);
/* replaces insert_async (volatile_store.cpp:174-188) */
int hps_vdb_insert_async(hps_vdb* vdb, const char* name, const uint64_t* keys,
                         size_t n, const float* vectors, size_t vectors_len);
/* replaces lookup (volatile_store.cpp:82-112): found keys / rows in input
 * order, missing keys in input order; each output holds n entries (rows:
 * n * dim). */
int hps_vdb_lookup(hps_vdb* vdb, const char* name, const uint64_t* keys, size_t n,
                   uint64_t* found_keys, float* found_vectors, size_t* n_found,
                   uint64_t* missing_keys, size_t* n_missing);
/* replaces drain (volatile_store.cpp:250-253) */
int hps_vdb_drain(hps_vdb* vdb);
/* replaces table_size / partition_size / table_clock / last_access */
int hps_vdb_table_size(hps_vdb* vdb, const char* name, uint64_t* out);
int hps_vdb_partition_size(hps_vdb* vdb, const char* name, uint32_t partition,
                           uint64_t* out);
int hps_vdb_table_clock(hps_vdb* vdb, const char* name, uint64_t* out);
/* *found = 0 when the key is absent */
int hps_vdb_last_access(hps_vdb* vdb, const char* name, uint64_t key, uint64_t* out,
                        int* found);
/* replaces evict (volatile_store.cpp:190-199) */
int hps_vdb_evict(hps_vdb* vdb, const char* name, uint32_t partition,
                  uint64_t* evicted, size_t evicted_cap, size_t* n_evicted);
/* The full evicted-key list of this thread's last hps_vdb_insert /
 * hps_vdb_evict (for callers whose evicted_cap was too small): copies up to
 * cap keys, *n = the list's length. */
int hps_vdb_last_evicted(uint64_t* out, size_t cap, size_t* n);
/* the table's registered dimension (TableId::dimension) */
int hps_vdb_dimension(hps_vdb* vdb, const char* name, uint32_t* out);
/* replaces partition_count (volatile_store.cpp:59-61) */
int hps_vdb_partition_count(hps_vdb* vdb, const char* name, uint32_t* out);
/* replaces keys (volatile_store.cpp:293-303): every resident key, partition
 * by partition; copies up to cap keys (out may be NULL), *n = the count. */
int hps_vdb_keys(hps_vdb* vdb, const char* name, uint64_t* out, size_t cap, size_t* n);

/* ---- cold tier callback (stands in for hps::PersistentStore::get,
 *      persistent_store.cpp:405-439, which stays CPU code) ---- */
typedef int (*hps_cold_fetch_fn)(void* ctx, const uint64_t* keys, size_t n,
                                 uint64_t* found_keys, float* found_vectors,
                                 size_t* n_found, uint64_t* missing_keys,
                                 size_t* n_missing);

/* ---- batched cold reads over the reference's persistent store files
 *      (replaces PersistentStore::get,
 *      persistent_store.cpp:405-439, one pread per key, for the read path).
 *      A read-only reader of <root>/<escaped table>/{MANIFEST, seg-<n>.log}
 *      (persistent_store.hpp:5-15): the newest-record-wins index is rebuilt
 *      as the reference's open does (persistent_store.cpp:229-268), the
 *      segments are memory-mapped, and a batch's probes and row copies fan
 *      out over `threads` host threads (0 = all cores). Records still in the
 *      writer's unflushed tail are invisible until flushed + refreshed. ---- */
int hps_pdb_open(const char* root, uint32_t threads, hps_pdb** out);
int hps_pdb_destroy(hps_pdb* pdb);
/* indexes the table (HPS_INVALID_ARGUMENT "persistent store has no table
 * named <t>" when absent; HPS_TIER_FAULT for a malformed MANIFEST) */
int hps_pdb_attach(hps_pdb* pdb, const char* table);
/* picks up flushed appends, new segments and compactions */
int hps_pdb_refresh(hps_pdb* pdb, const char* table);
int hps_pdb_info(hps_pdb* pdb, const char* table, uint32_t* dimension, uint64_t* keys,
                 uint64_t* segments);
/* PersistentStore::get: found keys / rows and missing keys in input order;
 * each output holds n entries (rows: n * dim) */
int hps_pdb_get(hps_pdb* pdb, const char* table, const uint64_t* keys, size_t n,
                uint64_t* found_keys, float* found_vectors, size_t* n_found,
                uint64_t* missing_keys, size_t* n_missing);
/* the engine's cold tier over one table: pass hps_pdb_cold_fetch as `cold`
 * and the context from hps_pdb_table_ctx (attaches the table; owned by pdb)
 * as `cold_ctx` to hps_engine_create / hps_tier_fetch / hps_refresh_cache */
int hps_pdb_table_ctx(hps_pdb* pdb, const char* table, void** ctx);
int hps_pdb_cold_fetch(void* ctx, const uint64_t* keys, size_t n, uint64_t* found_keys,
                       float* found_vectors, size_t* n_found, uint64_t* missing_keys,
                       size_t* n_missing);

/* replaces hps::tier_fetch (lookup_engine.cpp:50-89): VDB first (if vdb and
 * the table are present), then the cold tier for the rest; cold hits are
 * promoted to the VDB asynchronously. counters (may be NULL) receives
 * {vdb_hits, cold_hits, missing}. */
int hps_tier_fetch(hps_vdb* vdb, const char* table, uint32_t dimension,
                   hps_cold_fetch_fn cold, void* cold_ctx, const uint64_t* keys,
                   size_t n, uint64_t* found_keys, float* found_vectors,
                   size_t* n_found, uint64_t* missing_keys, size_t* n_missing,
                   uint64_t* counters);

/* replaces hps::refresh_cache (refresh_engine.cpp:5-22): every resident key,
 * in dump order and batches of dump_batch, re-fetched from the tiers (VDB
 * first, then the cold tier) and written back with the non-admitting update;
 * *refreshed = rows rewritten, unresolved (capacity unresolved_cap, may be
 * NULL) = resident keys absent from every tier, *n_unresolved their count.
 * The host tier fetch of one batch overlaps the device update of the last. */
int hps_refresh_cache(hps_cache* cache, hps_vdb* vdb, const char* table,
                      hps_cold_fetch_fn cold, void* cold_ctx, size_t dump_batch,
                      uint64_t* refreshed, uint64_t* unresolved, size_t unresolved_cap,
                      size_t* n_unresolved);

/* ---- lookup engine (replaces hps::LookupEngine, lookup_engine.hpp:152-196) ---- */

/* Mirrors EngineConfig (lookup_engine.hpp:29-37). */
typedef struct {
  double hit_rate_threshold;
  const float* default_vector; /* may be NULL = zeros; padded / cut to dim */
  uint32_t default_vector_len;
  uint32_t workspace_pool_size;
  uint32_t async_worker_count;
  int volatile_tier_enabled;
  uint32_t max_batch; /* largest accepted batch in keys; larger calls fail with
                         HPS_INVALID_ARGUMENT (0 = no limit below 2^32) */
} hps_engine_config;

/* Mirrors LookupOutcome (lookup_engine.hpp:145-150). */
typedef struct {
  int sync_branch;
  double unique_hit_rate;
  uint64_t unique_count;
  uint64_t defaults_returned;
} hps_lookup_outcome;

/* Mirrors EngineStatsSnapshot (lookup_engine.hpp:129-142), same order. */
typedef struct {
  uint64_t queries, queried_keys, unique_keys, cache_hits, cache_misses,
      sync_batches, async_batches, defaults_returned, vdb_hits, pdb_hits,
      tier_missing, async_faults;
} hps_engine_stats;

/* replaces LookupEngine::LookupEngine (lookup_engine.cpp:91-117); vdb and
 * cold may be NULL. The engine keeps pointers to cache / vdb, which must
 * outlive it. */
int hps_engine_create(const char* table, uint32_t dimension, hps_cache* cache,
                      hps_vdb* vdb, hps_cold_fetch_fn cold, void* cold_ctx,
                      const hps_engine_config* config, hps_engine** out);
int hps_engine_destroy(hps_engine* engine);

/* replaces LookupEngine::lookup (lookup_engine.cpp:130-241). out holds
 * n * dimension floats (out_len must equal that), miss_flags n bytes;
 * outcome may be NULL. */
int hps_engine_lookup(hps_engine* engine, const uint64_t* keys, size_t n, float* out,
                      size_t out_len, uint8_t* miss_flags, hps_lookup_outcome* outcome,
                      int mem, void* stream);

/* Several tables in one call (the reference's caller -- e.g. Node::lookup
 * per table, server.cpp:198-202 -- loops over tables): engines[t] looks up
 * keys[t][0..n[t]) into out[t] / miss_flags[t] with exactly the semantics of
 * hps_engine_lookup; all tables' device work is enqueued before the first
 * host wait, so the lookups overlap on the GPU. outcomes may be NULL. */
int hps_engine_lookup_multi(hps_engine* const* engines, size_t count,
                            const uint64_t* const* keys, const size_t* n, float* const* out,
                            uint8_t* const* miss_flags, hps_lookup_outcome* outcomes, int mem);

/* Multi-table lookup over engines whose caches form one cache group
 * (hps_cache_create_shared), one engine per table, batches of up to
 * max_batch keys per table: ONE H2D, ONE kernel launch for every table, one
 * D2H of all results, one host wait -- then each table's hit-rate switch and
 * miss path exactly as hps_engine_lookup (host buffers). */
int hps_multi_create(hps_engine* const* engines, size_t count, size_t max_batch,
                     hps_multi** out);
int hps_multi_destroy(hps_multi* multi);
int hps_multi_lookup(hps_multi* multi, const uint64_t* const* keys, const size_t* n,
                     float* const* out, uint8_t* const* miss_flags, hps_lookup_outcome* outcomes);

/* The paper's concurrent deployment in one process (no
 * reference counterpart -- the reference is single-GPU-less): engines[r] is
 * replica r -- its own cache on its own GPU -- and the engines share ONE host
 * VDB (create them all over the same hps_vdb). hps_replicas_lookup hands
 * replica r the batch keys[r][0..n[r]) on its own persistent host thread
 * (exactly hps_engine_lookup's semantics, NULL stream in device mode) and
 * returns when every replica is done; no collective. */
int hps_replicas_create(hps_engine* const* engines, size_t count, hps_replicas** out);
int hps_replicas_destroy(hps_replicas* group);
int hps_replicas_lookup(hps_replicas* group, const uint64_t* const* keys, const size_t* n,
                        float* const* out, uint8_t* const* miss_flags,
                        hps_lookup_outcome* outcomes, int mem);

/* B200 extension: allocates every workspace (device + pinned staging) and
 * the cache's replace scratch for batches of up to max_keys now, so no lookup
 * pays a first-use allocation (also done at creation when
 * hps_engine_config.max_batch is set). Call before serving. */
int hps_engine_reserve(hps_engine* engine, size_t max_keys);
/* replaces drain_async (lookup_engine.cpp:286-289) */
int hps_engine_drain_async(hps_engine* engine);
/* replaces stats (lookup_engine.cpp:291-294) */
int hps_engine_get_stats(hps_engine* engine, hps_engine_stats* out);
/* replaces WorkspacePool::size / outstanding / peak_outstanding */
int hps_engine_pool_info(hps_engine* engine, uint64_t* size, uint64_t* outstanding,
                         uint64_t* peak_outstanding);

/* ---- key-hash-sharded mode (tables larger than one GPU's HBM; SURVEY
 *      §8e -- no reference counterpart: the reference is single-process and
 *      the paper deploys one replica per GPU). Rank r of G owns
 *      the keys with hps_shard_of(key, G) == r; a lookup routes keys to their
 *      owners (NCCL all-to-all in paper_2210_08804_b200/sharded.py), each
 *      owner runs hps_cache_lookup_device on its shard, and the rows come
 *      back the same way. All pointers are device memory on `device`. ---- */
uint32_t hps_shard_of(uint64_t key, uint32_t world);
/* counts[world] (u64) = keys per owner */
int hps_shard_count(int device, const uint64_t* keys, size_t n, uint32_t world, uint64_t* counts,
                    void* stream);
/* cursor[world] = each owner's segment start in send_keys / send_pos (advanced
 * by the call); send_pos[j] = the original position of send_keys[j] */
int hps_shard_scatter(int device, const uint64_t* keys, size_t n, uint32_t world, uint64_t* cursor,
                      uint64_t* send_keys, uint32_t* send_pos, void* stream);
/* out[send_pos[j]] = rows[j] (dim floats), flags_out[send_pos[j]] = flags_in[j]
 * (flags may be NULL) */
int hps_shard_unroute(int device, size_t m, uint32_t dim, const uint32_t* send_pos,
                      const float* rows, const uint8_t* flags_in, float* out, uint8_t* flags_out,
                      void* stream);

/* ---- key-hash-sharded lookup over PEER MEMORY (the B200-native
 *      alternative to the two all-to-alls; no reference counterpart). Every
 *      rank exports its shard cache (CUDA IPC handles of its probe
 *      structures, rows and a miss inbox; the caller ships the blob to the
 *      other ranks over any transport), then maps every rank's shard. A
 *      lookup is ONE kernel: each key's owner shard is probed through mapped
 *      (NVLink peer) memory, the owner's counter stamped, its row copied
 *      straight into `out`; misses get default_row + flag and are appended
 *      to the owner's inbox. Owners admit their inbox keys between lookup
 *      phases (hps_cache_peer_drain, then a fetch + replace of their own);
 *      no peer may look up while an owner mutates its shard. Recency: while
 *      exported, a shard's clock lives in device memory; every lookup call
 *      ticks each owner's clock once and stamps that owner's hits with it,
 *      and a drain reads it back for the owner's replaces (use an exported
 *      shard only through its peer group). ---- */
size_t hps_peer_blob_size(void);
/* inbox_cap: miss keys the inbox holds between drains (first export only) */
int hps_cache_peer_export(hps_cache* cache, uint64_t inbox_cap, void* blob, size_t blob_cap,
                          size_t* blob_len);
/* blobs: world blobs of blob_len bytes each, rank order; self = this rank's cache */
int hps_peer_group_create(hps_cache* self, uint32_t rank, uint32_t world, const void* blobs,
                          size_t blob_len, hps_peer_group** out);
int hps_peer_group_destroy(hps_peer_group* group);
/* device pointers: keys[n], out[n * dim], miss_flags[n], default_row[dim] */
int hps_peer_lookup_device(hps_peer_group* group, const uint64_t* keys, size_t n, float* out,
                           uint8_t* miss_flags, const float* default_row, void* stream);
/* this shard's inbox: up to cap keys into keys_out (host), *n_appended = keys
 * appended since the last drain (beyond the inbox capacity they were
 * dropped); empties the inbox */
int hps_cache_peer_drain(hps_cache* cache, uint64_t* keys_out, size_t cap, size_t* n_appended);

/* ---- wire LOOKUP response frame (replaces encode_response_frame for
 *      Opcode::Lookup, wire.cpp:174-188; layout wire.hpp:18-21, byte-exact:
 *      [u32 body_len][u8 0][u32 count][u32 dim][count*dim f32][ceil(count/8)
 *      miss bitmap, bit i%8 of byte i/8]). rows / miss_flags are the lookup's
 *      output (HPS_MEM_HOST or, with HPS_MEM_DEVICE, device pointers on
 *      `device`: the bitmap is packed on the GPU and rows + bitmap are copied
 *      straight into `frame`, which should be pinned). frame = NULL queries
 *      the size. Synchronous: the frame is complete on return. ---- */
int hps_wire_lookup_frame(int device, const float* rows, const uint8_t* miss_flags,
                          uint32_t count, uint32_t dim, int mem, uint8_t* frame, size_t cap,
                          size_t* frame_len, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HPS_B200_H_ */
