// capi.cpp -- extern "C" boundary (include/hps_b200.h). Every entry point
// catches, maps the exception to a status code and stores the message in a
// thread-local for hps_last_error().
#include "hps_b200.h"

#include <algorithm>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cstring>

#include "device_cache.hpp"
#include "peer.hpp"
#include "engine.hpp"
#include "segment_store.hpp"
#include "volatile_store.hpp"

struct hps_cache {
  std::unique_ptr<hpsb::DeviceCache> impl;
};
struct hps_peer_group {
  std::unique_ptr<hpsb::PeerGroup> impl;
};
struct hps_vdb {
  std::unique_ptr<hpsb::VolatileStore> impl;
};
struct hps_pdb {
  std::unique_ptr<hpsb::SegmentStore> impl;
  std::mutex mu;
  // cold-callback contexts handed out by hps_pdb_table_ctx (stable addresses)
  std::map<std::string, std::unique_ptr<std::pair<hps_pdb*, std::string>>> ctx;
};
struct hps_engine {
  std::unique_ptr<hpsb::LookupEngine> impl;
};
struct hps_replicas {
  std::unique_ptr<hpsb::ReplicaGroup> impl;
};
struct hps_multi {
  std::unique_ptr<hpsb::MultiLookup> impl;
};
// A captured graph and what each of its caches consumes per replay.
struct hps_graph {
  cudaGraphExec_t exec = nullptr;
  std::vector<hpsb::GraphCacheUse> uses;
};

namespace {
thread_local std::string g_error;
// keys evicted by this thread's last hps_vdb_insert / hps_vdb_evict
thread_local std::vector<uint64_t> g_evicted;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return HPS_OK;
  } catch (const hpsb::Error& e) {
    g_error = e.what();
    return e.code();
  } catch (const std::bad_alloc& e) {
    g_error = e.what();
    return HPS_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_error = e.what();
    return HPS_INTERNAL;
  } catch (...) {
    g_error = "unknown error";
    return HPS_INTERNAL;
  }
}

void need(bool ok, const char* what) {
  if (!ok) throw hpsb::invalid_argument(what);
}

// NULL = the legacy default stream: device-mode work is ordered after it
// (and the caller's later default-stream work after ours).
inline cudaStream_t as_stream(void* s) {
  return s ? static_cast<cudaStream_t>(s) : cudaStreamLegacy;
}

// Process-wide per-device context for the stateless dedup entry point.
struct DedupContext {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  hpsb::DeviceBuffer dbuf;
  hpsb::PinnedBuffer hbuf;
  hpsb::ScanState scan;
  uint32_t epoch = 0;
  uint64_t cap = 0;
  void* last_base = nullptr;
};
std::mutex g_dedup_mu;
std::map<int, std::unique_ptr<DedupContext>> g_dedup;

DedupContext& dedup_ctx(int device) {
  std::lock_guard<std::mutex> lk(g_dedup_mu);
  auto& p = g_dedup[device];
  if (!p) {
    p = std::make_unique<DedupContext>();
    hpsb::DeviceGuard g(device);
    HPSB_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
  }
  return *p;
}
}  // namespace

extern "C" {

const char* hps_last_error(void) { return g_error.c_str(); }

uint64_t hps_kernel_launch_count(void) { return hpsb::launch_count(); }

uint64_t hps_xxh64_key(uint64_t key, uint64_t seed) { return hpsb::xxh64_key(key, seed); }

uint64_t hps_xxh64(const void* input, size_t len, uint64_t seed) {
  // general byte-string XXH64 (xxhash64.hpp:60-114)
  using namespace hpsb;
  const unsigned char* p = static_cast<const unsigned char*>(input);
  const unsigned char* end = p + len;
  auto rd64 = [](const unsigned char* q) {
    uint64_t v;
    std::memcpy(&v, q, 8);
    return v;
  };
  auto rd32 = [](const unsigned char* q) {
    uint32_t v;
    std::memcpy(&v, q, 4);
    return v;
  };
  auto round1 = [](uint64_t acc, uint64_t lane) { return rotl64(acc + lane * kP2, 31) * kP1; };
  uint64_t h;
  if (len >= 32) {
    uint64_t v1 = seed + kP1 + kP2, v2 = seed + kP2, v3 = seed, v4 = seed - kP1;
    const unsigned char* limit = end - 32;
    do {
      v1 = round1(v1, rd64(p));
      v2 = round1(v2, rd64(p + 8));
      v3 = round1(v3, rd64(p + 16));
      v4 = round1(v4, rd64(p + 24));
      p += 32;
    } while (p <= limit);
    h = rotl64(v1, 1) + rotl64(v2, 7) + rotl64(v3, 12) + rotl64(v4, 18);
    for (uint64_t v : {v1, v2, v3, v4}) {
      h ^= round1(0, v);
      h = h * kP1 + kP4;
    }
  } else {
    h = seed + kP5;
  }
  h += uint64_t(len);
  while (p + 8 <= end) {
    h ^= round1(0, rd64(p));
    h = rotl64(h, 27) * kP1 + kP4;
    p += 8;
  }
  if (p + 4 <= end) {
    h ^= uint64_t(rd32(p)) * kP1;
    h = rotl64(h, 23) * kP2 + kP3;
    p += 4;
  }
  while (p < end) {
    h ^= uint64_t(*p) * kP5;
    h = rotl64(h, 11) * kP1;
    ++p;
  }
  h ^= h >> 33;
  h *= kP2;
  h ^= h >> 29;
  h *= kP3;
  h ^= h >> 32;
  return h;
}

uint64_t hps_slabset_of(uint64_t key, uint64_t slabset_count) {
  return hpsb::xxh64_key(key, hpsb::kSlabsetSeed) % slabset_count;
}
uint32_t hps_first_slab_of(uint64_t key, uint32_t slabs_per_set) {
  return uint32_t(hpsb::xxh64_key(key, hpsb::kSlabSeed) % slabs_per_set);
}
uint32_t hps_partition_of(uint64_t key, uint32_t partition_count) {
  return hpsb::partition_of(key, partition_count);
}

int hps_dedup_keys(int device, const uint64_t* keys, size_t n, uint64_t* unique_out,
                   uint32_t* inverse_out, size_t* n_unique, int mem, void* stream) {
  return guarded([&] {
    need(n_unique != nullptr, "n_unique must not be null");
    need(n < (1ull << 32), "dedup batch too large");
    DedupContext& c = dedup_ctx(device);
    std::lock_guard<std::mutex> lk(c.mu);
    hpsb::DeviceGuard g(device);
    if (n == 0) {
      *n_unique = 0;
      return;
    }
    uint64_t tcap = 16;
    while (tcap < 2 * n) tcap <<= 1;
    // regions that persist across calls depend only on tcap and come first,
    // so their epoch-tagged contents never move between calls
    const uint64_t tiles = (tcap / 2 + hpsb::kScanTile - 1) / hpsb::kScanTile;
    auto a = [](uint64_t v) { return (v + 255) / 256 * 256; };
    const bool host = mem == HPS_MEM_HOST;
    const uint64_t fixed = a(tcap * 8) + a(tcap * 4) + a(8) + a(tiles * 8) + a(8);
    const uint64_t bytes = fixed + a(n * 4) + (host ? a(n * 8) * 2 + a(n * 4) : 0);
    if (tcap != c.cap) c.cap = 0;
    const bool fresh = c.cap == 0;
    char* p = static_cast<char*>(c.dbuf.ensure(bytes, c.stream));
    auto take = [&](uint64_t b) {
      char* r = p;
      p += a(b);
      return r;
    };
    hpsb::DedupScratch ds;
    ds.cap = tcap;
    ds.table = reinterpret_cast<uint64_t*>(take(tcap * 8));
    ds.rank_of_slot = reinterpret_cast<uint32_t*>(take(tcap * 4));
    ds.n_unique = reinterpret_cast<unsigned long long*>(take(8));
    c.scan.status = reinterpret_cast<uint64_t*>(take(tiles * 8));
    c.scan.tile_ctr = reinterpret_cast<unsigned long long*>(take(8));
    c.scan.capacity_tiles = tiles;
    ds.slot_of = reinterpret_cast<uint32_t*>(take(n * 4));
    if (fresh || c.dbuf.get() != c.last_base) {
      // new carve: clear the persistent regions once and restart the epochs
      HPSB_CUDA(cudaMemsetAsync(c.dbuf.get(), 0, fixed, c.stream));
      c.scan.tile_base = 0;
      c.scan.epoch = 0;
      c.epoch = 0;
      c.cap = tcap;
      c.last_base = c.dbuf.get();
    }
    if (++c.epoch == 0) {
      HPSB_CUDA(cudaMemsetAsync(ds.table, 0, tcap * 8, c.stream));
      c.epoch = 1;
    }
    const uint64_t* d_keys = keys;
    uint64_t* d_unique = unique_out;
    uint32_t* d_inv = inverse_out;
    if (host) {
      uint64_t* k = reinterpret_cast<uint64_t*>(take(n * 8));
      d_unique = reinterpret_cast<uint64_t*>(take(n * 8));
      d_inv = reinterpret_cast<uint32_t*>(take(n * 4));
      HPSB_CUDA(cudaMemcpyAsync(k, keys, n * 8, cudaMemcpyHostToDevice, c.stream));
      d_keys = k;
    } else {
      cudaEvent_t ev;
      HPSB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      HPSB_CUDA(cudaEventRecord(ev, as_stream(stream)));
      HPSB_CUDA(cudaStreamWaitEvent(c.stream, ev, 0));
      cudaEventDestroy(ev);
    }
    hpsb::launch_dedup(d_keys, n, d_unique, d_inv, ds, c.epoch, c.scan, c.stream);
    unsigned long long* h = static_cast<unsigned long long*>(c.hbuf.ensure(8));
    HPSB_CUDA(cudaMemcpyAsync(h, ds.n_unique, 8, cudaMemcpyDeviceToHost, c.stream));
    HPSB_CUDA(cudaStreamSynchronize(c.stream));
    *n_unique = size_t(*h);
    if (host) {
      HPSB_CUDA(cudaMemcpyAsync(unique_out, d_unique, *n_unique * 8, cudaMemcpyDeviceToHost,
                                c.stream));
      HPSB_CUDA(cudaMemcpyAsync(inverse_out, d_inv, n * 4, cudaMemcpyDeviceToHost, c.stream));
      HPSB_CUDA(cudaStreamSynchronize(c.stream));
    }
  });
}

// ------------------------------------------------------------------ cache --
int hps_cache_create(const hps_cache_config* config, int device, hps_cache** out) {
  return guarded([&] {
    need(config != nullptr && out != nullptr, "null argument");
    hpsb::CacheConfig c;
    c.slabset_count = config->slabset_count;
    c.slabs_per_set = config->slabs_per_set;
    c.dimension = config->dimension;
    c.worker_pool_size = config->worker_pool_size;
    c.tasks_per_worker = config->tasks_per_worker;
    auto h = std::make_unique<hps_cache>();
    h->impl = std::make_unique<hpsb::DeviceCache>(c, device);
    *out = h.release();
  });
}

int hps_cache_create_shared(const hps_cache_config* config, int device, hps_cache* share_with,
                            hps_cache** out) {
  return guarded([&] {
    need(config != nullptr && out != nullptr && share_with != nullptr, "null argument");
    hpsb::CacheConfig c;
    c.slabset_count = config->slabset_count;
    c.slabs_per_set = config->slabs_per_set;
    c.dimension = config->dimension;
    c.worker_pool_size = config->worker_pool_size;
    c.tasks_per_worker = config->tasks_per_worker;
    auto h = std::make_unique<hps_cache>();
    h->impl = std::make_unique<hpsb::DeviceCache>(c, device, share_with->impl.get());
    *out = h.release();
  });
}

int hps_cache_destroy(hps_cache* cache) {
  return guarded([&] { delete cache; });
}

int hps_cache_get_info(hps_cache* cache, hps_cache_info* out) {
  return guarded([&] {
    need(cache && out, "null argument");
    auto& c = *cache->impl;
    out->dimension = c.dimension();
    out->slabs_per_set = c.slabs_per_set();
    out->slabset_count = c.slabset_count();
    out->capacity = c.capacity();
    out->occupied = c.occupied();
    out->recency_clock = c.recency_clock();
    out->device = c.device();
    out->reserved = 0;
  });
}

void* hps_cache_stream(hps_cache* cache) { return cache ? cache->impl->stream() : nullptr; }

int hps_cache_query(hps_cache* cache, const uint64_t* keys, size_t n, float* out,
                    size_t out_len, uint32_t* miss_positions, uint64_t* miss_keys,
                    size_t* n_miss, int mem, void* stream) {
  return guarded([&] {
    need(cache && n_miss, "null argument");
    *n_miss = cache->impl->query(keys, n, out, out_len, miss_positions, miss_keys, mem,
                                 as_stream(stream));
  });
}

int hps_cache_lookup_device(hps_cache* cache, const uint64_t* keys, size_t n, float* out,
                            uint8_t* miss_flags, const float* default_row, uint64_t* miss_keys,
                            uint32_t* miss_firsts, uint64_t* counts, void* stream) {
  return guarded([&] {
    need(cache && counts, "null argument");
    need(n == 0 || (keys && out && miss_flags && default_row && miss_keys && miss_firsts),
         "null argument");
    cache->impl->lookup_device(keys, n, out, miss_flags, default_row, miss_keys, miss_firsts,
                               counts, as_stream(stream));
  });
}

int hps_cache_set_profile_events(hps_cache* cache, void* start_event, void* end_event) {
  return guarded([&] {
    need(cache != nullptr, "null argument");
    cache->impl->set_profile_events(static_cast<cudaEvent_t>(start_event),
                                    static_cast<cudaEvent_t>(end_event));
  });
}

int hps_stream_begin_capture(void* stream) {
  return guarded([&] {
    need(stream != nullptr, "capture needs an explicit stream");
    HPSB_CUDA(cudaStreamBeginCapture(static_cast<cudaStream_t>(stream),
                                     cudaStreamCaptureModeThreadLocal));
  });
}

int hps_stream_end_capture(void* stream, void** graph_exec) {
  return guarded([&] {
    need(stream != nullptr && graph_exec != nullptr, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    unsigned long long cid = 0;
    HPSB_CUDA(cudaStreamGetCaptureInfo(st, &cs, &cid));
    // close the caches' capture sessions whatever happens next (their host
    // clocks and view uses go back to the values at capture start)
    auto g = std::make_unique<hps_graph>();
    g->uses = hpsb::DeviceCache::end_capture(cid);
    cudaGraph_t gr = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(st, &gr);
    if (ec != cudaSuccess) {
      for (auto& u : g->uses)
        if (hpsb::DeviceCache::alive(u.cache, u.serial)) u.cache->release_rebase_slot(u.slot);
      g->uses.clear();
      HPSB_CUDA(ec);
    }
    const cudaError_t e = cudaGraphInstantiate(&g->exec, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) {
      for (auto& u : g->uses)
        if (hpsb::DeviceCache::alive(u.cache, u.serial)) u.cache->release_rebase_slot(u.slot);
      g->uses.clear();
      HPSB_CUDA(e);
    }
    *graph_exec = g.release();
  });
}

int hps_graph_launch(void* graph_exec, void* stream) {
  return guarded([&] {
    need(graph_exec != nullptr, "null graph");
    auto* g = static_cast<hps_graph*>(graph_exec);
    cudaStream_t x = as_stream(stream);
    // every cache of the graph is held for the whole launch (address order:
    // no lock-order inversion between concurrent launches)
    std::vector<hpsb::GraphCacheUse*> us;
    for (auto& u : g->uses) {
      need(hpsb::DeviceCache::alive(u.cache, u.serial),
           "a cache captured in this graph has been destroyed");
      us.push_back(&u);
    }
    std::sort(us.begin(), us.end(),
              [](const hpsb::GraphCacheUse* a, const hpsb::GraphCacheUse* b) { return a->cache < b->cache; });
    std::vector<std::unique_lock<std::mutex>> locks;
    for (size_t i = 0; i < us.size(); ++i)
      if (i == 0 || us[i]->cache != us[i - 1]->cache) locks.emplace_back(us[i]->cache->mutex());
    for (auto* u : us) u->cache->graph_before_launch_locked(*u, x);
    HPSB_CUDA(cudaGraphLaunch(g->exec, x));
    for (auto* u : us) u->cache->graph_after_launch_locked(x);
  });
}

int hps_event_record(void* event, void* stream) {
  return guarded([&] {
    need(event != nullptr, "null event");
    cudaStream_t st = as_stream(stream);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    HPSB_CUDA(cudaStreamIsCapturing(st, &cs));
    HPSB_CUDA(cudaEventRecordWithFlags(static_cast<cudaEvent_t>(event), st,
                                       cs == cudaStreamCaptureStatusActive
                                           ? cudaEventRecordExternal
                                           : cudaEventRecordDefault));
  });
}

int hps_graph_destroy(void* graph_exec) {
  return guarded([&] {
    auto* g = static_cast<hps_graph*>(graph_exec);
    if (g == nullptr) return;
    for (auto& u : g->uses)
      if (hpsb::DeviceCache::alive(u.cache, u.serial)) u.cache->release_rebase_slot(u.slot);
    if (g->exec) cudaGraphExecDestroy(g->exec);
    delete g;
  });
}

int hps_cache_replace(hps_cache* cache, const uint64_t* keys, size_t n, const float* vectors,
                      size_t vectors_len, int mem, void* stream) {
  return guarded([&] {
    need(cache != nullptr, "null argument");
    cache->impl->replace(keys, n, vectors, vectors_len, mem, as_stream(stream));
  });
}

int hps_cache_replace_device_async(hps_cache* cache, const uint64_t* keys, size_t n,
                                   const float* vectors, size_t vectors_len, void* stream) {
  return guarded([&] {
    need(cache != nullptr, "null argument");
    need(vectors_len == n * uint64_t(cache->impl->dimension()),
         "replace vector buffer has wrong size");
    need(n == 0 || (keys && vectors), "null argument");
    cache->impl->replace_device_async(keys, n, vectors, as_stream(stream));
  });
}

size_t hps_peer_blob_size(void) { return sizeof(hpsb::PeerBlob); }

int hps_cache_peer_export(hps_cache* cache, uint64_t inbox_cap, void* blob, size_t blob_cap,
                          size_t* blob_len) {
  return guarded([&] {
    need(cache && blob && blob_len, "null argument");
    need(blob_cap >= sizeof(hpsb::PeerBlob), "peer blob buffer too small");
    hpsb::PeerBlob b;
    cache->impl->peer_export(inbox_cap, &b);
    std::memcpy(blob, &b, sizeof(b));
    *blob_len = sizeof(b);
  });
}

int hps_peer_group_create(hps_cache* self, uint32_t rank, uint32_t world, const void* blobs,
                          size_t blob_len, hps_peer_group** out) {
  return guarded([&] {
    need(self && blobs && out, "null argument");
    need(blob_len == sizeof(hpsb::PeerBlob), "peer blob size mismatch");
    std::vector<hpsb::PeerBlob> v(world);
    for (uint32_t r = 0; r < world; ++r)
      std::memcpy(&v[r], static_cast<const char*>(blobs) + size_t(r) * blob_len, blob_len);
    auto g = std::make_unique<hps_peer_group>();
    g->impl = std::make_unique<hpsb::PeerGroup>(*self->impl, rank, v);
    *out = g.release();
  });
}

int hps_peer_group_destroy(hps_peer_group* group) {
  return guarded([&] { delete group; });
}

int hps_peer_lookup_device(hps_peer_group* group, const uint64_t* keys, size_t n, float* out,
                           uint8_t* miss_flags, const float* default_row, void* stream) {
  return guarded([&] {
    need(group != nullptr, "null argument");
    need(n == 0 || (keys && out && miss_flags && default_row), "null argument");
    need(n < 0xFFFFFFFFull, "lookup batch too large");
    group->impl->lookup(keys, n, out, miss_flags, default_row, as_stream(stream));
  });
}

int hps_cache_peer_drain(hps_cache* cache, uint64_t* keys_out, size_t cap, size_t* n_appended) {
  return guarded([&] {
    need(cache && n_appended && (cap == 0 || keys_out), "null argument");
    *n_appended = cache->impl->peer_drain(keys_out, cap);
  });
}

int hps_cache_set_replace_mode(hps_cache* cache, int mode) {
  return guarded([&] {
    need(cache != nullptr, "null argument");
    cache->impl->set_replace_mode(mode);
  });
}

int hps_cache_get_replace_mode(hps_cache* cache, int* mode, uint64_t* dropped) {
  return guarded([&] {
    need(cache != nullptr, "null argument");
    if (mode) *mode = cache->impl->replace_mode();
    if (dropped) *dropped = cache->impl->relaxed_dropped();
  });
}

int hps_cache_update(hps_cache* cache, const uint64_t* keys, size_t n, const float* vectors,
                     size_t vectors_len, size_t* written, int mem, void* stream) {
  return guarded([&] {
    need(cache && written, "null argument");
    *written = cache->impl->update(keys, n, vectors, vectors_len, mem, as_stream(stream));
  });
}

int hps_cache_update_device(hps_cache* cache, const uint64_t* keys, size_t n,
                            const float* vectors, size_t vectors_len, uint64_t* written,
                            void* stream) {
  return guarded([&] {
    need(cache != nullptr, "null argument");
    need(vectors_len == n * uint64_t(cache->impl->dimension()),
         "update vector buffer has wrong size");
    cache->impl->update_device(keys, n, vectors, written, as_stream(stream));
  });
}

int hps_cache_dump_device(hps_cache* cache, uint64_t set_begin, uint64_t set_end, uint64_t* out,
                          uint64_t* n_out, void* stream) {
  return guarded([&] {
    need(cache && out && n_out, "null argument");
    cache->impl->dump_device(set_begin, set_end, out, n_out, as_stream(stream));
  });
}

int hps_cache_dump(hps_cache* cache, uint64_t set_begin, uint64_t set_end, uint64_t* out,
                   size_t cap, size_t* n_out) {
  return guarded([&] {
    need(cache && n_out, "null argument");
    *n_out = cache->impl->dump(set_begin, set_end, out, cap);
  });
}

int hps_cache_check_invariants(hps_cache* cache) {
  return guarded([&] {
    need(cache != nullptr, "null argument");
    cache->impl->check_invariants();
  });
}

int hps_cache_export_state(hps_cache* cache, uint64_t* keys, uint64_t* counters,
                           uint32_t* masks, float* rows) {
  return guarded([&] {
    need(cache != nullptr, "null argument");
    cache->impl->export_state(keys, counters, masks, rows);
  });
}

int hps_cache_debug_trace(hps_cache* cache, uint64_t* out, size_t cap, uint64_t* n_calls) {
  return guarded([&] {
    need(cache != nullptr && n_calls != nullptr, "null argument");
    std::vector<unsigned long long> ring(hpsb::DeviceCache::kTraceRing * 8);
    *n_calls = cache->impl->trace(ring.data());
    if (out != nullptr) std::copy(ring.begin(), ring.begin() + std::min(cap, ring.size()), out);
  });
}

// ---------------------------------------------------------------- sharded --
uint32_t hps_shard_of(uint64_t key, uint32_t world) {
  return world == 0 ? 0u : hpsb::shard_of(key, world);
}

int hps_shard_count(int device, const uint64_t* keys, size_t n, uint32_t world, uint64_t* counts,
                    void* stream) {
  return guarded([&] {
    need(counts != nullptr && (n == 0 || keys != nullptr), "null argument");
    need(world >= 1 && world <= 64, "world size must be within [1, 64]");
    hpsb::DeviceGuard g(device);
    hpsb::launch_shard_count(keys, n, world, reinterpret_cast<unsigned long long*>(counts),
                             as_stream(stream));
  });
}

int hps_shard_scatter(int device, const uint64_t* keys, size_t n, uint32_t world, uint64_t* cursor,
                      uint64_t* send_keys, uint32_t* send_pos, void* stream) {
  return guarded([&] {
    need(cursor != nullptr && (n == 0 || (keys && send_keys && send_pos)), "null argument");
    need(world >= 1 && world <= 64, "world size must be within [1, 64]");
    need(n < (1ull << 32), "batch too large");
    hpsb::DeviceGuard g(device);
    hpsb::launch_shard_scatter(keys, n, world, reinterpret_cast<unsigned long long*>(cursor),
                               send_keys, send_pos, as_stream(stream));
  });
}

int hps_shard_unroute(int device, size_t m, uint32_t dim, const uint32_t* send_pos,
                      const float* rows, const uint8_t* flags_in, float* out, uint8_t* flags_out,
                      void* stream) {
  return guarded([&] {
    need(m == 0 || (send_pos && rows && out), "null argument");
    need(dim > 0, "dimension must be positive");
    need((flags_in == nullptr) == (flags_out == nullptr), "flags in / out must both be given");
    hpsb::DeviceGuard g(device);
    hpsb::launch_shard_unroute(m, dim, send_pos, rows, flags_in, out, flags_out, as_stream(stream));
  });
}

// ------------------------------------------------------------------- wire --
int hps_wire_lookup_frame(int device, const float* rows, const uint8_t* miss_flags,
                          uint32_t count, uint32_t dim, int mem, uint8_t* frame, size_t cap,
                          size_t* frame_len, void* stream) {
  return guarded([&] {
    need(frame_len != nullptr, "null argument");
    need(dim > 0, "dimension must be positive");
    const size_t bytes = hpsb::wire_lookup_frame_bytes(count, dim);
    need(bytes - 4 <= 0xFFFFFFFFull, "frame too large");
    *frame_len = bytes;
    if (frame == nullptr) return;  // size query
    need(cap >= bytes, "frame buffer too small");
    need(count == 0 || (rows && miss_flags), "null argument");
    if (mem == HPS_MEM_HOST) {
      hpsb::wire_encode_lookup_host(rows, miss_flags, count, dim, frame);
      return;
    }
    hpsb::DeviceGuard g(device);
    cudaStream_t st = as_stream(stream);
    uint8_t* bm = nullptr;
    if (count) HPSB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bm), (count + 7) / 8 + 4, st));
    try {
      hpsb::wire_encode_lookup_device(rows, miss_flags, count, dim, bm, frame, st);
    } catch (...) {
      if (bm) cudaFreeAsync(bm, st);
      throw;
    }
    if (bm) HPSB_CUDA(cudaFreeAsync(bm, st));
    HPSB_CUDA(cudaStreamSynchronize(st));
  });
}

// -------------------------------------------------------------------- vdb --
int hps_vdb_create(uint32_t lookup_threads, hps_vdb** out) {
  return guarded([&] {
    need(out != nullptr, "null argument");
    auto h = std::make_unique<hps_vdb>();
    h->impl = std::make_unique<hpsb::VolatileStore>(lookup_threads);
    *out = h.release();
  });
}
int hps_vdb_destroy(hps_vdb* vdb) {
  return guarded([&] { delete vdb; });
}
int hps_vdb_register_table(hps_vdb* vdb, const char* name, uint32_t dimension,
                           uint32_t partition_count, uint64_t overflow_margin) {
  return guarded([&] {
    need(vdb && name, "null argument");
    vdb->impl->register_table(name, dimension, partition_count, overflow_margin);
  });
}
int hps_vdb_has_table(hps_vdb* vdb, const char* name) {
  return (vdb && name && vdb->impl->has_table(name)) ? 1 : 0;
}
int hps_vdb_insert(hps_vdb* vdb, const char* name, const uint64_t* keys, size_t n,
                   const float* vectors, size_t vectors_len, uint64_t* evicted,
                   size_t evicted_cap, size_t* n_evicted) {
  return guarded([&] {
    need(vdb && name, "null argument");
    g_evicted = vdb->impl->insert(name, keys, n, vectors, vectors_len);
    const auto& ev = g_evicted;
    if (evicted) std::copy(ev.begin(), ev.begin() + std::min(ev.size(), evicted_cap), evicted);
    if (n_evicted) *n_evicted = ev.size();
  });
}
int hps_vdb_insert_async(hps_vdb* vdb, const char* name, const uint64_t* keys, size_t n,
                         const float* vectors, size_t vectors_len) {
  return guarded([&] {
    need(vdb && name, "null argument");
    vdb->impl->insert_async(name, std::vector<uint64_t>(keys, keys + n),
                            std::vector<float>(vectors, vectors + vectors_len));
  });
}
int hps_vdb_lookup(hps_vdb* vdb, const char* name, const uint64_t* keys, size_t n,
                   uint64_t* found_keys, float* found_vectors, size_t* n_found,
                   uint64_t* missing_keys, size_t* n_missing) {
  return guarded([&] {
    need(vdb && name && n_found && n_missing, "null argument");
    vdb->impl->lookup(name, keys, n, found_keys, found_vectors, nullptr, n_found, missing_keys,
                      n_missing);
  });
}
int hps_vdb_drain(hps_vdb* vdb) {
  return guarded([&] { vdb->impl->drain(); });
}
int hps_vdb_table_size(hps_vdb* vdb, const char* name, uint64_t* out) {
  return guarded([&] { *out = vdb->impl->table_size(name); });
}
int hps_vdb_partition_size(hps_vdb* vdb, const char* name, uint32_t partition, uint64_t* out) {
  return guarded([&] { *out = vdb->impl->partition_size(name, partition); });
}
int hps_vdb_table_clock(hps_vdb* vdb, const char* name, uint64_t* out) {
  return guarded([&] { *out = vdb->impl->table_clock(name); });
}
int hps_vdb_last_access(hps_vdb* vdb, const char* name, uint64_t key, uint64_t* out,
                        int* found) {
  return guarded([&] {
    uint64_t v = 0;
    *found = vdb->impl->last_access(name, key, &v) ? 1 : 0;
    *out = v;
  });
}
int hps_vdb_evict(hps_vdb* vdb, const char* name, uint32_t partition, uint64_t* evicted,
                  size_t evicted_cap, size_t* n_evicted) {
  return guarded([&] {
    g_evicted = vdb->impl->evict(name, partition);
    const auto& ev = g_evicted;
    if (evicted) std::copy(ev.begin(), ev.begin() + std::min(ev.size(), evicted_cap), evicted);
    if (n_evicted) *n_evicted = ev.size();
  });
}
int hps_vdb_last_evicted(uint64_t* out, size_t cap, size_t* n) {
  return guarded([&] {
    need(n != nullptr, "null argument");
    if (out) std::copy(g_evicted.begin(), g_evicted.begin() + std::min(g_evicted.size(), cap), out);
    *n = g_evicted.size();
  });
}
int hps_vdb_dimension(hps_vdb* vdb, const char* name, uint32_t* out) {
  return guarded([&] {
    need(vdb && name && out, "null argument");
    *out = vdb->impl->dimension(name);
  });
}
int hps_vdb_partition_count(hps_vdb* vdb, const char* name, uint32_t* out) {
  return guarded([&] {
    need(vdb && name && out, "null argument");
    *out = vdb->impl->partition_count(name);
  });
}
int hps_vdb_keys(hps_vdb* vdb, const char* name, uint64_t* out, size_t cap, size_t* n) {
  return guarded([&] {
    need(vdb && name && n, "null argument");
    auto k = vdb->impl->keys(name);
    if (out) std::copy(k.begin(), k.begin() + std::min(k.size(), cap), out);
    *n = k.size();
  });
}

// ------------------------------------------------------------- cold tier --
int hps_pdb_open(const char* root, uint32_t threads, hps_pdb** out) {
  return guarded([&] {
    need(root && out, "null argument");
    auto h = std::make_unique<hps_pdb>();
    h->impl = std::make_unique<hpsb::SegmentStore>(root, threads);
    *out = h.release();
  });
}
int hps_pdb_destroy(hps_pdb* pdb) {
  return guarded([&] { delete pdb; });
}
int hps_pdb_attach(hps_pdb* pdb, const char* table) {
  return guarded([&] {
    need(pdb && table, "null argument");
    pdb->impl->attach(table);
  });
}
int hps_pdb_refresh(hps_pdb* pdb, const char* table) {
  return guarded([&] {
    need(pdb && table, "null argument");
    pdb->impl->refresh(table);
  });
}
int hps_pdb_info(hps_pdb* pdb, const char* table, uint32_t* dimension, uint64_t* keys,
                 uint64_t* segments) {
  return guarded([&] {
    need(pdb && table, "null argument");
    if (dimension) *dimension = pdb->impl->dimension(table);
    if (keys) *keys = pdb->impl->key_count(table);
    if (segments) *segments = pdb->impl->segment_count(table);
  });
}
int hps_pdb_get(hps_pdb* pdb, const char* table, const uint64_t* keys, size_t n,
                uint64_t* found_keys, float* found_vectors, size_t* n_found,
                uint64_t* missing_keys, size_t* n_missing) {
  return guarded([&] {
    need(pdb && table && n_found && n_missing, "null argument");
    pdb->impl->get(table, keys, n, found_keys, found_vectors, nullptr, n_found, missing_keys,
                   n_missing);
  });
}
int hps_pdb_table_ctx(hps_pdb* pdb, const char* table, void** ctx) {
  return guarded([&] {
    need(pdb && table && ctx, "null argument");
    pdb->impl->attach(table);
    std::lock_guard<std::mutex> lk(pdb->mu);
    auto& c = pdb->ctx[table];
    if (!c) c = std::make_unique<std::pair<hps_pdb*, std::string>>(pdb, table);
    *ctx = c.get();
  });
}
int hps_pdb_cold_fetch(void* ctx, const uint64_t* keys, size_t n, uint64_t* found_keys,
                       float* found_vectors, size_t* n_found, uint64_t* missing_keys,
                       size_t* n_missing) {
  auto* c = static_cast<std::pair<hps_pdb*, std::string>*>(ctx);
  return hps_pdb_get(c->first, c->second.c_str(), keys, n, found_keys, found_vectors, n_found,
                     missing_keys, n_missing);
}

int hps_tier_fetch(hps_vdb* vdb, const char* table, uint32_t dimension, hps_cold_fetch_fn cold,
                   void* cold_ctx, const uint64_t* keys, size_t n, uint64_t* found_keys,
                   float* found_vectors, size_t* n_found, uint64_t* missing_keys,
                   size_t* n_missing, uint64_t* counters) {
  return guarded([&] {
    need(table && n_found && n_missing, "null argument");
    std::vector<int32_t> row_of(n);
    hpsb::TierCounters tc;
    hpsb::tier_fetch_staged(vdb ? vdb->impl.get() : nullptr, table, dimension, cold, cold_ctx,
                            keys, n, found_keys, found_vectors, row_of.data(), n_found,
                            missing_keys, n_missing, &tc);
    if (counters) {
      counters[0] = tc.vdb_hits;
      counters[1] = tc.cold_hits;
      counters[2] = tc.missing;
    }
  });
}

int hps_refresh_cache(hps_cache* cache, hps_vdb* vdb, const char* table,
                      hps_cold_fetch_fn cold, void* cold_ctx, size_t dump_batch,
                      uint64_t* refreshed, uint64_t* unresolved, size_t unresolved_cap,
                      size_t* n_unresolved) {
  return guarded([&] {
    need(cache && table && refreshed && n_unresolved, "null argument");
    auto r = hpsb::refresh_cache(*cache->impl, vdb ? vdb->impl.get() : nullptr, table, cold,
                                 cold_ctx, dump_batch);
    *refreshed = r.refreshed;
    *n_unresolved = r.unresolved.size();
    if (unresolved)
      std::copy(r.unresolved.begin(),
                r.unresolved.begin() + std::min(unresolved_cap, r.unresolved.size()), unresolved);
  });
}

// ----------------------------------------------------------------- engine --
int hps_engine_create(const char* table, uint32_t dimension, hps_cache* cache, hps_vdb* vdb,
                      hps_cold_fetch_fn cold, void* cold_ctx, const hps_engine_config* config,
                      hps_engine** out) {
  return guarded([&] {
    need(table && cache && config && out, "null argument");
    hpsb::EngineConfig c;
    c.hit_rate_threshold = config->hit_rate_threshold;
    if (config->default_vector && config->default_vector_len)
      c.default_vector.assign(config->default_vector,
                              config->default_vector + config->default_vector_len);
    c.workspace_pool_size = config->workspace_pool_size;
    c.async_worker_count = config->async_worker_count;
    c.volatile_tier_enabled = config->volatile_tier_enabled != 0;
    c.max_batch = config->max_batch;  // 0 = no limit (below 2^32)
    auto h = std::make_unique<hps_engine>();
    h->impl = std::make_unique<hpsb::LookupEngine>(table, dimension, cache->impl.get(),
                                                   vdb ? vdb->impl.get() : nullptr, cold,
                                                   cold_ctx, std::move(c));
    *out = h.release();
  });
}
int hps_engine_destroy(hps_engine* engine) {
  return guarded([&] { delete engine; });
}
int hps_engine_lookup(hps_engine* engine, const uint64_t* keys, size_t n, float* out,
                      size_t out_len, uint8_t* miss_flags, hps_lookup_outcome* outcome, int mem,
                      void* stream) {
  return guarded([&] {
    need(engine != nullptr, "null argument");
    hpsb::LookupOutcome o;
    engine->impl->lookup(keys, n, out, out_len, miss_flags, &o, mem, as_stream(stream));
    if (outcome) {
      outcome->sync_branch = o.sync_branch ? 1 : 0;
      outcome->unique_hit_rate = o.unique_hit_rate;
      outcome->unique_count = o.unique_count;
      outcome->defaults_returned = o.defaults_returned;
    }
  });
}
int hps_engine_lookup_multi(hps_engine* const* engines, size_t count,
                            const uint64_t* const* keys, const size_t* n, float* const* out,
                            uint8_t* const* miss_flags, hps_lookup_outcome* outcomes, int mem) {
  return guarded([&] {
    need(count == 0 || (engines && keys && n && out && miss_flags), "null argument");
    std::vector<hpsb::LookupEngine*> impls(count);
    for (size_t t = 0; t < count; ++t) {
      need(engines[t] != nullptr, "null engine");
      impls[t] = engines[t]->impl.get();
    }
    std::vector<hpsb::LookupOutcome> o(count);
    hpsb::LookupEngine::lookup_multi(impls.data(), count, keys, n, out, miss_flags, o.data(), mem);
    if (outcomes) {
      for (size_t t = 0; t < count; ++t) {
        outcomes[t].sync_branch = o[t].sync_branch ? 1 : 0;
        outcomes[t].unique_hit_rate = o[t].unique_hit_rate;
        outcomes[t].unique_count = o[t].unique_count;
        outcomes[t].defaults_returned = o[t].defaults_returned;
      }
    }
  });
}
int hps_multi_create(hps_engine* const* engines, size_t count, size_t max_batch,
                     hps_multi** out) {
  return guarded([&] {
    need(out != nullptr && (count == 0 || engines != nullptr), "null argument");
    std::vector<hpsb::LookupEngine*> v(count);
    for (size_t t = 0; t < count; ++t) {
      need(engines[t] != nullptr, "null engine");
      v[t] = engines[t]->impl.get();
    }
    auto h = std::make_unique<hps_multi>();
    h->impl = std::make_unique<hpsb::MultiLookup>(std::move(v), max_batch);
    *out = h.release();
  });
}

int hps_multi_destroy(hps_multi* multi) {
  return guarded([&] { delete multi; });
}

int hps_multi_lookup(hps_multi* multi, const uint64_t* const* keys, const size_t* n,
                     float* const* out, uint8_t* const* miss_flags,
                     hps_lookup_outcome* outcomes) {
  return guarded([&] {
    need(multi && keys && n && out && miss_flags, "null argument");
    const size_t T = multi->impl ? multi->impl->tables() : 0;
    std::vector<hpsb::LookupOutcome> o(T);
    multi->impl->lookup(keys, n, out, miss_flags, o.data());
    if (outcomes) {
      for (size_t t = 0; t < T; ++t) {
        outcomes[t].sync_branch = o[t].sync_branch ? 1 : 0;
        outcomes[t].unique_hit_rate = o[t].unique_hit_rate;
        outcomes[t].unique_count = o[t].unique_count;
        outcomes[t].defaults_returned = o[t].defaults_returned;
      }
    }
  });
}

int hps_replicas_create(hps_engine* const* engines, size_t count, hps_replicas** out) {
  return guarded([&] {
    need(engines && out, "null argument");
    std::vector<hpsb::LookupEngine*> e;
    for (size_t i = 0; i < count; ++i) e.push_back(engines[i] ? engines[i]->impl.get() : nullptr);
    auto h = std::make_unique<hps_replicas>();
    h->impl = std::make_unique<hpsb::ReplicaGroup>(std::move(e));
    *out = h.release();
  });
}
int hps_replicas_destroy(hps_replicas* group) {
  return guarded([&] { delete group; });
}
int hps_replicas_lookup(hps_replicas* group, const uint64_t* const* keys, const size_t* n,
                        float* const* out, uint8_t* const* miss_flags,
                        hps_lookup_outcome* outcomes, int mem) {
  return guarded([&] {
    need(group && keys && n && out && miss_flags, "null argument");
    const size_t g = group->impl->size();
    std::vector<hpsb::LookupOutcome> o(g);
    group->impl->lookup(keys, n, out, miss_flags, o.data(), mem);
    if (outcomes)
      for (size_t r = 0; r < g; ++r) {
        outcomes[r].sync_branch = o[r].sync_branch ? 1 : 0;
        outcomes[r].unique_hit_rate = o[r].unique_hit_rate;
        outcomes[r].unique_count = o[r].unique_count;
        outcomes[r].defaults_returned = o[r].defaults_returned;
      }
  });
}
int hps_engine_reserve(hps_engine* engine, size_t max_keys) {
  return guarded([&] {
    need(engine != nullptr, "null argument");
    engine->impl->reserve(max_keys);
  });
}
int hps_engine_drain_async(hps_engine* engine) {
  return guarded([&] { engine->impl->drain_async(); });
}
int hps_engine_get_stats(hps_engine* engine, hps_engine_stats* out) {
  return guarded([&] {
    const auto s = engine->impl->stats();
    *out = hps_engine_stats{s.queries,        s.queried_keys,  s.unique_keys,
                            s.cache_hits,     s.cache_misses,  s.sync_batches,
                            s.async_batches,  s.defaults_returned, s.vdb_hits,
                            s.pdb_hits,       s.tier_missing,  s.async_faults};
  });
}
int hps_engine_pool_info(hps_engine* engine, uint64_t* size, uint64_t* outstanding,
                         uint64_t* peak_outstanding) {
  return guarded([&] {
    auto& p = engine->impl->pool();
    if (size) *size = p.size();
    if (outstanding) *outstanding = p.outstanding();
    if (peak_outstanding) *peak_outstanding = p.peak_outstanding();
  });
}


}  // extern "C"
