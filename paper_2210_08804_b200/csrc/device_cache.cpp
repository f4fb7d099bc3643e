// device_cache.cpp -- see device_cache.hpp.
#include "device_cache.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <unordered_set>
#include <vector>

namespace hpsb {

namespace {
inline uint64_t align256(uint64_t v) { return (v + 255) / 256 * 256; }

// Bump allocator over one scratch block.
struct Carver {
  char* p;
  template <class T>
  T* take(uint64_t count) {
    T* r = reinterpret_cast<T*>(p);
    p += align256(count * sizeof(T));
    return r;
  }
};

// Live caches and the open capture sessions (capture id -> caches).
std::mutex g_reg_mu;
std::map<const DeviceCache*, uint64_t> g_alive;
std::map<unsigned long long, std::vector<DeviceCache*>> g_sessions;
uint64_t g_next_serial = 1;

int keys_per_warp_for(uint32_t tasks_per_worker) {
  // SlabCacheConfig::tasks_per_worker (slab_cache.hpp:33) becomes the number
  // of keys one warp keeps in flight (paper tasksPerWarp).
  if (tasks_per_worker >= 8) return 8;
  if (tasks_per_worker >= 4) return 4;
  if (tasks_per_worker >= 2) return 2;
  return 1;
}
}  // namespace

DeviceCache::DeviceCache(const CacheConfig& cfg, int device, const DeviceCache* share_stream_with)
    : cfg_(cfg), device_(device) {
  // same validation, same messages as slab_cache.cpp:18-29
  if (cfg.slabset_count == 0) throw invalid_argument("slabset_count must be positive");
  if (cfg.slabs_per_set == 0) throw invalid_argument("slabs_per_set must be positive");
  if (cfg.dimension == 0) throw invalid_argument("cache dimension must be positive");
  if (cfg.worker_pool_size == 0) throw invalid_argument("worker_pool_size must be positive");
  // device slot indices are u32 (probe.cuh); 0xFFFFFFFF is the no-slot mark
  if (cfg.slabset_count * cfg.slabs_per_set * 32ull >= 0xFFFFFFFFull ||
      cfg.slabset_count * cfg.slabs_per_set / cfg.slabs_per_set != cfg.slabset_count)
    throw invalid_argument("cache capacity must stay below 2^32 slots per replica");
  keys_per_warp_ = keys_per_warp_for(std::max<uint32_t>(1, cfg.tasks_per_worker));
  DeviceGuard g(device_);
  if (share_stream_with != nullptr) {
    // a cache group: several tables' caches ordered on one stream (the
    // multi-table lookup runs them in one launch)
    if (share_stream_with->device_ != device)
      throw invalid_argument("caches sharing a stream must be on the same device");
    stream_holder_ = share_stream_with->stream_holder_;
  } else {
    stream_holder_ = std::make_shared<StreamHolder>();
    HPSB_CUDA(cudaStreamCreateWithFlags(&stream_holder_->s, cudaStreamNonBlocking));
  }
  stream_ = stream_holder_->s;
  HPSB_CUDA(cudaEventCreateWithFlags(&ev_in_, cudaEventDisableTiming));
  HPSB_CUDA(cudaEventCreateWithFlags(&ev_out_, cudaEventDisableTiming));
  const uint64_t slabs = cfg.slabset_count * cfg.slabs_per_set;
  const uint64_t slots = slabs * 32ull;
  dev_.S = cfg.slabset_count;
  dev_.W = cfg.slabs_per_set;
  dev_.d = cfg.dimension;
  dev_.mS = ~0ull / cfg.slabset_count;
  dev_.mW = ~0ull / cfg.slabs_per_set;
  // keys, fingerprints, masks and counters in ONE allocation (one L2
  // persistence window covers the probe structures, below)
  const uint64_t tags_off = (slots * 8 + 255) / 256 * 256;
  const uint64_t masks_off = tags_off + (slots + 255) / 256 * 256;
  const uint64_t ctr_off = masks_off + (slabs * 4 + 255) / 256 * 256;
  HPSB_CUDA(cudaMalloc(&probe_mem_, ctr_off + slots * 8));
  char* pm = static_cast<char*>(probe_mem_);
  dev_.keys = reinterpret_cast<uint64_t*>(pm);
  dev_.tags = reinterpret_cast<uint8_t*>(pm + tags_off);
  dev_.masks = reinterpret_cast<decltype(dev_.masks)>(pm + masks_off);
  dev_.counters = reinterpret_cast<decltype(dev_.counters)>(pm + ctr_off);
  HPSB_CUDA(cudaMalloc(&dev_.rows, slots * uint64_t(cfg.dimension) * 4));
  HPSB_CUDA(cudaMalloc(&dev_.occupied, 8));
  // rebase slots of captured graphs (allocated up front: no allocation may
  // happen while a stream is being captured)
  HPSB_CUDA(cudaMalloc(&rebase_, kRebaseSlots * 16 * 8));
  HPSB_CUDA(cudaMemsetAsync(rebase_, 0, kRebaseSlots * 16 * 8, stream_));
  for (int i = kRebaseSlots - 1; i >= 0; --i) free_slots_.push_back(i);
  // update: last position per slot, two arrays (consecutive updates alternate)
  HPSB_CUDA(cudaMalloc(&winner_, 2 * slots * 4));
  HPSB_CUDA(cudaMemsetAsync(winner_, 0, 2 * slots * 4, stream_));
  HPSB_CUDA(cudaMemsetAsync(dev_.keys, 0, slots * 8, stream_));
  HPSB_CUDA(cudaMemsetAsync(dev_.counters, 0, slots * 8, stream_));
  HPSB_CUDA(cudaMemsetAsync(dev_.masks, 0, slabs * 4, stream_));
  HPSB_CUDA(cudaMemsetAsync(dev_.tags, 0, slots, stream_));
  // The probe structures (keys + fingerprints: 9 B per slot, 18 MB at cfg 2)
  // as a persisting L2 window on the cache stream, so the expanded output
  // streaming through L2 (33.5 MB per 65,536-key call) does not evict them
  // between calls (cfg 2: +3.5 % lookups/s; HPSB_L2_PERSIST=off disables).
  // Tables whose probe structures exceed the persisting capacity get none.
  {
    const char* e = std::getenv("HPSB_L2_PERSIST");
    if (!(e && std::string(e) == "off")) {
      int maxp = 0, maxw = 0;
      cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, device_);
      cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, device_);
      // default: keys + fingerprints + masks; HPSB_L2_PERSIST=all adds the counters
      const bool all = e && std::string(e) == "all";
      const size_t want = all ? ctr_off + slots * 8 : ctr_off;
      const size_t win = std::min<size_t>(want, size_t(maxw));
      // only when the whole region fits the persisting capacity: a random
      // sliver of a much larger table (cfg 5: 1.8 GB) would only take L2
      // away from everything else
      if (maxp > 0 && win > 0 && want <= size_t(maxp) && want <= size_t(maxw)) {
        const size_t persist = std::min<size_t>(win, size_t(maxp));
        size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
        if (cur < persist) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist);
        cudaStreamAttrValue av = {};
        av.accessPolicyWindow.base_ptr = probe_mem_;
        av.accessPolicyWindow.num_bytes = win;
        av.accessPolicyWindow.hitRatio = float(double(persist) / double(win));
        av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaStreamSetAttribute(stream_, cudaStreamAttributeAccessPolicyWindow, &av);
      }
      cudaGetLastError();  // best effort: no persistence support is not an error
    }
  }
  HPSB_CUDA(cudaMemsetAsync(dev_.rows, 0, slots * uint64_t(cfg.dimension) * 4, stream_));
  HPSB_CUDA(cudaMemsetAsync(dev_.occupied, 0, 8, stream_));
  HPSB_CUDA(cudaMalloc(&d_small_, 64));
  HPSB_CUDA(cudaMemsetAsync(d_small_, 0, 64, stream_));
  HPSB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_small_), 64, cudaHostAllocPortable));
  HPSB_CUDA(cudaMalloc(&scan_.tile_ctr, 8));
  HPSB_CUDA(cudaMemsetAsync(scan_.tile_ctr, 0, 8, stream_));
  ensure_scan_tiles(1024);
  HPSB_CUDA(cudaStreamSynchronize(stream_));
  std::lock_guard<std::mutex> rl(g_reg_mu);
  serial_ = g_next_serial++;
  g_alive[this] = serial_;
}

DeviceCache::~DeviceCache() {
  {
    std::lock_guard<std::mutex> rl(g_reg_mu);
    g_alive.erase(this);
    if (cap_.id != 0) {
      auto it = g_sessions.find(cap_.id);
      if (it != g_sessions.end()) {
        auto& v = it->second;
        v.erase(std::remove(v.begin(), v.end(), this), v.end());
      }
    }
  }
  DeviceGuard g(device_);
  cudaStreamSynchronize(stream_);
  cudaFree(probe_mem_);
  cudaFree(dev_.rows);
  cudaFree(dev_.occupied);
  cudaFree(d_small_);
  cudaFreeHost(h_small_);
  cudaFree(inbox_);
  cudaFree(scan_.tile_ctr);
  cudaFree(scan_.status);
  cudaFree(trace_);
  cudaFree(rebase_);
  cudaFree(winner_);
  cudaEventDestroy(ev_in_);
  cudaEventDestroy(ev_out_);
  stream_holder_.reset();  // the last cache of a group destroys the stream
}

void DeviceCache::ensure_scan_tiles(uint64_t tiles) {
  if (tiles <= scan_.capacity_tiles) return;
  uint64_t cap = std::max<uint64_t>(1024, scan_.capacity_tiles);
  while (cap < tiles) cap <<= 1;
  if (scan_.status) {
    HPSB_CUDA(cudaStreamSynchronize(stream_));
    HPSB_CUDA(cudaFree(scan_.status));
  }
  HPSB_CUDA(cudaMalloc(&scan_.status, cap * 8));
  HPSB_CUDA(cudaMemsetAsync(scan_.status, 0, cap * 8, stream_));
  scan_.capacity_tiles = cap;
  scan_.epoch = 0;
}

void DeviceCache::join_from(cudaStream_t user) {
  if (user == nullptr || user == stream_) return;
  mark_other_op();
  HPSB_CUDA(cudaEventRecord(ev_in_, user));
  HPSB_CUDA(cudaStreamWaitEvent(stream_, ev_in_, 0));
}

void DeviceCache::join_to(cudaStream_t user) {
  if (user == nullptr || user == stream_) return;
  mark_other_op();
  HPSB_CUDA(cudaEventRecord(ev_out_, stream_));
  HPSB_CUDA(cudaStreamWaitEvent(user, ev_out_, 0));
}

uint64_t DeviceCache::occupied() {
  std::lock_guard<std::mutex> lk(mu_);
  mark_other_op();
  DeviceGuard g(device_);
  HPSB_CUDA(cudaMemcpyAsync(h_small_ + 7, dev_.occupied, 8, cudaMemcpyDeviceToHost, stream_));
  HPSB_CUDA(cudaStreamSynchronize(stream_));
  return h_small_[7];
}

size_t DeviceCache::query(const uint64_t* keys, size_t n, float* out, size_t out_len,
                          uint32_t* miss_pos, uint64_t* miss_keys, int mem, cudaStream_t user) {
  std::lock_guard<std::mutex> lk(mu_);
  mark_other_op();
  // one tick per call, before anything else (slab_cache.cpp:73-74)
  const uint64_t stamp = bump_clock();
  if (out_len != n * uint64_t(cfg_.dimension))
    throw invalid_argument("query output buffer has wrong size");
  if (n == 0) return 0;
  DeviceGuard g(device_);
  const uint64_t d = cfg_.dimension;
  const bool host = mem == kHostMem;
  ensure_scan_tiles((n + kScanTile - 1) / kScanTile);
  if (host && n <= kZeroCopyQueryMax) {
    // Zero-copy (the reference's batch sizes): the kernels read the keys from
    // and write hit rows, hit flags, miss positions / keys and the miss count
    // to pinned host memory -- the caller's own buffers when they are pinned,
    // else a pinned staging area copied on the host (only HIT rows go back
    // into `out`: miss rows stay untouched, slab_cache.cpp:84-89). One host
    // wait, no copy-engine operations.
    const uint64_t sb = align256(n * 8) + align256(n * d * 4) + align256(n) + align256(n * 4) +
                        align256(n * 8);
    Carver hv{static_cast<char*>(qstage_.ensure(sb))};
    uint64_t* hk = hv.take<uint64_t>(n);
    float* hrows = hv.take<float>(n * d);
    uint8_t* hhit = hv.take<uint8_t>(n);
    uint32_t* hpos = hv.take<uint32_t>(n);
    uint64_t* hmk = hv.take<uint64_t>(n);
    const uint64_t* zk = static_cast<const uint64_t*>(host_mapped(keys));
    if (zk == nullptr) {
      std::memcpy(hk, keys, n * 8);
      zk = hk;
    }
    float* zo = static_cast<float*>(host_mapped(out));
    uint32_t* zp = static_cast<uint32_t*>(host_mapped(miss_pos));
    uint64_t* zm = static_cast<uint64_t*>(host_mapped(miss_keys));
    launch_cache_query(dev_, zk, n, zo ? zo : hrows, hhit, stamp, keys_per_warp_, stream_);
    launch_select_misses(zk, hhit, n, zp ? zp : hpos, zm ? zm : hmk, h_small_, scan_, stream_);
    HPSB_CUDA(cudaStreamSynchronize(stream_));
    const size_t n_miss = h_small_[0];
    if (zo == nullptr) {
      for (uint64_t i = 0; i < n; ++i)
        if (hhit[i]) std::memcpy(out + i * d, hrows + i * d, d * 4);
    }
    if (zp == nullptr) std::memcpy(miss_pos, hpos, n_miss * 4);
    if (zm == nullptr) std::memcpy(miss_keys, hmk, n_miss * 8);
    return n_miss;
  }
  const uint64_t bytes = align256(n) + (host ? align256(n * 8) * 2 + align256(n * d * 4) +
                                                   align256(n * 4)
                                             : 0);
  Carver cv{static_cast<char*>(scratch(bytes))};
  uint8_t* d_hit = cv.take<uint8_t>(n);
  const uint64_t* d_keys = keys;
  float* d_out = out;
  uint32_t* d_mpos = miss_pos;
  uint64_t* d_mkeys = miss_keys;
  if (host) {
    uint64_t* k = cv.take<uint64_t>(n);
    d_out = cv.take<float>(n * d);
    d_mpos = cv.take<uint32_t>(n);
    d_mkeys = cv.take<uint64_t>(n);
    HPSB_CUDA(cudaMemcpyAsync(k, keys, n * 8, cudaMemcpyHostToDevice, stream_));
    // miss rows must come back untouched: start from the caller's bytes
    HPSB_CUDA(cudaMemcpyAsync(d_out, out, n * d * 4, cudaMemcpyHostToDevice, stream_));
    d_keys = k;
  } else {
    join_from(user);
  }
  launch_cache_query(dev_, d_keys, n, d_out, d_hit, stamp, keys_per_warp_, stream_);
  launch_select_misses(d_keys, d_hit, n, d_mpos, d_mkeys, d_small_, scan_, stream_);
  HPSB_CUDA(cudaMemcpyAsync(h_small_, d_small_, 8, cudaMemcpyDeviceToHost, stream_));
  HPSB_CUDA(cudaStreamSynchronize(stream_));
  const size_t n_miss = h_small_[0];
  if (host) {
    HPSB_CUDA(cudaMemcpyAsync(out, d_out, n * d * 4, cudaMemcpyDeviceToHost, stream_));
    if (n_miss) {
      HPSB_CUDA(cudaMemcpyAsync(miss_pos, d_mpos, n_miss * 4, cudaMemcpyDeviceToHost, stream_));
      HPSB_CUDA(
          cudaMemcpyAsync(miss_keys, d_mkeys, n_miss * 8, cudaMemcpyDeviceToHost, stream_));
    }
    HPSB_CUDA(cudaStreamSynchronize(stream_));
  } else {
    join_to(user);
  }
  return n_miss;
}

void DeviceCache::lookup_device(const uint64_t* keys, size_t n, float* out, uint8_t* flags,
                                const float* default_row, uint64_t* miss_keys,
                                uint32_t* miss_firsts, uint64_t* counts, cudaStream_t user) {
  std::lock_guard<std::mutex> lk(mu_);
  DeviceGuard g(device_);
  join_from(user);
  // inside a stream capture (the cache's stream joined it through join_from):
  // the call's stamp and view generation become relative to the rebase words
  // of this cache's capture session (graph_before_launch_locked)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  unsigned long long cid = 0;
  HPSB_CUDA(cudaStreamGetCaptureInfo(stream_, &cs, &cid));
  const bool capturing = cs == cudaStreamCaptureStatusActive;
  if (capturing && cap_.id != cid) {
    if (cap_.id != 0) throw invalid_argument("cache is already part of another stream capture");
    if (free_slots_.empty()) throw invalid_argument("too many live captured graphs on this cache");
    cap_.id = cid;
    cap_.slot = free_slots_.back();
    free_slots_.pop_back();
    cap_.clock0 = clock_.load(std::memory_order_relaxed);
    for (int k = 0; k < kLookupViews; ++k) cap_.uses0[k] = lws_.uses[k];
    mark_other_op();  // the first captured lookup chains onto nothing
    std::lock_guard<std::mutex> rl(g_reg_mu);
    g_sessions[cid].push_back(this);
  }
  const uint64_t stamp = bump_clock();
  if (n == 0) {
    mark_other_op();
    HPSB_CUDA(cudaMemsetAsync(counts, 0, 16, stream_));
    join_to(user);
    return;
  }
  if (n >= (1ull << 32)) throw invalid_argument("lookup batch too large");
  if (n > lcap_) {
    if (capturing)
      throw invalid_argument("run one lookup of this batch size before capturing lookups");
    // (re)carve: miss table >= 2n entries, per-position slots, claim list,
    // counters, hit tables -- zeroed once, then kept clean by the kernels
    uint64_t cap = 1024;
    while (cap < n) cap <<= 1;
    const uint64_t bytes = lookup_scratch_bytes(cap);
    void* b = lbuf_.ensure(bytes, stream_);
    HPSB_CUDA(cudaMemsetAsync(b, 0, bytes, stream_));
    mark_other_op();
    lws_ = lookup_scratch_carve(b, cap);
    lcap_ = cap;
  }
  // programmatic dependent of the previous lookup when nothing else was
  // enqueued in between (the kernel orders itself against it)
  static const bool no_pdl = std::getenv("HPSB_NO_PDL") != nullptr;
  if (!capturing) prepare_hits(lws_, stamp);  // (may enqueue a clear first)
  const bool after_update = last_op_update_;
  // (never inside a cache group: other caches' work shares the stream)
  const bool chain = (last_op_lookup_ || last_op_update_) && !no_pdl &&
                     stream_holder_.use_count() == 1;
  LookupView v = lookup_next_view(lws_, chain);
  uint64_t kstamp = stamp;
  if (capturing) {
    kstamp = stamp - cap_.clock0;
    v.gen -= cap_.uses0[v.idx];
    if (v.prev_completed != nullptr) v.prev_target -= cap_.uses0[v.prev_idx];
    v.rebase = rebase_ + uint64_t(cap_.slot) * 16;
  }
  static const bool tracing = std::getenv("HPSB_TRACE") != nullptr;
  if (tracing) {
    if (trace_ == nullptr) {
      HPSB_CUDA(cudaMalloc(&trace_, kTraceRing * 64));
      HPSB_CUDA(cudaMemsetAsync(trace_, 0xFF, kTraceRing * 64, stream_));
      mark_other_op();
    }
    v.trace = trace_ + (trace_calls_++ % kTraceRing) * 8;
  }
  v.list_keys = miss_keys;
  v.list_firsts = miss_firsts;
  v.counts_out = reinterpret_cast<unsigned long long*>(counts);
  // profile events: external records when the stream is being captured into
  // a CUDA graph, so the timestamps stay readable after graph launches
  const unsigned rec_flags = capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
  if (prof_start_) {
    HPSB_CUDA(cudaEventRecordWithFlags(prof_start_, stream_, rec_flags));
    mark_other_op();
  }
  launch_lookup_probe(dev_, keys, n, out, flags, default_row, kstamp, v, chain, stream_,
                      /*wait_before_copy=*/after_update);
  mark_other_op();
  last_op_lookup_ = true;
  if (prof_end_) {
    HPSB_CUDA(cudaEventRecordWithFlags(prof_end_, stream_, rec_flags));
    mark_other_op();
  }
  join_to(user);
}

void DeviceCache::prepare_hits(LookupScratch& ls, uint64_t stamp) {
  if ((stamp >> 32) == ls.hit_epoch) return;
  // every 2^32 stamps: an entry of the previous epoch could carry this
  // call's tag (stream-ordered after every earlier lookup)
  HPSB_CUDA(cudaMemsetAsync(ls.hits_base, 0, ls.hits_bytes, stream_));
  mark_other_op();
  ls.hit_epoch = stamp >> 32;
}

std::vector<GraphCacheUse> DeviceCache::end_capture(unsigned long long capture_id) {
  std::vector<DeviceCache*> caches;
  {
    std::lock_guard<std::mutex> rl(g_reg_mu);
    auto it = g_sessions.find(capture_id);
    if (it == g_sessions.end()) return {};
    caches = std::move(it->second);
    g_sessions.erase(it);
  }
  std::vector<GraphCacheUse> out;
  for (DeviceCache* c : caches) {
    std::lock_guard<std::mutex> lk(c->mu_);
    GraphCacheUse u;
    u.cache = c;
    u.serial = c->serial_;
    u.slot = c->cap_.slot;
    // what one replay consumes; the capture itself consumed nothing
    u.stamps = c->clock_.load(std::memory_order_relaxed) - c->cap_.clock0;
    c->clock_.store(c->cap_.clock0, std::memory_order_relaxed);
    for (int k = 0; k < kLookupViews; ++k) {
      u.uses[k] = c->lws_.uses[k] - c->cap_.uses0[k];
      c->lws_.uses[k] = c->cap_.uses0[k];
    }
    c->cap_ = CaptureSession{};
    c->mark_other_op();
    out.push_back(u);
  }
  return out;
}

void DeviceCache::graph_before_launch_locked(const GraphCacheUse& u, cudaStream_t x) {
  DeviceGuard g(device_);
  if (x != stream_) {
    // earlier work of the cache precedes the graph
    HPSB_CUDA(cudaEventRecord(ev_in_, stream_));
    HPSB_CUDA(cudaStreamWaitEvent(x, ev_in_, 0));
  }
  if (u.stamps >= (1ull << 31)) throw invalid_argument("captured graph holds too many lookups");
  uint64_t base = clock_.load(std::memory_order_relaxed);
  if (u.stamps > 0) {
    // the replay's stamps base+1 .. base+stamps share their high 32 bits and
    // none has zero low bits (the tag value of a free hit-table entry)
    if (((base + 1) >> 32) != ((base + u.stamps) >> 32)) base = ((base + u.stamps) >> 32) << 32;
    const uint64_t epoch = (base + 1) >> 32;
    if (lws_.hits_base != nullptr && lws_.hit_epoch != epoch) {
      HPSB_CUDA(cudaMemsetAsync(lws_.hits_base, 0, lws_.hits_bytes, x));
      lws_.hit_epoch = epoch;
    }
  }
  unsigned long long ub[kLookupViews];
  for (int k = 0; k < kLookupViews; ++k) ub[k] = lws_.uses[k];
  launch_rebase(rebase_ + uint64_t(u.slot) * 16, base, ub, x);
  clock_.store(base + u.stamps, std::memory_order_relaxed);
  for (int k = 0; k < kLookupViews; ++k) lws_.uses[k] += u.uses[k];
  mark_other_op();
}

void DeviceCache::graph_after_launch_locked(cudaStream_t x) {
  DeviceGuard g(device_);
  if (x != stream_) {
    // later work of the cache follows the graph
    HPSB_CUDA(cudaEventRecord(ev_out_, x));
    HPSB_CUDA(cudaStreamWaitEvent(stream_, ev_out_, 0));
  }
  mark_other_op();
}

void DeviceCache::release_rebase_slot(int slot) {
  std::lock_guard<std::mutex> lk(mu_);
  if (slot >= 0) free_slots_.push_back(slot);
}

bool DeviceCache::alive(const DeviceCache* c, uint64_t serial) {
  std::lock_guard<std::mutex> rl(g_reg_mu);
  auto it = g_alive.find(c);
  return it != g_alive.end() && it->second == serial;
}

void DeviceCache::replace(const uint64_t* keys, size_t n, const float* vectors,
                          size_t vectors_len, int mem, cudaStream_t user) {
  std::lock_guard<std::mutex> lk(mu_);
  mark_other_op();
  if (vectors_len != n * uint64_t(cfg_.dimension))
    throw invalid_argument("replace vector buffer has wrong size");
  const bool host = mem == kHostMem;
  if (host) {
    std::unordered_set<uint64_t> distinct(keys, keys + n);
    if (distinct.size() != n) throw invalid_argument("replace batch contains duplicate keys");
  }
  if (n == 0) return;
  DeviceGuard g(device_);
  const uint64_t d = cfg_.dimension;
  const uint64_t stamp = clock_.load(std::memory_order_relaxed);  // no increment
  const ReplaceScratch& rs = replace_scratch_locked(n);
  const uint64_t bytes = host ? align256(n * 8) + align256(n * d * 4) : 256;
  Carver cv{static_cast<char*>(scratch(bytes))};
  const uint64_t* d_keys = keys;
  const float* d_rows = vectors;
  if (host && n <= kZeroCopyReplaceMax) {
    // zero-copy: the one-launch small replace reads the keys and rows from
    // pinned host memory (the caller's when pinned, else a pinned staging copy)
    const uint64_t sb = align256(n * 8) + align256(n * d * 4);
    Carver hv{static_cast<char*>(qstage_.ensure(sb))};
    uint64_t* hk = hv.take<uint64_t>(n);
    float* hr = hv.take<float>(n * d);
    d_keys = static_cast<const uint64_t*>(host_mapped(keys));
    d_rows = static_cast<const float*>(host_mapped(vectors));
    if (d_keys == nullptr) {
      std::memcpy(hk, keys, n * 8);
      d_keys = hk;
    }
    if (d_rows == nullptr) {
      std::memcpy(hr, vectors, n * d * 4);
      d_rows = hr;
    }
  } else if (host) {
    uint64_t* k = cv.take<uint64_t>(n);
    float* r = cv.take<float>(n * d);
    HPSB_CUDA(cudaMemcpyAsync(k, keys, n * 8, cudaMemcpyHostToDevice, stream_));
    HPSB_CUDA(cudaMemcpyAsync(r, vectors, n * d * 4, cudaMemcpyHostToDevice, stream_));
    d_keys = k;
    d_rows = r;
  } else {
    join_from(user);
  }
  launch_replace_mode(d_keys, n, d_rows, stamp, /*validate=*/!host, rs);
  if (host) {
    HPSB_CUDA(cudaStreamSynchronize(stream_));
    return;
  }
  HPSB_CUDA(cudaMemcpyAsync(h_small_ + 1, rs.cursor, 8, cudaMemcpyDeviceToHost, stream_));
  HPSB_CUDA(cudaStreamSynchronize(stream_));
  const uint32_t dup = reinterpret_cast<const uint32_t*>(h_small_ + 1)[1];
  if (dup) throw invalid_argument("replace batch contains duplicate keys");
  join_to(user);
}

void DeviceCache::replace_device_async(const uint64_t* keys, size_t n, const float* rows,
                                       cudaStream_t user) {
  std::lock_guard<std::mutex> lk(mu_);
  DeviceGuard g(device_);
  join_from(user);
  replace_device_locked(keys, n, rows);
  join_to(user);
}

void DeviceCache::reserve_replace(uint64_t n) {
  std::lock_guard<std::mutex> lk(mu_);
  DeviceGuard g(device_);
  replace_scratch_locked(n);
}

const ReplaceScratch& DeviceCache::replace_scratch_locked(uint64_t n) {
  if (n >= (1ull << 31)) throw invalid_argument("replace batch too large");
  if (n > rcap_) {
    // persistent: the replace kernels leave it clean, so calls need no
    // memsets; (re)initialised only when it grows
    uint64_t cap = 1024;
    while (cap < n) cap <<= 1;
    void* b = rbuf_.ensure(replace_scratch_bytes(cap), stream_);
    rs_ = replace_scratch_carve(b, cap);
    replace_scratch_init(rs_, stream_);
    relaxed_buf_.ensure(cap * 8, stream_);
    rcap_ = cap;
    mark_other_op();
  }
  return rs_;
}

void DeviceCache::replace_device_locked(const uint64_t* d_keys, size_t n, const float* d_rows) {
  mark_other_op();
  if (n == 0) return;
  const uint64_t stamp = clock_.load(std::memory_order_relaxed);
  const ReplaceScratch& rs = replace_scratch_locked(n);
  launch_replace_mode(d_keys, n, d_rows, stamp, /*validate=*/false, rs);
}

void DeviceCache::launch_replace_mode(const uint64_t* d_keys, uint64_t n, const float* d_rows,
                                      uint64_t stamp, bool validate, const ReplaceScratch& rs) {
  // slot d_small_[6]: the relaxed mode's dropped-key count
  if (!validate && replace_mode() == 1 && dev_.W <= 4) {
    // each key's claimed slot (sized with the replace scratch)
    uint64_t* claimed = static_cast<uint64_t*>(relaxed_buf_.get());
    launch_replace_relaxed(dev_, d_keys, n, d_rows, stamp, claimed, d_small_ + 6, stream_);
    return;
  }
  launch_replace(dev_, d_keys, n, d_rows, stamp, validate, rs, stream_, device_);
}

void DeviceCache::peer_export(uint64_t inbox_cap, PeerBlob* out) {
  std::lock_guard<std::mutex> lk(mu_);
  DeviceGuard g(device_);
  if (inbox_ == nullptr) {
    if (inbox_cap == 0) throw invalid_argument("peer inbox capacity must be positive");
    HPSB_CUDA(cudaMalloc(&inbox_, 256 + inbox_cap * 8));
    HPSB_CUDA(cudaMemsetAsync(inbox_, 0, 256, stream_));
    // from here on the recency clock lives in device memory ([1] of the
    // inbox header): peers tick it, drains read it back
    h_small_[4] = clock_.load(std::memory_order_relaxed);
    HPSB_CUDA(cudaMemcpyAsync(static_cast<char*>(inbox_) + 8, h_small_ + 4, 8,
                              cudaMemcpyHostToDevice, stream_));
    HPSB_CUDA(cudaStreamSynchronize(stream_));
    inbox_cap_ = inbox_cap;
  }
  PeerBlob b;
  b.magic = kPeerBlobMagic;
  b.S = cfg_.slabset_count;
  b.W = cfg_.slabs_per_set;
  b.d = cfg_.dimension;
  const char* pm = static_cast<const char*>(probe_mem_);
  b.tags_off = uint64_t(reinterpret_cast<const char*>(dev_.tags) - pm);
  b.masks_off = uint64_t(reinterpret_cast<const char*>(dev_.masks) - pm);
  b.ctr_off = uint64_t(reinterpret_cast<const char*>(dev_.counters) - pm);
  b.inbox_cap = inbox_cap_;
  b.device = device_;
  HPSB_CUDA(cudaIpcGetMemHandle(&b.probe, probe_mem_));
  HPSB_CUDA(cudaIpcGetMemHandle(&b.rows, dev_.rows));
  HPSB_CUDA(cudaIpcGetMemHandle(&b.inbox, inbox_));
  *out = b;
}

void DeviceCache::peer_inbox(unsigned long long** count, uint64_t** keys, uint64_t* cap) const {
  if (inbox_ == nullptr) throw invalid_argument("cache is not exported for peers");
  *count = static_cast<unsigned long long*>(inbox_);
  *keys = reinterpret_cast<uint64_t*>(static_cast<char*>(inbox_) + 256);
  *cap = inbox_cap_;
}

size_t DeviceCache::peer_drain(uint64_t* out, size_t cap) {
  std::lock_guard<std::mutex> lk(mu_);
  if (inbox_ == nullptr) throw invalid_argument("cache is not exported for peers");
  mark_other_op();
  DeviceGuard g(device_);
  // the peers' appends are done (caller's contract); the device is
  // synchronised so appends from other streams / processes have landed
  HPSB_CUDA(cudaDeviceSynchronize());
  HPSB_CUDA(cudaMemcpy(h_small_ + 4, inbox_, 16, cudaMemcpyDeviceToHost));
  const uint64_t appended = h_small_[4];
  // the shard's clock as the peers ticked it: this owner's replaces stamp
  // with it (slab_cache.cpp:105)
  uint64_t cur = clock_.load(std::memory_order_relaxed);
  while (cur < h_small_[5] && !clock_.compare_exchange_weak(cur, h_small_[5])) {
  }
  // and back: ticks of this cache's own host-side queries reach the peers
  h_small_[5] = clock_.load(std::memory_order_relaxed);
  HPSB_CUDA(cudaMemcpy(static_cast<char*>(inbox_) + 8, h_small_ + 5, 8, cudaMemcpyHostToDevice));
  const uint64_t m = std::min<uint64_t>({appended, inbox_cap_, uint64_t(cap)});
  if (m > 0)
    HPSB_CUDA(cudaMemcpy(out, static_cast<char*>(inbox_) + 256, m * 8, cudaMemcpyDeviceToHost));
  HPSB_CUDA(cudaMemset(inbox_, 0, 8));
  return size_t(appended);
}

void DeviceCache::set_replace_mode(int mode) {
  if (mode != 0 && mode != 1) throw invalid_argument("replace mode must be 0 (exact) or 1 (relaxed)");
  std::lock_guard<std::mutex> lk(mu_);
  replace_mode_.store(mode, std::memory_order_relaxed);
}

uint64_t DeviceCache::relaxed_dropped() {
  std::lock_guard<std::mutex> lk(mu_);
  mark_other_op();
  DeviceGuard g(device_);
  HPSB_CUDA(cudaMemcpyAsync(h_small_ + 6, d_small_ + 6, 8, cudaMemcpyDeviceToHost, stream_));
  HPSB_CUDA(cudaStreamSynchronize(stream_));
  return h_small_[6];
}

size_t DeviceCache::update(const uint64_t* keys, size_t n, const float* vectors,
                           size_t vectors_len, int mem, cudaStream_t user) {
  std::lock_guard<std::mutex> lk(mu_);
  mark_other_op();
  if (vectors_len != n * uint64_t(cfg_.dimension))
    throw invalid_argument("update vector buffer has wrong size");
  if (n == 0) return 0;
  if (n >= (1ull << 32) - 1) throw invalid_argument("update batch too large");
  DeviceGuard g(device_);
  const uint64_t d = cfg_.dimension;
  const bool host = mem == kHostMem;
  const uint64_t ub = update_scratch_bytes(n);
  const uint64_t bytes = align256(ub) + (host ? align256(n * 8) + align256(n * d * 4) : 0);
  Carver cv{static_cast<char*>(scratch(bytes))};
  void* scratch_u = cv.take<char>(ub);
  const uint64_t* d_keys = keys;
  const float* d_rows = vectors;
  if (host) {
    uint64_t* k = cv.take<uint64_t>(n);
    float* r = cv.take<float>(n * d);
    HPSB_CUDA(cudaMemcpyAsync(k, keys, n * 8, cudaMemcpyHostToDevice, stream_));
    HPSB_CUDA(cudaMemcpyAsync(r, vectors, n * d * 4, cudaMemcpyHostToDevice, stream_));
    d_keys = k;
    d_rows = r;
  } else {
    join_from(user);
  }
  launch_update(dev_, d_keys, n, d_rows, scratch_u, next_winner(), d_small_ + 2,
                /*after_lookup=*/false, stream_);
  HPSB_CUDA(cudaMemcpyAsync(h_small_ + 2, d_small_ + 2, 8, cudaMemcpyDeviceToHost, stream_));
  HPSB_CUDA(cudaStreamSynchronize(stream_));
  if (!host) join_to(user);
  return h_small_[2];
}

void DeviceCache::update_device(const uint64_t* keys, size_t n, const float* vectors,
                                uint64_t* written, cudaStream_t user) {
  std::lock_guard<std::mutex> lk(mu_);
  static const bool no_pdl = std::getenv("HPSB_NO_PDL") != nullptr;
  // right behind a lookup kernel: the probe overlaps that lookup (and
  // completes after it); the next lookup may overlap this update the same way
  const bool after_lookup = last_op_lookup_ && !no_pdl && stream_holder_.use_count() == 1 &&
                            (user == nullptr || user == stream_);
  mark_other_op();
  if (n >= (1ull << 32) - 1) throw invalid_argument("update batch too large");
  DeviceGuard g(device_);
  join_from(user);
  bool chain = after_lookup;
  // two scratch halves: the next update's probe may overlap this write
  if (n > ucap_) {
    uint64_t cap = 1024;
    while (cap < n) cap <<= 1;
    ubuf_.ensure(2 * (align256(update_scratch_bytes(cap)) + 256), stream_);
    ucap_ = cap;
    chain = false;  // (re)allocation enqueued work in between
  }
  uint32_t* winner = next_winner();
  const uint64_t half = align256(update_scratch_bytes(ucap_)) + 256;
  char* ub = static_cast<char*>(ubuf_.get()) + (winner == winner_ ? 0 : half);
  unsigned long long* w = written != nullptr
                              ? reinterpret_cast<unsigned long long*>(written)
                              : reinterpret_cast<unsigned long long*>(
                                    ub + align256(update_scratch_bytes(ucap_)));
  launch_update(dev_, keys, n, vectors, ub, winner, w, chain, stream_);
  last_op_update_ = n > 0 && (user == nullptr || user == stream_);
  join_to(user);
}

size_t DeviceCache::dump(uint64_t set_begin, uint64_t set_end, uint64_t* out, size_t cap) {
  std::lock_guard<std::mutex> lk(mu_);
  mark_other_op();
  set_end = std::min<uint64_t>(set_end, cfg_.slabset_count);
  if (set_begin >= set_end) return 0;
  DeviceGuard g(device_);
  const uint64_t slots = (set_end - set_begin) * cfg_.slabs_per_set * 32ull;
  ensure_scan_tiles(((set_end - set_begin) * cfg_.slabs_per_set + kDumpTile - 1) / kDumpTile);
  uint64_t* d_out = static_cast<uint64_t*>(scratch(slots * 8));
  launch_dump(dev_, set_begin, set_end, d_out, d_small_ + 3, scan_, stream_);
  HPSB_CUDA(cudaMemcpyAsync(h_small_ + 3, d_small_ + 3, 8, cudaMemcpyDeviceToHost, stream_));
  HPSB_CUDA(cudaStreamSynchronize(stream_));
  const size_t n = h_small_[3];
  const size_t take = std::min(n, cap);
  if (take) {
    HPSB_CUDA(cudaMemcpyAsync(out, d_out, take * 8, cudaMemcpyDeviceToHost, stream_));
    HPSB_CUDA(cudaStreamSynchronize(stream_));
  }
  return n;
}

uint64_t DeviceCache::trace(unsigned long long* out) {
  std::lock_guard<std::mutex> lk(mu_);
  if (trace_ == nullptr) return 0;
  mark_other_op();
  DeviceGuard g(device_);
  HPSB_CUDA(cudaMemcpyAsync(out, trace_, kTraceRing * 64, cudaMemcpyDeviceToHost, stream_));
  HPSB_CUDA(cudaMemsetAsync(trace_, 0xFF, kTraceRing * 64, stream_));
  HPSB_CUDA(cudaStreamSynchronize(stream_));
  const uint64_t n = trace_calls_;
  trace_calls_ = 0;
  return n;
}

void DeviceCache::dump_device(uint64_t set_begin, uint64_t set_end, uint64_t* out,
                              uint64_t* n_out, cudaStream_t user) {
  std::lock_guard<std::mutex> lk(mu_);
  mark_other_op();
  set_end = std::min<uint64_t>(set_end, cfg_.slabset_count);
  DeviceGuard g(device_);
  join_from(user);
  if (set_begin >= set_end) {
    HPSB_CUDA(cudaMemsetAsync(n_out, 0, 8, stream_));
  } else {
    ensure_scan_tiles(((set_end - set_begin) * cfg_.slabs_per_set + kDumpTile - 1) / kDumpTile);
    launch_dump(dev_, set_begin, set_end, out, reinterpret_cast<unsigned long long*>(n_out),
                scan_, stream_);
  }
  join_to(user);
}

void DeviceCache::export_state(uint64_t* keys, uint64_t* counters, uint32_t* masks,
                               float* rows) {
  std::lock_guard<std::mutex> lk(mu_);
  mark_other_op();
  DeviceGuard g(device_);
  const uint64_t slabs = cfg_.slabset_count * cfg_.slabs_per_set;
  const uint64_t slots = slabs * 32ull;
  if (keys) HPSB_CUDA(cudaMemcpyAsync(keys, dev_.keys, slots * 8, cudaMemcpyDeviceToHost, stream_));
  if (counters)
    HPSB_CUDA(
        cudaMemcpyAsync(counters, dev_.counters, slots * 8, cudaMemcpyDeviceToHost, stream_));
  if (masks) HPSB_CUDA(cudaMemcpyAsync(masks, dev_.masks, slabs * 4, cudaMemcpyDeviceToHost, stream_));
  if (rows)
    HPSB_CUDA(cudaMemcpyAsync(rows, dev_.rows, slots * uint64_t(cfg_.dimension) * 4,
                              cudaMemcpyDeviceToHost, stream_));
  HPSB_CUDA(cudaStreamSynchronize(stream_));
}

void DeviceCache::check_invariants() {
  const uint64_t S = cfg_.slabset_count, W = cfg_.slabs_per_set;
  const uint64_t slots = S * W * 32;
  std::vector<uint64_t> keys(slots), ctr(slots);
  std::vector<uint32_t> masks(S * W);
  std::vector<uint8_t> tags(slots);
  uint64_t occ = 0, clock_now = 0;
  {
    // one consistent snapshot: keys, counters, masks, fingerprints, the
    // occupancy counter and the clock under ONE hold of the cache mutex and
    // one stream sync (the reference holds every set gate for the whole
    // check, slab_cache.cpp:407-442), so a concurrent replace or engine fill
    // cannot slip in between the copies
    std::lock_guard<std::mutex> lk(mu_);
    mark_other_op();
    DeviceGuard g(device_);
    HPSB_CUDA(cudaMemcpyAsync(keys.data(), dev_.keys, slots * 8, cudaMemcpyDeviceToHost, stream_));
    HPSB_CUDA(cudaMemcpyAsync(ctr.data(), dev_.counters, slots * 8, cudaMemcpyDeviceToHost, stream_));
    HPSB_CUDA(cudaMemcpyAsync(masks.data(), dev_.masks, S * W * 4, cudaMemcpyDeviceToHost, stream_));
    HPSB_CUDA(cudaMemcpyAsync(tags.data(), dev_.tags, slots, cudaMemcpyDeviceToHost, stream_));
    HPSB_CUDA(cudaMemcpyAsync(h_small_ + 7, dev_.occupied, 8, cudaMemcpyDeviceToHost, stream_));
    HPSB_CUDA(cudaStreamSynchronize(stream_));
    occ = h_small_[7];
    clock_now = recency_clock();
  }
  std::unordered_set<uint64_t> seen;
  seen.reserve(occ);
  uint64_t populated = 0;
  for (uint64_t set = 0; set < S; ++set) {
    for (uint64_t slab = 0; slab < W; ++slab) {
      const uint32_t m = masks[set * W + slab];
      // masks only grow contiguously from bit 0 (no erase; eviction in place)
      if ((m & (m + 1)) != 0) throw logic_error("slab cache occupancy mask is not contiguous");
      for (uint32_t j = 0; j < 32; ++j) {
        if (!((m >> j) & 1u)) continue;
        ++populated;
        const uint64_t slot = (set * W + slab) * 32 + j;
        const uint64_t key = keys[slot];
        // same checks and messages as slab_cache.cpp:425-436
        if (hpsb::xxh64_key(key, kSlabsetSeed) % S != set)
          throw logic_error("slab cache key stored outside its slabset");
        if (!seen.insert(key).second) throw logic_error("slab cache holds a key in two slots");
        if (ctr[slot] > clock_now) throw logic_error("slab cache slot counter exceeds the clock");
        // B200 layout: the lookup kernel's probe filter must match the key
        if (tags[slot] != key_tag(hpsb::xxh64_key(key, kSlabSeed)))
          throw logic_error("slab cache key fingerprint is out of sync");
      }
    }
  }
  if (populated != occ) throw logic_error("slab cache occupancy counter is out of sync");
}

}  // namespace hpsb
