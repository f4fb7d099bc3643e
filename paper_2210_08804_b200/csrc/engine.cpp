// engine.cpp -- see engine.hpp. Reference: /root/reference/proj/core/src/
// lookup_engine.cpp (tier_fetch :50-89, ctor checks :91-117, lookup
// :130-241, async_loop :243-284, drain_async :286-289).
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <unordered_map>

namespace hpsb {

namespace {
inline uint64_t a256(uint64_t v) { return (v + 255) / 256 * 256; }

// HPSB_ENGINE_TRACE=1: per-phase host timeline of lookups slower than 2 ms
// (diagnostic, stderr).
// HPSB_ENGINE_TRACE=1: calls slower than 2 ms print their phase timeline
// (from the start of begin); HPSB_ENGINE_TRACE=<us>: calls slower than that.
struct PhaseTrace {
  static bool on() {
    static const bool v = std::getenv("HPSB_ENGINE_TRACE") != nullptr;
    return v;
  }
  static double min_us() {
    static const double v = [] {
      const char* e = std::getenv("HPSB_ENGINE_TRACE");
      const double x = e ? std::atof(e) : 0.0;
      return (e == nullptr || x == 1.0) ? 2000.0 : x;
    }();
    return v;
  }
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double at[10] = {};
  const char* name[10] = {};
  int k = 0;
  void mark(const char* what) {
    if (!on() || k >= 10) return;
    name[k] = what;
    at[k++] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
                  .count();
  }
  void report(uint64_t n, uint64_t um, bool sync) {
    if (!on() || k == 0 || at[k - 1] < min_us()) return;
    std::fprintf(stderr, "[hpsb trace] n=%llu misses=%llu sync=%d", (unsigned long long)n,
                 (unsigned long long)um, int(sync));
    for (int i = 0; i < k; ++i) std::fprintf(stderr, " %s=%.0fus", name[i], at[i]);
    std::fprintf(stderr, "\n");
  }
};

// Device-accessible address of pinned host memory (cudaHostAlloc'd or
// registered), nullptr for pageable memory.
const void* mapped(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}
}  // namespace

// ------------------------------------------------------------- tier fetch --
void tier_fetch_staged(VolatileStore* vdb, const std::string& table, uint32_t dim,
                       ColdFetchFn cold, void* cold_ctx, const uint64_t* keys, size_t n,
                       uint64_t* found_keys, float* rows, int32_t* row_of, size_t* n_found,
                       uint64_t* missing_keys, size_t* n_missing, TierCounters* counters) {
  *n_found = 0;
  *n_missing = 0;
  if (n == 0) return;
  const bool use_vdb = vdb != nullptr && vdb->has_table(table);
  size_t nf = 0, nm = 0;
  std::vector<uint64_t> remaining;
  if (use_vdb) {
    remaining.resize(n);
    vdb->lookup(table, keys, n, found_keys, rows, row_of, &nf, remaining.data(), &nm);
    remaining.resize(nm);
    if (counters) counters->vdb_hits += nf;
  } else {
    remaining.assign(keys, keys + n);
    nm = n;
    for (size_t i = 0; i < n; ++i) row_of[i] = -1;
  }
  if (nm == 0) {
    *n_found = nf;
    return;
  }
  if (cold == nullptr) {
    // no cold tier wired: everything left is absent
    std::copy(remaining.begin(), remaining.end(), missing_keys);
    if (counters) counters->missing += nm;
    *n_found = nf;
    *n_missing = nm;
    return;
  }
  std::vector<uint64_t> cf_keys(nm), cm_keys(nm);
  std::vector<float> cf_rows(nm * uint64_t(dim));
  size_t cf = 0, cm = 0;
  const int rc = cold(cold_ctx, remaining.data(), nm, cf_keys.data(), cf_rows.data(), &cf,
                      cm_keys.data(), &cm);
  if (rc != 0) throw tier_fault("cold tier fetch failed");
  if (counters) {
    counters->cold_hits += cf;
    counters->missing += cm;
  }
  if (use_vdb && cf) {
    // promote cold reads (lookup_engine.cpp:76-81)
    vdb->insert_async(table, std::vector<uint64_t>(cf_keys.begin(), cf_keys.begin() + cf),
                      std::vector<float>(cf_rows.begin(), cf_rows.begin() + cf * dim));
  }
  std::copy(cf_keys.begin(), cf_keys.begin() + cf, found_keys + nf);
  std::copy(cf_rows.begin(), cf_rows.begin() + cf * dim, rows + nf * dim);
  // cold hits in the cold tier's own order (a tier that reads through
  // further levels, like the reference's tier_fetch, need not keep input
  // order): map them back by key (keys are unique)
  std::unordered_map<uint64_t, int32_t> cold_row;
  cold_row.reserve(cf * 2);
  for (size_t j = 0; j < cf; ++j) cold_row.emplace(cf_keys[j], int32_t(nf + j));
  for (size_t i = 0; i < n; ++i) {
    if (row_of[i] >= 0) continue;
    auto it = cold_row.find(keys[i]);
    if (it != cold_row.end()) row_of[i] = it->second;
  }
  std::copy(cm_keys.begin(), cm_keys.begin() + cm, missing_keys);
  *n_found = nf + cf;
  *n_missing = cm;
}

// ---------------------------------------------------------------- refresh --
// refresh_engine.cpp:5-22 (refresh_cache): the resident keys in dump order,
// batch by batch fetched from the tiers and written back with the
// non-admitting update. B200 pipeline: the host tier fetch of batch i+1
// (found rows land straight in pinned staging) overlaps the H2D copy and the
// device update of batch i (two staging buffers, stream-ordered on the
// cache's stream); the written counts stay on the device until the end.
RefreshResult refresh_cache(DeviceCache& cache, VolatileStore* vdb, const std::string& table,
                            ColdFetchFn cold, void* cold_ctx, size_t dump_batch) {
  if (dump_batch == 0) throw invalid_argument("dump batch size must be positive");
  RefreshResult r;
  const uint32_t d = cache.dimension();
  const uint64_t S = cache.slabset_count();
  DeviceCache::RefreshBuffers& rb = cache.refresh_buffers();
  std::lock_guard<std::mutex> lk(rb.mu);
  std::vector<uint64_t>& keys = rb.keys;
  keys.resize(S * cache.slabs_per_set() * 32ull);
  keys.resize(cache.dump(0, S, keys.data(), keys.size()));
  if (keys.empty()) return r;
  DeviceGuard g(cache.device());
  cudaStream_t st = cache.stream();
  const uint64_t nb = (keys.size() + dump_batch - 1) / dump_batch;
  struct Stage {
    cudaEvent_t done = nullptr;
    uint64_t* h_keys = nullptr;
    float* h_rows = nullptr;
    uint64_t* d_keys = nullptr;
    float* d_rows = nullptr;
  } stage[2];
  std::vector<uint64_t> missing(dump_batch);
  std::vector<int32_t> row_of(dump_batch);
  uint64_t* written = static_cast<uint64_t*>(rb.written.ensure(nb * 8, st));
  HPSB_CUDA(cudaMemsetAsync(written, 0, nb * 8, st));
  for (int x = 0; x < 2; ++x) {
    Stage& sg = stage[x];
    HPSB_CUDA(cudaEventCreateWithFlags(&sg.done, cudaEventDisableTiming));
    char* hp = static_cast<char*>(rb.h[x].ensure(dump_batch * (8 + uint64_t(d) * 4)));
    sg.h_keys = reinterpret_cast<uint64_t*>(hp);
    sg.h_rows = reinterpret_cast<float*>(hp + dump_batch * 8);
    char* dp = static_cast<char*>(rb.dv[x].ensure(dump_batch * (8 + uint64_t(d) * 4) + 256, st));
    sg.d_keys = reinterpret_cast<uint64_t*>(dp);
    sg.d_rows = reinterpret_cast<float*>(dp + (dump_batch * 8 + 255) / 256 * 256);
  }
  std::exception_ptr err;
  try {
    for (uint64_t b = 0; b < nb; ++b) {
      Stage& sg = stage[b & 1];
      HPSB_CUDA(cudaEventSynchronize(sg.done));  // staging b is free again
      const uint64_t k0 = b * dump_batch;
      const uint64_t m = std::min<uint64_t>(dump_batch, keys.size() - k0);
      size_t nf = 0, nm = 0;
      TierCounters tc;
      tier_fetch_staged(vdb, table, d, cold, cold_ctx, keys.data() + k0, m, sg.h_keys, sg.h_rows,
                        row_of.data(), &nf, missing.data(), &nm, &tc);
      r.unresolved.insert(r.unresolved.end(), missing.begin(), missing.begin() + nm);
      if (nf > 0) {
        HPSB_CUDA(cudaMemcpyAsync(sg.d_keys, sg.h_keys, nf * 8, cudaMemcpyHostToDevice, st));
        HPSB_CUDA(cudaMemcpyAsync(sg.d_rows, sg.h_rows, nf * uint64_t(d) * 4,
                                  cudaMemcpyHostToDevice, st));
        HPSB_CUDA(cudaEventRecord(sg.done, st));
        cache.update_device(sg.d_keys, nf, sg.d_rows, written + b, st);
      }
    }
  } catch (...) {
    // a tier fault aborts the pass; batches already applied stay applied
    // (refresh_engine.hpp:35-39)
    err = std::current_exception();
  }
  std::vector<uint64_t> w(nb);
  HPSB_CUDA(cudaMemcpyAsync(w.data(), written, nb * 8, cudaMemcpyDeviceToHost, st));
  HPSB_CUDA(cudaStreamSynchronize(st));
  for (auto& sg : stage) cudaEventDestroy(sg.done);
  for (uint64_t x : w) r.refreshed += x;
  if (err) std::rethrow_exception(err);
  return r;
}

// -------------------------------------------------------------- workspace --
Workspace::~Workspace() {
  if (done) {
    cudaEventSynchronize(done);
    cudaEventDestroy(done);
  }
  if (uploaded) {
    cudaEventSynchronize(uploaded);
    cudaEventDestroy(uploaded);
  }
  if (rows_ready) cudaEventDestroy(rows_ready);
  if (counts_ready) cudaEventDestroy(counts_ready);
  for (auto& e : chunk_ev)
    if (e) cudaEventDestroy(e);
}

void Workspace::wait_idle() {
  if (pending) {
    HPSB_CUDA(cudaEventSynchronize(done));
    pending = false;
  }
}

void Workspace::ensure(uint64_t n, uint32_t d, cudaStream_t st) {
  if (done == nullptr) HPSB_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  if (rows_ready == nullptr)
    HPSB_CUDA(cudaEventCreateWithFlags(&rows_ready, cudaEventDisableTiming));
  if (counts_ready == nullptr)
    HPSB_CUDA(cudaEventCreateWithFlags(&counts_ready, cudaEventDisableTiming));
  if (uploaded == nullptr)
    HPSB_CUDA(cudaEventCreateWithFlags(&uploaded, cudaEventDisableTiming));
  for (auto& e : chunk_ev)
    if (e == nullptr) HPSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (n <= capacity && d == dim && dbuf.get() != nullptr) return;
  uint64_t cap = 1024;
  while (cap < n) cap <<= 1;
  // one lookup view: a workspace serves one call at a time (wait_idle)
  const uint64_t ls_bytes = lookup_scratch_bytes(cap, 1);
  const uint64_t hdr_bytes = 16 + cap * 4 + 8 + cap * 8 + cap;
  const uint64_t dev_bytes = a256(cap * 8) * 3 + a256(cap * uint64_t(d) * 4) * 2 + a256(cap) +
                             a256(cap * 4) + a256(ls_bytes);
  HPSB_CUDA(cudaStreamSynchronize(st));
  char* p = static_cast<char*>(dbuf.ensure(dev_bytes, st));
  auto take = [&](uint64_t bytes) {
    char* r = p;
    p += a256(bytes);
    return r;
  };
  d_keys = reinterpret_cast<uint64_t*>(take(cap * 8));
  d_out = reinterpret_cast<float*>(take(cap * uint64_t(d) * 4));
  d_flags = reinterpret_cast<uint8_t*>(take(cap));
  d_row_of = reinterpret_cast<int32_t*>(take(cap * 4));
  d_staged = reinterpret_cast<float*>(take(cap * uint64_t(d) * 4));
  d_found_keys = reinterpret_cast<uint64_t*>(take(cap * 8));
  char* ls_base = take(ls_bytes);
  HPSB_CUDA(cudaMemsetAsync(ls_base, 0, ls_bytes, st));
  ls = lookup_scratch_carve(ls_base, cap, 1);

  const uint64_t host_bytes = a256(cap * 8) * 5 + a256(16) + a256(cap * 4) * 3 +
                              a256(cap * uint64_t(d) * 4) * 2 + a256(cap) + a256(hdr_bytes);
  char* h = static_cast<char*>(hbuf.ensure(host_bytes));
  auto htake = [&](uint64_t bytes) {
    char* r = h;
    h += a256(bytes);
    return r;
  };
  h_keys = reinterpret_cast<uint64_t*>(htake(cap * 8));
  h_counts = reinterpret_cast<unsigned long long*>(htake(16));
  h_miss_keys = reinterpret_cast<uint64_t*>(htake(cap * 8));
  h_row_of = reinterpret_cast<int32_t*>(htake(cap * 4));
  h_staged = reinterpret_cast<float*>(htake(cap * uint64_t(d) * 4));
  h_found_keys = reinterpret_cast<uint64_t*>(htake(cap * 8));
  h_missing = reinterpret_cast<uint64_t*>(htake(cap * 8));
  h_flags = reinterpret_cast<uint8_t*>(htake(cap));
  h_out = reinterpret_cast<float*>(htake(cap * uint64_t(d) * 4));
  h_claim_keys = reinterpret_cast<uint64_t*>(htake(cap * 8));
  h_claim_firsts = reinterpret_cast<uint32_t*>(htake(cap * 4));
  h_row_of_claim = reinterpret_cast<int32_t*>(htake(cap * 4));
  h_hdr = htake(hdr_bytes);
  HPSB_CUDA(cudaStreamSynchronize(st));
  capacity = cap;
  dim = d;
}

WorkspacePool::WorkspacePool(size_t size, int device) {
  if (size == 0) throw invalid_argument("workspace pool size must be positive");
  for (size_t i = 0; i < size; ++i) {
    slots_.push_back(std::make_unique<Workspace>());
    slots_.back()->device = device;
    free_.push_back(slots_.back().get());
  }
}

Workspace* WorkspacePool::acquire() {
  std::unique_lock<std::mutex> lk(mu_);
  cv_.wait(lk, [&] { return !free_.empty(); });
  Workspace* ws = free_.back();
  free_.pop_back();
  ++outstanding_;
  peak_ = std::max(peak_, outstanding_);
  return ws;
}

void WorkspacePool::release(Workspace* ws) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    free_.push_back(ws);
    --outstanding_;
  }
  cv_.notify_one();
}

size_t WorkspacePool::outstanding() const {
  std::lock_guard<std::mutex> lk(mu_);
  return outstanding_;
}
size_t WorkspacePool::peak_outstanding() const {
  std::lock_guard<std::mutex> lk(mu_);
  return peak_;
}

// ----------------------------------------------------------------- engine --
LookupEngine::LookupEngine(const std::string& table, uint32_t dim, DeviceCache* cache,
                           VolatileStore* vdb, ColdFetchFn cold, void* cold_ctx,
                           EngineConfig cfg)
    : table_(table),
      dim_(dim),
      cache_(cache),
      vdb_(vdb),
      cold_(cold),
      cold_ctx_(cold_ctx),
      cfg_(std::move(cfg)),
      pool_(cfg_.workspace_pool_size, cache ? cache->device() : 0),
      copy_threads_([] {
        const char* e = std::getenv("HPSB_COPY_THREADS");  // A/B knob
        const unsigned want = e ? unsigned(std::max(1, std::atoi(e))) : 8u;
        return std::min(want, std::max(1u, std::thread::hardware_concurrency()));
      }()) {
  if (table.empty()) throw invalid_argument("table name must not be empty");
  if (table.size() > 255) throw invalid_argument("table name exceeds 255 bytes: " + table);
  if (dim == 0) throw invalid_argument("table dimension must be positive: " + table);
  if (cache == nullptr) throw invalid_argument("engine needs a cache");
  if (cache->dimension() != dim) throw invalid_argument("cache dimension does not match table");
  if (cfg_.hit_rate_threshold < 0.0 || cfg_.hit_rate_threshold > 1.0)
    throw invalid_argument("hit_rate_threshold must be within [0, 1]");
  if (cfg_.async_worker_count == 0) throw invalid_argument("async_worker_count must be positive");
  std::vector<float> def = cfg_.default_vector;
  def.resize(dim, 0.0f);  // padded with zeros / cut to the dimension
  DeviceGuard g(cache->device());
  HPSB_CUDA(cudaMalloc(&d_default_, dim * 4));
  HPSB_CUDA(cudaMemcpy(d_default_, def.data(), dim * 4, cudaMemcpyHostToDevice));
  HPSB_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
  for (uint32_t i = 0; i < cfg_.async_worker_count; ++i)
    workers_.emplace_back([this] { async_loop(); });
  if (cfg_.max_batch) reserve(cfg_.max_batch);
}

LookupEngine::~LookupEngine() {
  {
    std::lock_guard<std::mutex> lk(q_mu_);
    stopping_ = true;
  }
  q_cv_.notify_all();
  for (auto& w : workers_) w.join();
  DeviceGuard g(cache_->device());
  cudaFree(d_default_);
  if (copy_stream_) {
    cudaStreamSynchronize(copy_stream_);
    cudaStreamDestroy(copy_stream_);
  }
}

void LookupEngine::rows_d2h(Workspace& ws, const LookupCall& c, cudaStream_t st) {
  const uint64_t bytes = c.n * uint64_t(dim_) * 4;
  if (c.out_pinned) {
    ws.out_chunks = 0;
    HPSB_CUDA(cudaMemcpyAsync(c.out, c.d_out, bytes, cudaMemcpyDeviceToHost, st));
    return;
  }
  // ~512 KB chunks (HPSB_OUT_CHUNK_SHIFT): the copy-on of chunk i runs while
  // later chunks cross PCIe; small chunks keep the tail after the last chunk
  // lands short (2 MB chunks left a ~0.2 ms single-thread copy after the DMA)
  static const int shift = [] {
    const char* e = std::getenv("HPSB_OUT_CHUNK_SHIFT");
    const int v = e ? std::atoi(e) : 19;
    return std::clamp(v, 16, 24);
  }();
  const uint64_t nch = std::clamp<uint64_t>(bytes >> shift, 1, Workspace::kOutChunks);
  const uint64_t per = (bytes / nch + 255) / 256 * 256;
  ws.out_chunks = 0;
  for (uint64_t off = 0; off < bytes; off += per) {
    const uint64_t len = std::min(per, bytes - off);
    HPSB_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(ws.h_out) + off,
                              reinterpret_cast<const char*>(c.d_out) + off, len,
                              cudaMemcpyDeviceToHost, st));
    HPSB_CUDA(cudaEventRecord(ws.chunk_ev[ws.out_chunks++], st));
  }
}

void LookupEngine::host_scatter(Workspace& ws, size_t n, const uint64_t* keys, float* out,
                                uint64_t um, uint8_t* hflags) {
  // found misses (ws.h_miss_keys in miss order, ws.h_row_of: staged row or -1)
  uint64_t cap = 16;
  while (cap < 2 * um) cap <<= 1;
  if (ws.hs_keys.size() < cap) {
    ws.hs_keys.resize(cap);
    ws.hs_rows.resize(cap);
    ws.hs_used.resize(cap);
  }
  std::fill(ws.hs_used.begin(), ws.hs_used.begin() + cap, uint8_t(0));
  const uint64_t mask = cap - 1;
  bool any = false;
  for (uint64_t k = 0; k < um; ++k) {
    if (ws.h_row_of[k] < 0) continue;
    any = true;
    const uint64_t key = ws.scatter_keys[k];
    uint64_t h = fmix64(key) & mask;
    while (ws.hs_used[h]) h = (h + 1) & mask;
    ws.hs_used[h] = 1;
    ws.hs_keys[h] = key;
    ws.hs_rows[h] = ws.h_row_of[k];
  }
  if (!any) return;
  const uint32_t d = dim_;
  const size_t chunks = std::min<size_t>(copy_threads_.size(), (n + 4095) / 4096);
  const size_t per = (n + chunks - 1) / chunks;
  copy_threads_.parallel_for(chunks, 1, [&](size_t cb, size_t ce) {
    for (size_t ch = cb; ch < ce; ++ch) {
      const size_t e = std::min(n, (ch + 1) * per);
      for (size_t p = ch * per; p < e; ++p) {
        if (!hflags[p]) continue;
        const uint64_t key = keys[p];
        uint64_t h = fmix64(key) & mask;
        while (ws.hs_used[h] && ws.hs_keys[h] != key) h = (h + 1) & mask;
        if (!ws.hs_used[h]) continue;  // absent from every tier: default row, flagged
        std::memcpy(out + p * d, ws.h_staged + uint64_t(ws.hs_rows[h]) * d, d * 4ull);
        hflags[p] = 0;
      }
    }
  });
}

void LookupEngine::rows_to_pageable(Workspace& ws, const LookupCall& c) {
  const uint64_t bytes = c.n * uint64_t(dim_) * 4;
  const int nch = ws.out_chunks;
  if (nch == 0) return;
  const uint64_t per = (bytes / uint64_t(nch) + 255) / 256 * 256;
  auto copy_chunk = [&](size_t i) {
    HPSB_CUDA(cudaEventSynchronize(ws.chunk_ev[i]));
    const uint64_t off = i * per;
    if (off >= bytes) return;
    std::memcpy(reinterpret_cast<char*>(c.out) + off, reinterpret_cast<const char*>(ws.h_out) + off,
                std::min(per, bytes - off));
  };
  if (nch == 1) {
    copy_chunk(0);
    return;
  }
  // thread t takes chunks t, t + T, ...: every thread starts on an early chunk
  const size_t T = std::min<size_t>(copy_threads_.size(), size_t(nch));
  copy_threads_.parallel_for(T, 1, [&](size_t tb, size_t te) {
    for (size_t t = tb; t < te; ++t)
      for (size_t i = t; i < size_t(nch); i += T) copy_chunk(i);
  });
}

size_t LookupEngine::fetch_and_upload(Workspace& ws, const uint64_t* miss_keys, size_t n_miss,
                                      TierCounters* counters, size_t* n_found) {
  size_t nf = 0, nm = 0;
  tier_fetch_staged(cfg_.volatile_tier_enabled ? vdb_ : nullptr, table_, dim_, cold_, cold_ctx_,
                    miss_keys, n_miss, ws.h_found_keys, ws.h_staged, ws.h_row_of, &nf,
                    ws.h_missing, &nm, counters);
  *n_found = nf;
  return nm;
}

void LookupEngine::lookup(const uint64_t* keys, size_t n, float* out, size_t out_len,
                          uint8_t* flags, LookupOutcome* outcome, int mem, cudaStream_t user) {
  LookupCall call = begin(keys, n, out, out_len, flags, mem, user);
  finish(call, outcome);
}

void LookupEngine::lookup_multi(LookupEngine* const* engines, size_t count,
                                const uint64_t* const* keys, const size_t* n, float* const* out,
                                uint8_t* const* flags, LookupOutcome* outcomes, int mem) {
  // every table's keys, kernel and first copies are in flight before any
  // host waits: the tables' lookups overlap on the device
  std::vector<LookupCall> calls;
  calls.reserve(count);
  try {
    for (size_t t = 0; t < count; ++t)
      // device mode orders against the legacy default stream, exactly as
      // hps_engine_lookup with a NULL stream (join_from / join_to skip a
      // null stream, which would leave the caller's keys and later reads
      // unordered against the cache stream)
      calls.push_back(engines[t]->begin(keys[t], n[t], out[t], n[t] * engines[t]->dim_, flags[t],
                                        mem, cudaStreamLegacy));
  } catch (...) {
    for (auto& c : calls) c.engine->abandon(c);
    throw;
  }
  std::exception_ptr first_error;
  for (size_t t = 0; t < count; ++t) {
    try {
      calls[t].engine->finish(calls[t], outcomes ? outcomes + t : nullptr);
    } catch (...) {
      if (!first_error) first_error = std::current_exception();
    }
  }
  if (first_error) std::rethrow_exception(first_error);
}

void LookupEngine::abandon(LookupCall& c) {
  if (c.ws == nullptr) return;
  if (c.n > 0) cudaEventSynchronize(c.ws->done);
  pool_.release(c.ws);
  c.ws = nullptr;
}

LookupEngine::LookupCall LookupEngine::begin(const uint64_t* keys, size_t n, float* out,
                                             size_t out_len, uint8_t* flags, int mem,
                                             cudaStream_t user) {
  if (out_len != n * uint64_t(dim_)) throw invalid_argument("lookup output buffer has wrong size");
  // positions and first occurrences are u32 on the device
  if (n >= 0xFFFFFFFFull) throw invalid_argument("lookup batch too large");
  if (cfg_.max_batch != 0 && n > cfg_.max_batch)
    throw invalid_argument("lookup batch exceeds the engine's max_batch");
  LookupCall c;
  c.t0 = std::chrono::steady_clock::now();
  c.engine = this;
  c.n = n;
  c.out = out;
  c.flags = flags;
  c.mem = mem;
  c.user = user;
  c.host = mem == kHostMem;
  const bool host = c.host;
  const uint32_t d = dim_;
  Workspace* ws = pool_.acquire();
  c.ws = ws;
  try {
    ws->wait_idle();
    DeviceGuard g(cache_->device());
    cudaStream_t st = cache_->stream();
    ws->ensure(std::max<size_t>(n, 1), d, st);
    // host mode: rows and flags always come back with the counts -- an
    // async call's rows are final as the kernel leaves them, and a sync
    // call's fetched rows are scattered into the host output on the host
    // (host_scatter) while the cache fill runs on
    c.spec_rows = host;
    c.h_keys = host ? keys : nullptr;
    c.out_pinned = host && n > 0 && is_pinned(out);
    c.flags_pinned = host && n > 0 && is_pinned(flags);
    c.d_keys = keys;
    c.d_out = out;
    c.d_flags = flags;
    std::lock_guard<std::mutex> lk(cache_->mutex());
    const uint64_t stamp = cache_->bump_clock();  // query ticks even when empty
    if (n > 0) {
      // small host-mode call (packed): zero-copy -- the kernel reads the keys
      // from pinned host memory and writes rows, flags, counts and every
      // claim straight into pinned host memory ([counts | first positions |
      // keys | flags] in h_hdr); no copies, one host wait on the kernel
      static const uint64_t zero_copy_max = [] {
        const char* e = std::getenv("HPSB_ZERO_COPY_MAX");  // A/B knob
        return e ? uint64_t(std::strtoull(e, nullptr, 10)) : kPackedMax;
      }();
      c.packed = host && n <= zero_copy_max;
      if (c.packed) {
        const void* mk = mapped(keys);
        if (mk == nullptr) {
          std::memcpy(ws->h_keys, keys, n * 8);
          mk = ws->h_keys;
        }
        c.d_keys = static_cast<const uint64_t*>(mk);
        float* mo = c.out_pinned ? static_cast<float*>(const_cast<void*>(mapped(out))) : nullptr;
        c.out_direct = mo != nullptr;
        c.d_out = c.out_direct ? mo : ws->h_out;
      } else if (host) {
        if (is_pinned(keys)) {
          HPSB_CUDA(cudaMemcpyAsync(ws->d_keys, keys, n * 8, cudaMemcpyHostToDevice, st));
        } else {
          // pageable keys: staged by the copy threads (a 0.5 MB single-thread
          // memcpy was most of this call's 0.1 ms before the upload)
          const size_t bytes = n * 8;
          const size_t chunks = bytes >= (size_t(256) << 10) ? copy_threads_.size() : 1;
          const size_t per = (n + chunks - 1) / chunks;
          copy_threads_.parallel_for(chunks, 1, [&](size_t cb, size_t ce) {
            for (size_t ch = cb; ch < ce; ++ch) {
              const size_t b = ch * per, e = std::min(n, b + per);
              if (b < e) std::memcpy(ws->h_keys + b, keys + b, (e - b) * 8);
            }
          });
          HPSB_CUDA(cudaMemcpyAsync(ws->d_keys, ws->h_keys, n * 8, cudaMemcpyHostToDevice, st));
        }
        c.d_keys = ws->d_keys;
        c.d_out = ws->d_out;
        c.d_flags = ws->d_flags;
      } else {
        cache_->join_from(user);
      }
      cache_->prepare_hits(ws->ls, stamp);
      ws->lv = lookup_next_view(ws->ls, /*chain=*/false);
      if (c.packed) {
        const uint64_t fo = 16, ko = 16 + (n * 4 + 7) / 8 * 8, flo = ko + n * 8;
        ws->lv.counts_out = reinterpret_cast<unsigned long long*>(ws->h_hdr);
        ws->lv.list_firsts = reinterpret_cast<uint32_t*>(ws->h_hdr + fo);
        ws->lv.list_keys = reinterpret_cast<uint64_t*>(ws->h_hdr + ko);
        c.d_flags = reinterpret_cast<uint8_t*>(ws->h_hdr + flo);
        c.hc = reinterpret_cast<const unsigned long long*>(ws->h_hdr);
        c.hcf = reinterpret_cast<const uint32_t*>(ws->h_hdr + fo);
        c.hck = reinterpret_cast<const uint64_t*>(ws->h_hdr + ko);
        c.hfl = reinterpret_cast<const uint8_t*>(ws->h_hdr + flo);
        ws->lv.flags_dev = ws->d_flags;
        c.spec_claims = n;
      }
      cache_->note_stream_op();  // the engine's own copies follow on the stream
      launch_lookup_probe(cache_->dev(), c.d_keys, n, c.d_out, c.d_flags, d_default_, stamp,
                          ws->lv, /*after_lookup=*/false, st);
      if (!c.packed) {
        HPSB_CUDA(cudaMemcpyAsync(ws->h_counts, ws->lv.counts_out, 16, cudaMemcpyDeviceToHost, st));
        // One host round trip on the common path: the first claims and -- when
        // the previous call took the async branch, whose rows are final as the
        // kernel leaves them -- the rows and flags come back with the counts.
        c.spec_claims = std::min<uint64_t>(n, kSpeculativeClaims);
        c.hc = ws->h_counts;
        c.hcf = ws->h_claim_firsts;
        c.hck = ws->h_claim_keys;
        HPSB_CUDA(cudaMemcpyAsync(ws->h_claim_keys, ws->lv.list_keys, c.spec_claims * 8,
                                  cudaMemcpyDeviceToHost, st));
        HPSB_CUDA(cudaMemcpyAsync(ws->h_claim_firsts, ws->lv.list_firsts, c.spec_claims * 4,
                                  cudaMemcpyDeviceToHost, st));
        // the host decides the branch as soon as the counts land; the rows
        // copy on behind them
        HPSB_CUDA(cudaEventRecord(ws->counts_ready, st));
        if (host && c.spec_rows) {
          HPSB_CUDA(cudaMemcpyAsync(c.flags_pinned ? flags : ws->h_flags, c.d_flags, n,
                                    cudaMemcpyDeviceToHost, st));
          rows_d2h(*ws, c, st);
          HPSB_CUDA(cudaEventRecord(ws->rows_ready, st));
        }
      } else {
        HPSB_CUDA(cudaEventRecord(ws->counts_ready, st));
      }
      HPSB_CUDA(cudaEventRecord(ws->done, st));
      ws->pending = true;  // rows may still be crossing after the counts land
    }
  } catch (...) {
    pool_.release(ws);
    throw;
  }
  return c;
}

void LookupEngine::finish(LookupCall& c, LookupOutcome* outcome) {
  PhaseTrace tr;
  tr.t0 = c.t0;
  tr.mark("finish");
  Workspace* ws = c.ws;
  bool handed_off = false;
  struct LeaseGuard {
    WorkspacePool& pool;
    LookupCall& c;
    bool* handed;
    ~LeaseGuard() {
      if (!*handed && c.ws) pool.release(c.ws);
      c.ws = nullptr;
    }
  } guard{pool_, c, &handed_off};
  const size_t n = c.n;
  const bool host = c.host;
  const uint32_t d = dim_;
  float* out = c.out;
  uint8_t* flags = c.flags;
  float* d_out = c.d_out;
  uint8_t* d_flags = c.d_flags;
  DeviceGuard g(cache_->device());
  cudaStream_t st = cache_->stream();
  uint64_t uh = 0, um = 0;
  if (n > 0) {
    HPSB_CUDA(cudaEventSynchronize(ws->counts_ready));
    tr.mark("counts");
    uh = c.hc[0];
    um = c.hc[1];
    if (um > c.spec_claims) {
      // the rest of the claims, on the side stream (the kernel is done: the
      // copy need not queue behind the speculative rows on the cache stream)
      HPSB_CUDA(cudaMemcpyAsync(ws->h_claim_keys + c.spec_claims,
                                ws->lv.list_keys + c.spec_claims, (um - c.spec_claims) * 8,
                                cudaMemcpyDeviceToHost, copy_stream_));
      HPSB_CUDA(cudaMemcpyAsync(ws->h_claim_firsts + c.spec_claims,
                                ws->lv.list_firsts + c.spec_claims, (um - c.spec_claims) * 4,
                                cudaMemcpyDeviceToHost, copy_stream_));
      HPSB_CUDA(cudaEventRecord(ws->uploaded, copy_stream_));
      HPSB_CUDA(cudaEventSynchronize(ws->uploaded));
    }
    if (um > 0) {
      // the reference's miss order: unique misses by first occurrence
      // (types.cpp:20-34 + slab_cache.cpp:84-89)
      ws->order.resize(um);
      for (uint32_t e = 0; e < um; ++e) ws->order[e] = e;
      const uint32_t* fp = c.hcf;
      std::sort(ws->order.begin(), ws->order.end(),
                [fp](uint32_t a, uint32_t b) { return fp[a] < fp[b]; });
      for (uint64_t k = 0; k < um; ++k) ws->h_miss_keys[k] = c.hck[ws->order[k]];
    }
  }
  const uint64_t n_unique = uh + um;
  // lookup_engine.cpp:148-153
  const double h = n_unique == 0 ? 1.0 : 1.0 - double(um) / double(n_unique);
  const bool sync_branch = h < cfg_.hit_rate_threshold;
  TierCounters counters;
  uint64_t defaults = 0;
  if (sync_branch) {
    size_t nf = 0;
    const size_t absent = fetch_and_upload(*ws, ws->h_miss_keys, um, &counters, &nf);
    tr.mark("fetch");
    defaults = absent;
    std::lock_guard<std::mutex> lk(cache_->mutex());
    tr.mark("lock");
    if (host && c.packed) {
      // zero-copy call: the kernel has written rows and flags to host memory
      // already; the fetched rows go into the caller's output on the host
      // (below) and the fill's replace reads its keys and rows straight from
      // the pinned staging (small fills) or after an upload
      if (nf > 0) {
        if (nf <= kZeroCopyReplaceMax) {
          cache_->replace_device_locked(ws->h_found_keys, nf, ws->h_staged);
        } else {
          HPSB_CUDA(cudaMemcpyAsync(ws->d_staged, ws->h_staged, nf * uint64_t(d) * 4,
                                    cudaMemcpyHostToDevice, st));
          HPSB_CUDA(cudaMemcpyAsync(ws->d_found_keys, ws->h_found_keys, nf * 8,
                                    cudaMemcpyHostToDevice, st));
          cache_->replace_device_locked(ws->d_found_keys, nf, ws->d_staged);
        }
      }
    } else if (host && c.spec_rows) {
      // rows and flags are already crossing to the host: the fetched rows go
      // into the host output there (below); on the device only the fill
      if (nf > 0) {
        HPSB_CUDA(cudaMemcpyAsync(ws->d_staged, ws->h_staged, nf * uint64_t(d) * 4,
                                  cudaMemcpyHostToDevice, st));
        HPSB_CUDA(cudaMemcpyAsync(ws->d_found_keys, ws->h_found_keys, nf * 8,
                                  cudaMemcpyHostToDevice, st));
        cache_->replace_device_locked(ws->d_found_keys, nf, ws->d_staged);
      }
    } else if (nf > 0) {
      // device mode: the scatter kernel (row_of is in miss order; the kernel
      // indexes by claim) writes the caller's device rows / flags
      for (uint64_t k = 0; k < um; ++k) ws->h_row_of_claim[ws->order[k]] = ws->h_row_of[k];
      HPSB_CUDA(cudaMemcpyAsync(ws->d_row_of, ws->h_row_of_claim, um * 4,
                                cudaMemcpyHostToDevice, st));
      HPSB_CUDA(cudaMemcpyAsync(ws->d_staged, ws->h_staged, nf * uint64_t(d) * 4,
                                cudaMemcpyHostToDevice, st));
      HPSB_CUDA(cudaMemcpyAsync(ws->d_found_keys, ws->h_found_keys, nf * 8,
                                cudaMemcpyHostToDevice, st));
      cache_->note_stream_op();
      launch_lookup_scatter(n, d, d_flags, ws->lv, ws->d_row_of, ws->d_staged, d_out, st);
      cache_->replace_device_locked(ws->d_found_keys, nf, ws->d_staged);
    }
    HPSB_CUDA(cudaEventRecord(ws->done, st));
    ws->pending = true;
    tr.mark("enqueued");
  } else {
    defaults = um;
  }

  last_async_.store(!sync_branch, std::memory_order_relaxed);
  if (n > 0) {
    if (host && c.packed) {
      // zero-copy call: rows and flags are in host memory since the kernel
      // completed (counts_ready); a sync branch's fetched rows are written
      // into the caller's output here while its fill runs on
      if (!sync_branch) ws->pending = false;
      if (!c.out_direct) std::memcpy(out, ws->h_out, n * uint64_t(d) * 4);
      std::memcpy(flags, c.hfl, n);
      if (sync_branch && um > 0) {
        ws->scatter_keys = ws->h_miss_keys;
        host_scatter(*ws, n, c.h_keys, out, um, flags);
        tr.mark("scatter");
      }
    } else if (host) {
      if (!c.spec_rows) {
        HPSB_CUDA(cudaMemcpyAsync(c.flags_pinned ? flags : ws->h_flags, d_flags, n,
                                  cudaMemcpyDeviceToHost, st));
        rows_d2h(*ws, c, st);
        HPSB_CUDA(cudaEventRecord(ws->rows_ready, st));
        HPSB_CUDA(cudaEventRecord(ws->done, st));
      }
      // pageable rows: copied on chunk by chunk as they land
      if (!c.out_pinned) rows_to_pageable(*ws, c);
      HPSB_CUDA(cudaEventSynchronize(ws->rows_ready));
      tr.mark("rows");
      uint8_t* hf = c.flags_pinned ? flags : ws->h_flags;
      if (sync_branch && um > 0) {
        ws->scatter_keys = ws->h_miss_keys;
        host_scatter(*ws, n, c.h_keys, c.out, um, hf);
        tr.mark("scatter");
      }
      if (!sync_branch) {
        HPSB_CUDA(cudaEventSynchronize(ws->done));
        ws->pending = false;
      }  // sync: the fill runs on behind the return (ws->done, wait_idle)
      if (!c.flags_pinned) std::memcpy(flags, ws->h_flags, n);
    } else {
      cache_->join_to(c.user);
    }
  }

  tr.mark("done");
  tr.report(n, um, sync_branch);
  if (outcome) {
    outcome->sync_branch = sync_branch;
    outcome->unique_hit_rate = h;
    outcome->unique_count = n_unique;
    outcome->defaults_returned = defaults;
  }
  {
    std::lock_guard<std::mutex> lk(stats_mu_);
    stats_.queries += 1;
    stats_.queried_keys += n;
    stats_.unique_keys += n_unique;
    stats_.cache_hits += uh;
    stats_.cache_misses += um;
    stats_.defaults_returned += defaults;
    if (sync_branch) {
      stats_.sync_batches += 1;
      stats_.vdb_hits += counters.vdb_hits;
      stats_.pdb_hits += counters.cold_hits;
      stats_.tier_missing += counters.missing;
    } else {
      stats_.async_batches += 1;
    }
  }
  if (!sync_branch && um > 0) {
    // the workspace (and its miss list) rides along with the background fill
    ws->missing_keys.assign(ws->h_miss_keys, ws->h_miss_keys + um);
    {
      std::lock_guard<std::mutex> lk(q_mu_);
      queue_.push_back(AsyncTask{ws});
      handed_off = true;
    }
    q_cv_.notify_one();
  }
}

void LookupEngine::finish_group(const GroupResult& r, LookupOutcome* outcome) {
  const uint32_t d = dim_;
  const uint64_t n_unique = r.uh + r.um;
  // lookup_engine.cpp:148-153
  const double h = n_unique == 0 ? 1.0 : 1.0 - double(r.um) / double(n_unique);
  const bool sync_branch = h < cfg_.hit_rate_threshold;
  TierCounters counters;
  uint64_t defaults = 0;
  DeviceGuard g(cache_->device());
  cudaStream_t st = cache_->stream();
  if (sync_branch) {
    Workspace* ws = pool_.acquire();
    struct Release {
      WorkspacePool& p;
      Workspace* w;
      ~Release() { p.release(w); }
    } rel{pool_, ws};
    ws->wait_idle();
    ws->ensure(std::max<uint64_t>(r.um, 1), d, st);
    size_t nf = 0;
    defaults = fetch_and_upload(*ws, r.miss_keys, r.um, &counters, &nf);
    if (nf > 0) {
      // the table's rows and flags are in the caller's host buffers already:
      // the fetched rows are written there by the host, and the fill's
      // replace runs on behind the return (the workspace is reused only
      // after it, ws->done)
      {
        std::lock_guard<std::mutex> lk(cache_->mutex());
        if (nf <= kZeroCopyReplaceMax) {
          cache_->replace_device_locked(ws->h_found_keys, nf, ws->h_staged);
        } else {
          HPSB_CUDA(cudaMemcpyAsync(ws->d_staged, ws->h_staged, nf * uint64_t(d) * 4,
                                    cudaMemcpyHostToDevice, st));
          HPSB_CUDA(cudaMemcpyAsync(ws->d_found_keys, ws->h_found_keys, nf * 8,
                                    cudaMemcpyHostToDevice, st));
          cache_->replace_device_locked(ws->d_found_keys, nf, ws->d_staged);
        }
        HPSB_CUDA(cudaEventRecord(ws->done, st));
        ws->pending = true;
      }
      ws->scatter_keys = r.miss_keys;
      host_scatter(*ws, r.n, r.h_keys, r.out, r.um, r.flags);
    }
  } else {
    defaults = r.um;
  }
  last_async_.store(!sync_branch, std::memory_order_relaxed);
  if (outcome) {
    outcome->sync_branch = sync_branch;
    outcome->unique_hit_rate = h;
    outcome->unique_count = n_unique;
    outcome->defaults_returned = defaults;
  }
  {
    std::lock_guard<std::mutex> lk(stats_mu_);
    stats_.queries += 1;
    stats_.queried_keys += r.n;
    stats_.unique_keys += n_unique;
    stats_.cache_hits += r.uh;
    stats_.cache_misses += r.um;
    stats_.defaults_returned += defaults;
    if (sync_branch) {
      stats_.sync_batches += 1;
      stats_.vdb_hits += counters.vdb_hits;
      stats_.pdb_hits += counters.cold_hits;
      stats_.tier_missing += counters.missing;
    } else {
      stats_.async_batches += 1;
    }
  }
  if (!sync_branch && r.um > 0) {
    Workspace* ws = pool_.acquire();
    try {
      ws->wait_idle();
      ws->ensure(r.um, d, st);
      ws->missing_keys.assign(r.miss_keys, r.miss_keys + r.um);
    } catch (...) {
      pool_.release(ws);
      throw;
    }
    {
      std::lock_guard<std::mutex> lk(q_mu_);
      queue_.push_back(AsyncTask{ws});
    }
    q_cv_.notify_one();
  }
}

// ------------------------------------------------------------ multi-table --
namespace {
inline uint64_t a256m(uint64_t v) { return (v + 255) / 256 * 256; }
}  // namespace

MultiLookup::MultiLookup(std::vector<LookupEngine*> engines, uint64_t max_batch)
    : eng_(std::move(engines)), maxb_(std::max<uint64_t>(max_batch, 1)) {
  if (eng_.empty()) throw invalid_argument("multi-table lookup needs at least one engine");
  const DeviceCache* c0 = eng_[0]->cache();
  bool all8 = true, all4 = true;
  for (auto* e : eng_) {
    if (e == nullptr) throw invalid_argument("null engine");
    if (e->cache()->stream() != c0->stream() || e->cache()->device() != c0->device())
      throw invalid_argument("multi-table lookup needs the tables' caches in one cache group");
    all8 &= e->dim() % 8 == 0;
    all4 &= e->dim() % 4 == 0;
  }
  for (size_t i = 0; i < eng_.size(); ++i)
    for (size_t j = i + 1; j < eng_.size(); ++j)
      if (eng_[i]->cache() == eng_[j]->cache())
        throw invalid_argument("multi-table lookup needs one cache per table");
  ch_ = all8 ? 8 : (all4 ? 4 : 1);
  const uint64_t T = eng_.size();
  DeviceGuard g(c0->device());
  cudaStream_t st = c0->stream();
  uint64_t rows = 0;
  for (auto* e : eng_) rows += maxb_ * e->dim();
  // device: [desc][keys][counts][flags][claim keys][claim firsts][rows]
  uint64_t o = 0;
  d_desc_ = o;
  o += a256m(T * sizeof(TableLookup));
  d_keys_ = o;
  o += a256m(T * maxb_ * 8);
  d_counts_ = o;
  o += a256m(T * 16);
  d_flags_ = o;
  o += a256m(T * maxb_ + 32 * T);
  d_ckeys_ = o;
  o += a256m(T * maxb_ * 8);
  d_cfirsts_ = o;
  o += a256m(T * maxb_ * 4);
  d_rows_ = o;
  o += a256m(rows * 4 + 32 * T);
  dev_.ensure(o, st);
  host_.ensure(o);
  h_rows_ = d_rows_;
  // one view per table: every group call completes before the next starts
  const uint64_t sbytes = lookup_scratch_bytes(maxb_, 1);
  char* sp = static_cast<char*>(scratch_dev_.ensure(a256m(sbytes) * T, st));
  HPSB_CUDA(cudaMemsetAsync(sp, 0, a256m(sbytes) * T, st));
  for (uint64_t t = 0; t < T; ++t)
    ls_.push_back(lookup_scratch_carve(sp + t * a256m(sbytes), maxb_, 1));
  HPSB_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
  HPSB_CUDA(cudaStreamSynchronize(st));
}

MultiLookup::~MultiLookup() {
  if (done_) {
    cudaEventSynchronize(done_);
    cudaEventDestroy(done_);
  }
}

void MultiLookup::lookup(const uint64_t* const* keys, const size_t* n, float* const* out,
                         uint8_t* const* flags, LookupOutcome* outcomes) {
  std::lock_guard<std::mutex> lk(mu_);
  const uint64_t T = eng_.size();
  for (uint64_t t = 0; t < T; ++t)
    if (n[t] > maxb_) throw invalid_argument("multi-table batch exceeds the group's max batch");
  DeviceCache* c0 = eng_[0]->cache();
  DeviceGuard g(c0->device());
  cudaStream_t st = c0->stream();
  char* hb = static_cast<char*>(host_.get());
  char* db = static_cast<char*>(dev_.get());
  auto* desc = reinterpret_cast<TableLookup*>(hb + d_desc_);
  auto* hkeys = reinterpret_cast<uint64_t*>(hb + d_keys_);
  // packed per-call offsets: keys / flags / claims by position, rows by float
  std::vector<uint64_t> koff(T + 1, 0), roff(T + 1, 0);
  for (uint64_t t = 0; t < T; ++t) {
    koff[t + 1] = koff[t] + n[t];
    roff[t + 1] = roff[t] + n[t] * eng_[t]->dim() + 7;  // keep 32 B alignment
    roff[t + 1] &= ~7ull;
  }
  // small calls: zero-copy outputs -- the kernel writes counts, flags,
  // claims and rows straight into the pinned mirror (same offsets), no
  // device-to-host copies
  const bool packed_rows = roff[T] * 4 <= kPackedRowBytes;
  // pinned caller outputs (any size up to kDirectRowBytes): the kernel writes
  // each table's rows straight into the caller's buffer -- no row copies at
  // all (one D2H per table before); counts, flags and claims as above
  std::vector<float*> direct_out(T, nullptr);
  bool direct = roff[T] * 4 <= kDirectRowBytes;
  const uintptr_t align = ch_ == 8 ? 32 : (ch_ == 4 ? 16 : 4);
  for (uint64_t t = 0; t < T && direct; ++t) {
    if (n[t] == 0) continue;
    direct_out[t] = static_cast<float*>(host_mapped(out[t]));
    direct = direct_out[t] != nullptr && reinterpret_cast<uintptr_t>(direct_out[t]) % align == 0;
  }
  const bool zero_copy = packed_rows || direct;
  char* ob = zero_copy ? hb : db;
  uint32_t blocks = 0;
  std::vector<LookupView> views(T);
  for (uint64_t t = 0; t < T; ++t) {
    DeviceCache* c = eng_[t]->cache();
    std::memcpy(hkeys + koff[t], keys[t], n[t] * 8);
    std::lock_guard<std::mutex> clk(c->mutex());
    const uint64_t stamp = c->bump_clock();  // query ticks even when empty
    c->note_stream_op();
    TableLookup& tl = desc[t];
    if (n[t] == 0) {
      // no blocks run for an empty table: it takes no view (a view handed
      // out here would never be released, and its next use would wait
      // forever on the device)
      std::memset(static_cast<void*>(&tl), 0, sizeof(tl));
      tl.block_begin = blocks;
      continue;
    }
    c->prepare_hits(ls_[t], stamp);
    LookupView v = lookup_next_view(ls_[t], false);
    v.list_keys = reinterpret_cast<uint64_t*>(ob + d_ckeys_) + koff[t];
    v.list_firsts = reinterpret_cast<uint32_t*>(ob + d_cfirsts_) + koff[t];
    v.counts_out = reinterpret_cast<unsigned long long*>(ob + d_counts_) + 2 * t;
    views[t] = v;
    tl.c = c->dev();
    tl.keys = reinterpret_cast<const uint64_t*>(db + d_keys_) + koff[t];
    tl.n = n[t];
    tl.out = direct ? direct_out[t] : reinterpret_cast<float*>(ob + d_rows_) + roff[t];
    tl.flags = reinterpret_cast<uint8_t*>(ob + d_flags_) + koff[t];
    tl.default_row = eng_[t]->default_row();
    tl.stamp = stamp;
    tl.v = v;
    tl.block_begin = blocks;
    tl.nblocks = uint32_t((n[t] + kMultiBlockPositions - 1) / kMultiBlockPositions);
    blocks += tl.nblocks;
  }
  // one H2D (descriptors + packed keys), one launch
  HPSB_CUDA(cudaMemcpyAsync(db + d_desc_, hb + d_desc_, (d_keys_ - d_desc_) + koff[T] * 8,
                            cudaMemcpyHostToDevice, st));
  launch_lookup_multi(reinterpret_cast<const TableLookup*>(db + d_desc_), uint32_t(T), blocks,
                      ch_, st);
  // one D2H each: counts, flags, claims (whole packed regions), rows
  auto d2h = [&](uint64_t off, uint64_t bytes) {
    if (bytes) HPSB_CUDA(cudaMemcpyAsync(hb + off, db + off, bytes, cudaMemcpyDeviceToHost, st));
  };
  // large calls: one D2H each for counts, flags, claims (whole packed
  // regions), and the rows straight into each table's output (no extra host
  // copy of big rows)
  if (!zero_copy) {
    d2h(d_counts_, T * 16);
    d2h(d_flags_, koff[T]);
    d2h(d_ckeys_, koff[T] * 8);
    d2h(d_cfirsts_, koff[T] * 4);
    for (uint64_t t = 0; t < T; ++t)
      if (n[t])
        HPSB_CUDA(cudaMemcpyAsync(out[t], db + d_rows_ + roff[t] * 4,
                                  n[t] * uint64_t(eng_[t]->dim()) * 4, cudaMemcpyDeviceToHost, st));
  }
  HPSB_CUDA(cudaEventRecord(done_, st));
  HPSB_CUDA(cudaEventSynchronize(done_));
  const auto* hcounts = reinterpret_cast<const unsigned long long*>(hb + d_counts_);
  const auto* hflags = reinterpret_cast<const uint8_t*>(hb + d_flags_);
  const auto* hck = reinterpret_cast<const uint64_t*>(hb + d_ckeys_);
  const auto* hcf = reinterpret_cast<const uint32_t*>(hb + d_cfirsts_);
  const auto* hrows = reinterpret_cast<const float*>(hb + d_rows_);
  std::exception_ptr first_error;
  for (uint64_t t = 0; t < T; ++t) {
    try {
      const uint32_t d = eng_[t]->dim();
      if (zero_copy && !direct) std::memcpy(out[t], hrows + roff[t], n[t] * uint64_t(d) * 4);
      std::memcpy(flags[t], hflags + koff[t], n[t]);
      LookupEngine::GroupResult r;
      r.n = n[t];
      r.uh = n[t] ? hcounts[2 * t] : 0;
      r.um = n[t] ? hcounts[2 * t + 1] : 0;
      order_.resize(r.um);
      miss_.resize(r.um);
      for (uint32_t e = 0; e < r.um; ++e) order_[e] = e;
      const uint32_t* fp = hcf + koff[t];
      std::sort(order_.begin(), order_.end(), [fp](uint32_t a, uint32_t b) { return fp[a] < fp[b]; });
      for (uint64_t k = 0; k < r.um; ++k) miss_[k] = hck[koff[t] + order_[k]];
      r.miss_keys = miss_.data();
      r.out = out[t];
      r.flags = flags[t];
      r.h_keys = keys[t];
      eng_[t]->finish_group(r, outcomes ? outcomes + t : nullptr);
    } catch (...) {
      if (!first_error) first_error = std::current_exception();
    }
  }
  if (first_error) std::rethrow_exception(first_error);
}

void LookupEngine::async_loop() {
  for (;;) {
    AsyncTask task;
    {
      std::unique_lock<std::mutex> lk(q_mu_);
      q_cv_.wait(lk, [&] { return stopping_ || !queue_.empty(); });
      if (queue_.empty()) return;
      task = queue_.front();
      queue_.pop_front();
      ++active_;
    }
    Workspace& ws = *task.ws;
    TierCounters counters;
    try {
      DeviceGuard g(cache_->device());
      cudaStream_t st = cache_->stream();
      ws.wait_idle();
      size_t nf = 0;
      fetch_and_upload(ws, ws.missing_keys.data(), ws.missing_keys.size(), &counters, &nf);
      if (nf > kZeroCopyReplaceMax) {
        // the upload runs on the side stream and is waited for HERE, before
        // the replace is enqueued: lookups queued on the cache stream in the
        // meantime never wait behind the copy
        HPSB_CUDA(cudaMemcpyAsync(ws.d_staged, ws.h_staged, nf * uint64_t(dim_) * 4,
                                  cudaMemcpyHostToDevice, copy_stream_));
        HPSB_CUDA(cudaMemcpyAsync(ws.d_found_keys, ws.h_found_keys, nf * 8,
                                  cudaMemcpyHostToDevice, copy_stream_));
        HPSB_CUDA(cudaEventRecord(ws.uploaded, copy_stream_));
        HPSB_CUDA(cudaEventSynchronize(ws.uploaded));
      }
      if (nf > 0) {
        std::lock_guard<std::mutex> lk(cache_->mutex());
        if (nf <= kZeroCopyReplaceMax) {
          // small fill: the replace reads keys and rows from pinned host
          // memory (no copies queued ahead of the next lookup on the stream)
          cache_->replace_device_locked(ws.h_found_keys, nf, ws.h_staged);
        } else {
          cache_->replace_device_locked(ws.d_found_keys, nf, ws.d_staged);
        }
        HPSB_CUDA(cudaEventRecord(ws.done, st));
        ws.pending = true;
      }
      ws.wait_idle();
      std::lock_guard<std::mutex> lk(stats_mu_);
      stats_.vdb_hits += counters.vdb_hits;
      stats_.pdb_hits += counters.cold_hits;
      stats_.tier_missing += counters.missing;
    } catch (...) {
      // the caller already got default rows; a failed fill only costs hit rate
      std::lock_guard<std::mutex> lk(stats_mu_);
      stats_.async_faults += 1;
    }
    pool_.release(task.ws);
    {
      std::lock_guard<std::mutex> lk(q_mu_);
      --active_;
      if (queue_.empty() && active_ == 0) idle_cv_.notify_all();
    }
  }
}

void LookupEngine::reserve(uint64_t n) {
  if (n == 0) return;
  if (n >= 0xFFFFFFFFull) throw invalid_argument("lookup batch too large");
  DeviceGuard g(cache_->device());
  cudaStream_t st = cache_->stream();
  pool_.for_each([&](Workspace& ws) {
    ws.wait_idle();
    ws.ensure(n, dim_, st);
  });
  cache_->reserve_replace(n);
}

void LookupEngine::drain_async() {
  std::unique_lock<std::mutex> lk(q_mu_);
  idle_cv_.wait(lk, [&] { return queue_.empty() && active_ == 0; });
}

EngineStats LookupEngine::stats() const {
  std::lock_guard<std::mutex> lk(stats_mu_);
  return stats_;
}

// ------------------------------------------------------------ replicas --
ReplicaGroup::ReplicaGroup(std::vector<LookupEngine*> engines) : eng_(std::move(engines)) {
  if (eng_.empty()) throw invalid_argument("a replica group needs at least one engine");
  for (auto* e : eng_)
    if (e == nullptr) throw invalid_argument("null engine in replica group");
  jobs_.resize(eng_.size());
  errs_.resize(eng_.size());
  for (size_t r = 0; r < eng_.size(); ++r) threads_.emplace_back([this, r] { worker(r); });
}

ReplicaGroup::~ReplicaGroup() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : threads_) t.join();
}

void ReplicaGroup::worker(size_t r) {
  uint64_t seen = 0;
  for (;;) {
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
    }
    const Job& j = jobs_[r];
    try {
      eng_[r]->lookup(j.keys, j.n, j.out, j.n * uint64_t(eng_[r]->dimension()), j.flags, j.outcome,
                      j.mem, cudaStreamLegacy);
    } catch (...) {
      errs_[r] = std::current_exception();
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
}

void ReplicaGroup::lookup(const uint64_t* const* keys, const size_t* n, float* const* out,
                          uint8_t* const* flags, LookupOutcome* outcomes, int mem) {
  std::lock_guard<std::mutex> call(call_mu_);
  for (size_t r = 0; r < eng_.size(); ++r) {
    jobs_[r] = Job{keys[r], n[r], out[r], flags[r], outcomes ? outcomes + r : nullptr, mem};
    errs_[r] = nullptr;
  }
  {
    std::lock_guard<std::mutex> lk(mu_);
    pending_ = eng_.size();
    ++gen_;
  }
  cv_.notify_all();
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return pending_ == 0; });
  for (auto& e : errs_)
    if (e) std::rethrow_exception(e);
}

}  // namespace hpsb
