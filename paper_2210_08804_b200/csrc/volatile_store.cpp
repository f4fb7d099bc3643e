// volatile_store.cpp -- see volatile_store.hpp. Reference behaviour
// (volatile_store.cpp of /root/reference/proj):
//   partition_of            :10-13
//   register_table          :25-51 (same validation and messages)
//   lookup                  :82-112 (clock once per call, input order)
//   insert / insert_rows    :113-152 (clock once per call, upsert, prune)
//   prune_partition         :154-173 (smallest (last_access, key) first)
//   background refresh      :226-239 (max, never backwards)
#include "volatile_store.hpp"

#include <algorithm>
#include <cstring>
#include <atomic>
#include <cmath>

#include "common.cuh"

namespace hpsb {

uint32_t partition_of(uint64_t key, uint32_t partition_count) {
  return uint32_t(xxh64_key(key, kPartitionSeed) % partition_count);
}

namespace {
inline uint64_t idx_hash(uint64_t key) { return fmix64(key ^ 0xA5A5A5A5DEADBEEFull); }

void require_finite(const float* v, size_t n, const char* ctx) {
  for (size_t i = 0; i < n; ++i) {
    if (!std::isfinite(v[i]))
      throw invalid_argument(std::string(ctx) + ": embedding values must be finite");
  }
}

inline void atomic_max(uint64_t& slot, uint64_t v) {
  std::atomic_ref<uint64_t> a(slot);
  uint64_t cur = a.load(std::memory_order_relaxed);
  while (cur < v && !a.compare_exchange_weak(cur, v, std::memory_order_relaxed)) {
  }
}
}  // namespace

int64_t VolatileStore::Partition::find(uint64_t key) const {
  if (index.empty()) return -1;
  const uint64_t mask = index.size() - 1;
  uint64_t h = idx_hash(key) & mask;
  while (true) {
    const uint32_t e = index[h];
    if (e == 0) return -1;
    if (keys[e - 1] == key) return int64_t(e - 1);
    h = (h + 1) & mask;
  }
}

VolatileStore::VolatileStore(unsigned lookup_threads)
    : pool_(lookup_threads ? lookup_threads : std::max(1u, std::thread::hardware_concurrency())),
      worker_([this] { background_loop(); }) {}

VolatileStore::~VolatileStore() {
  {
    std::lock_guard<std::mutex> lk(q_mu_);
    stopping_ = true;
  }
  q_cv_.notify_all();
  worker_.join();
}

void VolatileStore::register_table(const std::string& name, uint32_t dim,
                                   uint32_t partition_count, uint64_t overflow_margin) {
  // validate_table_id (types.cpp:3-12) + register_table checks
  if (name.empty()) throw invalid_argument("table name must not be empty");
  if (name.size() > 255) throw invalid_argument("table name exceeds 255 bytes: " + name);
  if (dim == 0) throw invalid_argument("table dimension must be positive: " + name);
  if (partition_count == 0) throw invalid_argument("partition_count must be positive");
  if (overflow_margin == 0) throw invalid_argument("overflow_margin must be positive");
  std::lock_guard<std::mutex> lk(tables_mu_);
  auto it = tables_.find(name);
  if (it != tables_.end()) {
    if (it->second->dim != dim)
      throw invalid_argument("table already registered with dimension " +
                             std::to_string(it->second->dim));
    return;
  }
  auto t = std::make_unique<Table>();
  t->name = name;
  t->dim = dim;
  t->partition_count = partition_count;
  t->overflow_margin = overflow_margin;
  for (uint32_t i = 0; i < partition_count; ++i) t->parts.push_back(std::make_unique<Partition>());
  tables_.emplace(name, std::move(t));
}

bool VolatileStore::has_table(const std::string& name) const {
  std::lock_guard<std::mutex> lk(tables_mu_);
  return tables_.count(name) != 0;
}

VolatileStore::Table& VolatileStore::table_ref(const std::string& name) const {
  std::lock_guard<std::mutex> lk(tables_mu_);
  auto it = tables_.find(name);
  if (it == tables_.end()) throw invalid_argument("volatile store has no table named " + name);
  return *it->second;
}

uint32_t VolatileStore::dimension(const std::string& name) const { return table_ref(name).dim; }

uint32_t VolatileStore::partition_count(const std::string& name) const {
  return table_ref(name).partition_count;
}

std::vector<uint64_t> VolatileStore::keys(const std::string& name) const {
  Table& t = table_ref(name);
  std::vector<uint64_t> out;
  for (auto& p : t.parts) {
    std::shared_lock<std::shared_mutex> lk(p->mu);
    for (uint32_t s : p->index)
      if (s) out.push_back(p->keys[s - 1]);
  }
  return out;
}

void VolatileStore::upsert(Partition& p, uint32_t dim, uint64_t key, const float* row,
                           uint64_t stamp) {
  int64_t e = p.find(key);
  if (e < 0) {
    // grow the index to keep load <= 1/2
    if ((p.live + 1) * 2 > p.index.size()) {
      const size_t cap = std::max<size_t>(64, p.index.size() * 2);
      Arena<uint32_t> idx(cap, 0);
      for (size_t s = 0; s < p.index.size(); ++s) {
        const uint32_t v = p.index[s];
        if (!v) continue;
        uint64_t h = idx_hash(p.keys[v - 1]) & (cap - 1);
        while (idx[h]) h = (h + 1) & (cap - 1);
        idx[h] = v;
      }
      p.index.swap(idx);
    }
    uint32_t ent;
    if (!p.free_entries.empty()) {
      ent = p.free_entries.back();
      p.free_entries.pop_back();
      p.keys[ent] = key;
      p.last_access[ent] = 0;
    } else {
      ent = uint32_t(p.keys.size());
      p.keys.push_back(key);
      p.last_access.push_back(0);
      p.rows.resize(p.rows.size() + dim);
    }
    const uint64_t mask = p.index.size() - 1;
    uint64_t h = idx_hash(key) & mask;
    while (p.index[h]) h = (h + 1) & mask;
    p.index[h] = ent + 1;
    ++p.live;
    e = ent;
  }
  std::copy(row, row + dim, p.rows.begin() + size_t(e) * dim);
  p.last_access[size_t(e)] = stamp;  // upsert stamps (volatile_store.cpp:137-138)
}

void VolatileStore::erase_entry(Partition& p, uint32_t dim, uint64_t key) {
  (void)dim;
  const uint64_t mask = p.index.size() - 1;
  uint64_t h = idx_hash(key) & mask;
  while (p.index[h] && p.keys[p.index[h] - 1] != key) h = (h + 1) & mask;
  if (!p.index[h]) return;
  const uint32_t ent = p.index[h] - 1;
  // backward-shift deletion keeps probe chains intact
  uint64_t hole = h;
  uint64_t j = (h + 1) & mask;
  while (p.index[j]) {
    const uint64_t home = idx_hash(p.keys[p.index[j] - 1]) & mask;
    const bool movable = (hole <= j) ? (home <= hole || home > j) : (home <= hole && home > j);
    if (movable) {
      p.index[hole] = p.index[j];
      hole = j;
    }
    j = (j + 1) & mask;
  }
  p.index[hole] = 0;
  p.free_entries.push_back(ent);
  --p.live;
}

std::vector<uint64_t> VolatileStore::prune(Table& t, Partition& p) {
  std::vector<uint64_t> evicted;
  if (p.live <= t.overflow_margin) return evicted;
  // EvictOldest: smallest last-access first, ties by smaller key
  std::vector<std::pair<uint64_t, uint64_t>> order;
  order.reserve(p.live);
  for (uint32_t s : p.index) {
    if (s) order.emplace_back(p.last_access[s - 1], p.keys[s - 1]);
  }
  std::sort(order.begin(), order.end());
  const uint64_t excess = p.live - t.overflow_margin;
  for (uint64_t i = 0; i < excess; ++i) {
    erase_entry(p, t.dim, order[i].second);
    evicted.push_back(order[i].second);
  }
  return evicted;
}

std::vector<uint64_t> VolatileStore::insert_rows(Table& t, const uint64_t* keys, size_t n,
                                                 const float* vectors, uint64_t stamp) {
  std::vector<bool> touched(t.partition_count, false);
  for (size_t i = 0; i < n; ++i) {
    const uint32_t pi = partition_of(keys[i], t.partition_count);
    Partition& p = *t.parts[pi];
    std::unique_lock<std::shared_mutex> lk(p.mu);
    upsert(p, t.dim, keys[i], vectors + i * t.dim, stamp);
    touched[pi] = true;
  }
  std::vector<uint64_t> evicted;
  for (uint32_t pi = 0; pi < t.partition_count; ++pi) {
    if (!touched[pi]) continue;
    Partition& p = *t.parts[pi];
    std::unique_lock<std::shared_mutex> lk(p.mu);
    auto v = prune(t, p);
    evicted.insert(evicted.end(), v.begin(), v.end());
  }
  return evicted;
}

std::vector<uint64_t> VolatileStore::insert(const std::string& name, const uint64_t* keys,
                                            size_t n, const float* vectors,
                                            size_t vectors_len) {
  Table& t = table_ref(name);
  if (vectors_len != n * uint64_t(t.dim)) throw invalid_argument("insert vector buffer has wrong size");
  require_finite(vectors, vectors_len, "volatile insert");
  const uint64_t stamp = t.clock.fetch_add(1, std::memory_order_relaxed) + 1;
  return insert_rows(t, keys, n, vectors, stamp);
}

void VolatileStore::insert_async(const std::string& name, std::vector<uint64_t> keys,
                                 std::vector<float> vectors) {
  Table& t = table_ref(name);
  if (vectors.size() != keys.size() * uint64_t(t.dim))
    throw invalid_argument("insert vector buffer has wrong size");
  require_finite(vectors.data(), vectors.size(), "volatile insert");
  {
    std::lock_guard<std::mutex> lk(q_mu_);
    queue_.push_back(Task{&t, std::move(keys), std::move(vectors)});
  }
  q_cv_.notify_one();
}

std::vector<uint64_t> VolatileStore::evict(const std::string& name, uint32_t partition) {
  Table& t = table_ref(name);
  if (partition >= t.partition_count) throw invalid_argument("partition index out of range");
  Partition& p = *t.parts[partition];
  std::unique_lock<std::shared_mutex> lk(p.mu);
  return prune(t, p);
}

void VolatileStore::lookup(const std::string& name, const uint64_t* keys, size_t n,
                           uint64_t* found_keys, float* found_rows, int32_t* found_idx,
                           size_t* n_found, uint64_t* missing_keys, size_t* n_missing) {
  Table& t = table_ref(name);
  const uint64_t stamp = t.clock.fetch_add(1, std::memory_order_relaxed) + 1;
  const uint32_t dim = t.dim;
  // Every partition's shared lock for the whole call (one acquisition per
  // partition instead of per key): entry positions found in pass 1 stay
  // valid for the copies of pass 2. Writers (insert / evict) wait.
  std::vector<std::shared_lock<std::shared_mutex>> held;
  held.reserve(t.parts.size());
  for (auto& p : t.parts) held.emplace_back(p->mu);
  const size_t min_chunk = 512;
  const size_t nchunks =
      std::max<size_t>(1, std::min<size_t>(pool_.size(), (n + min_chunk - 1) / min_chunk));
  const size_t per = (n + nchunks - 1) / nchunks;
  std::vector<const float*> src(n);  // row of each found key, else null
  std::vector<size_t> nf(nchunks, 0);
  // pass 1: index probes, software-prefetched a few keys ahead
  pool_.parallel_for(nchunks, 1, [&](size_t cb, size_t ce) {
    constexpr size_t kAhead = 8;
    for (size_t c = cb; c < ce; ++c) {
      const size_t b = c * per, e = std::min(n, b + per);
      size_t found = 0;
      for (size_t i = b; i < e; ++i) {
        if (i + kAhead < e) {
          const uint64_t kp = keys[i + kAhead];
          const Partition& pp = *t.parts[partition_of(kp, t.partition_count)];
          if (!pp.index.empty())
            __builtin_prefetch(&pp.index[idx_hash(kp) & (pp.index.size() - 1)]);
        }
        const uint64_t k = keys[i];
        Partition& p = *t.parts[partition_of(k, t.partition_count)];
        const int64_t ent = p.find(k);
        if (ent < 0) {
          src[i] = nullptr;
        } else {
          src[i] = p.rows.data() + size_t(ent) * dim;
          __builtin_prefetch(src[i]);
          atomic_max(p.last_access[size_t(ent)], stamp);
          ++found;
        }
      }
      nf[c] = found;
    }
  });
  std::vector<size_t> foff(nchunks + 1, 0), moff(nchunks + 1, 0);
  for (size_t c = 0; c < nchunks; ++c) {
    const size_t len = std::min(n, (c + 1) * per) - std::min(n, c * per);
    foff[c + 1] = foff[c] + nf[c];
    moff[c + 1] = moff[c] + (len - nf[c]);
  }
  // pass 2: rows copied once, straight to their final (input-order) place
  pool_.parallel_for(nchunks, 1, [&](size_t cb, size_t ce) {
    for (size_t c = cb; c < ce; ++c) {
      const size_t b = c * per, e = std::min(n, b + per);
      size_t f = foff[c], m = moff[c];
      for (size_t i = b; i < e; ++i) {
        if (src[i] != nullptr) {
          if (i + 4 < e && src[i + 4] != nullptr) __builtin_prefetch(src[i + 4] + 16);
          found_keys[f] = keys[i];
          std::memcpy(found_rows + f * dim, src[i], size_t(dim) * 4);
          if (found_idx) found_idx[i] = int32_t(f);
          ++f;
        } else {
          missing_keys[m++] = keys[i];
          if (found_idx) found_idx[i] = -1;
        }
      }
    }
  });
  *n_found = foff[nchunks];
  *n_missing = moff[nchunks];
}

void VolatileStore::background_loop() {
  for (;;) {
    Task task;
    {
      std::unique_lock<std::mutex> lk(q_mu_);
      q_cv_.wait(lk, [&] { return stopping_ || !queue_.empty(); });
      if (queue_.empty()) return;
      task = std::move(queue_.front());
      queue_.pop_front();
      busy_ = true;
    }
    Table& t = *task.table;
    const uint64_t stamp = t.clock.fetch_add(1, std::memory_order_relaxed) + 1;
    insert_rows(t, task.keys.data(), task.keys.size(), task.vectors.data(), stamp);
    {
      std::lock_guard<std::mutex> lk(q_mu_);
      busy_ = false;
      if (queue_.empty()) idle_cv_.notify_all();
    }
  }
}

void VolatileStore::drain() {
  std::unique_lock<std::mutex> lk(q_mu_);
  idle_cv_.wait(lk, [&] { return queue_.empty() && !busy_; });
}

uint64_t VolatileStore::partition_size(const std::string& name, uint32_t partition) const {
  Table& t = table_ref(name);
  if (partition >= t.partition_count) throw invalid_argument("partition index out of range");
  Partition& p = *t.parts[partition];
  std::shared_lock<std::shared_mutex> lk(p.mu);
  return p.live;
}

uint64_t VolatileStore::table_size(const std::string& name) const {
  Table& t = table_ref(name);
  uint64_t total = 0;
  for (auto& p : t.parts) {
    std::shared_lock<std::shared_mutex> lk(p->mu);
    total += p->live;
  }
  return total;
}

uint64_t VolatileStore::table_clock(const std::string& name) const {
  return table_ref(name).clock.load(std::memory_order_relaxed);
}

bool VolatileStore::last_access(const std::string& name, uint64_t key, uint64_t* out) const {
  Table& t = table_ref(name);
  Partition& p = *t.parts[partition_of(key, t.partition_count)];
  std::shared_lock<std::shared_mutex> lk(p.mu);
  const int64_t e = p.find(key);
  if (e < 0) return false;
  *out = std::atomic_ref<uint64_t>(p.last_access[size_t(e)]).load();
  return true;
}

}  // namespace hpsb
