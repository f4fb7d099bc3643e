// volatile_store.hpp -- host volatile DB (level-2 tier) for the miss path.
//
// Same contract as hps::VolatileStore (volatile_store.hpp:45-137 of the
// reference): per-table hash partitions routed by xxh64(key, 0) % P,
// upsert + evict-oldest down to the overflow margin (ties by smaller key),
// one clock tick per lookup / insert call, last-access refresh that never
// moves a stamp backwards. Storage is built for the GPU miss path instead
// of per-key std::vector rows: each partition keeps an open-addressing index
// over one contiguous row arena, lookups fan out over a thread pool in
// input-order chunks, and found rows are copied straight into a (pinned)
// staging buffer in found order. Refreshes are applied inline with an
// atomic max (the reference queues them to a background thread; the
// drained state is identical).
#pragma once

#include <atomic>
#include <sys/mman.h>

#include <condition_variable>
#include <cstdlib>
#include <new>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "runtime.hpp"

namespace hpsb {

uint32_t partition_of(uint64_t key, uint32_t partition_count);  // volatile_store.cpp:10-13

class VolatileStore {
 public:
  explicit VolatileStore(unsigned lookup_threads);
  ~VolatileStore();

  void register_table(const std::string& name, uint32_t dim, uint32_t partition_count,
                      uint64_t overflow_margin);
  bool has_table(const std::string& name) const;
  uint32_t dimension(const std::string& name) const;
  uint32_t partition_count(const std::string& name) const;
  // Every resident key, partition by partition (volatile_store.cpp:293-303).
  std::vector<uint64_t> keys(const std::string& name) const;

  // Upsert + prune touched partitions; returns evicted keys.
  std::vector<uint64_t> insert(const std::string& name, const uint64_t* keys, size_t n,
                               const float* vectors, size_t vectors_len);
  void insert_async(const std::string& name, std::vector<uint64_t> keys,
                    std::vector<float> vectors);
  std::vector<uint64_t> evict(const std::string& name, uint32_t partition);

  // Lookup in input order. found_rows receives n_found * dim floats in found
  // order; found_idx (optional, n entries) gets the found row index of each
  // input key or -1. found_keys / missing_keys hold n entries.
  void lookup(const std::string& name, const uint64_t* keys, size_t n, uint64_t* found_keys,
              float* found_rows, int32_t* found_idx, size_t* n_found, uint64_t* missing_keys,
              size_t* n_missing);

  void drain();

  uint64_t partition_size(const std::string& name, uint32_t partition) const;
  uint64_t table_size(const std::string& name) const;
  uint64_t table_clock(const std::string& name) const;
  bool last_access(const std::string& name, uint64_t key, uint64_t* out) const;

 private:
  // Arena storage on transparent huge pages (2 MB): a table of 10 M rows of
  // 512 B is 5 GB, and a miss batch touches its rows at random -- with 4 KB
  // pages nearly every row copy is also a TLB miss.
  template <class T>
  struct HugePageAllocator {
    using value_type = T;
    static constexpr size_t kHuge = size_t(2) << 20;
    HugePageAllocator() = default;
    template <class U>
    HugePageAllocator(const HugePageAllocator<U>&) {}
    T* allocate(size_t n) {
      const size_t bytes = n * sizeof(T);
      if (bytes < kHuge) return static_cast<T*>(::operator new(bytes));
      const size_t rounded = (bytes + kHuge - 1) & ~(kHuge - 1);
      void* p = std::aligned_alloc(kHuge, rounded);
      if (p == nullptr) throw std::bad_alloc();
      (void)::madvise(p, rounded, MADV_HUGEPAGE);
      return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t n) {
      if (n * sizeof(T) < kHuge)
        ::operator delete(p);
      else
        std::free(p);
    }
    template <class U>
    bool operator==(const HugePageAllocator<U>&) const { return true; }
  };
  template <class T>
  using Arena = std::vector<T, HugePageAllocator<T>>;
  struct Partition {
    mutable std::shared_mutex mu;
    // open addressing: slot -> entry index + 1 (0 = empty)
    Arena<uint32_t> index;
    Arena<uint64_t> keys;                   // per entry
    Arena<uint64_t> last_access;            // per entry (updated with atomic_ref max)
    Arena<float> rows;                      // entry * dim
    std::vector<uint32_t> free_entries;
    uint64_t live = 0;
    int64_t find(uint64_t key) const;       // entry or -1
  };
  struct Table {
    std::string name;
    uint32_t dim = 0;
    uint32_t partition_count = 16;
    uint64_t overflow_margin = 1u << 20;
    std::atomic<uint64_t> clock{0};
    std::vector<std::unique_ptr<Partition>> parts;
  };
  struct Task {
    Table* table;
    std::vector<uint64_t> keys;
    std::vector<float> vectors;
  };

  Table& table_ref(const std::string& name) const;
  std::vector<uint64_t> insert_rows(Table& t, const uint64_t* keys, size_t n,
                                    const float* vectors, uint64_t stamp);
  static void upsert(Partition& p, uint32_t dim, uint64_t key, const float* row, uint64_t stamp);
  static std::vector<uint64_t> prune(Table& t, Partition& p);
  static void erase_entry(Partition& p, uint32_t dim, uint64_t key);
  void background_loop();

  mutable std::mutex tables_mu_;
  std::unordered_map<std::string, std::unique_ptr<Table>> tables_;
  ThreadPool pool_;

  std::mutex q_mu_;
  std::condition_variable q_cv_, idle_cv_;
  std::deque<Task> queue_;
  bool busy_ = false;
  bool stopping_ = false;
  std::thread worker_;
};

}  // namespace hpsb
