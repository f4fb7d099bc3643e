// include/hps/slab_cache.hpp -- drop-in replacement for the reference's
// core/include/hps/slab_cache.hpp (hps::SlabCache, slab_cache.hpp:23-178),
// backed by the B200 cache of libhps_b200.so through the C ABI
// (include/hps_b200.h). Same class, same members, same semantics and error
// behaviour; the embedding table lives in HBM on `device` and every call is
// synchronous host-pointer I/O like the reference's (the device-pointer,
// stream-ordered fast path is the C ABI's HPS_MEM_DEVICE mode).
//
// A reference build switches by putting this repo's include/ ahead of
// core/include on the include path and linking libhps_b200.so instead of
// compiling core/src/slab_cache.cpp. The reference's own
// unit test tests/unit/test_slab_cache.cpp compiles unchanged against this
// header (oracle/Makefile target _ref/test_slab_cache_b200).
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hps_b200.h"

#if __has_include("hps/types.hpp")
#include "hps/types.hpp"  // the reference's vocabulary, when present
#else
namespace hps {
using EmbeddingKey = std::uint64_t;
class TierFault : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
}  // namespace hps
#endif

namespace hps {

inline constexpr std::uint32_t kSlotsPerSlab = 32;

// slab_cache.hpp:27-34
struct SlabCacheConfig {
  std::size_t slabset_count = 1;
  std::uint32_t slabs_per_set = 2;
  std::uint32_t dimension = 0;
  // Accepted and validated like the reference (0 is rejected); on the GPU
  // they set how many keys one warp keeps in flight.
  std::uint32_t worker_pool_size = 1;
  std::uint32_t tasks_per_worker = 8;
};

// slab_cache.hpp:36-39
struct CacheMiss {
  std::size_t position;  // index into the query key span
  EmbeddingKey key;
};

namespace b200_detail {
// C ABI status -> the reference's exception types.
inline void check(int rc) {
  if (rc == HPS_OK) return;
  const std::string what = hps_last_error();
  switch (rc) {
    case HPS_INVALID_ARGUMENT: throw std::invalid_argument(what);
    case HPS_LOGIC_ERROR: throw std::logic_error(what);
    case HPS_TIER_FAULT: throw TierFault(what);
    case HPS_OUT_OF_MEMORY: throw std::bad_alloc();
    default: throw std::runtime_error(what);
  }
}
}  // namespace b200_detail

class SlabCache {
 public:
  // slab_cache.cpp:17-41 (same validation and messages); `device` selects
  // the GPU that holds this replica.
  explicit SlabCache(const SlabCacheConfig& config, int device = 0) {
    const hps_cache_config c{config.slabset_count, config.slabs_per_set, config.dimension,
                             config.worker_pool_size, config.tasks_per_worker};
    b200_detail::check(hps_cache_create(&c, device, &h_));
    hps_cache_info i{};
    b200_detail::check(hps_cache_get_info(h_, &i));
    dimension_ = i.dimension;
    slabs_per_set_ = i.slabs_per_set;
    slabset_count_ = i.slabset_count;
  }
  ~SlabCache() { hps_cache_destroy(h_); }

  SlabCache(const SlabCache&) = delete;
  SlabCache& operator=(const SlabCache&) = delete;

  // slab_cache.cpp:69-91: the clock advances once, even for an empty query
  // or a wrongly sized output; misses in ascending position order; miss
  // rows untouched.
  std::vector<CacheMiss> query(std::span<const EmbeddingKey> keys, std::span<float> out_vectors) {
    std::vector<std::uint32_t> pos(keys.size());
    std::vector<std::uint64_t> mk(keys.size());
    std::size_t n_miss = 0;
    b200_detail::check(hps_cache_query(h_, keys.data(), keys.size(), out_vectors.data(),
                                       out_vectors.size(), pos.data(), mk.data(), &n_miss,
                                       HPS_MEM_HOST, nullptr));
    std::vector<CacheMiss> misses(n_miss);
    for (std::size_t i = 0; i < n_miss; ++i) misses[i] = CacheMiss{pos[i], mk[i]};
    return misses;
  }

  // slab_cache.cpp:93-107: duplicates / wrong size rejected before any
  // mutation; resident keys only get their recency refreshed.
  void replace(std::span<const EmbeddingKey> keys, std::span<const float> vectors) {
    b200_detail::check(hps_cache_replace(h_, keys.data(), keys.size(), vectors.data(),
                                         vectors.size(), HPS_MEM_HOST, nullptr));
  }

  // slab_cache.cpp:109-125: overwrite resident rows, never admit, recency
  // untouched; returns the number of positions written.
  std::size_t update(std::span<const EmbeddingKey> keys, std::span<const float> vectors) {
    std::size_t written = 0;
    b200_detail::check(hps_cache_update(h_, keys.data(), keys.size(), vectors.data(),
                                        vectors.size(), &written, HPS_MEM_HOST, nullptr));
    return written;
  }

  // slab_cache.cpp:360-394: batches in set / slab / slot order; each range
  // of slabsets is read in one stream-ordered device pass, so every key
  // resident for the cursor's lifetime shows up exactly once.
  class DumpCursor {
   public:
    bool next(std::vector<EmbeddingKey>& out) {
      out.clear();
      for (;;) {
        while (staged_pos_ < staged_.size() && out.size() < batch_size_)
          out.push_back(staged_[staged_pos_++]);
        if (out.size() == batch_size_) return true;
        if (next_set_ == cache_->slabset_count_) return !out.empty();
        const std::size_t end = std::min(cache_->slabset_count_, next_set_ + kSetsPerStage);
        staged_.assign((end - next_set_) * cache_->slabs_per_set_ * kSlotsPerSlab, 0);
        std::size_t n = 0;
        b200_detail::check(hps_cache_dump(cache_->h_, next_set_, end, staged_.data(),
                                          staged_.size(), &n));
        staged_.resize(n);
        staged_pos_ = 0;
        next_set_ = end;
      }
    }

   private:
    friend class SlabCache;
    static constexpr std::size_t kSetsPerStage = 1024;
    DumpCursor(SlabCache* cache, std::size_t batch_size) : cache_(cache), batch_size_(batch_size) {}
    SlabCache* cache_;
    std::size_t batch_size_;
    std::size_t next_set_ = 0;
    std::vector<EmbeddingKey> staged_;
    std::size_t staged_pos_ = 0;
  };

  DumpCursor dump(std::size_t batch_size) {
    if (batch_size == 0) throw std::invalid_argument("dump batch size must be positive");
    return DumpCursor(this, batch_size);
  }
  std::vector<EmbeddingKey> dump_all() {
    std::vector<EmbeddingKey> all;
    auto cursor = dump(4096);
    std::vector<EmbeddingKey> batch;
    while (cursor.next(batch)) all.insert(all.end(), batch.begin(), batch.end());
    return all;
  }

  std::uint32_t dimension() const { return dimension_; }
  std::size_t slabset_count() const { return slabset_count_; }
  std::uint32_t slabs_per_set() const { return slabs_per_set_; }
  std::size_t capacity() const { return slabset_count_ * slabs_per_set_ * kSlotsPerSlab; }
  std::size_t occupied() const { return info().occupied; }
  std::uint64_t recency_clock() const { return info().recency_clock; }

  // slab_cache.cpp:60-67 (XXH64 placement, pinned by golden vectors)
  static std::size_t slabset_of(EmbeddingKey key, std::size_t slabset_count) {
    return hps_slabset_of(key, slabset_count);
  }
  static std::uint32_t first_slab_of(EmbeddingKey key, std::uint32_t slabs_per_set) {
    return hps_first_slab_of(key, slabs_per_set);
  }

  // slab_cache.cpp:407-442 (+ the device fingerprint array); throws
  // std::logic_error on violation.
  void check_invariants() const { b200_detail::check(hps_cache_check_invariants(h_)); }

  // B200 extras: the C handle (device-pointer / stream-ordered calls).
  hps_cache* handle() const { return h_; }
  // The opt-in relaxed replace mode (atomicCAS slot claims for replaces of
  // distinct keys; include/hps_b200.h hps_cache_set_replace_mode). The
  // default, exact mode is slot-exact with the reference.
  void set_relaxed_replace(bool relaxed) {
    b200_detail::check(
        hps_cache_set_replace_mode(h_, relaxed ? HPS_REPLACE_RELAXED : HPS_REPLACE_EXACT));
  }

 private:
  hps_cache_info info() const {
    hps_cache_info i{};
    b200_detail::check(hps_cache_get_info(h_, &i));
    return i;
  }
  hps_cache* h_ = nullptr;
  std::uint32_t dimension_ = 0;
  std::uint32_t slabs_per_set_ = 0;
  std::size_t slabset_count_ = 0;
};

}  // namespace hps
