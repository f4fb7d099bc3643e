// segment_store.hpp -- batched cold reads over the reference's persistent
// store files.
//
// The reference's PersistentStore::get (persistent_store.cpp:405-439) serves
// a cold-tier fetch key by key: an unordered_map probe and one pread(2) per
// key under the table's shared lock. This reader opens the SAME on-disk
// layout read-only (persistent_store.hpp:5-15):
//   <root>/<escaped table name>/MANIFEST   name=, dim=, version=1
//   <root>/<escaped table name>/seg-<n>.log records [u64 key][u32 dim][dim f32]
// rebuilds the newest-record-wins index exactly as the reference's open does
// (segments in ascending number, records in file order, a segment's scan
// stopping at its first incomplete / foreign-dimension record,
// persistent_store.cpp:229-268), memory-maps every segment, and answers a
// whole batch at once: index probes fan out over a thread pool, the rows are
// copied straight from the page cache into the caller's (pinned staging)
// buffer in input order -- no syscall per key, no per-key allocation.
//
// It is a READER: records the reference still holds in its unflushed
// in-memory tail are not visible until they are flushed and refresh() has
// picked them up (refresh() also follows compactions: a changed segment set
// is re-indexed from scratch). The serving deployment this is for -- a PDB
// written by the offline / update pipeline and read during serving -- is the
// reference's own (§3, initial cache rate < 1 => cold reads).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <shared_mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "runtime.hpp"

namespace hpsb {

// persistent_store.cpp:64-85 (%XX escaping of anything outside [A-Za-z0-9._-])
std::string escape_table_dir(const std::string& name);

class SegmentStore {
 public:
  SegmentStore(std::string root, unsigned threads);
  ~SegmentStore();

  // Indexes <root>/<escaped name>; throws invalid_argument when the table
  // directory or its MANIFEST is absent, tier_fault when it is malformed.
  void attach(const std::string& name);
  bool has_table(const std::string& name) const;
  uint32_t dimension(const std::string& name) const;
  uint64_t key_count(const std::string& name) const;
  uint64_t segment_count(const std::string& name) const;
  // Picks up flushed appends and new / compacted segments.
  void refresh(const std::string& name);

  // PersistentStore::get's contract: found keys / rows and missing keys, both
  // in input order; found_idx (optional, n entries) = each input key's found
  // row or -1. found_keys / missing_keys hold n entries, found_rows n * dim.
  void get(const std::string& name, const uint64_t* keys, size_t n, uint64_t* found_keys,
           float* found_rows, int32_t* found_idx, size_t* n_found, uint64_t* missing_keys,
           size_t* n_missing);

 private:
  struct Segment {
    uint64_t number = 0;
    std::string path;
    int fd = -1;
    const unsigned char* base = nullptr;  // read-only mapping
    uint64_t mapped = 0;                  // bytes mapped
    uint64_t good = 0;                    // scanned prefix (complete records)
  };
  struct Table {
    std::string name, dir;
    uint32_t dim = 0;
    mutable std::shared_mutex mu;
    std::vector<Segment> segs;
    // open addressing: key -> location (segment << 48 | payload offset);
    // kEmpty = free slot
    std::vector<uint64_t> keys, locs;
    uint64_t live = 0;
  };

  Table& table_ref(const std::string& name) const;
  void load(Table& t, bool from_scratch);
  void scan_from(Table& t, size_t slot);
  void index_put(Table& t, uint64_t key, uint64_t loc);
  int64_t index_find(const Table& t, uint64_t key) const;
  static void unmap(Segment& s);

  std::string root_;
  mutable std::mutex tables_mu_;
  std::unordered_map<std::string, std::unique_ptr<Table>> tables_;
  ThreadPool pool_;
};

}  // namespace hpsb
