// segment_store.cpp -- see segment_store.hpp. Reference behaviour
// (persistent_store.cpp of /root/reference/proj):
//   escape_table_dir        :64-85
//   MANIFEST parsing        :146-165 (same "malformed MANIFEST" fault)
//   segment naming / order  :41-56, :170-188 (seg-<n>.log, ascending n)
//   scan_segment            :229-268 (newest record wins, stop at the first
//                                     incomplete or foreign-dim record)
//   get                     :405-439 (found / missing in input order)
#include "segment_store.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstring>
#include <filesystem>
#include <fstream>

#include "common.cuh"

namespace hpsb {

namespace fs = std::filesystem;

namespace {
constexpr uint64_t kEmpty = ~0ull;
constexpr uint64_t kHeader = 12;  // u64 key + u32 dim
constexpr int kOffsetBits = 48;

inline uint64_t slot_hash(uint64_t key) { return fmix64(key ^ 0x5E65E65E65E65E65ull); }

inline uint64_t load_le64(const unsigned char* p) {
  uint64_t v;
  std::memcpy(&v, p, 8);  // little-endian host (x86-64 / aarch64 LE)
  return v;
}
inline uint32_t load_le32(const unsigned char* p) {
  uint32_t v;
  std::memcpy(&v, p, 4);
  return v;
}

bool parse_segment_number(const std::string& f, uint64_t* number) {
  if (f.size() < 9 || f.rfind("seg-", 0) != 0 || f.substr(f.size() - 4) != ".log") return false;
  const std::string digits = f.substr(4, f.size() - 8);
  if (digits.empty() ||
      !std::all_of(digits.begin(), digits.end(), [](unsigned char c) { return std::isdigit(c); }))
    return false;
  *number = std::stoull(digits);
  return true;
}
}  // namespace

std::string escape_table_dir(const std::string& name) {
  auto safe = [](char c) {
    return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || (c >= '0' && c <= '9') ||
           c == '.' || c == '_' || c == '-';
  };
  static const char* hex = "0123456789ABCDEF";
  std::string out;
  const bool dots = name == "." || name == "..";
  for (char c : name) {
    if (!dots && safe(c)) {
      out.push_back(c);
    } else {
      out.push_back('%');
      out.push_back(hex[(static_cast<unsigned char>(c) >> 4) & 0xF]);
      out.push_back(hex[static_cast<unsigned char>(c) & 0xF]);
    }
  }
  return out;
}

SegmentStore::SegmentStore(std::string root, unsigned threads)
    : root_(std::move(root)),
      pool_(threads ? threads : std::max(1u, std::thread::hardware_concurrency())) {}

SegmentStore::~SegmentStore() {
  for (auto& [name, t] : tables_)
    for (auto& s : t->segs) unmap(s);
}

void SegmentStore::unmap(Segment& s) {
  if (s.base) munmap(const_cast<unsigned char*>(s.base), s.mapped);
  if (s.fd >= 0) close(s.fd);
  s.base = nullptr;
  s.mapped = 0;
  s.fd = -1;
}

SegmentStore::Table& SegmentStore::table_ref(const std::string& name) const {
  std::lock_guard<std::mutex> lk(tables_mu_);
  auto it = tables_.find(name);
  if (it == tables_.end()) throw invalid_argument("persistent store has no table named " + name);
  return *it->second;
}

bool SegmentStore::has_table(const std::string& name) const {
  std::lock_guard<std::mutex> lk(tables_mu_);
  return tables_.count(name) != 0;
}

uint32_t SegmentStore::dimension(const std::string& name) const { return table_ref(name).dim; }

uint64_t SegmentStore::key_count(const std::string& name) const {
  Table& t = table_ref(name);
  std::shared_lock<std::shared_mutex> lk(t.mu);
  return t.live;
}

uint64_t SegmentStore::segment_count(const std::string& name) const {
  Table& t = table_ref(name);
  std::shared_lock<std::shared_mutex> lk(t.mu);
  return t.segs.size();
}

void SegmentStore::attach(const std::string& name) {
  if (has_table(name)) return;
  const fs::path dir = fs::path(root_) / escape_table_dir(name);
  std::ifstream manifest(dir / "MANIFEST");
  if (!manifest) throw invalid_argument("persistent store has no table named " + name);
  std::string mname, line;
  uint32_t dim = 0, version = 0;
  try {
    while (std::getline(manifest, line)) {
      if (line.rfind("name=", 0) == 0) mname = line.substr(5);
      else if (line.rfind("dim=", 0) == 0) dim = uint32_t(std::stoul(line.substr(4)));
      else if (line.rfind("version=", 0) == 0) version = uint32_t(std::stoul(line.substr(8)));
    }
  } catch (const std::exception&) {
    throw tier_fault("malformed MANIFEST in " + dir.string());
  }
  if (mname.empty() || dim == 0 || version != 1)
    throw tier_fault("malformed MANIFEST in " + dir.string());
  if (mname != name) throw tier_fault("MANIFEST in " + dir.string() + " names table " + mname);
  auto t = std::make_unique<Table>();
  t->name = name;
  t->dir = dir.string();
  t->dim = dim;
  {
    std::unique_lock<std::shared_mutex> lk(t->mu);
    load(*t, true);
  }
  std::lock_guard<std::mutex> lk(tables_mu_);
  tables_.emplace(name, std::move(t));
}

void SegmentStore::refresh(const std::string& name) {
  Table& t = table_ref(name);
  std::unique_lock<std::shared_mutex> lk(t.mu);
  load(t, false);
}

void SegmentStore::load(Table& t, bool from_scratch) {
  std::vector<std::pair<uint64_t, std::string>> found;
  for (const auto& e : fs::directory_iterator(t.dir)) {
    if (!e.is_regular_file()) continue;
    uint64_t num = 0;
    if (parse_segment_number(e.path().filename().string(), &num)) found.emplace_back(num, e.path());
  }
  std::sort(found.begin(), found.end());
  if (!from_scratch) {
    // appends only ever grow the last segment and compactions only add a
    // higher-numbered one and delete the old: the old list must survive as
    // a prefix, else re-index from scratch
    bool prefix = found.size() >= t.segs.size();
    for (size_t i = 0; prefix && i < t.segs.size(); ++i)
      prefix = found[i].first == t.segs[i].number;
    from_scratch = !prefix;
  }
  size_t first_scan = 0;
  if (from_scratch) {
    for (auto& s : t.segs) unmap(s);
    t.segs.clear();
    t.keys.assign(1024, 0);
    t.locs.assign(1024, kEmpty);
    t.live = 0;
  } else if (!t.segs.empty()) {
    first_scan = t.segs.size() - 1;  // the last known segment may have grown
  }
  for (size_t i = t.segs.size(); i < found.size(); ++i) {
    Segment s;
    s.number = found[i].first;
    s.path = found[i].second;
    t.segs.push_back(std::move(s));
  }
  if (t.segs.size() > (size_t(1) << (64 - kOffsetBits)))
    throw tier_fault("too many segments in " + t.dir);
  for (size_t i = first_scan; i < t.segs.size(); ++i) {
    Segment& s = t.segs[i];
    if (s.fd < 0) {
      s.fd = open(s.path.c_str(), O_RDONLY | O_CLOEXEC);
      if (s.fd < 0) throw tier_fault("cannot open segment " + s.path);
    }
    struct stat sb {};
    if (fstat(s.fd, &sb) != 0) throw tier_fault("cannot stat " + s.path);
    const uint64_t size = uint64_t(sb.st_size);
    if (size > s.mapped) {
      if (s.base) munmap(const_cast<unsigned char*>(s.base), s.mapped);
      s.base = nullptr;
      s.mapped = 0;
      void* p = mmap(nullptr, size, PROT_READ, MAP_SHARED, s.fd, 0);
      if (p == MAP_FAILED) throw tier_fault("cannot map segment " + s.path);
      madvise(p, size, MADV_RANDOM);
      s.base = static_cast<const unsigned char*>(p);
      s.mapped = size;
    }
    scan_from(t, i);
  }
}

void SegmentStore::scan_from(Table& t, size_t slot) {
  Segment& s = t.segs[slot];
  const uint64_t payload = 4ull * t.dim;
  uint64_t pos = s.good;
  while (s.mapped - pos >= kHeader) {
    const uint64_t key = load_le64(s.base + pos);
    const uint32_t rdim = load_le32(s.base + pos + 8);
    if (rdim != t.dim || s.mapped - pos - kHeader < payload) break;
    index_put(t, key, (uint64_t(slot) << kOffsetBits) | (pos + kHeader));
    pos += kHeader + payload;
  }
  s.good = pos;
}

void SegmentStore::index_put(Table& t, uint64_t key, uint64_t loc) {
  if ((t.live + 1) * 2 > t.locs.size()) {
    const size_t cap = t.locs.size() * 2;
    std::vector<uint64_t> k2(cap, 0), l2(cap, kEmpty);
    for (size_t i = 0; i < t.locs.size(); ++i) {
      if (t.locs[i] == kEmpty) continue;
      uint64_t h = slot_hash(t.keys[i]) & (cap - 1);
      while (l2[h] != kEmpty) h = (h + 1) & (cap - 1);
      k2[h] = t.keys[i];
      l2[h] = t.locs[i];
    }
    t.keys.swap(k2);
    t.locs.swap(l2);
  }
  const uint64_t mask = t.locs.size() - 1;
  uint64_t h = slot_hash(key) & mask;
  while (t.locs[h] != kEmpty) {
    if (t.keys[h] == key) {
      t.locs[h] = loc;  // a later record of the key wins
      return;
    }
    h = (h + 1) & mask;
  }
  t.keys[h] = key;
  t.locs[h] = loc;
  ++t.live;
}

int64_t SegmentStore::index_find(const Table& t, uint64_t key) const {
  const uint64_t mask = t.locs.size() - 1;
  uint64_t h = slot_hash(key) & mask;
  while (t.locs[h] != kEmpty) {
    if (t.keys[h] == key) return int64_t(h);
    h = (h + 1) & mask;
  }
  return -1;
}

void SegmentStore::get(const std::string& name, const uint64_t* keys, size_t n,
                       uint64_t* found_keys, float* found_rows, int32_t* found_idx,
                       size_t* n_found, uint64_t* missing_keys, size_t* n_missing) {
  Table& t = table_ref(name);
  std::shared_lock<std::shared_mutex> lk(t.mu);
  const uint32_t dim = t.dim;
  const size_t min_chunk = 256;
  const size_t nchunks =
      std::max<size_t>(1, std::min<size_t>(pool_.size(), (n + min_chunk - 1) / min_chunk));
  const size_t per = (n + nchunks - 1) / nchunks;
  std::vector<const unsigned char*> src(n);
  std::vector<size_t> nf(nchunks, 0);
  // pass 1: index probes (prefetched a few keys ahead); the payload's page
  // is touched here so the copies of pass 2 find it resident
  pool_.parallel_for(nchunks, 1, [&](size_t cb, size_t ce) {
    constexpr size_t kAhead = 8;
    const uint64_t mask = t.locs.size() - 1;
    for (size_t c = cb; c < ce; ++c) {
      const size_t b = c * per, e = std::min(n, b + per);
      size_t found = 0;
      for (size_t i = b; i < e; ++i) {
        if (i + kAhead < e) __builtin_prefetch(&t.locs[slot_hash(keys[i + kAhead]) & mask]);
        const int64_t h = index_find(t, keys[i]);
        if (h < 0) {
          src[i] = nullptr;
          continue;
        }
        const uint64_t loc = t.locs[size_t(h)];
        const Segment& s = t.segs[loc >> kOffsetBits];
        src[i] = s.base + (loc & ((uint64_t(1) << kOffsetBits) - 1));
        __builtin_prefetch(src[i]);
        ++found;
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
          if (i + 4 < e && src[i + 4] != nullptr) __builtin_prefetch(src[i + 4]);
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

}  // namespace hpsb
