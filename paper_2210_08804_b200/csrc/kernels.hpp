// kernels.hpp -- host-side launchers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace hpsb {

// Process-wide count of kernels launched by this library (bench.py reports
// it as gpu_launches for the timed region).
void note_launches(uint32_t kernels);
uint64_t launch_count();

// Look-back scan state of one serialised user (a cache or a workspace).
struct ScanState {
  uint64_t* status = nullptr;             // one word per tile
  unsigned long long* tile_ctr = nullptr; // cumulative tile ticket counter
  uint64_t capacity_tiles = 0;
  unsigned long long tile_base = 0;       // tickets issued so far
  uint32_t epoch = 0;                     // 24-bit epoch of the next launch
};

// Tile geometry of the ordered-compaction kernels.
constexpr int kScanBlock = 256;
constexpr int kScanItems = 4;
constexpr uint64_t kScanTile = uint64_t(kScanBlock) * kScanItems;
constexpr uint64_t kDumpTile = uint64_t(kScanBlock);  // slabs per dump tile

// Prepares `s` for one launch of `tiles` tiles; returns false if the status
// array had to be cleared (epoch wrap) -- handled internally.
void scan_begin(ScanState& s, uint64_t tiles, cudaStream_t st);

// ---- cache-level operations (slab_cache.cpp) ----
void launch_cache_query(const CacheDev& c, const uint64_t* keys, uint64_t n, float* out,
                        uint8_t* hit, uint64_t stamp, int keys_per_warp, cudaStream_t st);
void launch_select_misses(const uint64_t* keys, const uint8_t* hit, uint64_t n,
                          uint32_t* miss_pos, uint64_t* miss_keys,
                          unsigned long long* n_miss, ScanState& scan, cudaStream_t st);

// Replace scratch (persistent: the kernels leave it in its initial state --
// set1 / cnt zero, ovf / boff all-ones -- so calls need no memsets).
// A per-call table of the touched slabsets (open addressing on the set id):
// each key finds its set's entry and appends its index there (the first
// kReplaceInline inline, the rest on an overflow list); the key that arrived
// first leads the set.
constexpr uint32_t kReplaceInline = 8;
struct ReplaceScratch {
  uint64_t cap = 0;      // set-table entries (power of two >= 2 * ncap)
  uint64_t ncap = 0;     // keys per call
  unsigned long long* ent = nullptr;  // cap: (slabset + 1) << 32 | keys of the set (0 = free)
  uint32_t* idx = nullptr;    // cap * kReplaceInline: key indices, arrival order
  uint64_t* kin = nullptr;    // cap * kReplaceInline: the keys themselves
  uint32_t* hin = nullptr;    // cap * kReplaceInline: their slab-hash meta (tag << 24 | first slab)
  uint32_t* ovf = nullptr;    // cap: overflow list head (~0 = none)
  uint32_t* boff = nullptr;   // cap: sorted bucket of a set with > 32 keys (~0 = none)
  uint32_t* next = nullptr;   // ncap: overflow list links
  uint32_t* lead_e = nullptr; // ncap: touched sets' table entries, compact (~0 = none)
  uint32_t* lead_s = nullptr; // ncap: their slabsets
  uint32_t* bucket = nullptr; // ncap: buckets of sets with > 32 keys
  uint32_t* cursor = nullptr; // [0] bucket cursor, [1] duplicate flag, [2] touched-set count
  uint32_t* dup_flag = nullptr;
};
// Bytes of a scratch for calls of up to n keys; carving; the one-time
// initialisation (enqueued on st).
size_t replace_scratch_bytes(uint64_t n);
ReplaceScratch replace_scratch_carve(void* base, uint64_t n);
void replace_scratch_init(const ReplaceScratch& rs, cudaStream_t st);
void launch_replace(const CacheDev& c, const uint64_t* keys, uint64_t n, const float* rows,
                    uint64_t stamp, bool validate, const ReplaceScratch& rs, cudaStream_t st,
                    int device);
// The opt-in relaxed mode (atomicCAS slot claims, every key at once; keys
// must be distinct): false when the geometry has no relaxed kernel (W > 4),
// then the caller runs the exact path. `claimed` = n u64 of device scratch
// (each key's won slot); *dropped (device) counts keys that found no
// claimable slot.
bool launch_replace_relaxed(const CacheDev& c, const uint64_t* keys, uint64_t n, const float* rows,
                            uint64_t stamp, uint64_t* claimed, unsigned long long* dropped,
                            cudaStream_t st);

// Update (slab_cache.cpp:109-125): scratch = update_scratch_bytes(n) of
// device memory (per-position slots + per-block hit counts); winner = the
// cache's per-slot u32 array (all-zero between calls); *written = number of
// positions whose key is resident (device memory, no pre-zeroing needed).
// after_lookup: the previous operation on `st` is a lookup kernel -> the
// probe launches as its programmatic dependent (and completes after it).
size_t update_scratch_bytes(uint64_t n);
void launch_update(const CacheDev& c, const uint64_t* keys, uint64_t n, const float* rows,
                   void* scratch, uint32_t* winner, unsigned long long* written,
                   bool after_lookup, cudaStream_t st);

void launch_dump(const CacheDev& c, uint64_t set_begin, uint64_t set_end, uint64_t* out,
                 unsigned long long* n_out, ScanState& scan, cudaStream_t st);

// ---- dedup (types.cpp:20-34) ----
struct DedupScratch {
  uint64_t cap = 0;
  uint64_t* table = nullptr;       // cap, (epoch << 32) | first position
  uint32_t* slot_of = nullptr;     // n
  uint32_t* rank_of_slot = nullptr;  // cap
  unsigned long long* n_unique = nullptr;
};
void launch_dedup(const uint64_t* keys, uint64_t n, uint64_t* unique_out, uint32_t* inverse,
                  const DedupScratch& ds, uint32_t table_epoch, ScanState& scan,
                  cudaStream_t st);

// ---- lookup (lookup_engine.cpp:130-241) ----
// Scratch of ONE lookup call. A lookup's unique misses come out as a CLAIM
// LIST (one entry per missing key, in claim order) with each key's
// first-occurrence position; sorting the claims by that position gives the
// reference's order (dedup first-occurrence order, types.cpp:20-34, then
// ascending miss positions, slab_cache.cpp:84-89). Every field is back to
// its initial state (zero) when the call completes.
struct LookupView {
  uint64_t cap = 0;                       // miss table capacity (power of two >= 2 * batch)
  uint32_t* miss_table = nullptr;         // 0 = empty, else first position + 1
  uint32_t* claim_of_slot = nullptr;      // miss-table slot -> claim index
  uint32_t* miss_slot = nullptr;          // per position (valid where missed)
  uint32_t* list = nullptr;               // claim -> miss-table slot (capacity batch)
  uint64_t* list_keys = nullptr;          // claim -> key (per-call destination)
  uint32_t* list_firsts = nullptr;        // claim -> first position (per-call destination)
  unsigned long long* counts = nullptr;   // distributed (unique hit, unique miss) pairs
  unsigned long long* counts_out = nullptr;  // [2] per-call destination
  uint32_t* list_ctr = nullptr;           // claims so far
  uint32_t* done = nullptr;               // [2] block tickets (claims done, counts done)
  // diagnostic phase timeline (HPSB_TRACE): 8 u64 per call, filled with
  // 0xFF before the call; fields hold min(t) or min(~t) (= max t) over blocks
  unsigned long long* trace = nullptr;
  // ---- ordering between overlapping calls ----
  unsigned long long* completed = nullptr;  // uses of this view completed so far
  unsigned long long gen = 0;               // this call's use number of the view
  // the previous call on the stream (its completion precedes this call's)
  const unsigned long long* prev_completed = nullptr;
  unsigned long long prev_target = 0;
  // distinct hit slots of the call (open addressing, `cap` entries, 2^log2cap):
  // (low 32 bits of the call's stamp << 32) | slot. An entry whose tag is not
  // this call's stamp is free (a previous use of the view), so the table needs
  // no clearing between calls; inserting a slot for the first time counts one
  // unique hit. Cleared only when the stamps' high 32 bits change
  // (DeviceCache::prepare_hits).
  unsigned long long* hits = nullptr;
  uint32_t log2cap = 0;
  // graph replay (DeviceCache capture sessions): stamp, gen and prev_target
  // are relative to device words written before every launch of the graph
  // ([0] stamp base, [1 + view] use base of view `view`); nullptr = absolute
  const unsigned long long* rebase = nullptr;
  uint32_t idx = 0, prev_idx = 0;  // this call's / the previous call's view index
  // zero-copy engine calls: a device copy of the miss flags (the output flags
  // live in pinned host memory; the sync branch's scatter reads this copy)
  uint8_t* flags_dev = nullptr;
};
// A ring of views: consecutive lookups on one stream take consecutive views,
// so up to kLookupViews calls can be in flight (programmatic dependent
// launch); a call waits on the device until the previous use of its view
// has completed.
#ifndef HPSB_LOOKUP_VIEWS
#define HPSB_LOOKUP_VIEWS 8
#endif
constexpr int kLookupViews = HPSB_LOOKUP_VIEWS;
struct LookupScratch {
  LookupView v[kLookupViews];
  uint64_t uses[kLookupViews] = {};  // host: uses handed out per view
  int nviews = kLookupViews;         // views in the ring (1 for unchained users)
  int next = 0;
  int last = -1;
  // hit tables of every view, contiguous (one memset clears them)
  void* hits_base = nullptr;
  uint64_t hits_bytes = 0;
  uint64_t hit_epoch = ~0ull;  // stamp >> 32 the tables are valid for
};
// The view of the next call (host bookkeeping). chain: the call is launched
// as a programmatic dependent of the previous call taken from this scratch,
// whose completion it then waits for before completing.
LookupView lookup_next_view(LookupScratch& ls, bool chain);
// Bytes / carving of a LookupScratch of `nviews` views for batches of up to
// `cap` keys (the caller zero-fills the block once; carving resets the host
// bookkeeping).
size_t lookup_scratch_bytes(uint64_t cap, int nviews = kLookupViews);
LookupScratch lookup_scratch_carve(void* base, uint64_t cap, int nviews = kLookupViews);
// Writes the rebase words of a captured graph's lookups (one thread):
// w[0] = stamp base, w[1 + k] = use base of view k.
void launch_rebase(unsigned long long* w, unsigned long long stamp_base,
                   const unsigned long long (&use_base)[kLookupViews], cudaStream_t st);
// One launch per lookup (probe, claims, stamps, row gather / default rows,
// and the call's completion by its last block). after_lookup: the previous
// operation on `st` was a lookup or update kernel -> launched as its
// programmatic dependent; wait_before_copy (after an update): the rows are
// read only once that update's grid has completed. Returns the number of
// kernels launched.
unsigned launch_lookup_probe(const CacheDev& c, const uint64_t* keys, uint64_t n, float* out,
                             uint8_t* flags, const float* default_row, uint64_t stamp,
                             const LookupView& v, bool after_lookup, cudaStream_t st,
                             bool wait_before_copy = false);
// One table of a multi-table lookup launch (device-resident descriptor).
struct TableLookup {
  CacheDev c;
  const uint64_t* keys;
  uint64_t n;
  float* out;
  uint8_t* flags;
  const float* default_row;
  uint64_t stamp;
  LookupView v;
  uint32_t block_begin;  // first block of this table in the launch
  uint32_t nblocks;      // ceil(n / 256)
};
constexpr uint32_t kMultiBlockPositions = 256;  // positions per block of the multi kernel
// One launch for `count` tables (descriptors in device memory, block ranges
// consecutive); ch = row chunk width valid for every table (8, 4 or 1).
void launch_lookup_multi(const TableLookup* d_tables, uint32_t count, uint32_t total_blocks,
                         int ch, cudaStream_t st);
void launch_lookup_scatter(uint64_t n, uint32_t d, uint8_t* flags, const LookupView& v,
                           const int32_t* row_of_claim, const float* staged, float* out,
                           cudaStream_t st);

// ---- key-hash-sharded mode (shard_kernels.cu) ----
uint32_t shard_of(uint64_t key, uint32_t world);
void launch_shard_count(const uint64_t* keys, uint64_t n, uint32_t world,
                        unsigned long long* counts, cudaStream_t st);
void launch_shard_scatter(const uint64_t* keys, uint64_t n, uint32_t world,
                          unsigned long long* cursor, uint64_t* send_keys, uint32_t* send_pos,
                          cudaStream_t st);
void launch_shard_unroute(uint64_t m, uint32_t d, const uint32_t* send_pos, const float* rows,
                          const uint8_t* flags_in, float* out, uint8_t* flags_out,
                          cudaStream_t st);

// ---- wire LOOKUP response frames (wire.cu; wire.hpp:18-21) ----
size_t wire_lookup_frame_bytes(uint64_t count, uint32_t dim);
void wire_encode_lookup_host(const float* rows, const uint8_t* flags, uint32_t count, uint32_t dim,
                             uint8_t* frame);
void wire_encode_lookup_device(const float* d_rows, const uint8_t* d_flags, uint32_t count,
                               uint32_t dim, uint8_t* d_bitmap_scratch, uint8_t* frame,
                               cudaStream_t st);

}  // namespace hpsb
