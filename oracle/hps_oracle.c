/*
 * hps_oracle.c -- CPU restatement of the reference lookup path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker for the
 * B200 product path in paper_2210_08804_b200/. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it, and only as a checker or as the timed CPU baseline --
 * never as a fallback for the product.
 *
 * Parity status: PINNED. The hash is checked against the reference's golden
 * vectors (tests/golden/xxh64_vectors.json, taken from
 * proj/tests/unit/test_core.cpp:26-95), and the cache model is checked
 * op-for-op against the reference SlabCache built from its own sources
 * (oracle/_ref, see oracle/Makefile) and against committed fixtures
 * generated from it (tests/golden/gen_golden.py).
 *
 * What is restated (reference file:line, all under /root/reference/proj):
 *   xxh64 / xxh64_key            core/include/hps/xxhash64.hpp:60-124
 *   placement seeds              core/include/hps/xxhash64.hpp:127-129
 *   slabset_of / first_slab_of   core/src/slab_cache.cpp:60-67
 *   partition_of                 core/src/volatile_store.cpp:10-13
 *   dedup_keys                   core/src/types.cpp:20-34
 *   cache query                  core/src/slab_cache.cpp:69-91,228-259
 *                                (model: tests/oracles/reference_cache.hpp:32-47)
 *   cache replace                core/src/slab_cache.cpp:93-107,261-326
 *                                (model: tests/oracles/reference_cache.hpp:49-105)
 *   cache update                 core/src/slab_cache.cpp:109-125,328-358
 *   dump order                   core/src/slab_cache.cpp:367-394
 *
 * The cache is a deliberately naive slot matrix: slot index
 * ((set * W) + slab) * 32 + j, an explicit occupied flag per slot and
 * straight-line probe loops. The occupancy masks reported by
 * orc_cache_state() are derived from the flags, so the product's mask
 * bookkeeping is checked rather than copied.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define P1 0x9E3779B185EBCA87ull
#define P2 0xC2B2AE3D27D4EB4Full
#define P3 0x165667B19E3779F9ull
#define P4 0x85EBCA77C2B2AE63ull
#define P5 0x27D4EB2F165667C5ull

#define SLABSET_SEED 0x5EED5E7ull
#define SLAB_SEED 0x51ABull
#define PARTITION_SEED 0ull

static uint64_t rotl(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

static uint64_t rd64(const unsigned char* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}
static uint32_t rd32(const unsigned char* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) |
         ((uint32_t)p[3] << 24);
}
static uint64_t round1(uint64_t acc, uint64_t lane) {
  return rotl(acc + lane * P2, 31) * P1;
}
static uint64_t merge(uint64_t h, uint64_t v) {
  h ^= round1(0, v);
  return h * P1 + P4;
}

/* Canonical XXH64 (xxhash64.hpp:60-114). */
uint64_t orc_xxh64(const void* input, size_t len, uint64_t seed) {
  const unsigned char* p = (const unsigned char*)input;
  const unsigned char* end = p + len;
  uint64_t h;
  if (len >= 32) {
    uint64_t v1 = seed + P1 + P2, v2 = seed + P2, v3 = seed, v4 = seed - P1;
    const unsigned char* limit = end - 32;
    do {
      v1 = round1(v1, rd64(p));
      v2 = round1(v2, rd64(p + 8));
      v3 = round1(v3, rd64(p + 16));
      v4 = round1(v4, rd64(p + 24));
      p += 32;
    } while (p <= limit);
    h = rotl(v1, 1) + rotl(v2, 7) + rotl(v3, 12) + rotl(v4, 18);
    h = merge(h, v1);
    h = merge(h, v2);
    h = merge(h, v3);
    h = merge(h, v4);
  } else {
    h = seed + P5;
  }
  h += (uint64_t)len;
  while (p + 8 <= end) {
    h ^= round1(0, rd64(p));
    h = rotl(h, 27) * P1 + P4;
    p += 8;
  }
  if (p + 4 <= end) {
    h ^= (uint64_t)rd32(p) * P1;
    h = rotl(h, 23) * P2 + P3;
    p += 4;
  }
  while (p < end) {
    h ^= (uint64_t)(*p) * P5;
    h = rotl(h, 11) * P1;
    ++p;
  }
  h ^= h >> 33;
  h *= P2;
  h ^= h >> 29;
  h *= P3;
  h ^= h >> 32;
  return h;
}

/* Keys hash as their 8-byte little-endian encoding (xxhash64.hpp:118-124). */
uint64_t orc_xxh64_key(uint64_t key, uint64_t seed) {
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = (unsigned char)(key >> (8 * i));
  return orc_xxh64(b, 8, seed);
}

uint64_t orc_slabset_of(uint64_t key, uint64_t slabset_count) {
  return orc_xxh64_key(key, SLABSET_SEED) % slabset_count;
}
uint32_t orc_first_slab_of(uint64_t key, uint32_t slabs_per_set) {
  return (uint32_t)(orc_xxh64_key(key, SLAB_SEED) % slabs_per_set);
}
uint32_t orc_partition_of(uint64_t key, uint32_t partition_count) {
  return (uint32_t)(orc_xxh64_key(key, PARTITION_SEED) % partition_count);
}

/* ---------------------------------------------------------------------- */
/* dedup_keys (types.cpp:20-34): unique keys in first-occurrence order and a
 * u32 inverse index. Open addressing keyed by the key itself; returns the
 * unique count. */
size_t orc_dedup(const uint64_t* keys, size_t n, uint64_t* unique_out,
                 uint32_t* inverse_out) {
  size_t cap = 16;
  while (cap < 2 * n) cap <<= 1;
  uint64_t* tk = (uint64_t*)malloc(cap * sizeof(uint64_t));
  uint32_t* tv = (uint32_t*)malloc(cap * sizeof(uint32_t));
  unsigned char* used = (unsigned char*)calloc(cap, 1);
  size_t nu = 0;
  for (size_t i = 0; i < n; ++i) {
    size_t h = (size_t)orc_xxh64_key(keys[i], 0x0DDull) & (cap - 1);
    while (used[h] && tk[h] != keys[i]) h = (h + 1) & (cap - 1);
    if (!used[h]) {
      used[h] = 1;
      tk[h] = keys[i];
      tv[h] = (uint32_t)nu;
      unique_out[nu++] = keys[i];
    }
    inverse_out[i] = tv[h];
  }
  free(tk);
  free(tv);
  free(used);
  return nu;
}

/* ---------------------------------------------------------------------- */
/* Slot-matrix cache model. */
typedef struct orc_cache {
  uint64_t S;
  uint32_t W;
  uint32_t d;
  uint64_t clock;
  size_t occupied;
  unsigned char* occ; /* per slot */
  uint64_t* key;
  uint64_t* counter;
  float* vec;
} orc_cache;

orc_cache* orc_cache_create(uint64_t S, uint32_t W, uint32_t d) {
  if (S == 0 || W == 0 || d == 0) return NULL;
  orc_cache* c = (orc_cache*)calloc(1, sizeof(orc_cache));
  size_t slots = (size_t)S * W * 32;
  c->S = S;
  c->W = W;
  c->d = d;
  c->occ = (unsigned char*)calloc(slots, 1);
  c->key = (uint64_t*)calloc(slots, sizeof(uint64_t));
  c->counter = (uint64_t*)calloc(slots, sizeof(uint64_t));
  c->vec = (float*)calloc(slots * d, sizeof(float));
  return c;
}

void orc_cache_destroy(orc_cache* c) {
  if (!c) return;
  free(c->occ);
  free(c->key);
  free(c->counter);
  free(c->vec);
  free(c);
}

uint64_t orc_cache_clock(const orc_cache* c) { return c->clock; }
size_t orc_cache_occupied(const orc_cache* c) { return c->occupied; }

/* Probe in slab order from first_slab_of, scanning every slot of a slab and
 * stopping at the first slab with a free slot (reference_cache.hpp:153-173).
 * Returns the global slot or -1. */
static int64_t probe(const orc_cache* c, uint64_t k) {
  uint64_t set = orc_slabset_of(k, c->S);
  uint32_t first = orc_first_slab_of(k, c->W);
  for (uint32_t step = 0; step < c->W; ++step) {
    uint32_t slab = (first + step) % c->W;
    size_t base = ((size_t)set * c->W + slab) * 32;
    int full = 1;
    for (uint32_t j = 0; j < 32; ++j) {
      if (c->occ[base + j] && c->key[base + j] == k) return (int64_t)(base + j);
      if (!c->occ[base + j]) full = 0;
    }
    if (!full) return -1;
  }
  return -1;
}

/* query: clock bumps once per call (slab_cache.cpp:73-74), hits copy the
 * row and take the stamp; miss rows stay untouched. hit[i] = 1 on hit. */
void orc_cache_query(orc_cache* c, const uint64_t* keys, size_t n, float* out,
                     unsigned char* hit) {
  c->clock += 1;
  for (size_t i = 0; i < n; ++i) {
    int64_t s = probe(c, keys[i]);
    hit[i] = 0;
    if (s >= 0) {
      memcpy(out + i * c->d, c->vec + (size_t)s * c->d, c->d * sizeof(float));
      c->counter[s] = c->clock;
      hit[i] = 1;
    }
  }
}

/* replace (slab_cache.cpp:93-107,261-326). Returns 1 and mutates nothing if
 * keys holds duplicates. Keys are applied in input order; the stamp is the
 * current clock (no increment). */
int orc_cache_replace(orc_cache* c, const uint64_t* keys, size_t n,
                      const float* vecs) {
  if (n > 1) {
    /* duplicate check before any mutation (slab_cache.cpp:95-101): one
     * open-addressing pass instead of all pairs (million-key preloads) */
    size_t cap = 16;
    while (cap < 2 * n) cap <<= 1;
    uint64_t* tk = (uint64_t*)malloc(cap * sizeof(uint64_t));
    unsigned char* used = (unsigned char*)calloc(cap, 1);
    int dup = 0;
    for (size_t i = 0; i < n && !dup; ++i) {
      size_t h = (size_t)orc_xxh64_key(keys[i], 0x0DDull) & (cap - 1);
      while (used[h] && tk[h] != keys[i]) h = (h + 1) & (cap - 1);
      if (used[h]) dup = 1;
      used[h] = 1;
      tk[h] = keys[i];
    }
    free(tk);
    free(used);
    if (dup) return 1;
  }
  const size_t per_set = (size_t)c->W * 32;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t k = keys[i];
    const float* row = vecs + i * c->d;
    const uint64_t set = orc_slabset_of(k, c->S);
    const uint32_t first = orc_first_slab_of(k, c->W);
    int64_t found = -1, free_slot = -1;
    for (uint32_t step = 0; step < c->W && found < 0; ++step) {
      uint32_t slab = (first + step) % c->W;
      size_t base = ((size_t)set * c->W + slab) * 32;
      int64_t lowest_free = -1;
      for (uint32_t j = 0; j < 32; ++j) {
        if (c->occ[base + j] && c->key[base + j] == k) {
          found = (int64_t)(base + j);
          break;
        }
        if (!c->occ[base + j] && lowest_free < 0) lowest_free = (int64_t)(base + j);
      }
      if (found < 0 && lowest_free >= 0) {
        free_slot = lowest_free;
        break;
      }
    }
    if (found >= 0) {
      c->counter[found] = c->clock; /* resident: recency only */
      continue;
    }
    size_t s;
    if (free_slot >= 0) {
      s = (size_t)free_slot;
      c->occ[s] = 1;
      c->occupied += 1;
    } else {
      /* evict the smallest counter, ties to the lowest (slab, slot) */
      size_t base = (size_t)set * per_set;
      s = base;
      for (size_t j = 1; j < per_set; ++j)
        if (c->counter[base + j] < c->counter[s]) s = base + j;
    }
    c->key[s] = k;
    c->counter[s] = c->clock;
    memcpy(c->vec + s * c->d, row, c->d * sizeof(float));
  }
  return 0;
}

/* update (slab_cache.cpp:109-125,328-358): overwrite resident rows, count
 * every position written (duplicates twice), last occurrence wins. */
size_t orc_cache_update(orc_cache* c, const uint64_t* keys, size_t n,
                        const float* vecs) {
  size_t written = 0;
  for (size_t i = 0; i < n; ++i) {
    int64_t s = probe(c, keys[i]);
    if (s >= 0) {
      memcpy(c->vec + (size_t)s * c->d, vecs + i * c->d, c->d * sizeof(float));
      ++written;
    }
  }
  return written;
}

/* Resident keys of sets [set_begin, set_end) in set, slab, slot order
 * (slab_cache.cpp:367-394). Returns the count (writes at most cap). */
size_t orc_cache_dump(const orc_cache* c, uint64_t set_begin, uint64_t set_end,
                      uint64_t* out, size_t cap) {
  size_t n = 0;
  for (uint64_t set = set_begin; set < set_end && set < c->S; ++set) {
    size_t base = (size_t)set * c->W * 32;
    for (size_t j = 0; j < (size_t)c->W * 32; ++j) {
      if (c->occ[base + j]) {
        if (n < cap) out[n] = c->key[base + j];
        ++n;
      }
    }
  }
  return n;
}

/* Full state export for slot-for-slot comparison with the device table.
 * Unoccupied slots report key 0 / counter 0 / zero rows only if they were
 * never written; callers compare occupied slots. Masks are derived from the
 * per-slot flags. Any pointer may be NULL. */
void orc_cache_state(const orc_cache* c, uint64_t* keys, uint64_t* counters,
                     uint32_t* masks, float* rows) {
  size_t slots = (size_t)c->S * c->W * 32;
  if (keys) memcpy(keys, c->key, slots * sizeof(uint64_t));
  if (counters) memcpy(counters, c->counter, slots * sizeof(uint64_t));
  if (rows) memcpy(rows, c->vec, slots * c->d * sizeof(float));
  if (masks) {
    for (size_t slab = 0; slab < (size_t)c->S * c->W; ++slab) {
      uint32_t m = 0;
      for (uint32_t j = 0; j < 32; ++j)
        if (c->occ[slab * 32 + j]) m |= (1u << j);
      masks[slab] = m;
    }
  }
}

/* ---------------------------------------------------------------------- */
/* Power-law workload restatement (workload.cpp:18-20,24-70): inverse-CDF
 * over r^-alpha and an mt19937_64 Fisher-Yates rank->key permutation. Used
 * only to pin the product's own sampler. */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
               (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  static const uint64_t mag[2] = {0ull, 0xB5026F5AA96619E9ull};
  if (g->idx >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[i + 1] & 0x7FFFFFFFull);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ mag[(int)(x & 1ull)];
    }
    for (; i < 311; ++i) {
      x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[i + 1] & 0x7FFFFFFFull);
      g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[(int)(x & 1ull)];
    }
    x = (g->mt[311] & 0xFFFFFFFF80000000ull) | (g->mt[0] & 0x7FFFFFFFull);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ mag[(int)(x & 1ull)];
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= (x >> 43);
  return x;
}

uint64_t orc_mt64_first(uint64_t seed, size_t skip) {
  mt64 g;
  mt64_seed(&g, seed);
  for (size_t i = 0; i < skip; ++i) mt64_next(&g);
  return mt64_next(&g);
}

#include <math.h>

/* sample `count` keys; returns 0 on success. */
int orc_powerlaw_sample(double alpha, uint64_t keyspace, uint64_t permute_seed,
                        uint64_t draw_seed, size_t count, uint64_t* out) {
  if (keyspace == 0 || !(alpha > 0.0)) return 1;
  double* cdf = (double*)malloc(keyspace * sizeof(double));
  uint64_t* r2k = (uint64_t*)malloc(keyspace * sizeof(uint64_t));
  if (!cdf || !r2k) {
    free(cdf);
    free(r2k);
    return 2;
  }
  double running = 0.0;
  for (uint64_t r = 1; r <= keyspace; ++r) {
    running += pow((double)r, -alpha);
    cdf[r - 1] = running;
  }
  for (uint64_t r = 0; r < keyspace; ++r) cdf[r] /= running;
  cdf[keyspace - 1] = 1.0;
  for (uint64_t i = 0; i < keyspace; ++i) r2k[i] = i;
  mt64 g;
  mt64_seed(&g, permute_seed);
  for (uint64_t i = keyspace - 1; i > 0; --i) {
    uint64_t j = mt64_next(&g) % (i + 1);
    uint64_t t = r2k[i];
    r2k[i] = r2k[j];
    r2k[j] = t;
  }
  mt64_seed(&g, draw_seed);
  for (size_t i = 0; i < count; ++i) {
    double u = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
    /* upper_bound: first index with cdf > u */
    uint64_t lo = 0, hi = keyspace;
    while (lo < hi) {
      uint64_t mid = lo + (hi - lo) / 2;
      if (cdf[mid] > u)
        hi = mid;
      else
        lo = mid + 1;
    }
    uint64_t rank = lo + 1;
    if (rank > keyspace) rank = keyspace;
    out[i] = r2k[rank - 1];
  }
  free(cdf);
  free(r2k);
  return 0;
}
