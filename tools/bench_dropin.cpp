// bench_dropin.cpp -- the e2e lookup measured through the DROP-IN C++ API:
// hps::LookupEngine::lookup (include/hps/lookup_engine.hpp), which returns the
// reference's LookupResult (std::vector rows / flags, i.e. PAGEABLE memory,
// reference lookup_engine.hpp:161-162), over the drop-in hps::SlabCache and
// hps::VolatileStore, with the reference's own PersistentStore as the cold
// tier -- exactly what a reference build gets after the INTEGRATION.md swap.
//
// bench.py writes the workload (its calibrated cfg-2 batches) to files and
// runs this binary:
//   bench_dropin_b200 <dir> <S> <W> <dim> <batch> <steps> <warmup> <threshold>
// <dir>/preload.u64 -- keys replaced into the cache first (the bench preload)
// <dir>/vdb.u64     -- keys held by the volatile tier (the batches' misses)
// <dir>/batches.u64 -- K batches of <batch> keys, used round robin
// Rows are hash-derived (bench.py table_rows); after the timed region a few
// calls' rows are checked against them. Prints one JSON object.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <string>
#include <vector>

#include "hps/lookup_engine.hpp"
#include "hps/persistent_store.hpp"
#include "hps/slab_cache.hpp"
#include "hps/volatile_store.hpp"

namespace {

std::vector<std::uint64_t> read_u64(const std::filesystem::path& p) {
  std::ifstream f(p, std::ios::binary);
  f.seekg(0, std::ios::end);
  const auto bytes = static_cast<std::size_t>(f.tellg());
  f.seekg(0);
  std::vector<std::uint64_t> v(bytes / 8);
  f.read(reinterpret_cast<char*>(v.data()), std::streamsize(v.size() * 8));
  return v;
}

// bench.py table_rows
void rows_of(const std::uint64_t* keys, std::size_t n, std::uint32_t d, float* out) {
  for (std::size_t i = 0; i < n; ++i) {
    const std::uint64_t k = keys[i] * 0x9E3779B1ull;
    for (std::uint32_t c = 0; c < d; ++c) {
      const std::uint64_t v = (k + std::uint64_t(c) * 0x85EBCA77ull) & 0xFFFFFFull;
      out[i * d + c] = float(v) / 8388608.0f - 1.0f;
    }
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 9) {
    std::fprintf(stderr, "usage: %s dir S W dim batch steps warmup threshold\n", argv[0]);
    return 2;
  }
  const std::filesystem::path dir = argv[1];
  const std::size_t S = std::strtoull(argv[2], nullptr, 10);
  const std::uint32_t W = std::uint32_t(std::strtoul(argv[3], nullptr, 10));
  const std::uint32_t d = std::uint32_t(std::strtoul(argv[4], nullptr, 10));
  const std::size_t batch = std::strtoull(argv[5], nullptr, 10);
  const int steps = std::atoi(argv[6]);
  const int warmup = std::atoi(argv[7]);
  const double threshold = std::atof(argv[8]);

  const auto preload = read_u64(dir / "preload.u64");
  const auto vdb_keys = read_u64(dir / "vdb.u64");
  const auto all = read_u64(dir / "batches.u64");
  const std::size_t K = all.size() / batch;

  hps::SlabCache cache(hps::SlabCacheConfig{S, W, d, 1, 8});
  {
    std::vector<float> rows(batch * d);
    for (std::size_t i = 0; i < preload.size(); i += batch) {
      const std::size_t m = std::min(batch, preload.size() - i);
      rows_of(preload.data() + i, m, d, rows.data());
      cache.replace(std::span(preload.data() + i, m), std::span(rows.data(), m * d));
    }
  }
  const hps::TableId table{"bench", d};
  hps::VolatileStore vdb;
  vdb.register_table(table, hps::VolatileTableConfig{16, std::size_t(1) << 40});
  {
    std::vector<float> rows(262144ull * d);
    for (std::size_t i = 0; i < vdb_keys.size(); i += 262144) {
      const std::size_t m = std::min<std::size_t>(262144, vdb_keys.size() - i);
      rows_of(vdb_keys.data() + i, m, d, rows.data());
      vdb.insert(table.name, std::span(vdb_keys.data() + i, m), std::span(rows.data(), m * d));
    }
  }
  const auto pdb_dir = std::filesystem::temp_directory_path() / "hps_bench_dropin_pdb";
  std::filesystem::remove_all(pdb_dir);
  std::size_t checked = 0, bad = 0;
  double mean_h = 0.0;
  std::vector<double> lat;
  double el = 0.0;
  std::uint64_t sync_b = 0, async_b = 0;
  {
    hps::PersistentStore pdb(pdb_dir);
    pdb.create_table(table);
    hps::EngineConfig ec;
    ec.hit_rate_threshold = threshold;
    hps::LookupEngine eng(table, cache, &vdb, pdb, ec);
    eng.reserve(batch);  // serving setup (B200 extension)
    for (int s = 0; s < warmup; ++s)
      (void)eng.lookup(std::span(all.data() + (s % K) * batch, batch));
    eng.drain_async();
    const auto st0 = eng.stats();
    std::vector<float> want(batch * d);
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < steps; ++s) {
      const std::uint64_t* q = all.data() + (s % K) * batch;
      hps::LookupOutcome o;
      const auto c0 = std::chrono::steady_clock::now();
      hps::LookupResult r = eng.lookup(std::span(q, batch), &o);
      const auto c1 = std::chrono::steady_clock::now();
      lat.push_back(std::chrono::duration<double, std::micro>(c1 - c0).count());
      mean_h += o.unique_hit_rate / steps;
    }
    eng.drain_async();
    el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const auto st1 = eng.stats();
    sync_b = st1.sync_batches - st0.sync_batches;
    async_b = st1.async_batches - st0.async_batches;
    // rows check, after the timed region: unflagged rows are the stored rows
    for (std::size_t b = 0; b < std::min<std::size_t>(K, 4); ++b) {
      const std::uint64_t* q = all.data() + b * batch;
      hps::LookupResult r = eng.lookup(std::span(q, batch));
      rows_of(q, batch, d, want.data());
      for (std::size_t i = 0; i < batch; i += 7) {
        ++checked;
        if (r.miss_flags[i]) continue;  // default row (async branch miss)
        if (std::memcmp(&r.vectors[i * d], &want[i * d], d * 4) != 0) ++bad;
      }
    }
  }
  std::filesystem::remove_all(pdb_dir);
  std::vector<double> sl = lat;
  std::sort(sl.begin(), sl.end());
  auto pct = [&](double p) { return sl[std::min(sl.size() - 1, std::size_t(p * sl.size()))]; };
  std::printf(
      "{\"value\": %.1f, \"unit\": \"keys/s\", \"ms_per_step\": %.4f, \"p50_call_us\": %.1f, "
      "\"p99_call_us\": %.1f, \"mean_unique_hit_rate\": %.4f, \"sync_batches\": %llu, "
      "\"async_batches\": %llu, \"rows_checked\": %zu, \"rows_bad\": %zu, "
      "\"h2d_bytes_per_step\": %zu, \"d2h_bytes_per_step\": %zu, "
      "\"api\": \"hps::LookupEngine::lookup (include/hps/lookup_engine.hpp) -> LookupResult "
      "std::vector (pageable), drop-in SlabCache + VolatileStore, reference PersistentStore\"}\n",
      double(steps) * double(batch) / el, el * 1e3 / steps, pct(0.5), pct(0.99), mean_h,
      (unsigned long long)sync_b, (unsigned long long)async_b, checked, bad, batch * 8,
      batch * d * 4 + batch);
  return bad == 0 ? 0 : 1;
}
