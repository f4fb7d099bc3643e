// workload.cpp -- synthetic power-law key streams: HARNESS INPUT for the
// bench and the tests (tools/libhps_workload.so), not part of the product
// library.
//
// Bit-exact restatement of PowerLawSampler (workload.cpp:18-20, 24-70 of the
// reference; SURVEY.md §2 marks the sampler "reused verbatim" so the streams
// match the reference's bit for bit): inverse CDF over r^-alpha (running sum
// of std::pow, normalised, last entry forced to 1.0), mt19937_64
// Fisher-Yates rank -> key permutation (`gen() % (i + 1)`), uniform = top 53
// bits * 2^-53, upper_bound search. Serial, O(keyspace + count log keyspace).
#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <random>
#include <vector>

extern "C" int hps_powerlaw_sample(double alpha, uint64_t keyspace, uint64_t permute_seed,
                                   uint64_t draw_seed, size_t count, uint64_t* out) {
  if (keyspace == 0 || !(alpha > 0.0) || (count > 0 && out == nullptr)) return 1;
  std::vector<double> cdf(keyspace);
  double running = 0.0;
  for (uint64_t r = 1; r <= keyspace; ++r) {
    running += std::pow(static_cast<double>(r), -alpha);
    cdf[r - 1] = running;
  }
  for (double& c : cdf) c /= running;
  cdf.back() = 1.0;
  std::vector<uint64_t> rank_to_key(keyspace);
  for (uint64_t i = 0; i < keyspace; ++i) rank_to_key[i] = i;
  std::mt19937_64 perm(permute_seed);
  for (uint64_t i = keyspace - 1; i > 0; --i) {
    const uint64_t j = perm() % (i + 1);
    std::swap(rank_to_key[i], rank_to_key[j]);
  }
  std::mt19937_64 gen(draw_seed);
  for (size_t i = 0; i < count; ++i) {
    const double u = static_cast<double>(gen() >> 11) * 0x1.0p-53;
    const auto it = std::upper_bound(cdf.begin(), cdf.end(), u);
    uint64_t rank = static_cast<uint64_t>(it - cdf.begin()) + 1;
    rank = std::min(rank, keyspace);
    out[i] = rank_to_key[rank - 1];
  }
  return 0;
}
