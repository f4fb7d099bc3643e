// lookup_kernels.cu -- the fused lookup hot path (sm_100a).
//
// Restates LookupEngine::lookup (lookup_engine.cpp:130-241) for a batch of
// |Q| query positions without materialising the dedup step for hits:
//
//   K1 lookup_probe   one warp per P positions: placement hash, ballot probe
//                     of 32-key slabs, 128-bit gather of the hit row straight
//                     into the position's output row (the expansion of
//                     lookup_engine.cpp:194-203 is fused), recency stamp via
//                     atomicExch -- the exchange that first moves a slot to
//                     this call's stamp counts one UNIQUE hit, so |Q*| needs
//                     no dedup of hits. Missing positions get the default row
//                     (the async branch's answer) and are deduplicated in a
//                     per-call hash table keeping the first occurrence.
//   K2 lookup_compact ordered single-pass compaction of the first occurrences
//                     of missing keys -> the unique miss list in
//                     first-occurrence order (= reference order of
//                     CacheMiss after dedup, slab_cache.cpp:84-89), plus the
//                     rank of every miss-table entry.
//   K3 lookup_scatter (sync branch only) copies the rows fetched from the
//                     tiers into every position of their key, clearing the
//                     default flag (lookup_engine.cpp:165-181).
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "common.cuh"
#include "kernels.hpp"
#include "probe.cuh"

namespace hpsb {

namespace {
inline void check_launch(const char* what, uint32_t kernels) {
  note_launches(kernels);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
  }
}
constexpr int kLookupWarps = 8;
}  // namespace

__device__ __forceinline__ float4 ld_nc_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_cs_f4(float4* p, const float4& v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

template <int P>
__global__ void __launch_bounds__(kLookupWarps * 32)
    k_lookup_probe(CacheDev c, const uint64_t* __restrict__ keys, uint64_t n,
                   float* __restrict__ out, uint8_t* __restrict__ flags,
                   const float* __restrict__ default_row, uint64_t stamp, LookupScratch ls,
                   uint32_t epoch) {
  __shared__ unsigned int s_counts[2];
  if (threadIdx.x < 2) s_counts[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t warp = (uint64_t(blockIdx.x) * kLookupWarps) + (threadIdx.x >> 5);
  const uint64_t base = warp * P;
  const uint32_t lane = lane_id();
  uint32_t uh = 0, um = 0;
  if (base < n) {
    WarpKeys<P> wk;
    warp_load_keys<P>(c, keys, base, n, wk);
    int64_t slot[P];
    warp_probe<P>(c, wk, slot);
    const uint32_t d = c.d;
    if ((d & 3u) == 0) {
      // 128-bit path: the first 32 float4 chunks of every row are loaded for
      // all P positions before any store so P row reads are in flight.
      const uint32_t d4 = d >> 2;
      float4 v[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (wk.valid[p] && lane < d4) {
          const float* src = slot[p] >= 0 ? c.rows + uint64_t(slot[p]) * d : default_row;
          v[p] = ld_nc_f4(reinterpret_cast<const float4*>(src) + lane);
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (wk.valid[p] && lane < d4)
          st_cs_f4(reinterpret_cast<float4*>(out + (base + p) * d) + lane, v[p]);
      }
      for (uint32_t ch = lane + 32; ch < d4; ch += 32) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
          if (!wk.valid[p]) continue;
          const float* src = slot[p] >= 0 ? c.rows + uint64_t(slot[p]) * d : default_row;
          st_cs_f4(reinterpret_cast<float4*>(out + (base + p) * d) + ch,
                   ld_nc_f4(reinterpret_cast<const float4*>(src) + ch));
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < P; ++p) {
        if (!wk.valid[p]) continue;
        const float* src = slot[p] >= 0 ? c.rows + uint64_t(slot[p]) * d : default_row;
        for (uint32_t ch = lane; ch < d; ch += 32) out[(base + p) * d + ch] = src[ch];
      }
    }
    // bookkeeping: lane p owns position base + p
    if (lane < uint32_t(P)) {
      int64_t my_slot = -1;
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (uint32_t(p) == lane) my_slot = slot[p];
      const uint64_t i = base + lane;
      if (i < n) {
        if (my_slot >= 0) {
          const unsigned long long old = atomicExch(
              reinterpret_cast<unsigned long long*>(c.counters + my_slot), stamp);
          uh += (old != stamp) ? 1u : 0u;
          flags[i] = 0;
        } else {
          bool claimed;
          ls.miss_slot[i] =
              dedup_insert(ls.miss_table, ls.cap, keys, keys[i], uint32_t(i), epoch, &claimed);
          um += claimed ? 1u : 0u;
          flags[i] = 1;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uh += __shfl_xor_sync(0xFFFFFFFFu, uh, o);
    um += __shfl_xor_sync(0xFFFFFFFFu, um, o);
  }
  if (lane == 0 && (uh | um)) {
    atomicAdd(&s_counts[0], uh);
    atomicAdd(&s_counts[1], um);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_counts[0]) atomicAdd(ls.counts + 0, (unsigned long long)s_counts[0]);
    if (s_counts[1]) atomicAdd(ls.counts + 1, (unsigned long long)s_counts[1]);
  }
}

void launch_lookup_probe(const CacheDev& c, const uint64_t* keys, uint64_t n, float* out,
                         uint8_t* flags, const float* default_row, uint64_t stamp,
                         const LookupScratch& ls, uint32_t table_epoch, cudaStream_t st) {
  if (n == 0) return;
  constexpr int P = 4;
  const uint64_t warps = (n + P - 1) / P;
  const unsigned grid = unsigned((warps + kLookupWarps - 1) / kLookupWarps);
  k_lookup_probe<P><<<grid, kLookupWarps * 32, 0, st>>>(c, keys, n, out, flags, default_row,
                                                        stamp, ls, table_epoch);
  check_launch("lookup_probe", 1);
}

__global__ void __launch_bounds__(kScanBlock)
    k_lookup_compact(const uint64_t* __restrict__ keys, uint64_t n,
                     const uint8_t* __restrict__ flags, LookupScratch ls, ScanState scan) {
  if (ls.counts_out != nullptr && blockIdx.x == 0 && threadIdx.x < 2) {
    // K1 has fully completed (stream order): publish this call's counts
    const unsigned long long cum = ls.counts[threadIdx.x];
    ls.counts_out[threadIdx.x] = cum - ls.counts_prev[threadIdx.x];
    ls.counts_prev[threadIdx.x] = cum;
  }
  select_tile(
      n, scan,
      [&](uint64_t i) {
        return flags[i] != 0 && uint32_t(ls.miss_table[ls.miss_slot[i]]) == uint32_t(i);
      },
      [&](uint64_t i, uint64_t r) {
        ls.miss_keys[r] = keys[i];
        ls.rank_of_slot[ls.miss_slot[i]] = uint32_t(r);
      },
      nullptr);
}

void launch_lookup_compact(const uint64_t* keys, uint64_t n, const uint8_t* flags,
                           const LookupScratch& ls, uint32_t table_epoch, ScanState& scan,
                           cudaStream_t st) {
  (void)table_epoch;
  if (n == 0) return;
  const uint64_t tiles = (n + kScanTile - 1) / kScanTile;
  scan_begin(scan, tiles, st);
  k_lookup_compact<<<unsigned(tiles), kScanBlock, 0, st>>>(keys, n, flags, ls, scan);
  scan.tile_base += tiles;
  check_launch("lookup_compact", 1);
}

__global__ void __launch_bounds__(256)
    k_lookup_scatter(uint64_t n, uint32_t d, uint8_t* __restrict__ flags, LookupScratch ls,
                     const int32_t* __restrict__ row_of, const float* __restrict__ staged,
                     float* __restrict__ out) {
  const uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  if (flags[i] == 0) return;
  const uint32_t u = ls.rank_of_slot[ls.miss_slot[i]];
  const int32_t r = row_of[u];
  if (r < 0) return;  // absent from every tier: keep default + flag
  warp_copy_row(staged + uint64_t(r) * d, out + i * d, d);
  __syncwarp();
  if (lane_id() == 0) flags[i] = 0;
}

void launch_lookup_scatter(uint64_t n, uint32_t d, const uint8_t* flags_in, uint8_t* flags,
                           const LookupScratch& ls, const int32_t* row_of,
                           const float* staged, float* out, cudaStream_t st) {
  (void)flags_in;
  if (n == 0) return;
  const uint64_t threads = n * 32;
  k_lookup_scatter<<<unsigned((threads + 255) / 256), 256, 0, st>>>(n, d, flags, ls, row_of,
                                                                    staged, out);
  check_launch("lookup_scatter", 1);
}

}  // namespace hpsb
