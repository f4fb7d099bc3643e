// peer.hpp -- the key-hash-sharded lookup over PEER MEMORY (the
// B200-native alternative to the two all-to-alls): every rank maps the other
// ranks' shard caches into its address space (CUDA IPC handles; on an
// NVLink / NVSwitch node the loads, stores and atomics below travel over
// NVLink) and ONE kernel per call routes each key to its owner, probes the
// owner's slabs, stamps the owner's counter, copies the owner's row straight
// into the local output, and appends a missing key to the owner's miss inbox.
// No collective, no staging, no host synchronisation on the data path; the
// owners admit their inboxes' keys between lookup phases (PeerGroup users
// run a barrier around the fill, see paper_2210_08804_b200/sharded.py).
// Recency: while a shard is peer-mapped its clock lives in device memory
// next to its inbox; every lookup call ticks each owner's clock once
// (slab_cache.cpp:73-74: one tick per query) and stamps that owner's hits
// with it, and the owner's replace stamps with the same clock (it is read
// back at the drain), so the LRU order is the reference's per shard.
// No reference counterpart: the reference is single-process and the paper
// deploys one replica per GPU.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace hpsb {

class DeviceCache;

constexpr uint32_t kMaxPeers = 64;

// What a peer needs to map one rank's shard (plain bytes: it crosses
// process boundaries through the caller's transport).
struct PeerBlob {
  uint64_t magic = 0;
  uint64_t S = 0;
  uint32_t W = 0, d = 0;
  uint64_t tags_off = 0, masks_off = 0, ctr_off = 0;  // within the probe allocation
  uint64_t inbox_cap = 0;
  int device = 0, reserved = 0;
  cudaIpcMemHandle_t probe, rows, inbox;
};
constexpr uint64_t kPeerBlobMagic = 0x48505342504545ull;  // "HPSBPEE"

// One shard as the lookup kernel sees it.
struct PeerShard {
  CacheDev c;
  unsigned long long* inbox_count;  // inbox: [count | clock | pad | keys...]
  unsigned long long* clock;        // the shard's recency clock while peer-mapped
  uint64_t* inbox_keys;
  uint64_t inbox_cap;
};

// Kernel launcher (shard_kernels.cu).
// (two launches: each owner's clock ticks once for the call -- the stamps --
// then the lookup)
void launch_peer_lookup(const PeerShard* d_shards, uint32_t world, const uint64_t* keys,
                        uint64_t n, float* out, uint8_t* flags, const float* default_row,
                        uint32_t d, unsigned long long* d_stamps, cudaStream_t st);

class PeerGroup {
 public:
  // self: this rank's shard cache (exported already); blobs[r] of every rank
  PeerGroup(DeviceCache& self, uint32_t rank, const std::vector<PeerBlob>& blobs);
  ~PeerGroup();
  PeerGroup(const PeerGroup&) = delete;
  PeerGroup& operator=(const PeerGroup&) = delete;
  // the sharded lookup on device pointers, ordered after `user` (and the
  // cache stream after it): rows of every position (owner's row on a hit,
  // default_row on a miss) and miss flags
  void lookup(const uint64_t* keys, size_t n, float* out, uint8_t* flags,
              const float* default_row, cudaStream_t user);
  uint32_t world() const { return world_; }
  uint32_t rank() const { return rank_; }

 private:
  DeviceCache& self_;
  uint32_t rank_, world_;
  std::vector<void*> opened_;
  PeerShard* d_shards_ = nullptr;
  unsigned long long* d_stamps_ = nullptr;  // this call's stamp per owner
};

}  // namespace hpsb
