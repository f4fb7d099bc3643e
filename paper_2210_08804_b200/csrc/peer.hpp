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
  unsigned long long* inbox_count;  // inbox: [count | keys...]
  uint64_t* inbox_keys;
  uint64_t inbox_cap;
};

// Kernel launcher (shard_kernels.cu).
void launch_peer_lookup(const PeerShard* d_shards, uint32_t world, const uint64_t* keys,
                        uint64_t n, float* out, uint8_t* flags, const float* default_row,
                        uint32_t d, uint64_t stamp, cudaStream_t st);

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
};

}  // namespace hpsb
