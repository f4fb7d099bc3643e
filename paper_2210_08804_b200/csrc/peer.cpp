// peer.cpp -- see peer.hpp.
#include "peer.hpp"

#include <stdexcept>
#include <string>

#include "device_cache.hpp"
#include "runtime.hpp"

namespace hpsb {

PeerGroup::PeerGroup(DeviceCache& self, uint32_t rank, const std::vector<PeerBlob>& blobs)
    : self_(self), rank_(rank), world_(uint32_t(blobs.size())) {
  if (world_ == 0 || world_ > kMaxPeers) throw invalid_argument("peer group size out of range");
  if (rank_ >= world_) throw invalid_argument("peer rank out of range");
  DeviceGuard g(self.device());
  std::vector<PeerShard> shards(world_);
  try {
    for (uint32_t r = 0; r < world_; ++r) {
      const PeerBlob& b = blobs[r];
      if (b.magic != kPeerBlobMagic) throw invalid_argument("not a peer export blob");
      if (b.d != self.dimension())
        throw invalid_argument("peer shards must have the same dimension");
      PeerShard& s = shards[r];
      if (r == rank_) {
        s.c = self.dev();
        self.peer_inbox(&s.inbox_count, &s.inbox_keys, &s.inbox_cap);
        s.clock = s.inbox_count + 1;
        continue;
      }
      void *probe = nullptr, *rows = nullptr, *inbox = nullptr;
      HPSB_CUDA(cudaIpcOpenMemHandle(&probe, b.probe, cudaIpcMemLazyEnablePeerAccess));
      opened_.push_back(probe);
      HPSB_CUDA(cudaIpcOpenMemHandle(&rows, b.rows, cudaIpcMemLazyEnablePeerAccess));
      opened_.push_back(rows);
      HPSB_CUDA(cudaIpcOpenMemHandle(&inbox, b.inbox, cudaIpcMemLazyEnablePeerAccess));
      opened_.push_back(inbox);
      char* pm = static_cast<char*>(probe);
      CacheDev c{};
      c.keys = reinterpret_cast<uint64_t*>(pm);
      c.tags = reinterpret_cast<uint8_t*>(pm + b.tags_off);
      c.masks = reinterpret_cast<uint32_t*>(pm + b.masks_off);
      c.counters = reinterpret_cast<uint64_t*>(pm + b.ctr_off);
      c.rows = static_cast<float*>(rows);
      c.occupied = nullptr;  // a peer never admits into this shard
      c.S = b.S;
      c.W = b.W;
      c.d = b.d;
      c.mS = ~0ull / b.S;
      c.mW = ~0ull / b.W;
      s.c = c;
      s.inbox_count = static_cast<unsigned long long*>(inbox);
      s.clock = s.inbox_count + 1;
      s.inbox_keys = reinterpret_cast<uint64_t*>(static_cast<char*>(inbox) + 256);
      s.inbox_cap = b.inbox_cap;
    }
    HPSB_CUDA(cudaMalloc(&d_shards_, world_ * sizeof(PeerShard)));
    HPSB_CUDA(cudaMalloc(&d_stamps_, world_ * 8));
    HPSB_CUDA(cudaMemcpy(d_shards_, shards.data(), world_ * sizeof(PeerShard),
                         cudaMemcpyHostToDevice));
  } catch (...) {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    opened_.clear();
    throw;
  }
}

PeerGroup::~PeerGroup() {
  DeviceGuard g(self_.device());
  cudaDeviceSynchronize();
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  cudaFree(d_shards_);
  cudaFree(d_stamps_);
}

void PeerGroup::lookup(const uint64_t* keys, size_t n, float* out, uint8_t* flags,
                       const float* default_row, cudaStream_t user) {
  std::lock_guard<std::mutex> lk(self_.mutex());
  DeviceGuard g(self_.device());
  // recency: each owner's device clock ticks once for this call (peer.hpp)
  self_.note_stream_op();
  self_.join_from(user);
  launch_peer_lookup(d_shards_, world_, keys, n, out, flags, default_row, self_.dimension(),
                     d_stamps_, self_.stream());
  self_.join_to(user);
}

}  // namespace hpsb
