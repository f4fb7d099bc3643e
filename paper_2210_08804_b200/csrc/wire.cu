// wire.cu -- LOOKUP response frames straight from the lookup's output
// (reference: encode_response_frame, wire.cpp:174-188,
// used by handle_frame, server.cpp:284-294; layout in wire.hpp:18-21):
//
//   [u32 body_len][u8 status = 0][u32 count][u32 dim][count*dim f32]
//   [ceil(count/8) bytes: bit i (byte i/8, bit i%8) = row i is a default]
//
// all little-endian. Device mode: the miss bitmap is packed on the GPU (one
// ballot per 32 flags) and the rows and bitmap are copied from HBM straight
// into the caller's (pinned) frame buffer, at their unaligned frame offsets,
// by the copy engine; the host writes only the 13-byte header.
#include <cuda_runtime.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "kernels.hpp"

namespace hpsb {

namespace {
inline void check_launch(const char* what, uint32_t kernels) {
  note_launches(kernels);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
inline void put_le32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = uint8_t(v >> (8 * i));
}
}  // namespace

// bitmap[i / 8] bit (i % 8) = flags[i] != 0; one warp per 32 flags = 4 bytes
__global__ void __launch_bounds__(256)
    k_pack_bitmap(const uint8_t* __restrict__ flags, uint64_t n, uint8_t* __restrict__ bitmap) {
  const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t b = __ballot_sync(0xFFFFFFFFu, i < n && flags[i] != 0);
  const uint64_t byte0 = (i & ~31ull) / 8;
  const uint32_t lane = lane_id();
  if (lane < 4 && byte0 + lane < (n + 7) / 8) bitmap[byte0 + lane] = uint8_t(b >> (8 * lane));
}

size_t wire_lookup_frame_bytes(uint64_t count, uint32_t dim) {
  return 13 + count * uint64_t(dim) * 4 + (count + 7) / 8;
}

void wire_encode_lookup_host(const float* rows, const uint8_t* flags, uint32_t count, uint32_t dim,
                             uint8_t* frame) {
  const uint64_t body = wire_lookup_frame_bytes(count, dim) - 4;
  put_le32(frame, uint32_t(body));
  frame[4] = 0;  // Status::Ok
  put_le32(frame + 5, count);
  put_le32(frame + 9, dim);
  std::memcpy(frame + 13, rows, uint64_t(count) * dim * 4);  // f32 LE == host order (x86/arm LE)
  uint8_t* bm = frame + 13 + uint64_t(count) * dim * 4;
  std::memset(bm, 0, (uint64_t(count) + 7) / 8);
  for (uint32_t i = 0; i < count; ++i)
    if (flags[i]) bm[i / 8] |= uint8_t(1u << (i % 8));
}

void wire_encode_lookup_device(const float* d_rows, const uint8_t* d_flags, uint32_t count,
                               uint32_t dim, uint8_t* d_bitmap_scratch, uint8_t* frame,
                               cudaStream_t st) {
  const uint64_t body = wire_lookup_frame_bytes(count, dim) - 4;
  put_le32(frame, uint32_t(body));
  frame[4] = 0;
  put_le32(frame + 5, count);
  put_le32(frame + 9, dim);
  const uint64_t row_bytes = uint64_t(count) * dim * 4;
  if (count == 0) return;
  k_pack_bitmap<<<unsigned((count + 255) / 256), 256, 0, st>>>(d_flags, count, d_bitmap_scratch);
  check_launch("pack_bitmap", 1);
  cudaError_t e = cudaMemcpyAsync(frame + 13, d_rows, row_bytes, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(frame + 13 + row_bytes, d_bitmap_scratch, (uint64_t(count) + 7) / 8,
                        cudaMemcpyDeviceToHost, st);
  if (e != cudaSuccess) throw std::runtime_error(std::string("wire frame copy: ") + cudaGetErrorString(e));
}

}  // namespace hpsb
