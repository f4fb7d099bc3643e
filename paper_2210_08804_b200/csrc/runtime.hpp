// runtime.hpp -- host runtime pieces shared by the cache, the VDB and the
// engine: error types (mapped 1:1 onto the C ABI status codes), grow-only
// device / pinned buffers, a small fixed thread pool.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace hpsb {

// Status codes of include/hps_b200.h.
enum Status : int {
  kOk = 0,
  kInvalidArgument = 1,
  kInternal = 2,
  kOutOfMemory = 3,
  kLogicError = 4,
  kTierFault = 5,
};

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

// reference: std::invalid_argument
inline Error invalid_argument(const std::string& w) { return Error(kInvalidArgument, w); }
// reference: std::logic_error (check_invariants)
inline Error logic_error(const std::string& w) { return Error(kLogicError, w); }
// reference: hps::TierFault (types.hpp:14-20)
inline Error tier_fault(const std::string& w) { return Error(kTierFault, w); }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw Error(kOutOfMemory, std::string(what) + ": " + cudaGetErrorString(e));
  }
  throw Error(kInternal, std::string(what) + ": " + cudaGetErrorString(e));
}
#define HPSB_CUDA(expr) ::hpsb::cuda_check((expr), #expr)

// Grow-only device buffer. Growing synchronises `st` first so in-flight
// kernels never see the old allocation freed underneath them.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  void* ensure(size_t bytes, cudaStream_t st) {
    if (bytes <= bytes_) return p_;
    if (p_) {
      HPSB_CUDA(cudaStreamSynchronize(st));
      HPSB_CUDA(cudaFree(p_));
      p_ = nullptr;
      bytes_ = 0;
    }
    size_t b = 1;
    while (b < bytes) b <<= 1;
    HPSB_CUDA(cudaMalloc(&p_, b));
    bytes_ = b;
    return p_;
  }
  void* get() const { return p_; }
  size_t size() const { return bytes_; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

// Device-accessible address of pinned host memory (cudaHostAlloc'd or
// registered; the same address under unified addressing), nullptr for
// pageable memory.
inline void* host_mapped(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Grow-only page-locked host buffer (for async copies).
class PinnedBuffer {
 public:
  PinnedBuffer() = default;
  ~PinnedBuffer() {
    if (p_) cudaFreeHost(p_);
  }
  PinnedBuffer(const PinnedBuffer&) = delete;
  PinnedBuffer& operator=(const PinnedBuffer&) = delete;
  void* ensure(size_t bytes) {
    if (bytes <= bytes_) return p_;
    if (p_) cudaFreeHost(p_);
    p_ = nullptr;
    size_t b = 4096;
    while (b < bytes) b <<= 1;
    HPSB_CUDA(cudaHostAlloc(&p_, b, cudaHostAllocPortable));
    bytes_ = b;
    return p_;
  }
  void* get() const { return p_; }

 private:
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

// Fixed-size pool running index-range jobs: parallel_for(n, fn) calls
// fn(begin, end) over contiguous chunks and returns when all are done.
class ThreadPool {
 public:
  explicit ThreadPool(unsigned threads) {
    if (threads == 0) threads = 1;
    for (unsigned t = 1; t < threads; ++t) workers_.emplace_back([this] { loop(); });
    nthreads_ = threads;
  }
  ~ThreadPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& w : workers_) w.join();
  }
  unsigned size() const { return nthreads_; }

  void parallel_for(size_t n, size_t min_chunk,
                    const std::function<void(size_t, size_t)>& fn) {
    if (n == 0) return;
    size_t chunks = std::min<size_t>(nthreads_, (n + min_chunk - 1) / min_chunk);
    if (chunks <= 1) {
      fn(0, n);
      return;
    }
    const size_t per = (n + chunks - 1) / chunks;
    // The countdown lives on this frame: it is decremented UNDER done_mu, so
    // the waiter (which reads it under done_mu) cannot see zero -- and return,
    // destroying done_mu / done_cv -- before the last worker has finished
    // notifying and released the lock. (Decrementing first and locking after
    // let the waiter return in between: a rare use-after-scope of the mutex.)
    size_t left = chunks - 1;
    std::mutex done_mu;
    std::condition_variable done_cv;
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (size_t c = 1; c < chunks; ++c) {
        const size_t b = c * per, e = std::min(n, b + per);
        q_.push_back([&, b, e] {
          if (b < e) fn(b, e);
          std::lock_guard<std::mutex> dl(done_mu);
          if (--left == 0) done_cv.notify_all();
        });
      }
    }
    cv_.notify_all();
    fn(0, std::min(n, per));
    std::unique_lock<std::mutex> dl(done_mu);
    done_cv.wait(dl, [&] { return left == 0; });
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (q_.empty()) return;
        job = std::move(q_.front());
        q_.pop_front();
      }
      job();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  bool stop_ = false;
  unsigned nthreads_ = 1;
};

// Scoped device selection.
class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (prev_ != dev) cudaSetDevice(dev);
    dev_ = dev;
  }
  ~DeviceGuard() {
    if (prev_ != dev_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0;
  int dev_ = 0;
};

}  // namespace hpsb
