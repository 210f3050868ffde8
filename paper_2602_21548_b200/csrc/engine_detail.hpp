// Internal helpers shared by the executor's translation units.
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <deque>
#include <stdexcept>
#include <utility>
#include <string>
#include <vector>

#include "dualpath/kv_abi.h"

namespace dualpath::detail {

inline void check(int rc, const char* what) {
  if (rc != DP_OK) throw std::runtime_error(std::string(what) + ": " + dp_last_error());
}

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Executor streams come from a per-device pool created in one burst and
// reused (never destroyed): the driver maps streams to its hardware queues
// round-robin in creation order, so a burst of consecutive streams lands on
// distinct queues.  Engines that share a GPU (the 1-GPU DE read path) then
// never have one engine's blocked wait queued in front of the other's
// producer, however many streams came and went before.
cudaStream_t acquire_stream(int device, bool high_priority = false);
void release_stream(int device, cudaStream_t s);

// The reader's host staging bound (pe_buffer_bytes / de_buffer_bytes,
// types.hpp:22-23; try_admit's reservation, desim.cpp:587-599): a job's hit KV
// occupies the buffer from its StorageRead until its transfer has landed.
// Before a job is read the executor reserves its bytes; while the buffer is
// full it first launches what it has batched, then waits (host side) for the
// oldest launched transfers to complete -- an admission stall.
class BufferGate {
 public:
  explicit BufferGate(std::int64_t budget) : budget_(budget) {}
  ~BufferGate() {
    for (auto& e : q_) cudaEventDestroy(e.first);
  }
  BufferGate(const BufferGate&) = delete;
  BufferGate& operator=(const BufferGate&) = delete;
  // `flush` launches the batched (pending) jobs and calls launched()
  template <class Flush>
  void reserve(std::int64_t bytes, Flush&& flush) {
    if (budget_ <= 0) return;
    if (held_ + pending_ + bytes > budget_ && pending_ > 0) flush();
    while (held_ + pending_ + bytes > budget_ && !q_.empty()) {
      const auto t0 = std::chrono::steady_clock::now();
      check_cuda(cudaEventSynchronize(q_.front().first), "buffer gate sync");
      wait_ms_ += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      cudaEventDestroy(q_.front().first);
      held_ -= q_.front().second;
      q_.pop_front();
      ++stalls_;
    }
    pending_ += bytes;
  }
  // the pending jobs were launched on `s`: they leave the buffer when it gets here
  void launched(cudaStream_t s) {
    if (budget_ <= 0 || pending_ == 0) return;
    cudaEvent_t e;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    check_cuda(cudaEventRecord(e, s), "cudaEventRecord");
    q_.emplace_back(e, pending_);
    held_ += pending_;
    pending_ = 0;
  }
  std::int64_t stalls() const { return stalls_; }
  double wait_ms() const { return wait_ms_; }

 private:
  std::int64_t budget_, held_ = 0, pending_ = 0, stalls_ = 0;
  double wait_ms_ = 0;
  std::deque<std::pair<cudaEvent_t, std::int64_t>> q_;
};

template <class T>
T* upload(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* d = nullptr;
  check_cuda(cudaMalloc(reinterpret_cast<void**>(&d), v.size() * sizeof(T)), "cudaMalloc tables");
  check_cuda(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload tables");
  return d;
}

}  // namespace dualpath::detail
