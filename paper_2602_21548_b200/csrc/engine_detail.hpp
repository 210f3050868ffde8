// Internal helpers shared by the executor's translation units.
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
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

template <class T>
T* upload(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* d = nullptr;
  check_cuda(cudaMalloc(reinterpret_cast<void**>(&d), v.size() * sizeof(T)), "cudaMalloc tables");
  check_cuda(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload tables");
  return d;
}

}  // namespace dualpath::detail
