// The emulated storage NIC of the C ABI (include/dualpath/kv_abi.h, dp_nic_*):
// the rate cap of StorageRead, a flow over {snic_rd[node], dram[node]}
// (/root/reference/proj/src/desim.cpp:603-606) whose bandwidth is the node's
// storage_bandwidth (types.hpp:27-29).  Requests are served FIFO at the cap,
// like the reference's single flow per read once it holds the NIC alone.
#include <algorithm>
#include <chrono>
#include <mutex>
#include <string>
#include <thread>

#include "dualpath/kv_abi.h"

namespace dualpath::detail {
int set_error(int code, const std::string& msg);  // kv_abi.cu: thread-local dp_last_error
}

struct dp_nic {
  double rate = 0;  // bytes/s, 0 = unlimited
  std::mutex mu;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  double busy_until = 0;  // s since t0
};

extern "C" {

int dp_nic_create(double rate_Bps, dp_nic** out) {
  if (!out || !(rate_Bps >= 0)) return dualpath::detail::set_error(DP_EINVAL, "nic_create: bad argument");
  *out = new dp_nic;
  (*out)->rate = rate_Bps;
  return DP_OK;
}

int dp_nic_destroy(dp_nic* nic) {
  delete nic;
  return DP_OK;
}

int dp_nic_start(dp_nic* nic) {
  if (!nic) return dualpath::detail::set_error(DP_EINVAL, "nic_start: null nic");
  std::lock_guard<std::mutex> lk(nic->mu);
  nic->t0 = std::chrono::steady_clock::now();
  nic->busy_until = 0;
  return DP_OK;
}

int dp_nic_read(dp_nic* nic, int64_t bytes, double not_before_s, double* t_begin, double* t_end) {
  if (!nic || bytes < 0) return dualpath::detail::set_error(DP_EINVAL, "nic_read: bad argument");
  double begin, end;
  std::chrono::steady_clock::time_point t0;
  {
    std::lock_guard<std::mutex> lk(nic->mu);
    // an idle NIC starts the read now: no credit for the time it sat idle
    const double now = std::chrono::duration<double>(std::chrono::steady_clock::now() - nic->t0).count();
    begin = std::max({nic->busy_until, not_before_s, now});
    end = begin + (nic->rate > 0 ? static_cast<double>(bytes) / nic->rate : 0.0);
    nic->busy_until = end;
    t0 = nic->t0;
  }
  std::this_thread::sleep_until(t0 + std::chrono::duration<double>(end));
  if (t_begin) *t_begin = begin;
  if (t_end) *t_end = end;
  return DP_OK;
}

}  // extern "C"
