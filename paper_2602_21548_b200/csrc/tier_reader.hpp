// Storage-tier IO of the executor (internal): see TierReader below.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "dualpath/engine.hpp"
#include "engine_detail.hpp"

namespace dualpath {

// Storage tier IO for one step of one reader: `io_threads` host threads read
// each job's Full Blocks from the file into its staging-ring positions, in
// job order, first waiting (event) for the transfer that last read a ring
// position they overwrite; the launch thread issues a job once it is read.
class TierReader {
 public:
  TierReader(EngineRuntime& rt, const std::vector<int>& mine) : rt_(rt), mine_(mine) {
    const ExecPlan& x = *rt.plan_;
    void* host = nullptr;
    detail::check(dp_store_info(rt.store_, &host, nullptr, nullptr), "dp_store_info");
    staging_ = static_cast<char*>(host);
    read_.assign(mine.size(), 0);
    launched_.assign(mine.size(), 0);
    for (int t = 0; t < x.opt.io_threads; ++t) workers_.emplace_back([this] { work(); });
  }
  ~TierReader() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      failed_ = true;  // releases any worker still waiting (normal exit: all done)
      cv_.notify_all();
    }
    for (auto& t : workers_) t.join();
  }
  char* staging() const { return staging_; }
  bool ready(int i) {
    std::lock_guard<std::mutex> lk(mu_);
    if (err_) std::rethrow_exception(err_);
    return read_[i] != 0;
  }
  // Blocks until job i is read; returns the milliseconds waited.
  double wait(int i) {
    const auto t0 = std::chrono::steady_clock::now();
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return read_[i] || failed_; });
    if (err_) std::rethrow_exception(err_);
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  // The jobs were just enqueued on `s`: record their events, wake the readers.
  void launched(const std::vector<int>& jobs, cudaStream_t s) {
    for (int i : jobs) detail::check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(rt_.ev_job_[i]), s), "cudaEventRecord");
    std::lock_guard<std::mutex> lk(mu_);
    for (int i : jobs) launched_[i] = 1;
    cv_.notify_all();
  }

 private:
  void work() {
    const ExecPlan& x = *rt_.plan_;
    try {
      cudaSetDevice(rt_.device_);
      const std::int64_t fbb = x.cfg.full_block_bytes();
      for (int i = next_++; i < static_cast<int>(mine_.size()); i = next_++) {
        for (int w : rt_.ring_wait_local_[i]) {
          {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return launched_[w] || failed_; });
            if (failed_) return;
          }
          detail::check_cuda(cudaEventSynchronize(static_cast<cudaEvent_t>(rt_.ev_job_[w])), "ring reuse wait");
        }
        // one read per run of blocks consecutive both in the file and in
        // the ring (a session's pages are consecutive records)
        const LoadJob& j = x.jobs[mine_[i]];
        const std::int64_t* rec = x.tier_rec[rt_.engine_].data() + j.blk_off;
        const std::int64_t* pos = x.src_fb[rt_.engine_].data() + j.blk_off;
        constexpr std::int32_t kMaxRun = 8;  // 18 MB of DS-V3 Full Blocks per read
        for (std::int32_t k = 0; k < j.n_blk;) {
          std::int32_t run = 1;
          while (k + run < j.n_blk && run < kMaxRun && rec[k + run] == rec[k] + run && pos[k + run] == pos[k] + run)
            ++run;
          rt_.tier_file_->read_run(rec[k], run, staging_ + pos[k] * fbb);
          k += run;
        }
        std::lock_guard<std::mutex> lk(mu_);
        read_[i] = 1;
        cv_.notify_all();
      }
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu_);
      if (!err_) err_ = std::current_exception();
      failed_ = true;
      cv_.notify_all();
    }
  }

  EngineRuntime& rt_;
  const std::vector<int>& mine_;
  char* staging_ = nullptr;
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<char> read_, launched_;
  std::atomic<int> next_{0};
  bool failed_ = false;
  std::exception_ptr err_;
  std::vector<std::thread> workers_;
};

}  // namespace dualpath
