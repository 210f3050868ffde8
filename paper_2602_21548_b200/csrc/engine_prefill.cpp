// Prefill mode of the executor: quota-batched forwards
// of K5 over the landed KV, layer by layer.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <thread>

#include "dualpath/engine.hpp"
#include "engine_detail.hpp"
#include "tier_reader.hpp"

namespace dualpath {

using detail::check;
using detail::check_cuda;
using detail::DeviceScope;
using detail::upload;

void EngineRuntime::upload_prefill_tables() {
  const ExecPlan& x = *plan_;
  const auto& items = x.fwd_items[engine_];
  const auto& fwds = x.forwards[engine_];
  const std::int32_t L = x.cfg.n_layer;
  stream_c_ = detail::acquire_stream(device_);  // the compute stream: forwards
  // the load stream outranks the compute stream: as K5 CTAs retire, the
  // block scheduler places pending loader CTAs first
  detail::release_stream(device_, static_cast<cudaStream_t>(stream_));
  stream_ = detail::acquire_stream(device_, /*high_priority=*/true);
  d_fwd_slot_ = upload(x.fwd_slot[engine_]);
  const std::size_t rows = std::max<std::size_t>(1, x.fwd_rows[engine_].size());
  check_cuda(cudaMalloc(reinterpret_cast<void**>(&d_digest_), rows * L * sizeof(std::uint64_t)),
             "cudaMalloc digests");
  check_cuda(cudaMemset(d_digest_, 0, rows * L * sizeof(std::uint64_t)), "cudaMemset digests");
  std::vector<std::int32_t> wt;
  std::vector<std::uint32_t> wg;
  fwd_att_.assign(fwds.size(), {});
  fwd_done_.assign(fwds.size(), {});
  fwd_wait_off_.assign(fwds.size(), 0);
  fwd_wait_n_.assign(fwds.size(), 0);
  for (std::size_t f = 0; f < fwds.size(); ++f) {
    fwd_wait_off_[f] = static_cast<std::int64_t>(wt.size());
    for (std::int32_t i = fwds[f].begin; i < fwds[f].end; ++i) {
      const FwdItem& it = items[i];
      dp_attend_item a{};
      a.cached = it.cached;
      a.q_begin = it.q_begin;
      a.bsz = it.bsz;
      a.digest = d_digest_ + static_cast<std::int64_t>(it.row) * L;
      a.req = static_cast<std::uint32_t>(it.req);
      if (it.job >= 0) {
        const LoadJob& j = x.jobs[it.job];
        a.slot = d_fwd_slot_ + j.fwd_off;
        if (it.first) {  // the request's KV is read here first: gate every layer on it
          wt.push_back(j.ticket);
          wg.push_back(static_cast<std::uint32_t>(static_cast<std::int64_t>(j.n_blk) * x.items_per_block));
        }
        if (x.last_fwd[it.job] == static_cast<int>(f)) fwd_done_[f].push_back(j.ticket);
      }
      fwd_att_[f].push_back(a);
    }
    fwd_wait_n_[f] = static_cast<std::int32_t>(wt.size() - fwd_wait_off_[f]);
    cudaEvent_t e;
    check_cuda(cudaEventCreate(&e), "cudaEventCreate");  // timed: the handoff lag
    ev_fwd_.push_back(e);
  }
  d_fwt_ = upload(wt);
  d_fwg_ = upload(wg);
}

// Prefill step of a PE.  The load stream runs this PE's own reads (K1) in
// FIFO order; the compute stream runs the forwards, layer by layer: a wait
// on the landed counters of the requests the forward reads first, then K5.
// A forward is enqueued after the loads of its requests, so every wait is
// enqueued after its producer.  A load that reuses slots waits for the event
// of the forward that last read them; DE loads wait on the "consumed" rows
// the compute stream writes after that forward.
StepResult EngineRuntime::run_step_prefill(bool loads) {
  const ExecPlan& x = *plan_;
  DeviceScope ds(device_);
  auto s = static_cast<cudaStream_t>(stream_);
  auto c = static_cast<cudaStream_t>(stream_c_);
  StepResult res;
  const auto t0 = std::chrono::steady_clock::now();
  check(dp_nic_start(nic_), "dp_nic_start");
  auto start = static_cast<cudaEvent_t>(ev_start_);
  auto end = static_cast<cudaEvent_t>(ev_end_);
  check_cuda(cudaEventRecord(start, s), "cudaEventRecord");
  check_cuda(cudaStreamWaitEvent(c, start, 0), "cudaStreamWaitEvent");
  const std::int32_t L = x.cfg.n_layer;
  const auto& rows = x.fwd_rows[engine_];
  check_cuda(cudaMemsetAsync(d_digest_, 0, std::max<std::size_t>(1, rows.size()) * L * sizeof(std::uint64_t), c),
             "cudaMemsetAsync digests");
  const auto& fwds = x.forwards[engine_];
  std::size_t fi = 0;
  if (loads) {
    std::vector<int> job_of_row(rows.size(), -1);
    for (const FwdItem& it : x.fwd_items[engine_]) job_of_row[it.row] = it.job;
    const bool k1_ce = x.opt.k1_mode == 1;
    const bool k1_st = x.opt.k1_mode == 3 && stager_;
    const std::int64_t st_launch0 = stager_launches();
    std::vector<dp_job> batch;
    std::vector<int> batch_jobs;  // by_reader positions (the storage tier's job ids)
    detail::BufferGate buf(x.opt.buffer_bound ? buffer_budget() : 0);
    std::unique_ptr<TierReader> tier;
    if (x.tier && !x.by_reader[engine_].empty()) tier = std::make_unique<TierReader>(*this, x.by_reader[engine_]);
    int li = 0;  // by_reader position of the next own load
    auto flush = [&]() {
      if (batch.empty()) return;
      const auto n = static_cast<int32_t>(batch.size());
      if (k1_ce) {
        check(x.opt.copy_release_per_job ? dp_h2d_layer_copy_job(pool_, store_, batch.data(), n, s)
                                         : dp_h2d_layer_copy(pool_, store_, batch.data(), n, s),
              "dp_h2d_layer_copy");
      } else if (k1_st) {
        check(dp_h2d_layer_staged(pool_, store_, stager_, batch.data(), n, s), "dp_h2d_layer_staged");
      } else {
        check(dp_h2d_layer_gather(pool_, store_, batch.data(), n, s), "dp_h2d_layer_gather");
        res.launches += (n + DP_MAX_JOBS_PER_LAUNCH - 1) / DP_MAX_JOBS_PER_LAUNCH;
      }
      batch.clear();
      if (tier) tier->launched(batch_jobs, s);
      batch_jobs.clear();
      buf.launched(s);
    };
    const double cap = x.opt.storage_cap_per_engine.empty() ? x.opt.storage_cap_Bps
                                                            : x.opt.storage_cap_per_engine[engine_];
    const double pace = x.opt.pace_scale;
    // enqueue forwards whose requests' loads are all enqueued (row < r)
    auto forwards_before = [&](std::size_t r) {
      while (fi < fwds.size() && static_cast<std::size_t>(fwds[fi].last_row) < r) {
        flush();
        enqueue_forward(static_cast<int>(fi++), res);
      }
    };
    for (std::size_t r = 0; r < rows.size(); ++r) {
      const int ji = job_of_row[r];
      if (ji < 0 || x.jobs[ji].reader != engine_ || x.jobs[ji].n_blk == 0) continue;
      const LoadJob& j = x.jobs[ji];
      const std::int64_t bytes = j.cached * x.cfg.kv_bytes_per_token();
      const bool gated = cap > 0 || pace > 0;
      const int pos = li++;
      // loads run ahead of the forwards (the compute stream's queue may be
      // long); they stop only for a slot reuse, whose reader forward must be
      // enqueued first, and for the storage gate or a read still on the disk,
      // which let the forwards that are ready start before the host waits
      if (tier && !tier->ready(pos)) {
        forwards_before(r);
        flush();
        res.io_wait_ms += tier->wait(pos);
      }
      if (gated || !j.consumer_waits.empty()) forwards_before(r);
      if (gated || !j.consumer_waits.empty() || batch.size() == DP_MAX_JOBS_PER_LAUNCH) flush();
      buf.reserve(bytes, flush);
      for (int w : j.consumer_waits)
        check_cuda(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_fwd_[x.last_fwd[w]]), 0),
                   "cudaStreamWaitEvent");
      if (gated) {
        storage_read(j, bytes, res);
      }
      if (k1_ce)
        batch.push_back(dp_job{x.src_fb[engine_].data() + j.blk_off, x.slots[engine_].data() + j.blk_off,
                               j.cached, j.n_blk, 0, L, j.ticket});
      else if (k1_st)
        batch.push_back(dp_job{x.src_fb[engine_].data() + j.blk_off, stage_slots() + j.blk_off, j.cached,
                               j.n_blk, 0, L, j.ticket});
      else
        batch.push_back(dp_job{d_src_ + j.blk_off, d_slots_ + j.blk_off, j.cached, j.n_blk, 0, L, j.ticket});
      batch_jobs.push_back(pos);
      res.bytes_read += bytes;
      ++res.jobs;
    }
    flush();
    res.launches += stager_launches() - st_launch0;
    res.buffer_stalls = buf.stalls();
    res.buffer_wait_ms = buf.wait_ms();
  }
  while (fi < fwds.size()) enqueue_forward(static_cast<int>(fi++), res);
  // the step ends when both streams are drained
  check_cuda(cudaEventRecord(end, s), "cudaEventRecord");
  check_cuda(cudaStreamWaitEvent(c, end, 0), "cudaStreamWaitEvent");
  check_cuda(cudaEventRecord(end, c), "cudaEventRecord");
  check_cuda(cudaEventSynchronize(end), "step sync");
  check(dp_wait_status(pool_), "transfer watchdog");
  float ms = 0;
  check_cuda(cudaEventElapsedTime(&ms, start, end), "cudaEventElapsedTime");
  res.device_ms = ms;
  read_back_landed(res);
  res.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

void EngineRuntime::enqueue_forward(int f, StepResult& res) {
  const ExecPlan& x = *plan_;
  auto c = static_cast<cudaStream_t>(stream_c_);
  const std::int32_t L = x.cfg.n_layer;
  const auto& att = fwd_att_[f];
  std::int64_t work = 0;
  for (const dp_attend_item& a : att) work += (a.cached > 0 && a.bsz > 0) ? 1 : 0;
  for (std::int32_t layer = 0; layer < L; ++layer) {
    if (fwd_wait_n_[f] > 0) {
      check(dp_wait_tickets(pool_, d_fwt_ + fwd_wait_off_[f], d_fwg_ + fwd_wait_off_[f], fwd_wait_n_[f], layer,
                            x.opt.wait_timeout_ms, c),
            "dp_wait_tickets (forward gate)");
      ++res.launches;
    }
    // layerwise handoff: K5's last CTA out flags "forward f computed layer l"
    // (row fwd_row0_ + f of the pool's counters), which K3 gates on
    std::uint32_t* done = nullptr;
    if (layerwise_handoff()) {
      void* base = nullptr;
      std::uint32_t* ctr = nullptr;
      std::int64_t bytes = 0;
      check(dp_pool_info(pool_, &base, &ctr, &bytes), "dp_pool_info");
      done = ctr + static_cast<std::int64_t>(fwd_row0_ + f) * (L + 1) + layer;
    }
    check(dp_prefill_attend_signal(pool_, layer, att.data(), static_cast<int32_t>(att.size()), x.opt.seed, done, c),
          "dp_prefill_attend");
    res.launches += (work + DP_MAX_ATTEND_ITEMS_PER_LAUNCH - 1) / DP_MAX_ATTEND_ITEMS_PER_LAUNCH;
  }
  check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_fwd_[f]), c), "cudaEventRecord");
  if (!x.handoff)  // with the handoff, K3 (after the forward) marks the rows
    for (std::int32_t t : fwd_done_[f])
      check(dp_stream_write_counter(pool_, t + x.n_tickets[engine_], L, 1, c), "dp_stream_write_counter");
  ++res.forwards;
}

StepResult EngineRuntime::run_forwards() {
  if (!plan_->prefill || !is_pe()) throw std::logic_error("run_forwards: prefill mode, PE engines only");
  return run_step_prefill(false);
}

std::vector<std::uint64_t> EngineRuntime::prefill_digests() const {
  if (!plan_->prefill || !is_pe()) throw std::logic_error("prefill_digests: prefill mode, PE engines only");
  DeviceScope ds(device_);
  const std::size_t n = plan_->fwd_rows[engine_].size() * plan_->cfg.n_layer;
  std::vector<std::uint64_t> out(n);
  if (n) check_cuda(cudaMemcpy(out.data(), d_digest_, n * 8, cudaMemcpyDeviceToHost), "digests D2H");
  return out;
}

}  // namespace dualpath
