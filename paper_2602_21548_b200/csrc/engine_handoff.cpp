// PD handoff mode of the executor: K3 per request,
// the DE's fused dual reads, decode stand-in and K4 persistence, optionally
// with the prefill forwards in between.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <limits>
#include <thread>

#include "dualpath/engine.hpp"
#include "engine_detail.hpp"

namespace dualpath {

using detail::check;
using detail::check_cuda;
using detail::DeviceScope;

// PD handoff step.  A PE runs two streams: the load stream (its own reads,
// K1, gated by the storage NIC) and the handoff stream (per request: K3 =
// prefill stand-in + PeToDe / MissMerge, gated per layer on the request's hit
// KV).  A DE runs its reads as the fused dual gather (PE pool + its decode
// pool) and ends once every request of its decode pool is complete.
StepResult EngineRuntime::run_step_handoff() {
  const ExecPlan& x = *plan_;
  DeviceScope ds(device_);
  auto s = static_cast<cudaStream_t>(stream_);
  auto h = static_cast<cudaStream_t>(stream_h_);
  StepResult res;
  const auto t0 = std::chrono::steady_clock::now();
  check(dp_nic_start(nic_), "dp_nic_start");
  auto start = static_cast<cudaEvent_t>(ev_start_);
  check_cuda(cudaEventRecord(start, s), "cudaEventRecord");
  if (h) check_cuda(cudaStreamWaitEvent(h, start, 0), "cudaStreamWaitEvent");
  const std::int32_t L = x.cfg.n_layer;
  const double cap = x.opt.storage_cap_per_engine.empty() ? x.opt.storage_cap_Bps
                                                          : x.opt.storage_cap_per_engine[engine_];
  const double pace = x.opt.pace_scale;
  const bool gated = cap > 0 || pace > 0;
  auto storage_gate = [&](const LoadJob& j) {
    const std::int64_t bytes = j.cached * x.cfg.kv_bytes_per_token();
    if (gated) {
      storage_read(j, bytes, res);
    }
    res.bytes_read += bytes;
    ++res.jobs;
  };
  const auto nt = [&](int pe) { return x.n_tickets[pe]; };

  if (is_pe()) {
    const bool pf = x.prefill;
    auto c = static_cast<cudaStream_t>(stream_c_);
    const auto& mine = x.by_pe[engine_];
    std::vector<std::int32_t> row_of;  // prefill: FIFO row of each job of this PE
    if (pf) {
      check_cuda(cudaStreamWaitEvent(c, start, 0), "cudaStreamWaitEvent");
      const std::size_t rows = std::max<std::size_t>(1, x.fwd_rows[engine_].size());
      check_cuda(cudaMemsetAsync(d_digest_, 0, rows * L * sizeof(std::uint64_t), c), "cudaMemsetAsync digests");
      row_of.assign(x.jobs.size(), -1);
      for (const FwdItem& it : x.fwd_items[engine_])
        if (it.job >= 0) row_of[it.job] = it.row;
    }
    // K3 of a set of jobs on the handoff stream: each job's decode-slot
    // hazards, then one K3 call per decode engine (a layerwise forward's
    // requests in one launch: every request's layer l moves once the forward
    // has computed l), then each job's "K3 done" event
    const bool lw = pf && layerwise_handoff();
    auto enqueue_k3_set = [&](const std::vector<int>& set) {
      std::vector<std::pair<int, dp_handoff_job>> hjs;  // (decode engine, job)
      for (int ji : set) {
        const LoadJob& j = x.jobs[ji];
        if (pf && !lw)  // the prompt is handed off after its last forward
          check_cuda(cudaStreamWaitEvent(h, static_cast<cudaEvent_t>(ev_fwd_[x.last_fwd[ji]]), 0),
                     "cudaStreamWaitEvent");
        if (!j.de_preds.empty()) {
          const std::int64_t off = de_wait_off_[ji];
          check(dp_wait_tickets(de_views_[j.de], d_wt_ + off, d_wg_ + off,
                                static_cast<int32_t>(j.de_preds.size()), L, x.opt.wait_timeout_ms, h),
                "dp_wait_tickets (decode slots)");
          ++res.launches;
        }
        const bool layer_gate = x.opt.k3_layer_gate == 1;
        if (j.de_path && j.n_blk > 0 && !layer_gate && !lw) {
          // the whole request's hit KV, pushed by its DE: a one-thread spin
          // kernel with the watchdog (a DE that never pushes -- e.g. its rank
          // died -- fails the step with DP_ETIMEOUT instead of hanging it)
          check(dp_wait_layer(pool_, j.ticket, L,
                              static_cast<std::uint32_t>(static_cast<std::int64_t>(j.n_blk) * x.items_per_block * L),
                              x.opt.wait_timeout_ms, h),
                "dp_wait_layer (handoff gate)");
          ++res.launches;
        }
        dp_handoff_job hj{d_ho_src_ + j.ho_off,
                          d_ho_pe_ + j.ho_off,
                          d_ho_de_ + j.ho_off,
                          j.cached,
                          j.prompt,
                          j.n_pblk,
                          j.de_path ? 0 : 1,
                          // layerwise: layer l waits for the finishing forward's layer l (which
                          // itself waited for the request's hit KV of layer l)
                          lw ? fwd_row0_ + x.last_fwd[ji] : (j.de_path && j.n_blk > 0 && layer_gate) ? j.ticket : -1,
                          lw ? 1u : static_cast<std::uint32_t>(static_cast<std::int64_t>(j.n_blk) * x.items_per_block),
                          j.de_ticket,
                          j.ticket + nt(engine_)};
        hjs.emplace_back(j.de, hj);
      }
      std::vector<int> des;
      for (const auto& [de, hj] : hjs)
        if (std::find(des.begin(), des.end(), de) == des.end()) des.push_back(de);
      for (int de : des) {
        std::vector<dp_handoff_job> batch;
        for (const auto& [d, hj] : hjs)
          if (d == de) batch.push_back(hj);
        if (x.opt.k3_mode == 1) {
          // copy engines: the same jobs with host-readable block tables
          for (dp_handoff_job& hj : batch) {
            const std::int64_t off = hj.src_fb - d_ho_src_;
            hj.src_fb = x.ho_src_fb[engine_].data() + off;
            hj.pe_slot = x.ho_pe_slot[engine_].data() + off;
            hj.de_slot = x.ho_de_slot[engine_].data() + off;
          }
          std::int64_t n0 = 0, n1 = 0;
          check(dp_handoff_copy_launches(&n0), "dp_handoff_copy_launches");
          for (std::size_t b0 = 0; b0 < batch.size(); b0 += DP_MAX_HANDOFF_JOBS_PER_LAUNCH) {
            const auto nb = std::min<std::size_t>(DP_MAX_HANDOFF_JOBS_PER_LAUNCH, batch.size() - b0);
            check(dp_prefill_handoff_copy(pool_, de_views_[de], batch.data() + b0, static_cast<int32_t>(nb),
                                          x.opt.seed, x.opt.wait_timeout_ms, h),
                  "dp_prefill_handoff_copy");
          }
          check(dp_handoff_copy_launches(&n1), "dp_handoff_copy_launches");
          res.launches += n1 - n0;
          continue;
        }
        check(dp_prefill_handoff(pool_, de_views_[de], batch.data(), static_cast<int32_t>(batch.size()), x.opt.seed,
                                 x.opt.wait_timeout_ms, h),
              "dp_prefill_handoff");
        res.launches += (static_cast<std::int64_t>(batch.size()) + DP_MAX_HANDOFF_JOBS_PER_LAUNCH - 1) /
                        DP_MAX_HANDOFF_JOBS_PER_LAUNCH;
      }
      for (int ji : set)
        check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_k3_[pe_local_[ji]]), h), "cudaEventRecord");
    };
    auto enqueue_k3 = [&](int ji) { enqueue_k3_set({ji}); };
    // prefill: forwards whose requests' loads are all enqueued (row < r), and
    // the K3s of the requests they finish
    static const std::vector<Forward> kNone;
    const std::vector<Forward>& fwds = pf ? x.forwards[engine_] : kNone;
    std::size_t fi = 0, ki = 0;
    auto drain = [&](std::int64_t r) {
      while (fi < fwds.size() && fwds[fi].last_row < r) {
        enqueue_forward(static_cast<int>(fi++), res);
        std::vector<int> set;
        while (ki < mine.size() && x.last_fwd[mine[ki]] < static_cast<int>(fi)) set.push_back(mine[ki++]);
        if (lw) {
          if (!set.empty()) enqueue_k3_set(set);
        } else {
          for (int ji : set) enqueue_k3(ji);
        }
      }
    };
    for (int ji : mine) {
      const LoadJob& j = x.jobs[ji];
      const int li = pe_local_[ji];
      auto ev_load = static_cast<cudaEvent_t>(ev_load_[li]);
      if (!de_views_[j.de]) throw std::runtime_error("run_step: DE " + std::to_string(j.de) + " not attached");
      // a load reusing slots waits for K3s, which wait for forwards: enqueue them first
      if (pf && (!j.k3_waits.empty() || gated)) drain(row_of[ji]);
      // --- load stream: this PE's own reads (PE path)
      if (!j.de_path && j.n_blk > 0) {
        for (int w : j.k3_waits)
          check_cuda(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_k3_[pe_local_[w]]), 0),
                     "cudaStreamWaitEvent");
        storage_gate(j);
        dp_job job{d_src_ + j.blk_off, d_slots_ + j.blk_off, j.cached, j.n_blk, 0, L, j.ticket};
        if (x.opt.k1_mode == 1) {
          job.src_fb = x.src_fb[engine_].data() + j.blk_off;
          job.dst_slot = x.slots[engine_].data() + j.blk_off;
          check(x.opt.copy_release_per_job ? dp_h2d_layer_copy_job(pool_, store_, &job, 1, s)
                                           : dp_h2d_layer_copy(pool_, store_, &job, 1, s),
                "dp_h2d_layer_copy");
        } else if (x.opt.k1_mode == 3 && stager_) {
          job.src_fb = x.src_fb[engine_].data() + j.blk_off;
          job.dst_slot = stage_slots() + j.blk_off;
          const std::int64_t l0 = stager_launches();
          check(dp_h2d_layer_staged(pool_, store_, stager_, &job, 1, s), "dp_h2d_layer_staged");
          res.launches += stager_launches() - l0;
        } else {
          check(dp_h2d_layer_gather(pool_, store_, &job, 1, s), "dp_h2d_layer_gather");
          ++res.launches;
        }
        check_cuda(cudaEventRecord(ev_load, s), "cudaEventRecord");
        check_cuda(cudaStreamWaitEvent(h, ev_load, 0), "cudaStreamWaitEvent");
      } else if (!j.de_path) {
        // cold request on the PE path: only its K3 reuses slots
        for (int w : j.k3_waits)
          check_cuda(cudaStreamWaitEvent(h, static_cast<cudaEvent_t>(ev_k3_[pe_local_[w]]), 0),
                     "cudaStreamWaitEvent");
      }
      if (!pf) enqueue_k3(ji);
    }
    if (pf) {
      drain(std::numeric_limits<std::int64_t>::max());
      while (ki < mine.size()) enqueue_k3(mine[ki++]);
    }
    // the step ends when every stream is drained
    auto end_ev = static_cast<cudaEvent_t>(ev_end_);
    check_cuda(cudaEventRecord(end_ev, s), "cudaEventRecord");
    check_cuda(cudaStreamWaitEvent(h, end_ev, 0), "cudaStreamWaitEvent");
    if (pf) {
      check_cuda(cudaEventRecord(end_ev, c), "cudaEventRecord");
      check_cuda(cudaStreamWaitEvent(h, end_ev, 0), "cudaStreamWaitEvent");
    }
    check_cuda(cudaEventRecord(end_ev, h), "cudaEventRecord");
  } else {
    // A DE enqueues its work job by job in the global order, across its two
    // streams: every operation a wait depends on belongs to an earlier job,
    // so it was enqueued earlier -- even if the driver multiplexes both
    // streams onto one hardware queue, a blocked wait never sits in front of
    // its own producer.
    const std::int64_t T = x.cfg.block_size_tokens;
    // With the prefill the order is the plan's (ExecPlan::de_order): a
    // request's K3 follows forwards that may hold later requests, so global
    // order alone is not enough.
    std::size_t ri = 0, di = 0, oi = 0;
    const auto& reads = x.by_reader[engine_];
    const auto& decodes = x.by_de[engine_];
    const auto& order = x.prefill ? x.de_order[engine_] : std::vector<int>{};
    while (x.prefill ? oi < order.size() : (ri < reads.size() || (x.persist && di < decodes.size()))) {
      bool take_read;
      int next_read = -1;
      if (x.prefill) {
        const int code = order[oi++];
        take_read = code >= 0;
        if (take_read) next_read = code;
        else if (di >= decodes.size() || decodes[di] != -1 - code)
          throw std::logic_error("run_step: DE order out of step with its decodes");
      } else {
        take_read = ri < reads.size() && (!x.persist || di >= decodes.size() || reads[ri] <= decodes[di]);
        if (take_read) next_read = reads[ri++];
      }
      if (take_read) {  // DE read path: dual gather
        const int ji = next_read;
        const LoadJob& j = x.jobs[ji];
        if (!peers_[j.pe]) throw std::runtime_error("run_step: PE " + std::to_string(j.pe) + " not attached");
        if (!j.pe_done_preds.empty()) {
          const std::int64_t off = pe_done_off_[ji];
          check(dp_wait_tickets(peers_[j.pe], d_wt_ + off, d_wg_ + off,
                                static_cast<int32_t>(j.pe_done_preds.size()), L, x.opt.wait_timeout_ms, s),
                "dp_wait_tickets (prefill slots)");
          ++res.launches;
        }
        if (!j.de_preds.empty()) {
          const std::int64_t off = de_wait_off_[ji];
          check(dp_wait_tickets(pool_, d_wt_ + off, d_wg_ + off, static_cast<int32_t>(j.de_preds.size()),
                                L, x.opt.wait_timeout_ms, s),
                "dp_wait_tickets (decode slots)");
          ++res.launches;
        }
        storage_gate(j);
        dp_dual_job dj{{d_src_ + j.blk_off, d_slots_ + j.blk_off, j.cached, j.n_blk, 0, L, j.ticket},
                       d_dual_de_ + j.blk_off,
                       j.de_ticket,
                       0};
        if (x.opt.k2_mode == 2 && stager_) {  // staged: copy engine into the ring, then the dual scatter
          dj.pe.src_fb = x.src_fb[engine_].data() + j.blk_off;
          const std::int64_t l0 = stager_launches();
          check(dp_h2d_push_dual_staged(peers_[j.pe], pool_, store_, stager_, &dj, 1, s), "dp_h2d_push_dual_staged");
          res.launches += stager_launches() - l0;
        } else {
          check(dp_h2d_push_p2p_dual(peers_[j.pe], pool_, store_, &dj, 1, s), "dp_h2d_push_p2p_dual");
          ++res.launches;
        }
        continue;
      }
      // decode stream: once the request's whole prompt has landed, the
      // decode stand-in writes its generated tokens, K4 persists them chunk
      // by chunk, then its "persist done" row is set
      const std::int64_t pos = static_cast<std::int64_t>(di);
      const LoadJob& j = x.jobs[decodes[di++]];
      check(dp_wait_tickets(pool_, d_wt_ + final_wait_off_ + pos, d_wg_ + final_wait_off_ + pos, 1, L,
                            x.opt.wait_timeout_ms, h),
            "dp_wait_tickets (decode ready)");
      const std::int64_t blk0 = j.prompt / T;
      const std::int32_t nb = j.n_tblk - static_cast<std::int32_t>(blk0);
      const dp_span_job fill{d_dec_slot_ + j.dec_off + blk0, d_dec_fb_ + j.dec_off + blk0, blk0,
                             j.prompt, j.prompt + j.gen, nb, 0};
      check(dp_decode_fill(pool_, &fill, 1, x.opt.seed, h), "dp_decode_fill");
      std::vector<dp_span_job> chunks;
      for (const auto& [t0, t1] : x.persist_chunks(j))
        chunks.push_back(dp_span_job{fill.slot, fill.fb, blk0, t0, t1, nb, 0});
      if (persist_stager_) {  // staged: the block tables' host copy plans the copies
        for (dp_span_job& c : chunks) c.fb = x.dec_fb[engine_].data() + j.dec_off + blk0;
        const std::int64_t l0 = persist_launches();
        check(dp_persist_staged(pool_, persist_store_, persist_stager_, chunks.data(),
                                static_cast<int32_t>(chunks.size()), h),
              "dp_persist_staged");
        res.launches += persist_launches() - l0 - 1;  // its kernels (K4 is counted below)
      } else {
        check(dp_persist_d2h(pool_, persist_store_, chunks.data(), static_cast<int32_t>(chunks.size()), h),
              "dp_persist_d2h");
      }
      check(dp_stream_write_counter(pool_, j.de_ticket + x.n_de_tickets[engine_], L, 1, h),
            "dp_stream_write_counter");
      res.launches += 3;
    }
    if (x.persist) {
      check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_end_), s), "cudaEventRecord");
      check_cuda(cudaStreamWaitEvent(h, static_cast<cudaEvent_t>(ev_end_), 0), "cudaStreamWaitEvent");
      check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_end_), h), "cudaEventRecord");
    } else {
      if (final_wait_n_ > 0) {  // decode-ready: every prompt landed in this decode pool
        check(dp_wait_tickets(pool_, d_wt_ + final_wait_off_, d_wg_ + final_wait_off_, final_wait_n_, L,
                              x.opt.wait_timeout_ms, s),
              "dp_wait_tickets (decode ready)");
        ++res.launches;
      }
      check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_end_), s), "cudaEventRecord");
    }
  }
  check_cuda(cudaEventSynchronize(static_cast<cudaEvent_t>(ev_end_)), "step sync");
  if (pool_) check(dp_wait_status(pool_), "transfer watchdog");
  for (dp_pool* p : peers_)
    if (p && p != pool_) check(dp_wait_status(p), "transfer watchdog");
  for (dp_pool* p : de_views_)
    if (p) check(dp_wait_status(p), "transfer watchdog");
  float ms = 0;
  check_cuda(cudaEventElapsedTime(&ms, start, static_cast<cudaEvent_t>(ev_end_)), "cudaEventElapsedTime");
  res.device_ms = ms;
  persist_write(res);
  if (is_pe()) {  // per request: its prompt KV complete in the decode pool
    for (int ji : x.by_pe[engine_]) {
      float t = 0, tf = 0;
      check_cuda(cudaEventElapsedTime(&t, start, static_cast<cudaEvent_t>(ev_k3_[pe_local_[ji]])),
                 "cudaEventElapsedTime");
      res.ttft_ms.push_back(t);
      if (x.prefill) {
        check_cuda(cudaEventElapsedTime(&tf, start, static_cast<cudaEvent_t>(ev_fwd_[x.last_fwd[ji]])),
                   "cudaEventElapsedTime");
        res.handoff_lag_ms.push_back(t - tf);
      }
    }
  }
  read_back_landed(res);
  res.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

}  // namespace dualpath
