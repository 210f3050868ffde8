// GPU executor of the DualPath KV loading path (see dualpath/engine.hpp):
// the engine runtime and the plain load step.  The plan is built in
// exec_plan.cpp, the prefill and handoff steps live in engine_prefill.cpp and
// engine_handoff.cpp.
#include "dualpath/engine.hpp"
#include "engine_detail.hpp"
#include "tier_reader.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <limits>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <tuple>

namespace dualpath {

namespace detail {

namespace {
struct StreamPool {
  std::vector<cudaStream_t> free_lo, free_hi;
};
std::mutex g_stream_mu;
std::vector<StreamPool> g_stream_pools;
constexpr int kStreamBurst = 12;  // per priority; 24 < CUDA_DEVICE_MAX_CONNECTIONS = 32
}  // namespace

cudaStream_t acquire_stream(int device, bool high_priority) {
  std::lock_guard<std::mutex> lk(g_stream_mu);
  if (device < 0) throw std::invalid_argument("acquire_stream: bad device");
  if (g_stream_pools.size() <= static_cast<std::size_t>(device)) g_stream_pools.resize(device + 1);
  StreamPool& p = g_stream_pools[device];
  auto& list = high_priority ? p.free_hi : p.free_lo;
  if (list.empty()) {
    DeviceScope ds(device);
    int lo = 0, hi = 0;
    check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
    for (int i = 0; i < kStreamBurst; ++i) {
      cudaStream_t s;
      check_cuda(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, high_priority ? hi : lo),
                 "cudaStreamCreateWithPriority");
      list.insert(list.begin(), s);
    }
  }
  cudaStream_t s = list.back();
  list.pop_back();
  return s;
}

void release_stream(int device, cudaStream_t s) {
  if (!s) return;
  cudaStreamSynchronize(s);
  int lo = 0, hi = 0, prio = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStreamGetPriority(s, &prio);
  std::lock_guard<std::mutex> lk(g_stream_mu);
  auto& p = g_stream_pools[device];
  (prio == hi && hi != lo ? p.free_hi : p.free_lo).push_back(s);
}

}  // namespace detail

using detail::check;
using detail::check_cuda;
using detail::DeviceScope;
using detail::upload;

EngineRuntime::EngineRuntime(std::shared_ptr<const ExecPlan> plan, int engine, int device)
    : plan_(std::move(plan)), engine_(engine), device_(device) {
  if (!plan_) throw std::invalid_argument("EngineRuntime: null plan");
  if (engine < 0 || engine >= plan_->n_engines)
    throw std::invalid_argument("EngineRuntime: engine out of range");
  const ExecPlan& x = *plan_;
  DeviceScope ds(device_);
  stream_ = detail::acquire_stream(device_);
  cudaEvent_t a, b;
  check_cuda(cudaEventCreate(&a), "cudaEventCreate");
  check_cuda(cudaEventCreate(&b), "cudaEventCreate");
  ev_start_ = a;
  ev_end_ = b;
  peers_.assign(x.n_engines, nullptr);
  de_views_.assign(x.n_engines, nullptr);
  check(dp_nic_create(x.opt.storage_cap_per_engine.empty() ? x.opt.storage_cap_Bps
                                                           : x.opt.storage_cap_per_engine[engine_],
                      &nic_),
        "dp_nic_create");
  if (!x.by_reader[engine_].empty()) {
    // with the storage tier the store is the pinned staging ring the reads land in
    check(dp_store_create(device_, &x.geom, x.tier ? x.ring_fb : x.store_fb, x.opt.seed, &store_),
          "dp_store_create");
    if (x.tier) {
      tier_file_ = std::make_unique<FullBlockFile>(x.opt.tier_path, x.geom, x.store_fb, false, x.opt.tier_direct);
      const auto& mine = x.by_reader[engine_];
      std::vector<int> local(x.jobs.size(), -1);
      for (std::size_t i = 0; i < mine.size(); ++i) local[mine[i]] = static_cast<int>(i);
      for (int ji : mine) {
        cudaEvent_t e;
        check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        ev_job_.push_back(e);
        std::vector<int> w;
        for (int p : x.jobs[ji].ring_waits) w.push_back(local[p]);
        ring_wait_local_.push_back(std::move(w));
      }
    }
  }
  if (is_pe()) {
    // handoff: rows [0, n) hit-KV landed, rows [n, 2n) handoff (K3) done
    // handoff / prefill: rows [0, n) hit-KV landed, rows [n, 2n) handoff done / consumed
    // + with the layerwise handoff, one row per forward: its per-layer done flags
    fwd_row0_ = std::max<std::int32_t>(1, x.n_tickets[engine_]) * (x.handoff || x.prefill ? 2 : 1);
    const std::int32_t rows =
        fwd_row0_ + (layerwise_handoff() ? static_cast<std::int32_t>(x.forwards[engine_].size()) : 0);
    check(dp_pool_create_layout(device_, &x.geom, x.pool_slots, rows, x.opt.pool_layout, &pool_), "dp_pool_create");
    peers_[engine_] = pool_;
  } else if (x.handoff) {
    // rows [0, n) prompt landed; with persistence rows [n, 2n) persisted
    const std::int32_t rows = std::max<std::int32_t>(1, x.n_de_tickets[engine_]) * (x.persist ? 2 : 1);
    check(dp_pool_create(device_, &x.geom, x.de_pool_slots, rows, &pool_), "dp_pool_create (decode pool)");
    if (x.persist && !x.by_de[engine_].empty())  // content seed + 1: unwritten bytes differ
      check(dp_store_create(device_, &x.geom, x.store_fb, x.opt.seed + 1, &persist_store_),
            "dp_store_create (persist store)");
    if (x.persist && x.opt.persist_mode == 1 && !x.by_de[engine_].empty())
      check(dp_stager_create(device_, &x.geom, x.opt.stage_ring_bytes, &persist_stager_),
            "dp_stager_create (persist)");
    if (x.persist && !x.opt.persist_path.empty() && !x.by_de[engine_].empty())
      persist_file_ = std::make_unique<FullBlockFile>(x.opt.persist_path, x.geom, x.store_fb, false, false);
  }
  if (!x.by_reader[engine_].empty() && ((is_pe() && x.opt.k1_mode == 3) || (!is_pe() && x.opt.k2_mode == 2))) {
    check(dp_stager_create(device_, &x.geom, x.opt.stage_ring_bytes, &stager_), "dp_stager_create");
    check(dp_stager_set_ctas(stager_, is_pe() ? x.opt.stage_ctas : x.opt.stage_push_ctas), "dp_stager_set_ctas");
    check(dp_stager_set_mode(stager_, x.opt.stage_scatter), "dp_stager_set_mode");
  }
  if (x.handoff) {
    upload_handoff_tables();
  } else {
    upload_tables();
  }
  if (x.prefill && is_pe()) upload_prefill_tables();
  if (x.opt.k1_mode == 2 && is_pe() && !x.handoff && !x.prefill) {
    stream_ce_ = detail::acquire_stream(device_);
    for (int k = 0; k < 2; ++k) {
      cudaEvent_t e;
      check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
      ev_ce_.push_back(e);
    }
  }
  // K1 is PCIe-bound and keeps its rate down to ~32 CTAs; on a PE that also
  // runs K3 the remaining SMs go to the handoff
  // (and on a prefill PE, 32 CTAs keep 51 GB/s while costing K5 the least:
  // tools/prefill_interference.py)
  std::int32_t ctas = x.opt.gather_ctas;
  if (ctas < 0) ctas = !is_pe() ? 0 : x.prefill ? 32 : x.handoff ? 64 : 0;
  check(dp_set_gather_ctas(device_, ctas), "dp_set_gather_ctas");
  if (is_pe() && x.handoff) check(dp_set_handoff_tma(x.opt.handoff_tma ? 1 : 0), "dp_set_handoff_tma");
  // layerwise with the copy-engine K3: its gates are this PE's own forward
  // rows (released by K5 on this GPU), so stream waits, not spinning CTAs
  if (is_pe() && x.handoff)
    check(dp_set_handoff_gate_memop(layerwise_handoff() && x.opt.k3_mode == 1 ? 1 : 0), "dp_set_handoff_gate_memop");
  // layerwise K3 CTAs wait in-kernel for the forward's layers: 64 of them.
  // One per SM hung the 1P1D pipeline (profiles/r02_g15_pf_lw148_HANG.txt):
  // with a spinning K3 CTA resident on every SM, a producer the gates wait
  // for could not be scheduled; 64 leave SMs free of spinners.
  if (is_pe())
    check(dp_set_handoff_ctas(device_, x.opt.handoff_ctas ? x.opt.handoff_ctas : layerwise_handoff() ? 64 : 0),
          "dp_set_handoff_ctas");
  if (is_pe() && x.prefill) check(dp_set_attend_ctas(device_, x.opt.attend_ctas), "dp_set_attend_ctas");
}

EngineRuntime::~EngineRuntime() {
  DeviceScope ds(device_);
  if (stream_) cudaStreamSynchronize(static_cast<cudaStream_t>(stream_));
  if (stream_h_) cudaStreamSynchronize(static_cast<cudaStream_t>(stream_h_));
  if (stream_c_) cudaStreamSynchronize(static_cast<cudaStream_t>(stream_c_));
  if (stream_ce_) cudaStreamSynchronize(static_cast<cudaStream_t>(stream_ce_));
  for (int e = 0; e < static_cast<int>(peers_.size()); ++e)
    if (peers_[e] && peers_[e] != pool_) dp_pool_destroy(peers_[e]);
  for (dp_pool* v : de_views_)
    if (v) dp_pool_destroy(v);
  if (pool_) dp_pool_destroy(pool_);
  dp_stager_destroy(stager_);
  dp_stager_destroy(persist_stager_);
  if (store_) dp_store_destroy(store_);
  dp_nic_destroy(nic_);
  if (persist_store_) dp_store_destroy(persist_store_);
  for (void* p : {static_cast<void*>(d_src_), static_cast<void*>(d_slots_),
                  static_cast<void*>(d_wait_tickets_), static_cast<void*>(d_wait_targets_),
                  static_cast<void*>(d_pred_tickets_), static_cast<void*>(d_pred_targets_),
                  static_cast<void*>(d_ho_src_), static_cast<void*>(d_ho_pe_),
                  static_cast<void*>(d_ho_de_), static_cast<void*>(d_dual_de_),
                  static_cast<void*>(d_wt_), static_cast<void*>(d_wg_),
                  static_cast<void*>(d_dec_slot_), static_cast<void*>(d_dec_fb_),
                  static_cast<void*>(d_digest_), static_cast<void*>(d_fwd_slot_),
                  static_cast<void*>(d_fwt_), static_cast<void*>(d_fwg_)})
    if (p) cudaFree(p);
  for (void* e : ev_load_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  for (void* e : ev_k3_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  for (void* e : ev_fwd_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  for (void* e : ev_job_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  if (ev_start_) cudaEventDestroy(static_cast<cudaEvent_t>(ev_start_));
  if (ev_end_) cudaEventDestroy(static_cast<cudaEvent_t>(ev_end_));
  detail::release_stream(device_, static_cast<cudaStream_t>(stream_h_));
  detail::release_stream(device_, static_cast<cudaStream_t>(stream_c_));
  detail::release_stream(device_, static_cast<cudaStream_t>(stream_ce_));
  for (void* e : ev_ce_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  detail::release_stream(device_, static_cast<cudaStream_t>(stream_));
}

void EngineRuntime::upload_tables() {
  const ExecPlan& x = *plan_;
  d_src_ = upload(x.src_fb[engine_]);
  d_slots_ = upload(x.slots[engine_]);
  std::vector<std::int32_t> pt;
  std::vector<std::uint32_t> pg;
  pred_off_.clear();
  for (int ji : x.by_reader[engine_]) {
    pred_off_.push_back(static_cast<std::int64_t>(pt.size()));
    const LoadJob& j = x.jobs[ji];
    pt.insert(pt.end(), j.preds.begin(), j.preds.end());
    pg.insert(pg.end(), j.pred_targets.begin(), j.pred_targets.end());
  }
  d_pred_tickets_ = upload(pt);
  d_pred_targets_ = upload(pg);
  if (is_pe()) {
    std::vector<std::int32_t> wt;
    std::vector<std::uint32_t> wg;
    for (int ji : x.by_pe[engine_]) {
      const LoadJob& j = x.jobs[ji];
      if (j.reader == engine_) continue;  // own stream orders these already
      wt.push_back(j.ticket);
      wg.push_back(static_cast<std::uint32_t>(static_cast<std::int64_t>(j.n_blk) *
                                              x.items_per_block * x.cfg.n_layer));
    }
    n_wait_ = static_cast<std::int32_t>(wt.size());
    d_wait_tickets_ = upload(wt);
    d_wait_targets_ = upload(wg);
  }
}

void EngineRuntime::upload_handoff_tables() {
  const ExecPlan& x = *plan_;
  d_src_ = upload(x.src_fb[engine_]);
  d_slots_ = upload(x.slots[engine_]);
  d_dual_de_ = upload(x.dual_de_slot[engine_]);
  std::vector<std::int32_t> wt;
  std::vector<std::uint32_t> wg;
  de_wait_off_.assign(x.jobs.size(), -1);
  pe_done_off_.assign(x.jobs.size(), -1);
  pe_local_.assign(x.jobs.size(), -1);
  if (is_pe()) {
    d_ho_src_ = upload(x.ho_src_fb[engine_]);
    d_ho_pe_ = upload(x.ho_pe_slot[engine_]);
    d_ho_de_ = upload(x.ho_de_slot[engine_]);
    stream_h_ = detail::acquire_stream(device_);
    const auto& mine = x.by_pe[engine_];
    for (std::size_t i = 0; i < mine.size(); ++i) {
      pe_local_[mine[i]] = static_cast<int>(i);
      cudaEvent_t a, b;
      check_cuda(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "cudaEventCreate");
      check_cuda(cudaEventCreate(&b), "cudaEventCreate");  // timed: per-request TTFT
      ev_load_.push_back(a);
      ev_k3_.push_back(b);
      const LoadJob& j = x.jobs[mine[i]];
      de_wait_off_[mine[i]] = static_cast<std::int64_t>(wt.size());
      for (std::int32_t t : j.de_preds) wt.push_back(t + (x.persist ? x.n_de_tickets[j.de] : 0));
      wg.insert(wg.end(), j.de_pred_targets.begin(), j.de_pred_targets.end());
    }
  }
  // DE read path (dual): waits on the PE done-rows and on its own decode pool
  for (int ji : x.by_reader[engine_]) {
    const LoadJob& j = x.jobs[ji];
    if (!j.de_path) continue;
    pe_done_off_[ji] = static_cast<std::int64_t>(wt.size());
    for (std::int32_t t : j.pe_done_preds) wt.push_back(t + x.n_tickets[j.pe]);
    wg.insert(wg.end(), j.pe_done_targets.begin(), j.pe_done_targets.end());
    if (de_wait_off_[ji] < 0) {  // a DE reading for its own decode pool (always: reader == de)
      de_wait_off_[ji] = static_cast<std::int64_t>(wt.size());
      for (std::int32_t t : j.de_preds) wt.push_back(t + (x.persist ? x.n_de_tickets[j.de] : 0));
      wg.insert(wg.end(), j.de_pred_targets.begin(), j.de_pred_targets.end());
    }
  }
  if (!is_pe()) {  // decode-ready gate: every row of this decode pool complete
    final_wait_off_ = static_cast<std::int64_t>(wt.size());
    for (int ji : x.by_de[engine_]) {
      wt.push_back(x.jobs[ji].de_ticket);
      wg.push_back(x.de_total_items(x.jobs[ji]));
    }
    final_wait_n_ = static_cast<std::int32_t>(x.by_de[engine_].size());
  }
  d_wt_ = upload(wt);
  d_wg_ = upload(wg);
  if (x.persist && !is_pe()) {
    d_dec_slot_ = upload(x.dec_slot[engine_]);
    d_dec_fb_ = upload(x.dec_fb[engine_]);
    stream_h_ = detail::acquire_stream(device_);  // the decode stream: decode stand-in + persistence
  }
}

dp_pool_handle EngineRuntime::export_pool() const {
  if (!pool_) throw std::logic_error("export_pool: this engine owns no pool");
  dp_pool_handle h;
  check(dp_pool_export(pool_, &h), "dp_pool_export");
  return h;
}

void EngineRuntime::attach_peer(int engine, const dp_pool_handle& handle) {
  if (engine < 0 || engine >= plan_->n_engines || engine == engine_)
    throw std::invalid_argument("attach_peer: bad engine");
  auto& slot = engine < plan_->n_pe ? peers_[engine] : de_views_[engine];
  if (slot) return;
  dp_pool* v = nullptr;
  check(dp_pool_import(device_, &handle, &v), "dp_pool_import");
  slot = v;
}

void EngineRuntime::attach_peer_local(int engine, const EngineRuntime& other) {
  if (engine == engine_ || !other.pool_) throw std::invalid_argument("attach_peer_local: bad engine");
  auto& slot = engine < plan_->n_pe ? peers_[engine] : de_views_[engine];
  if (slot) return;
  dp_pool* v = nullptr;
  check(dp_pool_peer_view(device_, other.pool_, &v), "dp_pool_peer_view");
  slot = v;
}

void EngineRuntime::reset_counters() {
  // the watchdog flags of this engine's views of other pools are its own:
  // clear them too, so one fired watchdog does not fail every later step
  for (dp_pool* v : peers_)
    if (v && v != pool_) check(dp_wait_clear(v), "dp_wait_clear");
  for (dp_pool* v : de_views_)
    if (v) check(dp_wait_clear(v), "dp_wait_clear");
  if (!pool_) return;
  DeviceScope ds(device_);
  check(dp_pool_reset_counters(pool_, stream_), "dp_pool_reset_counters");
  check_cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)), "reset sync");
}

// The step's result, read back to the host: on a PE, the all-layer column of
// every hit-KV landed row (one 32-bit word per request), checked against the
// plan -- the host-side proof that each request's KV is in the pool.
void EngineRuntime::read_back_landed(StepResult& res) {
  const ExecPlan& x = *plan_;
  if (!is_pe() || !pool_) return;
  const std::int32_t n = x.n_tickets[engine_];
  if (n <= 0) return;
  if (landed_host_.size() < static_cast<std::size_t>(n)) landed_host_.resize(n);
  const std::size_t row = static_cast<std::size_t>(x.cfg.n_layer + 1) * sizeof(std::uint32_t);
  void* base = nullptr;
  std::uint32_t* ctr = nullptr;
  std::int64_t bytes = 0;
  check(dp_pool_info(pool_, &base, &ctr, &bytes), "dp_pool_info");
  check_cuda(cudaMemcpy2D(landed_host_.data(), sizeof(std::uint32_t), ctr + x.cfg.n_layer, row,
                          sizeof(std::uint32_t), n, cudaMemcpyDeviceToHost),
             "landed counters D2H");
  res.d2h_bytes += static_cast<std::int64_t>(n) * sizeof(std::uint32_t);
  for (int ji : x.by_pe[engine_]) {
    const LoadJob& j = x.jobs[ji];
    const std::uint32_t want =
        static_cast<std::uint32_t>(static_cast<std::int64_t>(j.n_blk) * x.items_per_block * x.cfg.n_layer);
    if (landed_host_[j.ticket] != want)
      throw std::runtime_error("step incomplete: request " + std::to_string(j.req) + " landed " +
                               std::to_string(landed_host_[j.ticket]) + " of " + std::to_string(want) +
                               " items");
  }
}

StepResult EngineRuntime::run_step() {
  const ExecPlan& x = *plan_;
  if (x.handoff) return run_step_handoff();
  if (x.prefill && is_pe()) return run_step_prefill(true);
  DeviceScope ds(device_);
  auto s = static_cast<cudaStream_t>(stream_);
  StepResult res;
  const auto t0 = std::chrono::steady_clock::now();
  check(dp_nic_start(nic_), "dp_nic_start");
  check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_start_), s), "cudaEventRecord");

  const auto& mine = x.by_reader[engine_];
  std::vector<dp_job> batch;
  batch.reserve(DP_MAX_JOBS_PER_LAUNCH);
  std::vector<int> batch_jobs;  // by_reader positions of the jobs in `batch`
  std::vector<char> in_batch(x.jobs.size(), 0);  // job index -> in `batch`
  int batch_pe = -1;
  const bool k1_ce = x.opt.k1_mode == 1;
  const bool k2_ce = x.opt.k2_mode == 1;
  const bool k1_st = x.opt.k1_mode == 3 && stager_;
  const bool k2_st = x.opt.k2_mode == 2 && stager_;
  const std::int64_t st_launch0 = stager_launches();
  // K1 hybrid (k1_mode 2): the PE's own jobs split by bytes between the SM
  // gather (load stream) and the copy engine (a second stream), run together
  const bool hybrid = x.opt.k1_mode == 2 && stream_ce_ != nullptr && !x.tier;
  auto sc = static_cast<cudaStream_t>(stream_ce_);
  std::vector<dp_job> batch_ce;
  double sm_bytes = 0, ce_bytes = 0;
  if (hybrid) check_cuda(cudaStreamWaitEvent(sc, static_cast<cudaEvent_t>(ev_start_), 0), "cudaStreamWaitEvent");

  // Storage tier: IO threads stage each job's Full Blocks (TierReader)
  std::unique_ptr<TierReader> tier;
  if (x.tier && !mine.empty()) tier = std::make_unique<TierReader>(*this, mine);

  detail::BufferGate buf(x.opt.buffer_bound && !hybrid ? buffer_budget() : 0);
  auto flush = [&]() {
    if (batch.empty()) return;
    dp_pool* dst = peers_[batch_pe];
    const auto n = static_cast<int32_t>(batch.size());
    int rc;
    const char* what;
    const bool per_job = x.opt.copy_release_per_job;
    if (batch_pe != engine_ && k2_ce) {
      rc = per_job ? dp_h2d_push_copy_job(dst, store_, batch.data(), n, s) : dp_h2d_push_copy(dst, store_, batch.data(), n, s);
      what = "dp_h2d_push_copy";
    } else if (batch_pe != engine_ && k2_st) {
      rc = dp_h2d_push_staged(dst, store_, stager_, batch.data(), n, s);
      what = "dp_h2d_push_staged";
    } else if (batch_pe == engine_ && k1_st) {
      rc = dp_h2d_layer_staged(dst, store_, stager_, batch.data(), n, s);
      what = "dp_h2d_layer_staged";
    } else if (batch_pe != engine_) {
      rc = dp_h2d_push_p2p_layer(dst, store_, batch.data(), n, s);
      what = "dp_h2d_push_p2p_layer";
    } else if (k1_ce) {
      rc = per_job ? dp_h2d_layer_copy_job(dst, store_, batch.data(), n, s) : dp_h2d_layer_copy(dst, store_, batch.data(), n, s);
      what = "dp_h2d_layer_copy";
    } else {
      rc = dp_h2d_layer_gather(dst, store_, batch.data(), n, s);
      what = "dp_h2d_layer_gather";
    }
    check(rc, what);
    buf.launched(s);
    const bool on_ce = batch_pe == engine_ ? (k1_ce || k1_st) : (k2_ce || k2_st);
    if (!on_ce)  // kernel launches (the copy engine paths have none; staged ones are counted below)
      res.launches += (static_cast<std::int64_t>(batch.size()) + DP_MAX_JOBS_PER_LAUNCH - 1) /
                      DP_MAX_JOBS_PER_LAUNCH;
    batch.clear();
    if (tier) tier->launched(batch_jobs, s);
    for (int i : batch_jobs) in_batch[mine[i]] = 0;
    batch_jobs.clear();
  };
  auto flush_ce = [&]() {
    if (batch_ce.empty()) return;
    check(dp_h2d_layer_copy(pool_, store_, batch_ce.data(), static_cast<int32_t>(batch_ce.size()), sc),
          "dp_h2d_layer_copy");
    batch_ce.clear();
  };
  // both streams see everything enqueued so far on either (slot reuse across them)
  auto join_streams = [&]() {
    flush();
    flush_ce();
    auto a = static_cast<cudaEvent_t>(ev_ce_[0]), b = static_cast<cudaEvent_t>(ev_ce_[1]);
    check_cuda(cudaEventRecord(a, sc), "cudaEventRecord");
    check_cuda(cudaStreamWaitEvent(s, a, 0), "cudaStreamWaitEvent");
    check_cuda(cudaEventRecord(b, s), "cudaEventRecord");
    check_cuda(cudaStreamWaitEvent(sc, b, 0), "cudaStreamWaitEvent");
  };
  const double cap = x.opt.storage_cap_per_engine.empty() ? x.opt.storage_cap_Bps
                                                          : x.opt.storage_cap_per_engine[engine_];
  const double pace = x.opt.pace_scale;
  for (std::size_t i = 0; i < mine.size(); ++i) {
    const LoadJob& j = x.jobs[mine[i]];
    if (!peers_[j.pe]) throw std::runtime_error("run_step: PE " + std::to_string(j.pe) + " not attached");
    const std::int64_t bytes = j.cached * x.cfg.kv_bytes_per_token();
    const bool gated = cap > 0 || pace > 0;
    const bool hazard = !j.preds.empty();
    // a same-reader slot reuse only needs a launch boundary when the previous
    // occupant is in the launch being built (launches on one stream are ordered)
    bool fence_now = false;
    for (int w : j.fence_jobs) fence_now = fence_now || in_batch[w];
    if (gated || hazard || fence_now || batch_pe != j.pe || batch.size() == DP_MAX_JOBS_PER_LAUNCH)
      flush();
    if (hybrid) {
      if (hazard || j.fence) join_streams();
      else if (gated || batch_ce.size() == DP_MAX_JOBS_PER_LAUNCH) flush_ce();
    }
    buf.reserve(bytes, flush);  // the reader's staging bound (may launch, then wait)
    if (gated) {
      // StorageRead of C*L*b bytes over this engine's storage NIC: starts
      // when the NIC is free (and, replaying online, not before the planned
      // admission), takes bytes / cap
      storage_read(j, bytes, res);
    }
    if (tier && !tier->ready(static_cast<int>(i))) {  // StorageRead: the job's Full Blocks in staging
      flush();  // never hold launched work while waiting on the disk
      res.io_wait_ms += tier->wait(static_cast<int>(i));
    }
    if (hazard) {
      const std::int64_t off = pred_off_[i];
      check(dp_wait_tickets(peers_[j.pe], d_pred_tickets_ + off, d_pred_targets_ + off,
                            static_cast<int32_t>(j.preds.size()), x.cfg.n_layer,
                            x.opt.wait_timeout_ms, s),
            "dp_wait_tickets");
      ++res.launches;
    }
    if (hybrid && j.pe == engine_) {
      // the copy engine takes a job when its queue would finish first
      // (measured side by side: copy engine 26.6, SM gather 28.4 GB/s)
      if (ce_bytes * 28.4 < sm_bytes * 26.6) {
        if (hazard) join_streams();  // the ticket wait ran on the load stream
        batch_ce.push_back(dp_job{x.src_fb[engine_].data() + j.blk_off, x.slots[engine_].data() + j.blk_off,
                                  j.cached, j.n_blk, 0, x.cfg.n_layer, j.ticket});
        ce_bytes += static_cast<double>(bytes);
        res.bytes_read += bytes;
        ++res.jobs;
        continue;
      }
      sm_bytes += static_cast<double>(bytes);
    }
    batch_pe = j.pe;
    if (j.pe == engine_ ? k1_st : k2_st)  // staged: host-readable sources; slots for the scatter
      batch.push_back(dp_job{x.src_fb[engine_].data() + j.blk_off, stage_slots() + j.blk_off, j.cached, j.n_blk,
                             0, x.cfg.n_layer, j.ticket});
    else if (j.pe == engine_ ? k1_ce : k2_ce)  // copy engine: host-readable block tables
      batch.push_back(dp_job{x.src_fb[engine_].data() + j.blk_off, x.slots[engine_].data() + j.blk_off,
                             j.cached, j.n_blk, 0, x.cfg.n_layer, j.ticket});
    else
      batch.push_back(dp_job{d_src_ + j.blk_off, d_slots_ + j.blk_off, j.cached, j.n_blk, 0,
                             x.cfg.n_layer, j.ticket});
    batch_jobs.push_back(static_cast<int>(i));
    in_batch[mine[i]] = 1;
    res.bytes_read += bytes;
    ++res.jobs;
  }
  flush();
  if (hybrid) join_streams();
  if (pool_ && n_wait_ > 0 && !x.prefill) {
    check(dp_wait_tickets(pool_, d_wait_tickets_, d_wait_targets_, n_wait_, x.cfg.n_layer,
                          x.opt.wait_timeout_ms, s),
          "dp_wait_tickets");
    ++res.launches;
  }
  res.launches += stager_launches() - st_launch0;
  res.buffer_stalls = buf.stalls();
  res.buffer_wait_ms = buf.wait_ms();
  check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_end_), s), "cudaEventRecord");
  check_cuda(cudaEventSynchronize(static_cast<cudaEvent_t>(ev_end_)), "step sync");
  for (dp_pool* p : peers_)
    if (p) check(dp_wait_status(p), "transfer watchdog");
  float ms = 0;
  check_cuda(cudaEventElapsedTime(&ms, static_cast<cudaEvent_t>(ev_start_),
                                  static_cast<cudaEvent_t>(ev_end_)),
             "cudaEventElapsedTime");
  res.device_ms = ms;
  read_back_landed(res);
  res.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

// This engine's host staging bound as a reader: its node's PE buffer when it
// is a PE, the DE buffer otherwise (types.hpp:22-23).
std::int64_t EngineRuntime::buffer_budget() const {
  const ExecPlan& x = *plan_;
  return is_pe() ? x.cfg.pe_buffer_bytes : x.cfg.de_buffer_bytes;
}

// The slot table the staged scatter reads: device memory for the kernel,
// host memory for the copy-engine scatter.
const std::int32_t* EngineRuntime::stage_slots() const {
  return plan_->opt.stage_scatter == DP_SCATTER_CE ? plan_->slots[engine_].data() : d_slots_;
}

std::int64_t EngineRuntime::persist_launches() const {
  std::int64_t n = 0;
  if (persist_stager_) check(dp_stager_launches(persist_stager_, &n), "dp_stager_launches");
  return n;
}

std::int64_t EngineRuntime::stager_launches() const {
  std::int64_t n = 0;
  if (stager_) check(dp_stager_launches(stager_, &n), "dp_stager_launches");
  return n;
}

// StorageRead of job j over this engine's emulated storage NIC (dp_nic): the
// read starts when the NIC is free (and, replaying online, not before the
// planned admission) and lasts bytes / cap; blocks until it is done.
void EngineRuntime::storage_read(const LoadJob& j, std::int64_t bytes, StepResult& res) {
  const double pace = plan_->opt.pace_scale;
  double b = 0, e = 0;
  check(dp_nic_read(nic_, bytes, pace > 0 ? j.t_admit * pace : 0.0, &b, &e), "dp_nic_read");
  res.spans.push_back({b, e, bytes});
}

std::vector<std::uint64_t> EngineRuntime::checksum(int layer, std::span<const std::int32_t> slots,
                                                    std::span<const std::int32_t> ntok) {
  if (!pool_) throw std::logic_error("checksum: this engine owns no pool");
  if (slots.size() != ntok.size()) throw std::invalid_argument("checksum: size mismatch");
  DeviceScope ds(device_);
  const std::size_t n = slots.size();
  std::vector<std::uint64_t> out(n);
  if (n == 0) return out;
  std::int32_t *ds_ = nullptr, *dn = nullptr;
  std::uint64_t* dout = nullptr;
  check_cuda(cudaMalloc(reinterpret_cast<void**>(&ds_), n * 4), "cudaMalloc");
  check_cuda(cudaMalloc(reinterpret_cast<void**>(&dn), n * 4), "cudaMalloc");
  check_cuda(cudaMalloc(reinterpret_cast<void**>(&dout), n * 8), "cudaMalloc");
  check_cuda(cudaMemcpy(ds_, slots.data(), n * 4, cudaMemcpyHostToDevice), "H2D");
  check_cuda(cudaMemcpy(dn, ntok.data(), n * 4, cudaMemcpyHostToDevice), "H2D");
  check(dp_pool_checksum(pool_, layer, ds_, dn, static_cast<int32_t>(n), dout, stream_),
        "dp_pool_checksum");
  check_cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)), "checksum sync");
  check_cuda(cudaMemcpy(out.data(), dout, n * 8, cudaMemcpyDeviceToHost), "D2H");
  cudaFree(ds_);
  cudaFree(dn);
  cudaFree(dout);
  return out;
}

// PersistWrite (desim.cpp:764-771): every Full Block this DE's K4 wrote in
// the step goes from the pinned persist store to its record in the storage
// tier file (pwrite), after the step's device work is done.
void EngineRuntime::persist_write(StepResult& res) {
  if (!persist_file_) return;
  const ExecPlan& x = *plan_;
  const auto t0 = std::chrono::steady_clock::now();
  void* host = nullptr;
  std::int64_t bytes = 0, n_fb = 0;
  check(dp_store_info(persist_store_, &host, &bytes, &n_fb), "dp_store_info");
  const std::int64_t T = x.cfg.block_size_tokens, fbb = x.cfg.full_block_bytes();
  const std::int64_t lb = x.cfg.layer_block_bytes(), b = x.cfg.kv_bytes_per_token_per_layer;
  // only the persisted tokens: per (Full Block, layer), each chunk's token range
  std::vector<std::tuple<std::int64_t, std::int64_t, std::int64_t>> ranges;  // (fb, tok a, tok z)
  for (int ji : x.by_de[engine_]) {
    const LoadJob& j = x.jobs[ji];
    for (const auto& [t0, t1] : x.persist_chunks(j))
      for (std::int64_t k = t0 / T; k < (t1 + T - 1) / T; ++k)
        ranges.emplace_back(x.fb_of(j.traj, k), std::max(t0, k * T) - k * T, std::min(t1, (k + 1) * T) - k * T);
  }
  std::sort(ranges.begin(), ranges.end());
  const char* base = static_cast<const char*>(host);
  for (std::size_t i = 0; i < ranges.size();) {  // merge touching ranges of one block
    auto [fb, a, z] = ranges[i];
    std::size_t k = i + 1;
    while (k < ranges.size() && std::get<0>(ranges[k]) == fb && std::get<1>(ranges[k]) <= z)
      z = std::max(z, std::get<2>(ranges[k++]));
    for (std::int32_t layer = 0; layer < x.cfg.n_layer; ++layer) {
      const std::int64_t off = layer * lb + a * b;
      persist_file_->write_bytes(fb, off, (z - a) * b, base + fb * fbb + off);
    }
    res.persist_write_bytes += (z - a) * b * x.cfg.n_layer;
    i = k;
  }
  res.persist_write_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

std::vector<std::uint8_t> EngineRuntime::read_persisted(std::int64_t fb, int layer) const {
  if (!persist_store_) throw std::logic_error("read_persisted: this engine persists nothing");
  void* host = nullptr;
  std::int64_t bytes = 0, n_fb = 0;
  check(dp_store_info(persist_store_, &host, &bytes, &n_fb), "dp_store_info");
  const ExecPlan& x = *plan_;
  if (fb < 0 || fb >= n_fb || layer < 0 || layer >= x.cfg.n_layer)
    throw std::out_of_range("read_persisted: Full Block / layer out of range");
  const std::int64_t lb = x.cfg.layer_block_bytes();
  const auto* p = static_cast<const std::uint8_t*>(host) + fb * x.cfg.full_block_bytes() + layer * lb;
  return std::vector<std::uint8_t>(p, p + lb);
}

std::vector<std::uint32_t> EngineRuntime::counters() const {
  if (!pool_) return {};
  DeviceScope ds(device_);
  void* base = nullptr;
  std::uint32_t* ctr = nullptr;
  std::int64_t bytes = 0;
  check(dp_pool_info(pool_, &base, &ctr, &bytes), "dp_pool_info");
  const ExecPlan& x = *plan_;
  const std::int32_t rows = is_pe() ? fwd_row0_ + (layerwise_handoff() ? static_cast<std::int32_t>(
                                                                            x.forwards[engine_].size())
                                                                      : 0)
                                    : std::max<std::int32_t>(1, x.n_de_tickets[engine_]) * (x.persist ? 2 : 1);
  const std::size_t n = static_cast<std::size_t>(rows) * (x.cfg.n_layer + 1);
  std::vector<std::uint32_t> out(n);
  check_cuda(cudaMemcpy(out.data(), ctr, n * 4, cudaMemcpyDeviceToHost), "counters D2H");
  return out;
}

std::vector<StepResult> run_step_all(std::span<EngineRuntime* const> engines) {
  std::vector<StepResult> out(engines.size());
  std::vector<std::exception_ptr> err(engines.size());
  std::vector<std::thread> th;
  th.reserve(engines.size());
  for (std::size_t i = 0; i < engines.size(); ++i)
    th.emplace_back([&, i] {
      try {
        out[i] = engines[i]->run_step();
      } catch (...) {
        err[i] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  return out;
}

}  // namespace dualpath
