// GPU executor of the DualPath KV loading path (see dualpath/engine.hpp).
#include "dualpath/engine.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <deque>
#include <stdexcept>
#include <thread>

namespace dualpath {

namespace {

void check(int rc, const char* what) {
  if (rc != DP_OK) throw std::runtime_error(std::string(what) + ": " + dp_last_error());
}

void check_cuda(cudaError_t e, const char* what) {
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

template <class T>
T* upload(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* d = nullptr;
  check_cuda(cudaMalloc(reinterpret_cast<void**>(&d), v.size() * sizeof(T)), "cudaMalloc tables");
  check_cuda(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload tables");
  return d;
}

}  // namespace

std::int64_t ExecPlan::fb_of(int traj, std::int64_t block) const {
  return (static_cast<std::int64_t>(traj) * fb_stride + block) % store_fb;
}

ExecPlan build_exec_plan(const pdsim::ClusterConfig& cfg,
                         std::span<const pdsim::Trajectory> trajectories,
                         const pdsim::desim::SimReport& plan, const ExecOptions& opt) {
  cfg.validate();
  ExecPlan x;
  x.cfg = cfg;
  x.opt = opt;
  x.n_engines = cfg.total_engines();
  x.n_pe = cfg.prefill_nodes * cfg.engines_per_node;
  x.geom = {cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer};
  check(dp_geom_check(&x.geom), "build_exec_plan");
  check(dp_layer_items(&x.geom, 1, &x.items_per_block), "build_exec_plan");
  const std::int64_t fb_bytes = cfg.full_block_bytes();
  const std::int64_t T = cfg.block_size_tokens;

  x.fb_stride = 1;
  for (const auto& t : trajectories)
    x.fb_stride = std::max(x.fb_stride, pdsim::blocks_for(t.total_tokens(), cfg));
  if (opt.store_fb > 0) {
    x.store_fb = opt.store_fb;
  } else {
    const std::int64_t want = x.fb_stride * static_cast<std::int64_t>(std::max<std::size_t>(1, trajectories.size()));
    const std::int64_t cap = std::max<std::int64_t>(1, opt.store_bytes_max / fb_bytes);
    x.store_fb = std::max<std::int64_t>(1, std::min(want, cap));
  }

  // jobs: every request with cached KV that reached the hit transfer
  struct Ev {
    double t;
    int kind;  // 0 = free, 1 = alloc
    int req;
    int job;
  };
  std::vector<Ev> evs;
  std::vector<LoadJob> jobs;
  for (const auto& r : plan.requests) {
    x.prompt_tokens += r.cached + r.append;
    ++x.requests;
    if (r.cached <= 0 || r.pe < 0 || r.t_read_done < 0) continue;
    if (r.traj_index < 0 || static_cast<std::size_t>(r.traj_index) >= trajectories.size())
      throw std::invalid_argument("build_exec_plan: plan does not match the trajectories");
    LoadJob j;
    j.req = r.request_id;
    j.traj = r.traj_index;
    j.round = r.round;
    j.pe = r.pe;
    j.de_path = r.path == pdsim::ReadPath::DEPath;
    j.reader = j.de_path ? r.de : r.pe;
    j.cached = r.cached;
    j.n_blk = static_cast<std::int32_t>((r.cached + T - 1) / T);
    j.t_admit = r.t_admit;
    j.t_read_done = r.t_read_done;
    const int idx = static_cast<int>(jobs.size());
    jobs.push_back(std::move(j));
    evs.push_back({r.t_read_done, 1, r.request_id, idx});
    if (r.t_pe_release >= 0) evs.push_back({r.t_pe_release, 0, r.request_id, idx});
  }
  std::sort(evs.begin(), evs.end(), [](const Ev& a, const Ev& b) {
    if (a.t != b.t) return a.t < b.t;
    if (a.kind != b.kind) return a.kind < b.kind;
    return a.req < b.req;
  });

  // pass 1: peak live blocks per PE
  {
    std::vector<std::int64_t> live(x.n_pe, 0);
    std::int64_t peak = 0;
    for (const Ev& e : evs) {
      const LoadJob& j = jobs[e.job];
      live[j.pe] += e.kind == 1 ? j.n_blk : -j.n_blk;
      peak = std::max(peak, live[j.pe]);
    }
    x.peak_slots = static_cast<std::int32_t>(peak);
  }
  const std::int64_t slot_cap = std::max<std::int64_t>(1, opt.pool_bytes_max / fb_bytes);
  if (opt.pool_slots > 0) {
    x.pool_slots = opt.pool_slots;
  } else {
    x.pool_slots = static_cast<std::int32_t>(
        std::min<std::int64_t>(slot_cap, std::max<std::int64_t>(1, 4 * static_cast<std::int64_t>(x.peak_slots))));
  }
  if (!opt.storage_cap_per_engine.empty() &&
      static_cast<int>(opt.storage_cap_per_engine.size()) != x.n_engines)
    throw std::invalid_argument("build_exec_plan: storage_cap_per_engine needs one entry per engine");
  if (x.pool_slots < x.peak_slots)
    throw std::invalid_argument("build_exec_plan: PE pool of " + std::to_string(x.pool_slots) +
                                " slots is below the plan's peak of " +
                                std::to_string(x.peak_slots) + " live blocks");

  // pass 2: slot allocation in virtual time.  Freed slots go back to a queue
  // of the engine that last wrote them; an allocation takes, in order, slots
  // its own reader last wrote (ordered by its stream: only a launch boundary
  // is needed), never-used slots, then other readers' slots (a cross-GPU
  // hazard wait).  FIFO within each queue.
  struct PeSlots {
    std::deque<std::int32_t> fresh;
    std::vector<std::deque<std::int32_t>> by_reader;
    std::vector<std::int32_t> owner;  // slot -> job index of its last writer
  };
  std::vector<PeSlots> ps(x.n_pe);
  for (int p = 0; p < x.n_pe; ++p) {
    ps[p].owner.assign(x.pool_slots, -1);
    ps[p].by_reader.assign(x.n_engines, {});
    for (std::int32_t s = 0; s < x.pool_slots; ++s) ps[p].fresh.push_back(s);
  }
  auto take = [&](PeSlots& q, int reader) -> std::int32_t {
    std::deque<std::int32_t>* src = nullptr;
    if (!q.by_reader[reader].empty()) {
      src = &q.by_reader[reader];
    } else if (!q.fresh.empty()) {
      src = &q.fresh;
    } else {
      for (int r = 0; r < x.n_engines && !src; ++r)
        if (!q.by_reader[r].empty()) src = &q.by_reader[r];
    }
    if (!src) throw std::logic_error("build_exec_plan: slot allocator ran dry below the peak");
    const std::int32_t s = src->front();
    src->pop_front();
    return s;
  };
  std::vector<std::vector<std::int32_t>> job_slots(jobs.size());
  x.n_tickets.assign(x.n_pe, 0);
  std::vector<int> order;
  order.reserve(jobs.size());
  for (const Ev& e : evs) {
    LoadJob& j = jobs[e.job];
    PeSlots& q = ps[j.pe];
    if (e.kind == 0) {
      for (std::int32_t s : job_slots[e.job]) q.by_reader[j.reader].push_back(s);
      continue;
    }
    j.ticket = x.n_tickets[j.pe]++;
    auto& mine = job_slots[e.job];
    mine.reserve(j.n_blk);
    for (std::int32_t k = 0; k < j.n_blk; ++k) {
      const std::int32_t s = take(q, j.reader);
      mine.push_back(s);
      const std::int32_t prev = q.owner[s];
      // same reader: stream order serialises launches, but items of one
      // launch run concurrently, so the reuse must start a new launch
      if (prev >= 0 && jobs[prev].reader == j.reader) j.fence = true;
      if (prev >= 0 && jobs[prev].reader != j.reader &&
          std::find(j.preds.begin(), j.preds.end(), jobs[prev].ticket) == j.preds.end()) {
        j.preds.push_back(jobs[prev].ticket);
        j.pred_targets.push_back(static_cast<std::uint32_t>(
            static_cast<std::int64_t>(jobs[prev].n_blk) * x.items_per_block * cfg.n_layer));
      }
      q.owner[s] = e.job;
    }
    order.push_back(e.job);
  }

  x.by_reader.assign(x.n_engines, {});
  x.by_pe.assign(x.n_pe, {});
  x.src_fb.assign(x.n_engines, {});
  x.slots.assign(x.n_engines, {});
  x.reader_bytes.assign(x.n_engines, 0);
  x.jobs.reserve(order.size());
  for (int old : order) {
    LoadJob j = std::move(jobs[old]);
    const int idx = static_cast<int>(x.jobs.size());
    auto& src = x.src_fb[j.reader];
    auto& dst = x.slots[j.reader];
    j.blk_off = static_cast<std::int64_t>(src.size());
    for (std::int32_t k = 0; k < j.n_blk; ++k) {
      src.push_back(x.fb_of(j.traj, k));
      dst.push_back(job_slots[old][k]);
    }
    const std::int64_t bytes = j.cached * cfg.kv_bytes_per_token();
    x.reader_bytes[j.reader] += bytes;
    x.hit_bytes += bytes;
    x.by_reader[j.reader].push_back(idx);
    x.by_pe[j.pe].push_back(idx);
    x.jobs.push_back(std::move(j));
  }
  return x;
}

EngineRuntime::EngineRuntime(std::shared_ptr<const ExecPlan> plan, int engine, int device)
    : plan_(std::move(plan)), engine_(engine), device_(device) {
  if (!plan_) throw std::invalid_argument("EngineRuntime: null plan");
  if (engine < 0 || engine >= plan_->n_engines)
    throw std::invalid_argument("EngineRuntime: engine out of range");
  DeviceScope ds(device_);
  cudaStream_t s;
  check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  stream_ = s;
  cudaEvent_t a, b;
  check_cuda(cudaEventCreate(&a), "cudaEventCreate");
  check_cuda(cudaEventCreate(&b), "cudaEventCreate");
  ev_start_ = a;
  ev_end_ = b;
  peers_.assign(plan_->n_engines, nullptr);
  if (!plan_->by_reader[engine_].empty())
    check(dp_store_create(device_, &plan_->geom, plan_->store_fb, plan_->opt.seed, &store_),
          "dp_store_create");
  if (is_pe()) {
    check(dp_pool_create(device_, &plan_->geom, plan_->pool_slots,
                         std::max<std::int32_t>(1, plan_->n_tickets[engine_]), &pool_),
          "dp_pool_create");
    peers_[engine_] = pool_;
  }
  upload_tables();
}

EngineRuntime::~EngineRuntime() {
  DeviceScope ds(device_);
  if (stream_) cudaStreamSynchronize(static_cast<cudaStream_t>(stream_));
  for (int e = 0; e < static_cast<int>(peers_.size()); ++e)
    if (peers_[e] && peers_[e] != pool_) dp_pool_destroy(peers_[e]);
  if (pool_) dp_pool_destroy(pool_);
  if (store_) dp_store_destroy(store_);
  for (void* p : {static_cast<void*>(d_src_), static_cast<void*>(d_slots_),
                  static_cast<void*>(d_wait_tickets_), static_cast<void*>(d_wait_targets_),
                  static_cast<void*>(d_pred_tickets_), static_cast<void*>(d_pred_targets_)})
    if (p) cudaFree(p);
  if (ev_start_) cudaEventDestroy(static_cast<cudaEvent_t>(ev_start_));
  if (ev_end_) cudaEventDestroy(static_cast<cudaEvent_t>(ev_end_));
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
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

dp_pool_handle EngineRuntime::export_pool() const {
  if (!pool_) throw std::logic_error("export_pool: engine is not a PE");
  dp_pool_handle h;
  check(dp_pool_export(pool_, &h), "dp_pool_export");
  return h;
}

void EngineRuntime::attach_peer(int pe_engine, const dp_pool_handle& handle) {
  if (pe_engine < 0 || pe_engine >= plan_->n_pe || pe_engine == engine_)
    throw std::invalid_argument("attach_peer: bad PE engine");
  if (peers_[pe_engine]) return;
  dp_pool* v = nullptr;
  check(dp_pool_import(device_, &handle, &v), "dp_pool_import");
  peers_[pe_engine] = v;
}

void EngineRuntime::attach_peer_local(int pe_engine, const EngineRuntime& pe) {
  if (pe_engine == engine_ || !pe.pool_) throw std::invalid_argument("attach_peer_local: bad PE");
  if (peers_[pe_engine]) return;
  dp_pool* v = nullptr;
  check(dp_pool_peer_view(device_, pe.pool_, &v), "dp_pool_peer_view");
  peers_[pe_engine] = v;
}

void EngineRuntime::reset_counters() {
  if (!pool_) return;
  DeviceScope ds(device_);
  check(dp_pool_reset_counters(pool_, stream_), "dp_pool_reset_counters");
  check_cuda(cudaStreamSynchronize(static_cast<cudaStream_t>(stream_)), "reset sync");
}

StepResult EngineRuntime::run_step() {
  const ExecPlan& x = *plan_;
  DeviceScope ds(device_);
  auto s = static_cast<cudaStream_t>(stream_);
  StepResult res;
  const auto t0 = std::chrono::steady_clock::now();
  check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_start_), s), "cudaEventRecord");

  const auto& mine = x.by_reader[engine_];
  std::vector<dp_job> batch;
  batch.reserve(DP_MAX_JOBS_PER_LAUNCH);
  int batch_pe = -1;
  const bool k1_ce = x.opt.k1_mode == 1;
  auto flush = [&]() {
    if (batch.empty()) return;
    dp_pool* dst = peers_[batch_pe];
    const auto n = static_cast<int32_t>(batch.size());
    int rc;
    const char* what;
    if (batch_pe != engine_) {
      rc = dp_h2d_push_p2p_layer(dst, store_, batch.data(), n, s);
      what = "dp_h2d_push_p2p_layer";
    } else if (k1_ce) {
      rc = dp_h2d_layer_copy(dst, store_, batch.data(), n, s);
      what = "dp_h2d_layer_copy";
    } else {
      rc = dp_h2d_layer_gather(dst, store_, batch.data(), n, s);
      what = "dp_h2d_layer_gather";
    }
    check(rc, what);
    if (!(k1_ce && batch_pe == engine_))  // kernel launches (the copy engine path has none)
      res.launches += (static_cast<std::int64_t>(batch.size()) + DP_MAX_JOBS_PER_LAUNCH - 1) /
                      DP_MAX_JOBS_PER_LAUNCH;
    batch.clear();
  };
  const double cap = x.opt.storage_cap_per_engine.empty() ? x.opt.storage_cap_Bps
                                                          : x.opt.storage_cap_per_engine[engine_];
  const double pace = x.opt.pace_scale;
  double gate_s = 0;  // emulated storage-NIC busy-until (FIFO token bucket), s since t0
  for (std::size_t i = 0; i < mine.size(); ++i) {
    const LoadJob& j = x.jobs[mine[i]];
    if (!peers_[j.pe]) throw std::runtime_error("run_step: PE " + std::to_string(j.pe) + " not attached");
    const std::int64_t bytes = j.cached * x.cfg.kv_bytes_per_token();
    const bool gated = cap > 0 || pace > 0;
    const bool hazard = !j.preds.empty();
    if (gated || hazard || j.fence || batch_pe != j.pe || batch.size() == DP_MAX_JOBS_PER_LAUNCH)
      flush();
    if (gated) {
      // StorageRead of C*L*b bytes over this engine's storage NIC: starts
      // when the NIC is free (and, replaying online, not before the planned
      // admission), takes bytes / cap
      const double begin = std::max(gate_s, pace > 0 ? j.t_admit * pace : 0.0);
      gate_s = begin + (cap > 0 ? static_cast<double>(bytes) / cap : 0.0);
      std::this_thread::sleep_until(t0 + std::chrono::duration<double>(gate_s));
      res.spans.push_back({begin, gate_s, bytes});
    }
    if (hazard) {
      const std::int64_t off = pred_off_[i];
      check(dp_wait_tickets(peers_[j.pe], d_pred_tickets_ + off, d_pred_targets_ + off,
                            static_cast<int32_t>(j.preds.size()), x.cfg.n_layer,
                            x.opt.wait_timeout_ms, s),
            "dp_wait_tickets");
      ++res.launches;
    }
    batch_pe = j.pe;
    if (k1_ce && j.pe == engine_)  // copy engine: host-readable block tables
      batch.push_back(dp_job{x.src_fb[engine_].data() + j.blk_off, x.slots[engine_].data() + j.blk_off,
                             j.cached, j.n_blk, 0, x.cfg.n_layer, j.ticket});
    else
      batch.push_back(dp_job{d_src_ + j.blk_off, d_slots_ + j.blk_off, j.cached, j.n_blk, 0,
                             x.cfg.n_layer, j.ticket});
    res.bytes_read += bytes;
    ++res.jobs;
  }
  flush();
  if (pool_ && n_wait_ > 0) {
    check(dp_wait_tickets(pool_, d_wait_tickets_, d_wait_targets_, n_wait_, x.cfg.n_layer,
                          x.opt.wait_timeout_ms, s),
          "dp_wait_tickets");
    ++res.launches;
  }
  check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_end_), s), "cudaEventRecord");
  check_cuda(cudaEventSynchronize(static_cast<cudaEvent_t>(ev_end_)), "step sync");
  for (dp_pool* p : peers_)
    if (p) check(dp_wait_status(p), "transfer watchdog");
  float ms = 0;
  check_cuda(cudaEventElapsedTime(&ms, static_cast<cudaEvent_t>(ev_start_),
                                  static_cast<cudaEvent_t>(ev_end_)),
             "cudaEventElapsedTime");
  res.device_ms = ms;
  res.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return res;
}

std::vector<std::uint64_t> EngineRuntime::checksum(int layer, std::span<const std::int32_t> slots,
                                                    std::span<const std::int32_t> ntok) {
  if (!pool_) throw std::logic_error("checksum: engine is not a PE");
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

std::vector<std::uint32_t> EngineRuntime::counters() const {
  if (!pool_) return {};
  DeviceScope ds(device_);
  void* base = nullptr;
  std::uint32_t* ctr = nullptr;
  std::int64_t bytes = 0;
  check(dp_pool_info(pool_, &base, &ctr, &bytes), "dp_pool_info");
  const std::size_t n = static_cast<std::size_t>(std::max<std::int32_t>(1, plan_->n_tickets[engine_])) *
                        (plan_->cfg.n_layer + 1);
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
