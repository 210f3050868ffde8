// Live-mode scheduling (include/dualpath/live.hpp): the reference's global
// scheduler (/root/reference/proj/src/desim.cpp:797-906) driven by real
// completions, the bytes moved by the C ABI's K1 / K2 on the GPUs (or by a
// timed backend for host-only tests).
#include "dualpath/live.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <mutex>
#include <queue>
#include <stdexcept>
#include <thread>
#include <unordered_map>

#include "dualpath/storage.hpp"
#include "engine_detail.hpp"
#include "pdsim/metrics.hpp"

namespace dualpath {
namespace {

using detail::check;
using detail::check_cuda;
using detail::DeviceScope;
using Clock = std::chrono::steady_clock;

struct Req {
  LiveRequest r;
  std::int64_t total() const { return r.cached + r.append + r.gen; }
  std::int32_t n_blk = 0;     // hit blocks ceil(C / T)
  std::int32_t n_pblk = 0;    // prompt blocks ceil((C + A) / T)
  std::int32_t n_tblk = 0;    // prompt + generated blocks ceil((C + A + G) / T)
  std::int32_t n_pe = 0;      // its PE-pool slots: n_pblk with the handoff, else n_blk
  std::int32_t n_de = 0;      // its decode-pool slots: n_tblk with persistence, else n_pblk
  std::int32_t n_tab = 0;     // its table entries: max(n_pe, n_de)
  std::int64_t tab_off = 0;   // its blocks in the slot / Full Block tables
};

struct Msg {
  enum Kind { ReadDone, Landed, Prefilled, Persisted } kind;
  int req;
};

// One DE's persistence (exec.persist): at a request's completion the decode
// stand-in writes its generated tokens into the decode pool and K4 persists
// them (64-token chunks + the final partial) into the DE's persist store; the
// decode-pool slots are freed when that is done.
struct Persister {
  int de = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<int> fifo;
  bool stop = false;
  std::thread th;
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  dp_stager* stager = nullptr;
  dp_store* store = nullptr;     // seed + 1: bytes never persisted differ from the content formula
  std::unique_ptr<FullBlockFile> file;  // exec.persist_path: PersistWrite into the storage tier
  std::int32_t* d_slot = nullptr;
  std::int64_t* d_fb = nullptr;
};

// One PE's prefill stand-in (exec.prefill): a FIFO of requests whose loads
// are launched, packed into forwards by build_forward_batch and run as K5
// layer by layer on the PE's compute stream, one forward at a time.
struct Computer {
  int pe = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<int> fifo;
  std::int64_t head_done = 0;  // query tokens of the head request already run
  bool stop = false;
  std::thread th;
  // gpu backend
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  std::int32_t* d_slot = nullptr;          // device copy of the block tables (by tab_off)
  std::uint64_t* d_digest = nullptr;       // [request][L]
  std::int32_t* h_wt = nullptr;            // mapped pinned: the forward's gate tickets
  std::uint32_t* h_wg = nullptr;           // ... and targets
};

// One reader engine's transfer pipeline: a FIFO worker (storage NIC, then
// the launch) and a completion thread (waits for each transfer in order).
struct Reader {
  int engine = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::deque<int> jobs;          // requests to read, FIFO
  std::deque<std::pair<int, cudaEvent_t>> inflight;
  std::deque<double> inflight_done;  // timed backend: completion times
  bool stop = false;
  bool worker_done = false;  // the completer drains in-flight transfers until then
  std::thread worker, completer;
};

class Live {
 public:
  Live(const pdsim::ClusterConfig& cfg, std::span<const pdsim::Trajectory> trajs, const LiveOptions& o)
      : cfg_(cfg), trajs_(trajs), o_(o) {
    cfg_.validate();
    g_ = cfg_.engines_per_node;
    n_pe_ = cfg_.prefill_nodes * g_;
    n_eng_ = cfg_.total_engines();
    tok_.assign(n_eng_, 0);
    seq_.assign(n_eng_, 0);
    hbm_free_.assign(n_eng_, cfg_.hbm_capacity_tokens);
    read_q_.assign(cfg_.prefill_nodes + cfg_.decode_nodes, 0);
    private_q_.assign(cfg_.prefill_nodes + cfg_.decode_nodes, {});
    next_round_.assign(trajs_.size(), 0);
    T_ = cfg_.block_size_tokens;
    L_ = cfg_.n_layer;
    // every turn of every session, ids in arrival order are assigned at arrival
    prefill_ = o_.exec.prefill;
    handoff_ = o_.exec.handoff;
    persist_ = o_.exec.persist;
    if (handoff_ && !prefill_) throw std::invalid_argument("run_live: exec.handoff needs exec.prefill");
    if (persist_ && !handoff_) throw std::invalid_argument("run_live: exec.persist needs exec.handoff");
    std::int64_t max_blk = 1, total_blk = 0;
    for (const auto& t : trajs_) {
      fb_stride_ = std::max(fb_stride_, pdsim::blocks_for(t.total_tokens(), cfg_));
      for (std::size_t k = 0; k < t.rounds.size(); ++k) {
        const std::int64_t c = pdsim::context_before(t, k) + (handoff_ ? t.rounds[k].append_tokens : 0) +
                               (persist_ ? t.rounds[k].gen_tokens : 0);
        const std::int64_t nb = (c + T_ - 1) / T_;
        max_blk = std::max(max_blk, nb);
        total_blk += nb;
        ++total_reqs_;
      }
    }
    reqs_.reserve(static_cast<std::size_t>(total_reqs_));  // workers hold references: never reallocate
    pool_slots_ = o_.pe_pool_slots > 0 ? o_.pe_pool_slots : static_cast<std::int32_t>(4 * max_blk);
    if (pool_slots_ < max_blk)
      throw pdsim::desim::ConfigError("run_live: pe_pool_slots smaller than the largest request");
    const std::int64_t fbb = cfg_.full_block_bytes();
    store_fb_ = std::max<std::int64_t>(
        1, std::min<std::int64_t>(fb_stride_ * static_cast<std::int64_t>(std::max<std::size_t>(1, trajs_.size())),
                                  o_.exec.store_bytes_max / fbb));
    free_slots_.assign(n_pe_, {});
    for (int p = 0; p < n_pe_; ++p)
      for (std::int32_t s = pool_slots_ - 1; s >= 0; --s) free_slots_[p].push_back(s);
    occupant_.assign(static_cast<std::size_t>(n_pe_) * pool_slots_, {-1, 0});
    if (handoff_) {  // decode pools: each DE holds the whole prompt of the requests it decodes
      de_slots_ = o_.de_pool_slots > 0 ? o_.de_pool_slots : static_cast<std::int32_t>(4 * max_blk);
      if (de_slots_ < max_blk)
        throw pdsim::desim::ConfigError("run_live: de_pool_slots smaller than the largest prompt");
      free_de_.assign(n_eng_ - n_pe_, {});
      for (auto& fl : free_de_)
        for (std::int32_t s = de_slots_ - 1; s >= 0; --s) fl.push_back(s);
      de_occupant_.assign(static_cast<std::size_t>(n_eng_ - n_pe_) * de_slots_, {-1, 0});
    }
    reader_bytes_.assign(n_eng_, 0);
    if (prefill_) {
      if (!(o_.exec.compute_quota > 0)) throw std::invalid_argument("run_live: exec.compute_quota must be > 0");
      for (int p = 0; p < n_pe_; ++p) {
        computers_.push_back(std::make_unique<Computer>());
        computers_.back()->pe = p;
      }
    }
    if (persist_)
      for (int d = 0; d < n_eng_ - n_pe_; ++d) {
        persisters_.push_back(std::make_unique<Persister>());
        persisters_.back()->de = d;
      }
    if (o_.gpu) setup_gpu(total_blk);
    else {
      tab_slot_h_ = new std::int32_t[std::max<std::int64_t>(1, total_blk)];
      tab_fb_h_ = new std::int64_t[std::max<std::int64_t>(1, total_blk)];
      tab_de_h_ = new std::int32_t[std::max<std::int64_t>(1, total_blk)];
    }
    for (int e = 0; e < n_eng_; ++e) {
      dp_nic* nic = nullptr;
      const double cap = o_.exec.storage_cap_per_engine.empty() ? o_.exec.storage_cap_Bps
                                                                : o_.exec.storage_cap_per_engine.at(e);
      check(dp_nic_create(cap, &nic), "dp_nic_create");
      nics_.push_back(nic);
    }
  }

  // Stop every reader: reads not yet started are dropped (a stopped online
  // run), transfers already launched are waited for before the pools go.
  void shutdown_readers() {
    for (auto& r : readers_) {
      {
        std::lock_guard<std::mutex> lk(r->mu);
        r->jobs.clear();
        r->stop = true;
      }
      r->cv.notify_all();
      if (r->worker.joinable()) r->worker.join();
      {
        std::lock_guard<std::mutex> lk(r->mu);
        r->worker_done = true;
      }
      r->cv.notify_all();
      if (r->completer.joinable()) r->completer.join();
    }
    readers_.clear();
  }

  void shutdown_computers() {
    for (auto& c : computers_) {
      {
        std::lock_guard<std::mutex> lk(c->mu);
        c->stop = true;
      }
      c->cv.notify_all();
      if (c->th.joinable()) c->th.join();
    }
  }

  void shutdown_persisters() {
    for (auto& p : persisters_) {
      {
        std::lock_guard<std::mutex> lk(p->mu);
        p->stop = true;
      }
      p->cv.notify_all();
      if (p->th.joinable()) p->th.join();
    }
  }

  ~Live() {
    shutdown_readers();
    shutdown_computers();
    shutdown_persisters();
    for (auto& p : persisters_) {
      if (p->done) cudaEventDestroy(p->done);
      if (p->stager) dp_stager_destroy(p->stager);
      if (p->store) dp_store_destroy(p->store);
      if (p->stream) detail::release_stream(devs_[n_pe_ + p->de], p->stream);
    }
    for (auto& c : computers_) {
      if (c->done) cudaEventDestroy(c->done);
      if (c->d_slot) cudaFree(c->d_slot);
      if (c->d_digest) cudaFree(c->d_digest);
      if (c->h_wt) cudaFreeHost(c->h_wt);
      if (c->h_wg) cudaFreeHost(c->h_wg);
      if (c->stream) detail::release_stream(devs_[c->pe], c->stream);
    }
    for (dp_nic* n : nics_) dp_nic_destroy(n);
    for (dp_stager* s : stagers_) dp_stager_destroy(s);
    for (auto& row : views_)
      for (dp_pool* v : row)
        if (v) dp_pool_destroy(v);
    for (dp_pool* p : pools_) dp_pool_destroy(p);
    for (dp_store* s : stores_) dp_store_destroy(s);
    for (std::size_t e = 0; e < streams_.size(); ++e)
      if (streams_[e]) detail::release_stream(devs_[e], streams_[e]);
    for (auto& row : de_views_)
      for (dp_pool* v : row)
        if (v) dp_pool_destroy(v);
    for (dp_pool* p : de_pools_) dp_pool_destroy(p);
    if (o_.gpu) {
      if (tab_slot_h_) cudaFreeHost(tab_slot_h_);
      if (tab_fb_h_) cudaFreeHost(tab_fb_h_);
      if (tab_de_h_) cudaFreeHost(tab_de_h_);
    } else {
      delete[] tab_slot_h_;
      delete[] tab_fb_h_;
      delete[] tab_de_h_;
    }
  }

  LiveReport run() {
    t0_ = Clock::now();
    for (dp_nic* n : nics_) check(dp_nic_start(n), "dp_nic_start");
    for (int e = 0; e < n_eng_; ++e) {
      readers_.push_back(std::make_unique<Reader>());
      Reader* rd = readers_.back().get();
      rd->engine = e;
      rd->worker = std::thread([this, rd] { worker(rd); });
      rd->completer = std::thread([this, rd] { completer(rd); });
    }
    for (auto& c : computers_) {
      Computer* cp = c.get();
      cp->th = std::thread([this, cp] { compute(cp); });
    }
    for (auto& ps : persisters_) {
      Persister* pp = ps.get();
      pp->th = std::thread([this, pp] { persist_loop(pp); });
    }
    if (!o_.arrival_times.empty() && o_.arrival_times.size() != trajs_.size())
      throw std::invalid_argument("run_live: one arrival time per trajectory");
    for (std::size_t t = 0; t < trajs_.size(); ++t) {
      const double at = o_.arrival_times.empty() ? 0.0 : o_.arrival_times[t];
      if (at <= 0) arrive(static_cast<int>(t));
      else timers_.push({at, -1 - static_cast<int>(t)});  // a session's first turn
    }
    if (o_.steady_window > 0) next_steady_ = o_.steady_window / 2;
    wake();
    auto last_progress = Clock::now();
    while ((completed_ < total_reqs_ || (persist_ && persisted_ < completed_)) && !stop_) {
      std::vector<Msg> msgs;
      {
        std::unique_lock<std::mutex> lk(mu_);
        const auto until = timers_.empty() ? Clock::now() + std::chrono::milliseconds(200)
                                           : t0_ + std::chrono::duration_cast<Clock::duration>(
                                                       std::chrono::duration<double>(timers_.top().first));
        cv_.wait_until(lk, until, [this] { return !msgs_.empty() || !worker_error_.empty(); });
        if (!worker_error_.empty()) throw std::runtime_error("run_live: " + worker_error_);
        msgs.swap(msgs_);
      }
      const bool progress = !msgs.empty();
      for (const Msg& m : msgs) handle(m);
      while (!timers_.empty() && timers_.top().first <= now()) {
        const int id = timers_.top().second;
        timers_.pop();
        if (id < 0) arrive(-1 - id);  // online arrival of a session
        else complete(id);
      }
      if (next_steady_ > 0 && now() >= next_steady_ && !stop_) {  // on_steady_check (desim.cpp:942-953)
        if (pdsim::detect_steady_state(rep_.ttft_series, o_.steady_window, o_.steady_lookback,
                                       o_.steady_threshold)) {
          rep_.steady_state = true;
          stop_ = true;
        }
        next_steady_ = now() + o_.steady_window / 2;
      }
      if (stop_) break;
      wake();
      if (progress) last_progress = Clock::now();
      if (std::chrono::duration<double>(Clock::now() - last_progress).count() > o_.timeout_s)
        throw std::runtime_error("run_live: no progress for " + std::to_string(o_.timeout_s) + " s");
    }
    rep_.wall_s = now();
    shutdown_readers();
    shutdown_computers();
    shutdown_persisters();
    if (o_.gpu && !stop_) final_occupants();
    if (o_.gpu && prefill_) final_digests();
    rep_.forwards = forwards_;
    for (auto& q : reqs_) rep_.requests.push_back(q.r);
    rep_.reader_bytes = reader_bytes_;
    rep_.pool_slots = pool_slots_;
    rep_.store_fb = store_fb_;
    rep_.fb_stride = fb_stride_;
    rep_.completed_requests = static_cast<std::size_t>(completed_);
    rep_.total_requests = static_cast<std::size_t>(total_reqs_);
    return std::move(rep_);
  }

 private:
  double now() const { return std::chrono::duration<double>(Clock::now() - t0_).count(); }
  int node_of(int e) const { return e / g_; }
  bool is_pe(int e) const { return e < n_pe_; }
  std::int64_t fb_of(int traj, std::int64_t k) const { return (traj * fb_stride_ + k) % store_fb_; }

  void post(Msg m) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      msgs_.push_back(m);
    }
    cv_.notify_one();
  }
  void fail_async(const std::string& what) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (worker_error_.empty()) worker_error_ = what;
    }
    cv_.notify_one();
  }

  // ---- the reference's request life cycle, on measured events ----------
  void arrive(int t) {  // on_arrival (desim.cpp:551-566)
    const pdsim::Trajectory& tr = trajs_[t];
    const int round = next_round_[t]++;
    Req q;
    q.r.id = static_cast<int>(reqs_.size());
    q.r.traj = t;
    q.r.round = round;
    q.r.cached = pdsim::context_before(tr, static_cast<std::size_t>(round));
    q.r.append = tr.rounds[round].append_tokens;
    q.r.gen = tr.rounds[round].gen_tokens;
    q.r.t_arrival = now();
    q.n_blk = static_cast<std::int32_t>((q.r.cached + T_ - 1) / T_);
    q.n_pblk = static_cast<std::int32_t>((q.r.cached + q.r.append + T_ - 1) / T_);
    q.n_tblk = static_cast<std::int32_t>((q.r.cached + q.r.append + q.r.gen + T_ - 1) / T_);
    q.n_pe = handoff_ ? q.n_pblk : q.n_blk;
    q.n_de = persist_ ? q.n_tblk : handoff_ ? q.n_pblk : 0;
    q.n_tab = std::max(q.n_pe, q.n_de);
    q.tab_off = tab_used_;
    tab_used_ += q.n_tab;
    reqs_.push_back(q);
    de_global_.push_back(q.r.id);
    arrived_in_wake_ = true;
  }

  pdsim::EngineSnapshot snapshot_of(int e) const {  // desim.cpp:797-807
    pdsim::EngineSnapshot s;
    s.engine_id = e;
    s.node_id = node_of(e);
    s.kind = is_pe(e) ? pdsim::EngineKind::PE : pdsim::EngineKind::DE;
    s.seq_e = seq_[e];
    s.tok_e = tok_[e];
    s.read_q = read_q_[node_of(e)];
    s.hbm_free_tokens = hbm_free_[e];
    return s;
  }

  void assign_de(Req& q, int de, int cat) {  // desim.cpp:809-817
    q.r.de = de;
    de_cat_[q.r.id] = cat;
    tok_[de] += q.total();
    seq_[de] += 1;
    hbm_free_[de] -= q.total();
    pe_waiting_.push_back(q.r.id);
  }

  void assign_pe(Req& q, int pe, int cat) {  // desim.cpp:819-849
    q.r.pe = pe;
    tok_[pe] += q.total();
    seq_[pe] += 1;
    q.r.t_sched = now();
    pdsim::ReadPath path;
    const auto& pol = o_.sim;
    if (pol.policy == pdsim::desim::Policy::PEOnly) {
      path = pdsim::ReadPath::PEPath;
    } else if (pol.sched_mode == pdsim::desim::SchedMode::RoundRobin) {
      path = (rr_path_++ % 2 == 0) ? pdsim::ReadPath::PEPath : pdsim::ReadPath::DEPath;
    } else {
      const std::int64_t a = read_q_[node_of(q.r.pe)], b = read_q_[node_of(q.r.de)];
      path = pdsim::select_read_path(a, b);
      LiveInvocation inv;
      inv.fn = "select_read_path";
      inv.t = now();
      inv.pe_read_q = a;
      inv.de_read_q = b;
      inv.path = path == pdsim::ReadPath::PEPath ? 0 : 1;
      rep_.invocations.push_back(std::move(inv));
    }
    q.r.path = path == pdsim::ReadPath::PEPath ? 0 : 1;
    q.r.reader = q.r.path == 0 ? q.r.pe : q.r.de;
    if (q.r.cached > 0 && pol.policy != pdsim::desim::Policy::Oracle) read_q_[node_of(q.r.reader)] += q.r.cached;
    admission_.push_back(q.r.id);
    rep_.decisions.push_back({q.r.t_sched, q.r.id, q.r.pe, q.r.de, path, cat, de_cat_[q.r.id]});
  }

  void schedule_adaptive() {  // desim.cpp:865-906
    if (!de_global_.empty()) {
      std::vector<pdsim::GroupLoad> groups;
      for (int n = cfg_.prefill_nodes; n < cfg_.prefill_nodes + cfg_.decode_nodes; ++n) {
        pdsim::GroupLoad gl{n, 0};
        for (int k = 0; k < g_; ++k) gl.tok_sum += tok_[n * g_ + k];
        for (int id : private_q_[n]) gl.tok_sum += reqs_[id].total();
        groups.push_back(gl);
      }
      std::vector<pdsim::PendingRequest> pending;
      for (int id : de_global_) pending.push_back({id, reqs_[id].total()});
      const auto out = pdsim::schedule_de_groups(pending, groups);
      LiveInvocation inv;
      inv.fn = "schedule_de_groups";
      inv.t = now();
      inv.queue = pending;
      inv.groups = groups;
      for (const auto& [req, group] : out) {
        private_q_[group].push_back(req);
        inv.out.push_back({req, group, 0});
      }
      rep_.invocations.push_back(std::move(inv));
      de_global_.clear();
    }
    for (int n = cfg_.prefill_nodes; n < cfg_.prefill_nodes + cfg_.decode_nodes; ++n) {
      auto& q = private_q_[n];
      if (q.empty()) continue;
      std::vector<pdsim::PendingRequest> pending;
      for (int id : q) pending.push_back({id, reqs_[id].total()});
      std::vector<pdsim::EngineSnapshot> snaps;
      for (int k = 0; k < g_; ++k) snaps.push_back(snapshot_of(n * g_ + k));
      const auto asg = pdsim::schedule_de_within_group(pending, snaps, o_.sim.sched);
      LiveInvocation inv;
      inv.fn = "schedule_de_within_group";
      inv.t = now();
      inv.queue = pending;
      inv.snapshots = snaps;
      inv.out = asg;
      rep_.invocations.push_back(std::move(inv));
      for (const auto& a : asg) assign_de(reqs_[a.request_id], a.engine_id, a.category);
      q.erase(q.begin(), q.begin() + static_cast<std::ptrdiff_t>(asg.size()));
    }
    if (!pe_waiting_.empty()) {
      std::vector<pdsim::PendingRequest> pending;
      for (int id : pe_waiting_) pending.push_back({id, reqs_[id].total()});
      std::vector<pdsim::EngineSnapshot> snaps;
      for (int e = 0; e < n_pe_; ++e) snaps.push_back(snapshot_of(e));
      const auto asg = pdsim::schedule_pe_fetch(pending, snaps, o_.sim.sched);
      LiveInvocation inv;
      inv.fn = "schedule_pe_fetch";
      inv.t = now();
      inv.queue = pending;
      inv.snapshots = snaps;
      inv.out = asg;
      rep_.invocations.push_back(std::move(inv));
      for (const auto& a : asg) assign_pe(reqs_[a.request_id], a.engine_id, a.category);
      pe_waiting_.erase(pe_waiting_.begin(), pe_waiting_.begin() + static_cast<std::ptrdiff_t>(asg.size()));
    }
  }

  void schedule_round_robin() {  // desim.cpp:908-933
    while (!de_global_.empty()) {
      Req& q = reqs_[de_global_.front()];
      const int n_de = n_eng_ - n_pe_;
      int chosen = -1;
      for (int i = 0; i < n_de; ++i) {
        const int e = n_pe_ + (rr_de_ + i) % n_de;
        if (hbm_free_[e] >= q.total()) {
          chosen = e;
          rr_de_ = (rr_de_ + i + 1) % n_de;
          break;
        }
      }
      if (chosen < 0) break;
      de_global_.pop_front();
      assign_de(q, chosen, 0);
    }
    while (!pe_waiting_.empty()) {
      Req& q = reqs_[pe_waiting_.front()];
      pe_waiting_.pop_front();
      const int pe = rr_pe_ % n_pe_;
      rr_pe_ = (rr_pe_ + 1) % n_pe_;
      assign_pe(q, pe, 0);
    }
  }

  void wake() {  // scheduler_wake (desim.cpp:851-863)
    // a cold turn lands at its admission and its session's next turn arrives
    // at once: schedule again until no arrival is left waiting
    do {
      wake_once();
    } while (!de_global_.empty() && !stop_ && arrived_in_wake_);
  }

  void wake_once() {
    arrived_in_wake_ = false;
    if (o_.sim.sched_mode == pdsim::desim::SchedMode::Adaptive) schedule_adaptive();
    else schedule_round_robin();
    // admission pass, FIFO; PEs progress independently.  The bounded
    // resource is the PE's paged pool: a request waits for its blocks.
    bool stalled = false;
    for (auto it = admission_.begin(); it != admission_.end();) {
      Req& q = reqs_[*it];
      auto& fl = free_slots_[q.r.pe];
      auto* dl = handoff_ ? &free_de_[q.r.de - n_pe_] : nullptr;
      if (static_cast<std::int64_t>(fl.size()) < q.n_pe ||
          (dl && static_cast<std::int64_t>(dl->size()) < q.n_de)) {
        stalled = true;
        ++it;
        continue;
      }
      // the PE pool holds the hit KV, with the handoff the whole prompt (the
      // prefill writes the miss KV there); the DE's decode pool the prompt
      const std::int64_t held = handoff_ ? q.r.cached + q.r.append : q.r.cached;
      const std::int64_t de_held = persist_ ? q.total() : held;  // the decode pool ends with the generated tokens
      for (std::int32_t k = 0; k < q.n_tab; ++k) {
        tab_fb_h_[q.tab_off + k] = fb_of(q.r.traj, k);
        if (k < q.n_pe) {
          const std::int32_t s = fl.back();
          fl.pop_back();
          tab_slot_h_[q.tab_off + k] = s;
          const auto ntok = static_cast<std::int32_t>(std::min<std::int64_t>(T_, held - k * T_));
          occupant_[static_cast<std::size_t>(q.r.pe) * pool_slots_ + s] = {tab_fb_h_[q.tab_off + k], ntok};
        }
        if (dl && k < q.n_de) {
          const std::int32_t d = dl->back();
          dl->pop_back();
          tab_de_h_[q.tab_off + k] = d;
          const auto ntok = static_cast<std::int32_t>(std::min<std::int64_t>(T_, de_held - k * T_));
          de_occupant_[static_cast<std::size_t>(q.r.de - n_pe_) * de_slots_ + d] = {tab_fb_h_[q.tab_off + k], ntok};
        }
      }
      q.r.t_admit = now();
      const int id = q.r.id;
      it = admission_.erase(it);
      if (q.r.cached == 0) {  // no hit KV: nothing to read (desim.cpp:709)
        q.r.t_read_done = q.r.t_landed = q.r.t_admit;
        if (prefill_) to_compute(q);
        else handle({Msg::Landed, id});
        continue;
      }
      Reader* rd = readers_[q.r.reader].get();
      {
        std::lock_guard<std::mutex> lk(rd->mu);
        rd->jobs.push_back(id);
      }
      rd->cv.notify_all();
    }
    if (stalled) ++rep_.admission_stalls;
  }

  void free_de_slots(const Req& q) {
    auto& dl = free_de_[q.r.de - n_pe_];
    for (std::int32_t k = 0; k < q.n_de; ++k) dl.push_back(tab_de_h_[q.tab_off + k]);
  }

  void handle(const Msg& m) {
    Req& q = reqs_[m.req];
    if (m.kind == Msg::Persisted) {
      free_de_slots(q);
      ++persisted_;
      return;
    }
    if (m.kind == Msg::ReadDone) {  // complete_stage(StorageRead): read_q -= C (desim.cpp:702-704)
      q.r.t_read_done = now();
      if (o_.sim.policy != pdsim::desim::Policy::Oracle) read_q_[node_of(q.r.reader)] -= q.r.cached;
      return;
    }
    if (m.kind == Msg::Landed) {
      if (q.r.t_landed < 0) q.r.t_landed = now();
      if (prefill_) {  // the PE holds the request until its prefill is done
        if (!o_.gpu) to_compute(q);  // timed backend: no counters to gate on
        return;
      }
    } else {
      q.r.t_prefilled = now();
    }
    // the load path's PE release at landing, or with the prefill at its end
    // (on_prefill_side_done, desim.cpp:642-652)
    const double t_rel = prefill_ ? q.r.t_prefilled : q.r.t_landed;
    // with the handoff the prompt is in the DE's decode pool at t_rel (the
    // DecodeH2D is done): the first token follows one decode step
    // (on_decode_token k = 1, desim.cpp:679-685)
    const double t_tok = handoff_ ? t_rel + o_.decode_s_per_token : t_rel;
    const double ttft = t_tok - q.r.t_arrival;
    rep_.ttft_series.emplace_back(t_tok, ttft);
    if (o_.slo_ttft_s > 0 && ttft > o_.slo_ttft_s) {  // the SLO stop (desim.cpp:679-685)
      rep_.slo_violated = true;
      stop_ = true;
    }
    tok_[q.r.pe] -= q.total();
    seq_[q.r.pe] -= 1;
    auto& fl = free_slots_[q.r.pe];
    for (std::int32_t k = 0; k < q.n_pe; ++k) fl.push_back(tab_slot_h_[q.tab_off + k]);
    if (o_.decode_s_per_token > 0)
      timers_.push({now() + static_cast<double>(q.r.gen) * o_.decode_s_per_token, q.r.id});
    else
      complete(q.r.id);
  }

  void complete(int id) {  // request done on its DE (desim.cpp:776-787), then the next turn
    Req& q = reqs_[id];
    q.r.t_done = now();
    if (persist_) {  // its generated tokens to storage; the slots are freed once persisted
      Persister* ps = persisters_[q.r.de - n_pe_].get();
      {
        std::lock_guard<std::mutex> lk(ps->mu);
        ps->fifo.push_back(q.r.id);
      }
      ps->cv.notify_all();
    } else if (handoff_) {  // the decode pool's slots are free once the request is done
      free_de_slots(q);
    }
    tok_[q.r.de] -= q.total();
    seq_[q.r.de] -= 1;
    hbm_free_[q.r.de] += q.total();
    ++completed_;
    if (next_round_[q.r.traj] < static_cast<int>(trajs_[q.r.traj].rounds.size())) arrive(q.r.traj);
  }

  // ---- reader threads ---------------------------------------------------
  void worker(Reader* rd) {
    const int e = rd->engine;
    try {
      if (o_.gpu) check_cuda(cudaSetDevice(devs_[e]), "cudaSetDevice");
      for (;;) {
        int id;
        {
          std::unique_lock<std::mutex> lk(rd->mu);
          rd->cv.wait(lk, [rd] { return rd->stop || !rd->jobs.empty(); });
          if (rd->jobs.empty()) return;
          id = rd->jobs.front();
          rd->jobs.pop_front();
        }
        const Req& q = reqs_[id];  // fields read here are fixed once admitted
        const std::int64_t bytes = q.r.cached * cfg_.kv_bytes_per_token();
        check(dp_nic_read(nics_[e], bytes, 0.0, nullptr, nullptr), "dp_nic_read");  // StorageRead
        post({Msg::ReadDone, id});
        reader_bytes_[e] += bytes;
        cudaEvent_t ev = nullptr;
        if (o_.gpu) ev = launch(e, q);
        {
          std::lock_guard<std::mutex> lk(rd->mu);
          rd->inflight.emplace_back(id, ev);
          if (!o_.gpu) {
            const double start = std::max(now(), rd->inflight_done.empty() ? 0.0 : rd->inflight_done.back());
            rd->inflight_done.push_back(start + static_cast<double>(bytes) / o_.link_Bps);
          }
        }
        rd->cv.notify_all();
        if (prefill_ && o_.gpu) to_compute(q);  // launched: the forwards gate on its landed counters
      }
    } catch (const std::exception& ex) {
      fail_async(ex.what());
    }
  }

  void to_compute(const Req& q) {
    Computer* c = computers_[q.r.pe].get();
    {
      std::lock_guard<std::mutex> lk(c->mu);
      c->fifo.push_back(q.r.id);
    }
    c->cv.notify_all();
  }

  // ---- prefill stand-in (exec.prefill) ---------------------------------
  void compute(Computer* c) {
    try {
      if (o_.gpu) check_cuda(cudaSetDevice(devs_[c->pe]), "cudaSetDevice");
      pdsim::SchedulerParams sp;
      sp.compute_quota = o_.exec.compute_quota;
      std::vector<pdsim::BatchItem> window;
      std::vector<dp_attend_item> att;
      for (;;) {
        std::int64_t head_done;
        {
          std::unique_lock<std::mutex> lk(c->mu);
          c->cv.wait(lk, [c] { return c->stop || !c->fifo.empty(); });
          if (c->stop) return;
          window.clear();
          for (std::size_t i = 0; i < c->fifo.size(); ++i) {
            const Req& q = reqs_[c->fifo[i]];
            window.push_back({q.r.id, q.r.cached, q.r.append - (i == 0 ? c->head_done : 0)});
          }
          head_done = c->head_done;
        }
        const pdsim::ForwardBatch fb = pdsim::build_forward_batch(window, sp, o_.exec.prefill_cost);
        if (o_.gpu) {
          run_forward(c, fb, head_done, att);
        } else {
          double ho = 0;  // the handoff of the requests this forward finishes
          for (std::int64_t k = 0; handoff_ && k < fb.consumed_whole; ++k) {
            const Req& q = reqs_[fb.items[k].request_id];
            ho += static_cast<double>((q.r.path == 0 ? q.r.cached : 0) + q.r.append) * cfg_.kv_bytes_per_token();
          }
          std::this_thread::sleep_for(std::chrono::duration<double>(fb.estimated_time * L_ + ho / o_.link_Bps));
        }
        std::vector<int> finished;
        {
          std::lock_guard<std::mutex> lk(c->mu);
          for (std::size_t k = 0; k < fb.items.size(); ++k) ++reqs_[fb.items[k].request_id].r.forwards;
          for (std::int64_t k = 0; k < fb.consumed_whole; ++k) {
            finished.push_back(c->fifo.front());
            c->fifo.pop_front();
          }
          if (fb.chunked)
            c->head_done = fb.consumed_whole == 0 ? c->head_done + fb.chunk_bsz : fb.chunk_bsz;
          else
            c->head_done = 0;
        }
        forwards_ += 1;
        for (int id : finished) post({Msg::Prefilled, id});
      }
    } catch (const std::exception& ex) {
      fail_async(ex.what());
    }
  }

  // ---- persistence (exec.persist) --------------------------------------
  void persist_loop(Persister* ps) {
    try {
      if (o_.gpu) check_cuda(cudaSetDevice(devs_[n_pe_ + ps->de]), "cudaSetDevice");
      for (;;) {
        int id;
        {
          std::unique_lock<std::mutex> lk(ps->mu);
          ps->cv.wait(lk, [ps] { return ps->stop || !ps->fifo.empty(); });
          if (ps->stop) return;
          id = ps->fifo.front();
          ps->fifo.pop_front();
        }
        const Req& q = reqs_[id];
        if (o_.gpu) {
          persist_gpu(ps, q);
        } else {
          const double bytes = static_cast<double>(q.r.gen) * cfg_.kv_bytes_per_token();
          std::this_thread::sleep_for(std::chrono::duration<double>(bytes / o_.link_Bps));
        }
        post({Msg::Persisted, id});
      }
    } catch (const std::exception& ex) {
      fail_async(ex.what());
    }
  }

  // The decode stand-in writes the generated tokens [P, P + G) into the
  // decode pool, staged K4 persists them in the reference's chunks (every 64
  // generated tokens + the final partial, desim.cpp:658-661, :690-693, :760)
  // into the DE's persist store; then the persisted ranges of layers 0 and
  // L-1 are hashed for the report (parity vs the oracle).
  void persist_gpu(Persister* ps, const Req& q) {
    const std::int64_t P = q.r.cached + q.r.append, G = q.r.gen;
    if (G <= 0) return;
    const std::int64_t blk0 = P / T_;
    const std::int32_t nb = q.n_tblk - static_cast<std::int32_t>(blk0);
    dp_pool* pool = de_pools_[ps->de];
    const dp_span_job fill{tab_de_h_ + q.tab_off + blk0, tab_fb_h_ + q.tab_off + blk0, blk0, P, P + G, nb, 0};
    check(dp_decode_fill(pool, &fill, 1, o_.exec.seed, ps->stream), "dp_decode_fill");
    std::vector<dp_span_job> chunks;
    std::int64_t done = 0;
    for (std::int64_t k = T_; k < G; k += T_) {
      chunks.push_back({fill.slot, fill.fb, blk0, P + done, P + k, nb, 0});
      done = k;
    }
    chunks.push_back({fill.slot, fill.fb, blk0, P + done, P + G, nb, 0});
    check(dp_persist_staged(pool, ps->store, ps->stager, chunks.data(), static_cast<std::int32_t>(chunks.size()),
                            ps->stream),
          "dp_persist_staged");
    check_cuda(cudaEventRecord(ps->done, ps->stream), "cudaEventRecord");
    check_cuda(cudaEventSynchronize(ps->done), "persist sync");
    void* host = nullptr;
    std::int64_t bytes = 0, n_fb = 0;
    check(dp_store_info(ps->store, &host, &bytes, &n_fb), "dp_store_info");
    const std::int64_t b = cfg_.kv_bytes_per_token_per_layer, lb = T_ * b, fbb = lb * L_;
    std::vector<LiveReport::Persisted> out;
    std::int64_t written = 0;
    for (std::int32_t i = 0; i < nb; ++i) {
      const std::int64_t k = blk0 + i;
      const std::int64_t t0 = std::max(P, k * T_) - k * T_, t1 = std::min(P + G, (k + 1) * T_) - k * T_;
      if (t1 <= t0) continue;
      const std::int64_t fb = tab_fb_h_[q.tab_off + k];
      if (ps->file)  // PersistWrite (desim.cpp:764-771): the generated tokens into the block's record
        for (std::int32_t layer = 0; layer < L_; ++layer) {
          const std::int64_t off = layer * lb + t0 * b;
          ps->file->write_bytes(fb, off, (t1 - t0) * b, static_cast<const char*>(host) + fb * fbb + off);
          written += (t1 - t0) * b;
        }
      for (std::int32_t layer : {0, L_ - 1}) {
        const auto* w = reinterpret_cast<const std::uint64_t*>(static_cast<const char*>(host) + fb * fbb +
                                                               layer * lb + t0 * b);
        out.push_back({q.r.id, fb, layer, static_cast<std::int32_t>(t0), static_cast<std::int32_t>(t1),
                       range_hash(w, (t1 - t0) * b / 8)});
      }
    }
    std::lock_guard<std::mutex> lk(persist_mu_);
    rep_.persisted.insert(rep_.persisted.end(), out.begin(), out.end());
    rep_.persist_write_bytes += written;
  }

  // H = sum_i splitmix64(word_i + (i + 1) * golden) (mod 2^64): the hash of
  // dp_pool_checksum over a byte range (the test restates it)
  static std::uint64_t range_hash(const std::uint64_t* w, std::int64_t n) {
    std::uint64_t h = 0;
    for (std::int64_t i = 0; i < n; ++i) {
      std::uint64_t z = w[i] + static_cast<std::uint64_t>(i + 1) * 0x9E3779B97F4A7C15ull + 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      h += z ^ (z >> 31);
    }
    return h;
  }

  // One forward: the block tables of its requests to the device, then per
  // layer the gate on the landed counters of the requests it reads first and
  // K5 over its items; waits for the forward to finish.
  void run_forward(Computer* c, const pdsim::ForwardBatch& fb, std::int64_t head_done,
                   std::vector<dp_attend_item>& att) {
    att.clear();
    std::int32_t n_gate = 0;
    for (std::size_t k = 0; k < fb.items.size(); ++k) {
      const Req& q = reqs_[fb.items[k].request_id];
      dp_attend_item a{};
      a.cached = q.r.cached;
      a.q_begin = k == 0 ? head_done : 0;
      a.bsz = fb.items[k].bsz;
      a.digest = c->d_digest + static_cast<std::int64_t>(q.r.id) * L_;
      a.req = static_cast<std::uint32_t>(q.r.id);
      a.slot = c->d_slot + q.tab_off;
      if (a.q_begin == 0 && q.n_blk > 0) {  // read here first: its table, and a gate on its KV
        check_cuda(cudaMemcpyAsync(c->d_slot + q.tab_off, tab_slot_h_ + q.tab_off, q.n_blk * sizeof(std::int32_t),
                                   cudaMemcpyHostToDevice, c->stream),
                   "cudaMemcpyAsync block table");
        if (n_gate >= kMaxGates) throw std::runtime_error("run_live: more gated requests in a forward than the gate table");
        c->h_wt[n_gate] = q.r.id;
        c->h_wg[n_gate] = static_cast<std::uint32_t>(q.n_blk) * items_per_block_;
        ++n_gate;
      }
      att.push_back(a);
    }
    for (std::int32_t l = 0; l < L_; ++l) {
      if (n_gate > 0)
        check(dp_wait_tickets(pools_[c->pe], c->h_wt, c->h_wg, n_gate, l, o_.exec.wait_timeout_ms, c->stream),
              "dp_wait_tickets (forward gate)");
      check(dp_prefill_attend(pools_[c->pe], l, att.data(), static_cast<std::int32_t>(att.size()), o_.exec.seed,
                              c->stream),
            "dp_prefill_attend");
    }
    if (handoff_) {
      // PeToDe / MissMerge of the requests this forward finishes (K3, after
      // the forward on its stream): the whole prompt into the DE's decode
      // pool, the PE path pushing the hit KV too (desim.cpp:630-652)
      std::vector<std::vector<dp_handoff_job>> by_de(n_eng_ - n_pe_);
      for (std::int64_t k = 0; k < fb.consumed_whole; ++k) {
        const Req& q = reqs_[fb.items[k].request_id];
        if (q.n_pblk == 0) continue;
        by_de[q.r.de - n_pe_].push_back(dp_handoff_job{tab_fb_h_ + q.tab_off, tab_slot_h_ + q.tab_off,
                                                       tab_de_h_ + q.tab_off, q.r.cached, q.r.cached + q.r.append,
                                                       q.n_pblk, q.r.path == 0 ? 1 : 0, -1, 0, q.r.id, -1});
      }
      for (std::size_t d = 0; d < by_de.size(); ++d) {
        if (by_de[d].empty()) continue;
        dp_pool* view = de_views_[c->pe][d];
        const auto n = static_cast<std::int32_t>(by_de[d].size());
        check(o_.exec.k3_mode == 1
                  ? dp_prefill_handoff_copy(pools_[c->pe], view, by_de[d].data(), n, o_.exec.seed,
                                            o_.exec.wait_timeout_ms, c->stream)
                  : dp_prefill_handoff(pools_[c->pe], view, by_de[d].data(), n, o_.exec.seed,
                                       o_.exec.wait_timeout_ms, c->stream),
              "prefill handoff (K3)");
      }
    }
    check_cuda(cudaEventRecord(c->done, c->stream), "cudaEventRecord");
    check_cuda(cudaEventSynchronize(c->done), "forward sync");
    check(dp_wait_status(pools_[c->pe]), "forward gate watchdog");
  }

  void completer(Reader* rd) {
    try {
      if (o_.gpu) check_cuda(cudaSetDevice(devs_[rd->engine]), "cudaSetDevice");
      for (;;) {
        int id;
        cudaEvent_t ev;
        double done_at = 0;
        {
          std::unique_lock<std::mutex> lk(rd->mu);
          rd->cv.wait(lk, [rd] { return !rd->inflight.empty() || rd->worker_done; });
          if (rd->inflight.empty()) return;
          std::tie(id, ev) = rd->inflight.front();
          rd->inflight.pop_front();
          if (!o_.gpu) {
            done_at = rd->inflight_done.front();
            rd->inflight_done.pop_front();
          }
        }
        if (o_.gpu) {
          check_cuda(cudaEventSynchronize(ev), "transfer sync");
          cudaEventDestroy(ev);
          const Req& q = reqs_[id];
          for (dp_pool* p : {pools_[q.r.pe], views_[rd->engine][q.r.pe]})
            if (p) check(dp_wait_status(p), "transfer watchdog");
        } else {
          std::this_thread::sleep_until(t0_ + std::chrono::duration_cast<Clock::duration>(
                                                  std::chrono::duration<double>(done_at)));
        }
        post({Msg::Landed, id});
      }
    } catch (const std::exception& ex) {
      fail_async(ex.what());
    }
  }

  // ---- gpu backend ------------------------------------------------------
  void setup_gpu(std::int64_t total_blk) {
    int ndev = 0;
    check_cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (ndev < 1) throw std::runtime_error("run_live: no CUDA device");
    devs_ = o_.devices;
    if (devs_.empty())
      for (int e = 0; e < n_eng_; ++e) devs_.push_back(e % ndev);
    if (static_cast<int>(devs_.size()) != n_eng_) throw std::invalid_argument("run_live: one device per engine");
    const dp_kv_geom geom{L_, T_, cfg_.kv_bytes_per_token_per_layer};
    check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&tab_slot_h_), std::max<std::int64_t>(1, total_blk) * 4,
                             cudaHostAllocMapped | cudaHostAllocPortable),
               "cudaHostAlloc tables");
    check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&tab_fb_h_), std::max<std::int64_t>(1, total_blk) * 8,
                             cudaHostAllocMapped | cudaHostAllocPortable),
               "cudaHostAlloc tables");
    check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&tab_de_h_), std::max<std::int64_t>(1, total_blk) * 4,
                             cudaHostAllocMapped | cudaHostAllocPortable),
               "cudaHostAlloc tables");
    for (int e = 0; e < n_eng_; ++e) {
      dp_store* st = nullptr;
      check(dp_store_create(devs_[e], &geom, store_fb_, o_.exec.seed, &st), "dp_store_create");
      stores_.push_back(st);
      streams_.push_back(detail::acquire_stream(devs_[e]));
      dp_stager* sg = nullptr;
      if ((is_pe(e) && o_.exec.k1_mode == 3) || (!is_pe(e) && o_.exec.k2_mode == 2)) {
        check(dp_stager_create(devs_[e], &geom, o_.exec.stage_ring_bytes, &sg), "dp_stager_create");
        check(dp_stager_set_ctas(sg, is_pe(e) ? o_.exec.stage_ctas : o_.exec.stage_push_ctas), "dp_stager_set_ctas");
        check(dp_stager_set_mode(sg, o_.exec.stage_scatter), "dp_stager_set_mode");
      }
      stagers_.push_back(sg);
    }
    for (int p = 0; p < n_pe_; ++p) {
      dp_pool* pool = nullptr;
      check(dp_pool_create(devs_[p], &geom, pool_slots_, static_cast<std::int32_t>(std::max<std::int64_t>(1, total_reqs_)),
                           &pool),
            "dp_pool_create");
      pools_.push_back(pool);
    }
    check(dp_layer_items(&geom, 1, &items_per_block_), "dp_layer_items");
    for (auto& c : computers_) {
      DeviceScope ds(devs_[c->pe]);
      c->stream = detail::acquire_stream(devs_[c->pe]);
      check_cuda(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming), "cudaEventCreate");
      check_cuda(cudaMalloc(reinterpret_cast<void**>(&c->d_slot), std::max<std::int64_t>(1, total_blk) * 4),
                 "cudaMalloc block tables");
      const std::size_t dig = static_cast<std::size_t>(std::max<std::int64_t>(1, total_reqs_)) * L_ * 8;
      check_cuda(cudaMalloc(reinterpret_cast<void**>(&c->d_digest), dig), "cudaMalloc digests");
      check_cuda(cudaMemset(c->d_digest, 0, dig), "cudaMemset digests");
      check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&c->h_wt), kMaxGates * 4, cudaHostAllocMapped),
                 "cudaHostAlloc gates");
      check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&c->h_wg), kMaxGates * 4, cudaHostAllocMapped),
                 "cudaHostAlloc gates");
    }
    if (handoff_) {
      for (int d = n_pe_; d < n_eng_; ++d) {
        dp_pool* pool = nullptr;
        check(dp_pool_create(devs_[d], &geom, de_slots_,
                             static_cast<std::int32_t>(std::max<std::int64_t>(1, total_reqs_)), &pool),
              "dp_pool_create (decode pool)");
        de_pools_.push_back(pool);
      }
      for (auto& ps : persisters_) {
        const int dev = devs_[n_pe_ + ps->de];
        DeviceScope ds(dev);
        ps->stream = detail::acquire_stream(dev);
        check_cuda(cudaEventCreateWithFlags(&ps->done, cudaEventDisableTiming), "cudaEventCreate");
        check(dp_stager_create(dev, &geom, o_.exec.stage_ring_bytes, &ps->stager), "dp_stager_create (persist)");
        check(dp_store_create(dev, &geom, store_fb_, o_.exec.seed + 1, &ps->store), "dp_store_create (persist)");
        if (!o_.exec.persist_path.empty())
          ps->file = std::make_unique<FullBlockFile>(o_.exec.persist_path, geom, store_fb_, false, false);
      }
      de_views_.assign(n_pe_, std::vector<dp_pool*>(n_eng_ - n_pe_, nullptr));
      for (int p = 0; p < n_pe_; ++p)
        for (int d = 0; d < n_eng_ - n_pe_; ++d)
          check(dp_pool_peer_view(devs_[p], de_pools_[d], &de_views_[p][d]), "dp_pool_peer_view (decode pool)");
    }
    views_.assign(n_eng_, std::vector<dp_pool*>(n_pe_, nullptr));
    for (int e = 0; e < n_eng_; ++e)
      for (int p = 0; p < n_pe_; ++p)
        if (e != p) check(dp_pool_peer_view(devs_[e], pools_[p], &views_[e][p]), "dp_pool_peer_view");
  }

  cudaEvent_t launch(int e, const Req& q) {
    DeviceScope ds(devs_[e]);
    const bool local = e == q.r.pe;
    dp_pool* dst = local ? pools_[q.r.pe] : views_[e][q.r.pe];
    dp_job job{tab_fb_h_ + q.tab_off, tab_slot_h_ + q.tab_off, q.r.cached, q.n_blk, 0, L_, q.r.id};
    cudaStream_t s = streams_[e];
    if (handoff_ && !local) {  // the DE read path fused with DecodeH2D: PE pool and the DE's decode pool
      dp_dual_job dj{job, tab_de_h_ + q.tab_off, q.r.id, 0};
      dp_pool* de_pool = de_pools_[e - n_pe_];
      check(stagers_[e] ? dp_h2d_push_dual_staged(dst, de_pool, stores_[e], stagers_[e], &dj, 1, s)
                        : dp_h2d_push_p2p_dual(dst, de_pool, stores_[e], &dj, 1, s),
            "dual transfer");
    } else if (stagers_[e]) {
      check(local ? dp_h2d_layer_staged(dst, stores_[e], stagers_[e], &job, 1, s)
                  : dp_h2d_push_staged(dst, stores_[e], stagers_[e], &job, 1, s),
            "staged transfer");
    } else {
      check(local ? dp_h2d_layer_gather(dst, stores_[e], &job, 1, s)
                  : dp_h2d_push_p2p_layer(dst, stores_[e], &job, 1, s),
            "gather transfer");
    }
    cudaEvent_t ev;
    check_cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    check_cuda(cudaEventRecord(ev, s), "cudaEventRecord");
    return ev;
  }

  void final_digests() {
    for (auto& c : computers_) {
      DeviceScope ds(devs_[c->pe]);
      std::vector<std::uint64_t> d(static_cast<std::size_t>(std::max<std::int64_t>(1, total_reqs_)) * L_);
      check_cuda(cudaMemcpy(d.data(), c->d_digest, d.size() * 8, cudaMemcpyDeviceToHost), "digests D2H");
      for (const Req& q : reqs_)
        if (q.r.pe == c->pe && q.r.t_prefilled >= 0)
          rep_.digests.push_back({q.r.id, d[static_cast<std::size_t>(q.r.id) * L_],
                                  d[static_cast<std::size_t>(q.r.id) * L_ + L_ - 1]});
    }
  }

  void final_occupants() {
    hash_occupants(pools_, occupant_, pool_slots_, 0, rep_.final_slots);
    if (handoff_) hash_occupants(de_pools_, de_occupant_, de_slots_, n_pe_, rep_.final_decode_slots);
  }

  void hash_occupants(const std::vector<dp_pool*>& pools, const std::vector<std::pair<std::int64_t, std::int32_t>>& occ,
                      std::int32_t n_slots, int engine0, std::vector<LiveReport::Occupant>& out) {
    for (int p = 0; p < static_cast<int>(pools.size()); ++p) {
      std::vector<std::int32_t> slots, ntok;
      std::vector<std::int64_t> fbs;
      for (std::int32_t s = 0; s < n_slots; ++s) {
        const auto& oc = occ[static_cast<std::size_t>(p) * n_slots + s];
        if (oc.first < 0) continue;
        slots.push_back(s);
        fbs.push_back(oc.first);
        ntok.push_back(oc.second);
      }
      if (slots.empty()) continue;
      DeviceScope ds(devs_[engine0 + p]);
      const std::size_t n = slots.size();
      std::int32_t *d_s = nullptr, *d_n = nullptr;
      std::uint64_t* d_o = nullptr;
      check_cuda(cudaMalloc(reinterpret_cast<void**>(&d_s), n * 4), "cudaMalloc");
      check_cuda(cudaMalloc(reinterpret_cast<void**>(&d_n), n * 4), "cudaMalloc");
      check_cuda(cudaMalloc(reinterpret_cast<void**>(&d_o), n * 8), "cudaMalloc");
      check_cuda(cudaMemcpy(d_s, slots.data(), n * 4, cudaMemcpyHostToDevice), "H2D");
      check_cuda(cudaMemcpy(d_n, ntok.data(), n * 4, cudaMemcpyHostToDevice), "H2D");
      std::vector<std::uint64_t> h0(n), h1(n);
      check(dp_pool_checksum(pools[p], 0, d_s, d_n, static_cast<std::int32_t>(n), d_o, nullptr), "checksum");
      check_cuda(cudaMemcpy(h0.data(), d_o, n * 8, cudaMemcpyDeviceToHost), "D2H");
      check(dp_pool_checksum(pools[p], L_ - 1, d_s, d_n, static_cast<std::int32_t>(n), d_o, nullptr), "checksum");
      check_cuda(cudaMemcpy(h1.data(), d_o, n * 8, cudaMemcpyDeviceToHost), "D2H");
      cudaFree(d_s);
      cudaFree(d_n);
      cudaFree(d_o);
      for (std::size_t i = 0; i < n; ++i)
        out.push_back({engine0 + p, slots[i], fbs[i], ntok[i], h0[i], h1[i]});
    }
  }

  pdsim::ClusterConfig cfg_;
  std::span<const pdsim::Trajectory> trajs_;
  LiveOptions o_;
  int g_ = 1, n_pe_ = 1, n_eng_ = 2;
  std::int32_t T_ = 64, L_ = 1;
  std::int64_t total_reqs_ = 0, completed_ = 0, fb_stride_ = 1, store_fb_ = 1, tab_used_ = 0;
  bool stop_ = false;
  bool arrived_in_wake_ = false;
  bool prefill_ = false;
  bool handoff_ = false;
  bool persist_ = false;
  std::int64_t persisted_ = 0;
  std::mutex persist_mu_;
  std::vector<std::unique_ptr<Persister>> persisters_;
  std::int32_t de_slots_ = 0;
  std::vector<std::vector<std::int32_t>> free_de_;
  std::vector<std::pair<std::int64_t, std::int32_t>> de_occupant_;
  std::vector<dp_pool*> de_pools_;                 // per DE: its decode pool
  std::vector<std::vector<dp_pool*>> de_views_;    // [pe][de]: decode pools mapped on the PE
  std::int32_t* tab_de_h_ = nullptr;               // decode-pool slots (by tab_off)
  static constexpr std::int32_t kMaxGates = 4096;
  std::int32_t items_per_block_ = 1;
  std::atomic<std::int64_t> forwards_{0};
  std::vector<std::unique_ptr<Computer>> computers_;
  double next_steady_ = 0;
  std::int32_t pool_slots_ = 0;
  Clock::time_point t0_;
  std::vector<Req> reqs_;
  std::vector<int> next_round_;
  std::vector<std::int64_t> tok_, seq_, hbm_free_, read_q_;
  std::deque<int> de_global_, pe_waiting_;
  std::vector<std::vector<int>> private_q_;
  std::vector<int> admission_;
  std::unordered_map<int, int> de_cat_;
  int rr_de_ = 0, rr_pe_ = 0;
  std::uint64_t rr_path_ = 0;
  std::vector<std::vector<std::int32_t>> free_slots_;
  std::vector<std::pair<std::int64_t, std::int32_t>> occupant_;
  using Timer = std::pair<double, int>;
  std::priority_queue<Timer, std::vector<Timer>, std::greater<Timer>> timers_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<Msg> msgs_;
  std::string worker_error_;
  std::vector<std::unique_ptr<Reader>> readers_;
  std::vector<dp_nic*> nics_;
  std::vector<std::int64_t> reader_bytes_;
  // gpu backend
  std::vector<int> devs_;
  std::vector<dp_store*> stores_;
  std::vector<dp_stager*> stagers_;
  std::vector<dp_pool*> pools_;
  std::vector<std::vector<dp_pool*>> views_;
  std::vector<cudaStream_t> streams_;
  std::int32_t* tab_slot_h_ = nullptr;
  std::int64_t* tab_fb_h_ = nullptr;
  LiveReport rep_;
};

}  // namespace

LiveReport run_live(const pdsim::ClusterConfig& cfg, std::span<const pdsim::Trajectory> trajectories,
                    const LiveOptions& options) {
  Live live(cfg, trajectories, options);
  return live.run();
}

}  // namespace dualpath
