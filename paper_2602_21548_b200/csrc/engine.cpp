// GPU executor of the DualPath KV loading path (see dualpath/engine.hpp).
#include "dualpath/engine.hpp"

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

// Free-slot queues of one pool.  Freed slots go back to a queue of the
// engine that last wrote them; an allocation takes, in order, never-used
// slots, the slots its own writer freed longest ago (ordered by its stream,
// and long done in real time), then other writers' slots (a cross-GPU
// hazard).  FIFO within each queue: reuse distance is maximal, so the
// hazard waits an allocation records are almost always already satisfied.
struct SlotQueues {
  std::deque<std::int32_t> fresh;
  std::vector<std::deque<std::int32_t>> by_writer;
  std::vector<std::int32_t> owner;  // slot -> job index of its last occupant

  SlotQueues(std::int32_t n_slots, int n_writers) : by_writer(n_writers), owner(n_slots, -1) {
    for (std::int32_t s = 0; s < n_slots; ++s) fresh.push_back(s);
  }
  std::int32_t take(int writer) {
    std::deque<std::int32_t>* src = nullptr;
    if (!fresh.empty()) {
      src = &fresh;
    } else if (!by_writer[writer].empty()) {
      src = &by_writer[writer];
    } else {
      for (auto& q : by_writer)
        if (!q.empty()) {
          src = &q;
          break;
        }
    }
    if (!src) throw std::logic_error("build_exec_plan: slot allocator ran dry below the peak");
    const std::int32_t s = src->front();
    src->pop_front();
    return s;
  }
};

struct TimedEv {
  double t;
  int kind;  // 0 = free, 1 = alloc
  int req;
  int job;
};

void sort_events(std::vector<TimedEv>& evs) {
  std::sort(evs.begin(), evs.end(), [](const TimedEv& a, const TimedEv& b) {
    if (a.t != b.t) return a.t < b.t;
    if (a.kind != b.kind) return a.kind < b.kind;
    return a.req < b.req;
  });
}

// Peak live blocks over a key (PE or DE) for alloc/free events.
std::int64_t peak_blocks(const std::vector<TimedEv>& evs, int n_keys,
                         const std::vector<int>& key_of_job,
                         const std::vector<std::int32_t>& blocks_of_job) {
  std::vector<std::int64_t> live(n_keys, 0);
  std::int64_t peak = 0;
  for (const TimedEv& e : evs) {
    const int k = key_of_job[e.job];
    live[k] += e.kind == 1 ? blocks_of_job[e.job] : -blocks_of_job[e.job];
    peak = std::max(peak, live[k]);
  }
  return peak;
}

std::int32_t size_pool(std::int32_t requested, std::int64_t peak, std::int64_t slot_cap,
                       const char* what) {
  const std::int64_t n = requested > 0
                             ? requested
                             : std::min<std::int64_t>(slot_cap, std::max<std::int64_t>(1, 4 * peak));
  if (n < peak)
    throw std::invalid_argument(std::string("build_exec_plan: ") + what + " of " + std::to_string(n) +
                                " slots is below the plan's peak of " + std::to_string(peak) +
                                " live blocks");
  return static_cast<std::int32_t>(n);
}

// Prefill forwards of every PE.  A PE's FIFO is its requests in the order
// their KV lands (t_read_done, then request id: the job order); forwards
// are build_forward_batch over a window of that FIFO.  The window stops
// before the first request whose slots reuse those of a request still in
// the window: that request's load waits for the forward reading the
// earlier one, so the two must not share a forward.
void build_forwards(ExecPlan& x, const pdsim::desim::SimReport& plan) {
  std::vector<int> job_of_req;
  for (std::size_t i = 0; i < x.jobs.size(); ++i) {
    const int r = x.jobs[i].req;
    if (r >= static_cast<int>(job_of_req.size())) job_of_req.resize(r + 1, -1);
    job_of_req[r] = static_cast<int>(i);
  }
  std::vector<std::vector<const pdsim::desim::RequestPlan*>> fifo(x.n_pe);
  for (const auto& r : plan.requests)
    if (r.pe >= 0 && r.pe < x.n_pe && r.t_read_done >= 0) fifo[r.pe].push_back(&r);
  pdsim::SchedulerParams sp;
  sp.compute_quota = x.opt.compute_quota;
  x.fwd_items.assign(x.n_pe, {});
  x.forwards.assign(x.n_pe, {});
  x.fwd_rows.assign(x.n_pe, {});
  x.last_fwd.assign(x.jobs.size(), -1);
  std::vector<int> row_of_job(x.jobs.size(), -1);
  for (int p = 0; p < x.n_pe; ++p) {
    auto& q = fifo[p];
    std::stable_sort(q.begin(), q.end(), [](const auto* a, const auto* b) {
      return a->t_read_done != b->t_read_done ? a->t_read_done < b->t_read_done : a->request_id < b->request_id;
    });
    const int n = static_cast<int>(q.size());
    std::vector<int> job(n, -1), pred_row(n, -1);
    for (int i = 0; i < n; ++i) {
      x.fwd_rows[p].push_back(q[i]->request_id);
      const int rid = q[i]->request_id;
      if (rid < static_cast<int>(job_of_req.size()) && job_of_req[rid] >= 0) {
        job[i] = job_of_req[rid];
        row_of_job[job[i]] = i;
      } else if (q[i]->cached > 0) {
        throw std::logic_error("build_exec_plan: a request with cached KV reached prefill without a load job");
      }
    }
    for (int i = 0; i < n; ++i)
      if (job[i] >= 0)
        for (int w : x.jobs[job[i]].consumer_waits) pred_row[i] = std::max(pred_row[i], row_of_job[w]);
    int head = 0, barrier = 0;
    std::int64_t head_done = 0;  // query tokens of the head request already run
    std::vector<pdsim::BatchItem> window;
    while (head < n) {
      barrier = std::max(barrier, head + 1);
      while (barrier < n && pred_row[barrier] < head) ++barrier;
      window.clear();
      for (int i = head; i < barrier; ++i)
        window.push_back({q[i]->request_id, q[i]->cached, q[i]->append - (i == head ? head_done : 0)});
      const pdsim::ForwardBatch fb = pdsim::build_forward_batch(window, sp, x.opt.prefill_cost);
      Forward f;
      f.begin = static_cast<std::int32_t>(x.fwd_items[p].size());
      f.estimated_time = fb.estimated_time;
      const int fi = static_cast<int>(x.forwards[p].size());
      for (std::size_t k = 0; k < fb.items.size(); ++k) {
        const int row = head + static_cast<int>(k);
        FwdItem it;
        it.req = fb.items[k].request_id;
        it.job = job[row];
        it.cached = fb.items[k].cached;
        it.q_begin = k == 0 ? head_done : 0;
        it.bsz = fb.items[k].bsz;
        it.row = row;
        it.first = it.q_begin == 0;
        x.fwd_items[p].push_back(it);
        if (it.job >= 0) x.last_fwd[it.job] = fi;
        f.last_row = row;
      }
      f.end = static_cast<std::int32_t>(x.fwd_items[p].size());
      x.forwards[p].push_back(f);
      int last_job = -1;
      for (std::int32_t i = f.begin; i < f.end; ++i) last_job = std::max(last_job, x.fwd_items[p][i].job);
      for (std::int32_t i = f.begin; i < f.end; ++i)
        if (x.fwd_items[p][i].job >= 0) x.jobs[x.fwd_items[p][i].job].k3_after = last_job;
      if (fb.chunked) {
        head_done = fb.consumed_whole == 0 ? head_done + fb.chunk_bsz : fb.chunk_bsz;
      } else {
        head_done = 0;
      }
      head += static_cast<int>(fb.consumed_whole);
    }
  }
}

// Storage tier tables.  The Full Block trie indexes every session's chain of
// Full Blocks (record = the page the procedural store holds for it, so the
// bytes are the same); a job's blocks are the records its session's chain
// matches.  Each reader stages them in a FIFO ring of pinned Full Blocks:
// src_fb becomes ring positions, and a job whose reads overwrite positions
// of earlier jobs waits for their transfers.
void build_tier(ExecPlan& x, std::span<const pdsim::Trajectory> trajectories) {
  FullBlockTrie trie;
  std::vector<std::vector<std::uint64_t>> chains(trajectories.size());
  for (std::size_t t = 0; t < trajectories.size(); ++t) {
    const std::int64_t nb = pdsim::blocks_for(trajectories[t].total_tokens(), x.cfg);
    chains[t] = session_chain(trajectories[t].id, nb);
    std::vector<std::int64_t> rec(static_cast<std::size_t>(nb));
    for (std::int64_t k = 0; k < nb; ++k) rec[k] = x.fb_of(static_cast<int>(t), k);
    trie.insert(chains[t], rec);
  }
  x.trie_nodes = trie.nodes();
  std::int32_t biggest = 1;
  for (const LoadJob& j : x.jobs) biggest = std::max(biggest, j.n_blk);
  std::int64_t ring = x.opt.tier_ring_fb > 0 ? x.opt.tier_ring_fb : std::max<std::int64_t>(4LL * biggest, 512);
  if (ring < biggest)
    throw std::invalid_argument("build_exec_plan: tier_ring_fb of " + std::to_string(ring) +
                                " is below the largest job (" + std::to_string(biggest) + " Full Blocks)");
  x.ring_fb = static_cast<std::int32_t>(ring);
  x.tier_rec.assign(x.n_engines, {});
  for (int e = 0; e < x.n_engines; ++e) {
    std::vector<int> owner(static_cast<std::size_t>(ring), -1);
    std::int64_t head = 0;
    for (int ji : x.by_reader[e]) {
      LoadJob& j = x.jobs[ji];
      const auto recs = trie.match(std::span<const std::uint64_t>(chains[j.traj]).first(j.n_blk));
      if (static_cast<std::int32_t>(recs.size()) != j.n_blk)
        throw std::logic_error("build_exec_plan: trie lookup missed a session block");
      for (std::int32_t k = 0; k < j.n_blk; ++k) {
        const std::int64_t pos = (head + k) % ring;
        if (owner[pos] >= 0 && std::find(j.ring_waits.begin(), j.ring_waits.end(), owner[pos]) == j.ring_waits.end())
          j.ring_waits.push_back(owner[pos]);
        owner[pos] = ji;
        x.src_fb[e][j.blk_off + k] = pos;
        x.tier_rec[e].push_back(recs[k]);
      }
      head = (head + j.n_blk) % ring;
    }
  }
}

}  // namespace

std::int64_t ExecPlan::fb_of(int traj, std::int64_t block) const {
  return (static_cast<std::int64_t>(traj) * fb_stride + block) % store_fb;
}

std::uint32_t ExecPlan::de_total_items(const LoadJob& j) const {
  const std::int64_t blocks = (j.de_path ? j.n_blk : 0) + j.n_pblk;
  return static_cast<std::uint32_t>(blocks * items_per_block * cfg.n_layer);
}

std::vector<std::pair<std::int64_t, std::int64_t>> ExecPlan::persist_chunks(const LoadJob& j) const {
  // persist_tokens(rq, k) at decode milestones k % T == 0 (k < gen) and at
  // completion with k = gen (desim.cpp:658-661, :690-693, :760)
  std::vector<std::pair<std::int64_t, std::int64_t>> out;
  const std::int64_t T = cfg.block_size_tokens;
  std::int64_t done = 0;
  for (std::int64_t k = T; k < j.gen; k += T) {
    out.emplace_back(j.prompt + done, j.prompt + k);
    done = k;
  }
  if (j.gen > done) out.emplace_back(j.prompt + done, j.prompt + j.gen);
  return out;
}

ExecPlan build_exec_plan(const pdsim::ClusterConfig& cfg,
                         std::span<const pdsim::Trajectory> trajectories,
                         const pdsim::desim::SimReport& plan, const ExecOptions& opt) {
  cfg.validate();
  ExecPlan x;
  x.cfg = cfg;
  x.opt = opt;
  x.handoff = opt.handoff;
  x.persist = opt.persist;
  if (x.persist && !x.handoff) throw std::invalid_argument("build_exec_plan: persist needs handoff");
  x.prefill = opt.prefill;
  if (x.prefill && !(opt.compute_quota > 0))
    throw std::invalid_argument("build_exec_plan: compute_quota must be > 0");
  x.tier = !opt.tier_path.empty();
  if (x.tier && (x.handoff || x.prefill))
    throw std::invalid_argument("build_exec_plan: the storage tier runs on the plain load path");
  if (x.tier && opt.io_threads < 1) throw std::invalid_argument("build_exec_plan: io_threads must be >= 1");
  x.n_engines = cfg.total_engines();
  x.n_pe = cfg.prefill_nodes * cfg.engines_per_node;
  x.geom = {cfg.n_layer, cfg.block_size_tokens, cfg.kv_bytes_per_token_per_layer};
  check(dp_geom_check(&x.geom), "build_exec_plan");
  check(dp_layer_items(&x.geom, 1, &x.items_per_block), "build_exec_plan");
  const std::int64_t fb_bytes = cfg.full_block_bytes();
  const std::int64_t T = cfg.block_size_tokens;
  const std::int64_t L = cfg.n_layer;

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
  if (!opt.storage_cap_per_engine.empty() &&
      static_cast<int>(opt.storage_cap_per_engine.size()) != x.n_engines)
    throw std::invalid_argument("build_exec_plan: storage_cap_per_engine needs one entry per engine");

  // jobs: every request with cached KV that reached the hit transfer (and,
  // with the handoff, every request that reached prefill)
  std::vector<TimedEv> pe_evs, de_evs;
  std::vector<LoadJob> jobs;
  std::vector<int> pe_of, de_of;
  std::vector<std::int32_t> pblocks, dblocks;
  for (const auto& r : plan.requests) {
    x.prompt_tokens += r.cached + r.append;
    ++x.requests;
    if (r.pe < 0 || r.t_read_done < 0) continue;
    if (r.cached <= 0 && !x.handoff) continue;
    if (x.handoff && r.de < 0) continue;
    if (r.traj_index < 0 || static_cast<std::size_t>(r.traj_index) >= trajectories.size())
      throw std::invalid_argument("build_exec_plan: plan does not match the trajectories");
    LoadJob j;
    j.req = r.request_id;
    j.traj = r.traj_index;
    j.round = r.round;
    j.pe = r.pe;
    j.de = r.de;
    j.de_path = r.path == pdsim::ReadPath::DEPath;
    j.reader = j.de_path ? r.de : r.pe;
    j.cached = r.cached;
    j.prompt = r.cached + r.append;
    j.n_blk = static_cast<std::int32_t>((r.cached + T - 1) / T);
    j.n_pblk = x.handoff ? static_cast<std::int32_t>((j.prompt + T - 1) / T) : j.n_blk;
    j.gen = r.gen;
    j.n_tblk = x.persist ? static_cast<std::int32_t>((j.prompt + j.gen + T - 1) / T) : j.n_pblk;
    j.t_admit = r.t_admit;
    j.t_read_done = r.t_read_done;
    const int idx = static_cast<int>(jobs.size());
    jobs.push_back(std::move(j));
    pe_of.push_back(r.pe);
    de_of.push_back(std::max(0, r.de));
    pblocks.push_back(jobs.back().n_pblk);
    dblocks.push_back(jobs.back().n_tblk);
    pe_evs.push_back({r.t_read_done, 1, r.request_id, idx});
    if (r.t_pe_release >= 0) pe_evs.push_back({r.t_pe_release, 0, r.request_id, idx});
    if (x.handoff) {
      de_evs.push_back({r.t_read_done, 1, r.request_id, idx});
      if (r.t_done >= 0) de_evs.push_back({r.t_done, 0, r.request_id, idx});
    }
  }
  sort_events(pe_evs);
  sort_events(de_evs);
  const std::int64_t slot_cap = std::max<std::int64_t>(1, opt.pool_bytes_max / fb_bytes);
  x.peak_slots = static_cast<std::int32_t>(peak_blocks(pe_evs, x.n_engines, pe_of, pblocks));
  x.pool_slots = size_pool(opt.pool_slots, x.peak_slots, slot_cap, "PE pool");
  if (x.handoff) {
    x.de_peak_slots = static_cast<std::int32_t>(peak_blocks(de_evs, x.n_engines, de_of, dblocks));
    x.de_pool_slots = size_pool(opt.de_pool_slots, x.de_peak_slots, slot_cap, "DE decode pool");
  }

  // pass 2: PE slot allocation in virtual time -> the global job order
  std::vector<SlotQueues> pe_q;
  for (int p = 0; p < x.n_pe; ++p) pe_q.emplace_back(x.pool_slots, x.n_engines);
  std::vector<std::vector<std::int32_t>> pe_slots(jobs.size()), de_slots(jobs.size());
  x.n_tickets.assign(x.n_pe, 0);
  std::vector<int> order;
  order.reserve(jobs.size());
  for (const TimedEv& e : pe_evs) {
    LoadJob& j = jobs[e.job];
    SlotQueues& q = pe_q[j.pe];
    if (e.kind == 0) {
      for (std::int32_t s : pe_slots[e.job]) q.by_writer[j.reader].push_back(s);
      continue;
    }
    j.ticket = x.n_tickets[j.pe]++;
    auto& mine = pe_slots[e.job];
    mine.reserve(j.n_pblk);
    for (std::int32_t k = 0; k < j.n_pblk; ++k) {
      const std::int32_t s = q.take(j.reader);
      mine.push_back(s);
      const std::int32_t prev = q.owner[s];
      q.owner[s] = e.job;
      if (prev < 0) continue;
      const LoadJob& pj = jobs[prev];
      if (x.prefill && !x.handoff) {
        // the previous occupant's KV is read by its forwards: the reuse
        // waits for the last of them (which implies it landed)
        if (std::find(j.consumer_waits.begin(), j.consumer_waits.end(), prev) == j.consumer_waits.end())
          j.consumer_waits.push_back(prev);
      } else if (!x.handoff) {
        // same reader: stream order serialises launches, but items of one
        // launch run concurrently, so the reuse must start a new launch
        if (pj.reader == j.reader) {
          j.fence = true;
        } else if (std::find(j.preds.begin(), j.preds.end(), pj.ticket) == j.preds.end()) {
          j.preds.push_back(pj.ticket);
          j.pred_targets.push_back(static_cast<std::uint32_t>(
              static_cast<std::int64_t>(pj.n_blk) * x.items_per_block * L));
        }
      } else if (!j.de_path) {
        // the previous occupant's K3 (same PE, handoff stream) must be done
        if (std::find(j.k3_waits.begin(), j.k3_waits.end(), prev) == j.k3_waits.end())
          j.k3_waits.push_back(prev);
        if (x.prefill && std::find(j.consumer_waits.begin(), j.consumer_waits.end(), prev) == j.consumer_waits.end())
          j.consumer_waits.push_back(prev);  // K3 runs after the forwards: keep them apart
      } else if (std::find(j.pe_done_preds.begin(), j.pe_done_preds.end(), pj.ticket) ==
                 j.pe_done_preds.end()) {
        j.pe_done_preds.push_back(pj.ticket);  // + n_tickets[pe] once known
        j.pe_done_targets.push_back(
            static_cast<std::uint32_t>(static_cast<std::int64_t>(pj.n_pblk) * x.items_per_block * L));
        if (x.prefill && std::find(j.consumer_waits.begin(), j.consumer_waits.end(), prev) == j.consumer_waits.end())
          j.consumer_waits.push_back(prev);
      }
    }
    order.push_back(e.job);
  }
  std::vector<int> pos(jobs.size(), -1);  // old job index -> global position
  for (std::size_t i = 0; i < order.size(); ++i) pos[order[i]] = static_cast<int>(i);

  // pass 3 (handoff): decode-pool slots, allocated at t_read_done and freed
  // when the request completes
  if (x.handoff) {
    std::vector<SlotQueues> de_q;
    for (int d = 0; d < x.n_engines; ++d) de_q.emplace_back(d >= x.n_pe ? x.de_pool_slots : 0, 1);
    x.n_de_tickets.assign(x.n_engines, 0);
    for (const TimedEv& e : de_evs) {
      LoadJob& j = jobs[e.job];
      SlotQueues& q = de_q[j.de];
      if (e.kind == 0) {
        for (std::int32_t s : de_slots[e.job]) q.by_writer[0].push_back(s);
        continue;
      }
      j.de_ticket = x.n_de_tickets[j.de]++;
      for (std::int32_t k = 0; k < j.n_tblk; ++k) {
        const std::int32_t s = q.take(0);
        de_slots[e.job].push_back(s);
        const std::int32_t prev = q.owner[s];
        q.owner[s] = e.job;
        if (prev < 0) continue;
        const LoadJob& pj = jobs[prev];
        if (pos[prev] >= pos[e.job])
          throw std::logic_error("build_exec_plan: decode-slot predecessor is not earlier");
        if (std::find(j.de_preds.begin(), j.de_preds.end(), pj.de_ticket) == j.de_preds.end()) {
          j.de_preds.push_back(pj.de_ticket);
          // with persistence the slot is free once the occupant is persisted
          // (its "persist done" row, resolved at run time, reads 1)
          j.de_pred_targets.push_back(x.persist ? 1u : x.de_total_items(pj));
        }
      }
    }
  }

  x.by_reader.assign(x.n_engines, {});
  x.by_pe.assign(x.n_pe, {});
  x.by_de.assign(x.n_engines, {});
  x.src_fb.assign(x.n_engines, {});
  x.slots.assign(x.n_engines, {});
  x.dual_de_slot.assign(x.n_engines, {});
  x.dec_slot.assign(x.n_engines, {});
  x.dec_fb.assign(x.n_engines, {});
  x.ho_src_fb.assign(x.n_pe, {});
  x.ho_pe_slot.assign(x.n_pe, {});
  x.ho_de_slot.assign(x.n_pe, {});
  x.reader_bytes.assign(x.n_engines, 0);
  x.fwd_slot.assign(x.n_pe, {});
  x.jobs.reserve(order.size());
  for (int old : order) {
    LoadJob j = std::move(jobs[old]);
    for (int& w : j.k3_waits) w = pos[w];
    for (int& w : j.consumer_waits) w = pos[w];
    if (x.prefill) {
      if (j.reader != j.pe && !x.handoff)  // a DE load waits on the PE's "consumed" rows [n, 2n)
        for (int w : j.consumer_waits) {
          j.preds.push_back(x.jobs[w].ticket + x.n_tickets[j.pe]);
          j.pred_targets.push_back(1u);
        }
      j.fwd_off = static_cast<std::int64_t>(x.fwd_slot[j.pe].size());
      x.fwd_slot[j.pe].insert(x.fwd_slot[j.pe].end(), pe_slots[old].begin(),
                              pe_slots[old].begin() + j.n_blk);
    }
    const int idx = static_cast<int>(x.jobs.size());
    auto& src = x.src_fb[j.reader];
    auto& dst = x.slots[j.reader];
    j.blk_off = static_cast<std::int64_t>(src.size());
    for (std::int32_t k = 0; k < j.n_blk; ++k) {
      src.push_back(x.fb_of(j.traj, k));
      dst.push_back(pe_slots[old][k]);
      if (x.handoff) x.dual_de_slot[j.reader].push_back(de_slots[old][k]);
    }
    if (x.handoff) {
      j.ho_off = static_cast<std::int64_t>(x.ho_src_fb[j.pe].size());
      for (std::int32_t k = 0; k < j.n_pblk; ++k) {
        x.ho_src_fb[j.pe].push_back(x.fb_of(j.traj, k));
        x.ho_pe_slot[j.pe].push_back(pe_slots[old][k]);
        x.ho_de_slot[j.pe].push_back(de_slots[old][k]);
      }
      x.handoff_bytes += (j.de_path ? j.prompt - j.cached : j.prompt) * cfg.kv_bytes_per_token();
      x.by_de[j.de].push_back(idx);
      if (x.persist) {
        j.dec_off = static_cast<std::int64_t>(x.dec_slot[j.de].size());
        for (std::int32_t k = 0; k < j.n_tblk; ++k) {
          x.dec_slot[j.de].push_back(de_slots[old][k]);
          x.dec_fb[j.de].push_back(x.fb_of(j.traj, k));
        }
        x.persist_bytes += j.gen * cfg.kv_bytes_per_token();
      }
    }
    const std::int64_t bytes = j.cached * cfg.kv_bytes_per_token();
    x.reader_bytes[j.reader] += bytes;
    x.hit_bytes += bytes;
    if (j.n_blk > 0) x.by_reader[j.reader].push_back(idx);
    x.by_pe[j.pe].push_back(idx);
    x.jobs.push_back(std::move(j));
  }
  if (x.prefill) build_forwards(x, plan);
  if (x.tier) build_tier(x, trajectories);
  return x;
}

EngineRuntime::EngineRuntime(std::shared_ptr<const ExecPlan> plan, int engine, int device)
    : plan_(std::move(plan)), engine_(engine), device_(device) {
  if (!plan_) throw std::invalid_argument("EngineRuntime: null plan");
  if (engine < 0 || engine >= plan_->n_engines)
    throw std::invalid_argument("EngineRuntime: engine out of range");
  const ExecPlan& x = *plan_;
  DeviceScope ds(device_);
  cudaStream_t s;
  check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
  stream_ = s;
  cudaEvent_t a, b;
  check_cuda(cudaEventCreate(&a), "cudaEventCreate");
  check_cuda(cudaEventCreate(&b), "cudaEventCreate");
  ev_start_ = a;
  ev_end_ = b;
  peers_.assign(x.n_engines, nullptr);
  de_views_.assign(x.n_engines, nullptr);
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
    const std::int32_t rows =
        std::max<std::int32_t>(1, x.n_tickets[engine_]) * (x.handoff || x.prefill ? 2 : 1);
    check(dp_pool_create(device_, &x.geom, x.pool_slots, rows, &pool_), "dp_pool_create");
    peers_[engine_] = pool_;
  } else if (x.handoff) {
    // rows [0, n) prompt landed; with persistence rows [n, 2n) persisted
    const std::int32_t rows = std::max<std::int32_t>(1, x.n_de_tickets[engine_]) * (x.persist ? 2 : 1);
    check(dp_pool_create(device_, &x.geom, x.de_pool_slots, rows, &pool_), "dp_pool_create (decode pool)");
    if (x.persist && !x.by_de[engine_].empty())  // content seed + 1: unwritten bytes differ
      check(dp_store_create(device_, &x.geom, x.store_fb, x.opt.seed + 1, &persist_store_),
            "dp_store_create (persist store)");
  }
  if (x.handoff) {
    upload_handoff_tables();
  } else {
    upload_tables();
  }
  if (x.prefill && is_pe()) upload_prefill_tables();
  if (x.opt.k1_mode == 2 && is_pe() && !x.handoff && !x.prefill) {
    cudaStream_t c;
    check_cuda(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking), "cudaStreamCreate");
    stream_ce_ = c;
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
  if (is_pe()) check(dp_set_handoff_ctas(device_, x.opt.handoff_ctas), "dp_set_handoff_ctas");
  if (is_pe() && x.prefill) check(dp_set_attend_ctas(device_, x.opt.attend_ctas), "dp_set_attend_ctas");
}

void EngineRuntime::upload_prefill_tables() {
  const ExecPlan& x = *plan_;
  const auto& items = x.fwd_items[engine_];
  const auto& fwds = x.forwards[engine_];
  const std::int32_t L = x.cfg.n_layer;
  cudaStream_t c;
  check_cuda(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking), "cudaStreamCreate");
  stream_c_ = c;  // the compute stream: forwards
  // the load stream outranks the compute stream: as K5 CTAs retire, the
  // block scheduler places pending loader CTAs first
  int lo = 0, hi = 0;
  check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
  cudaStream_t s;
  check_cuda(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi), "cudaStreamCreateWithPriority");
  check_cuda(cudaStreamDestroy(static_cast<cudaStream_t>(stream_)), "cudaStreamDestroy");
  stream_ = s;
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
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    ev_fwd_.push_back(e);
  }
  d_fwt_ = upload(wt);
  d_fwg_ = upload(wg);
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
  if (store_) dp_store_destroy(store_);
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
  if (stream_h_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_h_));
  if (stream_c_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_c_));
  if (stream_ce_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_ce_));
  for (void* e : ev_ce_) cudaEventDestroy(static_cast<cudaEvent_t>(e));
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
    cudaStream_t h;
    check_cuda(cudaStreamCreateWithFlags(&h, cudaStreamNonBlocking), "cudaStreamCreate");
    stream_h_ = h;
    const auto& mine = x.by_pe[engine_];
    for (std::size_t i = 0; i < mine.size(); ++i) {
      pe_local_[mine[i]] = static_cast<int>(i);
      cudaEvent_t a, b;
      check_cuda(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "cudaEventCreate");
      check_cuda(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "cudaEventCreate");
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
    cudaStream_t h;
    check_cuda(cudaStreamCreateWithFlags(&h, cudaStreamNonBlocking), "cudaStreamCreate");
    stream_h_ = h;  // the decode stream: decode stand-in + persistence
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
  check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_start_), s), "cudaEventRecord");

  const auto& mine = x.by_reader[engine_];
  std::vector<dp_job> batch;
  batch.reserve(DP_MAX_JOBS_PER_LAUNCH);
  std::vector<int> batch_jobs;  // by_reader positions of the jobs in `batch`
  int batch_pe = -1;
  const bool k1_ce = x.opt.k1_mode == 1;
  const bool k2_ce = x.opt.k2_mode == 1;
  // K1 hybrid (k1_mode 2): the PE's own jobs split by bytes between the SM
  // gather (load stream) and the copy engine (a second stream), run together
  const bool hybrid = x.opt.k1_mode == 2 && stream_ce_ != nullptr && !x.tier;
  auto sc = static_cast<cudaStream_t>(stream_ce_);
  std::vector<dp_job> batch_ce;
  double sm_bytes = 0, ce_bytes = 0;
  if (hybrid) check_cuda(cudaStreamWaitEvent(sc, static_cast<cudaEvent_t>(ev_start_), 0), "cudaStreamWaitEvent");

  // Storage tier: IO threads read each job's Full Blocks from the file into
  // its staging-ring positions, in job order (first reusing a position only
  // after the transfer that read it is done); a job is launched once read.
  struct Io {
    std::mutex mu;
    std::condition_variable cv;
    std::vector<char> read, launched;
    std::atomic<int> next{0};
    bool failed = false;
    std::exception_ptr err;
  } io;
  std::vector<std::thread> workers;
  char* staging = nullptr;
  if (x.tier && !mine.empty()) {
    void* host = nullptr;
    check(dp_store_info(store_, &host, nullptr, nullptr), "dp_store_info");
    staging = static_cast<char*>(host);
    io.read.assign(mine.size(), 0);
    io.launched.assign(mine.size(), 0);
    const std::int64_t fbb = x.cfg.full_block_bytes();
    const int dev = device_;
    for (int t = 0; t < x.opt.io_threads; ++t)
      workers.emplace_back([&, fbb, dev] {
        try {
          cudaSetDevice(dev);
          for (int i = io.next++; i < static_cast<int>(mine.size()); i = io.next++) {
            for (int w : ring_wait_local_[i]) {
              {
                std::unique_lock<std::mutex> lk(io.mu);
                io.cv.wait(lk, [&] { return io.launched[w] || io.failed; });
                if (io.failed) return;
              }
              check_cuda(cudaEventSynchronize(static_cast<cudaEvent_t>(ev_job_[w])), "ring reuse wait");
            }
            // one read per run of blocks consecutive both in the file and in
            // the ring (a session's pages are consecutive records)
            const LoadJob& j = x.jobs[mine[i]];
            const std::int64_t* rec = x.tier_rec[engine_].data() + j.blk_off;
            const std::int64_t* pos = x.src_fb[engine_].data() + j.blk_off;
            constexpr std::int32_t kMaxRun = 8;  // 18 MB of DS-V3 Full Blocks per read
            for (std::int32_t k = 0; k < j.n_blk;) {
              std::int32_t run = 1;
              while (k + run < j.n_blk && run < kMaxRun && rec[k + run] == rec[k] + run && pos[k + run] == pos[k] + run)
                ++run;
              tier_file_->read_run(rec[k], run, staging + pos[k] * fbb);
              k += run;
            }
            std::lock_guard<std::mutex> lk(io.mu);
            io.read[i] = 1;
            io.cv.notify_all();
          }
        } catch (...) {
          std::lock_guard<std::mutex> lk(io.mu);
          if (!io.err) io.err = std::current_exception();
          io.failed = true;
          io.cv.notify_all();
        }
      });
  }
  struct JoinWorkers {
    Io& io;
    std::vector<std::thread>& w;
    ~JoinWorkers() {
      {
        std::lock_guard<std::mutex> lk(io.mu);
        io.failed = true;  // releases any worker still waiting (normal exit: all done)
        io.cv.notify_all();
      }
      for (auto& t : w) t.join();
    }
  } join_workers{io, workers};

  auto flush = [&]() {
    if (batch.empty()) return;
    dp_pool* dst = peers_[batch_pe];
    const auto n = static_cast<int32_t>(batch.size());
    int rc;
    const char* what;
    if (batch_pe != engine_ && k2_ce) {
      rc = dp_h2d_push_copy(dst, store_, batch.data(), n, s);
      what = "dp_h2d_push_copy";
    } else if (batch_pe != engine_) {
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
    const bool on_ce = batch_pe == engine_ ? k1_ce : k2_ce;
    if (!on_ce)  // kernel launches (the copy engine paths have none)
      res.launches += (static_cast<std::int64_t>(batch.size()) + DP_MAX_JOBS_PER_LAUNCH - 1) /
                      DP_MAX_JOBS_PER_LAUNCH;
    batch.clear();
    if (staging) {
      for (int i : batch_jobs) check_cuda(cudaEventRecord(static_cast<cudaEvent_t>(ev_job_[i]), s), "cudaEventRecord");
      std::lock_guard<std::mutex> lk(io.mu);
      for (int i : batch_jobs) io.launched[i] = 1;
      io.cv.notify_all();
    }
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
  double gate_s = 0;  // emulated storage-NIC busy-until (FIFO token bucket), s since t0
  for (std::size_t i = 0; i < mine.size(); ++i) {
    const LoadJob& j = x.jobs[mine[i]];
    if (!peers_[j.pe]) throw std::runtime_error("run_step: PE " + std::to_string(j.pe) + " not attached");
    const std::int64_t bytes = j.cached * x.cfg.kv_bytes_per_token();
    const bool gated = cap > 0 || pace > 0;
    const bool hazard = !j.preds.empty();
    if (gated || hazard || j.fence || batch_pe != j.pe || batch.size() == DP_MAX_JOBS_PER_LAUNCH)
      flush();
    if (hybrid) {
      if (hazard || j.fence) join_streams();
      else if (gated || batch_ce.size() == DP_MAX_JOBS_PER_LAUNCH) flush_ce();
    }
    if (gated) {
      // StorageRead of C*L*b bytes over this engine's storage NIC: starts
      // when the NIC is free (and, replaying online, not before the planned
      // admission), takes bytes / cap
      const double begin = std::max(gate_s, pace > 0 ? j.t_admit * pace : 0.0);
      gate_s = begin + (cap > 0 ? static_cast<double>(bytes) / cap : 0.0);
      std::this_thread::sleep_until(t0 + std::chrono::duration<double>(gate_s));
      res.spans.push_back({begin, gate_s, bytes});
    }
    if (staging) {  // StorageRead: the job's Full Blocks must be in staging
      bool ready;
      {
        std::lock_guard<std::mutex> lk(io.mu);
        ready = io.read[i] || io.failed;
      }
      if (!ready) {
        flush();  // never hold launched work while waiting on the disk
        const auto w0 = std::chrono::steady_clock::now();
        std::unique_lock<std::mutex> lk(io.mu);
        io.cv.wait(lk, [&] { return io.read[i] || io.failed; });
        res.io_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
      }
      if (io.err) std::rethrow_exception(io.err);
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
    if (j.pe == engine_ ? k1_ce : k2_ce)  // copy engine: host-readable block tables
      batch.push_back(dp_job{x.src_fb[engine_].data() + j.blk_off, x.slots[engine_].data() + j.blk_off,
                             j.cached, j.n_blk, 0, x.cfg.n_layer, j.ticket});
    else
      batch.push_back(dp_job{d_src_ + j.blk_off, d_slots_ + j.blk_off, j.cached, j.n_blk, 0,
                             x.cfg.n_layer, j.ticket});
    batch_jobs.push_back(static_cast<int>(i));
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
    std::vector<dp_job> batch;
    auto flush = [&]() {
      if (batch.empty()) return;
      const auto n = static_cast<int32_t>(batch.size());
      if (k1_ce) {
        check(dp_h2d_layer_copy(pool_, store_, batch.data(), n, s), "dp_h2d_layer_copy");
      } else {
        check(dp_h2d_layer_gather(pool_, store_, batch.data(), n, s), "dp_h2d_layer_gather");
        res.launches += (n + DP_MAX_JOBS_PER_LAUNCH - 1) / DP_MAX_JOBS_PER_LAUNCH;
      }
      batch.clear();
    };
    const double cap = x.opt.storage_cap_per_engine.empty() ? x.opt.storage_cap_Bps
                                                            : x.opt.storage_cap_per_engine[engine_];
    const double pace = x.opt.pace_scale;
    double gate_s = 0;
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
      // loads run ahead of the forwards (the compute stream's queue may be
      // long); they stop only for a slot reuse, whose reader forward must be
      // enqueued first, and for the storage gate, which lets the forwards
      // that are ready start before the host sleeps
      if (gated || !j.consumer_waits.empty()) forwards_before(r);
      if (gated || !j.consumer_waits.empty() || batch.size() == DP_MAX_JOBS_PER_LAUNCH) flush();
      for (int w : j.consumer_waits)
        check_cuda(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ev_fwd_[x.last_fwd[w]]), 0),
                   "cudaStreamWaitEvent");
      if (gated) {
        const double begin = std::max(gate_s, pace > 0 ? j.t_admit * pace : 0.0);
        gate_s = begin + (cap > 0 ? static_cast<double>(bytes) / cap : 0.0);
        std::this_thread::sleep_until(t0 + std::chrono::duration<double>(gate_s));
        res.spans.push_back({begin, gate_s, bytes});
      }
      if (k1_ce)
        batch.push_back(dp_job{x.src_fb[engine_].data() + j.blk_off, x.slots[engine_].data() + j.blk_off,
                               j.cached, j.n_blk, 0, L, j.ticket});
      else
        batch.push_back(dp_job{d_src_ + j.blk_off, d_slots_ + j.blk_off, j.cached, j.n_blk, 0, L, j.ticket});
      res.bytes_read += bytes;
      ++res.jobs;
    }
    flush();
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
    check(dp_prefill_attend(pool_, layer, att.data(), static_cast<int32_t>(att.size()), x.opt.seed, c),
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
  auto start = static_cast<cudaEvent_t>(ev_start_);
  check_cuda(cudaEventRecord(start, s), "cudaEventRecord");
  if (h) check_cuda(cudaStreamWaitEvent(h, start, 0), "cudaStreamWaitEvent");
  const std::int32_t L = x.cfg.n_layer;
  const double cap = x.opt.storage_cap_per_engine.empty() ? x.opt.storage_cap_Bps
                                                          : x.opt.storage_cap_per_engine[engine_];
  const double pace = x.opt.pace_scale;
  const bool gated = cap > 0 || pace > 0;
  double gate_s = 0;
  auto storage_gate = [&](const LoadJob& j) {
    const std::int64_t bytes = j.cached * x.cfg.kv_bytes_per_token();
    if (gated) {
      const double begin = std::max(gate_s, pace > 0 ? j.t_admit * pace : 0.0);
      gate_s = begin + (cap > 0 ? static_cast<double>(bytes) / cap : 0.0);
      std::this_thread::sleep_until(t0 + std::chrono::duration<double>(gate_s));
      res.spans.push_back({begin, gate_s, bytes});
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
    // K3 of one job on the handoff stream: decode-slot hazards, then K3
    auto enqueue_k3 = [&](int ji) {
      const LoadJob& j = x.jobs[ji];
      auto ev_k3 = static_cast<cudaEvent_t>(ev_k3_[pe_local_[ji]]);
      if (pf)  // the prompt is handed off after its last forward
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
      if (j.de_path && j.n_blk > 0 && !layer_gate) {
        check(dp_stream_wait_counter(pool_, j.ticket, L,
                                     static_cast<std::uint32_t>(static_cast<std::int64_t>(j.n_blk) *
                                                                x.items_per_block * L),
                                     h),
              "dp_stream_wait_counter");
      }
      dp_handoff_job hj{d_ho_src_ + j.ho_off,
                        d_ho_pe_ + j.ho_off,
                        d_ho_de_ + j.ho_off,
                        j.cached,
                        j.prompt,
                        j.n_pblk,
                        j.de_path ? 0 : 1,
                        (j.de_path && j.n_blk > 0 && layer_gate) ? j.ticket : -1,
                        static_cast<std::uint32_t>(static_cast<std::int64_t>(j.n_blk) * x.items_per_block),
                        j.de_ticket,
                        j.ticket + nt(engine_)};
      check(dp_prefill_handoff(pool_, de_views_[j.de], &hj, 1, x.opt.seed, x.opt.wait_timeout_ms, h),
            "dp_prefill_handoff");
      ++res.launches;
      check_cuda(cudaEventRecord(ev_k3, h), "cudaEventRecord");
    };
    // prefill: forwards whose requests' loads are all enqueued (row < r), and
    // the K3s of the requests they finish
    static const std::vector<Forward> kNone;
    const std::vector<Forward>& fwds = pf ? x.forwards[engine_] : kNone;
    std::size_t fi = 0, ki = 0;
    auto drain = [&](std::int64_t r) {
      while (fi < fwds.size() && fwds[fi].last_row < r) {
        enqueue_forward(static_cast<int>(fi++), res);
        while (ki < mine.size() && x.last_fwd[mine[ki]] < static_cast<int>(fi)) enqueue_k3(mine[ki++]);
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
          check(dp_h2d_layer_copy(pool_, store_, &job, 1, s), "dp_h2d_layer_copy");
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
    std::size_t ri = 0, di = 0;
    const auto& reads = x.by_reader[engine_];
    const auto& decodes = x.by_de[engine_];
    while (ri < reads.size() || (x.persist && di < decodes.size())) {
      // with the prefill, a request's K3 (which its decode waits for) needs
      // the loads of every request in its last forward: read those first
      const auto decode_key = [&](int ji) { return std::max(ji, x.jobs[ji].k3_after); };
      const bool take_read = ri < reads.size() &&
                             (!x.persist || di >= decodes.size() || reads[ri] <= decode_key(decodes[di]));
      if (take_read) {  // DE read path: dual gather
        const int ji = reads[ri++];
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
        check(dp_h2d_push_p2p_dual(peers_[j.pe], pool_, store_, &dj, 1, s), "dp_h2d_push_p2p_dual");
        ++res.launches;
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
      check(dp_persist_d2h(pool_, persist_store_, chunks.data(), static_cast<int32_t>(chunks.size()), h),
            "dp_persist_d2h");
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
  read_back_landed(res);
  res.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return res;
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
  const std::int32_t rows = is_pe() ? std::max<std::int32_t>(1, x.n_tickets[engine_]) * (x.handoff || x.prefill ? 2 : 1)
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
