// Executor plan: planner decisions -> jobs, block tables, slots, hazards,
// prefill forwards and storage-tier staging (see dualpath/engine.hpp).
#include <algorithm>
#include <deque>
#include <stdexcept>
#include <string>
#include <limits>
#include <unordered_map>

#include "dualpath/engine.hpp"
#include "dualpath/storage.hpp"
#include "engine_detail.hpp"

namespace dualpath {

using detail::check;

namespace {

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

// The enqueue order of each DE in handoff + prefill mode.  Reads and
// decodes spin-wait on work of other engines, and in the worst case every
// stream of a device shares one hardware FIFO, so an operation also waits for
// everything enqueued before it on its device.  The orders are found by
// running the whole step in that model: each PE's sequence is the one its
// runtime enqueues (loads in FIFO order, forwards and the K3s they finish
// drained before a load that reuses slots or meets the storage gate), and
// each DE appends, among its next read per PE and its next decode, the one
// whose dependencies have completed (lowest job first).  A complete run of the
// model proves the orders cannot deadlock under one FIFO per device; a plan
// without one is rejected.
void build_de_orders(ExecPlan& x) {
  enum Kind : std::int64_t { kLoad = 0, kRead = 1, kK3 = 2, kDecode = 3, kFwd = 4 };
  const std::int64_t J = static_cast<std::int64_t>(x.jobs.size()) + 1;
  auto op = [&](Kind k, std::int64_t id) { return static_cast<std::int64_t>(k) * J * 64 + id; };
  auto fwd_op = [&](int p, int f) { return op(kFwd, static_cast<std::int64_t>(f) * 64 + p); };
  std::unordered_map<std::int64_t, char> done;
  auto is_done = [&](std::int64_t o) { return done.count(o) != 0; };
  const bool gated = x.opt.storage_cap_Bps > 0 || !x.opt.storage_cap_per_engine.empty() || x.opt.pace_scale > 0;
  if (x.n_pe > 64) throw std::invalid_argument("build_exec_plan: at most 64 PEs with handoff + prefill");

  auto fetch = [&](int y) { return x.jobs[y].reader == x.jobs[y].pe ? op(kLoad, y) : op(kRead, y); };
  auto add_release = [&](int q, std::vector<std::int64_t>& deps) {
    if (x.persist) {
      deps.push_back(op(kDecode, q));
    } else {
      deps.push_back(op(kK3, q));
      if (x.jobs[q].de_path && x.jobs[q].n_blk > 0) deps.push_back(op(kRead, q));
    }
  };
  struct Op {
    std::int64_t id;
    std::vector<std::int64_t> deps;
  };
  // each PE's enqueue sequence, as engine_handoff.cpp builds it
  std::vector<std::vector<Op>> pe_seq(x.n_pe);
  for (int p = 0; p < x.n_pe; ++p) {
    auto& seq = pe_seq[p];
    const auto& fwds = x.forwards[p];
    const auto& mine = x.by_pe[p];
    std::vector<int> row(x.jobs.size(), -1);
    for (const FwdItem& it : x.fwd_items[p])
      if (it.job >= 0) row[it.job] = it.row;
    std::size_t fi = 0, ki = 0;
    auto k3 = [&](int j) {
      Op o{op(kK3, j), {fwd_op(p, x.last_fwd[j])}};
      for (int q : x.jobs[j].de_pred_jobs) add_release(q, o.deps);
      seq.push_back(std::move(o));
    };
    auto drain = [&](std::int64_t r) {
      while (fi < fwds.size() && fwds[fi].last_row < r) {
        Op o{fwd_op(p, static_cast<int>(fi)), {}};
        for (std::int32_t i = fwds[fi].begin; i < fwds[fi].end; ++i) {
          const FwdItem& it = x.fwd_items[p][i];
          if (it.job >= 0 && it.cached > 0) o.deps.push_back(fetch(it.job));
        }
        seq.push_back(std::move(o));
        ++fi;
        while (ki < mine.size() && x.last_fwd[mine[ki]] < static_cast<int>(fi)) k3(mine[ki++]);
      }
    };
    for (int j : mine) {
      const LoadJob& lj = x.jobs[j];
      if (!lj.k3_waits.empty() || gated) drain(row[j]);
      if (!lj.de_path && lj.n_blk > 0) {
        Op o{op(kLoad, j), {}};
        for (int w : lj.k3_waits) o.deps.push_back(op(kK3, w));
        seq.push_back(std::move(o));
      }
    }
    drain(std::numeric_limits<std::int64_t>::max());
    while (ki < mine.size()) k3(mine[ki++]);
  }
  // the DEs' candidate operations
  const int n_de = x.n_engines - x.n_pe;
  std::vector<std::vector<std::vector<int>>> lists(n_de, std::vector<std::vector<int>>(x.n_pe));
  for (int d = 0; d < n_de; ++d)
    for (int ji : x.by_reader[x.n_pe + d]) lists[d][x.jobs[ji].pe].push_back(ji);
  std::vector<std::vector<std::size_t>> head(n_de, std::vector<std::size_t>(x.n_pe, 0));
  std::vector<std::size_t> dh(n_de, 0), ph(x.n_pe, 0);
  auto read_deps = [&](int ji) {
    std::vector<std::int64_t> deps;
    for (int q : x.jobs[ji].consumer_waits) deps.push_back(op(kK3, q));
    for (int q : x.jobs[ji].de_pred_jobs) add_release(q, deps);
    return deps;
  };
  auto decode_deps = [&](int j) {
    std::vector<std::int64_t> deps{op(kK3, j)};
    if (x.jobs[j].de_path && x.jobs[j].n_blk > 0) deps.push_back(op(kRead, j));
    return deps;
  };
  auto all_done = [&](const std::vector<std::int64_t>& deps) {
    for (std::int64_t d : deps)
      if (!is_done(d)) return false;
    return true;
  };
  x.de_order.assign(x.n_engines, {});
  std::size_t remaining = 0;
  for (int p = 0; p < x.n_pe; ++p) remaining += pe_seq[p].size();
  for (int d = 0; d < n_de; ++d)
    remaining += x.by_reader[x.n_pe + d].size() + (x.persist ? x.by_de[x.n_pe + d].size() : 0);
  while (remaining > 0) {
    bool progress = false;
    for (int p = 0; p < x.n_pe; ++p)
      while (ph[p] < pe_seq[p].size() && all_done(pe_seq[p][ph[p]].deps)) {
        done[pe_seq[p][ph[p]].id] = 1;
        ++ph[p];
        --remaining;
        progress = true;
      }
    for (int d = 0; d < n_de; ++d) {
      const int e = x.n_pe + d;
      const auto& decs = x.persist ? x.by_de[e] : std::vector<int>{};
      for (;;) {
        int best = -1;
        bool best_read = false;
        for (int p = 0; p < x.n_pe; ++p) {
          if (head[d][p] >= lists[d][p].size()) continue;
          const int ji = lists[d][p][head[d][p]];
          if ((best < 0 || ji < best) && all_done(read_deps(ji))) {
            best = ji;
            best_read = true;
          }
        }
        if (dh[d] < decs.size()) {
          const int jd = decs[dh[d]];
          if ((best < 0 || jd < best) && all_done(decode_deps(jd))) {
            best = jd;
            best_read = false;
          }
        }
        if (best < 0) break;
        if (best_read) {
          ++head[d][x.jobs[best].pe];
          done[op(kRead, best)] = 1;
          x.de_order[e].push_back(best);
        } else {
          ++dh[d];
          done[op(kDecode, best)] = 1;
          x.de_order[e].push_back(-1 - best);
        }
        --remaining;
        progress = true;
      }
    }
    if (!progress)
      throw std::logic_error("build_exec_plan: no deadlock-free enqueue order (handoff + prefill)");
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
  if (opt.pool_layout != 0 && opt.pool_layout != 1) throw std::invalid_argument("build_exec_plan: bad pool_layout");
  if (opt.pool_layout == 1 && x.handoff)
    throw std::invalid_argument("build_exec_plan: a block-major PE pool takes the load and prefill paths only");
  x.prefill = opt.prefill;
  if (x.prefill && !(opt.compute_quota > 0))
    throw std::invalid_argument("build_exec_plan: compute_quota must be > 0");
  x.tier = !opt.tier_path.empty();
  if (x.tier && x.handoff)
    throw std::invalid_argument("build_exec_plan: the storage tier runs on the load and prefill paths, not the handoff");
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
          if (std::find(j.fence_jobs.begin(), j.fence_jobs.end(), prev) == j.fence_jobs.end())
            j.fence_jobs.push_back(prev);
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
          j.de_pred_jobs.push_back(prev);  // -> global position below
          // with the prefill, the previous occupant is released after its
          // last forward (K3 follows it): on the same PE the two must not
          // share a forward
          if (x.prefill && pj.pe == j.pe &&
              std::find(j.consumer_waits.begin(), j.consumer_waits.end(), prev) == j.consumer_waits.end())
            j.consumer_waits.push_back(prev);
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
    for (int& w : j.de_pred_jobs) w = pos[w];
    for (int& w : j.fence_jobs) w = pos[w];
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
  if (x.prefill && x.handoff) build_de_orders(x);
  if (x.tier) build_tier(x, trajectories);
  return x;
}

}  // namespace dualpath
