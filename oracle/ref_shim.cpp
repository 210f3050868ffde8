// ref_shim — flat C entry points over the reference pdsim library, compiled
// from the reference's own sources where they lie (/root/reference/proj/src)
// into oracle/_ref/libpdsim_ref.so by oracle/Makefile.
//
// TEST INFRASTRUCTURE ONLY: the checker for scheduler decisions, byte ledgers
// and the synthetic-trace generator, and the CPU reference arm of bench.py.
// Nothing on the product path links or loads it.
//
// Reference interfaces wrapped (file:line under /root/reference/proj):
//   synthesize / save_trace / load_trace   src/workload.cpp:96-130, :78-94, :40-76
//   desim::run_offline / run_online        src/desim.cpp:1029-1051
//   schedule_pe_fetch                      src/scheduler.cpp:42-74
//   schedule_de_groups                     src/scheduler.cpp:76-93
//   schedule_de_within_group               src/scheduler.cpp:95-156
//   select_read_path                       src/scheduler.cpp:158-161
//   build_forward_batch                    src/scheduler.cpp:174-219
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "pdsim/desim.hpp"
#include "pdsim/scheduler.hpp"
#include "pdsim/types.hpp"
#include "pdsim/workload.hpp"

using namespace pdsim;

namespace {

thread_local std::string g_err;

std::map<std::string, std::string> parse_kv(const char* s) {
  std::map<std::string, std::string> out;
  std::string all = s ? s : "";
  size_t pos = 0;
  while (pos < all.size()) {
    size_t end = all.find(';', pos);
    if (end == std::string::npos) end = all.size();
    std::string item = all.substr(pos, end - pos);
    size_t eq = item.find('=');
    if (eq != std::string::npos) out[item.substr(0, eq)] = item.substr(eq + 1);
    pos = end + 1;
  }
  return out;
}

struct Kv {
  std::map<std::string, std::string> m;
  double d(const char* k, double def) const {
    auto it = m.find(k);
    return it == m.end() ? def : std::strtod(it->second.c_str(), nullptr);
  }
  long long i(const char* k, long long def) const {
    auto it = m.find(k);
    return it == m.end() ? def : std::strtoll(it->second.c_str(), nullptr, 10);
  }
  std::string s(const char* k, const char* def) const {
    auto it = m.find(k);
    return it == m.end() ? def : it->second;
  }
  bool has(const char* k) const { return m.count(k) != 0; }
};

void put(FILE* f, double v) { std::fprintf(f, "%.17g", v); }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_synthesize(int64_t max_len, double mean_turns, double mean_append, double mean_gen,
                   double sigma_turns, double sigma_append, double sigma_gen, int count,
                   uint64_t seed, const char* out_path) {
  try {
    SyntheticSpec spec;
    spec.max_len = max_len;
    spec.mean_turns = mean_turns;
    spec.mean_append = mean_append;
    spec.mean_gen = mean_gen;
    spec.sigma_turns = sigma_turns;
    spec.sigma_append = sigma_append;
    spec.sigma_gen = sigma_gen;
    spec.count = count;
    spec.seed = seed;
    const auto trajs = synthesize(spec);
    save_trace(std::string(out_path), trajs);
    return static_cast<int>(trajs.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// derive_variant / extend_with_synthetic_round of the reference
// (proj/src/workload.cpp:131-176) on a trace file, written back as a trace.
int ref_derive_variant(const char* in_path, double append_scale, double gen_scale,
                       int64_t max_len, const char* out_path) {
  try {
    const auto src = load_trace(std::string(in_path));
    save_trace(std::string(out_path), derive_variant(src, append_scale, gen_scale, max_len));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_extend_trace(const char* in_path, uint64_t seed, const char* out_path) {
  try {
    std::vector<Trajectory> out;
    for (const auto& t : load_trace(std::string(in_path)))
      out.push_back(extend_with_synthetic_round(t, seed));
    save_trace(std::string(out_path), out);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// poisson_arrivals (proj/src/workload.cpp:178-192): fills up to `cap` times,
// returns how many there are (may exceed cap), -1 on error.
int64_t ref_poisson(double rate, double horizon, uint64_t seed, double* out, int64_t cap) {
  try {
    const auto v = poisson_arrivals(rate, horizon, seed);
    for (int64_t i = 0; i < static_cast<int64_t>(v.size()) && i < cap; ++i) out[i] = v[i];
    return static_cast<int64_t>(v.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Runs the reference simulator on a trace file.  `kv` is "key=value;...".
// Writes a JSON report to out_path.  Returns 0, or -2 ConfigError,
// -3 SimulationError, -1 other.
int ref_simulate(const char* trace_path, const char* kv_str, const char* out_path) {
  try {
    Kv kv{parse_kv(kv_str)};
    ClusterConfig cfg;
    cfg.prefill_nodes = static_cast<int>(kv.i("P", cfg.prefill_nodes));
    cfg.decode_nodes = static_cast<int>(kv.i("D", cfg.decode_nodes));
    cfg.engines_per_node = static_cast<int>(kv.i("g", cfg.engines_per_node));
    cfg.cnic_bandwidth = kv.d("B", cfg.cnic_bandwidth);
    cfg.storage_multiple = kv.d("s", cfg.storage_multiple);
    cfg.dram_bandwidth = kv.d("M", cfg.dram_bandwidth);
    cfg.n_layer = static_cast<int>(kv.i("L", cfg.n_layer));
    cfg.kv_bytes_per_token_per_layer = kv.i("b", cfg.kv_bytes_per_token_per_layer);
    cfg.block_size_tokens = static_cast<int>(kv.i("T", cfg.block_size_tokens));
    cfg.hbm_capacity_tokens = kv.i("hbm", cfg.hbm_capacity_tokens);
    cfg.pe_buffer_bytes = kv.i("pe_buf", cfg.pe_buffer_bytes);
    cfg.de_buffer_bytes = kv.i("de_buf", cfg.de_buffer_bytes);

    desim::SimOptions opt;
    const std::string policy = kv.s("policy", "dual_path");
    if (policy == "dual_path") opt.policy = desim::Policy::DualPath;
    else if (policy == "pe_only") opt.policy = desim::Policy::PEOnly;
    else if (policy == "oracle") opt.policy = desim::Policy::Oracle;
    else throw std::invalid_argument("unknown policy " + policy);
    opt.sched_mode = kv.s("sched_mode", "adaptive") == "round_robin"
                         ? desim::SchedMode::RoundRobin
                         : desim::SchedMode::Adaptive;
    opt.sched.alpha = kv.i("alpha", opt.sched.alpha);
    opt.sched.beta = kv.i("beta", opt.sched.beta);
    opt.sched.z_factor = kv.d("z", opt.sched.z_factor);
    opt.sched.compute_quota = kv.d("quota", opt.sched.compute_quota);
    opt.cost.prefill.coeff_bilinear = kv.d("cb", 0);
    opt.cost.prefill.coeff_quadratic = kv.d("cq", 0);
    opt.cost.prefill.coeff_linear = kv.d("cl", 0);
    opt.cost.prefill.constant = kv.d("c0", 0);
    opt.cost.decode_per_ctx_token = kv.d("dctx", opt.cost.decode_per_ctx_token);
    opt.cost.decode_step_overhead = kv.d("dstep", opt.cost.decode_step_overhead);
    opt.submission_overhead = kv.d("sub", opt.submission_overhead);
    opt.batch_amortization = kv.d("amort", opt.batch_amortization);
    opt.bucket_width = kv.d("bucket", opt.bucket_width);
    opt.record_flows = kv.i("flows", 0) != 0;
    opt.record_events = kv.i("events", 0) != 0;
    opt.seed = static_cast<std::uint64_t>(kv.i("seed", 1));
    if (kv.has("burst_period")) {
      desim::BurstSpec b;
      b.period = kv.d("burst_period", b.period);
      b.bytes_per_burst = kv.d("burst_bytes", b.bytes_per_burst);
      b.start = kv.d("burst_start", b.start);
      b.stop = kv.d("burst_stop", b.stop);
      opt.bursts = b;
    }
    const auto trajs = load_trace(std::string(trace_path));
    desim::SimReport rep;
    const double aps = kv.d("aps", 0);
    if (aps > 0) {
      desim::SloSpec slo;
      slo.ttft_limit = kv.d("slo_ttft", slo.ttft_limit);
      slo.tpot_limit = kv.d("slo_tpot", slo.tpot_limit);
      desim::SteadySpec st;
      st.window = kv.d("steady_window", st.window);
      st.lookback = kv.d("steady_lookback", st.lookback);
      st.threshold = kv.d("steady_threshold", st.threshold);
      rep = desim::run_online(cfg, trajs, aps, slo, st, opt);
    } else {
      rep = desim::run_offline(cfg, trajs, opt);
    }
    FILE* f = std::fopen(out_path, "w");
    if (!f) throw std::runtime_error("cannot open output");
    std::fprintf(f, "{\"makespan\":");
    put(f, rep.makespan);
    std::fprintf(f, ",\"duration\":");
    put(f, rep.duration);
    std::fprintf(f, ",\"mean_jct\":");
    put(f, rep.mean_jct());
    std::fprintf(f, ",\"completed_requests\":%zu,\"total_requests\":%zu",
                 rep.completed_requests, rep.total_requests);
    std::fprintf(f, ",\"slo_violated\":%s,\"steady_state\":%s",
                 rep.slo_violated ? "true" : "false", rep.steady_state ? "true" : "false");
    std::fprintf(f, ",\"decisions\":[");
    for (size_t i = 0; i < rep.decisions.size(); ++i) {
      const auto& d = rep.decisions[i];
      std::fprintf(f, "%s[", i ? "," : "");
      put(f, d.t);
      std::fprintf(f, ",%d,%d,%d,%d,%d,%d]", d.request_id, d.pe, d.de,
                   d.path == ReadPath::PEPath ? 0 : 1, d.pe_category, d.de_category);
    }
    std::fprintf(f, "],\"flows\":[");
    for (size_t i = 0; i < rep.flows.size(); ++i) {
      const auto& fl = rep.flows[i];
      std::fprintf(f, "%s[%d,%d,", i ? "," : "", fl.request_id, static_cast<int>(fl.stage));
      put(f, fl.bytes);
      std::fprintf(f, ",");
      put(f, fl.t_start);
      std::fprintf(f, ",");
      put(f, fl.t_end);
      std::fprintf(f, "]");
    }
    std::fprintf(f, "],\"usage\":[");
    for (size_t i = 0; i < rep.usage.size(); ++i) {
      const auto& u = rep.usage[i];
      std::fprintf(f, "%s[\"%s\",%d,%d,", i ? "," : "", desim::to_string(u.kind), u.node_id,
                   u.engine_id);
      put(f, u.capacity);
      std::fprintf(f, ",");
      put(f, u.total_bytes);
      std::fprintf(f, ",[");
      for (size_t b = 0; b < u.buckets.size(); ++b) {
        if (b) std::fprintf(f, ",");
        put(f, u.buckets[b]);
      }
      std::fprintf(f, "]]");
    }
    std::fprintf(f, "],\"latencies\":[");
    for (size_t i = 0; i < rep.latencies.size(); ++i) {
      const auto& l = rep.latencies[i];
      std::fprintf(f, "%s[\"%s\"", i ? "," : "", l.request_id.c_str());
      for (double v : {l.ttft, l.ttst, l.tpot, l.sched_component, l.alloc_component,
                       l.read_component, l.prefill_component}) {
        std::fprintf(f, ",");
        put(f, v);
      }
      std::fprintf(f, "]");
    }
    std::fprintf(f, "],\"trajectory_jct\":[");
    for (size_t i = 0; i < rep.trajectory_jct.size(); ++i) {
      std::fprintf(f, "%s[\"%s\",", i ? "," : "", rep.trajectory_jct[i].first.c_str());
      put(f, rep.trajectory_jct[i].second);
      std::fprintf(f, "]");
    }
    std::fprintf(f, "],\"burst_latencies\":[");
    for (size_t i = 0; i < rep.burst_latencies.size(); ++i) {
      if (i) std::fprintf(f, ",");
      put(f, rep.burst_latencies[i]);
    }
    std::fprintf(f, "],\"event_log\":[");
    for (size_t i = 0; i < rep.event_log.size(); ++i)
      std::fprintf(f, "%s%s", i ? "," : "", rep.event_log[i].c_str());
    std::fprintf(f, "]}\n");
    std::fclose(f);
    return 0;
  } catch (const desim::ConfigError& e) {
    g_err = e.what();
    return -2;
  } catch (const desim::SimulationError& e) {
    g_err = e.what();
    return -3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// snaps: n x 6 int64 {engine_id, node_id, seq_e, tok_e, read_q, hbm_free_tokens}
static std::vector<EngineSnapshot> to_snaps(int n, const int64_t* s, EngineKind kind) {
  std::vector<EngineSnapshot> out(n);
  for (int i = 0; i < n; ++i) {
    out[i].engine_id = static_cast<int>(s[6 * i + 0]);
    out[i].node_id = static_cast<int>(s[6 * i + 1]);
    out[i].kind = kind;
    out[i].seq_e = s[6 * i + 2];
    out[i].tok_e = s[6 * i + 3];
    out[i].read_q = s[6 * i + 4];
    out[i].hbm_free_tokens = s[6 * i + 5];
  }
  return out;
}

static std::vector<PendingRequest> to_reqs(int n, const int* ids, const int64_t* tokens) {
  std::vector<PendingRequest> q(n);
  for (int i = 0; i < n; ++i) q[i] = {ids[i], tokens[i]};
  return q;
}

// out: up to n_req x 3 ints {request_id, engine_id, category}; returns count.
int ref_schedule_pe_fetch(int n_req, const int* ids, const int64_t* tokens, int n_pe,
                          const int64_t* snaps, int64_t alpha, int64_t beta, double z,
                          int* out) {
  try {
    SchedulerParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.z_factor = z;
    const auto q = to_reqs(n_req, ids, tokens);
    const auto s = to_snaps(n_pe, snaps, EngineKind::PE);
    const auto a = schedule_pe_fetch(q, s, p);
    for (size_t i = 0; i < a.size(); ++i) {
      out[3 * i] = a[i].request_id;
      out[3 * i + 1] = a[i].engine_id;
      out[3 * i + 2] = a[i].category;
    }
    return static_cast<int>(a.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_schedule_de_within_group(int n_req, const int* ids, const int64_t* tokens, int n_de,
                                 const int64_t* snaps, int64_t alpha, int64_t beta, double z,
                                 int* out) {
  try {
    SchedulerParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.z_factor = z;
    const auto q = to_reqs(n_req, ids, tokens);
    const auto s = to_snaps(n_de, snaps, EngineKind::DE);
    const auto a = schedule_de_within_group(q, s, p);
    for (size_t i = 0; i < a.size(); ++i) {
      out[3 * i] = a[i].request_id;
      out[3 * i + 1] = a[i].engine_id;
      out[3 * i + 2] = a[i].category;
    }
    return static_cast<int>(a.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// groups: n_grp x 2 int64 {group_id, tok_sum}; out: n_req x 2 {req, group}
int ref_schedule_de_groups(int n_req, const int* ids, const int64_t* tokens, int n_grp,
                           const int64_t* groups, int* out) {
  std::vector<GroupLoad> g(n_grp);
  for (int i = 0; i < n_grp; ++i) g[i] = {static_cast<int>(groups[2 * i]), groups[2 * i + 1]};
  const auto q = to_reqs(n_req, ids, tokens);
  const auto a = schedule_de_groups(q, g);
  for (size_t i = 0; i < a.size(); ++i) {
    out[2 * i] = a[i].first;
    out[2 * i + 1] = a[i].second;
  }
  return static_cast<int>(a.size());
}

int ref_select_read_path(int64_t pe_q, int64_t de_q) {
  return select_read_path(pe_q, de_q) == ReadPath::PEPath ? 0 : 1;
}

// build_forward_batch (src/scheduler.cpp:174-219).  items: n x 3 int64
// {request_id, cached, bsz}; cost: {bilinear, quadratic, linear, constant}.
// out_items: up to n x 3 {request_id, cached, bsz}; out_meta[4]: {chunked,
// chunked_request_id, chunk_bsz, consumed_whole}; *out_time = estimated_time.
// Returns the batch size, -2 on QuotaInfeasibleError, -1 on other errors.
int ref_build_forward_batch(int n, const int64_t* items, double quota, const double* cost,
                            int64_t* out_items, int64_t* out_meta, double* out_time) {
  try {
    std::vector<BatchItem> q(n);
    for (int i = 0; i < n; ++i)
      q[i] = {static_cast<int>(items[3 * i]), items[3 * i + 1], items[3 * i + 2]};
    SchedulerParams p;
    p.compute_quota = quota;
    AttentionCostModel m;
    m.coeff_bilinear = cost[0];
    m.coeff_quadratic = cost[1];
    m.coeff_linear = cost[2];
    m.constant = cost[3];
    const ForwardBatch fb = build_forward_batch(q, p, m);
    for (size_t i = 0; i < fb.items.size(); ++i) {
      out_items[3 * i] = fb.items[i].request_id;
      out_items[3 * i + 1] = fb.items[i].cached;
      out_items[3 * i + 2] = fb.items[i].bsz;
    }
    out_meta[0] = fb.chunked ? 1 : 0;
    out_meta[1] = fb.chunked_request_id;
    out_meta[2] = fb.chunk_bsz;
    out_meta[3] = fb.consumed_whole;
    *out_time = fb.estimated_time;
    return static_cast<int>(fb.items.size());
  } catch (const QuotaInfeasibleError& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int64_t ref_context_before_file(const char* trace_path, int traj, int round) {
  try {
    const auto t = load_trace(std::string(trace_path));
    return context_before(t.at(traj), static_cast<size_t>(round));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
