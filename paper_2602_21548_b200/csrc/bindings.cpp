// _core: the Python shim of the DualPath B200 engine.
//
// Mirrors the reference module /root/reference/proj/python/bindings.cpp:83-190
// (ClusterConfig, Round, Trajectory, synthesize, load_trace, save_trace,
// simulate -> dict, ConfigError, SimulationError) and adds what the GPU path
// needs: the decision log in simulate()'s result (the parity artefact the
// reference does not export), the per-request plan, and the
// executor (ExecPlan / EngineRuntime).  The GIL is released around planning
// and GPU steps.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>

#include "dualpath/engine.hpp"
#include "dualpath/kv_abi.h"
#include "dualpath/live.hpp"
#include "pdsim/desim.hpp"
#include "pdsim/metrics.hpp"
#include "pdsim/scheduler.hpp"
#include "pdsim/types.hpp"
#include "pdsim/workload.hpp"

namespace py = pybind11;
using namespace pdsim;

namespace {

py::dict report_dict(const desim::SimReport& rep, bool with_flows) {
  py::dict d;
  d["makespan"] = rep.makespan;
  d["duration"] = rep.duration;
  d["completed_requests"] = rep.completed_requests;
  d["total_requests"] = rep.total_requests;
  d["mean_jct"] = rep.mean_jct();
  d["slo_violated"] = rep.slo_violated;
  d["steady_state"] = rep.steady_state;
  py::list lat;
  for (const auto& r : rep.latencies) {
    py::dict e;
    e["request_id"] = r.request_id;
    e["ttft"] = r.ttft;
    e["ttst"] = r.ttst;
    e["tpot"] = r.tpot;
    e["sched_component"] = r.sched_component;
    e["alloc_component"] = r.alloc_component;
    e["read_component"] = r.read_component;
    e["prefill_component"] = r.prefill_component;
    lat.append(e);
  }
  d["latencies"] = lat;
  py::list jct;
  for (const auto& [id, v] : rep.trajectory_jct) jct.append(py::make_tuple(id, v));
  d["trajectory_jct"] = jct;
  py::list usage;
  for (const auto& u : rep.usage) {
    py::dict e;
    e["kind"] = std::string(desim::to_string(u.kind));
    e["node_id"] = u.node_id;
    e["engine_id"] = u.engine_id;
    e["capacity"] = u.capacity;
    e["total_bytes"] = u.total_bytes;
    e["buckets"] = u.buckets;
    usage.append(e);
  }
  d["usage"] = usage;
  // [B200] decision log: (t, request, pe, de, path 0=pe/1=de, pe_cat, de_cat)
  py::list dec;
  for (const auto& x : rep.decisions)
    dec.append(py::make_tuple(x.t, x.request_id, x.pe, x.de, x.path == ReadPath::PEPath ? 0 : 1,
                              x.pe_category, x.de_category));
  d["decisions"] = dec;
  if (with_flows) {
    py::list fl;
    for (const auto& f : rep.flows)
      fl.append(py::make_tuple(f.request_id, static_cast<int>(f.stage), f.bytes, f.t_start, f.t_end));
    d["flows"] = fl;
    d["event_log"] = rep.event_log;
  }
  d["burst_latencies"] = rep.burst_latencies;
  d["events_processed"] = rep.events_processed;
  return d;
}

desim::SimOptions make_options(const std::string& policy, const std::string& sched_mode,
                               double alpha, double beta, std::uint64_t seed) {
  desim::SimOptions opt;
  if (policy == "dual_path") opt.policy = desim::Policy::DualPath;
  else if (policy == "pe_only") opt.policy = desim::Policy::PEOnly;
  else if (policy == "oracle") opt.policy = desim::Policy::Oracle;
  else throw std::invalid_argument("unknown policy '" + policy + "'");
  if (sched_mode == "adaptive") opt.sched_mode = desim::SchedMode::Adaptive;
  else if (sched_mode == "round_robin") opt.sched_mode = desim::SchedMode::RoundRobin;
  else throw std::invalid_argument("unknown sched_mode '" + sched_mode + "'");
  opt.sched.alpha = static_cast<std::int64_t>(alpha);
  opt.sched.beta = static_cast<std::int64_t>(beta);
  opt.seed = seed;
  return opt;
}

py::bytes handle_bytes(const dp_pool_handle& h) {
  return py::bytes(reinterpret_cast<const char*>(&h), sizeof(h));
}

dp_pool_handle handle_from(const py::bytes& b) {
  std::string s = b;
  if (s.size() != sizeof(dp_pool_handle)) throw std::invalid_argument("bad pool handle size");
  dp_pool_handle h;
  std::memcpy(&h, s.data(), sizeof(h));
  return h;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
  m.doc() = "DualPath KV-Cache loading on B200: planner (pdsim-compatible) and GPU executor";

  py::class_<ClusterConfig>(m, "ClusterConfig")
      .def(py::init<>())
      .def_readwrite("prefill_nodes", &ClusterConfig::prefill_nodes)
      .def_readwrite("decode_nodes", &ClusterConfig::decode_nodes)
      .def_readwrite("engines_per_node", &ClusterConfig::engines_per_node)
      .def_readwrite("cnic_bandwidth", &ClusterConfig::cnic_bandwidth)
      .def_readwrite("storage_multiple", &ClusterConfig::storage_multiple)
      .def_readwrite("dram_bandwidth", &ClusterConfig::dram_bandwidth)
      .def_readwrite("n_layer", &ClusterConfig::n_layer)
      .def_readwrite("kv_bytes_per_token_per_layer", &ClusterConfig::kv_bytes_per_token_per_layer)
      .def_readwrite("block_size_tokens", &ClusterConfig::block_size_tokens)
      .def_readwrite("hbm_capacity_tokens", &ClusterConfig::hbm_capacity_tokens)
      .def_readwrite("pe_buffer_bytes", &ClusterConfig::pe_buffer_bytes)
      .def_readwrite("de_buffer_bytes", &ClusterConfig::de_buffer_bytes)
      .def_readwrite("storage_bandwidth_per_node", &ClusterConfig::storage_bandwidth_per_node)
      .def("validate", &ClusterConfig::validate)
      .def("kv_bytes_per_token", &ClusterConfig::kv_bytes_per_token)
      .def("layer_block_bytes", &ClusterConfig::layer_block_bytes)
      .def("full_block_bytes", &ClusterConfig::full_block_bytes)
      .def("node_storage_bandwidth",
           [](const ClusterConfig& c, int node) { return node < 0 ? c.node_storage_bandwidth() : c.node_storage_bandwidth(node); },
           py::arg("node") = -1)
      .def("total_engines", &ClusterConfig::total_engines);

  py::class_<Round>(m, "Round")
      .def(py::init<>())
      .def(py::init([](std::int64_t a, std::int64_t g) { return Round{a, g}; }))
      .def_readwrite("append_tokens", &Round::append_tokens)
      .def_readwrite("gen_tokens", &Round::gen_tokens);

  py::class_<Trajectory>(m, "Trajectory")
      .def(py::init<>())
      .def_readwrite("id", &Trajectory::id)
      .def_readwrite("rounds", &Trajectory::rounds)
      .def("total_tokens", &Trajectory::total_tokens)
      .def("validate", &Trajectory::validate);

  m.def("context_before", &context_before);
  m.def("blocks_for", &blocks_for);

  m.def(
      "synthesize",
      [](std::int64_t max_len, int count, std::uint64_t seed, double mean_turns,
         double mean_append, double mean_gen, double sigma_turns, double sigma_append,
         double sigma_gen) {
        SyntheticSpec spec;
        spec.max_len = max_len;
        spec.count = count;
        spec.seed = seed;
        spec.mean_turns = mean_turns;
        spec.mean_append = mean_append;
        spec.mean_gen = mean_gen;
        spec.sigma_turns = sigma_turns;
        spec.sigma_append = sigma_append;
        spec.sigma_gen = sigma_gen;
        return synthesize(spec);
      },
      py::arg("max_len") = 65536, py::arg("count") = 16, py::arg("seed") = 1,
      py::arg("mean_turns") = 157.0, py::arg("mean_append") = 429.0, py::arg("mean_gen") = 176.0,
      py::arg("sigma_turns") = 0.5, py::arg("sigma_append") = 0.6, py::arg("sigma_gen") = 0.6);

  m.def(
      "derive_variant",
      [](const std::vector<Trajectory>& t, double append_scale, double gen_scale,
         std::int64_t max_len) { return derive_variant(t, append_scale, gen_scale, max_len); },
      py::arg("trajectories"), py::arg("append_scale"), py::arg("gen_scale"), py::arg("max_len"));
  m.def("extend_with_synthetic_round", &extend_with_synthetic_round, py::arg("base"),
        py::arg("seed"));
  m.def("poisson_arrivals", &poisson_arrivals, py::arg("rate"), py::arg("horizon"),
        py::arg("seed"));
  m.def("load_trace", &load_trace);
  m.def("save_trace", [](const std::string& path, const std::vector<Trajectory>& t) {
    save_trace(path, t);
  });

  // scheduler pure functions (snapshots as dicts-free tuples for tests)
  m.def("select_read_path", [](std::int64_t pe_q, std::int64_t de_q) {
    return select_read_path(pe_q, de_q) == ReadPath::PEPath ? 0 : 1;
  });
  auto to_snaps = [](const std::vector<std::vector<std::int64_t>>& rows, EngineKind kind) {
    std::vector<EngineSnapshot> s;
    for (const auto& r : rows) {
      if (r.size() != 6) throw std::invalid_argument("snapshot rows are 6-tuples");
      EngineSnapshot e;
      e.engine_id = static_cast<int>(r[0]);
      e.node_id = static_cast<int>(r[1]);
      e.kind = kind;
      e.seq_e = r[2];
      e.tok_e = r[3];
      e.read_q = r[4];
      e.hbm_free_tokens = r[5];
      s.push_back(e);
    }
    return s;
  };
  auto to_reqs = [](const std::vector<std::pair<int, std::int64_t>>& q) {
    std::vector<PendingRequest> out;
    for (const auto& [id, t] : q) out.push_back({id, t});
    return out;
  };
  auto params = [](std::int64_t alpha, std::int64_t beta, double z) {
    SchedulerParams p;
    p.alpha = alpha;
    p.beta = beta;
    p.z_factor = z;
    return p;
  };
  // Intra-engine compute-quota batching (scheduler.hpp build_forward_batch).
  // items: [(request_id, cached, bsz)]; cost: (bilinear, quadratic, linear,
  // constant).  Returns (items, chunked, chunked_request_id, chunk_bsz,
  // consumed_whole, estimated_time).
  auto cost_of = [](const std::tuple<double, double, double, double>& c) {
    AttentionCostModel m;
    std::tie(m.coeff_bilinear, m.coeff_quadratic, m.coeff_linear, m.constant) = c;
    return m;
  };
  auto items_of = [](const std::vector<std::tuple<int, std::int64_t, std::int64_t>>& v) {
    std::vector<BatchItem> q;
    q.reserve(v.size());
    for (const auto& [id, cached, bsz] : v) q.push_back({id, cached, bsz});
    return q;
  };
  m.def(
      "estimate_attention_time",
      [=](const std::vector<std::tuple<int, std::int64_t, std::int64_t>>& batch,
          const std::tuple<double, double, double, double>& cost) {
        return estimate_attention_time(items_of(batch), cost_of(cost));
      },
      py::arg("batch"), py::arg("cost"));
  m.def(
      "build_forward_batch",
      [=](const std::vector<std::tuple<int, std::int64_t, std::int64_t>>& queue, double quota,
          const std::tuple<double, double, double, double>& cost) {
        SchedulerParams p;
        p.compute_quota = quota;
        const ForwardBatch fb = build_forward_batch(items_of(queue), p, cost_of(cost));
        std::vector<std::tuple<int, std::int64_t, std::int64_t>> items;
        for (const BatchItem& b : fb.items) items.emplace_back(b.request_id, b.cached, b.bsz);
        return py::make_tuple(items, fb.chunked, fb.chunked_request_id, fb.chunk_bsz,
                              fb.consumed_whole, fb.estimated_time);
      },
      py::arg("queue"), py::arg("quota"), py::arg("cost"));
  m.def("schedule_pe_fetch",
        [=](const std::vector<std::pair<int, std::int64_t>>& q,
            const std::vector<std::vector<std::int64_t>>& snaps, std::int64_t alpha,
            std::int64_t beta, double z) {
          std::vector<std::tuple<int, int, int>> out;
          for (const auto& a :
               schedule_pe_fetch(to_reqs(q), to_snaps(snaps, EngineKind::PE), params(alpha, beta, z)))
            out.emplace_back(a.request_id, a.engine_id, a.category);
          return out;
        });
  m.def("schedule_de_within_group",
        [=](const std::vector<std::pair<int, std::int64_t>>& q,
            const std::vector<std::vector<std::int64_t>>& snaps, std::int64_t alpha,
            std::int64_t beta, double z) {
          std::vector<std::tuple<int, int, int>> out;
          for (const auto& a : schedule_de_within_group(to_reqs(q), to_snaps(snaps, EngineKind::DE),
                                                        params(alpha, beta, z)))
            out.emplace_back(a.request_id, a.engine_id, a.category);
          return out;
        });
  m.def("schedule_de_groups", [=](const std::vector<std::pair<int, std::int64_t>>& q,
                                  const std::vector<std::pair<int, std::int64_t>>& groups) {
    std::vector<GroupLoad> g;
    for (const auto& [id, t] : groups) g.push_back({id, t});
    return schedule_de_groups(to_reqs(q), g);
  });

  // Full-control planner entry: every SimOptions field by keyword.
  m.def(
      "plan",
      [](const ClusterConfig& cfg, const std::vector<Trajectory>& trajs, const std::string& policy,
         const std::string& sched_mode, std::int64_t alpha, std::int64_t beta, double z,
         double quota, double cb, double cq, double cl, double c0, double dctx, double dstep,
         double sub, double amort, double bucket, bool flows, bool events, double aps,
         std::uint64_t seed, double slo_ttft, double slo_tpot, double steady_window,
         double steady_lookback, double steady_threshold, double burst_period,
         double burst_bytes, double burst_start, double burst_stop) {
        desim::SimOptions opt = make_options(policy, sched_mode, static_cast<double>(alpha),
                                             static_cast<double>(beta), seed);
        opt.sched.z_factor = z;
        opt.sched.compute_quota = quota;
        opt.cost.prefill = {cb, cq, cl, c0};
        opt.cost.decode_per_ctx_token = dctx;
        opt.cost.decode_step_overhead = dstep;
        opt.submission_overhead = sub;
        opt.batch_amortization = amort;
        opt.bucket_width = bucket;
        opt.record_flows = flows;
        opt.record_events = events;
        if (burst_period > 0) opt.bursts = desim::BurstSpec{burst_period, burst_bytes, burst_start, burst_stop};
        desim::SimReport rep;
        {
          py::gil_scoped_release nogil;
          if (aps > 0) {
            desim::SloSpec slo{slo_ttft, slo_tpot};
            desim::SteadySpec st{steady_window, steady_lookback, steady_threshold};
            rep = desim::run_online(cfg, trajs, aps, slo, st, opt);
          } else {
            rep = desim::run_offline(cfg, trajs, opt);
          }
        }
        py::dict d = report_dict(rep, flows || events);
        py::list reqs;
        for (const auto& r : rep.requests)
          reqs.append(py::make_tuple(r.request_id, r.traj_index, r.round, r.cached, r.append, r.gen,
                                     r.pe, r.de, r.path == ReadPath::PEPath ? 0 : 1, r.t_arrival,
                                     r.t_sched, r.t_admit, r.t_read_done, r.t_pe_release, r.t_done));
        d["requests"] = reqs;
        return d;
      },
      py::arg("cluster"), py::arg("trajectories"), py::arg("policy") = "dual_path",
      py::arg("sched_mode") = "adaptive", py::arg("alpha") = 100000, py::arg("beta") = 500000,
      py::arg("z") = 1.05, py::arg("quota") = 0.3, py::arg("cb") = 0.0, py::arg("cq") = 0.0,
      py::arg("cl") = 0.0, py::arg("c0") = 0.0, py::arg("dctx") = 0.0, py::arg("dstep") = 2e-3,
      py::arg("sub") = 1e-6, py::arg("amort") = 1.0, py::arg("bucket") = 0.5,
      py::arg("flows") = false, py::arg("events") = false, py::arg("aps") = 0.0,
      py::arg("seed") = 1, py::arg("slo_ttft") = 4.0, py::arg("slo_tpot") = 0.05,
      py::arg("steady_window") = 15.0, py::arg("steady_lookback") = 180.0,
      py::arg("steady_threshold") = 0.05, py::arg("burst_period") = 0.0,
      py::arg("burst_bytes") = 1e6, py::arg("burst_start") = 0.0, py::arg("burst_stop") = 1.0);

  // Reference-shaped entry (bindings.cpp:169-186) plus the decision log.
  m.def(
      "simulate",
      [](const ClusterConfig& cfg, const std::vector<Trajectory>& trajs, const std::string& policy,
         const std::string& sched_mode, double alpha, double beta, double aps, std::uint64_t seed) {
        desim::SimOptions opt = make_options(policy, sched_mode, alpha, beta, seed);
        desim::SimReport rep;
        {
          py::gil_scoped_release nogil;
          if (aps > 0) {
            desim::SloSpec slo;
            desim::SteadySpec st;
            rep = desim::run_online(cfg, trajs, aps, slo, st, opt);
          } else {
            rep = desim::run_offline(cfg, trajs, opt);
          }
        }
        return report_dict(rep, false);
      },
      py::arg("cluster"), py::arg("trajectories"), py::arg("policy") = "dual_path",
      py::arg("sched_mode") = "adaptive", py::arg("alpha") = 100000, py::arg("beta") = 500000,
      py::arg("aps") = 0.0, py::arg("seed") = 0);

  m.def("load_balance_ratio",
        [](const std::vector<std::vector<double>>& series, double bucket_width, int window) {
          std::vector<std::tuple<double, double, bool>> out;
          for (const auto& p : load_balance_ratio(series, bucket_width, window))
            out.emplace_back(p.t, p.max_avg, p.defined);
          return out;
        });

  py::register_exception<QuotaInfeasibleError>(m, "QuotaInfeasibleError", PyExc_RuntimeError);
  py::register_exception<desim::ConfigError>(m, "ConfigError");
  py::register_exception<desim::SimulationError>(m, "SimulationError");

  // ---------------------------------------------------------------- executor
  // ---- storage tier (dualpath/storage.hpp) ----
  auto geom_of = [](int L, int T, std::int64_t b) { return dp_kv_geom{L, T, b}; };
  m.def("session_chain", &dualpath::session_chain, py::arg("id"), py::arg("n_blocks"));
  py::class_<dualpath::FullBlockTrie>(m, "FullBlockTrie")
      .def(py::init<>())
      .def("insert",
           [](dualpath::FullBlockTrie& t, const std::vector<std::uint64_t>& chain,
              const std::vector<std::int64_t>& records) { return t.insert(chain, records); })
      .def("match", [](const dualpath::FullBlockTrie& t,
                       const std::vector<std::uint64_t>& chain) { return t.match(chain); })
      .def("nodes", &dualpath::FullBlockTrie::nodes)
      .def("save", &dualpath::FullBlockTrie::save)
      .def_static("load", &dualpath::FullBlockTrie::load);
  py::class_<dualpath::FullBlockFile>(m, "FullBlockFile")
      .def(py::init([=](const std::string& path, int L, int T, std::int64_t b, std::int64_t n_records,
                        bool create, bool direct) {
             return std::make_unique<dualpath::FullBlockFile>(path, geom_of(L, T, b), n_records, create, direct);
           }),
           py::arg("path"), py::arg("n_layer"), py::arg("block_tokens"), py::arg("bytes_per_token_layer"),
           py::arg("n_records"), py::arg("create") = false, py::arg("direct") = true)
      .def("populate", &dualpath::FullBlockFile::populate, py::arg("seed"), py::arg("threads") = 8,
           py::call_guard<py::gil_scoped_release>())
      .def("read",
           [](const dualpath::FullBlockFile& f, std::int64_t record) {
             std::string buf(static_cast<std::size_t>(f.record_bytes()), '\0');
             f.read(record, buf.data());
             return py::bytes(buf);
           })
      .def("read_run",
           [](const dualpath::FullBlockFile& f, std::int64_t record, std::int64_t n) {
             std::string buf(static_cast<std::size_t>(f.record_bytes() * std::max<std::int64_t>(0, n)), '\0');
             f.read_run(record, n, buf.data());
             return py::bytes(buf);
           })
      .def("records", &dualpath::FullBlockFile::records)
      .def("record_bytes", &dualpath::FullBlockFile::record_bytes)
      .def("stride", &dualpath::FullBlockFile::stride)
      .def("direct", &dualpath::FullBlockFile::direct);

  py::class_<dualpath::ExecOptions>(m, "ExecOptions")
      .def(py::init<>())
      .def_readwrite("storage_cap_Bps", &dualpath::ExecOptions::storage_cap_Bps)
      .def_readwrite("buffer_bound", &dualpath::ExecOptions::buffer_bound)
      .def_readwrite("persist_path", &dualpath::ExecOptions::persist_path)
      .def_readwrite("storage_cap_per_engine", &dualpath::ExecOptions::storage_cap_per_engine)
      .def_readwrite("pace_scale", &dualpath::ExecOptions::pace_scale)
      .def_readwrite("k1_mode", &dualpath::ExecOptions::k1_mode)
      .def_readwrite("k2_mode", &dualpath::ExecOptions::k2_mode)
      .def_readwrite("stage_ring_bytes", &dualpath::ExecOptions::stage_ring_bytes)
      .def_readwrite("stage_ctas", &dualpath::ExecOptions::stage_ctas)
      .def_readwrite("stage_scatter", &dualpath::ExecOptions::stage_scatter)
      .def_readwrite("copy_release_per_job", &dualpath::ExecOptions::copy_release_per_job)
      .def_readwrite("stage_push_ctas", &dualpath::ExecOptions::stage_push_ctas)
      .def_readwrite("handoff", &dualpath::ExecOptions::handoff)
      .def_readwrite("de_pool_slots", &dualpath::ExecOptions::de_pool_slots)
      .def_readwrite("gather_ctas", &dualpath::ExecOptions::gather_ctas)
      .def_readwrite("k3_layer_gate", &dualpath::ExecOptions::k3_layer_gate)
      .def_readwrite("handoff_layerwise", &dualpath::ExecOptions::handoff_layerwise)
      .def_readwrite("handoff_tma", &dualpath::ExecOptions::handoff_tma)
      .def_readwrite("k3_mode", &dualpath::ExecOptions::k3_mode)
      .def_readwrite("persist_mode", &dualpath::ExecOptions::persist_mode)
      .def_readwrite("pool_layout", &dualpath::ExecOptions::pool_layout)
      .def_readwrite("handoff_ctas", &dualpath::ExecOptions::handoff_ctas)
      .def_readwrite("persist", &dualpath::ExecOptions::persist)
      .def_readwrite("store_fb", &dualpath::ExecOptions::store_fb)
      .def_readwrite("store_bytes_max", &dualpath::ExecOptions::store_bytes_max)
      .def_readwrite("seed", &dualpath::ExecOptions::seed)
      .def_readwrite("pool_slots", &dualpath::ExecOptions::pool_slots)
      .def_readwrite("pool_bytes_max", &dualpath::ExecOptions::pool_bytes_max)
      .def_readwrite("wait_timeout_ms", &dualpath::ExecOptions::wait_timeout_ms)
      .def_readwrite("tier_path", &dualpath::ExecOptions::tier_path)
      .def_readwrite("tier_ring_fb", &dualpath::ExecOptions::tier_ring_fb)
      .def_readwrite("io_threads", &dualpath::ExecOptions::io_threads)
      .def_readwrite("tier_direct", &dualpath::ExecOptions::tier_direct)
      .def_readwrite("prefill", &dualpath::ExecOptions::prefill)
      .def_readwrite("compute_quota", &dualpath::ExecOptions::compute_quota)
      .def_readwrite("attend_ctas", &dualpath::ExecOptions::attend_ctas)
      .def_property(
          "prefill_cost",
          [](const dualpath::ExecOptions& o) {
            const auto& m = o.prefill_cost;
            return std::make_tuple(m.coeff_bilinear, m.coeff_quadratic, m.coeff_linear, m.constant);
          },
          [](dualpath::ExecOptions& o, const std::tuple<double, double, double, double>& c) {
            auto& m = o.prefill_cost;
            std::tie(m.coeff_bilinear, m.coeff_quadratic, m.coeff_linear, m.constant) = c;
          });

  py::class_<dualpath::ExecPlan, std::shared_ptr<dualpath::ExecPlan>>(m, "ExecPlan")
      .def_readonly("n_engines", &dualpath::ExecPlan::n_engines)
      .def_readonly("n_pe", &dualpath::ExecPlan::n_pe)
      .def_readonly("store_fb", &dualpath::ExecPlan::store_fb)
      .def_readonly("fb_stride", &dualpath::ExecPlan::fb_stride)
      .def_readonly("pool_slots", &dualpath::ExecPlan::pool_slots)
      .def_readonly("peak_slots", &dualpath::ExecPlan::peak_slots)
      .def_readonly("items_per_block", &dualpath::ExecPlan::items_per_block)
      .def_readonly("n_tickets", &dualpath::ExecPlan::n_tickets)
      .def_readonly("reader_bytes", &dualpath::ExecPlan::reader_bytes)
      .def_readonly("hit_bytes", &dualpath::ExecPlan::hit_bytes)
      .def_readonly("prompt_tokens", &dualpath::ExecPlan::prompt_tokens)
      .def_readonly("requests", &dualpath::ExecPlan::requests)
      .def_readonly("handoff", &dualpath::ExecPlan::handoff)
      .def_readonly("handoff_bytes", &dualpath::ExecPlan::handoff_bytes)
      .def_readonly("persist", &dualpath::ExecPlan::persist)
      .def_readonly("persist_bytes", &dualpath::ExecPlan::persist_bytes)
      .def("persist_chunks", [](const dualpath::ExecPlan& x, int job) { return x.persist_chunks(x.jobs.at(job)); })
      .def("job_gen", [](const dualpath::ExecPlan& x, int job) { return x.jobs.at(job).gen; })
      .def_readonly("de_pool_slots", &dualpath::ExecPlan::de_pool_slots)
      .def_readonly("de_peak_slots", &dualpath::ExecPlan::de_peak_slots)
      .def_readonly("n_de_tickets", &dualpath::ExecPlan::n_de_tickets)
      .def("fb_of", &dualpath::ExecPlan::fb_of)
      .def("jobs", [](const dualpath::ExecPlan& x) {
        // (req, traj, round, reader, pe, de_path, cached, n_blk, ticket, slots, src_fb, preds,
        //  fence, de, prompt, n_pblk, de_ticket, pe_prompt_slots, de_slots, de_preds, k3_waits,
        //  pe_done_preds)
        py::list out;
        for (const auto& j : x.jobs) {
          std::vector<std::int32_t> sl(x.slots[j.reader].begin() + j.blk_off,
                                       x.slots[j.reader].begin() + j.blk_off + j.n_blk);
          std::vector<std::int64_t> fb(x.src_fb[j.reader].begin() + j.blk_off,
                                       x.src_fb[j.reader].begin() + j.blk_off + j.n_blk);
          std::vector<std::int32_t> ps, dsl;
          if (x.handoff) {
            ps.assign(x.ho_pe_slot[j.pe].begin() + j.ho_off, x.ho_pe_slot[j.pe].begin() + j.ho_off + j.n_pblk);
            dsl.assign(x.ho_de_slot[j.pe].begin() + j.ho_off, x.ho_de_slot[j.pe].begin() + j.ho_off + j.n_pblk);
          } else {
            ps = sl;
          }
          py::tuple t = py::make_tuple(j.req, j.traj, j.round, j.reader, j.pe, j.de_path, j.cached,
                                       j.n_blk, j.ticket, sl, fb, j.preds);
          py::tuple u = py::make_tuple(j.fence, j.de, j.prompt, j.n_pblk, j.de_ticket, ps, dsl,
                                       j.de_preds, j.k3_waits, j.pe_done_preds);
          out.append(py::reinterpret_steal<py::tuple>(PySequence_Concat(t.ptr(), u.ptr())));
        }
        return out;
      })
      .def("by_reader", [](const dualpath::ExecPlan& x, int e) { return x.by_reader.at(e); })
      .def("by_pe", [](const dualpath::ExecPlan& x, int e) { return x.by_pe.at(e); })
      .def("by_de", [](const dualpath::ExecPlan& x, int e) { return x.by_de.at(e); })
      .def_readonly("prefill", &dualpath::ExecPlan::prefill)
      .def_readonly("tier", &dualpath::ExecPlan::tier)
      .def_readonly("ring_fb", &dualpath::ExecPlan::ring_fb)
      .def_readonly("trie_nodes", &dualpath::ExecPlan::trie_nodes)
      .def("tier_rec", [](const dualpath::ExecPlan& x, int e) { return x.tier_rec.at(e); })
      .def("src_fb", [](const dualpath::ExecPlan& x, int e) { return x.src_fb.at(e); })
      .def("ring_waits", [](const dualpath::ExecPlan& x, int job) { return x.jobs.at(job).ring_waits; })
      // forwards(pe) -> [(estimated_time, [(req, job, cached, q_begin, bsz, row)])]
      .def("forwards",
           [](const dualpath::ExecPlan& x, int pe) {
             py::list out;
             for (const dualpath::Forward& f : x.forwards.at(pe)) {
               py::list items;
               for (std::int32_t i = f.begin; i < f.end; ++i) {
                 const dualpath::FwdItem& it = x.fwd_items.at(pe)[i];
                 items.append(py::make_tuple(it.req, it.job, it.cached, it.q_begin, it.bsz, it.row));
               }
               out.append(py::make_tuple(f.estimated_time, items));
             }
             return out;
           })
      .def("fwd_rows", [](const dualpath::ExecPlan& x, int pe) { return x.fwd_rows.at(pe); })
      .def("consumer_waits", [](const dualpath::ExecPlan& x, int job) { return x.jobs.at(job).consumer_waits; })
      .def("last_fwd", [](const dualpath::ExecPlan& x, int job) { return x.last_fwd.at(job); })
      .def("de_order", [](const dualpath::ExecPlan& x, int e) {
        return e < static_cast<int>(x.de_order.size()) ? x.de_order[e] : std::vector<int>{};
      })
      .def("de_pred_jobs", [](const dualpath::ExecPlan& x, int job) { return x.jobs.at(job).de_pred_jobs; })
      .def("fwd_slots", [](const dualpath::ExecPlan& x, int job) {
        const dualpath::LoadJob& j = x.jobs.at(job);
        const auto& t = x.fwd_slot.at(j.pe);
        return std::vector<std::int32_t>(t.begin() + j.fwd_off, t.begin() + j.fwd_off + j.n_blk);
      });

  m.def(
      "build_exec_plan",
      [](const ClusterConfig& cfg, const std::vector<Trajectory>& trajs, const py::dict& planned,
         const dualpath::ExecOptions& opt) {
        // rebuild the RequestPlan list from plan()'s "requests" tuples
        desim::SimReport rep;
        for (const auto& item : planned["requests"].cast<py::list>()) {
          auto t = item.cast<py::tuple>();
          desim::RequestPlan r;
          r.request_id = t[0].cast<int>();
          r.traj_index = t[1].cast<int>();
          r.round = t[2].cast<int>();
          r.cached = t[3].cast<std::int64_t>();
          r.append = t[4].cast<std::int64_t>();
          r.gen = t[5].cast<std::int64_t>();
          r.pe = t[6].cast<int>();
          r.de = t[7].cast<int>();
          r.path = t[8].cast<int>() == 0 ? ReadPath::PEPath : ReadPath::DEPath;
          r.t_arrival = t[9].cast<double>();
          r.t_sched = t[10].cast<double>();
          r.t_admit = t[11].cast<double>();
          r.t_read_done = t[12].cast<double>();
          r.t_pe_release = t[13].cast<double>();
          r.t_done = t[14].cast<double>();
          rep.requests.push_back(r);
        }
        py::gil_scoped_release nogil;
        return std::make_shared<dualpath::ExecPlan>(dualpath::build_exec_plan(cfg, trajs, rep, opt));
      },
      py::arg("cluster"), py::arg("trajectories"), py::arg("planned"), py::arg("options"));

  py::class_<dualpath::StepResult>(m, "StepResult")
      .def_property_readonly("spans",
                             [](const dualpath::StepResult& r) {
                               std::vector<std::tuple<double, double, std::int64_t>> v;
                               for (const auto& s : r.spans) v.emplace_back(s.t_begin, s.t_end, s.bytes);
                               return v;
                             })
      .def_readonly("device_ms", &dualpath::StepResult::device_ms)
      .def_readonly("host_ms", &dualpath::StepResult::host_ms)
      .def_readonly("bytes_read", &dualpath::StepResult::bytes_read)
      .def_readonly("launches", &dualpath::StepResult::launches)
      .def_readonly("jobs", &dualpath::StepResult::jobs)
      .def_readonly("forwards", &dualpath::StepResult::forwards)
      .def_readonly("io_wait_ms", &dualpath::StepResult::io_wait_ms)
      .def_readonly("d2h_bytes", &dualpath::StepResult::d2h_bytes)
      .def_readonly("ttft_ms", &dualpath::StepResult::ttft_ms)
      .def_readonly("buffer_stalls", &dualpath::StepResult::buffer_stalls)
      .def_readonly("persist_write_ms", &dualpath::StepResult::persist_write_ms)
      .def_readonly("persist_write_bytes", &dualpath::StepResult::persist_write_bytes)
      .def_readonly("buffer_wait_ms", &dualpath::StepResult::buffer_wait_ms)
      .def_readonly("handoff_lag_ms", &dualpath::StepResult::handoff_lag_ms);

  py::class_<dualpath::EngineRuntime>(m, "EngineRuntime")
      .def(py::init([](std::shared_ptr<dualpath::ExecPlan> plan, int engine, int device) {
             py::gil_scoped_release nogil;
             return std::make_unique<dualpath::EngineRuntime>(plan, engine, device);
           }),
           py::arg("plan"), py::arg("engine"), py::arg("device"))
      .def_property_readonly("engine", &dualpath::EngineRuntime::engine)
      .def_property_readonly("device", &dualpath::EngineRuntime::device)
      .def_property_readonly("is_pe", &dualpath::EngineRuntime::is_pe)
      .def_property_readonly("has_pool", &dualpath::EngineRuntime::has_pool)
      .def("export_pool", [](const dualpath::EngineRuntime& e) { return handle_bytes(e.export_pool()); })
      .def("attach_peer", [](dualpath::EngineRuntime& e, int pe, const py::bytes& h) {
        e.attach_peer(pe, handle_from(h));
      })
      .def("attach_peer_local", &dualpath::EngineRuntime::attach_peer_local)
      .def("reset_counters", &dualpath::EngineRuntime::reset_counters)
      .def("run_step", &dualpath::EngineRuntime::run_step, py::call_guard<py::gil_scoped_release>())
      .def("run_forwards", &dualpath::EngineRuntime::run_forwards, py::call_guard<py::gil_scoped_release>())
      .def("prefill_digests", &dualpath::EngineRuntime::prefill_digests)
      .def("checksum",
           [](dualpath::EngineRuntime& e, int layer, const std::vector<std::int32_t>& slots,
              const std::vector<std::int32_t>& ntok) { return e.checksum(layer, slots, ntok); })
      .def("counters", &dualpath::EngineRuntime::counters)
      .def("read_persisted", [](const dualpath::EngineRuntime& e, std::int64_t fb, int layer) {
        const auto v = e.read_persisted(fb, layer);
        return py::bytes(reinterpret_cast<const char*>(v.data()), v.size());
      });

  // Live-mode scheduling (dualpath/live.hpp): the reference's scheduler on
  // measured state while K1 / K2 move the bytes; every invocation logged.
  m.def(
      "run_live",
      [](const ClusterConfig& cfg, const std::vector<Trajectory>& trajs, const std::string& policy,
         const std::string& sched_mode, std::int64_t alpha, std::int64_t beta, double z,
         const dualpath::ExecOptions& exec, std::int32_t pe_pool_slots, double decode_s_per_token, bool gpu,
         double link_Bps, const std::vector<int>& devices, double timeout_s,
         const std::vector<double>& arrival_times, double slo_ttft, double steady_window,
         double steady_lookback, double steady_threshold, std::int32_t de_pool_slots) {
        dualpath::LiveOptions o;
        o.arrival_times = arrival_times;
        o.slo_ttft_s = slo_ttft;
        o.steady_window = steady_window;
        o.steady_lookback = steady_lookback;
        o.steady_threshold = steady_threshold;
        o.sim = make_options(policy, sched_mode, static_cast<double>(alpha), static_cast<double>(beta), 1);
        o.sim.sched.z_factor = z;
        o.exec = exec;
        o.pe_pool_slots = pe_pool_slots;
        o.de_pool_slots = de_pool_slots;
        o.decode_s_per_token = decode_s_per_token;
        o.gpu = gpu;
        o.link_Bps = link_Bps;
        o.devices = devices;
        o.timeout_s = timeout_s;
        dualpath::LiveReport rep;
        {
          py::gil_scoped_release nogil;
          rep = dualpath::run_live(cfg, trajs, o);
        }
        py::dict d;
        py::list dec;
        for (const auto& x : rep.decisions)
          dec.append(py::make_tuple(x.t, x.request_id, x.pe, x.de, x.path == ReadPath::PEPath ? 0 : 1,
                                    x.pe_category, x.de_category));
        d["decisions"] = dec;
        py::list inv;
        for (const auto& v : rep.invocations) {
          py::dict e;
          e["fn"] = v.fn;
          e["t"] = v.t;
          py::list q, sn, gr, out;
          for (const auto& p : v.queue) q.append(py::make_tuple(p.id, p.tokens));
          for (const auto& x : v.snapshots)
            sn.append(py::make_tuple(x.engine_id, x.node_id, x.kind == EngineKind::PE ? 0 : 1, x.seq_e, x.tok_e,
                                     x.read_q, x.hbm_free_tokens));
          for (const auto& g : v.groups) gr.append(py::make_tuple(g.group_id, g.tok_sum));
          for (const auto& a : v.out) out.append(py::make_tuple(a.request_id, a.engine_id, a.category));
          e["queue"] = q;
          e["snapshots"] = sn;
          e["groups"] = gr;
          e["out"] = out;
          e["pe_read_q"] = v.pe_read_q;
          e["de_read_q"] = v.de_read_q;
          e["path"] = v.path;
          inv.append(e);
        }
        d["invocations"] = inv;
        py::list reqs;
        for (const auto& r : rep.requests)
          reqs.append(py::make_tuple(r.id, r.traj, r.round, r.cached, r.append, r.gen, r.pe, r.de, r.path, r.reader,
                                     r.t_arrival, r.t_sched, r.t_admit, r.t_read_done, r.t_landed, r.t_done,
                                     r.t_prefilled, r.forwards));
        d["requests"] = reqs;
        py::list occ;
        for (const auto& x : rep.final_slots)
          occ.append(py::make_tuple(x.pe, x.slot, x.fb, x.ntok, x.hash_first, x.hash_last));
        d["final_slots"] = occ;
        py::list docc;
        for (const auto& x : rep.final_decode_slots)
          docc.append(py::make_tuple(x.pe, x.slot, x.fb, x.ntok, x.hash_first, x.hash_last));
        d["final_decode_slots"] = docc;
        py::list pers;
        for (const auto& x : rep.persisted) pers.append(py::make_tuple(x.req, x.fb, x.layer, x.t0, x.t1, x.hash));
        d["persisted"] = pers;
        d["persist_write_bytes"] = rep.persist_write_bytes;
        py::list dig;
        for (const auto& x : rep.digests) dig.append(py::make_tuple(x.req, x.first, x.last));
        d["digests"] = dig;
        d["forwards"] = rep.forwards;
        d["wall_s"] = rep.wall_s;
        d["reader_bytes"] = rep.reader_bytes;
        d["admission_stalls"] = rep.admission_stalls;
        d["pool_slots"] = rep.pool_slots;
        d["store_fb"] = rep.store_fb;
        d["fb_stride"] = rep.fb_stride;
        d["slo_violated"] = rep.slo_violated;
        d["steady_state"] = rep.steady_state;
        d["completed_requests"] = rep.completed_requests;
        d["total_requests"] = rep.total_requests;
        d["ttft_series"] = rep.ttft_series;
        return d;
      },
      py::arg("cfg"), py::arg("trajectories"), py::arg("policy") = "dual_path",
      py::arg("sched_mode") = "adaptive", py::arg("alpha") = 100000, py::arg("beta") = 500000,
      py::arg("z") = 1.05, py::arg("exec") = dualpath::ExecOptions{}, py::arg("pe_pool_slots") = 0,
      py::arg("decode_s_per_token") = 0.0, py::arg("gpu") = true, py::arg("link_Bps") = 50e9,
      py::arg("devices") = std::vector<int>{}, py::arg("timeout_s") = 600.0,
      py::arg("arrival_times") = std::vector<double>{}, py::arg("slo_ttft") = 0.0,
      py::arg("steady_window") = 0.0, py::arg("steady_lookback") = 180.0, py::arg("steady_threshold") = 0.05,
      py::arg("de_pool_slots") = 0);

  m.def(
      "run_step_all",
      [](std::vector<dualpath::EngineRuntime*> engines) {
        py::gil_scoped_release nogil;
        return dualpath::run_step_all(engines);
      },
      py::arg("engines"));

  m.attr("ABI_VERSION") = dp_abi_version();
}
