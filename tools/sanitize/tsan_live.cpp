// ThreadSanitizer driver for the live-mode runtime's host threads (scheduler
// loop, per-reader worker and completion threads, per-PE prefill threads,
// the shared dp_nic) on the
// timed backend: no CUDA work, so every reported race is in this repo's
// host code.  Built and run by tools/sanitize/tsan_live.sh.
#include <cstdio>

#include "dualpath/live.hpp"
#include "pdsim/workload.hpp"

int main() {
  pdsim::ClusterConfig cfg;
  cfg.prefill_nodes = 2;
  cfg.decode_nodes = 2;
  cfg.engines_per_node = 1;
  cfg.n_layer = 4;
  cfg.kv_bytes_per_token_per_layer = 576;
  cfg.block_size_tokens = 64;
  cfg.hbm_capacity_tokens = 60000;
  pdsim::SyntheticSpec spec;
  spec.count = 16;
  spec.max_len = 16000;
  spec.mean_turns = 5;
  spec.sigma_turns = 0;
  spec.seed = 11;
  const auto trajs = pdsim::synthesize(spec);
  std::size_t total = 0;
  for (const auto& t : trajs) total += t.rounds.size();
  for (int mode = 0; mode < 6; ++mode) {
    dualpath::LiveOptions o;
    o.gpu = false;
    o.link_Bps = 8e9;
    o.exec.storage_cap_Bps = 1e9;
    o.decode_s_per_token = 2e-6;
    o.sim.sched.alpha = 20000;
    o.sim.sched.beta = 60000;
    if (mode == 1) o.sim.sched_mode = pdsim::desim::SchedMode::RoundRobin;
    if (mode == 2) o.pe_pool_slots = 260;  // tight: admission stalls
    if (mode >= 3) {  // the prefill stand-in: per-PE compute threads, release after the last forward
      o.exec.prefill = true;
      o.exec.compute_quota = 2e-4;
      o.exec.prefill_cost.coeff_bilinear = 576 / 2e12;
      o.exec.prefill_cost.constant = 2e-6;
      o.exec.handoff = mode >= 4;  // + the PD handoff: decode-pool slots, release after K3
      o.exec.persist = mode == 5;  // + persistence: per-DE persist threads, slots freed when persisted
    }
    const auto rep = dualpath::run_live(cfg, trajs, o);
    std::printf("mode %d: %zu requests (%zu expected), %zu invocations, %lld stalls, %.3f s\n", mode,
                rep.requests.size(), total, rep.invocations.size(),
                static_cast<long long>(rep.admission_stalls), rep.wall_s);
    if (rep.requests.size() != total) return 1;
  }
  return 0;
}
