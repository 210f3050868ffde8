// dualpath/live.hpp — live-mode scheduling: the reference's
// global scheduler run on MEASURED engine state while the bytes move.
//
// Plan mode (pdsim::desim) fixes every decision in virtual time, bit-exact
// with the reference for a trace and config, and the executor replays them.
// Live mode instead runs the reference's scheduler glue
// (/root/reference/proj/src/desim.cpp:851-906: DE phase 1 -> phase 2 per DE
// node -> PE fetch over the DE-assigned FIFO, then a FIFO admission pass) on
// counters that real completions update, as the reference's do:
//
//   read_q[node] += C at the decision (desim.cpp:833-835),
//                -= C when the request's StorageRead completes (:702-704),
//   tok_e / seq_e of the PE fall at its release (:646-647), of the DE at
//   the request's completion (:781-783, with hbm_free),
//   a session's next turn arrives when its previous turn completes.
//
// StorageRead is the engine's emulated storage NIC (dp_nic, the rate cap);
// the hit transfer is K1 / K2 (or their staged variants) on the GPUs.  Load
// path only (exec.prefill false): the PE is released when the request's KV
// has landed in its pool.  With exec.prefill, each PE runs the prefill
// stand-in as the plan-mode executor does -- forwards packed by
// build_forward_batch under exec.compute_quota (scheduler.cpp:174-219) from
// its FIFO of requests whose loads are launched, K5 per layer gated on the
// request's landed counters (maybe_start_compute, desim.cpp:623-628) -- and
// the PE is released when the request's last forward has computed its last
// layer (on_prefill_side_done, desim.cpp:642-652); a turn's TTFT is then
// arrival -> that point.  The DE holds the request for gen x
// decode_s_per_token.  With exec.handoff too, the PE pool holds each
// request's whole prompt, the DE read path is the dual gather (PE pool +
// the DE's decode pool), and after the forward that finishes a request K3
// (PeToDe / MissMerge, exec.k3_mode) moves its prompt into the DE's decode
// pool; the PE releases it when K3 is done (every layer computed and
// shipped) and its first token follows one decode step: TTFT as the
// reference's (desim.cpp:679-685).  Admission also reserves the prompt's
// decode-pool slots (bounded: de_pool_slots).  With exec.persist too, at a
// request's completion its DE writes the generated tokens into the decode
// pool (the decode stand-in) and persists them with staged K4 in the
// reference's chunks (PersistD2H, desim.cpp:658-661, :690-693, :760) into
// its persist store; the decode slots (prompt + generated blocks) are freed
// once that is done; with exec.persist_path each persisted range is also
// written into that block's record of the storage-tier file (PersistWrite).
// Admission reserves the request's blocks in the PE's paged pool (bounded:
// pe_pool_slots) and stalls, FIFO, while the pool is full -- the staging
// bound of try_admit (desim.cpp:587-599).
//
// Every scheduler invocation's inputs and outputs are logged, so each one can
// be replayed through the reference's own functions (oracle/_ref) for
// per-invocation parity (tests/test_live.py).  Decisions themselves depend
// on real timing; whole-run parity is plan mode's job.
#pragma once

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "dualpath/engine.hpp"
#include "pdsim/desim.hpp"
#include "pdsim/scheduler.hpp"
#include "pdsim/types.hpp"

namespace dualpath {

struct LiveOptions {
  pdsim::desim::SimOptions sim;      // policy, sched_mode, scheduler parameters
  ExecOptions exec;                  // storage cap, content seed, k1 / k2 modes, store size
  std::int32_t pe_pool_slots = 0;    // paged pool per PE; 0 = 4x the largest request's blocks
  std::int32_t de_pool_slots = 0;    // exec.handoff: decode pool per DE; 0 = 4x the largest prompt's blocks
  double decode_s_per_token = 0;     // emulated decode on the DE after the KV has landed
  bool gpu = true;                   // false: timed backend (transfers sleep bytes / link_Bps)
  double link_Bps = 50e9;            // timed backend: per-reader transfer rate
  std::vector<int> devices;          // engine -> CUDA device (gpu backend; default engine % count)
  double timeout_s = 600;            // whole-run watchdog
  // online (run_online, desim.cpp:1036-1051): session i's first turn arrives
  // at arrival_times[i] seconds (empty: all at 0, offline)
  std::vector<double> arrival_times;
  // the reference's online stops, on MEASURED latencies: a turn's TTFT here is
  // the load path's (arrival -> its hit KV landed in the PE pool), or with
  // exec.prefill arrival -> its prefill done (the PE release); the run
  // stops when one exceeds slo_ttft_s (> 0; desim.cpp:679-685) or when the
  // TTFT series is steady (steady_window > 0: detect_steady_state every
  // window / 2, desim.cpp:942-953)
  double slo_ttft_s = 0;
  double steady_window = 0, steady_lookback = 180, steady_threshold = 0.05;
};

// One scheduler function call, its inputs and result.
struct LiveInvocation {
  std::string fn;  // schedule_de_groups | schedule_de_within_group | schedule_pe_fetch | select_read_path
  double t = 0;
  std::vector<pdsim::PendingRequest> queue;
  std::vector<pdsim::EngineSnapshot> snapshots;
  std::vector<pdsim::GroupLoad> groups;
  std::vector<pdsim::Assignment> out;  // de_groups: {request, group, 0}
  std::int64_t pe_read_q = 0, de_read_q = 0;
  int path = 0;                        // select_read_path: 0 PE, 1 DE
};

struct LiveRequest {
  int id = 0, traj = 0, round = 0;
  std::int64_t cached = 0, append = 0, gen = 0;
  int pe = -1, de = -1, path = 0, reader = -1;
  double t_arrival = -1, t_sched = -1, t_admit = -1, t_read_done = -1, t_landed = -1, t_done = -1;
  double t_prefilled = -1;  // exec.prefill: its last forward done (the PE release)
  int forwards = 0;         // exec.prefill: forwards it took part in
};

struct LiveReport {
  std::vector<pdsim::desim::SchedDecision> decisions;
  std::vector<LiveInvocation> invocations;
  std::vector<LiveRequest> requests;
  double wall_s = 0;
  std::int64_t hit_bytes = 0;
  std::vector<std::int64_t> reader_bytes;  // per engine
  std::int64_t admission_stalls = 0;       // admission passes that left a request waiting for pool slots
  std::int32_t pool_slots = 0;
  // gpu backend, per PE: the final occupant of every slot (slot, Full Block,
  // valid tokens) and its content hash for layers 0 and L-1 (parity vs kvref)
  struct Occupant {
    int pe = 0;
    std::int32_t slot = 0;
    std::int64_t fb = 0;
    std::int32_t ntok = 0;
    std::uint64_t hash_first = 0, hash_last = 0;
  };
  std::vector<Occupant> final_slots;
  // exec.handoff: the same for every DE's decode pool (pe = the DE's engine id):
  // the whole prompt of its final occupant
  std::vector<Occupant> final_decode_slots;
  // exec.persist: per persisted request, block and layer (0 and L-1): the
  // generated tokens' range [t0, t1) of the block in its storage Full Block
  // and the hash of those bytes in the DE's persist store (dp_pool_checksum's
  // hash over the range)
  struct Persisted {
    int req = 0;
    std::int64_t fb = 0;
    std::int32_t layer = 0, t0 = 0, t1 = 0;
    std::uint64_t hash = 0;
  };
  std::vector<Persisted> persisted;
  std::int64_t persist_write_bytes = 0;  // exec.persist_path: bytes written into the storage-tier file
  // gpu backend with exec.prefill: the K5 digest of every prefilled request at
  // layers 0 and L-1 (parity vs the oracle: independent of the batching)
  struct Digest {
    int req = 0;
    std::uint64_t first = 0, last = 0;
  };
  std::vector<Digest> digests;
  std::int64_t forwards = 0;  // exec.prefill: forwards run over all PEs
  std::int64_t store_fb = 0, fb_stride = 0;  // content mapping fb = (traj * stride + k) % store_fb
  bool slo_violated = false, steady_state = false;
  std::size_t completed_requests = 0, total_requests = 0;
  std::vector<std::pair<double, double>> ttft_series;  // (t, ttft) per landed turn
};

LiveReport run_live(const pdsim::ClusterConfig& cfg, std::span<const pdsim::Trajectory> trajectories,
                    const LiveOptions& options);

}  // namespace dualpath
