// dualpath/engine.hpp — the GPU executor of the DualPath KV loading path.
//
// The reference's seam is start_flow(req, Stage, bytes) -> complete_stage(req,
// Stage) (/root/reference/proj/src/desim.cpp:468-499, :696-776): a simulated
// fluid flow per byte-moving Stage.  Here the planner (pdsim::desim, plan
// mode) fixes every scheduler decision bit-identically to the reference, and
// this executor turns the decisions into real transfers on B200s:
//
//   StorageRead  (desim.cpp:603-606) -> per-engine storage-NIC gate (token
//                                       bucket at storage_cap_Bps, FIFO), the
//                                       Full Blocks already in pinned host DRAM
//   LoopbackH2D  (desim.cpp:614-616) -> K1 dp_h2d_layer_gather on the PE
//   DeToPe       (desim.cpp:617-619) -> K2 dp_h2d_push_p2p_layer on the DE,
//                                       NVLink stores into the PE pool
//   layer gate   (desim.cpp:623-628) -> per-(ticket, layer) landed counters
//
// One EngineRuntime per GPU (engine e = one process per GPU under torchrun,
// or one thread per GPU in a single process).  Every runtime builds the same
// ExecPlan from the same plan, so block tables and slot ids agree without
// any host exchange; the only exchange is the PE pools' IPC handles.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "dualpath/kv_abi.h"
#include "dualpath/storage.hpp"
#include "pdsim/desim.hpp"
#include "pdsim/scheduler.hpp"
#include "pdsim/types.hpp"

namespace dualpath {

struct ExecOptions {
  double storage_cap_Bps = 0;          // per-engine storage NIC; 0 = uncapped (PCIe binds)
  // host staging bound of a reading engine (the plan's pe_buffer_bytes /
  // de_buffer_bytes): true = enforce it (BufferGate) on the load paths
  bool buffer_bound = true;
  std::vector<double> storage_cap_per_engine;  // overrides storage_cap_Bps per engine
  double pace_scale = 0;               // > 0: online replay, a job's storage read starts no
                                       // earlier than its planned t_admit * pace_scale
  std::int64_t store_fb = 0;           // Full Blocks per engine store; 0 = auto
  std::int64_t store_bytes_max = 8LL << 30;
  std::uint64_t seed = 9;              // content seed (oracle/kvref.c)
  std::int32_t pool_slots = 0;         // slots per PE pool; 0 = auto (plan peak)
  std::int64_t pool_bytes_max = 120LL << 30;
  std::int32_t wait_timeout_ms = 30000;
  // PE-path loads (K1): 0 = SM gather kernel, 1 = copy engine (no SMs: the
  // isolation mode while the PE computes), 2 = both at once, jobs split by
  // bytes (the plain load path; measured slower than 0, profiles/r01_SUMMARY.md)
  // 3 = staged: the copy engine moves whole Full-Block runs into an HBM ring at
  // the link's full rate, a small scatter kernel (stage_ctas CTAs) lands them
  // in the pool's layer planes (dp_h2d_layer_staged)
  std::int32_t k1_mode = 0;
  // PE pool layout: DP_POOL_LAYER_MAJOR (0, per-layer planes) or
  // DP_POOL_BLOCK_MAJOR (1, whole Full Blocks per slot: with k1_mode /
  // k2_mode 1 the copy engines land each run of Full Blocks in one copy, no
  // ring and no SM work); block-major takes the load and prefill paths only
  std::int32_t pool_layout = 0;
  // copy-engine modes (k1_mode / k2_mode 1): release a job's counters once
  // after its last layer (true) or after every layer (false; idles the copy
  // engine once per layer)
  bool copy_release_per_job = true;
  // DE-path loads (K2): 0 = SM gather pushing over NVLink, 1 = the DE's copy
  // engine writing into the PE pool (no SMs on the DE: its decode is untouched)
  // 2 = staged: the DE's copy engine into its HBM ring, then the scatter kernel
  // pushes over NVLink into the PE pool (dp_h2d_push_staged)
  std::int32_t k2_mode = 0;
  std::int64_t stage_ring_bytes = 1LL << 30;  // staged modes: HBM ring per engine
  std::int32_t stage_ctas = 32;               // staged K1: scatter CTAs (HBM -> HBM)
  std::int32_t stage_push_ctas = 148;         // staged K2: scatter CTAs pushing over NVLink
                                              // (peer stores need more in flight)
  std::int32_t stage_scatter = 0;             // staged modes: 0 = scatter kernel, 1 = copy engine
                                              // (DP_SCATTER_CE: no SM work at all)
  // PD handoff: every request's prompt KV also ends in its
  // DE's decode pool — prefill stand-in + PeToDe / MissMerge per layer (K3)
  // and the DE read path fused with DecodeH2D (dual store)
  bool handoff = false;
  std::int32_t de_pool_slots = 0;      // per DE decode pool; 0 = auto (4x plan peak)
  // CTA cap of the SM gathers (dp_set_gather_ctas) on this run's devices;
  // 0 = default (4 per SM), -1 = auto: 64 on a PE when the handoff shares it
  std::int32_t gather_ctas = -1;
  // DE-path gate of K3: 0 = the handoff stream waits (a one-thread spin kernel
  // with the watchdog) for the whole request's hit KV; 1 = K3 gates layer by
  // layer in-kernel
  std::int32_t k3_layer_gate = 0;
  std::int32_t handoff_ctas = 0;       // K3 CTA cap on PEs (0 = default)
  bool handoff_tma = false;            // K3's hit push through the TMA (dp_set_handoff_tma)
  // K3: 0 = the SM kernel (dp_prefill_handoff), 1 = the copy engines push the
  // hit runs over NVLink and a small side kernel per layer does the gates,
  // the miss KV and the releases (dp_prefill_handoff_copy; the default: 749 vs
  // 702 GB/s alone, and no SM pushes beside the prefill)
  std::int32_t k3_mode = 1;
  // handoff + prefill: K3 pushes layer l of a request as soon as the forward
  // that finishes it has computed layer l (the reference starts PeToDe /
  // MissMerge of layer l at LayerCompute l's completion, desim.cpp:630-640,
  // :721-738), gated in-kernel on per-(forward, layer) done counters the
  // compute stream writes; false: K3 waits for the forward's last layer
  // (default false: measured slower with the CUDA-core prefill stand-in, whose
  // forwards lose SM residency to the spinning K3 CTAs -- profiles/r02_SUMMARY.md)
  bool handoff_layerwise = false;
  // Decode-side persistence (needs `handoff`): each DE runs
  // the decode stand-in for the generated tokens and persists them (K4) every
  // 64 generated tokens plus the final partial, into its persist store
  bool persist = false;
  // K4: 0 = the SM kernel's zero-copy stores over PCIe (dp_persist_d2h),
  // 1 = staged: a gather kernel into an HBM ring of its own, then the copy
  // engine to the host (dp_persist_staged; the default: 57.2 GB/s = 0.999 of
  // the copy-engine D2H peak against 51.8 for the SM path)
  std::int32_t persist_mode = 1;
  // PersistWrite (desim.cpp:764-771): a FullBlockFile (record r = storage Full
  // Block r) each DE writes the Full Blocks its K4 persisted into at the end of
  // its step, so a later turn's StorageRead from the tier reads them back;
  // empty: the persisted blocks stay in the pinned persist store
  std::string persist_path;
  // Prefill stand-in (with or without `handoff`): every PE packs
  // its requests, in the order their KV lands, into forward batches with
  // pdsim::build_forward_batch under `compute_quota` (seconds per layer of
  // `prefill_cost`) and runs each batch layer by layer as K5
  // (dp_prefill_attend), layer l gated on the batch's landed counters.
  bool prefill = false;
  double compute_quota = 2e-3;
  pdsim::AttentionCostModel prefill_cost{};
  std::int32_t attend_ctas = 0;        // K5 CTA cap (0 = default)
  // Storage tier (the load and prefill paths): StorageRead
  // becomes real file reads — every Full Block a job needs is looked up in
  // the Full Block trie and read from `tier_path` (a FullBlockFile whose
  // record r is page r) by `io_threads` host threads into a pinned staging
  // ring, from which K1/K2 move its Layer Blocks.  Empty: procedural store.
  std::string tier_path;
  std::int32_t tier_ring_fb = 0;       // staging ring per reader, Full Blocks (0 = auto)
  std::int32_t io_threads = 8;
  bool tier_direct = true;             // O_DIRECT reads when the file system allows
};

// One request's hit-KV transfer (all layers), in global execution order.
struct LoadJob {
  int req = 0;              // plan request id
  int traj = 0;
  int round = 0;
  int reader = 0;           // engine reading storage: pe (PE path) or de (DE path)
  int pe = 0;               // destination engine (owner of the pool)
  bool de_path = false;
  std::int64_t cached = 0;  // C
  std::int32_t n_blk = 0;
  std::int64_t blk_off = 0; // offset of this job's blocks in the reader's tables
  std::int32_t ticket = 0;  // counter row in the PE pool
  double t_admit = 0;       // plan: StorageRead starts (virtual s)
  double t_read_done = 0;   // plan: hit transfer starts
  std::vector<std::int32_t> preds;         // tickets in the same PE pool whose slots this
  std::vector<std::uint32_t> pred_targets; // reuses (written by another engine), and their
                                           // all-layer landed-item targets
  bool fence = false;  // reuses a slot this reader wrote earlier: must not share a launch
  std::vector<int> fence_jobs;  // ... with these jobs (global order)
  // ---- PD handoff (ExecOptions::handoff) ----
  int de = -1;                   // the request's decode engine
  std::int64_t prompt = 0;       // C + A
  std::int32_t n_pblk = 0;       // prompt blocks (PE slots cover these in handoff mode)
  std::int64_t ho_off = 0;       // offset of the prompt tables in the PE's handoff tables
  std::int32_t de_ticket = -1;   // decode-pool row
  std::vector<std::int32_t> k3_waits;      // jobs (same PE) whose K3 must finish before this
                                           // job's K1 reuses their PE slots (event waits)
  std::vector<std::int32_t> pe_done_preds; // PE done-rows (ticket + n_tickets) a DE-path
  std::vector<std::uint32_t> pe_done_targets;  // job's dual gather waits for (PE slot reuse)
  std::vector<std::int32_t> de_preds;      // decode-pool rows of the previous occupants of
  std::vector<std::uint32_t> de_pred_targets;  // this job's DE slots
  // ---- persistence ----
  std::int64_t gen = 0;          // generated tokens of the turn
  std::int32_t n_tblk = 0;       // decode-pool blocks: ceil((C + A + gen) / T)
  std::int64_t dec_off = 0;      // offset of its blocks in the DE's decode tables
  // ---- prefill ----
  std::vector<int> consumer_waits;  // jobs whose slots this one reuses: their last forward
                                    // must be done before this job's load writes
  std::int64_t fwd_off = 0;         // offset of its slots in the PE's forward slot table
  std::vector<int> de_pred_jobs;    // jobs whose decode slots this one reuses (global order)
  // ---- storage tier ----
  std::vector<int> ring_waits;      // jobs (same reader) whose staging positions this
                                    // job's reads overwrite: their transfer must be done
};

// One request chunk of a forward batch (ExecOptions::prefill).
struct FwdItem {
  int req = 0;               // plan request id
  int job = -1;              // its load job (-1: no cached KV)
  std::int64_t cached = 0;   // C
  std::int64_t q_begin = 0;  // first query token of the chunk (offset into the append)
  std::int64_t bsz = 0;      // query tokens of the chunk
  std::int32_t row = 0;      // digest row of the request on its PE
  bool first = false;        // the request's first forward (gates on its KV)
};

struct Forward {
  std::int32_t begin = 0, end = 0;  // items [begin, end) of the PE's fwd_items
  double estimated_time = 0;        // per layer, the cost model's (pdsim::ForwardBatch)
  std::int32_t last_row = 0;        // FIFO row of its last item
};

struct ExecPlan {
  pdsim::ClusterConfig cfg;
  ExecOptions opt;
  int n_engines = 0;
  int n_pe = 0;
  dp_kv_geom geom{};
  std::int64_t store_fb = 0;
  std::int32_t pool_slots = 0;
  std::int32_t items_per_block = 1;        // landed-counter items per Layer Block
  std::vector<LoadJob> jobs;               // global execution (slot allocation) order
  std::vector<std::vector<int>> by_reader; // job indices per reading engine
  std::vector<std::vector<int>> by_pe;     // job indices per destination PE
  std::vector<std::vector<std::int64_t>> src_fb;  // per reader: flat Full Block ids
  std::vector<std::vector<std::int32_t>> slots;   // per reader: flat destination slots
  std::vector<std::int32_t> n_tickets;            // per PE
  std::vector<std::int64_t> reader_bytes;         // hit bytes read per engine
  std::int64_t hit_bytes = 0;                     // sum C * L * b
  std::int64_t prompt_tokens = 0;                 // sum (C + A) over all requests
  std::int64_t requests = 0;
  std::int32_t peak_slots = 0;                    // max live slots on any PE

  std::int64_t fb_of(int traj, std::int64_t block) const;  // storage mapping
  std::int64_t fb_stride = 1;                               // blocks per session

  // ---- PD handoff ----
  bool handoff = false;
  std::int32_t de_pool_slots = 0;
  std::int32_t de_peak_slots = 0;
  std::vector<std::int32_t> n_de_tickets;                  // per engine (0 for PEs)
  std::vector<std::vector<int>> by_de;                     // job indices per decode engine
  std::vector<std::vector<std::int64_t>> ho_src_fb;        // per PE: prompt blocks' Full Blocks
  std::vector<std::vector<std::int32_t>> ho_pe_slot;       // per PE: prompt blocks' PE slots
  std::vector<std::vector<std::int32_t>> ho_de_slot;       // per PE: prompt blocks' DE slots
  std::vector<std::vector<std::int32_t>> dual_de_slot;     // per reader: hit blocks' DE slots
  std::int64_t handoff_bytes = 0;  // pushed by K3: (C+A)*L*b PE path, A*L*b DE path
  bool persist = false;
  // PersistWrite (desim.cpp:764-771): a FullBlockFile (record r = storage Full
  // Block r) each DE writes the Full Blocks its K4 persisted into at the end of
  // its step, so a later turn's StorageRead from the tier reads them back;
  // empty: the persisted blocks stay in the pinned persist store
  std::string persist_path;
  std::vector<std::vector<std::int32_t>> dec_slot;         // per DE: all blocks' decode slots
  std::vector<std::vector<std::int64_t>> dec_fb;           // per DE: their storage Full Blocks
  std::int64_t persist_bytes = 0;                          // sum gen * L * b
  // persist chunks of a job, [token begin, end): the reference's
  // persist_tokens at every block_size generated tokens + the final partial
  std::vector<std::pair<std::int64_t, std::int64_t>> persist_chunks(const LoadJob& j) const;
  std::uint32_t de_total_items(const LoadJob& j) const;    // decode-pool row target (all layers)

  // ---- prefill ----
  bool prefill = false;
  std::vector<std::vector<FwdItem>> fwd_items;   // per PE: the items of its forwards, in order
  std::vector<std::vector<Forward>> forwards;    // per PE
  std::vector<std::vector<int>> fwd_rows;        // per PE: request id of each digest row (FIFO)
  std::vector<std::vector<std::int32_t>> fwd_slot;  // per PE: slots of the jobs landing there
  std::vector<int> last_fwd;                     // per job: the forward (on its PE) that reads it last
  // handoff + prefill: each DE's enqueue order; job j = a read, -1 - j = a decode
  std::vector<std::vector<int>> de_order;

  // ---- storage tier ----
  bool tier = false;
  std::int32_t ring_fb = 0;                       // staging ring per reader (Full Blocks)
  std::vector<std::vector<std::int64_t>> tier_rec;  // per reader: file record of each block
  std::int64_t trie_nodes = 0;                    // Full Block trie size
};

// Builds the executor plan from planner output.  Requests with C = 0 move no
// hit KV and get no job.  Slots are allocated per PE at t_read_done and freed
// at t_pe_release (virtual time, frees first at equal time), FIFO reuse.
ExecPlan build_exec_plan(const pdsim::ClusterConfig& cfg,
                         std::span<const pdsim::Trajectory> trajectories,
                         const pdsim::desim::SimReport& plan, const ExecOptions& opt);

struct StorageSpan {
  double t_begin = 0;  // s since the step started
  double t_end = 0;
  std::int64_t bytes = 0;
};

struct StepResult {
  std::vector<StorageSpan> spans;  // per job: its emulated storage read (gated runs)
  double device_ms = 0;         // CUDA-event time of this engine's step
  double host_ms = 0;           // wall time of run_step()
  std::int64_t bytes_read = 0;  // hit bytes this engine read from storage
  std::int64_t launches = 0;    // kernels launched by this engine
  std::int64_t jobs = 0;
  std::int64_t forwards = 0;    // prefill forwards run (PE, ExecOptions::prefill)
  double io_wait_ms = 0;        // storage tier: host time the launches waited for reads
  double persist_write_ms = 0;  // DE: PersistWrite of the step's persisted Full Blocks to the tier
  std::int64_t persist_write_bytes = 0;
  // handoff (PE): per request, ms from the step start until its whole prompt
  // KV is in its DE's decode pool (the offline TTFT of the prefill path), and
  // the handoff lag: that time minus the end of the forward finishing it
  std::int64_t buffer_stalls = 0;   // waits for the reader's host staging bound
  double buffer_wait_ms = 0;
  std::vector<float> ttft_ms;
  std::vector<float> handoff_lag_ms;
  std::int64_t d2h_bytes = 0;   // result read back (PE: landed-counter column)
};

class TierReader;

class EngineRuntime {
 public:
  EngineRuntime(std::shared_ptr<const ExecPlan> plan, int engine, int device);
  ~EngineRuntime();
  EngineRuntime(const EngineRuntime&) = delete;
  EngineRuntime& operator=(const EngineRuntime&) = delete;

  int engine() const { return engine_; }
  int device() const { return device_; }
  bool is_pe() const { return engine_ < plan_->n_pe; }

  // Pool export / import (cross-process) or same-process peer attach.  Every
  // PE exports its prefill pool; with PD handoff every DE exports its decode
  // pool too, and attach_* of a DE engine id gives a PE its view of it.
  dp_pool_handle export_pool() const;
  void attach_peer(int engine, const dp_pool_handle& handle);
  void attach_peer_local(int engine, const EngineRuntime& other);
  bool has_pool() const { return pool_ != nullptr; }

  // Zero this PE's landed counters (call on every PE, then barrier, before a step).
  void reset_counters();
  // Issue this engine's transfers for one pass over the plan and wait for
  // them (and, on a PE, for every push landing in its pool).
  StepResult run_step();
  // Prefill mode, PE only: run this PE's forwards again over the KV already
  // in the pool (after a run_step, counters not reset): the compute alone.
  StepResult run_forwards();
  // Prefill mode, PE only: the K5 digests [row][layer] of the last step.
  std::vector<std::uint64_t> prefill_digests() const;

  // Parity helpers: content hash of a pool Layer Block (PE only), and the
  // raw pool / counters for tests.
  std::vector<std::uint64_t> checksum(int layer, std::span<const std::int32_t> slots,
                                      std::span<const std::int32_t> ntok);
  std::vector<std::uint32_t> counters() const;
  const dp_pool* pool() const { return pool_; }
  const dp_store* store() const { return store_; }

 private:
  void upload_tables();
  bool layerwise_handoff() const {
    return plan_->handoff && plan_->prefill && plan_->opt.handoff_layerwise && is_pe();
  }
  std::int32_t fwd_row0_ = 0;               // PE: first per-forward layer-done row
  void storage_read(const LoadJob& j, std::int64_t bytes, StepResult& res);

  std::shared_ptr<const ExecPlan> plan_;
  int engine_;
  int device_;
  void* stream_ = nullptr;
  void* ev_start_ = nullptr;
  void* ev_end_ = nullptr;
  dp_store* store_ = nullptr;
  dp_nic* nic_ = nullptr;                   // emulated storage NIC (rate cap)
  dp_stager* persist_stager_ = nullptr;      // staged K4 (persist_mode 1): its own ring
  dp_stager* stager_ = nullptr;             // staged K1 / K2: HBM ring (k1_mode 3 / k2_mode 2)
  std::int64_t persist_launches() const;
  std::int64_t stager_launches() const;
  const std::int32_t* stage_slots() const;
  std::int64_t buffer_budget() const;
  dp_pool* pool_ = nullptr;                 // owned (PE only)
  std::vector<dp_pool*> peers_;             // per engine id: view of that PE's pool
  std::int64_t* d_src_ = nullptr;           // device block tables of this reader
  std::int32_t* d_slots_ = nullptr;
  std::int32_t* d_wait_tickets_ = nullptr;  // PE: DE-path tickets landing here
  std::uint32_t* d_wait_targets_ = nullptr;
  std::int32_t n_wait_ = 0;
  std::int32_t* d_pred_tickets_ = nullptr;  // hazard waits, flattened per job
  std::uint32_t* d_pred_targets_ = nullptr;
  std::vector<std::int64_t> pred_off_;      // per job index in by_reader: offset into preds

  // ---- PD handoff ----
  StepResult run_step_handoff();
  void upload_handoff_tables();
  void* stream_h_ = nullptr;                // PE: K3 (prefill stand-in + handoff) stream
  std::vector<void*> ev_load_, ev_k3_;      // PE: per job in by_pe order
  std::vector<int> pe_local_;               // job index -> position in by_pe (or -1)
  std::vector<dp_pool*> de_views_;          // PE: per engine id: view of that DE's pool
  std::int64_t* d_ho_src_ = nullptr;
  std::int32_t* d_ho_pe_ = nullptr;
  std::int32_t* d_ho_de_ = nullptr;
  std::int32_t* d_dual_de_ = nullptr;
  std::int32_t* d_wt_ = nullptr;            // flattened wait lists (tickets / targets)
  std::uint32_t* d_wg_ = nullptr;
  std::vector<std::int64_t> de_wait_off_;   // per job: offset of its de_preds in d_wt_
  std::vector<std::int64_t> pe_done_off_;   // per job: offset of its pe_done_preds
  std::int64_t final_wait_off_ = 0;         // DE: all own tickets (decode-ready gate)
  std::int32_t final_wait_n_ = 0;
  void read_back_landed(StepResult& res);
  std::vector<std::uint32_t> landed_host_;
  // ---- prefill ----
  StepResult run_step_prefill(bool loads);
  void enqueue_forward(int f, StepResult& res);
  void upload_prefill_tables();
  void* stream_c_ = nullptr;                // PE: the compute stream (forwards)
  void* stream_ce_ = nullptr;               // PE, k1_mode 2: the copy-engine share of K1
  std::vector<void*> ev_ce_;
  std::vector<void*> ev_fwd_;               // PE: per forward, recorded after its last layer
  std::vector<std::vector<dp_attend_item>> fwd_att_;  // PE: per forward, K5 items
  std::vector<std::int64_t> fwd_wait_off_;  // PE: per forward, offset of its KV waits in d_wt_
  std::vector<std::int32_t> fwd_wait_n_;
  std::vector<std::vector<std::int32_t>> fwd_done_;   // PE: per forward, tickets read last there
  std::uint64_t* d_digest_ = nullptr;
  std::int32_t* d_fwt_ = nullptr;           // PE: forward gate tickets / targets
  std::uint32_t* d_fwg_ = nullptr;
  std::int32_t* d_fwd_slot_ = nullptr;
  // ---- storage tier ----
  friend class TierReader;
  std::unique_ptr<FullBlockFile> tier_file_;
  std::vector<void*> ev_job_;               // per job in by_reader order: after its launch
  std::vector<std::vector<int>> ring_wait_local_;  // ring_waits as by_reader positions
  // ---- persistence (DE) ----
  dp_store* persist_store_ = nullptr;
  std::unique_ptr<FullBlockFile> persist_file_;   // PersistWrite target (ExecOptions::persist_path)
  void persist_write(StepResult& res);
  std::int32_t* d_dec_slot_ = nullptr;
  std::int64_t* d_dec_fb_ = nullptr;

 public:
  // Bytes of Layer Block `layer` of Full Block `fb` in this DE's persist store.
  std::vector<std::uint8_t> read_persisted(std::int64_t fb, int layer) const;
};

// Runs run_step() of several same-process engines concurrently (one host
// thread each) and returns their results in order.
std::vector<StepResult> run_step_all(std::span<EngineRuntime* const> engines);

}  // namespace dualpath
