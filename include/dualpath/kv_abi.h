/*
 * dualpath/kv_abi.h — C ABI of the B200 DualPath KV-Cache loading path.
 *
 * The reference (pdsim, /root/reference/proj) has no FFI for this path: KV
 * loading is a byte count inside a simulated flow.  The drop-in seam is the
 * Stage pair start_flow(req, Stage, bytes, path) ... complete_stage(req, Stage)
 * (proj/src/desim.cpp:468-499, :696-776).  Every entry point below replaces one
 * byte-moving Stage or one of the KV interfaces the reference defines:
 *
 *   dp_kv_geom            <- ClusterConfig KV fields (proj/include/pdsim/types.hpp:18-20,30-39)
 *   dp_store_*            <- StorageRead source: Full Blocks [L][T][b] in host DRAM
 *                            (desim.cpp:603-606)
 *   dp_h2d_layer_gather   <- Stage::LoopbackH2D, PE read path (desim.cpp:612-616)
 *   dp_h2d_push_p2p_layer <- Stage::DeToPe, DE read path (desim.cpp:617-619)
 *   dp_wait_layer         <- maybe_start_compute gate layer_h2d_done > layer_compute_done
 *                            (desim.cpp:623-628)
 *   dp_pool_*             <- the PE HBM KV pool (paged; not modelled by the reference,
 *                            SPEC.md:106) and BlockRef layer_block (types.cpp:62-71)
 *   dp_h2d_layer_copy     <- LoopbackH2D on the copy engine; dp_h2d_push_copy <- DeToPe
 *                            on the DE's copy engine (same Stages, no SMs)
 *   dp_h2d_push_p2p_dual  <- DeToPe fused with the hit half of DecodeH2D
 *                            (desim.cpp:617-619, :650-651)
 *   dp_prefill_handoff    <- Stage::PeToDe / Stage::MissMerge per layer (desim.cpp:630-640)
 *   dp_decode_fill,       <- Decode (stand-in) and Stage::PersistD2H, every 64 generated
 *   dp_persist_d2h           tokens + the final partial (desim.cpp:666-672, :690-693)
 *   dp_prefill_attend     <- Stage::LayerCompute of a forward batch
 *                            (layer_time desim.cpp:576-579; build_forward_batch
 *                            scheduler.cpp:174-219)
 *
 * Conventions (no exceptions cross this ABI):
 *   - every call returns int: 0 = ok, < 0 = dp_status error code;
 *   - dp_last_error() returns a thread-local message for the last failing call;
 *   - a dp_stream argument is a cudaStream_t (NULL = legacy default stream);
 *     calls taking one are asynchronous on that stream;
 *   - pointer fields inside dp_job must be device-accessible (device memory or
 *     mapped pinned host memory) on the device that runs the kernel.
 */
#ifndef DUALPATH_KV_ABI_H
#define DUALPATH_KV_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DP_ABI_VERSION 1
#define DP_MAX_JOBS_PER_LAUNCH 64

typedef void* dp_stream; /* cudaStream_t */

typedef enum dp_status {
  DP_OK = 0,
  DP_EINVAL = -1,  /* bad argument (reference: std::invalid_argument) */
  DP_ECUDA = -2,   /* CUDA runtime error */
  DP_ENOMEM = -3,  /* allocation failed */
  DP_ETIMEOUT = -4 /* a dp_wait_layer watchdog fired */
} dp_status;

/* KV geometry.  Layer Block = block_tokens * bytes_per_token_layer bytes;
 * Full Block = n_layer Layer Blocks concatenated (types.hpp:33-39). */
typedef struct dp_kv_geom {
  int32_t n_layer;
  int32_t block_tokens;
  int64_t bytes_per_token_layer; /* must be a multiple of 16 */
} dp_kv_geom;

/* One request's hit-KV transfer for a layer range (one or more Stage flows).
 * Blocks k = 0..n_blk-1 hold tokens [k*T, min((k+1)*T, n_tokens)); only the
 * valid bytes of the last (partial) block are moved, so a layer moves exactly
 * n_tokens * b bytes, the reference ledger kvb_layer (desim.cpp:569-571). */
typedef struct dp_job {
  const int64_t* src_fb;   /* [n_blk] Full Block index in the source store */
  const int32_t* dst_slot; /* [n_blk] slot in the destination pool (block table) */
  int64_t n_tokens;        /* hit tokens C of the request */
  int32_t n_blk;           /* ceil(C / T) (types.cpp:55-60) */
  int32_t layer_begin;     /* first layer to move */
  int32_t layer_end;       /* one past the last layer */
  int32_t ticket;          /* landed-counter row in the destination pool, or -1 */
} dp_job;

typedef struct dp_store dp_store; /* pinned, mapped host DRAM holding Full Blocks */
typedef struct dp_pool dp_pool;   /* paged HBM pool [n_layer][n_slots][T][b] + counters */

/* Cross-process export of a pool (CUDA IPC), 128 bytes. */
typedef struct dp_pool_handle {
  unsigned char ipc[64];
  dp_kv_geom geom;
  int32_t n_slots;
  int32_t n_tickets;
  int32_t device;
  int32_t reserved[9];
} dp_pool_handle;

int dp_abi_version(void);
const char* dp_last_error(void);
int dp_geom_check(const dp_kv_geom* geom);

/* Storage tier emulation.  Creates n_fb Full Blocks of pinned+mapped host
 * memory and fills them on `device` with the deterministic content
 *   word(p, w) = splitmix64((p << 32 | w) ^ (seed * 0xD1B54A32D192ED03))
 * for Full Block p, 8-byte word w (the oracle restates this, oracle/kvref.c). */
int dp_store_create(int device, const dp_kv_geom* geom, int64_t n_fb, uint64_t seed,
                    dp_store** out);
int dp_store_destroy(dp_store* store);
int dp_store_info(const dp_store* store, void** host_ptr, int64_t* bytes, int64_t* n_fb);

/* NUMA-placed staging (SURVEY.md §8(b) dp_staging_create): the PE / DE host
 * buffer (pe_buffer_bytes / de_buffer_bytes, types.hpp:22-23) as pinned,
 * device-mapped pages bound to one NUMA node (mmap + mbind + transparent huge
 * pages + cudaHostRegister).  numa_node >= 0 binds to that node,
 * DP_NUMA_DEVICE to the node of `device`'s PCIe root (sysfs), DP_NUMA_NONE
 * leaves placement to the kernel.  dp_store_create == ..._on_node(DP_NUMA_DEVICE). */
#define DP_NUMA_DEVICE (-1)
#define DP_NUMA_NONE (-2)
int dp_store_create_on_node(int device, const dp_kv_geom* geom, int64_t n_fb, uint64_t seed,
                            int32_t numa_node, dp_store** out);
/* The node the store's pages are bound to (-1: not bound / unknown). */
int dp_store_numa_node(const dp_store* store, int32_t* node);
/* NUMA node of the device's PCIe attachment (-1 when the platform has none). */
int dp_device_numa_node(int device, int32_t* node);

/* Emulated storage NIC (StorageRead over {snic_rd, dram}, desim.cpp:603-606):
 * a FIFO token bucket at rate_Bps (0 = unlimited).  dp_nic_read blocks the
 * calling thread until the NIC has delivered `bytes`: the transfer begins at
 * max(NIC free, not_before_s, now) and lasts bytes / rate; times are seconds
 * since dp_nic_start (optional outputs t_begin / t_end).  Thread-safe: the
 * IO threads of an engine share its NIC. */
typedef struct dp_nic dp_nic;
int dp_nic_create(double rate_Bps, dp_nic** out);
int dp_nic_destroy(dp_nic* nic);
int dp_nic_start(dp_nic* nic);
int dp_nic_read(dp_nic* nic, int64_t bytes, double not_before_s, double* t_begin, double* t_end);
/* StorageRead emulation (SURVEY.md §8(b) dp_storage_read): paced by `nic`
 * (may be NULL), materialise storage Full Blocks src_fb .. src_fb + n_fb - 1
 * (the content formula above, the staging's seed) into staging positions
 * dst_fb ..; synchronous. */
int dp_storage_read(dp_store* staging, int64_t dst_fb, int64_t src_fb, int64_t n_fb, dp_nic* nic);

/* Paged HBM pool with n_tickets rows of landed counters: row t holds one
 * counter per layer (items landed for that layer) and, in column n_layer,
 * the items landed over all layers of the ticket. */
int dp_pool_create(int device, const dp_kv_geom* geom, int32_t n_slots, int32_t n_tickets,
                   dp_pool** out);
/* Pool layouts.  Layer-major (dp_pool_create): one plane per layer,
 * [n_layer][n_slots][T][b], the per-layer paged layout attention kernels
 * read.  Block-major: [n_slots][n_layer][T][b], every slot a whole Full
 * Block, so the copy engine lands a run of storage Full Blocks in ONE
 * contiguous copy (dp_h2d_layer_copy / dp_h2d_push_copy and their _job
 * forms: no ring, no SM work) -- the loading path's kernels (K1 / K2 / staged
 * / K5 / checksum / copy-out) take either; the handoff and persistence
 * kernels take layer-major pools only (DP_EINVAL otherwise).  The layout
 * travels in dp_pool_handle (reserved[0]) to imported views. */
#define DP_POOL_LAYER_MAJOR 0
#define DP_POOL_BLOCK_MAJOR 1
int dp_pool_create_layout(int device, const dp_kv_geom* geom, int32_t n_slots, int32_t n_tickets, int32_t layout,
                          dp_pool** out);
int dp_pool_layout(const dp_pool* pool, int32_t* layout);
int dp_pool_destroy(dp_pool* pool);
int dp_pool_info(const dp_pool* pool, void** base, uint32_t** counters, int64_t* data_bytes);
int dp_pool_reset_counters(dp_pool* pool, dp_stream stream);
int dp_pool_export(const dp_pool* pool, dp_pool_handle* out);
/* Open an exported pool in another process (peer view used by DE engines). */
int dp_pool_import(int device, const dp_pool_handle* handle, dp_pool** out);
/* Same-process peer view of `pool` for `device` (enables P2P access). */
int dp_pool_peer_view(int device, const dp_pool* pool, dp_pool** out);

/* K1 (PE read path, LoopbackH2D): Layer Blocks from `src` (host, over the
 * PE's PCIe) into `pe` on the same device.  Bumps landed[ticket][layer] by
 * the number of items per layer (see dp_layer_items). */
int dp_h2d_layer_gather(dp_pool* pe, const dp_store* src, const dp_job* jobs, int32_t n_jobs,
                        dp_stream stream);
/* K2 (DE read path, DeToPe): run on the DE device: Layer Blocks from the DE's
 * store over the DE's PCIe, stored over NVLink into the PE pool `pe_view`
 * (from dp_pool_import / dp_pool_peer_view), then a system-scope release of
 * the PE's landed counters. */
int dp_h2d_push_p2p_layer(dp_pool* pe_view, const dp_store* de_src, const dp_job* jobs,
                          int32_t n_jobs, dp_stream de_stream);

/* ------------------------------------------------------------------------
 * PD handoff: PeToDe / MissMerge per layer
 * (desim.cpp:630-640) and DecodeH2D (desim.cpp:650-651, :740-747).
 *
 * B200 mapping: the DE's decode pool (a dp_pool on the DE) must end up
 * holding the whole prompt KV [0, C+A) of each request (de_need =
 * full(prompt), desim.cpp:592).  On one NVLink domain the DE's DRAM hop is
 * not needed:
 *   - DE read path: the DE reads each hit Layer Block from its host store
 *     ONCE and stores it both into the PE pool (NVLink, DeToPe) and into its
 *     own decode pool (local HBM: the hit half of DecodeH2D) —
 *     dp_h2d_push_p2p_dual;
 *   - per layer on the PE, after that layer's hit KV has landed, the
 *     prefill stand-in writes the miss tokens' KV [C, C+A) into the PE pool
 *     and the layer is pushed to the DE pool over NVLink: all prompt tokens
 *     on the PE read path (PeToDe), the miss tokens only on the DE read path
 *     (MissMerge) — dp_prefill_handoff (K3).
 * DE pool row of a request, per layer: (hit blocks if DE path, else 0) *
 * items_per_block from the dual gather + prompt blocks * items_per_block
 * from K3; column n_layer sums them over layers. */

typedef struct dp_dual_job {
  dp_job pe;               /* -> PE pool (peer view), as dp_h2d_push_p2p_layer */
  const int32_t* de_slot;  /* [pe.n_blk] slots in the DE's own decode pool */
  int32_t de_ticket;       /* DE pool landed-counter row, or -1 */
  int32_t reserved;
} dp_dual_job;

typedef struct dp_handoff_job {
  const int64_t* src_fb;   /* [n_blk] storage Full Block of each prompt block: the content
                              the prefill stand-in writes for the miss tokens */
  const int32_t* pe_slot;  /* [n_blk] the request's prompt blocks in the PE pool */
  const int32_t* de_slot;  /* [n_blk] its blocks in the DE decode pool */
  int64_t n_cached;        /* C: tokens [0, C) are hit KV (already in / landing in the PE pool) */
  int64_t n_prompt;        /* C + A */
  int32_t n_blk;           /* ceil((C + A) / T) */
  int32_t push_hit;        /* 1: PE read path (PeToDe moves C + A); 0: DE path (MissMerge moves A) */
  int32_t pe_ticket;       /* PE pool row whose layer l must reach pe_wait_items before layer l
                              is processed (the maybe_start_compute gate), or -1 (stream-ordered) */
  uint32_t pe_wait_items;  /* per-layer items of the hit KV */
  int32_t de_ticket;       /* DE pool row released per layer, or -1 */
  int32_t pe_done_ticket;  /* PE pool row released per item once its work (reads of the PE
                              pool included) is done, or -1: slot-reuse hazards */
} dp_handoff_job;

#define DP_MAX_DUAL_JOBS_PER_LAUNCH 48
#define DP_MAX_HANDOFF_JOBS_PER_LAUNCH 48

/* DE read path fused with DecodeH2D: run on the DE; one PCIe read per hit
 * Layer Block, stored to the PE pool (peer, system-scope release of its
 * counters) and to the DE's own decode pool `de_pool` (its counters too). */
int dp_h2d_push_p2p_dual(dp_pool* pe_view, dp_pool* de_pool, const dp_store* de_src,
                         const dp_dual_job* jobs, int32_t n_jobs, dp_stream de_stream);

/* K3, run on the PE: per layer (in order), per prompt block: wait for the
 * layer's hit KV (pe_ticket), write the miss tokens' KV (content formula of
 * the store, `seed`) into the PE pool, push the job's bytes of the layer to
 * the DE pool `de_view` (peer) and release the DE pool row.  A gate wait
 * longer than timeout_ms sets the PE pool's watchdog flag (dp_wait_status). */
int dp_prefill_handoff(dp_pool* pe_pool, dp_pool* de_view, const dp_handoff_job* jobs,
                       int32_t n_jobs, uint64_t seed, int32_t timeout_ms, dp_stream stream);

/* K3 on the copy engines: the transfer of dp_prefill_handoff with its bytes
 * moved by copy-engine copies over NVLink from the PE pool -- the whole
 * prompt on the PE path (PeToDe), the miss tokens on the DE path
 * (MissMerge); one copy per run of prompt blocks consecutive in both pools,
 * and with no gate (every pe_ticket -1) ONE 2D copy per run covers all
 * layers (rows = layers, pitches = the pools' layer planes).  Before a
 * layer's copies a small kernel (kv_handoff_side) releases the previous
 * layer's DE / pe_done rows (system scope, the same increments as K3's),
 * waits for the layer's gates (watchdog as K3's) and writes the miss
 * tokens' KV into the PE pool (gated calls: into both pools, the copies then
 * carry only PeToDe's hit part -- a few operations per layer, so a caller
 * that enqueues a gate's producer after this call on the same thread does
 * not fill the stream's queue behind the gate).  The final pools and
 * counters equal dp_prefill_handoff's.  Here the job arrays
 * (src_fb, pe_slot, de_slot) must be HOST-readable. */
int dp_prefill_handoff_copy(dp_pool* pe_pool, dp_pool* de_view, const dp_handoff_job* jobs, int32_t n_jobs,
                            uint64_t seed, int32_t timeout_ms, dp_stream stream);
/* Gates of dp_prefill_handoff_copy as stream waits (cuStreamWaitValue32 GEQ
 * on the PE pool's counter, no SM spinning, no watchdog) instead of the side
 * kernel's spin; process-wide.  For gates whose producer runs on the PE's own
 * GPU (the layerwise handoff's per-forward rows, released by K5). */
int dp_set_handoff_gate_memop(int32_t on);
/* Kernels dp_prefill_handoff_copy has launched in this process. */
int dp_handoff_copy_launches(int64_t* n);

/* ------------------------------------------------------------------------
 * Decode-side persistence: every 64 generated tokens
 * and at completion the DE persists the new tokens' KV to storage
 * (PersistD2H -> PersistWrite, desim.cpp:666-672, :690-693, :764-771).
 *
 * A span job names a session-token range [tok_begin, tok_end) that lies in
 * the session blocks blk0 .. blk0 + n_blk - 1; slot[i] is block blk0+i's slot
 * in the decode pool and fb[i] its storage Full Block. */
typedef struct dp_span_job {
  const int32_t* slot;  /* [n_blk] decode-pool slots */
  const int64_t* fb;    /* [n_blk] storage Full Blocks (content ids / persist targets) */
  int64_t blk0;         /* session block of slot[0] */
  int64_t tok_begin;    /* session tokens [tok_begin, tok_end) */
  int64_t tok_end;
  int32_t n_blk;
  int32_t reserved;
} dp_span_job;

#define DP_MAX_SPAN_JOBS_PER_LAUNCH 64

/* Decode stand-in: writes the KV of generated tokens (the storage content
 * formula with `seed`, i.e. what the turn will persist) into the decode pool. */
int dp_decode_fill(dp_pool* de_pool, const dp_span_job* jobs, int32_t n_jobs, uint64_t seed,
                   dp_stream stream);
/* K4 (PersistD2H): gathers the span's tokens of every layer from the decode
 * pool's layer planes into Full Blocks [L][T][b] of the pinned host `target`
 * (the storage tier), zero-copy stores over the DE's PCIe. */
int dp_persist_d2h(const dp_pool* de_pool, dp_store* target, const dp_span_job* jobs,
                   int32_t n_jobs, dp_stream stream);

/* ------------------------------------------------------------------------
 * Prefill stand-in driven by compute-quota batching (
 * build_forward_batch, proj/src/scheduler.cpp:174-219).
 *
 * K5 is the attention-score pass of one prefill layer for the items of one
 * forward batch: item i's query tokens [q_begin, q_begin + bsz) of its append
 * attend to its cached tokens [0, cached) of `layer`, read from the PE pool
 * (the KV the loader landed).  Queries are procedural bytes
 *   q(req, layer, q, w) = splitmix64(qbase ^ (q << 16 | w)),
 *   qbase = splitmix64((req << 20 | layer) ^ seed * 0xA24BAED4963EE407),
 * and the pass accumulates, exactly (mod 2^64), into digest[layer]
 *   sum_q sum_t dot_u8(Q[q], K[t])      (unsigned bytes, b per token)
 * on CUDA cores (dp4a): bsz * cached * b multiply-adds, the bilinear term of
 * the cost model.  Chunking a request over several forwards splits its
 * queries, so the digest of a request is independent of the batching. */
typedef struct dp_attend_item {
  const int32_t* slot;  /* [ceil(cached / T)] PE-pool slots of the cached blocks */
  int64_t cached;       /* keys: tokens [0, cached) */
  int64_t q_begin;      /* first query token (offset into the append) */
  int64_t bsz;          /* query tokens of this chunk */
  uint64_t* digest;     /* [n_layer] device accumulators of the request */
  uint32_t req;         /* request key of the procedural queries */
  int32_t reserved;
} dp_attend_item;

#define DP_MAX_ATTEND_ITEMS_PER_LAUNCH 48

/* K5 launches on one pool must be stream-ordered (they share the pool's
 * work-queue counter). */
int dp_prefill_attend(const dp_pool* pe_pool, int32_t layer, const dp_attend_item* items,
                      int32_t n_items, uint64_t seed, dp_stream stream);
/* The same, then *done = 1 (gpu-scope release by the last CTA out; a stream
 * write when there is nothing to compute): the layer's "computed" flag a
 * layerwise K3 gates on (desim.cpp:630-640). */
int dp_prefill_attend_signal(const dp_pool* pe_pool, int32_t layer, const dp_attend_item* items,
                             int32_t n_items, uint64_t seed, uint32_t* done, dp_stream stream);
/* Cap on the CTAs of a K5 launch on `device` (0 = default: every SM). */
int dp_set_attend_ctas(int device, int32_t ctas);

/* K1 on the copy engine (no SMs): the same transfer as dp_h2d_layer_gather,
 * issued as one strided cudaMemcpy2DAsync per contiguous run of blocks per
 * layer (Full-Block pitch -> Layer-Block pitch) plus the partial last block,
 * and after each layer a stream-ordered, fenced 32-bit write of the landed
 * counters (cuStreamWriteValue32): ctr[ticket][l] = items, ctr[ticket][L] =
 * items * layers done (absolute values: jobs start at layer 0 and a ticket
 * belongs to one job per call, else DP_EINVAL).  The isolation mode for a PE
 * that is computing.
 * HERE the dp_job block arrays (src_fb, dst_slot) must be HOST-readable. */
int dp_h2d_layer_copy(dp_pool* pe, const dp_store* src, const dp_job* jobs, int32_t n_jobs,
                      dp_stream stream);
/* K2 on the DE's copy engine (no SMs on either GPU): the transfer of
 * dp_h2d_push_p2p_layer as strided copies from the DE's pinned store into
 * the PE pool through its peer view (NVLink), then fenced stream writes of
 * the PE's landed counters.  Block arrays HOST-readable, as above. */
int dp_h2d_push_copy(dp_pool* pe_view, const dp_store* de_src, const dp_job* jobs, int32_t n_jobs,
                     dp_stream de_stream);
/* The same two, releasing each job's counters once after its last layer
 * (a stream write waits for the copies before it: per-layer releases idle
 * the copy engine once per layer).  Consumers see all layers land at once. */
int dp_h2d_layer_copy_job(dp_pool* pe, const dp_store* src, const dp_job* jobs, int32_t n_jobs,
                          dp_stream stream);
int dp_h2d_push_copy_job(dp_pool* pe_view, const dp_store* de_src, const dp_job* jobs, int32_t n_jobs,
                         dp_stream de_stream);

/* Staged K1 / K2: the copy engine moves whole Full-Block runs host -> an HBM
 * staging ring at the link's full rate (1D copies of contiguous runs, a 2D
 * copy of the valid rows of a partial last block), then the gather kernel
 * scatters the ring into the pool's layer planes (K2: over NVLink into the
 * PE pool) and releases the landed counters as K1 / K2 do.  The copies run
 * on the stager's own stream, the scatters on `stream` (ordered after its
 * earlier work; later work on `stream` sees the landed bytes).  Jobs move
 * all layers; src_fb HOST-readable, dst_slot device-readable.  A stager
 * serves one stream at a time.  ring_bytes 0 = 1 GiB. */
typedef struct dp_stager dp_stager;
int dp_stager_create(int device, const dp_kv_geom* geom, int64_t ring_bytes, dp_stager** out);
int dp_stager_destroy(dp_stager* stager);
int dp_stager_set_ctas(dp_stager* stager, int32_t ctas);  /* scatter CTAs (0 = 32) */
int dp_stager_launches(const dp_stager* stager, int64_t* n);  /* scatter kernels so far */
/* The scatter ring -> pool: DP_SCATTER_KERNEL (default; kv_gather from the
 * ring, dst_slot device-readable) or DP_SCATTER_CE (copy engines only: one 2D
 * copy per run of consecutive slots per layer + fenced stream writes of the
 * landed counters, absolute values as dp_h2d_layer_copy's; dst_slot
 * HOST-readable; no SM work on either GPU). */
#define DP_SCATTER_KERNEL 0
#define DP_SCATTER_CE 1
int dp_stager_set_mode(dp_stager* stager, int32_t mode);
int dp_h2d_layer_staged(dp_pool* pe, const dp_store* src, dp_stager* stager, const dp_job* jobs,
                        int32_t n_jobs, dp_stream stream);
int dp_h2d_push_staged(dp_pool* pe_view, const dp_store* de_src, dp_stager* stager, const dp_job* jobs,
                       int32_t n_jobs, dp_stream de_stream);
/* The DE read path fused with DecodeH2D (dp_h2d_push_p2p_dual), staged: the
 * copy engine into the ring, then the dual scatter stores each Layer Block to
 * the PE pool over NVLink and to the DE's decode pool.  src_fb HOST-readable,
 * dst_slot / de_slot device-readable; jobs move all layers. */
int dp_h2d_push_dual_staged(dp_pool* pe_view, dp_pool* de_pool, const dp_store* de_src, dp_stager* stager,
                            const dp_dual_job* jobs, int32_t n_jobs, dp_stream de_stream);

/* K4 staged (PersistD2H at the copy engine's rate): a gather kernel packs the
 * spans' tokens from the decode pool into Full Blocks of the stager's HBM
 * ring, the copy engine moves them to `target` (whole blocks as 1D runs, a
 * partial block as one 2D copy of its L token ranges); consecutive spans of
 * one request are merged.  The same bytes as dp_persist_d2h; later work on
 * `stream` sees them in host memory.  fb HOST-readable, slot device-readable.
 * Use a stager of its own (not one a loader uses on another stream). */
int dp_persist_staged(const dp_pool* de_pool, dp_store* target, dp_stager* stager, const dp_span_job* jobs,
                      int32_t n_jobs, dp_stream stream);

/* Cap on the CTAs a K1/K2 launch on `device` may use (0 = default, 4 per SM).
 * The transfer is PCIe-bound, so a few CTAs keep the link full while leaving
 * the SMs to the prefill compute (the isolation knob of config 4). */
int dp_set_gather_ctas(int device, int32_t ctas);

/* Cap on the CTAs of a K3 (dp_prefill_handoff) launch on `device` (0 =
 * default, 2 per SM: 699 GB/s of NVLink pushes, profiles/r01_SUMMARY.md). */
int dp_set_handoff_ctas(int device, int32_t ctas);
/* K3's PE-path hit push through the TMA (cp.async.bulk HBM -> shared -> peer
 * HBM, 4 x 16 KB stages per CTA) instead of 16-byte register copies; process-wide. */
int dp_set_handoff_tma(int32_t on);

/* Items (landed-counter increments) per layer for a job of n_blk blocks. */
int dp_layer_items(const dp_kv_geom* geom, int32_t n_blk, int32_t* out);

/* Block `stream` until landed[ticket][layer] >= target (acquire, system
 * scope; layer == n_layer waits on the all-layer column), with a watchdog of
 * timeout_ms (then DP_ETIMEOUT via dp_wait_status). */
int dp_wait_layer(const dp_pool* pool, int32_t ticket, int32_t layer, uint32_t target,
                  int32_t timeout_ms, dp_stream stream);
/* Same for n tickets at once (tickets/targets device-accessible). */
int dp_wait_tickets(const dp_pool* pool, const int32_t* tickets, const uint32_t* targets,
                    int32_t n, int32_t layer, int32_t timeout_ms, dp_stream stream);
/* Make `stream` wait, without occupying SMs (cuStreamWaitValue32, GEQ), until
 * the LOCAL pool's landed[ticket][layer] >= target.  No watchdog: use it for
 * producers that are known to run (the executor's whole-request gate). */
int dp_stream_wait_counter(const dp_pool* pool, int32_t ticket, int32_t layer, uint32_t target,
                           dp_stream stream);
/* Stream-ordered, fenced write of landed[ticket][layer] = value on a LOCAL
 * pool (cuStreamWriteValue32): marks the completion of copy-engine or
 * stream-ordered work that has no kernel of its own to release a counter. */
int dp_stream_write_counter(dp_pool* pool, int32_t ticket, int32_t layer, uint32_t value,
                            dp_stream stream);
/* Returns DP_ETIMEOUT if any wait issued through this pool (or view) has timed out. */
int dp_wait_status(const dp_pool* pool);
/* Clears that watchdog flag (dp_pool_reset_counters does it for an owned pool). */
int dp_wait_clear(dp_pool* pool);

/* 64-bit content hash of each listed Layer Block (valid tokens only):
 *   H = sum_i splitmix64(word_i + (i + 1) * 0x9E3779B97F4A7C15)  (mod 2^64)
 * slots/ntok/out are device-accessible arrays of length n. */
int dp_pool_checksum(const dp_pool* pool, int32_t layer, const int32_t* slots,
                     const int32_t* ntok, int32_t n, uint64_t* out, dp_stream stream);

/* Synchronous copy of `bytes` bytes of pool Layer Block (layer, slot) to
 * host memory (inspection / parity checks). */
int dp_pool_copy_out(const dp_pool* pool, int32_t layer, int32_t slot, int64_t bytes,
                     void* host_out);
/* Number of CUDA devices visible (0 when none). */
int dp_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* DUALPATH_KV_ABI_H */
