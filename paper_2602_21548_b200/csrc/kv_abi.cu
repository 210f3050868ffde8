// B200 (sm_100a) implementation of the DualPath KV loading C ABI
// (include/dualpath/kv_abi.h).
//
// Kernels:
//   K1 kv_gather<false>  — LoopbackH2D (proj/src/desim.cpp:614-616): Layer Blocks
//       of Full Blocks in pinned host DRAM -> paged PE HBM pool, zero-copy
//       16-byte loads over the PE's PCIe link.
//   K2 kv_gather<true>   — DeToPe (proj/src/desim.cpp:617-619): the same gather
//       run on the DE GPU, reading the DE's host DRAM over the DE's PCIe link
//       and storing straight into the PE pool over NVLink (peer pointer),
//       then a system-scope release of the PE's per-layer landed counter.
//   kv_wait_ge           — the layer gate of maybe_start_compute (desim.cpp:623-628).
//   kv_block_checksum    — per-Layer-Block content hash for parity checks.
//   kv_store_fill        — deterministic storage content (restated in oracle/kvref.c).
//
// Work decomposition: one CTA-sized item = one chunk (<= 64 KiB) of one
// Layer Block.  Items are ordered (job, layer, block, chunk) so a request's
// layer l lands before l+1 (layerwise prefill).  A launch
// carries up to DP_MAX_JOBS_PER_LAUNCH job headers in its parameter block;
// each warp decodes its item's job with a ballot over the job prefix sums.
#include <cuda.h>
#include <cuda_runtime.h>

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cctype>
#include <mutex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "dualpath/kv_abi.h"

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 8;
constexpr int64_t kChunkBytes = 64 * 1024;  // max bytes per item
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kSeedMul = 0xD1B54A32D192ED03ull;

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace

namespace dualpath::detail {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace dualpath::detail

namespace {

#define DP_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(DP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (dev != prev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + kGolden;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct GatherParams {
  const char* store;     // source Full Blocks (device-visible host pointer)
  char* pool;            // destination pool data base (local or peer)
  uint32_t* counters;    // destination landed counters [n_tickets][n_layer + 1]
  int64_t lb_bytes;      // Layer Block bytes T*b
  int64_t fb_bytes;      // Full Block bytes L*T*b
  int64_t bpt;           // b, bytes per token per layer
  int64_t layer_stride;  // pool: layer plane (layer-major) or Layer Block (block-major)
  int64_t slot_stride;   // pool: Layer Block (layer-major) or Full Block (block-major)
  int32_t n_layer;
  int32_t block_tokens;
  int32_t n_chunk;       // items per Layer Block
  int32_t n_jobs;
  int64_t item_begin[DP_MAX_JOBS_PER_LAUNCH + 1];
  dp_job jobs[DP_MAX_JOBS_PER_LAUNCH];
};
static_assert(sizeof(GatherParams) <= 4000, "kernel parameter block too large");
static_assert(sizeof(dp_pool_handle) == 128, "dp_pool_handle is a fixed 128-byte wire format");
static_assert(sizeof(dp_job) == 40, "dp_job layout");

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Warp-cooperative decode of the job owning `item`: lane j tests job
// j (and j+32), the ballot's population count is the job index.
template <class Params>
__device__ __forceinline__ int decode_job(const Params& p, int64_t item) {
  const int lane = threadIdx.x & 31;
  const unsigned lo = __ballot_sync(
      0xffffffffu, lane + 1 < p.n_jobs && p.item_begin[lane + 1] <= item);
  const unsigned hi = __ballot_sync(
      0xffffffffu, lane + 33 < p.n_jobs && p.item_begin[lane + 33] <= item);
  return __popc(lo) + __popc(hi);
}

// L2 evict-first variants for the staged scatter (ring -> pool): the bytes
// pass through L2 once, so they should not displace a co-running kernel's
// working set (config 4's GEMM stand-in).
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_stream_ef(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_v4_ef(uint4* p, const uint4& v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

// kStream: the staged scatter's ring -> pool copy (L2 evict-first both ways).
template <bool kPeer, bool kStream = false>
__global__ void __launch_bounds__(kThreads) kv_gather(const __grid_constant__ GatherParams p) {
  const int64_t total = p.item_begin[p.n_jobs];
  const int tid = threadIdx.x;
  const uint64_t pol = kStream ? evict_first_policy() : 0;
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
    const int j = decode_job(p, item);
    const dp_job& job = p.jobs[j];
    const int64_t local = item - p.item_begin[j];
    const int64_t per_layer = static_cast<int64_t>(job.n_blk) * p.n_chunk;
    const int layer = job.layer_begin + static_cast<int>(local / per_layer);
    const int64_t rem = local % per_layer;
    const int blk = static_cast<int>(rem / p.n_chunk);
    const int chunk = static_cast<int>(rem % p.n_chunk);

    const int64_t fb = job.src_fb[blk];
    const int64_t slot = job.dst_slot[blk];
    const int64_t tok0 = static_cast<int64_t>(blk) * p.block_tokens;
    const int64_t ntok = min(static_cast<int64_t>(p.block_tokens), job.n_tokens - tok0);
    const int64_t valid = ntok * p.bpt;
    const int64_t beg = static_cast<int64_t>(chunk) * kChunkBytes;
    const int64_t end = min(beg + kChunkBytes, valid);

    if (end > beg) {
      const uint4* src = reinterpret_cast<const uint4*>(p.store + fb * p.fb_bytes +
                                                        layer * p.lb_bytes + beg);
      uint4* dst = reinterpret_cast<uint4*>(p.pool + layer * p.layer_stride +
                                            slot * p.slot_stride + beg);
      const int n16 = static_cast<int>((end - beg) >> 4);
      for (int base = 0; base < n16; base += kThreads * kUnroll) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int i = base + u * kThreads + tid;
          if (i < n16) v[u] = kStream ? ld_stream_ef(src + i, pol) : ld_stream(src + i);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int i = base + u * kThreads + tid;
          if (i < n16) {
            if (kStream && !kPeer) st_v4_ef(dst + i, v[u], pol);
            else st_v4(dst + i, v[u]);
          }
        }
      }
    }
    if (job.ticket >= 0) {
      // all of this CTA's stores are ordered before the counter release
      __syncthreads();
      if (tid == 0) {
        uint32_t* row = p.counters + static_cast<int64_t>(job.ticket) * (p.n_layer + 1);
        // one fence after the CTA barrier, then relaxed reductions (a
        // release pattern; consumers acquire)
        if (kPeer) {
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(row + layer) : "memory");
          asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(row + p.n_layer) : "memory");
        } else {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(row + layer) : "memory");
          asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(row + p.n_layer) : "memory");
        }
      }
    }
  }
}

__device__ __forceinline__ uint64_t global_timer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void kv_wait_ge(const uint32_t* ctr, uint32_t target, uint64_t timeout_ns,
                           int* err_flag) {
  const uint64_t t0 = global_timer_ns();
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    if (global_timer_ns() - t0 > timeout_ns) {
      atomicExch_system(err_flag, 1);
      break;
    }
    __nanosleep(256);
  }
}

// One thread per (counter, target) pair; used to make an engine's step end
// cover every push that lands in its pool, and for slot-reuse hazards.
__global__ void kv_wait_many(const uint32_t* counters, int32_t row_len, const int32_t* tickets,
                             const uint32_t* targets, int32_t n, int32_t col,
                             uint64_t timeout_ns, int* err_flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* ctr = counters + static_cast<int64_t>(tickets[i]) * row_len + col;
  const uint32_t target = targets[i];
  const uint64_t t0 = global_timer_ns();
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    if (global_timer_ns() - t0 > timeout_ns) {
      atomicExch_system(err_flag, 1);
      break;
    }
    __nanosleep(512);
  }
}

__global__ void __launch_bounds__(kThreads)
    kv_block_checksum(const char* pool, int64_t layer_off, int64_t slot_stride, int64_t bpt,
                      const int32_t* slots, const int32_t* ntok, int32_t n, uint64_t* out) {
  __shared__ uint64_t partial[kThreads / 32];
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const uint64_t* words =
        reinterpret_cast<const uint64_t*>(pool + layer_off + static_cast<int64_t>(slots[b]) * slot_stride);
    const int64_t nw = static_cast<int64_t>(ntok[b]) * bpt / 8;
    uint64_t acc = 0;
    for (int64_t i = threadIdx.x; i < nw; i += kThreads)
      acc += splitmix64(words[i] + static_cast<uint64_t>(i + 1) * kGolden);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) partial[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t s = 0;
      for (int w = 0; w < kThreads / 32; ++w) s += partial[w];
      out[b] = s;
    }
    __syncthreads();
  }
}

// word(p, w) = splitmix64((p << 32 | w) ^ seed*kSeedMul), two words per thread;
// dst holds Full Blocks fb0, fb0 + 1, ... (the content is keyed on p).
__global__ void kv_store_fill(uint64_t* dst, int64_t n_pairs, int64_t words_per_fb,
                              uint64_t seed_mix, int64_t fb0) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_pairs;
       i += stride) {
    const int64_t w0 = 2 * i;
    const uint64_t fb = static_cast<uint64_t>(fb0 + w0 / words_per_fb);
    const uint64_t w = static_cast<uint64_t>(w0 % words_per_fb);
    const uint64_t a = splitmix64(((fb << 32) | w) ^ seed_mix);
    const uint64_t b = splitmix64(((fb << 32) | (w + 1)) ^ seed_mix);
    asm volatile("st.global.v2.u64 [%0], {%1,%2};" ::"l"(dst + w0), "l"(a), "l"(b) : "memory");
  }
}

constexpr int kMaxDevices = 64;
// per-device CTA caps (0 = default); set by one thread, read by launching ones
std::atomic<int> g_gather_ctas[kMaxDevices] = {};
std::atomic<int> g_handoff_ctas[kMaxDevices] = {};
std::atomic<bool> g_handoff_tma{false};  // K3 hit push through the TMA (dp_set_handoff_tma)

int sm_count(int device) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  return n > 0 ? n : 148;
}

int64_t chunks_per_block(const dp_kv_geom& g) {
  const int64_t lb = static_cast<int64_t>(g.block_tokens) * g.bytes_per_token_layer;
  return (lb + kChunkBytes - 1) / kChunkBytes;
}

bool geom_equal(const dp_kv_geom& a, const dp_kv_geom& b) {
  return a.n_layer == b.n_layer && a.block_tokens == b.block_tokens &&
         a.bytes_per_token_layer == b.bytes_per_token_layer;
}

}  // namespace

struct dp_store {
  int device = -1;
  dp_kv_geom geom{};
  int64_t n_fb = 0;
  uint64_t seed = 0;
  char* host = nullptr;
  int64_t bytes = 0;
  int numa_node = -1;       // node the pages are bound to (-1: not bound)
  bool registered = false;  // mmap + cudaHostRegister (else cudaHostAlloc)
  int64_t map_bytes = 0;
};

struct dp_pool {
  int device = -1;  // device whose address space `base` lives in
  int home_device = -1;
  dp_kv_geom geom{};
  int32_t n_slots = 0;
  int32_t n_tickets = 0;
  char* base = nullptr;
  uint32_t* counters = nullptr;
  int64_t data_bytes = 0;
  bool owner = false;
  bool ipc_opened = false;
  int* err_host = nullptr;  // mapped pinned watchdog flag
  uint32_t* att_ctr = nullptr;  // K5 work-queue counters {next unit, CTAs done} (owner pools)
  int32_t layout = 0;           // DP_POOL_LAYER_MAJOR or DP_POOL_BLOCK_MAJOR
};

namespace {

int64_t counters_offset(int64_t data_bytes) { return (data_bytes + 255) / 256 * 256; }

// Layer Block (layer, slot) of a pool lives at layer * layer_stride + slot *
// slot_stride: layer planes [L][slots][T][b] (layer-major, the default) or
// whole Full Blocks per slot [slots][L][T][b] (block-major).
int64_t pool_lb(const dp_pool* p) { return static_cast<int64_t>(p->geom.block_tokens) * p->geom.bytes_per_token_layer; }
int64_t layer_stride(const dp_pool* p) {
  return p->layout == DP_POOL_BLOCK_MAJOR ? pool_lb(p) : pool_lb(p) * p->n_slots;
}
int64_t slot_stride(const dp_pool* p) {
  return p->layout == DP_POOL_BLOCK_MAJOR ? pool_lb(p) * p->geom.n_layer : pool_lb(p);
}

// Loads every kernel of this library on `device` (defined at the end of the
// file, after the last kernel).  With CUDA's lazy loading a kernel is loaded
// at its first launch, and a load waits for the device's running kernels: a
// spin-waiting consumer (K3's layer gate, kv_wait_many) would then hold back
// the very launch of its producer when both share a GPU.
int preload_kernels(int device);

// The dual gather (DeToPe + the hit half of DecodeH2D) from any device-visible
// Full-Block source: the DE's host store, or a stager ring.
int launch_dual(dp_pool* pe_view, dp_pool* de_pool, const dp_store* src, const dp_dual_job* jobs, int32_t n_jobs,
                dp_stream stream, int ctas_override);

int launch_gather(dp_pool* pool, const dp_store* src, const dp_job* jobs, int32_t n_jobs,
                  dp_stream stream, bool peer, int ctas_override = 0, bool stream_hint = false) {
  if (!pool || !src || (n_jobs > 0 && !jobs) || n_jobs < 0)
    return fail(DP_EINVAL, "gather: null argument");
  if (!geom_equal(pool->geom, src->geom))
    return fail(DP_EINVAL, "gather: pool and store geometry differ");
  if (peer == pool->owner)
    return fail(DP_EINVAL, peer ? "push_p2p: destination must be a peer view of the PE pool"
                                : "h2d_gather: destination must be the local PE pool");
  const dp_kv_geom& g = pool->geom;
  DeviceGuard guard(pool->device);
  GatherParams p;
  std::memset(&p, 0, sizeof(p));
  p.store = src->host;
  p.pool = pool->base;
  p.counters = pool->counters;
  p.lb_bytes = static_cast<int64_t>(g.block_tokens) * g.bytes_per_token_layer;
  p.fb_bytes = p.lb_bytes * g.n_layer;
  p.bpt = g.bytes_per_token_layer;
  p.layer_stride = layer_stride(pool);
  p.slot_stride = slot_stride(pool);
  p.n_layer = g.n_layer;
  p.block_tokens = g.block_tokens;
  p.n_chunk = static_cast<int32_t>(chunks_per_block(g));
  const int dev_cap = (pool->device >= 0 && pool->device < kMaxDevices) ? g_gather_ctas[pool->device].load() : 0;
  const int grid_cap = ctas_override > 0 ? ctas_override : dev_cap > 0 ? dev_cap : sm_count(pool->device) * 4;
  auto s = static_cast<cudaStream_t>(stream);
  for (int32_t j0 = 0; j0 < n_jobs; j0 += DP_MAX_JOBS_PER_LAUNCH) {
    const int32_t nj = std::min<int32_t>(DP_MAX_JOBS_PER_LAUNCH, n_jobs - j0);
    p.n_jobs = 0;
    int64_t items = 0;
    for (int32_t j = 0; j < nj; ++j) {
      const dp_job& job = jobs[j0 + j];
      if (job.n_tokens < 0 || job.n_blk < 0 || job.layer_begin < 0 ||
          job.layer_end > g.n_layer || job.layer_begin > job.layer_end)
        return fail(DP_EINVAL, "gather: job " + std::to_string(j0 + j) + " out of range");
      const int64_t need_blk = (job.n_tokens + g.block_tokens - 1) / g.block_tokens;
      if (need_blk != job.n_blk)
        return fail(DP_EINVAL, "gather: job " + std::to_string(j0 + j) +
                                   " n_blk != ceil(n_tokens / block_tokens)");
      if (job.ticket >= pool->n_tickets)
        return fail(DP_EINVAL, "gather: ticket out of range");
      if (job.n_blk > 0 && (!job.src_fb || !job.dst_slot))
        return fail(DP_EINVAL, "gather: null block arrays");
      const int64_t n = static_cast<int64_t>(job.n_blk) * p.n_chunk *
                        (job.layer_end - job.layer_begin);
      if (n == 0) continue;
      p.jobs[p.n_jobs] = job;
      p.item_begin[p.n_jobs] = items;
      ++p.n_jobs;
      items += n;
    }
    p.item_begin[p.n_jobs] = items;
    if (items == 0) continue;
    const int grid = static_cast<int>(std::min<int64_t>(items, grid_cap));
    if (peer && stream_hint)
      kv_gather<true, true><<<grid, kThreads, 0, s>>>(p);
    else if (peer)
      kv_gather<true><<<grid, kThreads, 0, s>>>(p);
    else if (stream_hint)
      kv_gather<false, true><<<grid, kThreads, 0, s>>>(p);
    else
      kv_gather<false><<<grid, kThreads, 0, s>>>(p);
    DP_CUDA(cudaGetLastError());
  }
  return DP_OK;
}

}  // namespace

extern "C" {

int dp_abi_version(void) { return DP_ABI_VERSION; }

const char* dp_last_error(void) { return g_last_error.c_str(); }

int dp_geom_check(const dp_kv_geom* g) {
  if (!g) return fail(DP_EINVAL, "geom: null");
  if (g->n_layer < 1) return fail(DP_EINVAL, "geom: n_layer must be >= 1");
  if (g->block_tokens < 1) return fail(DP_EINVAL, "geom: block_tokens must be >= 1");
  if (g->bytes_per_token_layer <= 0 || g->bytes_per_token_layer % 16 != 0)
    return fail(DP_EINVAL, "geom: bytes_per_token_layer must be a positive multiple of 16");
  const int64_t fb = static_cast<int64_t>(g->n_layer) * g->block_tokens * g->bytes_per_token_layer;
  if (fb / 8 >= (int64_t{1} << 32)) return fail(DP_EINVAL, "geom: Full Block too large");
  return DP_OK;
}

int dp_device_numa_node(int device, int32_t* node) {
  if (!node) return fail(DP_EINVAL, "device_numa_node: null out");
  *node = -1;
  char bus[64] = {0};
  DP_CUDA(cudaDeviceGetPCIBusId(bus, sizeof(bus), device));
  for (char* c = bus; *c; ++c) *c = static_cast<char>(std::tolower(static_cast<unsigned char>(*c)));
  const std::string path = std::string("/sys/bus/pci/devices/") + bus + "/numa_node";
  if (FILE* f = std::fopen(path.c_str(), "r")) {
    int n = -1;
    if (std::fscanf(f, "%d", &n) == 1 && n >= 0) *node = n;
    std::fclose(f);
  }
  return DP_OK;
}

namespace {

// Pinned, device-mapped host memory whose pages live on NUMA node `node`
// (mmap + mbind(MPOL_BIND) + transparent huge pages + cudaHostRegister);
// falls back to cudaHostAlloc when the node is unknown or binding fails.
int alloc_store_pages(dp_store* st, int node) {
  if (node >= 0 && node < 128) {
    const int64_t huge = int64_t{2} << 20;
    const int64_t len = (st->bytes + huge - 1) / huge * huge;
    void* p = mmap(nullptr, static_cast<size_t>(len), PROT_READ | PROT_WRITE,
                   MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p != MAP_FAILED) {
      unsigned long mask[2] = {0, 0};
      mask[node / 64] = 1ul << (node % 64);
      const long rc = syscall(SYS_mbind, p, static_cast<unsigned long>(len), 2 /* MPOL_BIND */, mask,
                              129ul, 0u);
      madvise(p, static_cast<size_t>(len), MADV_HUGEPAGE);  // fewer IOMMU / TLB entries
      if (rc == 0 && cudaHostRegister(p, static_cast<size_t>(len),
                                      cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
        st->host = static_cast<char*>(p);
        st->registered = true;
        st->map_bytes = len;
        st->numa_node = node;
        return DP_OK;
      }
      cudaGetLastError();
      munmap(p, static_cast<size_t>(len));
    }
  }
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&st->host), st->bytes,
                                cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess)
    return fail(DP_ENOMEM, std::string("store_create: cudaHostAlloc: ") + cudaGetErrorString(e));
  return DP_OK;
}

void free_store_pages(dp_store* st) {
  if (!st->host) return;
  if (st->registered) {
    cudaHostUnregister(st->host);
    munmap(st->host, static_cast<size_t>(st->map_bytes));
  } else {
    cudaFreeHost(st->host);
  }
  cudaGetLastError();
  st->host = nullptr;
}

// Full Blocks [dst_fb, dst_fb + n) of `st` <- content of Full Blocks src_fb.. (GPU fill
// on the store's device, zero-copy stores over its PCIe link), synchronous.
int fill_store_range(dp_store* st, int64_t dst_fb, int64_t src_fb, int64_t n) {
  const dp_kv_geom& g = st->geom;
  const int64_t fb = static_cast<int64_t>(g.n_layer) * g.block_tokens * g.bytes_per_token_layer;
  DeviceGuard guard(st->device);
  cudaStream_t s;
  DP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  kv_store_fill<<<sm_count(st->device) * 8, kThreads, 0, s>>>(
      reinterpret_cast<uint64_t*>(st->host + dst_fb * fb), n * fb / 16, fb / 8, st->seed * kSeedMul, src_fb);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return fail(DP_ECUDA, std::string("store fill: ") + cudaGetErrorString(e));
  return DP_OK;
}

}  // namespace

int dp_store_create_on_node(int device, const dp_kv_geom* geom, int64_t n_fb, uint64_t seed,
                            int32_t numa_node, dp_store** out) {
  if (!out) return fail(DP_EINVAL, "store_create: null out");
  *out = nullptr;
  if (int rc = dp_geom_check(geom)) return rc;
  if (n_fb < 1) return fail(DP_EINVAL, "store_create: n_fb must be >= 1");
  if (numa_node < DP_NUMA_NONE) return fail(DP_EINVAL, "store_create: bad NUMA node");
  if (int rc = preload_kernels(device)) return rc;
  int32_t node = numa_node;
  if (numa_node == DP_NUMA_DEVICE)
    if (int rc = dp_device_numa_node(device, &node)) return rc;
  auto* st = new dp_store;
  st->device = device;
  st->geom = *geom;
  st->n_fb = n_fb;
  st->seed = seed;
  st->bytes = static_cast<int64_t>(geom->n_layer) * geom->block_tokens * geom->bytes_per_token_layer * n_fb;
  if (int rc = alloc_store_pages(st, node == DP_NUMA_NONE ? -1 : node)) {
    delete st;
    return rc;
  }
  if (int rc = fill_store_range(st, 0, 0, n_fb)) {
    free_store_pages(st);
    delete st;
    return rc;
  }
  *out = st;
  return DP_OK;
}

int dp_store_create(int device, const dp_kv_geom* geom, int64_t n_fb, uint64_t seed,
                    dp_store** out) {
  return dp_store_create_on_node(device, geom, n_fb, seed, DP_NUMA_DEVICE, out);
}

int dp_store_destroy(dp_store* st) {
  if (!st) return DP_OK;
  free_store_pages(st);
  delete st;
  return DP_OK;
}

int dp_storage_read(dp_store* staging, int64_t dst_fb, int64_t src_fb, int64_t n_fb, dp_nic* nic) {
  if (!staging || n_fb < 0 || dst_fb < 0 || src_fb < 0 || dst_fb + n_fb > staging->n_fb ||
      src_fb > (int64_t{1} << 31) - n_fb)
    return fail(DP_EINVAL, "storage_read: range out of bounds");
  if (n_fb == 0) return DP_OK;
  const dp_kv_geom& g = staging->geom;
  const int64_t bytes = static_cast<int64_t>(g.n_layer) * g.block_tokens * g.bytes_per_token_layer * n_fb;
  if (nic)
    if (int rc = dp_nic_read(nic, bytes, 0.0, nullptr, nullptr)) return rc;
  return fill_store_range(staging, dst_fb, src_fb, n_fb);
}

int dp_store_numa_node(const dp_store* st, int32_t* node) {
  if (!st || !node) return fail(DP_EINVAL, "store_numa_node: null argument");
  *node = st->numa_node;
  return DP_OK;
}

int dp_store_info(const dp_store* st, void** host_ptr, int64_t* bytes, int64_t* n_fb) {
  if (!st) return fail(DP_EINVAL, "store_info: null store");
  if (host_ptr) *host_ptr = st->host;
  if (bytes) *bytes = st->bytes;
  if (n_fb) *n_fb = st->n_fb;
  return DP_OK;
}

int dp_pool_create(int device, const dp_kv_geom* geom, int32_t n_slots, int32_t n_tickets,
                   dp_pool** out) {
  return dp_pool_create_layout(device, geom, n_slots, n_tickets, DP_POOL_LAYER_MAJOR, out);
}

int dp_pool_create_layout(int device, const dp_kv_geom* geom, int32_t n_slots, int32_t n_tickets, int32_t layout,
                          dp_pool** out) {
  if (!out) return fail(DP_EINVAL, "pool_create: null out");
  if (layout != DP_POOL_LAYER_MAJOR && layout != DP_POOL_BLOCK_MAJOR) return fail(DP_EINVAL, "pool_create: bad layout");
  *out = nullptr;
  if (int rc = dp_geom_check(geom)) return rc;
  if (n_slots < 1 || n_tickets < 0) return fail(DP_EINVAL, "pool_create: bad sizes");
  if (int rc = preload_kernels(device)) return rc;
  DeviceGuard guard(device);
  auto* pool = new dp_pool;
  pool->device = pool->home_device = device;
  pool->geom = *geom;
  pool->n_slots = n_slots;
  pool->n_tickets = n_tickets;
  pool->layout = layout;
  pool->data_bytes = static_cast<int64_t>(geom->n_layer) * n_slots * geom->block_tokens *
                     geom->bytes_per_token_layer;
  const int64_t ctr_bytes = static_cast<int64_t>(n_tickets) * (geom->n_layer + 1) * 4;
  const int64_t total = counters_offset(pool->data_bytes) + std::max<int64_t>(ctr_bytes, 256);
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&pool->base), total);
  if (e != cudaSuccess) {
    delete pool;
    return fail(DP_ENOMEM, std::string("pool_create: cudaMalloc: ") + cudaGetErrorString(e));
  }
  pool->counters = reinterpret_cast<uint32_t*>(pool->base + counters_offset(pool->data_bytes));
  pool->owner = true;
  e = cudaMemset(pool->counters, 0, std::max<int64_t>(ctr_bytes, 256));
  if (e == cudaSuccess)
    e = cudaHostAlloc(reinterpret_cast<void**>(&pool->err_host), sizeof(int), cudaHostAllocMapped |
                                                                            cudaHostAllocPortable);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&pool->att_ctr), 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(pool->att_ctr, 0, 2 * sizeof(uint32_t));
  if (e != cudaSuccess) {
    if (pool->att_ctr) cudaFree(pool->att_ctr);
    if (pool->err_host) cudaFreeHost(pool->err_host);
    cudaFree(pool->base);
    delete pool;
    return fail(DP_ECUDA, std::string("pool_create: ") + cudaGetErrorString(e));
  }
  *pool->err_host = 0;
  *out = pool;
  return DP_OK;
}

int dp_pool_destroy(dp_pool* pool) {
  if (!pool) return DP_OK;
  {
    DeviceGuard guard(pool->device);
    if (pool->owner && pool->base) cudaFree(pool->base);
    if (pool->ipc_opened && pool->base) cudaIpcCloseMemHandle(pool->base);
    if (pool->err_host) cudaFreeHost(pool->err_host);
    if (pool->owner && pool->att_ctr) cudaFree(pool->att_ctr);
    cudaGetLastError();  // a teardown failure must not surface in the next caller's check
  }
  delete pool;
  return DP_OK;
}

int dp_pool_layout(const dp_pool* pool, int32_t* layout) {
  if (!pool || !layout) return fail(DP_EINVAL, "pool_layout: null argument");
  *layout = pool->layout;
  return DP_OK;
}

int dp_pool_info(const dp_pool* pool, void** base, uint32_t** counters, int64_t* data_bytes) {
  if (!pool) return fail(DP_EINVAL, "pool_info: null pool");
  if (base) *base = pool->base;
  if (counters) *counters = pool->counters;
  if (data_bytes) *data_bytes = pool->data_bytes;
  return DP_OK;
}

int dp_pool_reset_counters(dp_pool* pool, dp_stream stream) {
  if (!pool) return fail(DP_EINVAL, "pool_reset_counters: null pool");
  DeviceGuard guard(pool->device);
  const int64_t ctr_bytes = static_cast<int64_t>(pool->n_tickets) * (pool->geom.n_layer + 1) * 4;
  if (ctr_bytes > 0)
    DP_CUDA(cudaMemsetAsync(pool->counters, 0, ctr_bytes, static_cast<cudaStream_t>(stream)));
  if (pool->err_host) *pool->err_host = 0;
  return DP_OK;
}

int dp_pool_export(const dp_pool* pool, dp_pool_handle* out) {
  if (!pool || !out) return fail(DP_EINVAL, "pool_export: null argument");
  if (!pool->owner) return fail(DP_EINVAL, "pool_export: only the owning pool can be exported");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "unexpected IPC handle size");
  DeviceGuard guard(pool->device);
  cudaIpcMemHandle_t h;
  DP_CUDA(cudaIpcGetMemHandle(&h, pool->base));
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out->ipc, &h, 64);
  out->geom = pool->geom;
  out->n_slots = pool->n_slots;
  out->n_tickets = pool->n_tickets;
  out->device = pool->device;
  out->reserved[0] = pool->layout;
  return DP_OK;
}

int dp_pool_import(int device, const dp_pool_handle* h, dp_pool** out) {
  if (!h || !out) return fail(DP_EINVAL, "pool_import: null argument");
  *out = nullptr;
  if (int rc = dp_geom_check(&h->geom)) return rc;
  if (int rc = preload_kernels(device)) return rc;
  DeviceGuard guard(device);
  cudaIpcMemHandle_t ih;
  std::memcpy(&ih, h->ipc, 64);
  void* ptr = nullptr;
  DP_CUDA(cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess));
  auto* v = new dp_pool;
  v->device = device;
  v->home_device = h->device;
  v->geom = h->geom;
  v->n_slots = h->n_slots;
  v->n_tickets = h->n_tickets;
  v->layout = h->reserved[0];
  v->base = static_cast<char*>(ptr);
  v->data_bytes = static_cast<int64_t>(h->geom.n_layer) * h->n_slots * h->geom.block_tokens *
                  h->geom.bytes_per_token_layer;
  v->counters = reinterpret_cast<uint32_t*>(v->base + counters_offset(v->data_bytes));
  v->ipc_opened = true;
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&v->err_host), sizeof(int),
                                cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaIpcCloseMemHandle(ptr);
    delete v;
    return fail(DP_ECUDA, std::string("pool_import: ") + cudaGetErrorString(e));
  }
  *v->err_host = 0;
  *out = v;
  return DP_OK;
}

int dp_pool_peer_view(int device, const dp_pool* pool, dp_pool** out) {
  if (!pool || !out) return fail(DP_EINVAL, "pool_peer_view: null argument");
  *out = nullptr;
  // A view on the pool's own device is a second, non-owning handle on the same
  // allocation: a PE and a DE engine sharing one GPU (the 1-GPU DE read path)
  // then run the very kernels (K2 / dual / K3, system-scope releases) of the
  // cross-GPU case, their stores landing in local HBM instead of over NVLink.
  if (device != pool->device) {
    int can = 0;
    DP_CUDA(cudaDeviceCanAccessPeer(&can, device, pool->device));
    if (!can) return fail(DP_EINVAL, "pool_peer_view: no P2P path between devices");
  }
  if (int rc = preload_kernels(device)) return rc;
  DeviceGuard guard(device);
  if (device != pool->device) {
    cudaError_t pe = cudaDeviceEnablePeerAccess(pool->device, 0);
    if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
      return fail(DP_ECUDA, std::string("pool_peer_view: ") + cudaGetErrorString(pe));
    cudaGetLastError();
  }
  cudaError_t e = cudaSuccess;
  auto* v = new dp_pool(*pool);
  v->device = device;
  v->owner = false;
  v->ipc_opened = false;
  v->err_host = nullptr;
  v->att_ctr = nullptr;  // owner-only resources stay with the owner
  e = cudaHostAlloc(reinterpret_cast<void**>(&v->err_host), sizeof(int),
                    cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) {
    delete v;
    return fail(DP_ECUDA, std::string("pool_peer_view: ") + cudaGetErrorString(e));
  }
  *v->err_host = 0;
  *out = v;
  return DP_OK;
}

int dp_h2d_layer_gather(dp_pool* pe, const dp_store* src, const dp_job* jobs, int32_t n_jobs,
                        dp_stream stream) {
  return launch_gather(pe, src, jobs, n_jobs, stream, /*peer=*/false);
}

int dp_h2d_push_p2p_layer(dp_pool* pe_view, const dp_store* de_src, const dp_job* jobs,
                          int32_t n_jobs, dp_stream de_stream) {
  return launch_gather(pe_view, de_src, jobs, n_jobs, de_stream, /*peer=*/true);
}

namespace {

using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

WaitValue32Fn wait_value32() {
  static WaitValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WaitValue32Fn>(p);
    cudaGetLastError();
  });
  return fn;
}

// cuStreamWriteValue32 through the runtime's driver entry point (no link
// dependency on libcuda, so the library still loads on a machine without a
// driver; the copy-engine path then fails with DP_ECUDA).
WriteValue32Fn write_value32() {
  static WriteValue32Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<WriteValue32Fn>(p);
    cudaGetLastError();
  });
  return fn;
}

using BatchMemOpFn = CUresult (*)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

BatchMemOpFn batch_memop() {
  static BatchMemOpFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<BatchMemOpFn>(p);
    cudaGetLastError();
  });
  return fn;
}

// Stream-ordered 32-bit writes of (counter, value) pairs: ONE batched
// stream memory operation (cuStreamBatchMemOp) when the driver has it --
// each separate write waits for the copies before it, so L + 1 of them per
// job left the copy engine idle between jobs -- else one write each.
int write_counters(cudaStream_t s, const std::vector<std::pair<uint32_t*, uint32_t>>& writes, const std::string& who) {
  if (writes.empty()) return DP_OK;
  const BatchMemOpFn batch = batch_memop();
  if (batch) {
    constexpr std::size_t kMaxOps = 256;
    for (std::size_t i0 = 0; i0 < writes.size(); i0 += kMaxOps) {
      const std::size_t n = std::min(kMaxOps, writes.size() - i0);
      std::vector<CUstreamBatchMemOpParams> ops(n);
      std::memset(ops.data(), 0, n * sizeof(CUstreamBatchMemOpParams));
      for (std::size_t k = 0; k < n; ++k) {
        ops[k].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
        ops[k].writeValue.address = reinterpret_cast<CUdeviceptr>(writes[i0 + k].first);
        ops[k].writeValue.value = writes[i0 + k].second;
        ops[k].writeValue.flags = 0;
      }
      if (batch(reinterpret_cast<CUstream>(s), static_cast<unsigned int>(n), ops.data(), 0) != CUDA_SUCCESS)
        return fail(DP_ECUDA, who + ": cuStreamBatchMemOp failed");
    }
    return DP_OK;
  }
  const WriteValue32Fn wv = write_value32();
  if (!wv) return fail(DP_ECUDA, who + ": cuStreamWriteValue32 unavailable");
  for (const auto& [ptr, v] : writes)
    if (wv(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(ptr), v, 0) != CUDA_SUCCESS)
      return fail(DP_ECUDA, who + ": cuStreamWriteValue32 failed");
  return DP_OK;
}

}  // namespace

namespace {

// K1 / K2 on the copy engine: one strided copy per contiguous block run per
// layer (Full-Block pitch -> Layer-Block pitch), then fenced stream writes of
// the layer's landed counter and the all-layer column.  With a peer view the
// destination (pool and counters) is the PE's memory over NVLink and the
// stream is the DE's.
int copy_transfer(const char* who, dp_pool* pool, const dp_store* src, const dp_job* jobs, int32_t n_jobs,
                  dp_stream stream, bool peer, bool per_layer = true) {
  const std::string w(who);
  if (!pool || !src || (n_jobs > 0 && !jobs) || n_jobs < 0) return fail(DP_EINVAL, w + ": null argument");
  if (!peer && !pool->owner) return fail(DP_EINVAL, w + ": destination must be the local PE pool");
  if (peer && pool->owner) return fail(DP_EINVAL, w + ": destination must be a peer view of a PE pool");
  if (peer && pool->device != src->device)
    return fail(DP_EINVAL, w + ": the peer view must be mapped on the store's device");
  if (!geom_equal(pool->geom, src->geom)) return fail(DP_EINVAL, w + ": pool and store geometry differ");
  const WriteValue32Fn wv = write_value32();
  if (!wv) return fail(DP_ECUDA, w + ": cuStreamWriteValue32 unavailable");
  const dp_kv_geom& g = pool->geom;
  const int64_t lb = static_cast<int64_t>(g.block_tokens) * g.bytes_per_token_layer;
  const int64_t fbb = lb * g.n_layer;
  const int64_t plane = layer_stride(pool), sstride = slot_stride(pool);
  const int32_t items = static_cast<int32_t>(chunks_per_block(g));
  DeviceGuard guard(pool->device);
  auto s = static_cast<cudaStream_t>(stream);
  // The counter writes are absolute (ctr[l] = items, ctr[L] = items * layers
  // done), not the kernels' increments: a job must start at layer 0 and own
  // its ticket within the call, or a column could go backwards.
  std::vector<int32_t> seen;
  for (int32_t j = 0; j < n_jobs; ++j) {
    const dp_job& job = jobs[j];
    if (job.ticket < 0) continue;
    if (std::find(seen.begin(), seen.end(), job.ticket) != seen.end())
      return fail(DP_EINVAL, w + ": ticket " + std::to_string(job.ticket) + " used by two jobs of one call");
    seen.push_back(job.ticket);
  }
  for (int32_t j = 0; j < n_jobs; ++j) {
    const dp_job& job = jobs[j];
    const int64_t need_blk = (job.n_tokens + g.block_tokens - 1) / g.block_tokens;
    if (job.n_tokens < 0 || job.n_blk != need_blk || job.layer_begin != 0 ||
        job.layer_end > g.n_layer || job.layer_begin > job.layer_end || job.ticket >= pool->n_tickets)
      return fail(DP_EINVAL, w + ": job " + std::to_string(j) + " out of range (copy mode starts at layer 0)");
    if (job.n_blk == 0) continue;
    for (int32_t k = 0; k < job.n_blk; ++k)
      if (job.src_fb[k] < 0 || job.src_fb[k] >= src->n_fb || job.dst_slot[k] < 0 ||
          job.dst_slot[k] >= pool->n_slots)
        return fail(DP_EINVAL, w + ": block " + std::to_string(k) + " out of range");
    const int32_t full = job.n_tokens % g.block_tokens == 0 ? job.n_blk : job.n_blk - 1;
    uint32_t* row = pool->counters + static_cast<int64_t>(job.ticket) * (g.n_layer + 1);
    if (pool->layout == DP_POOL_BLOCK_MAJOR && !per_layer && job.layer_end == g.n_layer) {
      // a block-major pool holds whole Full Blocks: a run of consecutive
      // storage Full Blocks into consecutive slots is ONE contiguous copy
      // (every layer), the partial last block a 2D copy of its L token ranges
      for (int32_t k = 0; k < full;) {
        int32_t run = 1;
        while (k + run < full && job.src_fb[k + run] == job.src_fb[k] + run &&
               job.dst_slot[k + run] == job.dst_slot[k] + run)
          ++run;
        DP_CUDA(cudaMemcpyAsync(pool->base + job.dst_slot[k] * sstride, src->host + job.src_fb[k] * fbb, run * fbb,
                                cudaMemcpyHostToDevice, s));
        k += run;
      }
      if (full < job.n_blk) {
        const int32_t k = full;
        const int64_t bytes = (job.n_tokens - static_cast<int64_t>(k) * g.block_tokens) * g.bytes_per_token_layer;
        DP_CUDA(cudaMemcpy2DAsync(pool->base + job.dst_slot[k] * sstride, lb, src->host + job.src_fb[k] * fbb, lb,
                                  bytes, g.n_layer, cudaMemcpyHostToDevice, s));
      }
    } else {
      for (int32_t layer = job.layer_begin; layer < job.layer_end; ++layer) {
        for (int32_t k = 0; k < full;) {
          int32_t run = 1;
          while (k + run < full && job.src_fb[k + run] == job.src_fb[k] + run &&
                 job.dst_slot[k + run] == job.dst_slot[k] + run)
            ++run;
          DP_CUDA(cudaMemcpy2DAsync(pool->base + layer * plane + job.dst_slot[k] * sstride, sstride,
                                    src->host + job.src_fb[k] * fbb + layer * lb, fbb, lb, run,
                                    cudaMemcpyHostToDevice, s));
          k += run;
        }
        if (full < job.n_blk) {
          const int32_t k = full;
          const int64_t bytes = (job.n_tokens - static_cast<int64_t>(k) * g.block_tokens) * g.bytes_per_token_layer;
          DP_CUDA(cudaMemcpyAsync(pool->base + layer * plane + job.dst_slot[k] * sstride,
                                  src->host + job.src_fb[k] * fbb + layer * lb, bytes,
                                  cudaMemcpyHostToDevice, s));
        }
        if (job.ticket >= 0 && per_layer) {
          const uint32_t n_items = static_cast<uint32_t>(job.n_blk) * items;
          if (wv(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(row + layer), n_items, 0) !=
                  CUDA_SUCCESS ||
              wv(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(row + g.n_layer),
                 n_items * static_cast<uint32_t>(layer - job.layer_begin + 1), 0) != CUDA_SUCCESS)
            return fail(DP_ECUDA, w + ": cuStreamWriteValue32 failed");
        }
      }
    }
    if (job.ticket >= 0 && !per_layer) {
      // one release per job: every layer's counter, then the all-layer column,
      // as one batched memory operation (per-layer writes would idle the copy
      // engine once per layer)
      const uint32_t n_items = static_cast<uint32_t>(job.n_blk) * items;
      std::vector<std::pair<uint32_t*, uint32_t>> writes;
      for (int32_t layer = job.layer_begin; layer <= job.layer_end; ++layer) {
        const bool all = layer == job.layer_end;
        writes.emplace_back(row + (all ? g.n_layer : layer),
                            all ? n_items * static_cast<uint32_t>(job.layer_end - job.layer_begin) : n_items);
      }
      if (int rc = write_counters(s, writes, w)) return rc;
    }
  }
  return DP_OK;
}

}  // namespace

int dp_h2d_layer_copy(dp_pool* pool, const dp_store* src, const dp_job* jobs, int32_t n_jobs,
                      dp_stream stream) {
  return copy_transfer("h2d_layer_copy", pool, src, jobs, n_jobs, stream, /*peer=*/false);
}

int dp_h2d_push_copy(dp_pool* pe_view, const dp_store* de_src, const dp_job* jobs, int32_t n_jobs,
                     dp_stream de_stream) {
  return copy_transfer("h2d_push_copy", pe_view, de_src, jobs, n_jobs, de_stream, /*peer=*/true);
}

int dp_h2d_layer_copy_job(dp_pool* pool, const dp_store* src, const dp_job* jobs, int32_t n_jobs,
                          dp_stream stream) {
  return copy_transfer("h2d_layer_copy_job", pool, src, jobs, n_jobs, stream, /*peer=*/false, /*per_layer=*/false);
}

int dp_h2d_push_copy_job(dp_pool* pe_view, const dp_store* de_src, const dp_job* jobs, int32_t n_jobs,
                         dp_stream de_stream) {
  return copy_transfer("h2d_push_copy_job", pe_view, de_src, jobs, n_jobs, de_stream, /*peer=*/true,
                       /*per_layer=*/false);
}

int dp_stream_wait_counter(const dp_pool* pool, int32_t ticket, int32_t layer, uint32_t target,
                           dp_stream stream) {
  if (!pool) return fail(DP_EINVAL, "stream_wait_counter: null pool");
  if (!pool->owner) return fail(DP_EINVAL, "stream_wait_counter: the pool must be local");
  if (ticket < 0 || ticket >= pool->n_tickets || layer < 0 || layer > pool->geom.n_layer)
    return fail(DP_EINVAL, "stream_wait_counter: ticket/layer out of range");
  const WaitValue32Fn wv = wait_value32();
  if (!wv) return fail(DP_ECUDA, "stream_wait_counter: cuStreamWaitValue32 unavailable");
  DeviceGuard guard(pool->device);
  const uint32_t* ctr =
      pool->counters + static_cast<int64_t>(ticket) * (pool->geom.n_layer + 1) + layer;
  if (wv(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(ctr), target,
         CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    return fail(DP_ECUDA, "stream_wait_counter: cuStreamWaitValue32 failed");
  return DP_OK;
}

int dp_stream_write_counter(dp_pool* pool, int32_t ticket, int32_t layer, uint32_t value,
                            dp_stream stream) {
  if (!pool) return fail(DP_EINVAL, "stream_write_counter: null pool");
  if (!pool->owner) return fail(DP_EINVAL, "stream_write_counter: the pool must be local");
  if (ticket < 0 || ticket >= pool->n_tickets || layer < 0 || layer > pool->geom.n_layer)
    return fail(DP_EINVAL, "stream_write_counter: ticket/layer out of range");
  const WriteValue32Fn wv = write_value32();
  if (!wv) return fail(DP_ECUDA, "stream_write_counter: cuStreamWriteValue32 unavailable");
  DeviceGuard guard(pool->device);
  uint32_t* ctr = pool->counters + static_cast<int64_t>(ticket) * (pool->geom.n_layer + 1) + layer;
  if (wv(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(ctr), value, 0) != CUDA_SUCCESS)
    return fail(DP_ECUDA, "stream_write_counter: cuStreamWriteValue32 failed");
  return DP_OK;
}

int dp_set_handoff_ctas(int device, int32_t ctas) {
  if (device < 0 || device >= kMaxDevices || ctas < 0)
    return fail(DP_EINVAL, "set_handoff_ctas: bad argument");
  g_handoff_ctas[device] = ctas;
  return DP_OK;
}

int dp_set_handoff_tma(int32_t on) {
  g_handoff_tma = on != 0;
  return DP_OK;
}

int dp_set_gather_ctas(int device, int32_t ctas) {
  if (device < 0 || device >= kMaxDevices || ctas < 0)
    return fail(DP_EINVAL, "set_gather_ctas: bad argument");
  g_gather_ctas[device] = ctas;
  return DP_OK;
}

int dp_layer_items(const dp_kv_geom* geom, int32_t n_blk, int32_t* out) {
  if (int rc = dp_geom_check(geom)) return rc;
  if (!out || n_blk < 0) return fail(DP_EINVAL, "layer_items: bad argument");
  *out = static_cast<int32_t>(n_blk * chunks_per_block(*geom));
  return DP_OK;
}

int dp_wait_layer(const dp_pool* pool, int32_t ticket, int32_t layer, uint32_t target,
                  int32_t timeout_ms, dp_stream stream) {
  if (!pool) return fail(DP_EINVAL, "wait_layer: null pool");
  if (ticket < 0 || ticket >= pool->n_tickets || layer < 0 || layer > pool->geom.n_layer)
    return fail(DP_EINVAL, "wait_layer: ticket/layer out of range");
  if (timeout_ms <= 0) return fail(DP_EINVAL, "wait_layer: timeout must be > 0");
  DeviceGuard guard(pool->device);
  const uint32_t* ctr =
      pool->counters + static_cast<int64_t>(ticket) * (pool->geom.n_layer + 1) + layer;
  kv_wait_ge<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      ctr, target, static_cast<uint64_t>(timeout_ms) * 1000000ull, pool->err_host);
  DP_CUDA(cudaGetLastError());
  return DP_OK;
}

int dp_wait_tickets(const dp_pool* pool, const int32_t* tickets, const uint32_t* targets,
                    int32_t n, int32_t layer, int32_t timeout_ms, dp_stream stream) {
  if (!pool || n < 0 || (n > 0 && (!tickets || !targets)))
    return fail(DP_EINVAL, "wait_tickets: bad argument");
  if (layer < 0 || layer > pool->geom.n_layer)
    return fail(DP_EINVAL, "wait_tickets: layer out of range");
  if (timeout_ms <= 0) return fail(DP_EINVAL, "wait_tickets: timeout must be > 0");
  if (n == 0) return DP_OK;
  DeviceGuard guard(pool->device);
  kv_wait_many<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      pool->counters, pool->geom.n_layer + 1, tickets, targets, n, layer,
      static_cast<uint64_t>(timeout_ms) * 1000000ull, pool->err_host);
  DP_CUDA(cudaGetLastError());
  return DP_OK;
}

int dp_wait_status(const dp_pool* pool) {
  if (!pool) return fail(DP_EINVAL, "wait_status: null pool");
  if (pool->err_host && *reinterpret_cast<volatile int*>(pool->err_host))
    return fail(DP_ETIMEOUT, "wait_layer: watchdog fired (producer never released the layer)");
  return DP_OK;
}

int dp_wait_clear(dp_pool* pool) {
  if (!pool) return fail(DP_EINVAL, "wait_clear: null pool");
  if (pool->err_host) *reinterpret_cast<volatile int*>(pool->err_host) = 0;
  return DP_OK;
}

int dp_pool_checksum(const dp_pool* pool, int32_t layer, const int32_t* slots,
                     const int32_t* ntok, int32_t n, uint64_t* out, dp_stream stream) {
  if (!pool || n < 0 || (n > 0 && (!slots || !ntok || !out)))
    return fail(DP_EINVAL, "pool_checksum: bad argument");
  if (layer < 0 || layer >= pool->geom.n_layer)
    return fail(DP_EINVAL, "pool_checksum: layer out of range");
  if (n == 0) return DP_OK;
  DeviceGuard guard(pool->device);
  const int64_t lb = static_cast<int64_t>(pool->geom.block_tokens) * pool->geom.bytes_per_token_layer;
  const int grid = std::min(n, sm_count(pool->device) * 8);
  (void)lb;
  kv_block_checksum<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      pool->base, layer * layer_stride(pool), slot_stride(pool), pool->geom.bytes_per_token_layer, slots, ntok,
      n, out);
  DP_CUDA(cudaGetLastError());
  return DP_OK;
}

int dp_pool_copy_out(const dp_pool* pool, int32_t layer, int32_t slot, int64_t bytes,
                     void* host_out) {
  if (!pool || !host_out || bytes < 0) return fail(DP_EINVAL, "pool_copy_out: bad argument");
  const int64_t lb = static_cast<int64_t>(pool->geom.block_tokens) * pool->geom.bytes_per_token_layer;
  if (layer < 0 || layer >= pool->geom.n_layer || slot < 0 || slot >= pool->n_slots || bytes > lb)
    return fail(DP_EINVAL, "pool_copy_out: out of range");
  DeviceGuard guard(pool->device);
  const char* src = pool->base + layer * layer_stride(pool) + slot * slot_stride(pool);
  DP_CUDA(cudaMemcpy(host_out, src, bytes, cudaMemcpyDeviceToHost));
  return DP_OK;
}

int dp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

}  // extern "C"

// ============================================================= PD handoff
// dp_h2d_push_p2p_dual (the DE read path fused with DecodeH2D) and
// dp_prefill_handoff (K3: prefill stand-in + PeToDe / MissMerge per layer).
namespace {

struct DualParams {
  const char* store;
  char* pe_pool;        // peer
  uint32_t* pe_ctr;
  int64_t pe_stride;    // PE pool layer plane
  char* de_pool;        // local decode pool
  uint32_t* de_ctr;
  int64_t de_stride;
  int64_t lb_bytes, fb_bytes, bpt;
  int32_t n_layer, block_tokens, n_chunk, n_jobs;
  int64_t item_begin[DP_MAX_DUAL_JOBS_PER_LAUNCH + 1];
  dp_dual_job jobs[DP_MAX_DUAL_JOBS_PER_LAUNCH];
};
static_assert(sizeof(DualParams) <= 4000, "kernel parameter block too large");

struct HandoffParams {
  char* pe_pool;        // local
  char* de_pool;        // peer
  uint32_t* pe_ctr;
  uint32_t* de_ctr;
  int64_t pe_stride, de_stride;
  int* err_flag;
  uint64_t timeout_ns;
  uint64_t seed_mix;
  int64_t lb_bytes, bpt;
  int32_t n_layer, block_tokens, n_chunk, n_jobs;
  int64_t item_begin[DP_MAX_HANDOFF_JOBS_PER_LAUNCH + 1];
  dp_handoff_job jobs[DP_MAX_HANDOFF_JOBS_PER_LAUNCH];
};
static_assert(sizeof(HandoffParams) <= 4000, "kernel parameter block too large");
static_assert(sizeof(dp_dual_job) == 56, "dp_dual_job layout");
static_assert(sizeof(dp_handoff_job) == 64, "dp_handoff_job layout");

// Release pattern: ONE system-scope fence (after the CTA barrier, it orders
// every store of the CTA), then relaxed reductions.  The consumers acquire.
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ void add_relaxed_sys(uint32_t* row, int layer, int n_layer, uint32_t n) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(row + layer), "r"(n) : "memory");
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(row + n_layer), "r"(n) : "memory");
}


__global__ void __launch_bounds__(kThreads) kv_gather_dual(const __grid_constant__ DualParams p) {
  const int64_t total = p.item_begin[p.n_jobs];
  const int tid = threadIdx.x;
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
    const int j = decode_job(p, item);
    const dp_dual_job& dj = p.jobs[j];
    const dp_job& job = dj.pe;
    const int64_t local = item - p.item_begin[j];
    const int64_t per_layer = static_cast<int64_t>(job.n_blk) * p.n_chunk;
    const int layer = job.layer_begin + static_cast<int>(local / per_layer);
    const int64_t rem = local % per_layer;
    const int blk = static_cast<int>(rem / p.n_chunk);
    const int chunk = static_cast<int>(rem % p.n_chunk);
    const int64_t tok0 = static_cast<int64_t>(blk) * p.block_tokens;
    const int64_t valid = min(static_cast<int64_t>(p.block_tokens), job.n_tokens - tok0) * p.bpt;
    const int64_t beg = static_cast<int64_t>(chunk) * kChunkBytes;
    const int64_t end = min(beg + kChunkBytes, valid);
    if (end > beg) {
      const uint4* src = reinterpret_cast<const uint4*>(p.store + job.src_fb[blk] * p.fb_bytes +
                                                        layer * p.lb_bytes + beg);
      uint4* d_pe = reinterpret_cast<uint4*>(p.pe_pool + layer * p.pe_stride +
                                             static_cast<int64_t>(job.dst_slot[blk]) * p.lb_bytes + beg);
      uint4* d_de = reinterpret_cast<uint4*>(p.de_pool + layer * p.de_stride +
                                             static_cast<int64_t>(dj.de_slot[blk]) * p.lb_bytes + beg);
      const int n16 = static_cast<int>((end - beg) >> 4);
      for (int base = 0; base < n16; base += kThreads * kUnroll) {
        uint4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int i = base + u * kThreads + tid;
          if (i < n16) v[u] = ld_stream(src + i);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
          const int i = base + u * kThreads + tid;
          if (i < n16) {
            st_v4(d_pe + i, v[u]);
            st_v4(d_de + i, v[u]);
          }
        }
      }
    }
    if (job.ticket >= 0 || dj.de_ticket >= 0) {
      __syncthreads();
      if (tid == 0) {
        fence_sys();
        if (job.ticket >= 0)
          add_relaxed_sys(p.pe_ctr + static_cast<int64_t>(job.ticket) * (p.n_layer + 1), layer, p.n_layer, 1);
        if (dj.de_ticket >= 0)
          add_relaxed_sys(p.de_ctr + static_cast<int64_t>(dj.de_ticket) * (p.n_layer + 1), layer,
                          p.n_layer, 1);
      }
    }
  }
}

// Two consecutive content words of Full Block fb, word index w (even).
__device__ __forceinline__ uint4 content_pair(uint64_t fb, uint64_t w, uint64_t seed_mix) {
  const uint64_t a = splitmix64(((fb << 32) | w) ^ seed_mix);
  const uint64_t b = splitmix64(((fb << 32) | (w + 1)) ^ seed_mix);
  return make_uint4(static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32),
                    static_cast<uint32_t>(b), static_cast<uint32_t>(b >> 32));
}

// K3 work unit: (layer, group of up to kHandoffGroup pieces), a piece being
// one chunk of one prompt block; counters advance by the group's piece count,
// so one system-scope fence covers up to kHandoffGroup * 36 KB of pushes.
constexpr int kHandoffGroup = 4;

// TMA bulk-copy helpers (sm_90+ async proxy): global -> shared completing on
// an mbarrier, shared -> global in bulk groups.
constexpr int kBulkStages = 4;
constexpr int kBulkBytes = 16 * 1024;
constexpr int kHandoffTmaSmem = kBulkStages * kBulkBytes;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// K3's hit push by one thread through the TMA: HBM -> shared -> peer HBM in
// kBulkBytes pieces over kBulkStages buffers; returns once every store has
// completed (the caller's system-scope release then publishes them).
__device__ void tma_push(char* dst, const char* src, int64_t bytes, char* smem, uint64_t* bars, uint32_t& phases) {
  const int64_t n = (bytes + kBulkBytes - 1) / kBulkBytes;
  auto piece = [&](int64_t i) {
    const int64_t left = bytes - i * kBulkBytes;
    return static_cast<uint32_t>(left < kBulkBytes ? left : kBulkBytes);
  };
  for (int64_t i = 0; i <= n; ++i) {
    if (i < n) {
      const int st = static_cast<int>(i % kBulkStages);
      // stores 0 .. i-2 are committed; the buffer's last reader, store
      // i - stages, must be done: at most stages - 2 may still be reading
      if (i >= kBulkStages) bulk_wait_read<kBulkStages - 2>();
      bulk_load(smem + st * kBulkBytes, src + i * kBulkBytes, piece(i), &bars[st]);
    }
    if (i >= 1) {
      const int64_t k = i - 1;
      const int st = static_cast<int>(k % kBulkStages);
      mbar_wait(&bars[st], (phases >> st) & 1u);
      phases ^= 1u << st;
      bulk_store(dst + k * kBulkBytes, smem + st * kBulkBytes, piece(k));
    }
  }
  bulk_wait_all();
}

constexpr int kHoUnroll = 4;  // K3's register-staged copy depth (fits the 40-register cap)

// Items are LAYER-major: item = layer * G + g, g a group of one job's pieces
// (item_begin = prefix sums of the jobs' groups, G their total), so every
// job's layer l is pushed before any job's layer l+1 -- what a gated,
// layerwise handoff of a whole forward's requests needs.  <= 40 registers:
// a K3 CTA beside two K5 CTAs still fits an SM's register file.
template <bool kTma>
__global__ void __launch_bounds__(kThreads, 6) kv_prefill_handoff(const __grid_constant__ HandoffParams p) {
  const int64_t G = p.item_begin[p.n_jobs];
  const int64_t total = G * p.n_layer;
  const int tid = threadIdx.x;
  const int64_t lb = p.lb_bytes;
  extern __shared__ __align__(128) char tma_smem[];
  __shared__ __align__(8) uint64_t tma_bars[kBulkStages];
  uint32_t tma_phases = 0;  // thread 0's parity per stage
  if (kTma) {
    if (tid == 0) {
      for (int st = 0; st < kBulkStages; ++st) mbar_init(&tma_bars[st]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
    const int layer = static_cast<int>(item / G);
    const int64_t gi = item - layer * G;
    const int j = decode_job(p, gi);
    const dp_handoff_job& job = p.jobs[j];
    const int64_t pieces = static_cast<int64_t>(job.n_blk) * p.n_chunk;
    const int64_t piece0 = (gi - p.item_begin[j]) * kHandoffGroup;
    const int64_t piece1 = min(piece0 + kHandoffGroup, pieces);
    // the layer gate: layer l's hit KV must have landed before "computing" l
    if (job.pe_ticket >= 0) {
      if (tid == 0) {
        const uint32_t* ctr = p.pe_ctr + static_cast<int64_t>(job.pe_ticket) * (p.n_layer + 1) + layer;
        const uint64_t t0 = global_timer_ns();
        while (true) {
          uint32_t v;
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
          if (v >= job.pe_wait_items) break;
          if (global_timer_ns() - t0 > p.timeout_ns) {  // watchdog: report, do not hang
            atomicExch_system(p.err_flag, 1);
            break;
          }
          __nanosleep(1024);  // a layer of compute takes tens of microseconds
        }
      }
      __syncthreads();
    }
    for (int64_t piece = piece0; piece < piece1; ++piece) {
      const int blk = static_cast<int>(piece / p.n_chunk);
      const int chunk = static_cast<int>(piece % p.n_chunk);
      const int64_t tok0 = static_cast<int64_t>(blk) * p.block_tokens;
      const int64_t hit_end = max(int64_t{0}, min(lb, (job.n_cached - tok0) * p.bpt));
      const int64_t prompt_end = max(int64_t{0}, min(lb, (job.n_prompt - tok0) * p.bpt));
      const int64_t beg = static_cast<int64_t>(chunk) * kChunkBytes;
      const int64_t end = min(beg + kChunkBytes, prompt_end);
      const int64_t pe_off = layer * p.pe_stride + static_cast<int64_t>(job.pe_slot[blk]) * lb;
      const int64_t de_off = layer * p.de_stride + static_cast<int64_t>(job.de_slot[blk]) * lb;
      // hit part: PeToDe pushes it, MissMerge leaves it to the DE
      const int64_t h1 = min(end, hit_end);
      if (kTma && job.push_hit && h1 > beg) {
        if (tid == 0) tma_push(p.de_pool + de_off + beg, p.pe_pool + pe_off + beg, h1 - beg, tma_smem, tma_bars,
                               tma_phases);
      } else if (job.push_hit && h1 > beg) {
        const uint4* src = reinterpret_cast<const uint4*>(p.pe_pool + pe_off + beg);
        uint4* dst = reinterpret_cast<uint4*>(p.de_pool + de_off + beg);
        const int n16 = static_cast<int>((h1 - beg) >> 4);
        for (int base = 0; base < n16; base += kThreads * kHoUnroll) {
          uint4 v[kHoUnroll];
#pragma unroll
          for (int u = 0; u < kHoUnroll; ++u) {
            const int i = base + u * kThreads + tid;
            if (i < n16) v[u] = __ldcg(src + i);  // landed by another GPU: bypass L1
          }
#pragma unroll
          for (int u = 0; u < kHoUnroll; ++u) {
            const int i = base + u * kThreads + tid;
            if (i < n16) st_v4(dst + i, v[u]);
          }
        }
      }
      // miss part: the prefill stand-in's KV for tokens [C, C+A), written into
      // the PE pool (its KV cache) and pushed to the DE pool
      const int64_t m0 = max(beg, hit_end);
      if (end > m0) {
        const uint64_t fb = static_cast<uint64_t>(job.src_fb[blk]);
        const uint64_t w_base = static_cast<uint64_t>((layer * lb) >> 3);
        uint4* pe_dst = reinterpret_cast<uint4*>(p.pe_pool + pe_off);
        uint4* de_dst = reinterpret_cast<uint4*>(p.de_pool + de_off);
        for (int64_t i = (m0 >> 4) + tid; i < (end >> 4); i += kThreads) {
          const uint4 v = content_pair(fb, w_base + 2 * static_cast<uint64_t>(i), p.seed_mix);
          st_v4(pe_dst + i, v);
          st_v4(de_dst + i, v);
        }
      }
    }
    if (job.de_ticket >= 0 || job.pe_done_ticket >= 0) {
      __syncthreads();
      if (tid == 0) {
        const uint32_t n = static_cast<uint32_t>(piece1 - piece0);
        fence_sys();
        if (job.de_ticket >= 0)
          add_relaxed_sys(p.de_ctr + static_cast<int64_t>(job.de_ticket) * (p.n_layer + 1), layer,
                          p.n_layer, n);
        if (job.pe_done_ticket >= 0)
          add_relaxed_sys(p.pe_ctr + static_cast<int64_t>(job.pe_done_ticket) * (p.n_layer + 1), layer,
                          p.n_layer, n);
      }
    }
  }
}

}  // namespace

extern "C" {

int dp_h2d_push_p2p_dual(dp_pool* pe_view, dp_pool* de_pool, const dp_store* src,
                         const dp_dual_job* jobs, int32_t n_jobs, dp_stream stream) {
  return launch_dual(pe_view, de_pool, src, jobs, n_jobs, stream, 0);
}

}  // extern "C"

namespace {

int launch_dual(dp_pool* pe_view, dp_pool* de_pool, const dp_store* src, const dp_dual_job* jobs, int32_t n_jobs,
                dp_stream stream, int ctas_override) {
  if (!pe_view || !de_pool || !src || (n_jobs > 0 && !jobs) || n_jobs < 0)
    return fail(DP_EINVAL, "push_p2p_dual: null argument");
  if (pe_view->owner) return fail(DP_EINVAL, "push_p2p_dual: PE destination must be a peer view");
  if (!de_pool->owner) return fail(DP_EINVAL, "push_p2p_dual: decode pool must be the local pool");
  if (pe_view->device != de_pool->device)
    return fail(DP_EINVAL, "push_p2p_dual: the PE view must be mapped on the decode pool's device");
  if (pe_view->layout != DP_POOL_LAYER_MAJOR || de_pool->layout != DP_POOL_LAYER_MAJOR)
    return fail(DP_EINVAL, "push_p2p_dual: layer-major pools only");
  if (!geom_equal(pe_view->geom, src->geom) || !geom_equal(de_pool->geom, src->geom))
    return fail(DP_EINVAL, "push_p2p_dual: geometry differs");
  const dp_kv_geom& g = src->geom;
  DeviceGuard guard(de_pool->device);
  DualParams p;
  std::memset(&p, 0, sizeof(p));
  p.store = src->host;
  p.pe_pool = pe_view->base;
  p.pe_ctr = pe_view->counters;
  p.de_pool = de_pool->base;
  p.de_ctr = de_pool->counters;
  p.lb_bytes = static_cast<int64_t>(g.block_tokens) * g.bytes_per_token_layer;
  p.fb_bytes = p.lb_bytes * g.n_layer;
  p.bpt = g.bytes_per_token_layer;
  p.pe_stride = p.lb_bytes * pe_view->n_slots;
  p.de_stride = p.lb_bytes * de_pool->n_slots;
  p.n_layer = g.n_layer;
  p.block_tokens = g.block_tokens;
  p.n_chunk = static_cast<int32_t>(chunks_per_block(g));
  const int dev_cap = de_pool->device < kMaxDevices ? g_gather_ctas[de_pool->device].load() : 0;
  const int grid_cap = ctas_override > 0 ? ctas_override : dev_cap > 0 ? dev_cap : sm_count(de_pool->device) * 4;
  auto s = static_cast<cudaStream_t>(stream);
  for (int32_t j0 = 0; j0 < n_jobs; j0 += DP_MAX_DUAL_JOBS_PER_LAUNCH) {
    const int32_t nj = std::min<int32_t>(DP_MAX_DUAL_JOBS_PER_LAUNCH, n_jobs - j0);
    p.n_jobs = 0;
    int64_t items = 0;
    for (int32_t j = 0; j < nj; ++j) {
      const dp_dual_job& dj = jobs[j0 + j];
      const dp_job& job = dj.pe;
      const int64_t need = (job.n_tokens + g.block_tokens - 1) / g.block_tokens;
      if (job.n_tokens < 0 || job.n_blk != need || job.layer_begin < 0 || job.layer_end > g.n_layer ||
          job.layer_begin > job.layer_end || job.ticket >= pe_view->n_tickets ||
          dj.de_ticket >= de_pool->n_tickets || (job.n_blk > 0 && (!job.src_fb || !job.dst_slot || !dj.de_slot)))
        return fail(DP_EINVAL, "push_p2p_dual: job " + std::to_string(j0 + j) + " out of range");
      const int64_t n = static_cast<int64_t>(job.n_blk) * p.n_chunk * (job.layer_end - job.layer_begin);
      if (n == 0) continue;
      p.jobs[p.n_jobs] = dj;
      p.item_begin[p.n_jobs] = items;
      ++p.n_jobs;
      items += n;
    }
    p.item_begin[p.n_jobs] = items;
    if (items == 0) continue;
    kv_gather_dual<<<static_cast<int>(std::min<int64_t>(items, grid_cap)), kThreads, 0, s>>>(p);
    DP_CUDA(cudaGetLastError());
  }
  return DP_OK;
}

}  // namespace

extern "C" {

int dp_prefill_handoff(dp_pool* pe_pool, dp_pool* de_view, const dp_handoff_job* jobs,
                       int32_t n_jobs, uint64_t seed, int32_t timeout_ms, dp_stream stream) {
  if (!pe_pool || !de_view || (n_jobs > 0 && !jobs) || n_jobs < 0)
    return fail(DP_EINVAL, "prefill_handoff: null argument");
  if (!pe_pool->owner) return fail(DP_EINVAL, "prefill_handoff: the PE pool must be local");
  if (de_view->owner) return fail(DP_EINVAL, "prefill_handoff: the DE pool must be a peer view");
  if (de_view->device != pe_pool->device)
    return fail(DP_EINVAL, "prefill_handoff: the DE view must be mapped on the PE's device");
  if (!geom_equal(pe_pool->geom, de_view->geom)) return fail(DP_EINVAL, "prefill_handoff: geometry differs");
  if (pe_pool->layout != DP_POOL_LAYER_MAJOR || de_view->layout != DP_POOL_LAYER_MAJOR)
    return fail(DP_EINVAL, "prefill_handoff: layer-major pools only");
  if (timeout_ms <= 0) return fail(DP_EINVAL, "prefill_handoff: timeout must be > 0");
  const dp_kv_geom& g = pe_pool->geom;
  DeviceGuard guard(pe_pool->device);
  HandoffParams p;
  std::memset(&p, 0, sizeof(p));
  p.pe_pool = pe_pool->base;
  p.de_pool = de_view->base;
  p.pe_ctr = pe_pool->counters;
  p.de_ctr = de_view->counters;
  p.lb_bytes = static_cast<int64_t>(g.block_tokens) * g.bytes_per_token_layer;
  p.bpt = g.bytes_per_token_layer;
  p.pe_stride = p.lb_bytes * pe_pool->n_slots;
  p.de_stride = p.lb_bytes * de_view->n_slots;
  p.err_flag = pe_pool->err_host;
  p.timeout_ns = static_cast<uint64_t>(timeout_ms) * 1000000ull;
  p.seed_mix = seed * kSeedMul;
  p.n_layer = g.n_layer;
  p.block_tokens = g.block_tokens;
  p.n_chunk = static_cast<int32_t>(chunks_per_block(g));
  const int ho_cap = pe_pool->device < kMaxDevices ? g_handoff_ctas[pe_pool->device].load() : 0;
  const int grid_cap = ho_cap > 0 ? ho_cap : sm_count(pe_pool->device) * 2;  // 699 GB/s NVLink (r01)
  auto s = static_cast<cudaStream_t>(stream);
  for (int32_t j0 = 0; j0 < n_jobs; j0 += DP_MAX_HANDOFF_JOBS_PER_LAUNCH) {
    const int32_t nj = std::min<int32_t>(DP_MAX_HANDOFF_JOBS_PER_LAUNCH, n_jobs - j0);
    p.n_jobs = 0;
    int64_t items = 0;
    for (int32_t j = 0; j < nj; ++j) {
      const dp_handoff_job& job = jobs[j0 + j];
      const int64_t need = (job.n_prompt + g.block_tokens - 1) / g.block_tokens;
      if (job.n_cached < 0 || job.n_prompt < job.n_cached || job.n_blk != need ||
          job.pe_ticket >= pe_pool->n_tickets || job.de_ticket >= de_view->n_tickets ||
          job.pe_done_ticket >= pe_pool->n_tickets ||
          (job.n_blk > 0 && (!job.src_fb || !job.pe_slot || !job.de_slot)))
        return fail(DP_EINVAL, "prefill_handoff: job " + std::to_string(j0 + j) + " out of range");
      const int64_t pieces = static_cast<int64_t>(job.n_blk) * p.n_chunk;
      const int64_t n = (pieces + kHandoffGroup - 1) / kHandoffGroup;  // groups per layer
      if (n == 0) continue;
      p.jobs[p.n_jobs] = job;
      p.item_begin[p.n_jobs] = items;
      ++p.n_jobs;
      items += n;
    }
    p.item_begin[p.n_jobs] = items;
    if (items == 0) continue;
    const int grid = static_cast<int>(std::min<int64_t>(items * g.n_layer, grid_cap));
    if (g_handoff_tma.load())
      kv_prefill_handoff<true><<<grid, kThreads, kHandoffTmaSmem, s>>>(p);
    else
      kv_prefill_handoff<false><<<grid, kThreads, 0, s>>>(p);
    DP_CUDA(cudaGetLastError());
  }
  return DP_OK;
}

}  // extern "C"

// ============================================== K3 on the copy engines
// dp_prefill_handoff_copy: one small kernel per layer (kv_handoff_side)
// releases the previous layer (its copies precede it on the stream), waits
// for this layer's gates and writes the miss tokens' KV into the PE pool;
// then copy-engine copies push the layer's PeToDe / MissMerge bytes from the
// PE pool to the DE pool (whole runs of Layer Blocks consecutive in both).
namespace {

constexpr int kHoMissDescs = 112;  // miss pieces per side-kernel launch (parameter block)
constexpr int kHoSideCtas = 32;

struct HoMissDesc {  // one block's miss tokens: bytes [b0, b1) of its Layer Block
  int64_t fb;
  int32_t pe_slot, de_slot;
  int32_t b0, b1;
};
struct HoGate {
  int32_t ticket;
  uint32_t target;
};
struct HoRelease {
  int32_t de_ticket, pe_done_ticket;
  uint32_t n;  // items per layer
};

struct HoSideParams {
  char* pe_pool;
  char* de_pool;
  uint32_t* pe_ctr;
  uint32_t* de_ctr;
  int64_t pe_stride, de_stride, lb_bytes;
  int* err_flag;
  uint64_t timeout_ns, seed_mix;
  int32_t n_layer;
  int32_t miss_l0, miss_l1;  // layers whose miss KV this launch writes (after the gates)
  int32_t rel_l0, rel_l1;    // layers released first by CTA 0 (work stream-ordered before this launch)
  int32_t n_gate, n_miss, n_rel;
  int32_t miss_to_de;        // gated calls: the miss KV is also stored into the DE pool (no copies of it)
  HoGate gate[DP_MAX_HANDOFF_JOBS_PER_LAUNCH];
  HoRelease rel[DP_MAX_HANDOFF_JOBS_PER_LAUNCH];
  HoMissDesc miss[kHoMissDescs];
};
static_assert(sizeof(HoSideParams) <= 4000, "kernel parameter block too large");

__global__ void __launch_bounds__(kThreads) kv_handoff_side(const __grid_constant__ HoSideParams p) {
  const int tid = threadIdx.x;
  if (blockIdx.x == 0 && tid == 0 && p.n_rel > 0 && p.rel_l1 > p.rel_l0) {
    // everything of layers [rel_l0, rel_l1) -- copies and earlier launches --
    // precedes this kernel on the stream
    fence_sys();
    const uint32_t layers = static_cast<uint32_t>(p.rel_l1 - p.rel_l0);
    for (int r = 0; r < p.n_rel; ++r) {
      const HoRelease& h = p.rel[r];
      for (int l = p.rel_l0; l < p.rel_l1; ++l) {
        if (h.de_ticket >= 0)
          asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(
                           p.de_ctr + static_cast<int64_t>(h.de_ticket) * (p.n_layer + 1) + l),
                       "r"(h.n)
                       : "memory");
        if (h.pe_done_ticket >= 0)
          asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(
                           p.pe_ctr + static_cast<int64_t>(h.pe_done_ticket) * (p.n_layer + 1) + l),
                       "r"(h.n)
                       : "memory");
      }
      if (h.de_ticket >= 0)
        asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(
                         p.de_ctr + static_cast<int64_t>(h.de_ticket) * (p.n_layer + 1) + p.n_layer),
                     "r"(h.n * layers)
                     : "memory");
      if (h.pe_done_ticket >= 0)
        asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(
                         p.pe_ctr + static_cast<int64_t>(h.pe_done_ticket) * (p.n_layer + 1) + p.n_layer),
                     "r"(h.n * layers)
                     : "memory");
    }
  }
  if (p.miss_l1 <= p.miss_l0) return;
  // the gates of the miss layers (the maybe_start_compute gate of each job)
  if (p.n_gate > 0) {
    if (tid == 0) {
      const uint64_t t0 = global_timer_ns();
      for (int gi = 0; gi < p.n_gate; ++gi)
        for (int l = p.miss_l0; l < p.miss_l1; ++l) {
          const uint32_t* ctr = p.pe_ctr + static_cast<int64_t>(p.gate[gi].ticket) * (p.n_layer + 1) + l;
          while (true) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= p.gate[gi].target) break;
            if (global_timer_ns() - t0 > p.timeout_ns) {
              atomicExch_system(p.err_flag, 1);
              break;
            }
            __nanosleep(1024);
          }
        }
    }
    __syncthreads();
  }
  // miss KV: the prefill stand-in's content for the miss tokens, into the PE
  // pool (its KV cache, local HBM); the copies that follow push it to the DE
  // (gated calls store it into the DE pool here as well)
  const int64_t lb = p.lb_bytes;
  const int64_t per_layer = p.n_miss;
  const int64_t total = per_layer * (p.miss_l1 - p.miss_l0);
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
    const int layer = p.miss_l0 + static_cast<int>(item / per_layer);
    const HoMissDesc& d = p.miss[item % per_layer];
    const uint64_t w_base = static_cast<uint64_t>((layer * lb) >> 3);
    uint4* pe_dst = reinterpret_cast<uint4*>(p.pe_pool + layer * p.pe_stride + static_cast<int64_t>(d.pe_slot) * lb);
    uint4* de_dst = reinterpret_cast<uint4*>(p.de_pool + layer * p.de_stride + static_cast<int64_t>(d.de_slot) * lb);
    for (int64_t i = (d.b0 >> 4) + tid; i < (d.b1 >> 4); i += kThreads) {
      const uint4 v = content_pair(static_cast<uint64_t>(d.fb), w_base + 2 * static_cast<uint64_t>(i), p.seed_mix);
      st_v4(pe_dst + i, v);
      if (p.miss_to_de) st_v4(de_dst + i, v);
    }
  }
}

// Launches kv_handoff_side: releases of layers [r0, r1) (CTA 0, first),
// then -- with `gate` -- the jobs' gates at layers [l0, l1), then the miss KV
// of layers [l0, l1), the descriptors split over as many launches as the
// parameter block needs (the releases and gates ride on the first).
int launch_side(HoSideParams& p, const std::vector<HoMissDesc>& miss, int l0, int l1, int r0, int r1, bool gate,
                cudaStream_t s, int64_t* launches, int max_ctas = kHoSideCtas) {
  const int32_t n_rel = p.n_rel, n_gate = p.n_gate;
  if (!gate) p.n_gate = 0;
  p.miss_l0 = l0;
  p.miss_l1 = l1;
  p.rel_l0 = r0;
  p.rel_l1 = r1;
  std::size_t i = 0;
  bool first = true;
  while (first || i < miss.size()) {
    const std::size_t n = std::min<std::size_t>(kHoMissDescs, miss.size() - i);
    p.n_miss = static_cast<int32_t>(n);
    for (std::size_t k = 0; k < n; ++k) p.miss[k] = miss[i + k];
    const bool work = (p.n_rel > 0 && r1 > r0) || (l1 > l0 && (p.n_gate > 0 || n > 0));
    if (work) {
      const int64_t units = static_cast<int64_t>(n) * std::max(0, l1 - l0);
      const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(units, max_ctas)));
      kv_handoff_side<<<grid, kThreads, 0, s>>>(p);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        p.n_rel = n_rel;
        p.n_gate = n_gate;
        return fail(DP_ECUDA, std::string("kv_handoff_side: ") + cudaGetErrorString(e));
      }
      ++*launches;
    }
    p.n_rel = 0;  // released / gated once: later launches are stream-ordered after it
    p.n_gate = 0;
    first = false;
    i += n;
  }
  p.n_rel = n_rel;
  p.n_gate = n_gate;
  return DP_OK;
}

std::atomic<int64_t> g_handoff_copy_launches{0};  // side kernels, process-wide
std::atomic<bool> g_handoff_gate_memop{false};     // dp_set_handoff_gate_memop

}  // namespace

extern "C" {

int dp_prefill_handoff_copy(dp_pool* pe_pool, dp_pool* de_view, const dp_handoff_job* jobs, int32_t n_jobs,
                            uint64_t seed, int32_t timeout_ms, dp_stream stream) {
  if (!pe_pool || !de_view || (n_jobs > 0 && !jobs) || n_jobs < 0)
    return fail(DP_EINVAL, "prefill_handoff_copy: null argument");
  if (!pe_pool->owner) return fail(DP_EINVAL, "prefill_handoff_copy: the PE pool must be local");
  if (de_view->owner) return fail(DP_EINVAL, "prefill_handoff_copy: the DE pool must be a peer view");
  if (de_view->device != pe_pool->device)
    return fail(DP_EINVAL, "prefill_handoff_copy: the DE view must be mapped on the PE's device");
  if (!geom_equal(pe_pool->geom, de_view->geom))
    return fail(DP_EINVAL, "prefill_handoff_copy: geometry differs");
  if (pe_pool->layout != DP_POOL_LAYER_MAJOR || de_view->layout != DP_POOL_LAYER_MAJOR)
    return fail(DP_EINVAL, "prefill_handoff_copy: layer-major pools only");
  if (timeout_ms <= 0) return fail(DP_EINVAL, "prefill_handoff_copy: timeout must be > 0");
  if (n_jobs > DP_MAX_HANDOFF_JOBS_PER_LAUNCH) {  // in groups of the parameter block's job capacity
    for (int32_t j0 = 0; j0 < n_jobs; j0 += DP_MAX_HANDOFF_JOBS_PER_LAUNCH)
      if (int rc = dp_prefill_handoff_copy(pe_pool, de_view, jobs + j0,
                                           std::min<int32_t>(DP_MAX_HANDOFF_JOBS_PER_LAUNCH, n_jobs - j0), seed,
                                           timeout_ms, stream))
        return rc;
    return DP_OK;
  }
  const dp_kv_geom& g = pe_pool->geom;
  const int L = g.n_layer;
  const int64_t T = g.block_tokens, bpt = g.bytes_per_token_layer, lb = T * bpt;
  const int64_t pe_plane = lb * pe_pool->n_slots, de_plane = lb * de_view->n_slots;
  const uint32_t items = static_cast<uint32_t>(chunks_per_block(g));
  DeviceGuard guard(pe_pool->device);
  auto s = static_cast<cudaStream_t>(stream);
  HoSideParams p;
  std::memset(&p, 0, sizeof(p));
  p.pe_pool = pe_pool->base;
  p.de_pool = de_view->base;
  p.pe_ctr = pe_pool->counters;
  p.de_ctr = de_view->counters;
  p.pe_stride = pe_plane;
  p.de_stride = de_plane;
  p.lb_bytes = lb;
  p.err_flag = pe_pool->err_host;
  p.timeout_ns = static_cast<uint64_t>(timeout_ms) * 1000000ull;
  p.seed_mix = seed * kSeedMul;
  p.n_layer = L;
  // per job: the hit runs to copy, the miss pieces, the gate and the release
  struct Run {
    int64_t pe_off, de_off, bytes;  // within a layer plane
  };
  std::vector<Run> runs;
  std::vector<HoMissDesc> miss;
  bool gated_call = false;  // any gate: the per-layer path
  for (int32_t j = 0; j < n_jobs; ++j) gated_call = gated_call || jobs[j].pe_ticket >= 0;
  p.miss_to_de = gated_call ? 1 : 0;
  for (int32_t j = 0; j < n_jobs; ++j) {
    const dp_handoff_job& job = jobs[j];
    const int64_t need = (job.n_prompt + T - 1) / T;
    if (job.n_cached < 0 || job.n_prompt < job.n_cached || job.n_blk != need ||
        job.pe_ticket >= pe_pool->n_tickets || job.de_ticket >= de_view->n_tickets ||
        job.pe_done_ticket >= pe_pool->n_tickets || (job.n_blk > 0 && (!job.src_fb || !job.pe_slot || !job.de_slot)))
      return fail(DP_EINVAL, "prefill_handoff_copy: job " + std::to_string(j) + " out of range");
    for (int32_t k = 0; k < job.n_blk; ++k)
      if (job.pe_slot[k] < 0 || job.pe_slot[k] >= pe_pool->n_slots || job.de_slot[k] < 0 ||
          job.de_slot[k] >= de_view->n_slots)
        return fail(DP_EINVAL, "prefill_handoff_copy: job " + std::to_string(j) + " block " +
                                   std::to_string(k) + " slot out of range");
    if (job.n_blk == 0) continue;
    // the copied tokens: the whole prompt [0, C + A) on the PE path
    // (PeToDe), the miss tokens [C, C + A) on the DE path (MissMerge), from
    // the PE pool once the side kernel has written the miss KV there; runs of
    // blocks consecutive in both pools, only the range's first and last
    // blocks partial.  Gated calls copy only the hit part [0, C) of the PE
    // path, per layer, and the side kernel stores the miss KV into both
    // pools: a few operations per layer (a long chain of copies queued behind
    // a gate can block the enqueueing thread until the queue drains, and so
    // deadlock a caller that enqueues the gate's producer after this call)
    const int64_t push0 = job.push_hit ? 0 : job.n_cached;
    const int64_t push1 = gated_call ? (job.push_hit ? job.n_cached : 0) : job.n_prompt;
    const int32_t blk1 = static_cast<int32_t>((push1 + T - 1) / T);
    for (int64_t k = push0 / T; k < blk1 && push1 > push0;) {
      int32_t run = 1;
      while (k + run < blk1 && job.pe_slot[k + run] == job.pe_slot[k] + run &&
             job.de_slot[k + run] == job.de_slot[k] + run)
        ++run;
      const int64_t last = k + run - 1;
      const int64_t head = std::max<int64_t>(0, push0 - k * T) * bpt;
      const int64_t tail = std::min<int64_t>(T, push1 - last * T) * bpt;
      const int64_t bytes = (run - 1) * lb + tail - head;
      if (bytes > 0) runs.push_back({job.pe_slot[k] * lb + head, job.de_slot[k] * lb + head, bytes});
      k += run;
    }
    // miss part: tokens [C, C + A) block by block
    for (int64_t k = job.n_cached / T; k < job.n_blk; ++k) {
      const int64_t b0 = std::max<int64_t>(0, job.n_cached - k * T) * bpt;
      const int64_t b1 = std::min<int64_t>(T, job.n_prompt - k * T) * bpt;
      if (b1 > b0)
        miss.push_back({job.src_fb[k], job.pe_slot[k], job.de_slot[k], static_cast<int32_t>(b0),
                        static_cast<int32_t>(b1)});
    }
    if (job.pe_ticket >= 0) {
      bool dup = false;
      for (int gi = 0; gi < p.n_gate; ++gi)
        if (p.gate[gi].ticket == job.pe_ticket) {
          p.gate[gi].target = std::max(p.gate[gi].target, job.pe_wait_items);
          dup = true;
        }
      if (!dup) p.gate[p.n_gate++] = {job.pe_ticket, job.pe_wait_items};
    }
    if (job.de_ticket >= 0 || job.pe_done_ticket >= 0)
      p.rel[p.n_rel++] = {job.de_ticket, job.pe_done_ticket, static_cast<uint32_t>(job.n_blk) * items};
  }
  int64_t launches = 0;
  if (p.n_gate == 0) {
    // no gates: the miss KV of every layer (a full-width side kernel), then
    // one 2D copy per run (rows = layers), then the releases of every layer.
    // All on `stream`: a helper stream overlapping the miss writes with the
    // copies gained ~0.5 % alone but deadlocked engines sharing a GPU (its
    // kernel queued behind another engine's spin-wait in one hardware queue)
    if (!miss.empty())
      if (int rc = launch_side(p, miss, 0, L, 0, 0, false, s, &launches, 2 * sm_count(pe_pool->device))) return rc;
    for (const Run& r : runs)
      DP_CUDA(cudaMemcpy2DAsync(de_view->base + r.de_off, de_plane, pe_pool->base + r.pe_off, pe_plane, r.bytes,
                                L, cudaMemcpyDeviceToDevice, s));
    if (int rc = launch_side(p, {}, 0, 0, 0, L, false, s, &launches)) return rc;
  } else {
    // layer by layer: side(l) = release of l - 1, the gates of l, the miss
    // KV of l; then l's copies.  With dp_set_handoff_gate_memop the gates are
    // stream waits (cuStreamWaitValue32, no SM) and side(l) does not spin
    const bool memop = g_handoff_gate_memop.load();
    const WaitValue32Fn wait = memop ? wait_value32() : nullptr;
    if (memop && !wait) return fail(DP_ECUDA, "prefill_handoff_copy: cuStreamWaitValue32 unavailable");
    for (int l = 0; l < L; ++l) {
      for (int gi = 0; memop && gi < p.n_gate; ++gi) {
        const uint32_t* ctr = pe_pool->counters + static_cast<int64_t>(p.gate[gi].ticket) * (L + 1) + l;
        if (wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(ctr), p.gate[gi].target,
                 CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
          return fail(DP_ECUDA, "prefill_handoff_copy: cuStreamWaitValue32 failed");
      }
      if (int rc = launch_side(p, miss, l, l + 1, l > 0 ? l - 1 : 0, l, !memop, s, &launches)) return rc;
      for (const Run& r : runs)
        DP_CUDA(cudaMemcpyAsync(de_view->base + l * de_plane + r.de_off, pe_pool->base + l * pe_plane + r.pe_off,
                                r.bytes, cudaMemcpyDeviceToDevice, s));
    }
    if (int rc = launch_side(p, {}, 0, 0, L - 1, L, false, s, &launches)) return rc;
  }
  g_handoff_copy_launches += launches;
  return DP_OK;
}

int dp_set_handoff_gate_memop(int32_t on) {
  g_handoff_gate_memop = on != 0;
  return DP_OK;
}

int dp_handoff_copy_launches(int64_t* n) {
  if (!n) return fail(DP_EINVAL, "handoff_copy_launches: null argument");
  *n = g_handoff_copy_launches.load();
  return DP_OK;
}

}  // extern "C"

// ============================================================ persistence
// dp_decode_fill (decode stand-in) and dp_persist_d2h (K4, PersistD2H).
namespace {

struct SpanParams {
  char* pool;
  char* host;            // K4: target Full Blocks (device-visible host pointer)
  int64_t pool_stride;   // layer plane
  int64_t lb_bytes, fb_bytes, bpt;
  uint64_t seed_mix;
  int32_t n_layer, block_tokens, n_chunk, n_jobs;
  int64_t item_begin[DP_MAX_SPAN_JOBS_PER_LAUNCH + 1];
  dp_span_job jobs[DP_MAX_SPAN_JOBS_PER_LAUNCH];
};
static_assert(sizeof(SpanParams) <= 4000, "kernel parameter block too large");
static_assert(sizeof(dp_span_job) == 48, "dp_span_job layout");

// item -> (job, block i, layer, chunk) and the byte range of the span inside
// that Layer Block; false when the chunk holds none of the span.
struct SpanItem {
  int j, i, layer;
  int64_t beg, end;  // bytes within the Layer Block
};

__device__ __forceinline__ bool span_item(const SpanParams& p, int64_t item, SpanItem& it) {
  it.j = decode_job(p, item);
  const dp_span_job& job = p.jobs[it.j];
  const int64_t local = item - p.item_begin[it.j];
  const int64_t per_block = static_cast<int64_t>(p.n_layer) * p.n_chunk;
  it.i = static_cast<int>(local / per_block);
  const int64_t rem = local % per_block;
  it.layer = static_cast<int>(rem / p.n_chunk);
  const int chunk = static_cast<int>(rem % p.n_chunk);
  const int64_t blk_tok0 = (job.blk0 + it.i) * p.block_tokens;
  const int64_t t0 = max(job.tok_begin, blk_tok0) - blk_tok0;
  const int64_t t1 = min(job.tok_end, blk_tok0 + p.block_tokens) - blk_tok0;
  it.beg = max(t0 * p.bpt, static_cast<int64_t>(chunk) * kChunkBytes);
  it.end = min(t1 * p.bpt, static_cast<int64_t>(chunk + 1) * kChunkBytes);
  return it.end > it.beg;
}

__global__ void __launch_bounds__(kThreads) kv_decode_fill(const __grid_constant__ SpanParams p) {
  const int64_t total = p.item_begin[p.n_jobs];
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
    SpanItem it;
    if (!span_item(p, item, it)) continue;
    const dp_span_job& job = p.jobs[it.j];
    uint4* dst = reinterpret_cast<uint4*>(p.pool + it.layer * p.pool_stride +
                                          static_cast<int64_t>(job.slot[it.i]) * p.lb_bytes);
    const uint64_t fb = static_cast<uint64_t>(job.fb[it.i]);
    const uint64_t w_base = static_cast<uint64_t>((it.layer * p.lb_bytes) >> 3);
    for (int64_t v = (it.beg >> 4) + threadIdx.x; v < (it.end >> 4); v += kThreads)
      st_v4(dst + v, content_pair(fb, w_base + 2 * static_cast<uint64_t>(v), p.seed_mix));
  }
}

__global__ void __launch_bounds__(kThreads) kv_persist_d2h(const __grid_constant__ SpanParams p) {
  const int64_t total = p.item_begin[p.n_jobs];
  const int tid = threadIdx.x;
  for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
    SpanItem it;
    if (!span_item(p, item, it)) continue;
    const dp_span_job& job = p.jobs[it.j];
    const uint4* src = reinterpret_cast<const uint4*>(p.pool + it.layer * p.pool_stride +
                                                      static_cast<int64_t>(job.slot[it.i]) * p.lb_bytes + it.beg);
    uint4* dst = reinterpret_cast<uint4*>(p.host + job.fb[it.i] * p.fb_bytes + it.layer * p.lb_bytes + it.beg);
    const int n16 = static_cast<int>((it.end - it.beg) >> 4);
    for (int base = 0; base < n16; base += kThreads * kUnroll) {
      uint4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int i = base + u * kThreads + tid;
        if (i < n16) v[u] = __ldcg(src + i);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int i = base + u * kThreads + tid;
        if (i < n16) st_v4(dst + i, v[u]);
      }
    }
  }
}

template <class Kernel>
int launch_span(const dp_pool* pool, const dp_store* target, const dp_span_job* jobs, int32_t n_jobs,
                uint64_t seed, dp_stream stream, Kernel kernel, const char* what) {
  if (!pool || (n_jobs > 0 && !jobs) || n_jobs < 0) return fail(DP_EINVAL, std::string(what) + ": bad argument");
  if (!pool->owner) return fail(DP_EINVAL, std::string(what) + ": the decode pool must be local");
  if (pool->layout != DP_POOL_LAYER_MAJOR) return fail(DP_EINVAL, std::string(what) + ": layer-major pools only");
  if (target && !geom_equal(pool->geom, target->geom))
    return fail(DP_EINVAL, std::string(what) + ": geometry differs");
  const dp_kv_geom& g = pool->geom;
  DeviceGuard guard(pool->device);
  SpanParams p;
  std::memset(&p, 0, sizeof(p));
  p.pool = pool->base;
  p.host = target ? target->host : nullptr;
  p.lb_bytes = static_cast<int64_t>(g.block_tokens) * g.bytes_per_token_layer;
  p.fb_bytes = p.lb_bytes * g.n_layer;
  p.bpt = g.bytes_per_token_layer;
  p.pool_stride = p.lb_bytes * pool->n_slots;
  p.seed_mix = seed * kSeedMul;
  p.n_layer = g.n_layer;
  p.block_tokens = g.block_tokens;
  p.n_chunk = static_cast<int32_t>(chunks_per_block(g));
  auto s = static_cast<cudaStream_t>(stream);
  const int grid_cap = sm_count(pool->device) * 4;
  for (int32_t j0 = 0; j0 < n_jobs; j0 += DP_MAX_SPAN_JOBS_PER_LAUNCH) {
    const int32_t nj = std::min<int32_t>(DP_MAX_SPAN_JOBS_PER_LAUNCH, n_jobs - j0);
    p.n_jobs = 0;
    int64_t items = 0;
    for (int32_t j = 0; j < nj; ++j) {
      const dp_span_job& job = jobs[j0 + j];
      const int64_t T = g.block_tokens;
      if (job.n_blk < 0 || job.blk0 < 0 || job.tok_begin < job.blk0 * T || job.tok_end < job.tok_begin ||
          job.tok_end > (job.blk0 + job.n_blk) * T || (job.n_blk > 0 && (!job.slot || !job.fb)))
        return fail(DP_EINVAL, std::string(what) + ": job " + std::to_string(j0 + j) + " out of range");
      const int64_t n = static_cast<int64_t>(job.n_blk) * g.n_layer * p.n_chunk;
      if (n == 0 || job.tok_end == job.tok_begin) continue;
      p.jobs[p.n_jobs] = job;
      p.item_begin[p.n_jobs] = items;
      ++p.n_jobs;
      items += n;
    }
    p.item_begin[p.n_jobs] = items;
    if (items == 0) continue;
    kernel<<<static_cast<int>(std::min<int64_t>(items, grid_cap)), kThreads, 0, s>>>(p);
    DP_CUDA(cudaGetLastError());
  }
  return DP_OK;
}

}  // namespace

extern "C" {

int dp_decode_fill(dp_pool* de_pool, const dp_span_job* jobs, int32_t n_jobs, uint64_t seed,
                   dp_stream stream) {
  return launch_span(de_pool, nullptr, jobs, n_jobs, seed, stream, kv_decode_fill, "decode_fill");
}

int dp_persist_d2h(const dp_pool* de_pool, dp_store* target, const dp_span_job* jobs, int32_t n_jobs,
                   dp_stream stream) {
  if (!target) return fail(DP_EINVAL, "persist_d2h: null target");
  // (the block arrays are device memory: their contents are not checked here)
  return launch_span(de_pool, target, jobs, n_jobs, 0, stream, kv_persist_d2h, "persist_d2h");
}

}  // extern "C"

// ============================================================ prefill stand-in
// K5 dp_prefill_attend: the attention-score pass of one prefill layer over
// the KV the loader landed.  Work unit = (item, 64-query
// tile, group of kAttGroup 64-token key tiles).  A CTA stages the query tile
// (procedural) and each key tile (from the pool, 16-byte loads) in shared
// memory, row stride 37 x 16 B so the per-lane LDS.128 of 8 distinct rows is
// bank-conflict free, and each thread accumulates a 4 x 4 block of
// (query, key) dot products with dp4a.  Integer sums are order-independent,
// so the digest is exact whatever the grid.
namespace {

constexpr int kAttRows = 64;     // query rows and key rows per tile
constexpr int kAttWords = 144;   // 32-bit words per staged row chunk (576 B)
constexpr int kAttStride = 148;  // padded row stride in words
constexpr int kAttGroup = 4;     // key tiles per unit
constexpr int kAttSmem = 3 * kAttRows * kAttStride * 4;  // query tile + 2 key tiles: 113,664 B
constexpr uint64_t kQueryMul = 0xA24BAED4963EE407ull;
std::atomic<int> g_attend_ctas[kMaxDevices] = {};
bool g_attend_init[kMaxDevices] = {};
std::mutex g_attend_mu;

struct AttendParams {
  const char* pool;
  uint32_t* ctr;  // {next unit, CTAs done}: zero at launch, zeroed again by the last CTA
  uint32_t* done; // or null: set to 1 by the last CTA out (the layer's "computed" flag)
  int64_t bpt;
  int64_t lb_bytes;
  int64_t layer_off;    // layer * the pool's layer stride
  int64_t slot_stride;  // the pool's slot stride (Layer Block or Full Block)
  uint64_t seed_q;
  int32_t layer;
  int32_t block_tokens;
  int32_t words;  // b / 4
  int32_t n_jobs;
  int64_t item_begin[DP_MAX_ATTEND_ITEMS_PER_LAUNCH + 1];
  dp_attend_item jobs[DP_MAX_ATTEND_ITEMS_PER_LAUNCH];
};
static_assert(sizeof(AttendParams) <= 4000, "kernel parameter block too large");
static_assert(sizeof(dp_attend_item) == 48, "dp_attend_item layout");

// 16-byte asynchronous global -> shared copy; src_size 0 zero-fills.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ int64_t attend_key_tiles(int64_t cached) {
  return (cached + kAttRows - 1) / kAttRows;
}

// <= 96 registers: the two K5 CTAs a default grid puts on
// an SM leave room for a loader CTA (K1) beside them.
__global__ void __maxnreg__(96) kv_prefill_attend(const __grid_constant__ AttendParams p) {
  extern __shared__ uint4 att_smem[];
  __shared__ uint64_t red[kThreads / 32];
  uint32_t* qs = reinterpret_cast<uint32_t*>(att_smem);
  uint32_t* const kbuf0 = qs + kAttRows * kAttStride;  // key tiles: kbuf0 + (i & 1) * tile
  constexpr int kTile = kAttRows * kAttStride;
  const int tid = threadIdx.x;
  const int tq = tid >> 4, tt = tid & 15;
  __shared__ int64_t fetched;
  const int64_t total = p.item_begin[p.n_jobs];
  // units are handed out by an atomic counter: an SM slowed by a neighbour
  // (a loader CTA) takes fewer, so no straggler holds the layer back
  for (;;) {
    __syncthreads();  // every thread has read the previous `fetched`
    if (tid == 0) fetched = atomicAdd(p.ctr, 1u);
    __syncthreads();
    const int64_t unit = fetched;
    if (unit >= total) break;
    const int j = decode_job(p, unit);
    const dp_attend_item& it = p.jobs[j];
    const int64_t local = unit - p.item_begin[j];
    const int64_t n_kt = attend_key_tiles(it.cached);
    const int64_t ng = (n_kt + kAttGroup - 1) / kAttGroup;
    const int64_t q0 = (local / ng) * kAttRows;
    const int64_t kt0 = (local % ng) * kAttGroup;
    const int64_t kt1 = min(n_kt, kt0 + kAttGroup);
    const int nq = static_cast<int>(min(static_cast<int64_t>(kAttRows), it.bsz - q0));
    const uint64_t qbase =
        splitmix64(((static_cast<uint64_t>(it.req) << 20) | static_cast<uint64_t>(p.layer)) ^ p.seed_q);
    uint64_t sum = 0;
    for (int c0 = 0; c0 < p.words; c0 += kAttWords) {
      const int cw = min(kAttWords, p.words - c0);  // a multiple of 4 (b % 16 == 0)
      const int half = cw / 2;
      const int vec = cw / 4;
      // key tile kt -> kbuf[b], asynchronously (rows past `cached` zero-filled)
      auto issue_tile = [&](int64_t kt, uint32_t* dst) {
        for (int e = tid; e < kAttRows * vec; e += kThreads) {
          const int r = e / vec, v4 = e - (e / vec) * vec;
          const int64_t t = kt * kAttRows + r;
          const bool valid = t < it.cached;
          const char* src = p.pool;
          if (valid) {
            const int64_t blk = t / p.block_tokens;
            src = p.pool + p.layer_off + static_cast<int64_t>(it.slot[blk]) * p.slot_stride +
                  (t - blk * p.block_tokens) * p.bpt + static_cast<int64_t>(c0) * 4 + v4 * 16;
          }
          cp_async16(dst + r * kAttStride + v4 * 4, src, valid);
        }
        cp_async_commit();
      };
      __syncthreads();  // the previous chunk's readers are done with qs / kbuf
      issue_tile(kt0, kbuf0);  // in flight while the query tile is generated
      for (int e = tid; e < kAttRows * half; e += kThreads) {
        const int r = e / half, k = e - (e / half) * half;
        uint64_t v = 0;
        if (r < nq) {
          const uint64_t qpos = static_cast<uint64_t>(it.q_begin + q0 + r);
          v = splitmix64(qbase ^ ((qpos << 16) | static_cast<uint64_t>(c0 / 2 + k)));
        }
        *reinterpret_cast<uint64_t*>(qs + r * kAttStride + 2 * k) = v;
      }
      for (int64_t kt = kt0; kt < kt1; ++kt) {
        const uint32_t* ks = kbuf0 + ((kt - kt0) & 1) * kTile;
        if (kt + 1 < kt1) {  // double buffer: the next tile loads during this one's math
          issue_tile(kt + 1, kbuf0 + ((kt + 1 - kt0) & 1) * kTile);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();  // tile kt (every thread's copies) and the query tile are visible
        uint32_t acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = 0;
#pragma unroll 1
        for (int k = 0; k < cw; k += 4) {
          uint4 qa[4], kb[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) qa[a] = *reinterpret_cast<const uint4*>(qs + (tq + 16 * a) * kAttStride + k);
#pragma unroll
          for (int b = 0; b < 4; ++b) kb[b] = *reinterpret_cast<const uint4*>(ks + (tt + 16 * b) * kAttStride + k);
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              acc[a][b] = __dp4a(qa[a].x, kb[b].x, acc[a][b]);
              acc[a][b] = __dp4a(qa[a].y, kb[b].y, acc[a][b]);
              acc[a][b] = __dp4a(qa[a].z, kb[b].z, acc[a][b]);
              acc[a][b] = __dp4a(qa[a].w, kb[b].w, acc[a][b]);
            }
        }
        // each acc <= 144 * 4 * 255^2 < 2^26, so the 16 fit a 32-bit sum
        uint32_t s32 = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) s32 += acc[a][b];
        sum += s32;
        __syncthreads();  // every reader is done with this buffer before it is refilled
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
    if ((tid & 31) == 0) red[tid >> 5] = sum;
    __syncthreads();
    if (tid == 0) {
      uint64_t all = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) all += red[w];
      atomicAdd(reinterpret_cast<unsigned long long*>(it.digest + p.layer),
                static_cast<unsigned long long>(all));
    }
  }
  if (tid == 0 && atomicAdd(p.ctr + 1, 1u) == gridDim.x - 1) {  // the last CTA out resets
    p.ctr[0] = 0;
    p.ctr[1] = 0;
    if (p.done) {  // every unit of the layer is done: release its flag
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.done), "r"(1u) : "memory");
    }
  }
}

}  // namespace

extern "C" {

int dp_set_attend_ctas(int device, int32_t ctas) {
  if (device < 0 || device >= kMaxDevices || ctas < 0) return fail(DP_EINVAL, "set_attend_ctas: bad argument");
  g_attend_ctas[device] = ctas;
  return DP_OK;
}

int dp_prefill_attend(const dp_pool* pool, int32_t layer, const dp_attend_item* items, int32_t n_items,
                      uint64_t seed, dp_stream stream) {
  return dp_prefill_attend_signal(pool, layer, items, n_items, seed, nullptr, stream);
}

int dp_prefill_attend_signal(const dp_pool* pool, int32_t layer, const dp_attend_item* items, int32_t n_items,
                             uint64_t seed, uint32_t* done, dp_stream stream) {
  if (!pool || (n_items > 0 && !items) || n_items < 0) return fail(DP_EINVAL, "prefill_attend: null argument");
  if (!pool->owner) return fail(DP_EINVAL, "prefill_attend: the PE pool must be local");
  const dp_kv_geom& g = pool->geom;
  if (layer < 0 || layer >= g.n_layer || layer >= (1 << 20))
    return fail(DP_EINVAL, "prefill_attend: layer out of range");
  if (g.bytes_per_token_layer >= (int64_t{1} << 19))
    return fail(DP_EINVAL, "prefill_attend: b must be < 512 KiB (query word index is 16-bit)");
  if (pool->device >= kMaxDevices) return fail(DP_EINVAL, "prefill_attend: device id too large");
  DeviceGuard guard(pool->device);
  {
    std::lock_guard<std::mutex> lk(g_attend_mu);
    if (!g_attend_init[pool->device]) {
      DP_CUDA(cudaFuncSetAttribute(kv_prefill_attend, cudaFuncAttributeMaxDynamicSharedMemorySize, kAttSmem));
      g_attend_init[pool->device] = true;
    }
  }
  if (!pool->att_ctr) return fail(DP_EINVAL, "prefill_attend: pool has no work-queue counter");
  AttendParams p;
  std::memset(&p, 0, sizeof(p));
  p.pool = pool->base;
  p.ctr = pool->att_ctr;
  p.bpt = g.bytes_per_token_layer;
  p.lb_bytes = static_cast<int64_t>(g.block_tokens) * g.bytes_per_token_layer;
  p.layer_off = static_cast<int64_t>(layer) * layer_stride(pool);
  p.slot_stride = slot_stride(pool);
  p.seed_q = seed * kQueryMul;
  p.layer = layer;
  p.block_tokens = g.block_tokens;
  p.words = static_cast<int32_t>(g.bytes_per_token_layer / 4);
  const int cap = g_attend_ctas[pool->device].load();
  const int grid_cap = cap > 0 ? cap : sm_count(pool->device) * 2;
  const int64_t max_tokens = static_cast<int64_t>(pool->n_slots) * g.block_tokens;
  auto s = static_cast<cudaStream_t>(stream);
  bool signalled = false;
  for (int32_t i0 = 0; i0 < n_items; i0 += DP_MAX_ATTEND_ITEMS_PER_LAUNCH) {
    const int32_t ni = std::min<int32_t>(DP_MAX_ATTEND_ITEMS_PER_LAUNCH, n_items - i0);
    p.done = i0 + ni >= n_items ? done : nullptr;  // the call's last launch signals
    p.n_jobs = 0;
    int64_t units = 0;
    for (int32_t i = 0; i < ni; ++i) {
      const dp_attend_item& it = items[i0 + i];
      if (it.cached < 0 || it.bsz < 0 || it.q_begin < 0 || it.q_begin + it.bsz >= (int64_t{1} << 47) ||
          it.cached > max_tokens || (it.cached > 0 && !it.slot) || (it.cached > 0 && it.bsz > 0 && !it.digest))
        return fail(DP_EINVAL, "prefill_attend: item " + std::to_string(i0 + i) + " out of range");
      const int64_t n_kt = (it.cached + kAttRows - 1) / kAttRows;
      const int64_t n = (it.bsz + kAttRows - 1) / kAttRows * ((n_kt + kAttGroup - 1) / kAttGroup);
      if (n == 0) continue;
      p.jobs[p.n_jobs] = it;
      p.item_begin[p.n_jobs] = units;
      ++p.n_jobs;
      units += n;
    }
    p.item_begin[p.n_jobs] = units;
    if (units == 0) continue;
    kv_prefill_attend<<<static_cast<int>(std::min<int64_t>(units, grid_cap)), kThreads, kAttSmem, s>>>(p);
    DP_CUDA(cudaGetLastError());
    signalled = signalled || p.done != nullptr;
  }
  if (done && !signalled) {  // nothing to compute in the last launch: a stream-ordered write instead
    const WriteValue32Fn wv = write_value32();
    if (!wv) return fail(DP_ECUDA, "prefill_attend: cuStreamWriteValue32 unavailable");
    if (wv(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(done), 1, 0) != CUDA_SUCCESS)
      return fail(DP_ECUDA, "prefill_attend: cuStreamWriteValue32 failed");
  }
  return DP_OK;
}

}  // extern "C"

// ============================================================ staged K1 / K2
// The copy engine moves whole Full-Block runs host -> an HBM staging ring at
// the link's full rate (one 1D copy per contiguous run, a 2D copy of the
// valid rows of a partial last block); the gather kernel then scatters the
// ring's Full Blocks [L][T][b] into the pool's layer planes (HBM -> HBM, or
// over NVLink into a peer PE pool) and releases the landed counters exactly
// as K1 / K2 do.  The ring is split into kStageSegs segments used round
// robin: the copies into a segment wait for the scatter that last read it
// (ev_free), the scatter waits for its copies (ev_copied).
namespace {
constexpr int kStageSegs = 4;
}  // namespace

struct dp_stager {
  int device = -1;
  dp_kv_geom geom{};
  int64_t seg_fb = 0;        // Full Blocks per segment
  dp_store ring;             // device ring of kStageSegs * seg_fb Full Blocks (base in ring.host)
  int64_t* iota = nullptr;   // device [0, 1, ..., ring_fb): ring positions as a src_fb table
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_copied[kStageSegs] = {};
  cudaEvent_t ev_free[kStageSegs] = {};
  int seg = 0;
  int32_t ctas = 32;         // scatter CTAs (HBM-bound: a few keep up with the link)
  int64_t launches = 0;      // scatter kernels launched so far
  int32_t mode = 0;          // DP_SCATTER_KERNEL or DP_SCATTER_CE
};

namespace {

void stager_free(dp_stager* st) {
  DeviceGuard guard(st->device);
  if (st->copy) cudaStreamSynchronize(st->copy);
  for (int i = 0; i < kStageSegs; ++i) {
    if (st->ev_copied[i]) cudaEventDestroy(st->ev_copied[i]);
    if (st->ev_free[i]) cudaEventDestroy(st->ev_free[i]);
  }
  if (st->copy) cudaStreamDestroy(st->copy);
  if (st->ring.host) cudaFree(st->ring.host);
  if (st->iota) cudaFree(st->iota);
  cudaGetLastError();
  delete st;
}

// Copy-engine leg of blocks [k0, k1) of `job` into ring positions base..:
// runs of consecutive storage Full Blocks as 1D copies, a partial last block
// as a 2D copy of its valid rows (exactly the hit bytes cross PCIe).
int stage_copy(dp_stager* st, const dp_store* src, const dp_job& job, int32_t k0, int32_t k1, int64_t base) {
  const dp_kv_geom& g = src->geom;
  const int64_t T = g.block_tokens, b = g.bytes_per_token_layer;
  const int64_t lb = T * b, fbb = lb * g.n_layer;
  const bool last_partial = k1 == job.n_blk && job.n_tokens % T != 0;
  const int32_t full_end = last_partial ? k1 - 1 : k1;
  for (int32_t k = k0; k < full_end;) {
    int32_t run = 1;
    while (k + run < full_end && job.src_fb[k + run] == job.src_fb[k] + run) ++run;
    DP_CUDA(cudaMemcpyAsync(st->ring.host + (base + (k - k0)) * fbb, src->host + job.src_fb[k] * fbb, run * fbb,
                            cudaMemcpyHostToDevice, st->copy));
    k += run;
  }
  if (last_partial) {
    const int32_t k = k1 - 1;
    const int64_t ntok = job.n_tokens - static_cast<int64_t>(k) * T;
    DP_CUDA(cudaMemcpy2DAsync(st->ring.host + (base + (k - k0)) * fbb, lb, src->host + job.src_fb[k] * fbb, lb,
                              ntok * b, g.n_layer, cudaMemcpyHostToDevice, st->copy));
  }
  return DP_OK;
}

// One staged transfer.  The jobs' src_fb arrays are HOST-readable (the copies
// are planned on the host), dst_slot device-readable (the kernel reads it).
int staged_transfer(const char* who, dp_pool* pool, const dp_store* src, dp_stager* st, const dp_job* jobs,
                    int32_t n_jobs, dp_stream stream, bool peer) {
  const std::string w(who);
  if (!pool || !src || !st || (n_jobs > 0 && !jobs) || n_jobs < 0) return fail(DP_EINVAL, w + ": null argument");
  if (peer == pool->owner)
    return fail(DP_EINVAL, w + (peer ? ": destination must be a peer view" : ": destination must be the local pool"));
  if (pool->device != st->device || src->device != st->device)
    return fail(DP_EINVAL, w + ": pool view, store and stager must be on one device");
  if (!geom_equal(pool->geom, src->geom) || !geom_equal(st->geom, src->geom))
    return fail(DP_EINVAL, w + ": geometry differs");
  const dp_kv_geom& g = src->geom;
  const int64_t T = g.block_tokens, b = g.bytes_per_token_layer;
  const int64_t lb = T * b, fbb = lb * g.n_layer;
  for (int32_t j = 0; j < n_jobs; ++j) {  // validate everything before enqueueing anything
    const dp_job& job = jobs[j];
    const int64_t need_blk = (job.n_tokens + T - 1) / T;
    if (job.n_tokens < 0 || job.n_blk != need_blk || job.layer_begin != 0 || job.layer_end != g.n_layer ||
        job.ticket >= pool->n_tickets || (job.n_blk > 0 && (!job.src_fb || !job.dst_slot)))
      return fail(DP_EINVAL, w + ": job " + std::to_string(j) + " out of range (staged jobs move all layers)");
    for (int32_t k = 0; k < job.n_blk; ++k)
      if (job.src_fb[k] < 0 || job.src_fb[k] >= src->n_fb)
        return fail(DP_EINVAL, w + ": job " + std::to_string(j) + ": source block out of range");
    if (st->mode == DP_SCATTER_CE)  // absolute counter writes: one job per ticket and call
      for (int32_t i = 0; i < j; ++i)
        if (job.ticket >= 0 && jobs[i].ticket == job.ticket)
          return fail(DP_EINVAL, w + ": ticket used by two jobs of one call (copy-engine scatter)");
  }
  DeviceGuard guard(st->device);
  auto s = static_cast<cudaStream_t>(stream);
  std::vector<dp_job> sub;
  int64_t used = 0;     // Full Blocks of the open segment
  bool open = false;
  std::vector<int64_t> sub_cum;  // CE mode: the job's items per layer landed after each sub-job
  auto flush = [&]() -> int {
    if (!open) return DP_OK;
    const int seg = st->seg;
    DP_CUDA(cudaEventRecord(st->ev_copied[seg], st->copy));
    DP_CUDA(cudaStreamWaitEvent(s, st->ev_copied[seg], 0));
    if (!sub.empty() && st->mode == DP_SCATTER_CE) {
      // the scatter on a copy engine too: per run of consecutive pool slots and
      // layer one 2D copy ring (Full-Block pitch) -> layer plane (Layer-Block
      // pitch), then fenced stream writes of the landed counters (absolute:
      // the job's items landed so far, per layer and over all layers)
      const int64_t plane = layer_stride(pool), sstride = slot_stride(pool);
      for (size_t q = 0; q < sub.size(); ++q) {
        const dp_job& jb = sub[q];
        const int64_t pos0 = jb.src_fb - st->iota;  // ring position of the sub-job's first block
        const bool part = jb.n_tokens % T != 0;
        const int32_t full = part ? jb.n_blk - 1 : jb.n_blk;
        for (int32_t k = 0; k < jb.n_blk;) {
          int32_t run = 1;
          const bool pk = part && k == jb.n_blk - 1;
          if (!pk)
            while (k + run < full && jb.dst_slot[k + run] == jb.dst_slot[k] + run) ++run;
          const int64_t width = pk ? (jb.n_tokens - static_cast<int64_t>(k) * T) * b : lb;
          for (int32_t layer = 0; layer < g.n_layer; ++layer)
            DP_CUDA(cudaMemcpy2DAsync(pool->base + layer * plane + static_cast<int64_t>(jb.dst_slot[k]) * sstride,
                                      sstride, st->ring.host + (pos0 + k) * fbb + layer * lb, fbb, width, run,
                                      cudaMemcpyDeviceToDevice, s));
          k += run;
        }
        if (jb.ticket >= 0) {
          uint32_t* row = pool->counters + static_cast<int64_t>(jb.ticket) * (g.n_layer + 1);
          const uint32_t v = static_cast<uint32_t>(sub_cum[q]);
          std::vector<std::pair<uint32_t*, uint32_t>> writes;
          for (int32_t layer = 0; layer <= g.n_layer; ++layer)
            writes.emplace_back(row + layer, layer == g.n_layer ? v * static_cast<uint32_t>(g.n_layer) : v);
          if (int rc = write_counters(s, writes, w)) return rc;
        }
      }
    } else if (!sub.empty()) {
      if (int rc = launch_gather(pool, &st->ring, sub.data(), static_cast<int32_t>(sub.size()), stream, peer,
                                 st->ctas, /*stream_hint=*/true))
        return rc;
      ++st->launches;
    }
    sub_cum.clear();
    DP_CUDA(cudaEventRecord(st->ev_free[seg], s));
    st->seg = (seg + 1) % kStageSegs;
    sub.clear();
    used = 0;
    open = false;
    return DP_OK;
  };
  for (int32_t j = 0; j < n_jobs; ++j) {
    const dp_job& job = jobs[j];
    for (int32_t k0 = 0; k0 < job.n_blk;) {
      if (open && (used == st->seg_fb || sub.size() == DP_MAX_JOBS_PER_LAUNCH))
        if (int rc = flush()) return rc;
      if (!open) {  // the segment's copies wait for the scatter that last read it
        DP_CUDA(cudaStreamWaitEvent(st->copy, st->ev_free[st->seg], 0));
        open = true;
      }
      const int32_t k1 = static_cast<int32_t>(std::min<int64_t>(job.n_blk, k0 + (st->seg_fb - used)));
      const int64_t base = st->seg * st->seg_fb + used;  // ring position of block k0
      if (int rc = stage_copy(st, src, job, k0, k1, base)) return rc;
      const int64_t tok0 = static_cast<int64_t>(k0) * T;
      sub.push_back(dp_job{st->iota + base, job.dst_slot + k0, std::min<int64_t>(job.n_tokens, k1 * T) - tok0,
                           k1 - k0, 0, g.n_layer, job.ticket});
      sub_cum.push_back(static_cast<int64_t>(k1) * chunks_per_block(g));
      used += k1 - k0;
      k0 = k1;
    }
  }
  return flush();
}

}  // namespace

extern "C" {

int dp_stager_create(int device, const dp_kv_geom* geom, int64_t ring_bytes, dp_stager** out) {
  if (!out) return fail(DP_EINVAL, "stager_create: null out");
  *out = nullptr;
  if (int rc = dp_geom_check(geom)) return rc;
  if (ring_bytes < 0) return fail(DP_EINVAL, "stager_create: negative ring size");
  if (int rc = preload_kernels(device)) return rc;
  const int64_t fbb = static_cast<int64_t>(geom->n_layer) * geom->block_tokens * geom->bytes_per_token_layer;
  const int64_t seg_fb = std::max<int64_t>(1, (ring_bytes > 0 ? ring_bytes : int64_t{1} << 30) / fbb / kStageSegs);
  DeviceGuard guard(device);
  auto* st = new dp_stager;
  st->device = device;
  st->geom = *geom;
  st->seg_fb = seg_fb;
  st->ring.device = device;
  st->ring.geom = *geom;
  st->ring.n_fb = seg_fb * kStageSegs;
  st->ring.bytes = st->ring.n_fb * fbb;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&st->ring.host), st->ring.bytes);
  if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&st->iota), st->ring.n_fb * sizeof(int64_t));
  if (e == cudaSuccess) {
    std::vector<int64_t> iota(st->ring.n_fb);
    for (int64_t i = 0; i < st->ring.n_fb; ++i) iota[i] = i;
    e = cudaMemcpy(st->iota, iota.data(), iota.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st->copy, cudaStreamNonBlocking);
  for (int i = 0; i < kStageSegs && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&st->ev_copied[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->ev_free[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    stager_free(st);
    return fail(e == cudaErrorMemoryAllocation ? DP_ENOMEM : DP_ECUDA,
                std::string("stager_create: ") + cudaGetErrorString(e));
  }
  *out = st;
  return DP_OK;
}

int dp_stager_destroy(dp_stager* st) {
  if (st) stager_free(st);
  return DP_OK;
}

int dp_stager_launches(const dp_stager* st, int64_t* n) {
  if (!st || !n) return fail(DP_EINVAL, "stager_launches: null argument");
  *n = st->launches;
  return DP_OK;
}

int dp_stager_set_mode(dp_stager* st, int32_t mode) {
  if (!st || (mode != DP_SCATTER_KERNEL && mode != DP_SCATTER_CE)) return fail(DP_EINVAL, "stager_set_mode: bad argument");
  st->mode = mode;
  return DP_OK;
}

int dp_stager_set_ctas(dp_stager* st, int32_t ctas) {
  if (!st || ctas < 0) return fail(DP_EINVAL, "stager_set_ctas: bad argument");
  st->ctas = ctas > 0 ? ctas : 32;
  return DP_OK;
}

int dp_h2d_layer_staged(dp_pool* pe, const dp_store* src, dp_stager* st, const dp_job* jobs, int32_t n_jobs,
                        dp_stream stream) {
  return staged_transfer("h2d_layer_staged", pe, src, st, jobs, n_jobs, stream, /*peer=*/false);
}

int dp_h2d_push_staged(dp_pool* pe_view, const dp_store* de_src, dp_stager* st, const dp_job* jobs,
                       int32_t n_jobs, dp_stream de_stream) {
  return staged_transfer("h2d_push_staged", pe_view, de_src, st, jobs, n_jobs, de_stream, /*peer=*/true);
}

int dp_h2d_push_dual_staged(dp_pool* pe_view, dp_pool* de_pool, const dp_store* de_src, dp_stager* st,
                            const dp_dual_job* jobs, int32_t n_jobs, dp_stream de_stream) {
  if (!pe_view || !de_pool || !de_src || !st || (n_jobs > 0 && !jobs) || n_jobs < 0)
    return fail(DP_EINVAL, "push_dual_staged: null argument");
  if (de_pool->device != st->device || de_src->device != st->device)
    return fail(DP_EINVAL, "push_dual_staged: decode pool, store and stager must be on one device");
  if (pe_view->layout != DP_POOL_LAYER_MAJOR || de_pool->layout != DP_POOL_LAYER_MAJOR)
    return fail(DP_EINVAL, "push_dual_staged: layer-major pools only");
  if (!geom_equal(st->geom, de_src->geom)) return fail(DP_EINVAL, "push_dual_staged: geometry differs");
  const dp_kv_geom& g = de_src->geom;
  const int64_t T = g.block_tokens;
  for (int32_t j = 0; j < n_jobs; ++j) {
    const dp_job& job = jobs[j].pe;
    if (job.n_tokens < 0 || job.n_blk != (job.n_tokens + T - 1) / T || job.layer_begin != 0 ||
        job.layer_end != g.n_layer || (job.n_blk > 0 && (!job.src_fb || !job.dst_slot || !jobs[j].de_slot)))
      return fail(DP_EINVAL, "push_dual_staged: job " + std::to_string(j) + " out of range (all layers)");
    for (int32_t k = 0; k < job.n_blk; ++k)
      if (job.src_fb[k] < 0 || job.src_fb[k] >= de_src->n_fb)
        return fail(DP_EINVAL, "push_dual_staged: source block out of range");
  }
  DeviceGuard guard(st->device);
  auto s = static_cast<cudaStream_t>(de_stream);
  std::vector<dp_dual_job> sub;
  int64_t used = 0;
  bool open = false;
  auto flush = [&]() -> int {
    if (!open) return DP_OK;
    const int seg = st->seg;
    DP_CUDA(cudaEventRecord(st->ev_copied[seg], st->copy));
    DP_CUDA(cudaStreamWaitEvent(s, st->ev_copied[seg], 0));
    if (!sub.empty()) {
      if (int rc = launch_dual(pe_view, de_pool, &st->ring, sub.data(), static_cast<int32_t>(sub.size()), de_stream,
                               st->ctas))
        return rc;
      ++st->launches;
    }
    DP_CUDA(cudaEventRecord(st->ev_free[seg], s));
    st->seg = (seg + 1) % kStageSegs;
    sub.clear();
    used = 0;
    open = false;
    return DP_OK;
  };
  for (int32_t j = 0; j < n_jobs; ++j) {
    const dp_dual_job& dj = jobs[j];
    for (int32_t k0 = 0; k0 < dj.pe.n_blk;) {
      if (open && (used == st->seg_fb || sub.size() == DP_MAX_DUAL_JOBS_PER_LAUNCH))
        if (int rc = flush()) return rc;
      if (!open) {
        DP_CUDA(cudaStreamWaitEvent(st->copy, st->ev_free[st->seg], 0));
        open = true;
      }
      const int32_t k1 = static_cast<int32_t>(std::min<int64_t>(dj.pe.n_blk, k0 + (st->seg_fb - used)));
      const int64_t base = st->seg * st->seg_fb + used;
      if (int rc = stage_copy(st, de_src, dj.pe, k0, k1, base)) return rc;
      dp_dual_job part = dj;
      part.pe = dp_job{st->iota + base, dj.pe.dst_slot + k0,
                       std::min<int64_t>(dj.pe.n_tokens, static_cast<int64_t>(k1) * T) - static_cast<int64_t>(k0) * T,
                       k1 - k0, 0, g.n_layer, dj.pe.ticket};
      part.de_slot = dj.de_slot + k0;
      sub.push_back(part);
      used += k1 - k0;
      k0 = k1;
    }
  }
  return flush();
}

}  // extern "C"

// ================================================ K4 staged (PersistD2H)
// dp_persist_staged: the gather kernel (kv_persist_d2h with the ring as its
// target) packs each span's tokens from the decode pool's layer planes into
// Full Blocks [L][T][b] of the HBM ring; the copy engine moves them to the
// host Full Blocks: a run of whole blocks as one 1D copy, a partial block as
// one 2D copy of its L token ranges.  Consecutive spans of one request (the
// 64-token persist chunks) are merged first, so only a request's first and
// last blocks are partial.
namespace {

int persist_copy(dp_stager* st, dp_store* target, const dp_span_job& job, int64_t pos0) {
  const dp_kv_geom& g = st->geom;
  const int64_t T = g.block_tokens, b = g.bytes_per_token_layer;
  const int64_t lb = T * b, fbb = lb * g.n_layer;
  for (int32_t i = 0; i < job.n_blk;) {
    const int64_t bt0 = (job.blk0 + i) * T;
    const int64_t t0 = std::max(job.tok_begin, bt0) - bt0, t1 = std::min(job.tok_end, bt0 + T) - bt0;
    if (t1 <= t0) {
      ++i;
      continue;
    }
    if (t0 == 0 && t1 == T) {  // whole blocks: runs of consecutive target Full Blocks
      int32_t run = 1;
      while (i + run < job.n_blk && job.fb[i + run] == job.fb[i] + run &&
             (job.blk0 + i + run + 1) * T <= job.tok_end)
        ++run;
      DP_CUDA(cudaMemcpyAsync(target->host + job.fb[i] * fbb, st->ring.host + (pos0 + i) * fbb, run * fbb,
                              cudaMemcpyDeviceToHost, st->copy));
      i += run;
      continue;
    }
    DP_CUDA(cudaMemcpy2DAsync(target->host + job.fb[i] * fbb + t0 * b, lb, st->ring.host + (pos0 + i) * fbb + t0 * b,
                              lb, (t1 - t0) * b, g.n_layer, cudaMemcpyDeviceToHost, st->copy));
    ++i;
  }
  return DP_OK;
}

}  // namespace

extern "C" {

int dp_persist_staged(const dp_pool* de_pool, dp_store* target, dp_stager* st, const dp_span_job* jobs,
                      int32_t n_jobs, dp_stream stream) {
  if (!de_pool || !target || !st || (n_jobs > 0 && !jobs) || n_jobs < 0)
    return fail(DP_EINVAL, "persist_staged: null argument");
  if (!de_pool->owner) return fail(DP_EINVAL, "persist_staged: the decode pool must be local");
  if (de_pool->layout != DP_POOL_LAYER_MAJOR) return fail(DP_EINVAL, "persist_staged: layer-major pools only");
  if (de_pool->device != st->device) return fail(DP_EINVAL, "persist_staged: pool and stager on different devices");
  if (!geom_equal(de_pool->geom, target->geom) || !geom_equal(st->geom, target->geom))
    return fail(DP_EINVAL, "persist_staged: geometry differs");
  const dp_kv_geom& g = target->geom;
  const int64_t T = g.block_tokens;
  // merge consecutive spans of one request (same tables, contiguous tokens)
  std::vector<dp_span_job> merged;
  for (int32_t j = 0; j < n_jobs; ++j) {
    const dp_span_job& job = jobs[j];
    if (job.n_blk < 0 || job.blk0 < 0 || job.tok_begin < job.blk0 * T || job.tok_end < job.tok_begin ||
        job.tok_end > (job.blk0 + job.n_blk) * T || (job.n_blk > 0 && (!job.slot || !job.fb)))
      return fail(DP_EINVAL, "persist_staged: job " + std::to_string(j) + " out of range");
    for (int32_t i = 0; i < job.n_blk; ++i)
      if (job.fb[i] < 0 || job.fb[i] >= target->n_fb)
        return fail(DP_EINVAL, "persist_staged: job " + std::to_string(j) + ": target block out of range");
    if (job.tok_end == job.tok_begin || job.n_blk == 0) continue;
    if (!merged.empty()) {
      dp_span_job& m = merged.back();
      if (m.slot == job.slot && m.fb == job.fb && m.blk0 == job.blk0 && m.n_blk == job.n_blk &&
          m.tok_end == job.tok_begin) {
        m.tok_end = job.tok_end;
        continue;
      }
    }
    merged.push_back(job);
  }
  DeviceGuard guard(st->device);
  auto s = static_cast<cudaStream_t>(stream);
  struct Part {
    dp_span_job job;  // host fb table, ring positions from pos0
    int64_t pos0;
  };
  std::vector<dp_span_job> sub;  // kernel view: fb = ring positions
  std::vector<Part> parts;
  int64_t used = 0;
  bool open = false;
  int last_seg = -1;
  auto flush = [&]() -> int {
    if (!open) return DP_OK;
    const int seg = st->seg;
    if (int rc = launch_span(de_pool, &st->ring, sub.data(), static_cast<int32_t>(sub.size()), 0, stream,
                             kv_persist_d2h, "persist_staged"))
      return rc;
    ++st->launches;
    DP_CUDA(cudaEventRecord(st->ev_copied[seg], s));  // gathered into the segment
    DP_CUDA(cudaStreamWaitEvent(st->copy, st->ev_copied[seg], 0));
    for (const Part& pt : parts)
      if (int rc = persist_copy(st, target, pt.job, pt.pos0)) return rc;
    DP_CUDA(cudaEventRecord(st->ev_free[seg], st->copy));  // drained to the host
    last_seg = seg;
    st->seg = (seg + 1) % kStageSegs;
    sub.clear();
    parts.clear();
    used = 0;
    open = false;
    return DP_OK;
  };
  for (const dp_span_job& job : merged) {
    // blocks holding none of the span are skipped
    int32_t first = 0, end = job.n_blk;
    while (first < end && (job.blk0 + first + 1) * T <= job.tok_begin) ++first;
    while (end > first && (job.blk0 + end - 1) * T >= job.tok_end) --end;
    for (int32_t i0 = first; i0 < end;) {
      if (open && (used == st->seg_fb || sub.size() == DP_MAX_SPAN_JOBS_PER_LAUNCH))
        if (int rc = flush()) return rc;
      if (!open) {  // the gather into the segment waits for the copies that last drained it
        DP_CUDA(cudaStreamWaitEvent(s, st->ev_free[st->seg], 0));
        open = true;
      }
      const int32_t i1 = static_cast<int32_t>(std::min<int64_t>(end, i0 + (st->seg_fb - used)));
      const int64_t base = st->seg * st->seg_fb + used;
      dp_span_job part = job;
      part.blk0 = job.blk0 + i0;
      part.n_blk = i1 - i0;
      part.tok_begin = std::max(job.tok_begin, part.blk0 * T);
      part.tok_end = std::min(job.tok_end, (part.blk0 + part.n_blk) * T);
      part.slot = job.slot + i0;
      part.fb = job.fb + i0;
      parts.push_back({part, base});
      part.fb = st->iota + base;
      sub.push_back(part);
      used += i1 - i0;
      i0 = i1;
    }
  }
  if (int rc = flush()) return rc;
  if (last_seg >= 0) DP_CUDA(cudaStreamWaitEvent(s, st->ev_free[last_seg], 0));  // later work sees the host bytes
  return DP_OK;
}

}  // extern "C"

// ============================================================ eager loading
namespace {

std::once_flag g_preload_once[kMaxDevices];
int g_preload_rc[kMaxDevices] = {};

int preload_kernels(int device) {
  if (device < 0 || device >= kMaxDevices) return fail(DP_EINVAL, "device id out of range");
  std::call_once(g_preload_once[device], [device] {
    DeviceGuard guard(device);
    const void* fns[] = {reinterpret_cast<const void*>(kv_gather<false>),
                         reinterpret_cast<const void*>(kv_gather<true>),
                         reinterpret_cast<const void*>(kv_gather<false, true>),
                         reinterpret_cast<const void*>(kv_gather<true, true>),
                         reinterpret_cast<const void*>(kv_wait_ge),
                         reinterpret_cast<const void*>(kv_wait_many),
                         reinterpret_cast<const void*>(kv_block_checksum),
                         reinterpret_cast<const void*>(kv_store_fill),
                         reinterpret_cast<const void*>(kv_gather_dual),
                         reinterpret_cast<const void*>(kv_prefill_handoff<false>),
                         reinterpret_cast<const void*>(kv_prefill_handoff<true>),
                         reinterpret_cast<const void*>(kv_handoff_side),
                         reinterpret_cast<const void*>(kv_decode_fill),
                         reinterpret_cast<const void*>(kv_persist_d2h),
                         reinterpret_cast<const void*>(kv_prefill_attend)};
    if (cudaFuncSetAttribute(kv_prefill_handoff<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kHandoffTmaSmem) != cudaSuccess) {
      g_preload_rc[device] = fail(DP_ECUDA, "preload_kernels: K3 TMA shared memory");
      return;
    }
    for (const void* f : fns) {
      cudaFuncAttributes a;
      if (cudaFuncGetAttributes(&a, f) != cudaSuccess) {
        g_preload_rc[device] = fail(DP_ECUDA, std::string("preload_kernels: ") +
                                                  cudaGetErrorString(cudaGetLastError()));
        return;
      }
    }
  });
  return g_preload_rc[device];
}

}  // namespace
