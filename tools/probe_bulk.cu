// Probe: can the bulk-copy (TMA) engine source host-mapped pinned memory, and
// does it beat SM LDG.128 zero-copy on PCIe H2D?  Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_bulk tools/probe_bulk.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Each CTA: STAGES smem buffers of CH bytes; thread 0 streams chunks
// host --(cp.async.bulk)--> smem --(cp.async.bulk store)--> global.
template <int STAGES>
__global__ void bulk_copy(const char* __restrict__ src, char* __restrict__ dst, size_t bytes, int ch) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  size_t nch = (bytes + ch - 1) / ch;
  uint32_t phase[STAGES];
  for (int s = 0; s < STAGES; ++s) phase[s] = 0;
  // prologue
  size_t c0 = blockIdx.x;
  size_t stride = gridDim.x;
  int s = 0;
  size_t issued = 0;
  size_t cs[STAGES];
  for (int k = 0; k < STAGES; ++k) {
    size_t c = c0 + (size_t)k * stride;
    cs[k] = c;
    if (c >= nch) continue;
    uint32_t n = (uint32_t)((c + 1) * ch <= bytes ? ch : bytes - c * ch);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[k])), "r"(n) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(smem + (size_t)k * ch)), "l"(src + c * ch), "r"(n), "r"(smem_u32(&bar[k])) : "memory");
    ++issued;
  }
  for (size_t c = c0; c < nch; c += stride) {
    uint32_t n = (uint32_t)((c + 1) * ch <= bytes ? ch : bytes - c * ch);
    // wait for stage s
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(smem_u32(&bar[s])), "r"(phase[s]) : "memory");
    }
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 :: "l"(dst + c * ch), "r"(smem_u32(smem + (size_t)s * ch)), "r"(n) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    size_t cn = c + (size_t)STAGES * stride;
    if (cn < nch) {
      uint32_t nn = (uint32_t)((cn + 1) * ch <= bytes ? ch : bytes - cn * ch);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(nn) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(smem_u32(smem + (size_t)s * ch)), "l"(src + cn * ch), "r"(nn), "r"(smem_u32(&bar[s])) : "memory");
    }
    s = (s + 1) % STAGES;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const size_t BYTES = 1ull << 30;
  CK(cudaSetDevice(0));
  char* host; CK(cudaHostAlloc(&host, BYTES, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < BYTES; i += 8) *(uint64_t*)(host + i) = i * 0x9E3779B97F4A7C15ull;
  char* dev; CK(cudaMalloc(&dev, BYTES));
  char* dptr; CK(cudaHostGetDevicePointer((void**)&dptr, host, 0));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  for (int ch : {16384, 36864, 65536}) for (int grid : {148, 296}) {
    const int STG = 3;
    size_t smem = (size_t)STG * ch;
    CK(cudaFuncSetAttribute(bulk_copy<STG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (smem * (grid / 148) > 220 * 1024) continue;
    double best = 1e30;
    for (int r = 0; r < 4; ++r) {
      CK(cudaMemsetAsync(dev, 0, BYTES, st));
      CK(cudaEventRecord(a, st));
      bulk_copy<STG><<<grid, 32, smem, st>>>(dptr, dev, BYTES, ch);
      CK(cudaGetLastError());
      CK(cudaEventRecord(b, st));
      CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, (double)ms);
    }
    // verify a sample
    uint64_t probe[4];
    for (int k = 0; k < 4; ++k) {
      size_t off = ((size_t)k * 0x3FFFF1ull * 8) % BYTES;
      CK(cudaMemcpy(&probe[k], dev + off, 8, cudaMemcpyDeviceToHost));
      if (probe[k] != off * 0x9E3779B97F4A7C15ull) { std::printf("MISMATCH ch %d off %zu\n", ch, off); }
    }
    std::printf("bulk ch %d grid %d stages %d: %.1f GB/s\n", ch, grid, STG, BYTES / (best * 1e-3) / 1e9);
  }
  std::printf("done\n");
  return 0;
}
