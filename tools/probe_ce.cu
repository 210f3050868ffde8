// Probe: can the copy engine carry Layer Blocks faster than SM zero-copy?
//  (1) cudaMemcpy2DAsync of Layer-Block runs (width = T*b, src pitch = Full
//      Block, dst pitch = Layer Block): the strided shape of one layer of one
//      request, per call;
//  (2) copy engine and SM zero-copy at the same time on one GPU: does the
//      PCIe link carry more than either alone?
// Not product code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_ce tools/probe_ce.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <chrono>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

__global__ void zc(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = __ldg(src + i);
}

int main() {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const size_t L = 61, LB = 36864, FB = L * LB;
  const size_t NFB = 2048;                    // 4.6 GB host store
  char* host; CK(cudaHostAlloc(&host, NFB * FB, cudaHostAllocMapped | cudaHostAllocPortable));
  for (size_t i = 0; i < NFB * FB; i += 4096) host[i] = (char)i;
  char* dev; CK(cudaMalloc(&dev, NFB * FB));
  cudaStream_t s1, s2; CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b, c, d; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b)); CK(cudaEventCreate(&c)); CK(cudaEventCreate(&d));
  // (1) 2D copies: runs of `run` blocks, one call per (run, layer)
  for (int run : {16, 64, 128, 512}) {
    const int runs = (int)(NFB / run);
    const size_t plane = NFB * LB;  // pool layer plane
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(a, s1));
      for (int r = 0; r < runs; ++r)
        for (size_t l = 0; l < L; ++l)
          CK(cudaMemcpy2DAsync(dev + l * plane + (size_t)r * run * LB, LB, host + (size_t)r * run * FB + l * LB, FB,
                               LB, run, cudaMemcpyHostToDevice, s1));
      CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
    }
    std::printf("ce2d run=%d blocks: %.1f GB/s (%d calls)\n", run, NFB * FB / (best * 1e-3) / 1e9, runs * (int)L);
  }
  // (1b) the same 2D copies spread round-robin over k streams: is the gap to
  // the 1-D copy peak a per-call latency that concurrency hides?
  {
    cudaStream_t ss[4];
    for (auto& x : ss) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    cudaEvent_t done[4];
    for (auto& x : done) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    for (int k : {1, 2, 4})
      for (int run : {16, 64, 128}) {
        const int runs = (int)(NFB / run);
        const size_t plane = NFB * LB;
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
          CK(cudaDeviceSynchronize());
          CK(cudaEventRecord(a, s1));
          for (int i = 0; i < k; ++i) CK(cudaStreamWaitEvent(ss[i], a, 0));
          int n = 0;
          for (size_t l = 0; l < L; ++l)
            for (int r = 0; r < runs; ++r, ++n)
              CK(cudaMemcpy2DAsync(dev + l * plane + (size_t)r * run * LB, LB,
                                   host + (size_t)r * run * FB + l * LB, FB, LB, run,
                                   cudaMemcpyHostToDevice, ss[n % k]));
          for (int i = 0; i < k; ++i) { CK(cudaEventRecord(done[i], ss[i])); CK(cudaStreamWaitEvent(s1, done[i], 0)); }
          CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
          float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
        }
        std::printf("ce2d %d streams run=%d: %.1f GB/s\n", k, run, NFB * FB / (best * 1e-3) / 1e9);
      }
  }
  // (1c) the 2D copies captured once into a CUDA graph and replayed: if the
  // per-call gap is host submission cost, the replay closes it.
  for (int run : {16, 64, 128}) {
    const int runs = (int)(NFB / run);
    const size_t plane = NFB * LB;
    cudaGraph_t graph; cudaGraphExec_t exec;
    CK(cudaStreamBeginCapture(s1, cudaStreamCaptureModeThreadLocal));
    for (size_t l = 0; l < L; ++l)
      for (int r = 0; r < runs; ++r)
        CK(cudaMemcpy2DAsync(dev + l * plane + (size_t)r * run * LB, LB,
                             host + (size_t)r * run * FB + l * LB, FB, LB, run,
                             cudaMemcpyHostToDevice, s1));
    CK(cudaStreamEndCapture(s1, &graph));
    CK(cudaGraphInstantiate(&exec, graph, 0));
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(a, s1)); CK(cudaGraphLaunch(exec, s1)); CK(cudaEventRecord(b, s1));
      CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
    }
    std::printf("ce2d graph run=%d: %.1f GB/s\n", run, NFB * FB / (best * 1e-3) / 1e9);
    CK(cudaGraphExecDestroy(exec)); CK(cudaGraphDestroy(graph));
  }
  // host-side submission cost of one 2D call, no GPU wait
  {
    CK(cudaDeviceSynchronize());
    const int n = 2000;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i)
      CK(cudaMemcpy2DAsync(dev + (size_t)(i % 64) * LB, LB, host + (size_t)(i % 64) * FB, FB, LB, 1,
                           cudaMemcpyHostToDevice, s1));
    auto t1 = std::chrono::steady_clock::now();
    CK(cudaStreamSynchronize(s1));
    std::printf("host submit cost per 2D call: %.2f us\n",
                std::chrono::duration<double, std::micro>(t1 - t0).count() / n);
  }
  // one contiguous 1-D copy per (run, layer), same bytes: the layer-major staging shape
  for (int run : {16, 64, 128}) {
    const int runs = (int)(NFB / run);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(a, s1));
      for (size_t l = 0; l < L; ++l)
        for (int r = 0; r < runs; ++r) {
          const size_t off = (l * NFB + (size_t)r * run) * LB;
          CK(cudaMemcpyAsync(dev + off, host + off, (size_t)run * LB, cudaMemcpyHostToDevice, s1));
        }
      CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
    }
    std::printf("ce1d run=%d: %.1f GB/s\n", run, NFB * FB / (best * 1e-3) / 1e9);
  }
  // (2) CE and SM together: CE copies the first half, SM the second half
  const size_t half = (NFB * FB / 2) & ~(size_t)15;
  char* dptr; CK(cudaHostGetDevicePointer((void**)&dptr, host, 0));
  for (int grid : {148, 592}) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, s1)); CK(cudaEventRecord(c, s2));
      CK(cudaMemcpyAsync(dev, host, half, cudaMemcpyHostToDevice, s1));
      zc<<<grid, 256, 0, s2>>>((const uint4*)(dptr + half), (uint4*)(dev + half), half / 16);
      CK(cudaEventRecord(b, s1)); CK(cudaEventRecord(d, s2));
      CK(cudaDeviceSynchronize());
      float m1, m2; CK(cudaEventElapsedTime(&m1, a, b)); CK(cudaEventElapsedTime(&m2, c, d));
      float m = m1 > m2 ? m1 : m2; if (m < best) best = m;
      if (rep == 2) std::printf("  ce %.1f ms, sm %.1f ms\n", m1, m2);
    }
    std::printf("ce+sm concurrent (grid %d): %.1f GB/s total\n", grid, 2 * half / (best * 1e-3) / 1e9);
  }
  // CE alone and SM alone on the same bytes for reference
  {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaEventRecord(a, s1)); CK(cudaMemcpyAsync(dev, host, 2 * half, cudaMemcpyHostToDevice, s1));
      CK(cudaEventRecord(b, s1)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
    }
    std::printf("ce alone: %.1f GB/s\n", 2 * half / (best * 1e-3) / 1e9);
  }
  // (3) DE-stream copy engine writing host -> PEER device memory: which PCIe
  // link does it read over?  Run it concurrently with the PE's own H2D.
  int ndev = 0; CK(cudaGetDeviceCount(&ndev));
  if (ndev >= 2) {
    CK(cudaSetDevice(1));
    cudaError_t pe = cudaDeviceEnablePeerAccess(0, 0); if (pe != cudaSuccess) cudaGetLastError();
    cudaStream_t s3; CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    CK(cudaSetDevice(0));
    const size_t q = half;  // GPU0 own copy: first half; GPU1 -> GPU0 peer: second half
    for (int mode = 0; mode < 2; ++mode) {
      CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize()); CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(1)); CK(cudaEventRecord(e0, s3));
      CK(cudaMemcpyAsync(dev + q, host + q, q, cudaMemcpyHostToDevice, s3));  // dst lives on GPU0
      CK(cudaEventRecord(e1, s3));
      CK(cudaSetDevice(0));
      if (mode == 1) { CK(cudaEventRecord(a, s1)); CK(cudaMemcpyAsync(dev, host, q, cudaMemcpyHostToDevice, s1)); CK(cudaEventRecord(b, s1)); }
      CK(cudaSetDevice(1)); CK(cudaEventSynchronize(e1)); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
      float m1; CK(cudaEventElapsedTime(&m1, e0, e1));
      float m0 = 0; if (mode == 1) CK(cudaEventElapsedTime(&m0, a, b));
      std::printf("gpu1-stream H2D into gpu0 memory: %.1f GB/s%s", q / (m1 * 1e-3) / 1e9, mode ? "" : " (alone)\n");
      if (mode) std::printf(" while gpu0 own H2D: %.1f GB/s\n", q / (m0 * 1e-3) / 1e9);
    }
  }
  std::printf("done\n");
  return 0;
}
