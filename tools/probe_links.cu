// Link probe for the B200 box: PCIe H2D (copy engine vs zero-copy SM loads),
// concurrency across GPUs (shared PCIe switches), NVLink peer copies, and the
// fused host->peer pattern used by the DE read path.  Not product code; the
// numbers it prints are recorded under profiles/.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o probe tools/probe_links.cu -lpthread
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <chrono>
#include <string>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  std::fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); std::exit(1);} } while (0)

__global__ void zc_read(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  constexpr int U = 8;
  size_t i = tid;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n16; i += stride) dst[i] = __ldg(src + i);
}

// contiguous chunk per CTA (blocks of 36864B like DS-V3 layer blocks)
__global__ void zc_read_chunk(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16, int chunk16) {
  size_t nchunks = (n16 + chunk16 - 1) / chunk16;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    size_t base = c * chunk16;
    size_t end = base + chunk16 < n16 ? base + chunk16 : n16;
    constexpr int U = 9;
    uint4 v[U];
    size_t i0 = base + threadIdx.x;
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = i0 + u * blockDim.x; if (i < end) v[u] = __ldg(src + i); }
#pragma unroll
    for (int u = 0; u < U; ++u) { size_t i = i0 + u * blockDim.x; if (i < end) dst[i] = v[u]; }
  }
}

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Gpu {
  int dev;
  void* host = nullptr;   // pinned mapped
  void* dev_buf = nullptr;
  cudaStream_t s;
};

static const size_t BYTES = 1ull << 30;

static double time_memcpy_h2d(Gpu& g, size_t bytes, int reps) {
  CK(cudaSetDevice(g.dev));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a, g.s));
    CK(cudaMemcpyAsync(g.dev_buf, g.host, bytes, cudaMemcpyHostToDevice, g.s));
    CK(cudaEventRecord(b, g.s));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, (double)ms);
  }
  return bytes / (best * 1e-3) / 1e9;
}

static double time_memcpy_d2h(Gpu& g, size_t bytes, int reps) {
  CK(cudaSetDevice(g.dev));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a, g.s));
    CK(cudaMemcpyAsync(g.host, g.dev_buf, bytes, cudaMemcpyDeviceToHost, g.s));
    CK(cudaEventRecord(b, g.s));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, (double)ms);
  }
  return bytes / (best * 1e-3) / 1e9;
}

static double time_zc(Gpu& g, size_t bytes, int grid, int block, int reps, int chunk16 = 0, void* dst = nullptr) {
  CK(cudaSetDevice(g.dev));
  void* dptr;
  CK(cudaHostGetDevicePointer(&dptr, g.host, 0));
  if (!dst) dst = g.dev_buf;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  double best = 1e30;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a, g.s));
    if (chunk16)
      zc_read_chunk<<<grid, block, 0, g.s>>>((const uint4*)dptr, (uint4*)dst, bytes / 16, chunk16);
    else
      zc_read<<<grid, block, 0, g.s>>>((const uint4*)dptr, (uint4*)dst, bytes / 16);
    CK(cudaGetLastError());
    CK(cudaEventRecord(b, g.s));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, (double)ms);
  }
  return bytes / (best * 1e-3) / 1e9;
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  std::printf("devices %d\n", n);
  std::vector<Gpu> gs(n);
  for (int d = 0; d < n; ++d) {
    gs[d].dev = d;
    CK(cudaSetDevice(d));
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, d));
    std::printf("dev %d %s sm=%d pci %04x:%02x:%02x l2=%d MB\n", d, p.name, p.multiProcessorCount,
                p.pciDomainID, p.pciBusID, p.pciDeviceID, p.l2CacheSize >> 20);
    double t0 = now_s();
    CK(cudaHostAlloc(&gs[d].host, BYTES, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(gs[d].host, d + 1, BYTES);
    double t1 = now_s();
    CK(cudaMalloc(&gs[d].dev_buf, BYTES));
    CK(cudaStreamCreateWithFlags(&gs[d].s, cudaStreamNonBlocking));
    std::printf("  hostalloc+touch 1GiB: %.2f s\n", t1 - t0);
  }
  // 1. per-GPU alone
  for (int d = 0; d < n; ++d) {
    double h2d = time_memcpy_h2d(gs[d], BYTES, 5);
    double d2h = time_memcpy_d2h(gs[d], BYTES, 5);
    std::printf("alone dev %d: memcpy H2D %.1f GB/s  D2H %.1f GB/s\n", d, h2d, d2h);
  }
  // zero-copy configs on dev 0
  for (int grid : {148, 296, 592, 1184}) for (int block : {256, 512}) {
    double zc = time_zc(gs[0], BYTES, grid, block, 4);
    std::printf("zc dev0 grid %d block %d: %.1f GB/s\n", grid, block, zc);
  }
  for (int grid : {148, 296, 592, 1184}) {
    double zc = time_zc(gs[0], BYTES, grid, 256, 4, 2304);
    std::printf("zc-chunk36864 dev0 grid %d: %.1f GB/s\n", grid, zc);
  }
  for (int d = 1; d < n; ++d) {
    double zc = time_zc(gs[d], BYTES, 592, 256, 3);
    std::printf("zc dev %d grid 592: %.1f GB/s\n", d, zc);
  }
  // 2. concurrent: all GPUs memcpy H2D; then pairs
  auto concurrent = [&](std::vector<int> devs, bool zc) {
    std::vector<double> r(devs.size());
    std::vector<std::thread> th;
    for (size_t i = 0; i < devs.size(); ++i)
      th.emplace_back([&, i] { r[i] = zc ? time_zc(gs[devs[i]], BYTES, 592, 256, 3) : time_memcpy_h2d(gs[devs[i]], BYTES, 3); });
    for (auto& t : th) t.join();
    std::string s; double sum = 0;
    for (size_t i = 0; i < devs.size(); ++i) { s += std::to_string(devs[i]) + ":" + std::to_string((int)r[i]) + " "; sum += r[i]; }
    std::printf("concurrent %s [%s] sum %.1f GB/s\n", zc ? "zc" : "memcpy", s.c_str(), sum);
  };
  std::vector<int> all; for (int d = 0; d < n; ++d) all.push_back(d);
  concurrent(all, false);
  concurrent(all, true);
  for (int j = 1; j < n; ++j) concurrent({0, j}, false);
  if (n >= 4) { concurrent({0, 1, 2, 3}, true); }
  if (n >= 8) { concurrent({0, 1, 2, 3}, false); concurrent({4, 5, 6, 7}, false); concurrent({0, 2, 4, 6}, false); }
  // 3. peer
  if (n >= 2) {
    for (int a = 0; a < n; ++a) for (int b = 0; b < n; ++b) if (a != b) {
      int can; CK(cudaDeviceCanAccessPeer(&can, a, b));
      if (can) { CK(cudaSetDevice(a)); cudaError_t e = cudaDeviceEnablePeerAccess(b, 0); if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e); cudaGetLastError(); }
    }
    // memcpyPeer 1->0
    CK(cudaSetDevice(1));
    cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    double best = 1e30;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(a, gs[1].s));
      CK(cudaMemcpyPeerAsync(gs[0].dev_buf, 0, gs[1].dev_buf, 1, BYTES, gs[1].s));
      CK(cudaEventRecord(b, gs[1].s)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); best = std::min(best, (double)ms);
    }
    std::printf("memcpyPeer 1->0: %.1f GB/s\n", BYTES / (best * 1e-3) / 1e9);
    // fused: dev1 zero-copy reads its pinned host, stores into dev0 memory (peer)
    for (int grid : {296, 592}) {
      double zc = time_zc(gs[1], BYTES, grid, 256, 4, 0, gs[0].dev_buf);
      std::printf("fused host->dev1 SM->peer dev0 grid %d: %.1f GB/s\n", grid, zc);
    }
    for (int grid : {296, 592}) {
      double zc = time_zc(gs[1], BYTES, grid, 256, 4, 2304, gs[0].dev_buf);
      std::printf("fused-chunk host->dev1 SM->peer dev0 grid %d: %.1f GB/s\n", grid, zc);
    }
    // concurrent: dev0 zc own host + dev1 pushes into dev0 (the 1P1D dual path)
    {
      std::vector<double> r(2);
      std::thread t0([&] { r[0] = time_zc(gs[0], BYTES, 592, 256, 3); });
      std::thread t1([&] { r[1] = time_zc(gs[1], BYTES, 592, 256, 3, 0, (char*)gs[0].dev_buf); });
      t0.join(); t1.join();
      std::printf("dual 1P1D: pe zc %.1f + de push %.1f = %.1f GB/s\n", r[0], r[1], r[0] + r[1]);
    }
  }
  std::printf("done\n");
  return 0;
}
