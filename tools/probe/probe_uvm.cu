// UVM residence-restore strategies for C3 (16 GiB managed, alternating 1 MiB runs)
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
__global__ void write_runs(char* p, size_t n, size_t run, int which) {
  // write every other run (which = 0: even runs, 1: odd runs)
  size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x * 16)
    if (((i / run) & 1) == (size_t)which) *reinterpret_cast<uint4*>(p + i) = make_uint4(1, 2, 3, 4);
}
__global__ void read_all(const char* p, size_t n, unsigned long long* sink) {
  unsigned long long s = 0;
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16; i < n; i += (size_t)gridDim.x * blockDim.x * 16)
    s += reinterpret_cast<const uint4*>(p + i)->x;
  if (s == 42) *sink = s;
}
int main() {
  const size_t N = 4ull << 30, RUN = 1 << 20;  // 4 GiB per test
  int dev = 0; cudaSetDevice(0); cudaFree(0);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  cudaStream_t st; cudaStreamCreate(&st);
  auto host_fill = [&](char* p, int which) {
    unsigned T = 16; std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) pool.emplace_back([=] { for (size_t r = t; r < N / RUN; r += T) if ((r & 1) == (size_t)which) memset(p + r * RUN, 7, RUN); });
    for (auto& x : pool) x.join();
  };
  // A: prefetch per run (device runs even, host runs odd)
  { char* p; cudaMallocManaged(&p, N); double t0 = now();
    for (size_t r = 0; r < N / RUN; ++r) cudaMemPrefetchAsync(p + r * RUN, RUN, (r & 1) ? cudaCpuDeviceId : dev, st);
    cudaStreamSynchronize(st); printf("A per-run prefetch (%zu calls): %.3fs\n", N / RUN, now() - t0); cudaFree(p); }
  // B: GPU first-touch writes even runs + CPU first-touch odd runs (concurrently)
  { char* p; cudaMallocManaged(&p, N); double t0 = now();
    write_runs<<<148 * 8, 256, 0, st>>>(p, N, RUN, 0);
    host_fill(p, 1); cudaStreamSynchronize(st); printf("B first-touch GPU even + CPU odd: %.3fs\n", now() - t0);
    // read back all from the GPU with AccessedBy set: remote reads of host runs
    cudaMemAdvise(p, N, cudaMemAdviseSetAccessedBy, dev);
    t0 = now(); read_all<<<148 * 8, 256, 0, st>>>(p, N, sink); cudaStreamSynchronize(st);
    printf("   GPU read all w/ AccessedBy: %.3fs (%.1f GB/s)\n", now() - t0, N / (now() - t0) / 1e9);
    t0 = now(); read_all<<<148 * 8, 256, 0, st>>>(p, N, sink); cudaStreamSynchronize(st);
    printf("   again: %.3fs\n", now() - t0);
    cudaMemAdvise(p, N, cudaMemAdviseUnsetAccessedBy, dev);
    t0 = now(); read_all<<<148 * 8, 256, 0, st>>>(p, N, sink); cudaStreamSynchronize(st);
    printf("   GPU read all w/o AccessedBy (migrating): %.3fs\n", now() - t0);
    cudaFree(p); }
  // C: advise PreferredLocation per run, then first touch
  { char* p; cudaMallocManaged(&p, N); double t0 = now();
    for (size_t r = 0; r < N / RUN; ++r) cudaMemAdvise(p + r * RUN, RUN, cudaMemAdviseSetPreferredLocation, (r & 1) ? cudaCpuDeviceId : dev);
    double t1 = now();
    write_runs<<<148 * 8, 256, 0, st>>>(p, N, RUN, 0); host_fill(p, 1); cudaStreamSynchronize(st);
    printf("C advise per run %.3fs + first touch %.3fs\n", t1 - t0, now() - t1); cudaFree(p); }
  // D: whole prefetch to device then CPU fill odd runs (migrating back)
  { char* p; cudaMallocManaged(&p, N); double t0 = now();
    cudaMemPrefetchAsync(p, N, dev, st); cudaStreamSynchronize(st); double t1 = now();
    host_fill(p, 1); printf("D prefetch whole to GPU %.3fs + CPU fill odd %.3fs\n", t1 - t0, now() - t1); cudaFree(p); }
  return 0;
}
