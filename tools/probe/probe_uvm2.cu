// C3 refill first-touch alternatives (16 GiB managed, alternating 1 MiB runs):
//   B  GPU first-touch of the device runs || CPU first-touch of the host runs (current)
//   D  whole-allocation prefetch to the CPU, then B (host runs need no faults)
//   E  whole-allocation prefetch to the GPU, then B (device runs need no faults)
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
__global__ void write_runs(char* p, size_t n, size_t run, int which) {
  size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x * 16)
    if (((i / run) & 1) == (size_t)which) *reinterpret_cast<uint4*>(p + i) = make_uint4(1, 2, 3, 4);
}
int main(int argc, char** argv) {
  const size_t N = (argc > 1 ? atol(argv[1]) : 16ull) << 30, RUN = 1 << 20;
  cudaSetDevice(0); cudaFree(0);
  cudaStream_t st; cudaStreamCreate(&st);
  auto host_fill = [&](char* p, int which) {
    unsigned T = 16; std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t) pool.emplace_back([=] { for (size_t r = t; r < N / RUN; r += T) if ((r & 1) == (size_t)which) memset(p + r * RUN, 7, RUN); });
    for (auto& x : pool) x.join();
  };
  for (int mode = 0; mode < 3; ++mode) {
    char* p; cudaMallocManaged(&p, N);
    double t0 = now();
    if (mode == 1) cudaMemPrefetchAsync(p, N, cudaCpuDeviceId, st);
    if (mode == 2) cudaMemPrefetchAsync(p, N, 0, st);
    cudaStreamSynchronize(st);
    double t1 = now();
    write_runs<<<148 * 8, 256, 0, st>>>(p, N, RUN, 0);
    double tg0 = now();
    host_fill(p, 1);
    double th = now();
    cudaStreamSynchronize(st);
    double t2 = now();
    printf("%s: prefetch %.3fs, then GPU even runs || CPU odd runs %.3fs (cpu part %.3fs) total %.3fs  err=%s\n",
           mode == 0 ? "B none" : mode == 1 ? "D cpu-prefetch" : "E gpu-prefetch", t1 - t0, t2 - t1, th - tg0, t2 - t0,
           cudaGetErrorString(cudaGetLastError()));
    t0 = now(); cudaFree(p); printf("   cudaFree %.3fs\n", now() - t0);
  }
  return 0;
}
