// C3 refill: ways to populate fresh managed memory with split residence
// (16 GiB, alternating 1 MiB runs: even runs device-resident, odd runs host).
// Host side: the odd runs get 8 GiB copied in from a pinned buffer.
//   cpuT     first-touch memcpy with T threads
//   popT     madvise(MADV_POPULATE_WRITE) per run (T threads), then memcpy
//   pfcpu    cudaMemPrefetchAsync(run -> CPU) per run, then memcpy (16 threads)
// Device side: the even runs get written by a kernel.
//   gft      kernel first touch (GPU page faults)
//   gpf      cudaMemPrefetchAsync(run -> GPU) per run, then the kernel
//   gpfth    the same prefetches issued from a second thread on its own stream
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void write_runs(char* p, size_t n, size_t run, int which) {
  size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x * 16)
    if (((i / run) & 1) == (size_t)which) *reinterpret_cast<uint4*>(p + i) = make_uint4(1, 2, 3, 4);
}

int main(int argc, char** argv) {
  const size_t N = (argc > 1 ? atol(argv[1]) : 16ull) << 30, RUN = 1 << 20, R = N / RUN;
  printf("nproc %ld\n", sysconf(_SC_NPROCESSORS_ONLN));
  cudaSetDevice(0);
  cudaFree(0);
  cudaStream_t st, st2;
  cudaStreamCreate(&st);
  cudaStreamCreate(&st2);
  char* src;
  cudaHostAlloc(&src, N / 2, 0);
  memset(src, 3, N / 2);
  auto threads = [&](unsigned T, auto fn) {
    std::vector<std::thread> pool;
    std::atomic<size_t> next{0};
    for (unsigned t = 0; t < T; ++t)
      pool.emplace_back([&] {
        for (size_t r; (r = next.fetch_add(2)) < R;) fn(r + 1);  // odd runs
      });
    for (auto& x : pool) x.join();
  };
  auto copy_in = [&](char* p, size_t r) { memcpy(p + r * RUN, src + (r / 2) * RUN, RUN); };
  auto fresh = [&]() {
    char* p;
    cudaMallocManaged(&p, N);
    return p;
  };
  auto release = [&](char* p) {
    double t0 = now();
    cudaFree(p);
    return now() - t0;
  };
  // host side
  for (unsigned T : {16u, 32u, 64u}) {
    char* p = fresh();
    double t0 = now();
    threads(T, [&](size_t r) { copy_in(p, r); });
    printf("cpu%u first-touch memcpy 8 GiB: %.3fs  (free %.2fs)\n", T, now() - t0, release(p));
  }
  for (unsigned T : {16u, 32u}) {
    char* p = fresh();
    double t0 = now();
    std::atomic<int> bad{0};
    threads(T, [&](size_t r) {
      if (madvise(p + r * RUN, RUN, MADV_POPULATE_WRITE)) bad = errno;
    });
    double t1 = now();
    threads(16, [&](size_t r) { copy_in(p, r); });
    printf("pop%u populate %.3fs (errno %d) + memcpy %.3fs = %.3fs (free %.2fs)\n", T, t1 - t0,
           bad.load(), now() - t1, now() - t0, release(p));
  }
  {
    char* p = fresh();
    double t0 = now();
    for (size_t r = 1; r < R; r += 2) cudaMemPrefetchAsync(p + r * RUN, RUN, cudaCpuDeviceId, st);
    cudaStreamSynchronize(st);
    double t1 = now();
    threads(16, [&](size_t r) { copy_in(p, r); });
    printf("pfcpu prefetch %.3fs + memcpy %.3fs = %.3fs  err=%s (free %.2fs)\n", t1 - t0, now() - t1,
           now() - t0, cudaGetErrorString(cudaGetLastError()), release(p));
  }
  // device side
  {
    char* p = fresh();
    double t0 = now();
    write_runs<<<148 * 8, 256, 0, st>>>(p, N, RUN, 0);
    cudaStreamSynchronize(st);
    printf("gft kernel first touch of even runs: %.3fs (free %.2fs)\n", now() - t0, release(p));
  }
  {
    char* p = fresh();
    double t0 = now();
    for (size_t r = 0; r < R; r += 2) cudaMemPrefetchAsync(p + r * RUN, RUN, 0, st);
    double t1 = now();
    cudaStreamSynchronize(st);
    double t2 = now();
    write_runs<<<148 * 8, 256, 0, st>>>(p, N, RUN, 0);
    cudaStreamSynchronize(st);
    printf("gpf per-run prefetch: calls %.3fs, done %.3fs, kernel %.3fs, total %.3fs err=%s (free %.2fs)\n",
           t1 - t0, t2 - t0, now() - t2, now() - t0, cudaGetErrorString(cudaGetLastError()), release(p));
  }
  {
    // both sides at once, the way a refill would: prefetch thread + kernel
    // after it, CPU threads copying the host runs meanwhile
    char* p = fresh();
    double t0 = now(), tg = 0;
    std::thread g([&] {
      for (size_t r = 0; r < R; r += 2) cudaMemPrefetchAsync(p + r * RUN, RUN, 0, st2);
      write_runs<<<148 * 8, 256, 0, st2>>>(p, N, RUN, 0);
      cudaStreamSynchronize(st2);
      tg = now() - t0;
    });
    threads(16, [&](size_t r) { copy_in(p, r); });
    double th = now() - t0;
    g.join();
    printf("both: gpu prefetch+kernel %.3fs || cpu16 first-touch %.3fs -> %.3fs (free %.2fs)\n", tg,
           th, now() - t0, release(p));
  }
  {
    char* p = fresh();
    double t0 = now(), tg = 0;
    std::thread g([&] {
      write_runs<<<148 * 8, 256, 0, st2>>>(p, N, RUN, 0);
      cudaStreamSynchronize(st2);
      tg = now() - t0;
    });
    threads(16, [&](size_t r) { copy_in(p, r); });
    double th = now() - t0;
    g.join();
    printf("both (no prefetch): gpu first touch %.3fs || cpu16 first-touch %.3fs -> %.3fs\n", tg, th,
           now() - t0);
    cudaFree(p);
  }
  return 0;
}
