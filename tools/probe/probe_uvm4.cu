// C3 refill, device side: populate the device-resident runs of fresh managed
// memory (16 GiB, alternating 1 MiB runs; the even runs, 8 GiB, are meant to
// end up device-resident) by
//   gft   kernel first touch (GPU page faults; what the scatter does today)
//   h2d   cudaMemcpyAsync from pinned host straight into each even run
//   h2d+  the same with the odd runs copied in by 16 host threads meanwhile
// then a read kernel over the even runs shows where they ended up (fast =
// device-resident; slow = the read faults / migrates).
#include <cuda_runtime.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void write_runs(char* p, size_t n, size_t run, int which) {
  size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x * 16)
    if (((i / run) & 1) == (size_t)which) *reinterpret_cast<uint4*>(p + i) = make_uint4(1, 2, 3, 4);
}

__global__ void read_runs(const char* p, size_t n, size_t run, int which, unsigned* out) {
  unsigned acc = 0;
  size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 16;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x * 16)
    if (((i / run) & 1) == (size_t)which) acc ^= reinterpret_cast<const uint4*>(p + i)->x;
  if (acc == 0x12345678u) *out = acc;
}

int main(int argc, char** argv) {
  const size_t N = (argc > 1 ? atol(argv[1]) : 16ull) << 30, RUN = 1 << 20, R = N / RUN;
  cudaSetDevice(0);
  cudaFree(0);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  char* src;
  cudaHostAlloc(&src, N / 2, 0);
  memset(src, 3, N / 2);
  unsigned* d_out;
  cudaMalloc(&d_out, 4);
  auto host_copy = [&](char* p) {
    std::vector<std::thread> pool;
    std::atomic<size_t> next{1};
    for (unsigned t = 0; t < 16; ++t)
      pool.emplace_back([&] {
        for (size_t r; (r = next.fetch_add(2)) < R;) memcpy(p + r * RUN, src + (r / 2) * RUN, RUN);
      });
    for (auto& x : pool) x.join();
  };
  auto check = [&](char* p) {
    double t0 = now();
    read_runs<<<148 * 8, 256, 0, st>>>(p, N, RUN, 0, d_out);
    cudaStreamSynchronize(st);
    double t1 = now();
    read_runs<<<148 * 8, 256, 0, st>>>(p, N, RUN, 0, d_out);
    cudaStreamSynchronize(st);
    return std::make_pair(t1 - t0, now() - t1);
  };
  for (int rep = 0; rep < 2; ++rep) {
    {
      char* p;
      cudaMallocManaged(&p, N);
      double t0 = now();
      write_runs<<<148 * 8, 256, 0, st>>>(p, N, RUN, 0);
      cudaStreamSynchronize(st);
      double t1 = now();
      auto c = check(p);
      printf("gft  even runs %.3fs | read after %.4fs, again %.4fs\n", t1 - t0, c.first, c.second);
      cudaFree(p);
    }
    {
      char* p;
      cudaMallocManaged(&p, N);
      double t0 = now();
      for (size_t r = 0; r < R; r += 2)
        cudaMemcpyAsync(p + r * RUN, src + (r / 2) * RUN, RUN, cudaMemcpyHostToDevice, st);
      double t1 = now();
      cudaStreamSynchronize(st);
      double t2 = now();
      auto c = check(p);
      printf("h2d  even runs calls %.3fs done %.3fs (%.1f GB/s) err=%s | read after %.4fs, again %.4fs\n",
             t1 - t0, t2 - t0, N / 2 / (t2 - t0) / 1e9, cudaGetErrorString(cudaGetLastError()),
             c.first, c.second);
      cudaFree(p);
    }
    {
      char* p;
      cudaMallocManaged(&p, N);
      double t0 = now(), tg = 0;
      std::thread g([&] {
        for (size_t r = 0; r < R; r += 2)
          cudaMemcpyAsync(p + r * RUN, src + (r / 2) * RUN, RUN, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
        tg = now() - t0;
      });
      host_copy(p);
      double th = now() - t0;
      g.join();
      double t1 = now();
      auto c = check(p);
      printf("h2d+ gpu %.3fs || cpu16 %.3fs -> %.3fs | read after %.4fs, again %.4fs\n", tg, th,
             t1 - t0, c.first, c.second);
      cudaFree(p);
    }
    {
      char* p;
      cudaMallocManaged(&p, N);
      double t0 = now(), tg = 0;
      std::thread g([&] {
        write_runs<<<148 * 8, 256, 0, st>>>(p, N, RUN, 0);
        cudaStreamSynchronize(st);
        tg = now() - t0;
      });
      host_copy(p);
      double th = now() - t0;
      g.join();
      double t1 = now();
      auto c = check(p);
      printf("gft+ gpu %.3fs || cpu16 %.3fs -> %.3fs | read after %.4fs, again %.4fs\n", tg, th,
             t1 - t0, c.first, c.second);
      cudaFree(p);
    }
  }
  return 0;
}
