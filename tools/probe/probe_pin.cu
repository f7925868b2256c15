// pinning strategies for a large host image
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char** argv) {
  size_t gib = argc > 1 ? atol(argv[1]) : 16;
  size_t n = gib << 30;
  cudaFree(0);
  double t = now(); void* p = nullptr; cudaHostAlloc(&p, n, cudaHostAllocDefault); printf("cudaHostAlloc %zu GiB: %.2fs\n", gib, now() - t); cudaFreeHost(p);
  // mmap + THP + parallel touch + register
  t = now();
  void* m = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
  madvise(m, n, MADV_HUGEPAGE);
  double t1 = now();
  unsigned th = std::thread::hardware_concurrency();
  std::vector<std::thread> pool;
  for (unsigned i = 0; i < th; ++i) pool.emplace_back([&, i] { size_t a = n * i / th, b = n * (i + 1) / th; for (size_t o = a; o < b; o += 4096) ((volatile char*)m)[o] = 0; });
  for (auto& x : pool) x.join();
  double t2 = now();
  cudaError_t e = cudaHostRegister(m, n, cudaHostRegisterDefault);
  double t3 = now();
  printf("mmap+THP: madvise %.3fs touch(%u thr) %.2fs register %.2fs (%s) total %.2fs\n", t1 - t, th, t2 - t1, t3 - t2, cudaGetErrorString(e), t3 - t);
  // bandwidth check D2H into registered memory
  void* d; cudaMalloc(&d, 1ull << 30);
  cudaStream_t s; cudaStreamCreate(&s);
  t = now(); for (int i = 0; i < 8; ++i) cudaMemcpyAsync((char*)m + ((size_t)i << 30), d, 1ull << 30, cudaMemcpyDeviceToHost, s); cudaStreamSynchronize(s);
  printf("D2H into registered THP memory: %.1f GB/s\n", 8.0 * (1ull << 30) / (now() - t) / 1e9);
  t = now(); cudaHostUnregister(m); munmap(m, n); printf("unregister+munmap %.2fs\n", now() - t);
  // without THP, MAP_POPULATE
  t = now();
  m = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_POPULATE, -1, 0);
  t1 = now(); e = cudaHostRegister(m, n, cudaHostRegisterDefault);
  printf("mmap POPULATE %.2fs register %.2fs (%s)\n", t1 - t, now() - t1, cudaGetErrorString(e));

  system("cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag");
  return 0;
}
