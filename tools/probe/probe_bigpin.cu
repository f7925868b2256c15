// D2H / H2D rate across a large THP-backed registered host image, per 8 GiB
// segment, to see whether the link or host DRAM binds a 120 GiB drain.
//   probe_bigpin <GiB> [piece_MiB]
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static long anon_huge_kb() {
  FILE* f = fopen("/proc/meminfo", "r");
  char line[256];
  long v = -1;
  while (f && fgets(line, sizeof line, f))
    if (!strncmp(line, "AnonHugePages:", 14)) v = atol(line + 14);
  if (f) fclose(f);
  return v;
}
int main(int argc, char** argv) {
  size_t gib = argc > 1 ? atol(argv[1]) : 32;
  size_t piece = (argc > 2 ? atol(argv[2]) : 16) << 20;
  size_t n = gib << 30;
  cudaFree(0);
  long h0 = anon_huge_kb();
  double t = now();
  char* m = (char*)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
  madvise(m, n, MADV_HUGEPAGE);
  unsigned th = std::thread::hardware_concurrency();
  std::vector<std::thread> pool;
  for (unsigned i = 0; i < th; ++i)
    pool.emplace_back([&, i] {
      size_t a = n * i / th, b = n * (i + 1) / th;
      for (size_t o = a; o < b; o += 4096) ((volatile char*)m)[o] = 0;
    });
  for (auto& x : pool) x.join();
  double t1 = now();
  cudaError_t e = cudaHostRegister(m, n, cudaHostRegisterDefault);
  printf("touch %.2fs register %.2fs (%s); AnonHugePages +%ld MiB of %zu\n", t1 - t, now() - t1,
         cudaGetErrorString(e), (anon_huge_kb() - h0) >> 10, n >> 20);
  const size_t dev_bytes = 1ull << 30;
  char* d;
  cudaMalloc(&d, dev_bytes);
  cudaMemset(d, 1, dev_bytes);
  cudaStream_t s[2];
  cudaStreamCreateWithFlags(&s[0], cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s[1], cudaStreamNonBlocking);
  const size_t seg = 8ull << 30;
  for (int dir = 0; dir < 2; ++dir) {
    printf("%s per 8 GiB segment (GB/s):", dir ? "H2D" : "D2H");
    double tot_t = 0;
    for (size_t a = 0; a < n; a += seg) {
      size_t b = a + seg < n ? a + seg : n;
      double t0 = now();
      int k = 0;
      for (size_t o = a; o < b; o += piece, ++k) {
        size_t len = piece < b - o ? piece : b - o;
        if (dir == 0)
          cudaMemcpyAsync(m + o, d + (o % dev_bytes), len, cudaMemcpyDeviceToHost, s[k & 1]);
        else
          cudaMemcpyAsync(d + (o % dev_bytes), m + o, len, cudaMemcpyHostToDevice, s[k & 1]);
      }
      cudaStreamSynchronize(s[0]);
      cudaStreamSynchronize(s[1]);
      double dt = now() - t0;
      tot_t += dt;
      printf(" %.1f", (b - a) / dt / 1e9);
      fflush(stdout);
    }
    printf("  | whole %.1f GB/s\n", n / tot_t / 1e9);
  }
  // host DRAM write bandwidth (all threads, memset) as the other candidate bound
  pool.clear();
  t = now();
  for (unsigned i = 0; i < th; ++i)
    pool.emplace_back([&, i] { size_t a = n * i / th, b = n * (i + 1) / th; memset(m + a, 7, b - a); });
  for (auto& x : pool) x.join();
  printf("host memset %u threads: %.1f GB/s\n", th, n / (now() - t) / 1e9);
  printf("cuda error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
