// Copy-engine probe: does spreading one big pinned transfer over several
// streams (so several copy engines) beat one stream?  D2H and H2D of `gib`
// GiB between device memory and one page-locked buffer, pieces handed out
// round-robin to S streams, best of 3 per (direction, S, piece).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a probe_ce.cu -o probe_ce
//   ./probe_ce [gib]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::printf("%s failed: %s\n", #x, cudaGetErrorString(e_));              \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

int main(int argc, char** argv) {
  const size_t gib = argc > 1 ? std::atoi(argv[1]) : 8;
  const size_t n = gib << 30;
  char *d = nullptr, *h = nullptr;
  CK(cudaMalloc(&d, n));
  CK(cudaHostAlloc(&h, n, cudaHostAllocDefault));
  CK(cudaMemset(d, 1, n));
  for (size_t i = 0; i < n; i += 4096) h[i] = 2;  // fault the host pages in
  std::vector<cudaStream_t> st(8);
  for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  int ces = 0;
  CK(cudaDeviceGetAttribute(&ces, cudaDevAttrAsyncEngineCount, 0));
  std::printf("async engines %d, %zu GiB per transfer\n", ces, gib);
  for (int dir = 0; dir < 3; ++dir) {
    for (size_t piece_mib : {16, 64}) {
      for (int S : {1, 2, 3, 4}) {
        const size_t piece = piece_mib << 20;
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
          CK(cudaDeviceSynchronize());
          CK(cudaEventRecord(a, st[0]));
          for (int s = 1; s < 8; ++s) CK(cudaStreamWaitEvent(st[s], a, 0));
          size_t k = 0;
          for (size_t off = 0; off < n; off += piece, ++k) {
            const size_t len = std::min(piece, n - off);
            if (dir == 2) {  // both directions at once: half the pieces each way
              if (k % 2) CK(cudaMemcpyAsync(h + off, d + off, len, cudaMemcpyDeviceToHost, st[(k / 2) % S]));
              else CK(cudaMemcpyAsync(d + off, h + off, len, cudaMemcpyHostToDevice, st[4 + (k / 2) % S]));
            } else if (dir == 0) {
              CK(cudaMemcpyAsync(h + off, d + off, len, cudaMemcpyDeviceToHost, st[k % S]));
            } else {
              CK(cudaMemcpyAsync(d + off, h + off, len, cudaMemcpyHostToDevice, st[k % S]));
            }
          }
          for (int s = 1; s < 8; ++s) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            CK(cudaEventRecord(e, st[s]));
            CK(cudaStreamWaitEvent(st[0], e, 0));
            CK(cudaEventDestroy(e));
          }
          CK(cudaEventRecord(b, st[0]));
          CK(cudaEventSynchronize(b));
          float ms = 0;
          CK(cudaEventElapsedTime(&ms, a, b));
          best = std::min(best, ms);
        }
        std::printf("%s piece %3zu MiB streams %d: %.2f GB/s%s\n",
                    dir == 0 ? "D2H " : dir == 1 ? "H2D " : "BOTH", piece_mib, S, n / (best * 1e6),
                    dir == 2 ? " (sum of both directions)" : "");
      }
    }
  }
  return 0;
}
