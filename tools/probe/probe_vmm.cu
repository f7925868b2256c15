// Where a cold arena map spends its time, and whether VMM calls wait for
// copies in flight (the cold refill's ordering question):
//   1. cuMemCreate / cuMemMap / cuMemSetAccess of N GiB, one handle and 2 GiB handles;
//   2. the same map issued while a 4 GiB H2D copy is in flight on another
//      stream: does the map call return before the copy completes?
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

static double now() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
#define CK(x)                                                        \
  do {                                                               \
    CUresult r_ = (x);                                               \
    if (r_ != CUDA_SUCCESS) {                                        \
      std::printf("FAIL %s = %d at line %d\n", #x, int(r_), __LINE__); \
      std::exit(1);                                                  \
    }                                                                \
  } while (0)

struct Timing {
  double create = 0, map = 0, access = 0, unmap = 0, release = 0;
};

static Timing map_range(CUdeviceptr va, size_t bytes, size_t piece, bool release_after) {
  Timing t;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  CUmemAccessDesc ad = {};
  ad.location = prop.location;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  std::vector<CUmemGenericAllocationHandle> hs;
  for (size_t o = 0; o < bytes; o += piece) {
    const size_t n = std::min(piece, bytes - o);
    CUmemGenericAllocationHandle h;
    double t0 = now();
    CK(cuMemCreate(&h, n, &prop, 0));
    double t1 = now();
    CK(cuMemMap(va + o, n, 0, h, 0));
    double t2 = now();
    CK(cuMemSetAccess(va + o, n, &ad, 1));
    double t3 = now();
    t.create += t1 - t0;
    t.map += t2 - t1;
    t.access += t3 - t2;
    hs.push_back(h);
  }
  if (release_after) {
    double t0 = now();
    CK(cuMemUnmap(va, bytes));
    double t1 = now();
    for (auto h : hs) CK(cuMemRelease(h));
    t.unmap = t1 - t0;
    t.release = now() - t1;
  }
  return t;
}

int main(int argc, char** argv) {
  const size_t gib = argc > 1 ? std::atol(argv[1]) : 100;
  const size_t bytes = gib << 30;
  cudaSetDevice(0);
  cudaFree(0);
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, bytes + (8ull << 30), 2 << 20, 0, 0));
  for (size_t piece : {bytes, size_t(8) << 30, size_t(2) << 30}) {
    Timing t = map_range(va, bytes, piece, true);
    std::printf("%zu GiB in %zu GiB handles: create %.1f map %.1f access %.1f | unmap %.1f release %.1f ms\n",
                gib, piece >> 30, t.create, t.map, t.access, t.unmap, t.release);
  }
  // a 4 GiB H2D in flight while mapping a fresh 8 GiB range
  const size_t cb = 4ull << 30;
  void* host;
  cudaHostAlloc(&host, cb, 0);
  void* dev;
  cudaMalloc(&dev, cb);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double t0 = now();
    cudaEventRecord(e0, st);
    cudaMemcpyAsync(dev, host, cb, cudaMemcpyHostToDevice, st);
    cudaEventRecord(e1, st);
    double t1 = now();
    Timing t = map_range(va, 8ull << 30, 8ull << 30, false);
    double t2 = now();
    cudaEventSynchronize(e1);
    double t3 = now();
    float copy_ms = 0;
    cudaEventElapsedTime(&copy_ms, e0, e1);
    std::printf("map 8 GiB beside a 4 GiB H2D: enqueue %.2f, map calls %.1f ms (create %.1f map %.1f access %.1f), "
                "copy done at +%.1f ms, copy %.1f ms\n",
                t1 - t0, t2 - t1, t.create, t.map, t.access, t3 - t0, copy_ms);
    CK(cuMemUnmap(va, 8ull << 30));
    // (handles leaked on purpose: the probe exits)
  }
  return 0;
}
