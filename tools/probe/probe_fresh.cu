// Fresh-mapping probe: is the first write into freshly created and mapped
// VMM memory (cuMemCreate + cuMemMap + cuMemSetAccess, as a cold refill's
// arena) slower than a later one?  Times, on `gib` GiB mapped as one handle:
//   * a kernel storing 64 MiB blocks (first pass, second pass)
//   * H2D copies of 64 MiB pieces from page-locked memory (into fresh memory,
//     then again into the same memory)
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a probe_fresh.cu -lcuda -o probe_fresh
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::printf("%s failed: %s\n", #x, cudaGetErrorString(e_));              \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)
#define CU(x)                                                                  \
  do {                                                                         \
    CUresult r_ = (x);                                                         \
    if (r_ != CUDA_SUCCESS) {                                                  \
      std::printf("%s failed: %d\n", #x, int(r_));                             \
      std::exit(1);                                                            \
    }                                                                          \
  } while (0)

__global__ void k_store(uint4* p, size_t words) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < words;
       i += size_t(gridDim.x) * blockDim.x)
    p[i] = make_uint4(1, 2, 3, 4);
}

struct Mapping {
  CUdeviceptr va = 0;
  CUmemGenericAllocationHandle h = 0;
  size_t n = 0;
};

Mapping map_fresh(size_t n) {
  Mapping m;
  m.n = n;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = 0;
  CU(cuMemAddressReserve(&m.va, n, 0, 0, 0));
  CU(cuMemCreate(&m.h, n, &prop, 0));
  CU(cuMemMap(m.va, n, 0, m.h, 0));
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CU(cuMemSetAccess(m.va, n, &acc, 1));
  return m;
}

void unmap(Mapping& m) {
  CU(cuMemUnmap(m.va, m.n));
  CU(cuMemRelease(m.h));
  CU(cuMemAddressFree(m.va, m.n));
}

int main(int argc, char** argv) {
  const size_t gib = argc > 1 ? std::atoi(argv[1]) : 8;
  const size_t n = gib << 30, blk = 64ull << 20;
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  char* h = nullptr;
  CK(cudaHostAlloc(&h, n, cudaHostAllocDefault));
  for (size_t i = 0; i < n; i += 4096) h[i] = 1;
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto timed = [&](auto&& body) {
    CK(cudaEventRecord(a, st));
    body();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    return ms;
  };
  for (int round = 0; round < 2; ++round) {
    Mapping m = map_fresh(n);
    // kernel stores, 64 MiB at a time: first touch then second pass
    float first = 0, second = 0, first_max = 0;
    for (size_t off = 0; off < n; off += blk) {
      const float t = timed([&] { k_store<<<592, 512, 0, st>>>(reinterpret_cast<uint4*>(m.va + off), blk / 16); });
      first += t;
      if (t > first_max) first_max = t;
    }
    for (size_t off = 0; off < n; off += blk)
      second += timed([&] { k_store<<<592, 512, 0, st>>>(reinterpret_cast<uint4*>(m.va + off), blk / 16); });
    const size_t blocks = n / blk;
    std::printf("round %d kernel store per 64 MiB: fresh %.1f us (max %.1f), again %.1f us\n", round,
                1e3f * first / blocks, 1e3f * first_max, 1e3f * second / blocks);
    unmap(m);
    m = map_fresh(n);
    const float h2d_fresh = timed([&] {
      for (size_t off = 0; off < n; off += blk)
        CK(cudaMemcpyAsync(reinterpret_cast<void*>(m.va + off), h + off, blk, cudaMemcpyHostToDevice, st));
    });
    const float h2d_again = timed([&] {
      for (size_t off = 0; off < n; off += blk)
        CK(cudaMemcpyAsync(reinterpret_cast<void*>(m.va + off), h + off, blk, cudaMemcpyHostToDevice, st));
    });
    std::printf("round %d H2D %zu GiB in 64 MiB pieces: fresh %.2f GB/s, again %.2f GB/s\n", round, gib,
                n / (h2d_fresh * 1e6), n / (h2d_again * 1e6));
    // a fresh mapping first written by H2D, then a kernel store pass over it
    unmap(m);
    m = map_fresh(n);
    float after_h2d = 0;
    timed([&] {
      for (size_t off = 0; off < n; off += blk)
        CK(cudaMemcpyAsync(reinterpret_cast<void*>(m.va + off), h + off, blk, cudaMemcpyHostToDevice, st));
    });
    for (size_t off = 0; off < n; off += blk)
      after_h2d += timed([&] { k_store<<<592, 512, 0, st>>>(reinterpret_cast<uint4*>(m.va + off), blk / 16); });
    std::printf("round %d kernel store per 64 MiB after an H2D touched it: %.1f us\n", round,
                1e3f * after_h2d / blocks);
    unmap(m);
  }
  return 0;
}
