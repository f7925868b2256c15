// Box probe: PCIe D2H/H2D bandwidth vs size/alignment/streams, fixed-VA VMM reserve.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

typedef CUresult (*PFN_reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PFN_create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
typedef CUresult (*PFN_map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
typedef CUresult (*PFN_setaccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
typedef CUresult (*PFN_gran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main() {
  CK(cudaSetDevice(0));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("dev %s sms %d l2 %d MB memclk %d busw %d\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.memoryClockRate, p.memoryBusWidth);
  int pma = 0; cudaDeviceGetAttribute(&pma, cudaDevAttrPageableMemoryAccess, 0);
  int cma = 0; cudaDeviceGetAttribute(&cma, cudaDevAttrConcurrentManagedAccess, 0);
  int ae = 0; cudaDeviceGetAttribute(&ae, cudaDevAttrAsyncEngineCount, 0);
  printf("pageableMemoryAccess %d concurrentManagedAccess %d asyncEngines %d\n", pma, cma, ae);

  // VMM fixed VA
  PFN_reserve reserve; PFN_create create; PFN_map map; PFN_setaccess setaccess; PFN_gran gran;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuMemAddressReserve", (void**)&reserve, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuMemCreate", (void**)&create, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuMemMap", (void**)&map, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuMemSetAccess", (void**)&setaccess, cudaEnableDefault, &q));
  CK(cudaGetDriverEntryPoint("cuMemGetAllocationGranularity", (void**)&gran, cudaEnableDefault, &q));
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED; prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE; prop.location.id = 0;
  size_t g = 0; gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM); printf("vmm granularity %zu\n", g);
  CUdeviceptr va = 0; size_t vsz = 130ull << 30;
  CUresult r = reserve(&va, vsz, 0, (CUdeviceptr)0x0D0000000000ull, 0);
  printf("reserve rc %d va %llx (want d0000000000)\n", (int)r, (unsigned long long)va);
  double t0 = now();
  CUmemGenericAllocationHandle h; r = create(&h, 120ull << 30, &prop, 0); printf("create 120GiB rc %d %.3fs\n", (int)r, now() - t0);
  t0 = now();
  r = map(va, 120ull << 30, 0, h, 0); printf("map rc %d %.3fs\n", (int)r, now() - t0);
  CUmemAccessDesc ad = {}; ad.location = prop.location; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  t0 = now();
  r = setaccess(va, 120ull << 30, &ad, 1); printf("setaccess rc %d %.3fs\n", (int)r, now() - t0);
  t0 = now(); CK(cudaMemset((void*)va, 0, 120ull << 30)); CK(cudaDeviceSynchronize()); printf("memset 120GiB %.3fs\n", now() - t0);

  // pinned host
  size_t HB = 16ull << 30;
  t0 = now(); uint8_t* hp = nullptr; CK(cudaHostAlloc(&hp, HB + 4096, cudaHostAllocDefault)); printf("cudaHostAlloc 16GiB %.3fs\n", now() - t0);
  t0 = now(); memset(hp, 1, HB); printf("host memset 16GiB %.3fs\n", now() - t0);
  uint8_t* dp = (uint8_t*)va;
  cudaStream_t s[4]; for (int i = 0; i < 4; ++i) CK(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  size_t sizes[] = {64 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20};
  for (int dir = 0; dir < 2; ++dir) for (size_t sz : sizes) for (int nst : {1, 2, 4}) for (int mis : {0, 3}) {
    size_t total = 8ull << 30; size_t n = total / sz;
    CK(cudaDeviceSynchronize());
    double a = now();
    for (size_t i = 0; i < n; ++i) {
      uint8_t* h = hp + i * sz + mis; uint8_t* d = dp + i * sz;
      if (dir == 0) CK(cudaMemcpyAsync(h, d, sz, cudaMemcpyDeviceToHost, s[i % nst]));
      else CK(cudaMemcpyAsync(d, h, sz, cudaMemcpyHostToDevice, s[i % nst]));
    }
    CK(cudaDeviceSynchronize());
    double b = now();
    printf("%s sz %8zu streams %d mis %d : %.2f GB/s\n", dir ? "H2D" : "D2H", sz, nst, mis, total / (b - a) / 1e9);
  }
  // bidirectional concurrently
  {
    size_t sz = 64 << 20; size_t total = 8ull << 30; size_t n = total / sz;
    CK(cudaDeviceSynchronize()); double a = now();
    for (size_t i = 0; i < n; ++i) {
      CK(cudaMemcpyAsync(hp + i * sz, dp + i * sz, sz, cudaMemcpyDeviceToHost, s[0]));
      CK(cudaMemcpyAsync(dp + (64ull << 30) + i * sz, hp + (8ull << 30) + i * sz, sz, cudaMemcpyHostToDevice, s[1]));
    }
    CK(cudaDeviceSynchronize()); double b = now();
    printf("bidir 64MiB each way: %.2f GB/s per direction\n", total / (b - a) / 1e9);
  }
  // device-side D2D copy bandwidth
  {
    size_t sz = 8ull << 30;
    CK(cudaEventRecord(e0, s[0]));
    for (int i = 0; i < 5; ++i) CK(cudaMemcpyAsync(dp + (32ull << 30), dp, sz, cudaMemcpyDeviceToDevice, s[0]));
    CK(cudaEventRecord(e1, s[0])); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("D2D 8GiB x5: %.1f GB/s (r+w)\n", 2.0 * 5 * sz / (ms * 1e-3) / 1e9);
  }
  printf("done\n");
  return 0;
}
