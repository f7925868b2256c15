#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
typedef CUresult (*PFN_reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PFN_free)(CUdeviceptr, size_t);
int main() {
  cudaFree(0);
  PFN_reserve reserve; PFN_free fr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuMemAddressReserve", (void**)&reserve, cudaEnableDefault, &q);
  cudaGetDriverEntryPoint("cuMemAddressFree", (void**)&fr, cudaEnableDefault, &q);
  size_t sizes[] = {4ull << 20, 16ull << 20, 1ull << 30, 130ull << 30};
  size_t aligns[] = {0, 2ull << 20};
  for (size_t sz : sizes) for (size_t al : aligns) {
    CUdeviceptr va = 0;
    CUresult r = reserve(&va, sz, al, (CUdeviceptr)0x0D0000000000ull, 0);
    printf("size %zu align %zu -> rc %d va %llx\n", sz, al, (int)r, (unsigned long long)va);
    if (r == CUDA_SUCCESS) fr(va, sz);
  }
  // flags: CU_MEM_ADDRESS_RESERVE? none in 12.9 except 0
  return 0;
}
