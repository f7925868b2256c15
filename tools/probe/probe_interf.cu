// Does PCIe copy traffic slow any HBM-bound copy kernel, or only the pack?
// Times device->device copy kernels (64 MiB per launch) alone and beside a
// continuous D2H (or H2D) of 16 MiB pieces on another stream.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int kWords, bool kHint>
__global__ void __launch_bounds__(256) copy_tiles(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t words) {
  const size_t tile = size_t(blockIdx.x) * 256 * kWords;
  uint4 v[kWords];
#pragma unroll
  for (int k = 0; k < kWords; ++k) {
    const size_t w = tile + threadIdx.x + k * 256;
    if (w < words) {
      if (kHint) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(src + w));
      else v[k] = src[w];
    }
  }
#pragma unroll
  for (int k = 0; k < kWords; ++k) {
    const size_t w = tile + threadIdx.x + k * 256;
    if (w < words) {
      if (kHint) asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(dst + w), "r"(v[k].x), "r"(v[k].y), "r"(v[k].z), "r"(v[k].w));
      else dst[w] = v[k];
    }
  }
}

// persistent grid-stride copy
template <int kUnroll>
__global__ void __launch_bounds__(512) copy_persist(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t words) {
  const size_t stride = size_t(gridDim.x) * 512 * kUnroll;
  for (size_t base = size_t(blockIdx.x) * 512 * kUnroll + threadIdx.x; base < words; base += stride) {
    uint4 v[kUnroll];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) if (base + k * 512 < words) v[k] = src[base + k * 512];
#pragma unroll
    for (int k = 0; k < kUnroll; ++k) if (base + k * 512 < words) dst[base + k * 512] = v[k];
  }
}

int main() {
  const size_t W = 64ull << 20, N = 64;  // 64 launches over 4 GiB of source
  uint8_t *src, *dst, *stage, *host;
  CK(cudaMalloc(&src, W * N));
  CK(cudaMalloc(&dst, W * 4));
  CK(cudaMalloc(&stage, 256ull << 20));
  CK(cudaHostAlloc(&host, 256ull << 20, 0));
  CK(cudaMemset(src, 1, W * N));
  cudaStream_t sk, sc;
  CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<cudaEvent_t> e0(N), e1(N);
  for (size_t i = 0; i < N; ++i) { cudaEventCreate(&e0[i]); cudaEventCreate(&e1[i]); }
  const size_t words = W / 16;
  auto run = [&](const char* name, auto launch) {
    for (int mode = 0; mode < 3; ++mode) {  // 0 alone, 1 beside D2H, 2 beside H2D
      CK(cudaDeviceSynchronize());
      if (mode) for (int i = 0; i < 200; ++i) {
        if (mode == 1) CK(cudaMemcpyAsync(host + (i % 16) * (16 << 20), stage + (i % 16) * (16 << 20), 16 << 20, cudaMemcpyDeviceToHost, sc));
        else CK(cudaMemcpyAsync(stage + (i % 16) * (16 << 20), host + (i % 16) * (16 << 20), 16 << 20, cudaMemcpyHostToDevice, sc));
      }
      for (size_t i = 0; i < N; ++i) {
        cudaEventRecord(e0[i], sk);
        launch((const uint4*)(src + i * W), (uint4*)(dst + (i % 4) * W), words);
        cudaEventRecord(e1[i], sk);
      }
      CK(cudaDeviceSynchronize());
      std::vector<float> t(N);
      for (size_t i = 0; i < N; ++i) cudaEventElapsedTime(&t[i], e0[i], e1[i]);
      std::sort(t.begin(), t.end());
      const float med = t[N / 2] * 1000;
      printf("%-28s %-10s median %7.1f us  %6.0f GB/s (r+w)\n", name, mode == 0 ? "alone" : mode == 1 ? "+D2H" : "+H2D", med, 2.0 * W / (med * 1e3));
    }
  };
  run("tiles 16w (pack-like)", [&](const uint4* s, uint4* d, size_t n) { copy_tiles<16, false><<<unsigned((n + 4095) / 4096), 256, 0, sk>>>(s, d, n); });
  run("tiles 16w nc/cs hints", [&](const uint4* s, uint4* d, size_t n) { copy_tiles<16, true><<<unsigned((n + 4095) / 4096), 256, 0, sk>>>(s, d, n); });
  run("tiles 4w", [&](const uint4* s, uint4* d, size_t n) { copy_tiles<4, false><<<unsigned((n + 1023) / 1024), 256, 0, sk>>>(s, d, n); });
  run("persistent 148x2 u8", [&](const uint4* s, uint4* d, size_t n) { copy_persist<8><<<sms * 2, 512, 0, sk>>>(s, d, n); });
  run("persistent 148x4 u4", [&](const uint4* s, uint4* d, size_t n) { copy_persist<4><<<sms * 4, 512, 0, sk>>>(s, d, n); });
  run("cudaMemcpyAsync D2D", [&](const uint4* s, uint4* d, size_t n) { cudaMemcpyAsync(d, s, n * 16, cudaMemcpyDeviceToDevice, sk); });
  return 0;
}
