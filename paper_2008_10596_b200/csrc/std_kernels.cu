// Standard kernel bodies (fixtures for workloads and tests; not the hot path).
// Compiled with -fmad=false: the reference builds with -ffp-contract=off
// (ref: proj/CMakeLists.txt:11) and its f32 sums must match bit for bit.
#include <cuda_runtime.h>

#include "cracsim/kernels.hpp"

namespace cracsim {
namespace {

__global__ void k_fill8(uint8_t* p, uint64_t n, uint8_t v) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void k_affine8(uint8_t* p, uint64_t n, uint8_t mul, uint8_t add) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    p[i] = uint8_t(p[i] * mul + add);
}

// ref: kernels.cpp:34-48 — four lanes, fixed combine order.
__device__ float dot4(const float* x, const float* y, uint64_t n, uint64_t sy = 1) {
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  uint64_t i = 0;
  for (; i + 4 <= n; i += 4) {
    a0 += x[i] * y[i * sy];
    a1 += x[i + 1] * y[(i + 1) * sy];
    a2 += x[i + 2] * y[(i + 2) * sy];
    a3 += x[i + 3] * y[(i + 3) * sy];
  }
  float acc = (a0 + a1) + (a2 + a3);
  for (; i < n; ++i) acc += x[i] * y[i * sy];
  return acc;
}

__global__ void k_dot(const float* x, const float* y, float* out, uint64_t n) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = dot4(x, y, n);
}

__global__ void k_gemv(const float* a, const float* x, float* y, uint64_t m, uint64_t k) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < m) y[i] = dot4(a + i * k, x, k);
}

__global__ void k_gemm(const float* a, const float* b, float* c, uint64_t m, uint64_t k,
                       uint64_t n) {
  const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (idx >= m * n) return;
  const uint64_t i = idx / n, j = idx % n;
  c[idx] = dot4(a + i * k, b + j, k, n);
}

unsigned grid_for(uint64_t n) {
  const uint64_t g = (n + 255) / 256;
  return unsigned(g == 0 ? 1 : (g > 4096 ? 4096 : g));
}

void fill8(KernelArgs& a) {
  auto out = a.write(0, 0, a.scalars()[1]);
  if (out.empty()) return;
  k_fill8<<<grid_for(out.size()), 256, 0, a.stream()>>>(out.data(), out.size(),
                                                        uint8_t(a.scalars()[0]));
}

void add8(KernelArgs& a) {
  auto out = a.write(0, 0, a.scalars()[1]);
  if (out.empty()) return;
  k_affine8<<<grid_for(out.size()), 256, 0, a.stream()>>>(out.data(), out.size(), 1,
                                                          uint8_t(a.scalars()[0]));
}

void affine8(KernelArgs& a) {
  auto out = a.write(0, 0, a.scalars()[2]);
  if (out.empty()) return;
  k_affine8<<<grid_for(out.size()), 256, 0, a.stream()>>>(
      out.data(), out.size(), uint8_t(a.scalars()[0]), uint8_t(a.scalars()[1]));
}

void dot_f32(KernelArgs& a) {
  const uint64_t n = a.scalars()[0];
  auto x = a.read(0, 0, n * 4);
  auto y = a.read(1, 0, n * 4);
  auto o = a.write(2, 0, 4);
  k_dot<<<1, 32, 0, a.stream()>>>(reinterpret_cast<const float*>(x.data()),
                                  reinterpret_cast<const float*>(y.data()),
                                  reinterpret_cast<float*>(o.data()), n);
}

void gemv_f32(KernelArgs& a) {
  const uint64_t m = a.scalars()[0], k = a.scalars()[1];
  auto A = a.read(0, 0, m * k * 4);
  auto x = a.read(1, 0, k * 4);
  auto y = a.write(2, 0, m * 4);
  if (!m) return;
  k_gemv<<<grid_for(m), 256, 0, a.stream()>>>(reinterpret_cast<const float*>(A.data()),
                                              reinterpret_cast<const float*>(x.data()),
                                              reinterpret_cast<float*>(y.data()), m, k);
}

void gemm_f32(KernelArgs& a) {
  const uint64_t m = a.scalars()[0], k = a.scalars()[1], n = a.scalars()[2];
  auto A = a.read(0, 0, m * k * 4);
  auto B = a.read(1, 0, k * n * 4);
  auto C = a.write(2, 0, m * n * 4);
  if (!m || !n) return;
  k_gemm<<<unsigned((m * n + 255) / 256), 256, 0, a.stream()>>>(
      reinterpret_cast<const float*>(A.data()), reinterpret_cast<const float*>(B.data()),
      reinterpret_cast<float*>(C.data()), m, k, n);
}

}  // namespace

std::vector<KernelDescriptor> standard_kernels() {
  return {{"fill8", 1, 2, fill8},       {"add8", 1, 2, add8},
          {"affine8", 1, 3, affine8},   {"dot_f32", 3, 1, dot_f32},
          {"gemv_f32", 3, 2, gemv_f32}, {"gemm_f32", 3, 3, gemm_f32}};
}

const KernelCatalog& standard_catalog() {
  static const KernelCatalog cat = [] {
    KernelCatalog c;
    for (auto& d : standard_kernels()) c.emplace(d.name, d.body);
    return c;
  }();
  return cat;
}

}  // namespace cracsim
