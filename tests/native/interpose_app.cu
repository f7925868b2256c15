// A plain CUDA application (links the shared CUDA runtime, knows nothing of
// cracsim) used to test libcrac_preload.so.
//
//   interpose_app run <image>   allocate, fill with its own kernels and host
//                               writes, free a temporary, checkpoint through
//                               crac_preload_checkpoint if the preload is there
//   interpose_app spin <ms>     the same state, then keeps the device busy
//                               (the target of a SIGUSR2 checkpoint)
//   interpose_app resume        (under CRAC_RESTART_FROM) find its pointers in
//                               its saved state and verify every byte with
//                               its own kernels / host reads
// Exit 0 on success.  Content is a pure function of the index, restated by
// tests/test_gpu_interpose.py to build the reference image of the same calls.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      std::fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 2;                                                                          \
    }                                                                                    \
  } while (0)

constexpr size_t kA = 3 * 1024 * 1024 + 12;  // floats
constexpr size_t kB = 1000003;                // bytes, odd
constexpr size_t kM = 6 * 4096 + 100;         // managed bytes
constexpr size_t kH = 70000;                  // pinned bytes

struct Saved {
  uint64_t magic;
  float* a;
  uint8_t* b;
  uint8_t* m;
  uint8_t* h;
  uint64_t step;
};

__global__ void fill_a(float* a, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    a[i] = float(i % 65536) * 0.5f + 1.0f;
}
__global__ void fill_b(uint8_t* b, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    b[i] = uint8_t(i * 7 + 3);
}
__global__ void fill_m(uint8_t* m, size_t n) {  // device writes the first half
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n / 2; i += size_t(gridDim.x) * blockDim.x)
    m[i] = uint8_t(i * 13 + 1);
}
__global__ void count_bad(const float* a, size_t na, const uint8_t* b, size_t nb, unsigned long long* bad) {
  unsigned long long k = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < na; i += size_t(gridDim.x) * blockDim.x)
    k += a[i] != float(i % 65536) * 0.5f + 1.0f;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nb; i += size_t(gridDim.x) * blockDim.x)
    k += b[i] != uint8_t(i * 7 + 3);
  if (k) atomicAdd(bad, k);
}

template <typename F>
F hook(const char* name) {
  return reinterpret_cast<F>(dlsym(RTLD_DEFAULT, name));
}

// Allocates and fills everything; leaves the streams in *s1 / *s2.
int setup(Saved& sv, cudaStream_t* s1, cudaStream_t* s2) {
  CK(cudaStreamCreate(s1));
  CK(cudaStreamCreateWithFlags(s2, cudaStreamNonBlocking));
  sv = Saved{0x5341564544ull, nullptr, nullptr, nullptr, nullptr, 41};
  CK(cudaMalloc(&sv.a, kA * sizeof(float)));
  void* tmp;
  CK(cudaMalloc(&tmp, 1000));
  CK(cudaMalloc(&sv.b, kB));
  CK(cudaFree(tmp));  // leaves a hole the log must replay
  CK(cudaMallocManaged(&sv.m, kM));
  CK(cudaMallocHost(&sv.h, kH));
  fill_a<<<148, 256, 0, *s1>>>(sv.a, kA);
  fill_b<<<148, 256, 0, *s2>>>(sv.b, kB);
  fill_m<<<4, 256, 0, *s1>>>(sv.m, kM);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(*s1));
  CK(cudaStreamSynchronize(*s2));
  for (size_t i = kM / 2; i < kM; ++i) sv.m[i] = uint8_t(i ^ 0xA5);
  for (size_t i = 0; i < kH; ++i) sv.h[i] = uint8_t(i * 3 + 11);
  CK(cudaDeviceSynchronize());
  std::printf("a=%p b=%p m=%p h=%p\n", (void*)sv.a, (void*)sv.b, (void*)sv.m, (void*)sv.h);
  return 0;
}

int run(const char* image) {
  cudaStream_t s1, s2;
  Saved sv;
  if (int rc = setup(sv, &s1, &s2)) return rc;
  auto set_state = hook<int (*)(const void*, uint64_t)>("crac_preload_set_app_state");
  auto ckpt = hook<int (*)(const char*)>("crac_preload_checkpoint");
  if (!set_state || !ckpt) {
    std::printf("no preload: ran without a checkpoint\n");
    return 0;
  }
  if (set_state(&sv, sizeof sv) || ckpt(image)) return 3;
  // the application keeps running after the checkpoint
  fill_b<<<148, 256, 0, s2>>>(sv.b, kB);
  CK(cudaStreamSynchronize(s2));
  std::printf("checkpointed to %s\n", image);
  return 0;
}

// Keeps the device busy for `ms` milliseconds (rewriting b with the same
// values on both streams) so an asynchronous checkpoint lands mid-run.
int spin(long ms) {
  cudaStream_t s1, s2;
  Saved sv;
  if (int rc = setup(sv, &s1, &s2)) return rc;
  auto set_state = hook<int (*)(const void*, uint64_t)>("crac_preload_set_app_state");
  if (set_state && set_state(&sv, sizeof sv)) return 3;
  std::printf("spinning\n");
  std::fflush(stdout);
  const auto t0 = std::chrono::steady_clock::now();
  long iters = 0;
  while (std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(ms)) {
    fill_b<<<148, 256, 0, (iters & 1) ? s1 : s2>>>(sv.b, kB);
    fill_a<<<148, 256, 0, (iters & 1) ? s2 : s1>>>(sv.a, kA);
    if (++iters % 16 == 0) CK(cudaDeviceSynchronize());
  }
  CK(cudaDeviceSynchronize());
  std::printf("spun %ld iterations\n", iters);
  return 0;
}

// Device memory only (the pre-copy path of the preload's checkpoint): a and
// b rewritten with their own values on two streams for `ms` milliseconds.
int devspin(long ms) {
  cudaStream_t s1, s2;
  CK(cudaStreamCreate(&s1));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  Saved sv{0x4445564f4e4cull, nullptr, nullptr, nullptr, nullptr, 43};
  CK(cudaMalloc(&sv.a, kA * sizeof(float)));
  CK(cudaMalloc(&sv.b, kB));
  fill_a<<<148, 256, 0, s1>>>(sv.a, kA);
  fill_b<<<148, 256, 0, s2>>>(sv.b, kB);
  CK(cudaDeviceSynchronize());
  auto set_state = hook<int (*)(const void*, uint64_t)>("crac_preload_set_app_state");
  if (set_state && set_state(&sv, sizeof sv)) return 3;
  std::printf("a=%p b=%p\nspinning\n", (void*)sv.a, (void*)sv.b);
  std::fflush(stdout);
  const auto t0 = std::chrono::steady_clock::now();
  long iters = 0;
  while (std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(ms)) {
    fill_b<<<148, 256, 0, (iters & 1) ? s1 : s2>>>(sv.b, kB);
    fill_a<<<148, 256, 0, (iters & 1) ? s2 : s1>>>(sv.a, kA);
    if (++iters % 16 == 0) CK(cudaDeviceSynchronize());
  }
  CK(cudaDeviceSynchronize());
  std::printf("spun %ld iterations\n", iters);
  return 0;
}

int devresume() {
  auto get_state = hook<int (*)(const void**, uint64_t*)>("crac_preload_app_state");
  const void* p = nullptr;
  uint64_t n = 0;
  if (!get_state || get_state(&p, &n) || n != sizeof(Saved)) return 5;
  Saved sv;
  std::memcpy(&sv, p, sizeof sv);
  if (sv.magic != 0x4445564f4e4cull || sv.step != 43) return 6;
  unsigned long long* bad;
  CK(cudaMalloc(&bad, sizeof *bad));
  CK(cudaMemset(bad, 0, sizeof *bad));
  count_bad<<<148, 256>>>(sv.a, kA, sv.b, kB, bad);
  unsigned long long host_bad = 0;
  CK(cudaMemcpy(&host_bad, bad, sizeof host_bad, cudaMemcpyDeviceToHost));
  std::printf("resumed: device mismatches %llu\n", host_bad);
  return host_bad ? 9 : 0;
}

int resume() {
  auto restarted = hook<int (*)()>("crac_preload_restarted");
  auto get_state = hook<int (*)(const void**, uint64_t*)>("crac_preload_app_state");
  auto translate = hook<void* (*)(const void*)>("crac_preload_translate");
  if (!restarted || !restarted()) {
    std::fprintf(stderr, "not restarted\n");
    return 4;
  }
  const void* p = nullptr;
  uint64_t n = 0;
  if (get_state(&p, &n) || n != sizeof(Saved)) return 5;
  Saved sv;
  std::memcpy(&sv, p, sizeof sv);
  if (sv.magic != 0x5341564544ull || sv.step != 41) return 6;
  // device memory sits at the same addresses; pinned/managed are re-issued
  if (translate(sv.a) != sv.a || translate(sv.b) != sv.b) return 7;
  uint8_t* m = static_cast<uint8_t*>(translate(sv.m));
  uint8_t* h = static_cast<uint8_t*>(translate(sv.h));
  if (!m || !h) return 8;
  unsigned long long* bad;
  CK(cudaMallocManaged(&bad, sizeof *bad));  // a new allocation after restart
  *bad = 0;
  count_bad<<<148, 256>>>(sv.a, kA, sv.b, kB, bad);
  CK(cudaDeviceSynchronize());
  unsigned long long host_bad = 0;
  for (size_t i = 0; i < kM; ++i) host_bad += m[i] != (i < kM / 2 ? uint8_t(i * 13 + 1) : uint8_t(i ^ 0xA5));
  for (size_t i = 0; i < kH; ++i) host_bad += h[i] != uint8_t(i * 3 + 11);
  std::printf("resumed: device mismatches %llu, host-visible mismatches %llu\n", *bad, host_bad);
  return (*bad || host_bad) ? 9 : 0;
}

int main(int argc, char** argv) {
  if (argc >= 3 && !std::strcmp(argv[1], "run")) return run(argv[2]);
  if (argc >= 2 && !std::strcmp(argv[1], "resume")) return resume();
  if (argc >= 3 && !std::strcmp(argv[1], "spin")) return spin(std::atol(argv[2]));
  if (argc >= 3 && !std::strcmp(argv[1], "devspin")) return devspin(std::atol(argv[2]));
  if (argc >= 2 && !std::strcmp(argv[1], "devresume")) return devresume();
  std::fprintf(stderr, "usage: interpose_app run <image> | resume\n");
  return 1;
}
