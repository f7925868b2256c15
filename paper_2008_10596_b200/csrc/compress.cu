// Host side of the GPU CRACSIMZ compressor (K5, deflate.cu): batches of the
// image go to the device, K5 deflates them segment by segment, the host
// prefix-sums the piece lengths and folds the per-segment Adler-32s
// (zlib's adler32_combine), a gather kernel packs the pieces, and the stream
// comes back.  Wrapper layout as the reference writes it
// (/root/reference/proj/src/image.cpp:419-430): "CRACSIMZ", u64 raw length,
// then a zlib stream (2-byte header, deflate, big-endian Adler-32).
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <zlib.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "crac_gpu.h"
#include "cracsim/ckpt_engine.hpp"

namespace cracsim {
namespace {

template <typename T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(uint64_t n) {
    check_cuda(cudaMalloc(reinterpret_cast<void**>(&p), std::max<uint64_t>(n, 1) * sizeof(T)),
               "deflate buffer");
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace

// Host memory for a compressed image: 2 MiB-aligned and THP-advised, so the
// D2H into it takes one fault per 2 MiB instead of per 4 KiB (a fresh 16 GiB
// malloc faulted at ~2 GB/s, slower than the deflate).  Free with std::free.
uint8_t* alloc_compressed_host(uint64_t bytes) {
  constexpr uint64_t kHuge = 2ull << 20;
  const uint64_t cap = (bytes + kHuge - 1) / kHuge * kHuge;
  void* p = std::aligned_alloc(kHuge, cap);
  if (!p) raise(Errc::InvalidArgument, "compress: out of host memory");
  madvise(p, cap, MADV_HUGEPAGE);
  return static_cast<uint8_t*>(p);
}

uint64_t compressed_bound_gpu(uint64_t n) {
  return 16 + 2 + n + 5 * (n / CRAC_DEFLATE_SEGMENT + 1) + 4;
}

std::vector<uint8_t> compress_image_gpu(std::span<const uint8_t> image, double* ms) {
  std::vector<uint8_t> out(compressed_bound_gpu(image.size()));
  out.resize(compress_image_gpu_into(image, out.data(), out.size(), ms));
  return out;
}

uint64_t compress_image_gpu_into(std::span<const uint8_t> image, uint8_t* dst, uint64_t cap,
                                 double* ms) {
  const auto t0 = std::chrono::steady_clock::now();
  constexpr uint64_t kSeg = CRAC_DEFLATE_SEGMENT;
  constexpr uint64_t kBatch = 1ull << 30;  // a multiple of the segment
  const uint64_t n = image.size();
  if (cap < compressed_bound_gpu(n)) raise(Errc::InvalidArgument, "compress: output too small");
  const uint64_t batch = std::min<uint64_t>(kBatch, std::max<uint64_t>(n, 1));
  const uint64_t seg_max = (batch + kSeg - 1) / kSeg;

  uint64_t at_out = 0;
  auto emit = [&](const void* p, uint64_t k) {
    std::memcpy(dst + at_out, p, k);
    at_out += k;
  };
  emit(kCompressedMagic, 8);
  uint8_t hdr[10];
  for (int i = 0; i < 8; ++i) hdr[i] = uint8_t(n >> (8 * i));
  hdr[8] = 0x78;  // zlib header: deflate, 32 KiB window
  hdr[9] = 0x9C;  // (0x789C % 31 == 0, no dictionary)
  emit(hdr, 10);
  if (n == 0) {  // a final empty stored block
    const uint8_t empty[5] = {1, 0, 0, 0xFF, 0xFF};
    emit(empty, 5);
  }

  DevBuf<uint8_t> d_in(batch), d_slots(seg_max * CRAC_DEFLATE_SLOT), d_out(batch + 5 * seg_max);
  DevBuf<uint32_t> d_len(seg_max), d_adler(seg_max);
  DevBuf<uint64_t> d_off(seg_max);
  cudaStream_t st = nullptr;
  check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "deflate stream");
  std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> keep(st, &cudaStreamDestroy);
  std::vector<uint32_t> len(seg_max), adl(seg_max);
  std::vector<uint64_t> off(seg_max);
  uLong adler = adler32(0L, Z_NULL, 0);
  for (uint64_t at = 0; at < n; at += batch) {
    const uint64_t m = std::min(batch, n - at), segs = (m + kSeg - 1) / kSeg;
    check_cuda(cudaMemcpyAsync(d_in.p, image.data() + at, m, cudaMemcpyHostToDevice, st),
               "deflate H2D");
    check_cuda(cudaError_t(crac_deflate_segments(d_in.p, m, d_slots.p, d_len.p, d_adler.p,
                                                 at + m == n ? 1 : 0, st)),
               "deflate");
    check_cuda(cudaMemcpyAsync(len.data(), d_len.p, segs * 4, cudaMemcpyDeviceToHost, st), "lens");
    check_cuda(cudaMemcpyAsync(adl.data(), d_adler.p, segs * 4, cudaMemcpyDeviceToHost, st),
               "adler");
    check_cuda(cudaStreamSynchronize(st), "deflate sync");
    uint64_t total = 0;
    for (uint64_t k = 0; k < segs; ++k) {
      off[k] = total;
      total += len[k] & 0x7FFFFFFFu;  // (bit 31: a stored piece)
      const uint64_t sl = std::min(kSeg, m - k * kSeg);
      adler = adler32_combine(adler, adl[k], z_off_t(sl));
    }
    check_cuda(cudaMemcpyAsync(d_off.p, off.data(), segs * 8, cudaMemcpyHostToDevice, st),
               "offsets");
    check_cuda(cudaError_t(crac_gather_segments(d_in.p, m, d_slots.p, d_len.p, d_off.p, d_out.p,
                                                at + m == n ? 1 : 0, st)),
               "gather");
    check_cuda(cudaMemcpyAsync(dst + at_out, d_out.p, total, cudaMemcpyDeviceToHost, st),
               "deflate D2H");
    check_cuda(cudaStreamSynchronize(st), "deflate sync");
    at_out += total;
  }
  uint8_t tail[4];
  for (int i = 0; i < 4; ++i) tail[i] = uint8_t(adler >> (8 * (3 - i)));
  emit(tail, 4);
  if (ms)
    *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return at_out;
}

}  // namespace cracsim
