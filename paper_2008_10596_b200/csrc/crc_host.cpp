// Host CRC-32/IEEE (zlib's crc32, bit-identical) by carry-less multiplication.
//
// The host threads of the drain and the refill hash every host-resident
// managed page (C3: 8 GiB), which zlib's table CRC does at ~2.6 GB/s per core.
// This folds 64 bytes per step with PCLMULQDQ (4 x 128-bit lanes, fold
// distance 512 bits), then 128 -> 64 -> 32 bits with a Barrett reduction --
// the standard reflected-CRC folding scheme for the polynomial 0xEDB88320.
// The fold constants are x^k mod P (bit-reflected) for the fold distances;
// they are re-derived and checked against zlib by tests/test_host_logic.py.
// Inputs shorter than 64 bytes and the sub-16-byte tail go through zlib.
#include <immintrin.h>
#include <zlib.h>

#include <cstdint>
#include <cstring>

namespace cracsim::codec {
namespace {

#define CRAC_PCLMUL __attribute__((target("pclmul,sse4.1")))

CRAC_PCLMUL inline __m128i load16(const uint8_t* q) {
  return _mm_loadu_si128(reinterpret_cast<const __m128i*>(q));
}

// x folded forward by the distance k encodes, plus the next 16 input bytes
CRAC_PCLMUL inline __m128i fold16(__m128i x, __m128i k, __m128i next) {
  return _mm_xor_si128(
      _mm_xor_si128(_mm_clmulepi64_si128(x, k, 0x00), _mm_clmulepi64_si128(x, k, 0x11)), next);
}

CRAC_PCLMUL uint32_t fold_crc(uint32_t crc, const uint8_t* p, size_t len) {
  // len >= 64, multiple of 16; crc is the raw (non-inverted) register
  const __m128i k1k2 = _mm_set_epi64x(0x1c6e41596LL, 0x154442bd4LL);  // fold by 512 bits
  const __m128i k3k4 = _mm_set_epi64x(0x0ccaa009eLL, 0x1751997d0LL);  // fold by 128 bits
  const __m128i k5 = _mm_set_epi64x(0, 0x163cd6124LL);               // 64 -> 32
  const __m128i poly = _mm_set_epi64x(0x1f7011641LL, 0x1db710641LL);  // Barrett: u, P'
  const __m128i mask32 = _mm_set_epi32(0, 0, 0, -1);
  __m128i x0 = _mm_xor_si128(load16(p), _mm_cvtsi32_si128(int(crc)));
  __m128i x1 = load16(p + 16), x2 = load16(p + 32), x3 = load16(p + 48);
  p += 64;
  len -= 64;
  for (; len >= 64; len -= 64, p += 64) {
    x0 = fold16(x0, k1k2, load16(p));
    x1 = fold16(x1, k1k2, load16(p + 16));
    x2 = fold16(x2, k1k2, load16(p + 32));
    x3 = fold16(x3, k1k2, load16(p + 48));
  }
  x0 = fold16(x0, k3k4, x1);
  x0 = fold16(x0, k3k4, x2);
  x0 = fold16(x0, k3k4, x3);
  for (; len >= 16; len -= 16, p += 16) x0 = fold16(x0, k3k4, load16(p));
  // 128 -> 64
  x0 = _mm_xor_si128(_mm_clmulepi64_si128(x0, k3k4, 0x10), _mm_srli_si128(x0, 8));
  // 64 -> 32
  x0 = _mm_xor_si128(_mm_clmulepi64_si128(_mm_and_si128(x0, mask32), k5, 0x00),
                     _mm_srli_si128(x0, 4));
  // Barrett reduction
  __m128i t = _mm_clmulepi64_si128(_mm_and_si128(x0, mask32), poly, 0x10);
  t = _mm_clmulepi64_si128(_mm_and_si128(t, mask32), poly, 0x00);
  return uint32_t(_mm_extract_epi32(_mm_xor_si128(t, x0), 1));
}

// fold_crc that also copies the bytes it folds to `dst` (16-byte aligned)
// with non-temporal stores: the destination lines are written without being
// read first (no read-for-ownership), and the source is read once
CRAC_PCLMUL uint32_t fold_crc_copy(uint32_t crc, const uint8_t* p, uint8_t* d, size_t len) {
  const __m128i k1k2 = _mm_set_epi64x(0x1c6e41596LL, 0x154442bd4LL);
  const __m128i k3k4 = _mm_set_epi64x(0x0ccaa009eLL, 0x1751997d0LL);
  const __m128i k5 = _mm_set_epi64x(0, 0x163cd6124LL);
  const __m128i poly = _mm_set_epi64x(0x1f7011641LL, 0x1db710641LL);
  const __m128i mask32 = _mm_set_epi32(0, 0, 0, -1);
  auto out = [&](size_t o, __m128i v) { _mm_stream_si128(reinterpret_cast<__m128i*>(d + o), v); };
  __m128i y0 = load16(p), y1 = load16(p + 16), y2 = load16(p + 32), y3 = load16(p + 48);
  out(0, y0), out(16, y1), out(32, y2), out(48, y3);
  __m128i x0 = _mm_xor_si128(y0, _mm_cvtsi32_si128(int(crc))), x1 = y1, x2 = y2, x3 = y3;
  p += 64;
  d += 64;
  len -= 64;
  for (; len >= 64; len -= 64, p += 64, d += 64) {
    y0 = load16(p), y1 = load16(p + 16), y2 = load16(p + 32), y3 = load16(p + 48);
    out(0, y0), out(16, y1), out(32, y2), out(48, y3);
    x0 = fold16(x0, k1k2, y0);
    x1 = fold16(x1, k1k2, y1);
    x2 = fold16(x2, k1k2, y2);
    x3 = fold16(x3, k1k2, y3);
  }
  x0 = fold16(x0, k3k4, x1);
  x0 = fold16(x0, k3k4, x2);
  x0 = fold16(x0, k3k4, x3);
  for (; len >= 16; len -= 16, p += 16, d += 16) {
    y0 = load16(p);
    out(0, y0);
    x0 = fold16(x0, k3k4, y0);
  }
  x0 = _mm_xor_si128(_mm_clmulepi64_si128(x0, k3k4, 0x10), _mm_srli_si128(x0, 8));
  x0 = _mm_xor_si128(_mm_clmulepi64_si128(_mm_and_si128(x0, mask32), k5, 0x00),
                     _mm_srli_si128(x0, 4));
  __m128i t = _mm_clmulepi64_si128(_mm_and_si128(x0, mask32), poly, 0x10);
  t = _mm_clmulepi64_si128(_mm_and_si128(t, mask32), poly, 0x00);
  return uint32_t(_mm_extract_epi32(_mm_xor_si128(t, x0), 1));
}

bool have_pclmul() {
  static const bool ok = __builtin_cpu_supports("pclmul") && __builtin_cpu_supports("sse4.1");
  return ok;
}

}  // namespace

uint32_t crc32_fast(const uint8_t* p, size_t n, uint32_t crc) {
  if (n < 64 || !have_pclmul()) return uint32_t(::crc32_z(crc, p, n));
  const size_t body = n & ~size_t(15);
  crc = ~fold_crc(~crc, p, body);
  if (n > body) crc = uint32_t(::crc32_z(crc, p + body, n - body));
  return crc;
}

uint32_t crc32_copy_stream(uint8_t* dst, const uint8_t* src, size_t n, uint32_t crc) {
  if (n < 64 || !have_pclmul() || reinterpret_cast<uintptr_t>(dst) % 16) {
    std::memcpy(dst, src, n);
    return crc32_fast(src, n, crc);
  }
  const size_t body = n & ~size_t(15);
  crc = ~fold_crc_copy(~crc, src, dst, body);
  if (n > body) {
    std::memcpy(dst + body, src + body, n - body);
    crc = uint32_t(::crc32_z(crc, src + body, n - body));
  }
  return crc;
}

void stream_fence() { _mm_sfence(); }

}  // namespace cracsim::codec
