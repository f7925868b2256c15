// GF(2) arithmetic behind the reference's section checksum.
//
// The reference stores zlib crc32 (CRC-32/IEEE, reflected poly 0xEDB88320,
// init/xorout 0xFFFFFFFF) after each image section (ref: src/image.cpp:16-26,
// :396).  Everything the B200 path does with CRCs follows from two facts:
//
//   1. The CRC register update is linear over GF(2):
//        run(state, data) = A^|data|(state) xor L(data)
//      where A is "advance one zero byte" = multiplication by x^8 mod P and
//      L(data) = run(0, data).  Hence  crc32(data) = L(data) xor K(|data|),
//      K(n) = A^n(0xFFFFFFFF) xor 0xFFFFFFFF.
//   2. L(X || Y) = A^|Y|(L(X)) xor L(Y), and zlib's crc32_combine uses the
//      same operator on finalized CRCs.
//
// Polynomials use zlib's reflected convention: bit 31 is the x^0 coefficient.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define CRAC_HD __host__ __device__ __forceinline__
#else
#define CRAC_HD inline
#endif

namespace crac {

constexpr uint32_t kCrcPoly = 0xEDB88320u;

// a * b mod P (reflected).  Bit-serial; used for one-off shifts only.
CRAC_HD uint32_t gf_mul(uint32_t a, uint32_t b) {
  uint32_t prod = 0;
  for (int k = 0; k < 32; ++k) {
    if (a & (0x80000000u >> k)) prod ^= b;
    b = (b & 1u) ? (b >> 1) ^ kCrcPoly : (b >> 1);
  }
  return prod;
}

// x^(8 n) mod P by square-and-multiply.  `pow2` may supply x^(8*2^k) for
// k = 0..63 (saves the squarings); pass nullptr to compute them inline.
CRAC_HD uint32_t x8n(uint64_t n, const uint32_t* pow2 = nullptr) {
  uint32_t result = 0x80000000u;  // x^0
  uint32_t sq = 0x00800000u;      // x^8
  for (int k = 0; n; ++k, n >>= 1) {
    const uint32_t p = pow2 ? pow2[k] : sq;
    if (n & 1) result = gf_mul(p, result);
    if (!pow2) sq = gf_mul(sq, sq);
  }
  return result;
}

// State `s` advanced by n zero bytes.
CRAC_HD uint32_t advance(uint32_t s, uint64_t n, const uint32_t* pow2 = nullptr) {
  return gf_mul(x8n(n, pow2), s);
}

// zlib crc32_combine: crc(A||B) from crc(A), crc(B), |B|.
CRAC_HD uint32_t crc_combine(uint32_t crc_a, uint32_t crc_b, uint64_t len_b,
                             const uint32_t* pow2 = nullptr) {
  return advance(crc_a, len_b, pow2) ^ crc_b;
}

// K(n): the affine part of crc32 for an n-byte message.
CRAC_HD uint32_t crc_affine(uint64_t n, const uint32_t* pow2 = nullptr) {
  return advance(0xFFFFFFFFu, n, pow2) ^ 0xFFFFFFFFu;
}

// Byte-table CRC update (host side small inputs and the device tail path).
CRAC_HD uint32_t byte_step(uint32_t s, uint8_t b, const uint32_t* t0) {
  return (s >> 8) ^ t0[(s ^ b) & 0xFFu];
}

}  // namespace crac
