// K5: GPU deflate for the CRACSIMZ wrapper (the reference's
// compress_image, /root/reference/proj/src/image.cpp:419-430, is zlib
// compress2 level 6 on the host, and maybe_decompress :347-379 inflates it).
//
// The reference's compressed bytes are zlib's level-6 output, which no
// parallel compressor reproduces.  What restart parity needs is weaker: a
// zlib stream that inflates to the exact image.  This one is built the way
// parallel gzip builds its streams:
//   * the image is cut into 32 KiB segments, one GPU thread each;
//   * a thread compresses its segment alone (greedy LZ77 over a small
//     hash table of 16-bit positions in shared memory (512 entries), RFC 1951 fixed Huffman
//     codes) and ends it with an empty stored block (the "sync flush"), so
//     every segment starts and ends on a byte boundary and the segments
//     concatenate into one deflate stream; a segment that would not shrink
//     (or shows no match in its first 4 KiB while its codes already outgrow
//     its bytes) is written as a stored block instead (never more than 5
//     bytes of growth), built by the gather straight from the input;
//   * the same thread folds the segment into a (partial) Adler-32; the host
//     combines the per-segment values with zlib's adler32_combine.
// A second kernel gathers the variable-length segment outputs into one
// contiguous stream at the host-computed offsets.
#include <cuda_runtime.h>

#include <cstdint>

#include "crac_gpu.h"

namespace {

constexpr uint32_t kSeg = CRAC_DEFLATE_SEGMENT;     // 32 KiB
constexpr uint32_t kSlot = CRAC_DEFLATE_SLOT;       // worst-case fixed-Huffman segment
constexpr int kHashBits = 9;  // 512 x u16 per thread: 32 KiB of static smem per CTA
constexpr int kThreads = 32;                         // segments per CTA
constexpr uint32_t kWindow = 32768;                  // deflate's maximum distance
constexpr uint32_t kMaxMatch = 258;
constexpr uint32_t kProbe = 4096;                    // bytes before giving up on a segment
constexpr uint32_t kStoredFlag = 0x80000000u;        // out_len: a stored piece

__constant__ uint16_t c_len_base[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                        31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2,
                                        2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dist_base[30] = {1,    2,    3,    4,    5,    7,     9,     13,    17,  25,
                                         33,   49,   65,   97,   129,  193,   257,   385,   513, 769,
                                         1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t c_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2,  3,  3,  4,  4,  5,  5,  6,
                                         6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

struct BitWriter {
  uint8_t* out;
  uint64_t acc = 0;
  uint32_t nbits = 0, pos = 0;
  __device__ __forceinline__ void put(uint32_t v, uint32_t n) {  // LSB-first, n <= 24
    acc |= uint64_t(v) << nbits;
    nbits += n;
    while (nbits >= 8) {
      out[pos++] = uint8_t(acc);
      acc >>= 8;
      nbits -= 8;
    }
  }
  // a Huffman code: its bits go out most significant first
  __device__ __forceinline__ void code(uint32_t c, uint32_t n) { put(__brev(c) >> (32 - n), n); }
  __device__ __forceinline__ void align() {
    if (nbits) {
      out[pos++] = uint8_t(acc);
      acc = 0;
      nbits = 0;
    }
  }
};

// RFC 1951 3.2.6 fixed literal/length code of symbol s
__device__ __forceinline__ void put_litlen(BitWriter& w, uint32_t s) {
  if (s < 144) w.code(0x30 + s, 8);
  else if (s < 256) w.code(0x190 + (s - 144), 9);
  else if (s < 280) w.code(s - 256, 7);
  else w.code(0xC0 + (s - 280), 8);
}

__device__ __forceinline__ void put_match(BitWriter& w, uint32_t len, uint32_t dist) {
  int l = 28;
  while (c_len_base[l] > len) --l;  // 29 entries, descending scan
  put_litlen(w, 257 + l);
  if (c_len_extra[l]) w.put(len - c_len_base[l], c_len_extra[l]);
  int d = 29;
  while (c_dist_base[d] > dist) --d;
  w.code(d, 5);
  if (c_dist_extra[d]) w.put(dist - c_dist_base[d], c_dist_extra[d]);
}

__device__ __forceinline__ uint32_t hash3(uint32_t v) {
  return ((v & 0xFFFFFFu) * 2654435761u) >> (32 - kHashBits);
}

__global__ void __launch_bounds__(kThreads)
    k_deflate_segments(const uint8_t* __restrict__ in, uint64_t n, uint64_t n_seg,
                       uint8_t* __restrict__ slots, uint32_t* __restrict__ out_len,
                       uint32_t* __restrict__ adler, int last_is_final) {
  __shared__ uint16_t table[kThreads][1 << kHashBits];
  const uint64_t seg = blockIdx.x * uint64_t(kThreads) + threadIdx.x;
  if (seg >= n_seg) return;
  uint16_t* tab = table[threadIdx.x];
  for (int i = 0; i < (1 << kHashBits); ++i) tab[i] = 0;  // 0 = empty, else position + 1
  const uint8_t* s = in + seg * kSeg;
  const uint64_t rest = n - seg * kSeg;
  const uint32_t len = rest < kSeg ? uint32_t(rest) : kSeg;
  const bool final_seg = last_is_final && seg + 1 == n_seg;

  // Adler-32 of the segment alone (a from 1), folded on the host; 16-byte
  // loads (segments start 32 KiB-aligned in the batch buffer)
  uint32_t a = 1, b = 0;
  {
    const uint32_t words = len / 16;
    const uint4* s4 = reinterpret_cast<const uint4*>(s);
    for (uint32_t wbeg = 0; wbeg < words;) {
      const uint32_t wend = min(words, wbeg + 340u);  // 5440 bytes: no 32-bit overflow
      for (uint32_t k = wbeg; k < wend; ++k) {
        const uint4 v = __ldg(s4 + k);
        const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            a += (x[q] >> (8 * r)) & 0xFFu;
            b += a;
          }
      }
      a %= 65521u;
      b %= 65521u;
      wbeg = wend;
    }
    for (uint32_t i = words * 16; i < len; ++i) {
      a += __ldg(s + i);
      b += a;
    }
    a %= 65521u;
    b %= 65521u;
  }
  adler[seg] = (b << 16) | a;

  BitWriter w{slots + seg * uint64_t(kSlot)};
  w.put(final_seg ? 1u : 0u, 1);  // BFINAL
  w.put(1u, 2);                    // BTYPE 01: fixed Huffman codes
  uint32_t pos = 0;
  uint32_t win = 0;  // next three bytes (little-endian)
  if (len >= 3) win = __ldg(s) | (uint32_t(__ldg(s + 1)) << 8) | (uint32_t(__ldg(s + 2)) << 16);
  bool matched = false;
  while (pos < len) {
    // incompressible so far (no match in the first kProbe bytes and the codes
    // already longer than the bytes): the whole segment goes stored
    if (pos >= kProbe && !matched && w.pos >= pos) break;
    if (pos + 3 <= len) {
      const uint32_t h = hash3(win);
      const uint32_t cand = tab[h];
      tab[h] = uint16_t(pos + 1);
      if (cand && pos - (cand - 1) <= kWindow) {
        const uint32_t c = cand - 1;
        const uint32_t maxl = min(kMaxMatch, len - pos);
        uint32_t l = 0;
        while (l < maxl && __ldg(s + c + l) == __ldg(s + pos + l)) ++l;
        if (l >= 3) {
          matched = true;
          put_match(w, l, pos - c);
          pos += l;
          if (pos + 3 <= len)
            win = __ldg(s + pos) | (uint32_t(__ldg(s + pos + 1)) << 8) |
                  (uint32_t(__ldg(s + pos + 2)) << 16);
          continue;
        }
      }
    }
    put_litlen(w, __ldg(s + pos));
    ++pos;
    if (pos + 3 <= len) win = (win >> 8) | (uint32_t(__ldg(s + pos + 2)) << 16);
  }
  if (pos < len) {  // gave up: stored
    out_len[seg] = kStoredFlag | (len + 5);
    return;
  }
  put_litlen(w, 256);  // end of block
  if (final_seg) {
    w.align();
  } else {  // sync flush: an empty stored block ends the segment on a byte boundary
    w.put(0, 3);
    w.align();
    w.put(0x0000, 16);
    w.put(0xFFFF, 16);
  }
  // did not shrink: one stored block of the raw bytes, written by the gather
  out_len[seg] = w.pos > len + 5 ? (kStoredFlag | (len + 5)) : w.pos;
}

// One CTA per segment: the piece -> the stream at its offset.  Stored pieces
// (kStoredFlag) are built here from the input: BFINAL/BTYPE byte, LEN, NLEN,
// then the raw bytes, copied by the whole CTA.
__global__ void k_gather_segments(const uint8_t* __restrict__ in, uint64_t n_in,
                                  const uint8_t* __restrict__ slots,
                                  const uint32_t* __restrict__ out_len,
                                  const uint64_t* __restrict__ offset, uint8_t* __restrict__ out,
                                  int last_is_final) {
  const uint64_t seg = blockIdx.x;
  uint8_t* dst = out + offset[seg];
  const uint32_t v = out_len[seg];
  const uint32_t n = v & ~kStoredFlag;
  if (v & kStoredFlag) {
    const uint32_t len = n - 5;
    const uint8_t* s = in + seg * kSeg;
    if (threadIdx.x == 0) {
      dst[0] = (last_is_final && seg + 1 == gridDim.x) ? 1 : 0;
      dst[1] = uint8_t(len);
      dst[2] = uint8_t(len >> 8);
      dst[3] = uint8_t(~len);
      dst[4] = uint8_t((~len) >> 8);
    }
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) dst[5 + i] = __ldg(s + i);
    return;
  }
  const uint8_t* src = slots + seg * uint64_t(kSlot);
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

}  // namespace

extern "C" {

int crac_deflate_segments(const uint8_t* d_in, uint64_t n, uint8_t* d_slots, uint32_t* d_len,
                          uint32_t* d_adler, int last_is_final, void* stream) {
  const uint64_t n_seg = n ? (n + kSeg - 1) / kSeg : 0;
  if (!n_seg) return 0;
  k_deflate_segments<<<unsigned((n_seg + kThreads - 1) / kThreads), kThreads, 0,
                       cudaStream_t(stream)>>>(d_in, n, n_seg, d_slots, d_len, d_adler,
                                               last_is_final);
  return int(cudaGetLastError());
}

int crac_gather_segments(const uint8_t* d_in, uint64_t n, const uint8_t* d_slots,
                         const uint32_t* d_len, const uint64_t* d_offset, uint8_t* d_out,
                         int last_is_final, void* stream) {
  const uint64_t n_seg = n ? (n + kSeg - 1) / kSeg : 0;
  if (!n_seg) return 0;
  k_gather_segments<<<unsigned(n_seg), 256, 0, cudaStream_t(stream)>>>(
      d_in, n, d_slots, d_len, d_offset, d_out, last_is_final);
  return int(cudaGetLastError());
}

}  // extern "C"
