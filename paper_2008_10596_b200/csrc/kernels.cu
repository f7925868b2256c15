// sm_100a kernels of the checkpoint drain / restart refill.  C-ABI: crac_gpu.h.
//
// K1  k1_chunk_crc      zlib-identical CRC-32 per region-relative chunk
// K2a k_pack_records    framed section stream (ALLOC_PAYLOADS / UVM_PAGES) -> staging
// K3  k_scatter_records staging -> regions (restart refill)
// K2b k_diff_count / k_diff_write / k_gather   incremental dirty-chunk drain
//     k_fill_synth / k_mutate                  synthetic workload fixtures
//
// K1 design (HBM-bound target):
//   * one warp per chunk, rows of 512 B: lane i owns 16-byte word i of every
//     row, so every LDG.128 is fully coalesced (4 sectors per 512 B);
//   * each lane runs the CRC register over its column with slicing-by-4
//     lookups.  The 496-byte gap to its next word is folded into the tables
//     used for the 4th step of each word (group B = A^496 o group A), so the
//     whole chunk costs exactly one table lookup per byte;
//   * lane columns are combined with x^(128*(31-i)) mod P and a shuffle-XOR
//     reduction; the affine part K(n) finishes the zlib value;
//   * tables live in shared memory half-replicated (16 copies) and the two
//     half-warps always read different tables of a 256-byte row, so every
//     LDS is bank-conflict-free by construction; the PRMT instruction forms
//     each lookup address (byte << 8 | table/replica offset) in one ALU op.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <type_traits>
#include <vector>

#include "crac_gpu.h"
#include "crc_math.hpp"

namespace {

constexpr int kK1Threads = 512;
constexpr int kK1Warps = kK1Threads / 32;
constexpr uint32_t kTabWords = 2 * 256 * 64;  // 2 groups x 256 rows x 64 words = 128 KiB
constexpr uint32_t kTabBytes = kTabWords * 4;
constexpr uint32_t kGroupB = 256 * 64 * 4;    // byte offset of group B
constexpr uint32_t kRowGap = 496;             // bytes between a lane's words
// in-flight rows of the K1 variants that also compute the dirty-key lane: 16
// (the CRC-only depth) spills the key's registers (ptxas -v), 8 does not
constexpr int kKeyRows = 8;
// rows per chain of the paired (two chunks per warp) key-lane variants
constexpr int kKeyPairRows = 4;

__device__ uint32_t g_tab[kTabWords];  // smem image of the lookup tables
__device__ uint32_t g_t0[256];         // plain byte table
__device__ uint32_t g_xp16[33];        // x^(128 k) mod P, k = 0..32
__device__ uint32_t g_xpt[512];        // x^(8 t) mod P, t = 0..511
__device__ uint32_t g_pow2[64];        // x^(8 * 2^k) mod P

// ---------------------------------------------------------------------------
// host: table construction
// ---------------------------------------------------------------------------
struct HostTables {
  std::vector<uint32_t> tab, t0, xp16, xpt, pow2;
};

HostTables build_tables() {
  HostTables h;
  h.t0.resize(256);
  for (uint32_t b = 0; b < 256; ++b) {
    uint32_t c = b;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ crac::kCrcPoly : c >> 1;
    h.t0[b] = c;
  }
  h.pow2.resize(64);
  h.pow2[0] = 0x00800000u;  // x^8
  for (int k = 1; k < 64; ++k) h.pow2[k] = crac::gf_mul(h.pow2[k - 1], h.pow2[k - 1]);
  // position tables: byte p of a 4-byte step is followed by (3 - p) bytes
  uint32_t pos[4][256];
  for (int p = 0; p < 4; ++p)
    for (uint32_t b = 0; b < 256; ++b) pos[p][b] = crac::advance(h.t0[b], 3 - p, h.pow2.data());
  const uint32_t gap = crac::x8n(kRowGap, h.pow2.data());
  h.tab.assign(kTabWords, 0);
  for (int g = 0; g < 2; ++g)
    for (uint32_t b = 0; b < 256; ++b)
      for (int t = 0; t < 4; ++t) {
        const uint32_t v = g == 0 ? pos[t][b] : crac::gf_mul(gap, pos[t][b]);
        for (int r = 0; r < 16; ++r) h.tab[g * 256 * 64 + b * 64 + t * 16 + r] = v;
      }
  h.xp16.resize(33);
  for (int k = 0; k <= 32; ++k) h.xp16[k] = crac::x8n(16ull * k, h.pow2.data());
  h.xpt.resize(512);
  for (int t = 0; t < 512; ++t) h.xpt[t] = crac::x8n(t, h.pow2.data());
  return h;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

// Per-lane lookup addressing: lookup j of a step reads table t_j = (j + half)
// & 3 (the table of byte position t_j) at replica (lane & 15).
struct LaneLut {
  uint32_t base;    // shared address of the table image
  uint32_t lr[4];   // byte 0: t_j << 6 | replica << 2; bytes 1..3 zero
  uint32_t sel[4];  // PRMT selector: (x.byte t_j << 8) | lr.byte0
};

__device__ __forceinline__ LaneLut make_lut(uint32_t smem_base, uint32_t lane) {
  LaneLut l;
  l.base = smem_base;
  const uint32_t half = lane >> 4, rep = lane & 15;
  for (int j = 0; j < 4; ++j) {
    const uint32_t t = (j + half) & 3;
    l.lr[j] = (t << 6) | (rep << 2);
    l.sel[j] = 4u | (t << 4) | (5u << 8) | (5u << 12);
  }
  return l;
}

// One slicing-by-4 step: returns sum_p table_p[x.byte p] of table group g.
template <uint32_t kGroup>
__device__ __forceinline__ uint32_t step4(const LaneLut& l, uint32_t x) {
  const uint32_t a0 = lds32(l.base + kGroup + prmt(x, l.lr[0], l.sel[0]));
  const uint32_t a1 = lds32(l.base + kGroup + prmt(x, l.lr[1], l.sel[1]));
  const uint32_t a2 = lds32(l.base + kGroup + prmt(x, l.lr[2], l.sel[2]));
  const uint32_t a3 = lds32(l.base + kGroup + prmt(x, l.lr[3], l.sel[3]));
  return (a0 ^ a1) ^ (a2 ^ a3);
}

// Runs the CRC register over one 16-byte word; the final step uses group B
// (which also advances past the 496-byte gap) unless this is the last row.
template <bool kGap>
__device__ __forceinline__ uint32_t word16(const LaneLut& l, uint32_t s, uint4 w) {
  s = step4<0>(l, s ^ w.x);
  s = step4<0>(l, s ^ w.y);
  s = step4<0>(l, s ^ w.z);
  return step4<kGap ? kGroupB : 0>(l, s ^ w.w);
}

__device__ __forceinline__ uint32_t warp_xor(uint32_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v ^= __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

__device__ __forceinline__ uint32_t find_span(const uint64_t* chunk_first, uint32_t n_spans,
                                              uint64_t c) {
  uint32_t lo = 0, hi = n_spans;  // invariant: chunk_first[lo] <= c < chunk_first[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(chunk_first + mid) <= c) lo = mid;
    else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// byte-shift helper: the 16 bytes starting at byte d (0..15) of (a || b)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 shift16(uint4 a, uint4 b, uint32_t d) {
  uint32_t x0, x1, x2, x3, x4;
  switch (d >> 2) {
    case 0: x0 = a.x; x1 = a.y; x2 = a.z; x3 = a.w; x4 = b.x; break;
    case 1: x0 = a.y; x1 = a.z; x2 = a.w; x3 = b.x; x4 = b.y; break;
    case 2: x0 = a.z; x1 = a.w; x2 = b.x; x3 = b.y; x4 = b.z; break;
    default: x0 = a.w; x1 = b.x; x2 = b.y; x3 = b.z; x4 = b.w; break;
  }
  const uint32_t sh = (d & 3) * 8;
  uint4 r;
  r.x = __funnelshift_r(x0, x1, sh);
  r.y = __funnelshift_r(x1, x2, sh);
  r.z = __funnelshift_r(x2, x3, sh);
  r.w = __funnelshift_r(x3, x4, sh);
  return r;
}

__device__ __forceinline__ uint4 load_shifted(const uint8_t* p) {
  const uint64_t a = reinterpret_cast<uint64_t>(p);
  const uint4* q = reinterpret_cast<const uint4*>(a & ~uint64_t(15));
  const uint32_t d = uint32_t(a & 15);
  const uint4 lo = q[0];
  if (d == 0) return lo;
  return shift16(lo, q[1], d);
}

// Row sinks of k1_rows: called once per hashed row with the lane's word of
// that row and, when it is in registers, the lane's word of the next row.
struct NoSink {
  __device__ __forceinline__ void operator()(uint32_t, uint4, uint4, bool) const {}
};

// Second dirty-key lane (crac_gpu.h "chunk key"): an integer-arithmetic hash
// computed from the same registers as the CRC, so a change that preserves a
// chunk's CRC-32 (GF(2)-linear: four compensating bytes suffice) still
// changes the 64-bit dirty key (CRC, key) with probability ~1 - 2^-32.
// 16-byte word j of a chunk, (x, y, z, w), row r = j / 32, lane l = j % 32:
//   k = (l + 1) * 0x27D4EB2F + r * 0x9E3779B9
//   t = (x + k) * (y + 0x85EBCA6B) + (z + (k ^ 0xC2B2AE35)) * (w + 0x165667B1)
// (32 x 32 -> 64-bit products, sums mod 2^64); a trailing partial word is
// zero-padded; key = fold(mix64(sum ^ len * 0x9E3779B97F4A7C15)).  ~0.4
// integer op per byte beside the CRC's one table lookup per byte.
struct NoKey {
  __device__ __forceinline__ void add(uint32_t, uint4) {}
};
struct Key2 {
  uint64_t sum = 0;
  uint32_t kl = 0;  // (lane + 1) * 0x27D4EB2F
  __device__ __forceinline__ void add(uint32_t r, uint4 w) {
    const uint32_t k = kl + r * 0x9E3779B9u;
    sum += uint64_t(w.x + k) * (w.y + 0x85EBCA6Bu) + uint64_t(w.z + (k ^ 0xC2B2AE35u)) * (w.w + 0x165667B1u);
  }
};

__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

__device__ __forceinline__ uint32_t key_final(uint64_t sum, uint32_t len) {
  uint64_t x = sum ^ (uint64_t(len) * 0x9E3779B97F4A7C15ull);
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return uint32_t(x) ^ uint32_t(x >> 32);
}

__device__ __forceinline__ uint4 shfl4(uint4 v, uint32_t src) {
  v.x = __shfl_sync(0xFFFFFFFFu, v.x, src);
  v.y = __shfl_sync(0xFFFFFFFFu, v.y, src);
  v.z = __shfl_sync(0xFFFFFFFFu, v.z, src);
  v.w = __shfl_sync(0xFFFFFFFFu, v.w, src);
  return v;
}

// Hash + copy from registers: writes every 16-byte destination word that
// lies wholly inside [dst, dst + rows * 512) while the chunk is hashed, so
// the chunk is read from HBM once.  dst may be misaligned by m (uniform per
// chunk): lane i then writes the aligned word that takes the last m bytes
// of its word and the first 16 - m of lane i+1's (lane 31: of lane 0 in the
// next row).  The first 16 - m bytes and everything from rows * 512 - m on
// are left to the caller (byte-exact edges).  A re-read of the chunk after
// hashing instead costs 1.6x (64 GiB: 54.7 ms against 33.9 ms misaligned).
template <bool kAligned>  // kAligned: the caller guarantees m == 0 (no realignment code)
struct CopySink {
  uint8_t* dal;       // dst rounded down to 16 bytes
  const uint8_t* p0;  // this lane's word in row 0 (lane 0: the row's first word)
  uint32_t m, rows, lane;
  __device__ __forceinline__ void operator()(uint32_t r, uint4 w, uint4 nx, bool have_nx) const {
    if (kAligned || m == 0) {
      *reinterpret_cast<uint4*>(dal + r * 512 + 16 * lane) = w;
      return;
    }
    if (!have_nx && lane == 0 && r + 1 < rows) nx = ldg_stream(p0 + (r + 1) * 512);
    const uint4 y = shfl4(lane == 0 ? nx : w, (lane + 1) & 31);
    if (lane < 31 || r + 1 < rows)
      *reinterpret_cast<uint4*>(dal + r * 512 + 16 * (lane + 1)) = shift16(w, y, 16 - m);
  }
};

// Runs one lane's column over `rows` rows of 512 B starting at p (the lane's
// first word).  Loads of the next kRows rows are in flight while the current
// kRows rows are hashed.  The last row uses group A (no trailing gap).
template <int kRows, typename Sink, typename Key>
__device__ __forceinline__ uint32_t k1_rows(const LaneLut& lut, const uint8_t* p, uint32_t rows,
                                            const Sink& sink, Key& key) {
  uint32_t acc = 0, r = 0;
  if (rows >= uint32_t(kRows)) {
    uint4 cur[kRows];
#pragma unroll
    for (int k = 0; k < kRows; ++k) cur[k] = ldg_stream(p + k * 512);
    for (; r + 2 * kRows <= rows; r += kRows) {
      uint4 nxt[kRows];
#pragma unroll
      for (int k = 0; k < kRows; ++k) nxt[k] = ldg_stream(p + (r + kRows + k) * 512);
#pragma unroll
      for (int k = 0; k < kRows; ++k) {
        acc = word16<true>(lut, acc, cur[k]);
        key.add(r + k, cur[k]);
        sink(r + k, cur[k], k + 1 < kRows ? cur[(k + 1) % kRows] : nxt[0], true);
      }
#pragma unroll
      for (int k = 0; k < kRows; ++k) cur[k] = nxt[k];
    }
#pragma unroll
    for (int k = 0; k < kRows - 1; ++k) {
      acc = word16<true>(lut, acc, cur[k]);
      key.add(r + k, cur[k]);
      sink(r + k, cur[k], cur[k + 1], true);
    }
    acc = (r + kRows == rows) ? word16<false>(lut, acc, cur[kRows - 1])
                              : word16<true>(lut, acc, cur[kRows - 1]);
    key.add(r + kRows - 1, cur[kRows - 1]);
    sink(r + kRows - 1, cur[kRows - 1], cur[kRows - 1], false);
    r += kRows;
  }
  for (; r < rows; ++r) {
    const uint4 w = ldg_stream(p + r * 512);
    acc = (r + 1 == rows) ? word16<false>(lut, acc, w) : word16<true>(lut, acc, w);
    key.add(r, w);
    sink(r, w, w, false);
  }
  return acc;
}

// Two chunks of `rows` rows (rows % kRows == 0) hashed together by the same
// lanes: two independent CRC chains (and key lanes) per lane, interleaved so
// the lookups of one chain fill the latency of the other's.
template <int kRows, typename Key>
__device__ __forceinline__ void k1_rows2(const LaneLut& lut, const uint8_t* p0, const uint8_t* p1,
                                         uint32_t rows, Key& k0, Key& k1, uint32_t& a0,
                                         uint32_t& a1) {
  uint32_t acc0 = 0, acc1 = 0, r = 0;
  uint4 c0[kRows], c1[kRows];
#pragma unroll
  for (int k = 0; k < kRows; ++k) {
    c0[k] = ldg_stream(p0 + k * 512);
    c1[k] = ldg_stream(p1 + k * 512);
  }
  for (; r + 2 * kRows <= rows; r += kRows) {
    uint4 n0[kRows], n1[kRows];
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      n0[k] = ldg_stream(p0 + (r + kRows + k) * 512);
      n1[k] = ldg_stream(p1 + (r + kRows + k) * 512);
    }
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      acc0 = word16<true>(lut, acc0, c0[k]);
      acc1 = word16<true>(lut, acc1, c1[k]);
      k0.add(r + k, c0[k]);
      k1.add(r + k, c1[k]);
    }
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      c0[k] = n0[k];
      c1[k] = n1[k];
    }
  }
#pragma unroll
  for (int k = 0; k < kRows - 1; ++k) {
    acc0 = word16<true>(lut, acc0, c0[k]);
    acc1 = word16<true>(lut, acc1, c1[k]);
    k0.add(r + k, c0[k]);
    k1.add(r + k, c1[k]);
  }
  a0 = word16<false>(lut, acc0, c0[kRows - 1]);
  a1 = word16<false>(lut, acc1, c1[kRows - 1]);
  k0.add(r + kRows - 1, c0[kRows - 1]);
  k1.add(r + kRows - 1, c1[kRows - 1]);
}

// ---------------------------------------------------------------------------
// K1
// ---------------------------------------------------------------------------
// Fused incremental drain (K1 + K2b in one pass): after a chunk is hashed,
// the same warp compares it with the previous image's CRC and, if it changed,
// writes the chunk straight into the pinned host image at its final offset.
// PCIe writes of dirty chunks overlap the hashing of the others; no
// compaction list, no host round trip, one read of HBM (plus an L2/HBM
// re-read of dirty chunks only).
struct HashDrain {
  uint32_t* prev;                // previous chunk CRCs; updated for dirty chunks
  uint32_t* prev_key;            // previous chunk keys (second lane); may be null
  const uint64_t* dst_off;       // per span: image offset of its first payload byte
  uint8_t* host;                 // pinned image (UVA)
  unsigned long long* counters;  // [0] dirty chunks, [1] dirty bytes
  // kMode 4 (split drain): the last n_writers CTAs write the dirty chunks the
  // others push into `queue` (chunk index + 1, 0 = not yet); qctl[0] pushed,
  // qctl[1] claimed by writers, qctl[2] hasher warps finished
  unsigned long long* queue;
  unsigned long long* qctl;
  uint32_t n_writers;
  uint32_t bulk_writers;  // 1: writers move chunks with cp.async.bulk (TMA) where aligned
};


__device__ __forceinline__ void chunk_to_host(uint8_t* dst, const uint8_t* src, uint32_t len,
                                              uint32_t lane) {
  if ((reinterpret_cast<uint64_t>(dst) & 15) == 0) {
    const uint32_t words = len >> 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (uint32_t w0 = lane; w0 < words; w0 += 32 * 8) {
      uint4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (w0 + 32 * k < words) v[k] = s4[w0 + 32 * k];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (w0 + 32 * k < words) d4[w0 + 32 * k] = v[k];
    }
    for (uint32_t i = (words << 4) + lane; i < len; i += 32) dst[i] = src[i];
    return;
  }
  const uint32_t head = uint32_t((16 - (reinterpret_cast<uint64_t>(dst) & 15)) & 15);
  const uint32_t h = head < len ? head : len;
  for (uint32_t i = lane; i < h; i += 32) dst[i] = src[i];
  const uint32_t body = (len - h) >> 4;
  uint4* d4 = reinterpret_cast<uint4*>(dst + h);
  for (uint32_t w = lane; w < body; w += 32) d4[w] = load_shifted(src + h + 16 * w);
  for (uint32_t i = h + 16 * body + lane; i < len; i += 32) dst[i] = src[i];
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
// Bulk shared -> global copy (TMA engine; global may be pinned host memory
// through UVA) in the CTA's bulk group, and its completion waits.
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_le1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// One dirty chunk through the copy engine of the SM (cp.async.bulk): HBM ->
// this warp's two staging buffers -> pinned image, lane 0 issuing, the store
// of one piece overlapping the load of the next.  Needs 16-byte-aligned
// source, destination and length.
constexpr uint32_t kWriterPiece = 3584;  // x2 per warp x 16 warps + barriers fit 128 KiB
__device__ void chunk_to_host_bulk(uint8_t* dst, const uint8_t* src, uint32_t len,
                                   uint32_t stage0, uint32_t bar0, uint32_t& phase) {
  for (uint32_t o = 0, i = 0; o < len; o += kWriterPiece, ++i) {
    const uint32_t b = i & 1, n = min(kWriterPiece, len - o);
    const uint32_t stage = stage0 + b * kWriterPiece, bar = bar0 + 8 * b;
    bulk_wait_read_le1();  // the store that last read this buffer is done with it
    mbar_expect_tx(bar, n);
    bulk_g2s(stage, src + o, n, bar);
    mbar_wait(bar, (phase >> b) & 1);
    phase ^= 1u << b;
    bulk_s2g(dst + o, stage, n);
  }
}

// Split-drain writer warp: claims queue slots in order and copies each dirty
// chunk into the image; exits once every hasher warp has finished and no
// pushed slot is left.  Hashers never wait for writers, so the kernel cannot
// deadlock as long as n_writers < the CTAs the GPU can hold at once.
__device__ void drain_writer(const crac_span_t* __restrict__ spans,
                             const uint64_t* __restrict__ chunk_first, uint32_t n_spans,
                             uint32_t chunk_bytes, const HashDrain& hd, uint32_t hasher_warps,
                             uint32_t lane, bool bulk, uint32_t smem) {
  // bulk (TMA) mode: this warp's staging buffers and mbarriers in the CTA's
  // dynamic shared memory (writer CTAs never load the CRC tables)
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t stage0 = smem + warp * 2 * kWriterPiece;
  const uint32_t bar0 = smem + kK1Warps * 2 * kWriterPiece + warp * 16;
  uint32_t phase = 0;
  if (bulk && lane == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  struct Drain {
    bool on;
    uint32_t lane;
    __device__ ~Drain() {
      if (on && lane == 0) bulk_wait_all();  // staging must outlive its stores
    }
  } drain_guard{bulk, lane};
  for (;;) {
    unsigned long long slot = 0;
    if (lane == 0) slot = atomicAdd(&hd.qctl[1], 1ull);
    slot = __shfl_sync(0xFFFFFFFFu, slot, 0);
    unsigned long long v = 0;
    for (;;) {
      if (lane == 0) {
        v = *reinterpret_cast<volatile unsigned long long*>(&hd.queue[slot]);
        if (!v) {
          const unsigned long long done = *reinterpret_cast<volatile unsigned long long*>(&hd.qctl[2]);
          if (done == hasher_warps) {
            __threadfence();
            const unsigned long long tail =
                *reinterpret_cast<volatile unsigned long long*>(&hd.qctl[0]);
            v = *reinterpret_cast<volatile unsigned long long*>(&hd.queue[slot]);
            if (!v && slot >= tail) v = ~0ull;
          }
        }
      }
      v = __shfl_sync(0xFFFFFFFFu, v, 0);
      if (v) break;
      __nanosleep(256);
    }
    if (v == ~0ull) return;
    const uint64_t c = v - 1;
    const uint32_t s = find_span(chunk_first, n_spans, c);
    const crac_span_t sp = spans[s];
    const uint64_t off = (c - __ldg(chunk_first + s)) * chunk_bytes;
    const uint64_t rem = sp.len - off;
    const uint32_t len = rem < chunk_bytes ? uint32_t(rem) : chunk_bytes;
    uint8_t* dst = hd.host + hd.dst_off[s] + off;
    const uint8_t* src = reinterpret_cast<const uint8_t*>(sp.ptr + off);
    if (bulk && ((reinterpret_cast<uint64_t>(dst) | reinterpret_cast<uint64_t>(src) | len) & 15) == 0) {
      if (lane == 0) chunk_to_host_bulk(dst, src, len, stage0, bar0, phase);
      __syncwarp();
    } else {
      chunk_to_host(dst, src, len, lane);
    }
  }
}

// kMode: 0 hash only; 1 fused incremental drain (dirty chunks to the image);
// 2 hash + copy every chunk from registers (stall-reduced snapshot), every
// destination 16-byte aligned; 3 the same for any destination alignment;
// 4 split incremental drain (hashers push dirty chunks, writer CTAs copy).
// kKey: also the second dirty-key lane (Key2) into out_key[c] (and, in the
// drain modes, compared with / stored to hd.prev_key).
template <int kRows, int kMode, bool kKey, bool kPair = false>
__global__ void __launch_bounds__(kK1Threads, 1)
    k1_chunk_crc(const crac_span_t* __restrict__ spans, const uint64_t* __restrict__ chunk_first,
                 uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                 uint32_t* __restrict__ out, uint32_t* __restrict__ out_key, uint32_t k_full,
                 HashDrain hd) {
  extern __shared__ __align__(16) uint32_t s_tab[];
  const uint32_t lane = threadIdx.x & 31;
  // split drain: the writers are the LAST n_wr CTAs, so hashers (which never
  // wait) are dispatched first; a writer only spins once every hasher CTA
  // has been placed (crac_hash_drain_split checks they all fit at once)
  const uint32_t n_wr = kMode == 4 ? hd.n_writers : 0;
  if (kMode == 4 && blockIdx.x >= gridDim.x - n_wr) {
    drain_writer(spans, chunk_first, n_spans, chunk_bytes, hd, (gridDim.x - n_wr) * kK1Warps, lane,
                 hd.bulk_writers != 0, static_cast<uint32_t>(__cvta_generic_to_shared(s_tab)));
    return;
  }
  {
    const uint4* src = reinterpret_cast<const uint4*>(g_tab);
    uint4* dst = reinterpret_cast<uint4*>(s_tab);
    for (uint32_t i = threadIdx.x; i < kTabWords / 4; i += kK1Threads) dst[i] = src[i];
  }
  __syncthreads();
  const LaneLut lut = make_lut(static_cast<uint32_t>(__cvta_generic_to_shared(s_tab)), lane);
  const uint64_t gw = blockIdx.x * uint64_t(kK1Warps) + (threadIdx.x >> 5);
  const uint64_t tw = (gridDim.x - n_wr) * uint64_t(kK1Warps);
  const uint64_t total_chunks = c_hi - c_lo;
  const uint64_t c_begin = c_lo + total_chunks * gw / tw, c_end = c_lo + total_chunks * (gw + 1) / tw;
  if (c_begin >= c_end) {
    if (kMode == 4 && lane == 0) {
      __threadfence();
      atomicAdd(&hd.qctl[2], 1ull);
    }
    return;
  }

  // Post-hash work of one chunk: lane columns -> the chunk's zlib CRC (and
  // key), then the mode's output (CRC store / dirty compare + drain).
  auto finish = [&](uint64_t c, uint32_t s, uint32_t L, uint32_t K, uint32_t len,
                    const uint8_t* base, uint64_t off) {
    if (kMode == 0) {
      if (lane == 0) {
        out[c] = L;
        if constexpr (kKey) out_key[c] = K;
      }
      return;
    }
    const uint32_t crc = __shfl_sync(0xFFFFFFFFu, L, 0);
    if (lane == 0) out[c] = crc;
    bool changed = crc != hd.prev[c];
    if constexpr (kKey) {  // the 64-bit dirty key (CRC, key), when the caller keeps keys
      if (hd.prev_key) {
        if (lane == 0) out_key[c] = K;
        changed |= K != hd.prev_key[c];
      }
    }
    if (changed) {  // warp-uniform
      if (lane == 0) {
        hd.prev[c] = crc;
        if constexpr (kKey)
          if (hd.prev_key) hd.prev_key[c] = K;
        atomicAdd(&hd.counters[0], 1ull);
        atomicAdd(&hd.counters[1], (unsigned long long)len);
        if (kMode == 4) {  // hand the chunk to the writers and keep hashing
          const unsigned long long slot = atomicAdd(&hd.qctl[0], 1ull);
          *reinterpret_cast<volatile unsigned long long*>(&hd.queue[slot]) = c + 1;
          __threadfence();
        }
      }
      if (kMode != 4) chunk_to_host(hd.host + hd.dst_off[s] + off, base, len, lane);
    }
  };

  uint32_t s = find_span(chunk_first, n_spans, c_begin);
  uint64_t s_next = __ldg(chunk_first + s + 1);
  for (uint64_t c = c_begin; c < c_end; ++c) {
    while (c >= s_next) {
      ++s;
      s_next = __ldg(chunk_first + s + 1);
    }
    const crac_span_t sp = spans[s];
    const uint64_t off = (c - __ldg(chunk_first + s)) * chunk_bytes;
    const uint64_t rem_len = sp.len - off;
    const uint32_t len = rem_len < chunk_bytes ? uint32_t(rem_len) : chunk_bytes;
    const uint8_t* base = reinterpret_cast<const uint8_t*>(sp.ptr + off);
    const uint32_t rows = len >> 9;

    if constexpr (kPair) {
      // two whole chunks at once: two independent CRC chains per lane (the
      // chain is a serial PRMT -> LDS -> XOR dependency; ncu shows the warps
      // stalled on the lookups' latency, not on a pipe)
      if (len == chunk_bytes && rows % kRows == 0 && c + 1 < c_end) {
        uint32_t s1 = s;
        uint64_t s1_next = s_next;
        while (c + 1 >= s1_next) {
          ++s1;
          s1_next = __ldg(chunk_first + s1 + 1);
        }
        const crac_span_t sp1 = spans[s1];
        const uint64_t off1 = (c + 1 - __ldg(chunk_first + s1)) * chunk_bytes;
        if (sp1.len - off1 >= chunk_bytes) {
          const uint8_t* base1 = reinterpret_cast<const uint8_t*>(sp1.ptr + off1);
          std::conditional_t<kKey, Key2, NoKey> key0, key1;
          if constexpr (kKey) key0.kl = key1.kl = (lane + 1) * 0x27D4EB2Fu;
          uint32_t a0, a1;
          k1_rows2<kRows>(lut, base + lane * 16, base1 + lane * 16, rows, key0, key1, a0, a1);
          uint32_t L0 = warp_xor(crac::gf_mul(g_xp16[31 - lane], a0));
          uint32_t L1 = warp_xor(crac::gf_mul(g_xp16[31 - lane], a1));
          if (lane == 0) {
            L0 ^= k_full;
            L1 ^= k_full;
          }
          uint32_t K0 = 0, K1 = 0;
          if constexpr (kKey) {
            K0 = key_final(warp_sum64(key0.sum), len);
            K1 = key_final(warp_sum64(key1.sum), len);
          }
          finish(c, s, L0, K0, len, base, off);
          finish(c + 1, s1, L1, K1, len, base1, off1);
          ++c;
          s = s1;
          s_next = s1_next;
          continue;
        }
      }
    }

    // ---- main body: rows of 512 B, kRows-deep double-buffered loads ----
    uint32_t acc;
    uint8_t* dst = nullptr;
    std::conditional_t<kKey, Key2, NoKey> key;
    if constexpr (kKey) key.kl = (lane + 1) * 0x27D4EB2Fu;
    if ((kMode == 2 || kMode == 3)) {
      dst = hd.host + hd.dst_off[s] + off;
      const uint32_t m = uint32_t(reinterpret_cast<uint64_t>(dst) & 15);
      acc = k1_rows<kRows>(lut, base + lane * 16, rows,
                           CopySink<kMode == 2>{dst - m, base + lane * 16, m, rows, lane}, key);
    } else {
      acc = k1_rows<kRows>(lut, base + lane * 16, rows, NoSink{}, key);
    }
    uint32_t L = rows ? warp_xor(crac::gf_mul(g_xp16[31 - lane], acc)) : 0u;

    // ---- tail (< 512 B): whole words per lane, then bytes on lane 0 ----
    const uint32_t t = len & 511;
    if (t) {
      const uint32_t nt = t >> 4;
      uint32_t part = 0;
      if (lane < nt) {
        const uint4 w = *reinterpret_cast<const uint4*>(base + rows * 512 + lane * 16);
        part = crac::gf_mul(g_xp16[nt - 1 - lane], word16<false>(lut, 0u, w));
        key.add(rows, w);
      }
      uint32_t lt = warp_xor(part);
      if (lane == 0) {
        const uint8_t* tb = base + rows * 512 + nt * 16;
        uint4 pw = make_uint4(0, 0, 0, 0);  // the trailing partial word, zero-padded
        for (uint32_t i = 0; i < (t & 15); ++i) {
          lt = (lt >> 8) ^ g_t0[(lt ^ tb[i]) & 0xFFu];
          if constexpr (kKey) (&pw.x)[i >> 2] |= uint32_t(tb[i]) << (8 * (i & 3));
        }
        L = crac::gf_mul(g_xpt[t], L) ^ lt;
        if constexpr (kKey) {
          if (t & 15) {  // word j = 32 rows + nt: the key of lane slot nt
            Key2 tail;
            tail.kl = (nt + 1) * 0x27D4EB2Fu;
            tail.add(rows, pw);
            key.sum += tail.sum;
          }
        }
      }
    }
    if (lane == 0) L ^= (len == chunk_bytes ? k_full : crac::crc_affine(len, g_pow2));
    uint32_t K = 0;
    if constexpr (kKey) K = key_final(warp_sum64(key.sum), len);
    if ((kMode == 2 || kMode == 3)) {
      if (lane == 0) {
        out[c] = L;
        if constexpr (kKey) out_key[c] = K;
      }
      // byte-exact edges the register copy left: the head word (misaligned
      // destination), the m bytes of the last main row's straddling word,
      // and the tail (< 512 B, source aligned again)
      const uint32_t m = uint32_t(reinterpret_cast<uint64_t>(dst) & 15);
      if (rows == 0) {
        chunk_to_host(dst, base, len, lane);
        continue;
      }
      if (m && lane < 16 - m) dst[lane] = base[lane];
      if (m && lane < m) dst[rows * 512 - m + lane] = base[rows * 512 - m + lane];
      chunk_to_host(dst + rows * 512, base + rows * 512, len - rows * 512, lane);
      continue;
    }
    finish(c, s, L, K, len, base, off);
  }
  if (kMode == 4 && lane == 0) {
    __threadfence();
    atomicAdd(&hd.qctl[2], 1ull);
  }
}

// ---------------------------------------------------------------------------
// K1-TMA: the same hash with rows staged through shared memory by the bulk
// copy engine (cp.async.bulk + mbarrier) instead of register loads.  Kept as
// the measured alternative the north star names (CRAC_K1_TMA=A|B|C selects
// it for crac_chunk_crc32_range); DESIGN.md "K1 design" has the numbers.
// The 128 KiB of lookup tables leave <= 99 KiB for staging, and every staged
// word costs one extra LDS.128 on the shared-memory pipe the lookups already
// keep busy.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

template <int kWarps, int kStages, int kStageRows>
constexpr uint32_t k1_tma_smem() {
  return kTabBytes + kWarps * kStages * kStageRows * 512 + kWarps * kStages * 8;
}

template <int kWarps, int kStages, int kStageRows>
__global__ void __launch_bounds__(kWarps * 32, 1)
    k1_chunk_crc_tma(const crac_span_t* __restrict__ spans, const uint64_t* __restrict__ chunk_first,
                     uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                     uint32_t* __restrict__ out, uint32_t k_full) {
  extern __shared__ __align__(128) uint32_t s_tab[];
  {
    const uint4* src = reinterpret_cast<const uint4*>(g_tab);
    uint4* dst = reinterpret_cast<uint4*>(s_tab);
    for (uint32_t i = threadIdx.x; i < kTabWords / 4; i += kWarps * 32) dst[i] = src[i];
  }
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t smem0 = static_cast<uint32_t>(__cvta_generic_to_shared(s_tab));
  constexpr uint32_t kStageBytes = kStageRows * 512;
  const uint32_t stage0 = smem0 + kTabBytes + warp * kStages * kStageBytes;
  const uint32_t bar0 = smem0 + kTabBytes + kWarps * kStages * kStageBytes + warp * kStages * 8;
  if (lane == 0) {
    for (int k = 0; k < kStages; ++k) mbar_init(bar0 + 8 * k, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const LaneLut lut = make_lut(smem0, lane);
  const uint64_t gw = blockIdx.x * uint64_t(kWarps) + warp;
  const uint64_t tw = gridDim.x * uint64_t(kWarps);
  const uint64_t total_chunks = c_hi - c_lo;
  const uint64_t c_begin = c_lo + total_chunks * gw / tw, c_end = c_lo + total_chunks * (gw + 1) / tw;
  if (c_begin >= c_end) return;

  // producer cursor (lane 0 issues; all lanes track it): chunk pc, stage pst
  uint64_t pc = c_begin;
  uint32_t ps = find_span(chunk_first, n_spans, pc);
  uint32_t pst = 0, issued = 0;
  auto chunk_rows = [&](uint64_t c, uint32_t s) -> uint32_t {
    const uint64_t off = (c - __ldg(chunk_first + s)) * chunk_bytes;
    const uint64_t rem = spans[s].len - off;
    return uint32_t((rem < chunk_bytes ? rem : chunk_bytes) >> 9);
  };
  auto issue = [&]() {  // next stage of the producer cursor, if any
    while (pc < c_end) {
      while (pc >= __ldg(chunk_first + ps + 1)) ++ps;
      const uint32_t rows = chunk_rows(pc, ps);
      if (pst * kStageRows < rows) {
        const uint32_t nr = min(uint32_t(kStageRows), rows - pst * kStageRows);
        const uint8_t* src = reinterpret_cast<const uint8_t*>(spans[ps].ptr) +
                             (pc - __ldg(chunk_first + ps)) * chunk_bytes + pst * kStageBytes;
        const uint32_t slot = issued % kStages;
        if (lane == 0) {
          mbar_expect_tx(bar0 + 8 * slot, nr * 512);
          bulk_g2s(stage0 + slot * kStageBytes, src, nr * 512, bar0 + 8 * slot);
        }
        ++issued;
        ++pst;
        return;
      }
      ++pc;
      pst = 0;
    }
  };
  for (int k = 0; k < kStages; ++k) issue();

  uint32_t consumed = 0;
  uint32_t s = find_span(chunk_first, n_spans, c_begin);
  for (uint64_t c = c_begin; c < c_end; ++c) {
    while (c >= __ldg(chunk_first + s + 1)) ++s;
    const crac_span_t sp = spans[s];
    const uint64_t off = (c - __ldg(chunk_first + s)) * chunk_bytes;
    const uint64_t rem_len = sp.len - off;
    const uint32_t len = rem_len < chunk_bytes ? uint32_t(rem_len) : chunk_bytes;
    const uint8_t* base = reinterpret_cast<const uint8_t*>(sp.ptr + off);
    const uint32_t rows = len >> 9;
    uint32_t acc = 0;
    for (uint32_t r0 = 0; r0 < rows; r0 += kStageRows) {
      const uint32_t slot = consumed % kStages, parity = (consumed / kStages) & 1;
      mbar_wait(bar0 + 8 * slot, parity);
      const uint32_t nr = min(uint32_t(kStageRows), rows - r0);
      const uint32_t buf = stage0 + slot * kStageBytes + lane * 16;
#pragma unroll
      for (uint32_t k = 0; k < uint32_t(kStageRows); ++k) {
        if (k < nr) {
          const uint4 w = lds128(buf + k * 512);
          acc = (r0 + k + 1 == rows) ? word16<false>(lut, acc, w) : word16<true>(lut, acc, w);
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      ++consumed;
      issue();
    }
    uint32_t L = rows ? warp_xor(crac::gf_mul(g_xp16[31 - lane], acc)) : 0u;
    const uint32_t t = len & 511;
    if (t) {
      const uint32_t nt = t >> 4;
      uint32_t part = 0;
      if (lane < nt) {
        const uint4 w = *reinterpret_cast<const uint4*>(base + rows * 512 + lane * 16);
        part = crac::gf_mul(g_xp16[nt - 1 - lane], word16<false>(lut, 0u, w));
      }
      uint32_t lt = warp_xor(part);
      if (lane == 0) {
        const uint8_t* tb = base + rows * 512 + nt * 16;
        for (uint32_t i = 0; i < (t & 15); ++i) lt = (lt >> 8) ^ g_t0[(lt ^ tb[i]) & 0xFFu];
        L = crac::gf_mul(g_xpt[t], L) ^ lt;
      }
    }
    if (lane == 0) out[c] = L ^ (len == chunk_bytes ? k_full : crac::crc_affine(len, g_pow2));
  }
}

__device__ __forceinline__ void set_byte(uint4& v, uint32_t i, uint32_t b) {
  const uint32_t sh = (i & 3) * 8, keep = ~(0xFFu << sh), put = b << sh;
  switch (i >> 2) {  // register-resident (no local-memory indexing)
    case 0: v.x = (v.x & keep) | put; break;
    case 1: v.y = (v.y & keep) | put; break;
    case 2: v.z = (v.z & keep) | put; break;
    default: v.w = (v.w & keep) | put; break;
  }
}

// Zeroes bytes [valid, 16) of v.
__device__ __forceinline__ void keep_prefix(uint4& v, uint32_t valid) {
  auto mask = [&](uint32_t word) -> uint32_t {
    const int n = int(valid) - int(4 * word);  // valid bytes in this word
    return n >= 4 ? 0xFFFFFFFFu : n <= 0 ? 0u : (0xFFFFFFFFu >> (32 - 8 * n));
  };
  v.x &= mask(0);
  v.y &= mask(1);
  v.z &= mask(2);
  v.w &= mask(3);
}

constexpr int kPackThreads = 512;
constexpr uint32_t kSubTile = 512;
constexpr uint32_t kTileWords = CRAC_TILE_BYTES / 16;             // 4096

__device__ __forceinline__ uint4 shfl_down4(uint4 v, int d) {
  v.x = __shfl_down_sync(0xFFFFFFFFu, v.x, d);
  v.y = __shfl_down_sync(0xFFFFFFFFu, v.y, d);
  v.z = __shfl_down_sync(0xFFFFFFFFu, v.z, d);
  v.w = __shfl_down_sync(0xFFFFFFFFu, v.w, d);
  return v;
}

// Copies `nwords` 16-byte words dst[i] = bytes [16 i + shift, +16) of the
// 16-byte-aligned source `src` (shift 0..15 uniform).  Thread t owns words
// t, t + 256, ... (coalesced); all loads are issued before any store, and
// the upper half of a misaligned word comes from the neighbouring lane.
template <uint32_t kThreads>
__device__ __forceinline__ void tile_copy(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                          uint32_t nwords, uint32_t shift) {
  const uint32_t lane = threadIdx.x & 31;
  constexpr uint32_t kWords = kTileWords / kThreads;  // per thread
  uint4 lo[kWords];
#pragma unroll
  for (uint32_t k = 0; k < kWords; ++k) {
    const uint32_t w = threadIdx.x + k * kThreads;
    // one word past the end when misaligned: it is the upper half of the
    // last word, inside the source's 16-byte-rounded extent
    if (w < nwords || (shift && w == nwords)) lo[k] = ldg_stream(src + w);
  }
  if (shift == 0) {
#pragma unroll
    for (uint32_t k = 0; k < kWords; ++k) {
      const uint32_t w = threadIdx.x + k * kThreads;
      if (w < nwords) dst[w] = lo[k];
    }
    return;
  }
#pragma unroll
  for (uint32_t k = 0; k < kWords; ++k) {
    const uint32_t w = threadIdx.x + k * kThreads;
    uint4 hi = shfl_down4(lo[k], 1);
    if (lane == 31 && w < nwords) hi = ldg_stream(src + w + 1);
    if (w < nwords) dst[w] = shift16(lo[k], hi, shift);
  }
}

// Byte at stream position x, walking the record cursor forward from r.
__device__ __forceinline__ uint32_t stream_byte(const crac_record_t* recs, uint32_t n,
                                                uint32_t& r, uint64_t x) {
  while (r + 1 < n && __ldg(&recs[r + 1].out_off) <= x) ++r;
  const crac_record_t& R = recs[r];
  if (x < R.out_off) return 0;
  const uint64_t rel = x - R.out_off;
  if (rel < R.frame_len) return R.frame[rel];
  const uint64_t pl = rel - R.frame_len;
  if (pl < R.len && R.ptr) return reinterpret_cast<const uint8_t*>(R.ptr)[pl];
  return 0;  // outside any record, or host-filled content (ptr == 0)
}

// ---------------------------------------------------------------------------
// K2a: pack
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kPackThreads)
    k_pack_records(const crac_record_t* __restrict__ recs, uint32_t n,
                   const uint32_t* __restrict__ tile_rec, uint64_t win_off, uint64_t win_len,
                   uint8_t* __restrict__ dst) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t tile0 = win_off + uint64_t(blockIdx.x) * CRAC_TILE_BYTES;
  const uint64_t win_end = win_off + win_len;
  const uint64_t tile1 = min(tile0 + CRAC_TILE_BYTES, win_end);
  uint32_t rec = tile_rec[blockIdx.x];
  while (rec + 1 < n && __ldg(&recs[rec + 1].out_off) <= tile0) ++rec;
  {
    // whole tile inside one payload (the common case for large regions)
    const crac_record_t& R = recs[rec];
    const uint64_t P = R.out_off + R.frame_len;
    if (P <= tile0 && tile1 <= P + R.len) {
      if (!R.ptr) {  // host-filled content: the host writes it after the D2H
        uint4* o = reinterpret_cast<uint4*>(dst + (tile0 - win_off));
        for (uint32_t w = threadIdx.x; w < ((tile1 - tile0 + 15) >> 4); w += kPackThreads)
          o[w] = make_uint4(0, 0, 0, 0);
        return;
      }
      const uint64_t rel = tile0 - P;
      tile_copy<kPackThreads>(reinterpret_cast<uint4*>(dst + (tile0 - win_off)),
                reinterpret_cast<const uint4*>(R.ptr) + (rel >> 4),
                uint32_t((tile1 - tile0 + 15) >> 4), uint32_t(rel & 15));
      return;
    }
  }
  for (uint32_t st = warp; st < CRAC_TILE_BYTES / kSubTile; st += kPackThreads / 32) {
    const uint64_t o = tile0 + uint64_t(st) * kSubTile;
    if (o >= win_end) break;
    while (rec + 1 < n && __ldg(&recs[rec + 1].out_off) <= o) ++rec;
    const uint64_t x = o + lane * 16;
    uint4* out = reinterpret_cast<uint4*>(dst + (x - win_off));
    const crac_record_t& R = recs[rec];
    const uint64_t P = R.out_off + R.frame_len;
    if (o >= P && o + kSubTile <= P + R.len) {
      // whole sub-tile inside one payload: aligned stores, shifted loads
      if (x < win_end)
        *out = R.ptr ? load_shifted(reinterpret_cast<const uint8_t*>(R.ptr) + (x - P))
                     : make_uint4(0, 0, 0, 0);
    } else if (x < win_end) {
      uint32_t r = rec;
      uint4 v = make_uint4(0, 0, 0, 0);
#pragma unroll
      for (uint32_t i = 0; i < 16; ++i) set_byte(v, i, stream_byte(recs, n, r, x + i));
      *out = v;
    }
  }
}

// Frame bytes of records [0, n) at dst + out_off, byte by byte: the words
// they share with payload bytes are written by other warps (the hash+copy
// pass), so nothing outside the frame may be stored.
__global__ void k_write_frames(const crac_record_t* __restrict__ recs, uint32_t n,
                               uint8_t* __restrict__ dst) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t r = i / 32, b = i % 32;
  if (r >= n) return;
  const crac_record_t& R = recs[r];
  if (b < R.frame_len) dst[R.out_off + b] = R.frame[b];
}

// ---------------------------------------------------------------------------
// K3: scatter
// ---------------------------------------------------------------------------
// Destination word of record R whose first stream byte lies in [x, x + 16):
// returns its index or UINT64_MAX.
__device__ __forceinline__ uint64_t dest_word_at(const crac_record_t& R, uint64_t x) {
  const uint64_t P = R.out_off + R.frame_len;
  if (R.len == 0) return ~0ull;
  const uint64_t d = x <= P ? 0 : (x - P + 15) >> 4;
  const uint64_t f = P + 16 * d;
  if (f >= x + 16 || 16 * d >= R.len) return ~0ull;
  return d;
}

__global__ void __launch_bounds__(kPackThreads)
    k_scatter_records(const crac_record_t* __restrict__ recs, uint32_t n,
                      const uint32_t* __restrict__ tile_rec, const uint8_t* __restrict__ win,
                      uint64_t win_off, uint64_t win_len) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t tile0 = win_off + uint64_t(blockIdx.x) * CRAC_TILE_BYTES;
  const uint64_t win_end = win_off + win_len;
  const uint64_t tile1 = min(tile0 + CRAC_TILE_BYTES, win_end);
  uint32_t rec = tile_rec[blockIdx.x];
  while (rec + 1 < n && __ldg(&recs[rec + 1].out_off) <= tile0) ++rec;
  {
    // every destination word starting in this tile is a full data word of
    // one record: the words are consecutive, sources share one misalignment
    const crac_record_t& R = recs[rec];
    const uint64_t P = R.out_off + R.frame_len;
    if (P <= tile0 && tile1 + 16 <= P + R.len) {
      if (!R.ptr) return;  // host-filled content
      const uint64_t d0 = (tile0 - P + 15) >> 4;                 // first dest word
      const uint64_t d1 = (tile1 - P + 15) >> 4;                 // one past the last
      const uint64_t f0 = P + 16 * d0 - win_off;                 // its window offset
      tile_copy<kPackThreads>(reinterpret_cast<uint4*>(R.ptr) + d0,
                reinterpret_cast<const uint4*>(win) + (f0 >> 4), uint32_t(d1 - d0),
                uint32_t(f0 & 15));
      return;
    }
  }
  for (uint32_t st = warp; st < CRAC_TILE_BYTES / kSubTile; st += kPackThreads / 32) {
    const uint64_t o = tile0 + uint64_t(st) * kSubTile;
    if (o >= win_end) break;
    while (rec + 1 < n && __ldg(&recs[rec + 1].out_off) <= o) ++rec;
    const uint64_t x = o + lane * 16;
    const crac_record_t& R = recs[rec];
    const uint64_t P = R.out_off + R.frame_len;
    if (o >= P && o + kSubTile + 16 <= P + R.len) {
      // fast path: every lane owns one full data word of R
      if (!R.ptr) continue;
      const uint64_t d = (x - P + 15) >> 4;
      const uint64_t f = P + 16 * d;
      *reinterpret_cast<uint4*>(R.ptr + 16 * d) = load_shifted(win + (f - win_off));
      continue;
    }
    if (x >= win_end) continue;
    // slow path: the record owning a destination word that starts in [x, x+16)
    uint32_t r = rec;
    while (r + 1 < n && __ldg(&recs[r + 1].out_off) <= x + 15) ++r;
    uint64_t d = dest_word_at(recs[r], x);
    if (d == ~0ull && r > 0) {
      --r;
      d = dest_word_at(recs[r], x);
    }
    if (d == ~0ull) continue;
    const crac_record_t& Q = recs[r];
    if (!Q.ptr) continue;  // host-filled content
    const uint64_t Pq = Q.out_off + Q.frame_len;
    const uint64_t f = Pq + 16 * d;
    uint4 v = load_shifted(win + (f - win_off));
    const uint64_t valid = Q.len - 16 * d;  // >= 1
    if (valid < 16) keep_prefix(v, uint32_t(valid));
    uint4* dstw = reinterpret_cast<uint4*>(Q.ptr) + d;
    *dstw = v;
    if (16 * (d + 1) >= Q.len) {  // last data word: zero the padding words
      const uint4 z = make_uint4(0, 0, 0, 0);
      for (uint64_t e = d + 1; 16 * e < Q.ext; ++e) dstw[e - d] = z;
    }
  }
}

// ---------------------------------------------------------------------------
// K4: section CRCs on the device
// ---------------------------------------------------------------------------
// crc(S) = L(S) ^ K(|S|) and L(S) = XOR over pieces p of A^(bytes after p)(L(p)),
// L(p) = crc(p) ^ K(|p|).  One thread per piece (a payload chunk, a page, or a
// 16-byte frame) computes its shifted linear term; the XOR is reduced per
// warp and folded into out[section] with one atomic.  The host applies the
// final K(|S|).  Record `reserved` carries the index of the record's first
// CRC (payload span index for ALLOC_PAYLOADS records, page index for pages).
constexpr int kFoldThreads = 256;

__device__ __forceinline__ uint32_t frame_linear(const uint8_t* f, uint32_t n) {
  uint32_t s = 0;
  for (uint32_t i = 0; i < n; ++i) s = (s >> 8) ^ g_t0[(s ^ f[i]) & 0xFFu];
  return s;
}

__global__ void __launch_bounds__(kFoldThreads)
    k_fold_sections(const crac_record_t* __restrict__ recs, uint32_t n_recs,
                    const uint64_t* __restrict__ pay_first, const uint32_t* __restrict__ pay_crc,
                    uint32_t n_pay, const uint32_t* __restrict__ page_crc, uint64_t len3,
                    uint64_t total_chunks, uint32_t* __restrict__ out) {
  const uint64_t t = blockIdx.x * uint64_t(kFoldThreads) + threadIdx.x;
  uint32_t term = 0;
  int sec = -1;
  if (t < total_chunks) {
    // an ALLOC_PAYLOADS chunk
    const uint32_t s = find_span(pay_first, n_pay, t);
    const crac_record_t& R = recs[s];
    const uint64_t off = (t - pay_first[s]) * 65536ull;
    const uint64_t len = min(uint64_t(65536), R.len - off);
    const uint64_t end = R.out_off + R.frame_len + off + len;
    term = crac::advance(pay_crc[t] ^ crac::crc_affine(len, g_pow2), len3 - end, g_pow2);
    sec = 0;
  } else if (t - total_chunks < n_recs) {
    const crac_record_t& R = recs[t - total_chunks];
    if (R.out_off < len3) {  // an ALLOC_PAYLOADS frame
      term = crac::advance(frame_linear(R.frame, 16), len3 - (R.out_off + 16), g_pow2);
      sec = 0;
    } else if (R.out_off >= len3 + 20) {  // a UVM_PAGES header or page
      // sec4 offsets are relative to the first byte after the 20-byte gap;
      // the section end is the end of the stream (the last record's end)
      const crac_record_t& last = recs[n_recs - 1];
      const uint64_t sec_end = last.out_off + last.frame_len + last.len;
      uint32_t l = crac::advance(frame_linear(R.frame, 16), R.len, g_pow2);
      if (R.len) l ^= page_crc[R.reserved] ^ crac::crc_affine(R.len, g_pow2);
      term = crac::advance(l, sec_end - (R.out_off + 16 + R.len), g_pow2);
      sec = 1;
    }
  }
  // reduce per warp and section
  const uint32_t lane = threadIdx.x & 31;
  for (int which = 0; which < 2; ++which) {
    uint32_t v = sec == which ? term : 0u;
    for (int o = 16; o; o >>= 1) v ^= __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0 && v) atomicXor(out + which, v);
  }
}

// ---------------------------------------------------------------------------
// K2b: dirty detection + compaction + gather
// ---------------------------------------------------------------------------
constexpr int kDiffThreads = 256;
constexpr uint32_t kDiffPerThread = 16;
constexpr uint32_t kDiffPerBlock = kDiffThreads * kDiffPerThread;  // 4096

__global__ void __launch_bounds__(kDiffThreads)
    k_diff_count(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t n,
                 uint32_t* __restrict__ block_counts) {
  const uint64_t i0 = uint64_t(blockIdx.x) * kDiffPerBlock + threadIdx.x * kDiffPerThread;
  uint32_t cnt = 0;
  for (uint32_t k = 0; k < kDiffPerThread; ++k) {
    const uint64_t i = i0 + k;
    if (i < n && a[i] != b[i]) ++cnt;
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  __shared__ uint32_t ws[kDiffThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kDiffThreads / 32; ++w) t += ws[w];
    block_counts[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(kDiffThreads)
    k_diff_write(const uint32_t* __restrict__ a, uint32_t* __restrict__ b, uint64_t n,
                 const uint32_t* __restrict__ block_counts, uint64_t* __restrict__ idx,
                 uint64_t* __restrict__ count, uint64_t index_base) {
  __shared__ uint64_t s_base;
  __shared__ uint32_t s_warp[kDiffThreads / 32];
  // block offset = sum of the counts of all preceding blocks
  uint64_t part = 0;
  for (uint32_t k = threadIdx.x; k < blockIdx.x; k += kDiffThreads) part += block_counts[k];
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, o);
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_base), part);

  const uint64_t i0 = uint64_t(blockIdx.x) * kDiffPerBlock + threadIdx.x * kDiffPerThread;
  uint32_t mask = 0;
  for (uint32_t k = 0; k < kDiffPerThread; ++k) {
    const uint64_t i = i0 + k;
    if (i < n && a[i] != b[i]) mask |= 1u << k;
  }
  const uint32_t mine = __popc(mask);
  // exclusive scan of `mine` across the block
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t before = 0;
  for (uint32_t w = 0; w < warp; ++w) before += s_warp[w];
  uint64_t pos = s_base + before + incl - mine;
  for (uint32_t k = 0; k < kDiffPerThread; ++k)
    if (mask & (1u << k)) idx[pos++] = index_base + i0 + k;
  if (blockIdx.x + 1 == gridDim.x && threadIdx.x == kDiffThreads - 1) *count = pos;
  __syncthreads();
  for (uint32_t k = 0; k < kDiffPerThread; ++k) {
    const uint64_t i = i0 + k;
    if (i < n) b[i] = a[i];
  }
}

constexpr int kGatherThreads = 256;

__global__ void __launch_bounds__(kGatherThreads)
    k_gather(const crac_span_t* __restrict__ spans, const uint64_t* __restrict__ chunk_first,
             uint32_t n_spans, uint32_t chunk_bytes, const uint64_t* __restrict__ dirty,
             uint64_t first, uint64_t count, uint8_t* __restrict__ staging) {
  for (uint64_t k = blockIdx.x; k < count; k += gridDim.x) {
    const uint64_t c = dirty[first + k];
    const uint32_t s = find_span(chunk_first, n_spans, c);
    const crac_span_t sp = spans[s];
    const uint64_t off = (c - chunk_first[s]) * chunk_bytes;
    const uint64_t len = min(uint64_t(chunk_bytes), sp.len - off);
    const uint4* src = reinterpret_cast<const uint4*>(sp.ptr + off);
    uint4* dst = reinterpret_cast<uint4*>(staging + k * chunk_bytes);
    const uint64_t words = (len + 15) >> 4;
    for (uint64_t w = threadIdx.x; w < words; w += kGatherThreads) dst[w] = ldg_stream(src + w);
  }
}

// Dirty chunks written by the SMs straight into the pinned image.  The host
// destination may be misaligned: aligned 16-byte stores cover the interior,
// byte stores the two edges.
__global__ void __launch_bounds__(kGatherThreads)
    k_gather_to_host(const crac_span_t* __restrict__ spans, const uint64_t* __restrict__ chunk_first,
                     uint32_t n_spans, uint32_t chunk_bytes, const uint64_t* __restrict__ dirty,
                     uint64_t first, uint64_t count, const uint64_t* __restrict__ d_count,
                     const uint64_t* __restrict__ dst_off, uint8_t* __restrict__ host) {
  if (d_count) count = min(count, *d_count);  // produced on the device by the diff
  for (uint64_t k = blockIdx.x; k < count; k += gridDim.x) {
    const uint64_t c = dirty[first + k];
    const uint32_t s = find_span(chunk_first, n_spans, c);
    const crac_span_t sp = spans[s];
    const uint64_t off = (c - chunk_first[s]) * chunk_bytes;
    const uint64_t len = min(uint64_t(chunk_bytes), sp.len - off);
    const uint8_t* src = reinterpret_cast<const uint8_t*>(sp.ptr + off);
    uint8_t* dst = host + dst_off[s] + off;
    if ((reinterpret_cast<uint64_t>(dst) & 15) == 0 && len == kTileWords * 16) {
      // aligned full chunk: every load in flight before the PCIe stores
      tile_copy<kGatherThreads>(reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src),
                                kTileWords, 0);
      continue;
    }
    const uint32_t head = uint32_t((16 - (reinterpret_cast<uint64_t>(dst) & 15)) & 15);
    const uint32_t h = uint32_t(min(uint64_t(head), len));
    for (uint32_t i = threadIdx.x; i < h; i += kGatherThreads) dst[i] = src[i];
    const uint64_t body = (len - h) >> 4;
    uint4* d4 = reinterpret_cast<uint4*>(dst + h);
    for (uint64_t w = threadIdx.x; w < body; w += kGatherThreads)
      d4[w] = load_shifted(src + h + 16 * w);
    for (uint64_t i = h + 16 * body + threadIdx.x; i < len; i += kGatherThreads) dst[i] = src[i];
  }
}

// ---------------------------------------------------------------------------
// fixtures
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t crac_mix64(uint64_t x) {  // common.hpp:55-60
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t synth_word(uint64_t seed, uint64_t id, uint64_t k) {
  return crac_mix64(k + 0x1000003ull * id + (seed << 56));
}

__global__ void k_fill_synth(uint8_t* __restrict__ dst, uint64_t len, uint64_t seed, uint64_t id,
                             uint64_t word_offset) {
  const uint64_t words = len / 8;
  const uint64_t pairs = words / 2;
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < pairs;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t w0 = synth_word(seed, id, word_offset + 2 * i);
    const uint64_t w1 = synth_word(seed, id, word_offset + 2 * i + 1);
    d4[i] = make_uint4(uint32_t(w0), uint32_t(w0 >> 32), uint32_t(w1), uint32_t(w1 >> 32));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (uint64_t k = 2 * pairs; k * 8 < len; ++k) {
      const uint64_t w = synth_word(seed, id, word_offset + k);
      for (uint32_t b = 0; b < 8 && k * 8 + b < len; ++b) dst[k * 8 + b] = uint8_t(w >> (8 * b));
    }
  }
}

// Restart check against regenerated content (bench "verified", tests): sets
// *flag = 1 if any byte of the allocation differs from synth_word.
__global__ void k_verify_synth(const uint8_t* __restrict__ src, uint64_t len, uint64_t seed,
                               uint64_t id, uint32_t* __restrict__ flag) {
  const uint64_t pairs = len / 16;
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint32_t diff = 0;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < pairs;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint4 v = ldg_stream(s4 + i);
    const uint64_t w0 = synth_word(seed, id, 2 * i), w1 = synth_word(seed, id, 2 * i + 1);
    diff |= (v.x ^ uint32_t(w0)) | (v.y ^ uint32_t(w0 >> 32)) | (v.z ^ uint32_t(w1)) |
            (v.w ^ uint32_t(w1 >> 32));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (uint64_t b = pairs * 16; b < len; ++b)
      diff |= src[b] ^ uint8_t(synth_word(seed, id, b / 8) >> (8 * (b % 8)));
  if (__syncthreads_or(diff != 0) && threadIdx.x == 0) *flag = 1u;
}

// Managed-populate ceiling probe (crac_probe_managed_populate): writes the
// even `run`-byte runs of a fresh managed range (first touch on the GPU).
__global__ void k_touch_even_runs(uint8_t* p, uint64_t n, uint64_t run) {
  for (uint64_t i = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) * 16; i < n;
       i += uint64_t(gridDim.x) * blockDim.x * 16)
    if (((i / run) & 1) == 0) *reinterpret_cast<uint4*>(p + i) = make_uint4(1, 2, 3, 4);
}

__global__ void k_mutate(const crac_span_t* __restrict__ spans, const uint64_t* __restrict__ ids,
                         const uint64_t* __restrict__ chunk_first, uint32_t n_spans,
                         uint32_t chunk_bytes, uint64_t total_chunks, uint64_t seed,
                         uint64_t epoch, uint64_t threshold) {
  for (uint64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
    if (crac_mix64(seed ^ (epoch << 40) ^ c) >= threshold) continue;
    const uint32_t s = find_span(chunk_first, n_spans, c);
    const crac_span_t sp = spans[s];
    const uint64_t off = (c - chunk_first[s]) * chunk_bytes;
    const uint64_t len = min(uint64_t(chunk_bytes), sp.len - off);
    uint8_t* dst = reinterpret_cast<uint8_t*>(sp.ptr + off);
    const uint64_t words = len / 8;
    for (uint64_t k = threadIdx.x; k < words; k += blockDim.x) {
      const uint64_t w = synth_word(seed + epoch, ids[s], off / 8 + k);
      reinterpret_cast<uint64_t*>(dst)[k] = w;
    }
    if (threadIdx.x == 0)
      for (uint64_t b = words * 8; b < len; ++b)
        dst[b] = uint8_t(synth_word(seed + epoch, ids[s], off / 8 + words) >> (8 * (b - words * 8)));
  }
}

std::once_flag g_init_once;
int g_init_rc = 0;
uint32_t g_k_full_cache_bytes = 0;
uint32_t g_k_full_cache = 0;
std::mutex g_kfull_mu;

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

// The split drain's writers move 16-byte-aligned dirty chunks with
// cp.async.bulk (TMA: HBM -> shared -> pinned image), unaligned ones with SM
// stores.  C5 at 64 GiB: 1/5/25 % dirty 13.6 / 66.6 / 331.5 ms against 13.9 /
// 68.8 / 342 ms with SM stores for all (profiles/r02/tma_writers.txt).
// CRAC_WRITER_TMA=0 turns it off.
bool bulk_writers_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("CRAC_WRITER_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

bool getenv_flag(const char* name) {
  const char* e = std::getenv(name);
  return e && e[0] && e[0] != '0';
}

uint32_t k_full_for(uint32_t chunk_bytes) {
  std::lock_guard<std::mutex> lk(g_kfull_mu);
  if (g_k_full_cache_bytes != chunk_bytes) {
    g_k_full_cache = crac::crc_affine(chunk_bytes);
    g_k_full_cache_bytes = chunk_bytes;
  }
  return g_k_full_cache;
}

}  // namespace

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

int crac_gpu_init(void) {
  std::call_once(g_init_once, [] {
    const HostTables h = build_tables();
    cudaError_t e = cudaMemcpyToSymbol(g_tab, h.tab.data(), kTabBytes);
    if (!e) e = cudaMemcpyToSymbol(g_t0, h.t0.data(), 256 * 4);
    if (!e) e = cudaMemcpyToSymbol(g_xp16, h.xp16.data(), 33 * 4);
    if (!e) e = cudaMemcpyToSymbol(g_xpt, h.xpt.data(), 512 * 4);
    if (!e) e = cudaMemcpyToSymbol(g_pow2, h.pow2.data(), 64 * 4);
    for (auto k : {k1_chunk_crc<4, 0, false>, k1_chunk_crc<8, 0, false>, k1_chunk_crc<16, 0, false>,
                   k1_chunk_crc<4, 0, true>, k1_chunk_crc<8, 0, true>, k1_chunk_crc<16, 0, true>,
                   k1_chunk_crc<12, 0, true>, k1_chunk_crc<kKeyRows, 1, true>,
                   k1_chunk_crc<16, 2, false>, k1_chunk_crc<8, 3, false>,
                   k1_chunk_crc<kKeyRows, 2, true>, k1_chunk_crc<8, 3, true>,
                   k1_chunk_crc<kKeyRows, 4, true>, k1_chunk_crc<4, 0, true, true>,
                   k1_chunk_crc<kKeyPairRows, 4, true, true>,
                   k1_chunk_crc<8, 0, true, true>, k1_chunk_crc<4, 0, false, true>,
                   k1_chunk_crc<8, 0, false, true>})
      if (!e) e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTabBytes));
    if (!e) e = cudaFuncSetAttribute(k1_chunk_crc_tma<16, 3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(k1_tma_smem<16, 3, 4>()));
    if (!e) e = cudaFuncSetAttribute(k1_chunk_crc_tma<8, 6, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(k1_tma_smem<8, 6, 4>()));
    if (!e) e = cudaFuncSetAttribute(k1_chunk_crc_tma<8, 3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(k1_tma_smem<8, 3, 8>()));
    g_init_rc = int(e);
  });
  return g_init_rc;
}

int crac_chunk_crc32(const crac_span_t* d_spans, const uint64_t* d_chunk_first, uint32_t n_spans,
                     uint32_t chunk_bytes, uint64_t total_chunks, uint32_t* d_crc, void* stream) {
  return crac_chunk_crc32_range(d_spans, d_chunk_first, n_spans, chunk_bytes, 0, total_chunks,
                                d_crc, 0, stream);
}

int crac_chunk_crc32_range(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                           uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                           uint32_t* d_crc, uint32_t max_ctas, void* stream) {
  return crac_chunk_key_range(d_spans, d_chunk_first, n_spans, chunk_bytes, c_lo, c_hi, d_crc,
                              nullptr, max_ctas, stream);
}

int crac_chunk_key_range(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                         uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                         uint32_t* d_crc, uint32_t* d_key, uint32_t max_ctas, void* stream) {
  if (c_hi <= c_lo) return 0;
  if (chunk_bytes == 0 || chunk_bytes % 512) return int(cudaErrorInvalidValue);
  if (int rc = crac_gpu_init()) return rc;
  const uint64_t warps_needed = c_hi - c_lo;
  uint64_t blocks = (warps_needed + kK1Warps - 1) / kK1Warps;
  // max_ctas may exceed the SM count: K1 then runs in waves of CTAs, so SMs
  // free up for higher-priority streams (the drain's pack) as CTAs retire
  const uint64_t cap = max_ctas ? max_ctas : sm_count();
  if (blocks > cap) blocks = cap;
  // prefetch depth: 16 rows in flight for 64 KiB chunks; 8 for 4 KiB pages
  // (one batch covers the page, so remote host-resident pages are read with
  // every load in flight)
  static const int forced = [] {
    const char* e = std::getenv("CRAC_K1_ROWS");
    return e ? std::atoi(e) : 0;
  }();
  static const char tma = [] {
    const char* e = std::getenv("CRAC_K1_TMA");
    return e ? e[0] : '\0';
  }();
  if (tma && !d_key) {  // measured alternative (see k1_chunk_crc_tma)
    const uint64_t w = tma == 'A' ? 16 : 8;
    const uint64_t b = std::min<uint64_t>((warps_needed + w - 1) / w, cap);
    const cudaStream_t st = cudaStream_t(stream);
    const uint32_t kf = k_full_for(chunk_bytes);
    if (tma == 'A')
      k1_chunk_crc_tma<16, 3, 4><<<unsigned(b), 512, k1_tma_smem<16, 3, 4>(), st>>>(
          d_spans, d_chunk_first, n_spans, chunk_bytes, c_lo, c_hi, d_crc, kf);
    else if (tma == 'B')
      k1_chunk_crc_tma<8, 6, 4><<<unsigned(b), 256, k1_tma_smem<8, 6, 4>(), st>>>(
          d_spans, d_chunk_first, n_spans, chunk_bytes, c_lo, c_hi, d_crc, kf);
    else
      k1_chunk_crc_tma<8, 3, 8><<<unsigned(b), 256, k1_tma_smem<8, 3, 8>(), st>>>(
          d_spans, d_chunk_first, n_spans, chunk_bytes, c_lo, c_hi, d_crc, kf);
    return int(cudaGetLastError());
  }
  // Default: two chunks per warp (two independent CRC chains per lane, see
  // k1_rows2), 8 rows in flight per chain for the CRC alone and 4 with the key
  // lane (8 spills); 32 GiB hash-only on one B200: 6875 / 6136 GB/s against
  // 6277 / 5518 for one chain (profiles/r02/k1_pair_chains.txt).
  // CRAC_K1_PAIR=0 selects the one-chain kernels (CRAC_K1_ROWS /
  // CRAC_K1_KEY_ROWS their depth), =4|8 the chain depth.
  static const int forced_key = [] {
    const char* e = std::getenv("CRAC_K1_KEY_ROWS");
    return e ? std::atoi(e) : 0;
  }();
  static const int pair_env = [] {
    const char* e = std::getenv("CRAC_K1_PAIR");
    return e ? std::atoi(e) : -1;
  }();
  const int pair = pair_env >= 0 ? pair_env : (d_key ? 4 : 8);
  const int rows_nokey = forced ? forced : (chunk_bytes >= 32 * 512 ? 16 : chunk_bytes >= 8 * 512 ? 8 : 4);
  const int rows = d_key ? (forced_key ? forced_key : kKeyRows) : rows_nokey;
  auto kern = d_key ? (rows == 4 ? k1_chunk_crc<4, 0, true>
                       : rows == 16 ? k1_chunk_crc<16, 0, true>
                       : rows == 12 ? k1_chunk_crc<12, 0, true> : k1_chunk_crc<8, 0, true>)
                    : (rows == 4 ? k1_chunk_crc<4, 0, false>
                       : rows == 16 ? k1_chunk_crc<16, 0, false> : k1_chunk_crc<8, 0, false>);
  if (pair && chunk_bytes >= 8 * 512)
    kern = d_key ? (pair == 8 ? k1_chunk_crc<8, 0, true, true> : k1_chunk_crc<4, 0, true, true>)
                 : (pair == 4 ? k1_chunk_crc<4, 0, false, true> : k1_chunk_crc<8, 0, false, true>);
  kern<<<unsigned(blocks), kK1Threads, kTabBytes, cudaStream_t(stream)>>>(
      d_spans, d_chunk_first, n_spans, chunk_bytes, c_lo, c_hi, d_crc, d_key,
      k_full_for(chunk_bytes), HashDrain{});
  return int(cudaGetLastError());
}

int crac_hash_drain_range(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                          uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                          uint32_t* d_crc, uint32_t* d_crc_prev, uint32_t* d_key,
                          uint32_t* d_key_prev, const uint64_t* d_dst_off,
                          uint8_t* host_image, unsigned long long* d_counters, void* stream) {
  if (c_hi <= c_lo) return 0;
  if (chunk_bytes == 0 || chunk_bytes % 512) return int(cudaErrorInvalidValue);
  if (int rc = crac_gpu_init()) return rc;
  uint64_t blocks = (c_hi - c_lo + kK1Warps - 1) / kK1Warps;
  if (blocks > uint64_t(sm_count())) blocks = sm_count();
  if (!d_crc_prev || !d_counters || (!d_key) != (!d_key_prev)) return int(cudaErrorInvalidValue);
  // (not paired: the inline chunk copy beside two chains spills 468 B)
  k1_chunk_crc<kKeyRows, 1, true><<<unsigned(blocks), kK1Threads, kTabBytes, cudaStream_t(stream)>>>(
      d_spans, d_chunk_first, n_spans, chunk_bytes, c_lo, c_hi, d_crc, d_key,
      k_full_for(chunk_bytes),
      HashDrain{d_crc_prev, d_key_prev, d_dst_off, host_image, d_counters, nullptr, nullptr, 0});
  return int(cudaGetLastError());
}

int crac_hash_drain_split(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                          uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                          uint32_t* d_crc, uint32_t* d_crc_prev, uint32_t* d_key,
                          uint32_t* d_key_prev, const uint64_t* d_dst_off,
                          uint8_t* host_image, unsigned long long* d_counters,
                          unsigned long long* d_queue, uint32_t n_writers, void* stream) {
  if (c_hi <= c_lo) return 0;
  if (chunk_bytes == 0 || chunk_bytes % 512) return int(cudaErrorInvalidValue);
  if (!d_crc_prev || !d_counters || !d_queue || n_writers == 0 || (!d_key) != (!d_key_prev))
    return int(cudaErrorInvalidValue);
  if (int rc = crac_gpu_init()) return rc;
  // one CTA per SM (128 KiB of tables each): every CTA of the grid is resident
  // at once, writers included, and hashers get all the other SMs
  const uint32_t sms = uint32_t(sm_count());
  if (n_writers * 4 > sms) return int(cudaErrorInvalidValue);
  uint64_t hashers = (c_hi - c_lo + kK1Warps - 1) / kK1Warps;
  if (hashers > sms - n_writers) hashers = sms - n_writers;
  cudaStream_t st = cudaStream_t(stream);
  // every CTA must be resident at once (writers spin until the hashers are
  // done): if this context cannot hold the grid (MPS / green-context SM
  // limits, 128 KiB of tables per CTA), drain fused instead
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, k1_chunk_crc<kKeyPairRows, 4, true, true>, kK1Threads, kTabBytes) != cudaSuccess ||
      uint64_t(per_sm) * sms < hashers + n_writers || getenv_flag("CRAC_FORCE_FUSED")) {
    cudaGetLastError();
    return crac_hash_drain_range(d_spans, d_chunk_first, n_spans, chunk_bytes, c_lo, c_hi, d_crc,
                                 d_crc_prev, d_key, d_key_prev, d_dst_off, host_image, d_counters,
                                 stream);
  }
  const uint64_t q = c_hi - c_lo + uint64_t(n_writers) * kK1Warps + 1;
  if (cudaError_t e = cudaMemsetAsync(d_queue, 0, q * 8, st); e != cudaSuccess) return int(e);
  k1_chunk_crc<kKeyPairRows, 4, true, true><<<unsigned(hashers + n_writers), kK1Threads, kTabBytes, st>>>(
      d_spans, d_chunk_first, n_spans, chunk_bytes, c_lo, c_hi, d_crc, d_key,
      k_full_for(chunk_bytes),
      HashDrain{d_crc_prev, d_key_prev, d_dst_off, host_image, d_counters, d_queue, d_counters + 2,
                n_writers, bulk_writers_enabled() ? 1u : 0u});
  return int(cudaGetLastError());
}

int crac_hash_copy_range(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                         uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                         uint32_t* d_crc, uint32_t* d_key, const uint64_t* d_dst_off,
                         uint8_t* d_dst, int dst_aligned, void* stream) {
  if (c_hi <= c_lo) return 0;
  if (chunk_bytes == 0 || chunk_bytes % 512) return int(cudaErrorInvalidValue);
  if (int rc = crac_gpu_init()) return rc;
  uint64_t blocks = (c_hi - c_lo + kK1Warps - 1) / kK1Warps;
  if (blocks > uint64_t(sm_count())) blocks = sm_count();
  auto kern = d_key ? (dst_aligned ? k1_chunk_crc<kKeyRows, 2, true> : k1_chunk_crc<8, 3, true>)
                    : (dst_aligned ? k1_chunk_crc<16, 2, false> : k1_chunk_crc<8, 3, false>);
  kern<<<unsigned(blocks), kK1Threads, kTabBytes, cudaStream_t(stream)>>>(
      d_spans, d_chunk_first, n_spans, chunk_bytes, c_lo, c_hi, d_crc, d_key,
      k_full_for(chunk_bytes), HashDrain{nullptr, nullptr, d_dst_off, d_dst, nullptr});
  return int(cudaGetLastError());
}

int crac_write_frames(const crac_record_t* d_recs, uint32_t n_recs, uint8_t* d_stream,
                      void* stream) {
  if (n_recs == 0) return 0;
  const uint64_t threads = uint64_t(n_recs) * 32;
  k_write_frames<<<unsigned((threads + 255) / 256), 256, 0, cudaStream_t(stream)>>>(d_recs, n_recs,
                                                                                   d_stream);
  return int(cudaGetLastError());
}

int crac_fold_sections(const crac_record_t* d_recs, uint32_t n_recs, const uint64_t* d_pay_first,
                       const uint32_t* d_pay_crc, uint32_t n_pay, const uint32_t* d_page_crc,
                       uint64_t len3, uint64_t total_pay_chunks, uint32_t* d_out, void* stream) {
  cudaStream_t st = cudaStream_t(stream);
  if (cudaError_t e = cudaMemsetAsync(d_out, 0, 8, st)) return int(e);
  if (int rc = crac_gpu_init()) return rc;
  const uint64_t threads = total_pay_chunks + n_recs;
  if (threads == 0) return 0;
  k_fold_sections<<<unsigned((threads + kFoldThreads - 1) / kFoldThreads), kFoldThreads, 0, st>>>(
      d_recs, n_recs, d_pay_first, d_pay_crc, n_pay, d_page_crc, len3, total_pay_chunks, d_out);
  return int(cudaGetLastError());
}

int crac_pack_records(const crac_record_t* d_recs, uint32_t n_recs, const uint32_t* d_tile_rec,
                      uint64_t win_off, uint64_t win_len, uint8_t* d_out, void* stream) {
  if (win_len == 0 || n_recs == 0) return 0;
  // tile b of the launch starts at win_off + b * TILE; d_tile_rec[b] (the
  // record of the aligned tile containing that) never lies past its record
  if (win_off % 16) return int(cudaErrorInvalidValue);
  const uint64_t tiles = (win_len + CRAC_TILE_BYTES - 1) / CRAC_TILE_BYTES;
  k_pack_records<<<unsigned(tiles), kPackThreads, 0, cudaStream_t(stream)>>>(
      d_recs, n_recs, d_tile_rec, win_off, win_len, d_out);
  return int(cudaGetLastError());
}

int crac_scatter_records(const crac_record_t* d_recs, uint32_t n_recs,
                         const uint32_t* d_tile_rec, const uint8_t* d_win, uint64_t win_off,
                         uint64_t win_len, void* stream) {
  if (win_len == 0 || n_recs == 0) return 0;
  if (win_off % CRAC_TILE_BYTES) return int(cudaErrorInvalidValue);
  const uint64_t tiles = (win_len + CRAC_TILE_BYTES - 1) / CRAC_TILE_BYTES;
  k_scatter_records<<<unsigned(tiles), kPackThreads, 0, cudaStream_t(stream)>>>(
      d_recs, n_recs, d_tile_rec, d_win, win_off, win_len);
  return int(cudaGetLastError());
}

int crac_diff_compact(const uint32_t* d_crc_new, uint32_t* d_crc_prev, uint64_t n_chunks,
                      uint32_t* d_block_counts, uint64_t* d_dirty_idx, uint64_t* d_dirty_count,
                      void* stream) {
  cudaStream_t st = cudaStream_t(stream);
  if (n_chunks == 0) return int(cudaMemsetAsync(d_dirty_count, 0, 8, st));
  const uint64_t blocks = (n_chunks + kDiffPerBlock - 1) / kDiffPerBlock;
  k_diff_count<<<unsigned(blocks), kDiffThreads, 0, st>>>(d_crc_new, d_crc_prev, n_chunks,
                                                          d_block_counts);
  k_diff_write<<<unsigned(blocks), kDiffThreads, 0, st>>>(d_crc_new, d_crc_prev, n_chunks,
                                                          d_block_counts, d_dirty_idx,
                                                          d_dirty_count, 0);
  return int(cudaGetLastError());
}

int crac_diff_compact_range(const uint32_t* d_crc_new, uint32_t* d_crc_prev, uint64_t c_lo,
                            uint64_t c_hi, uint32_t* d_block_counts, uint64_t* d_dirty_idx,
                            uint64_t* d_dirty_count, void* stream) {
  cudaStream_t st = cudaStream_t(stream);
  const uint64_t n = c_hi > c_lo ? c_hi - c_lo : 0;
  if (n == 0) return int(cudaMemsetAsync(d_dirty_count, 0, 8, st));
  const uint64_t blocks = (n + kDiffPerBlock - 1) / kDiffPerBlock;
  k_diff_count<<<unsigned(blocks), kDiffThreads, 0, st>>>(d_crc_new + c_lo, d_crc_prev + c_lo, n,
                                                          d_block_counts);
  k_diff_write<<<unsigned(blocks), kDiffThreads, 0, st>>>(d_crc_new + c_lo, d_crc_prev + c_lo, n,
                                                          d_block_counts, d_dirty_idx,
                                                          d_dirty_count, c_lo);
  return int(cudaGetLastError());
}

int crac_gather_chunks(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                       uint32_t n_spans, uint32_t chunk_bytes, const uint64_t* d_dirty_idx,
                       uint64_t first, uint64_t count, uint8_t* d_staging, void* stream) {
  if (count == 0) return 0;
  if (chunk_bytes % 16) return int(cudaErrorInvalidValue);
  uint64_t blocks = count;
  if (blocks > uint64_t(sm_count()) * 16) blocks = uint64_t(sm_count()) * 16;
  k_gather<<<unsigned(blocks), kGatherThreads, 0, cudaStream_t(stream)>>>(
      d_spans, d_chunk_first, n_spans, chunk_bytes, d_dirty_idx, first, count, d_staging);
  return int(cudaGetLastError());
}

int crac_gather_chunks_to_host(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                               uint32_t n_spans, uint32_t chunk_bytes,
                               const uint64_t* d_dirty_idx, uint64_t first, uint64_t count,
                               const uint64_t* d_dst_off, uint8_t* host_image, void* stream) {
  if (count == 0) return 0;
  uint64_t blocks = count;
  if (blocks > uint64_t(sm_count()) * 8) blocks = uint64_t(sm_count()) * 8;
  k_gather_to_host<<<unsigned(blocks), kGatherThreads, 0, cudaStream_t(stream)>>>(
      d_spans, d_chunk_first, n_spans, chunk_bytes, d_dirty_idx, first, count, nullptr, d_dst_off,
      host_image);
  return int(cudaGetLastError());
}

int crac_gather_chunks_to_host_dev(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                                   uint32_t n_spans, uint32_t chunk_bytes,
                                   const uint64_t* d_dirty_idx, const uint64_t* d_count,
                                   uint64_t max_count, uint32_t max_ctas,
                                   const uint64_t* d_dst_off, uint8_t* host_image, void* stream) {
  if (max_count == 0) return 0;
  uint64_t blocks = max_count;
  const uint64_t cap = max_ctas ? max_ctas : uint64_t(sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  k_gather_to_host<<<unsigned(blocks), kGatherThreads, 0, cudaStream_t(stream)>>>(
      d_spans, d_chunk_first, n_spans, chunk_bytes, d_dirty_idx, 0, max_count, d_count, d_dst_off,
      host_image);
  return int(cudaGetLastError());
}

int crac_verify_synth(const uint8_t* d_src, uint64_t len, uint64_t seed, uint64_t id,
                      uint32_t* d_flag, void* stream) {
  if (len == 0) return 0;
  const uint64_t pairs = std::max<uint64_t>(1, len / 16);
  const uint64_t blocks = std::min<uint64_t>((pairs + 255) / 256, uint64_t(sm_count()) * 8);
  k_verify_synth<<<unsigned(blocks), 256, 0, cudaStream_t(stream)>>>(d_src, len, seed, id, d_flag);
  return int(cudaGetLastError());
}

int crac_touch_even_runs(uint8_t* d_managed, uint64_t len, uint64_t run, void* stream) {
  if (!len || !run || run % 16) return int(cudaErrorInvalidValue);
  k_touch_even_runs<<<unsigned(sm_count() * 8), 256, 0, cudaStream_t(stream)>>>(d_managed, len, run);
  return int(cudaGetLastError());
}

int crac_fill_synth(uint8_t* d_dst, uint64_t len, uint64_t seed, uint64_t id,
                    uint64_t word_offset, void* stream) {
  if (len == 0) return 0;
  if (reinterpret_cast<uint64_t>(d_dst) % 16) return int(cudaErrorInvalidValue);
  uint64_t blocks = (len / 16 + 255) / 256;
  if (blocks > uint64_t(sm_count()) * 8) blocks = uint64_t(sm_count()) * 8;
  if (blocks == 0) blocks = 1;
  k_fill_synth<<<unsigned(blocks), 256, 0, cudaStream_t(stream)>>>(d_dst, len, seed, id,
                                                                   word_offset);
  return int(cudaGetLastError());
}

int crac_mutate_chunks(const crac_span_t* d_spans, const uint64_t* d_ids,
                       const uint64_t* d_chunk_first, uint32_t n_spans, uint32_t chunk_bytes,
                       uint64_t total_chunks, uint64_t seed, uint64_t epoch, uint64_t threshold,
                       void* stream) {
  if (total_chunks == 0) return 0;
  uint64_t blocks = total_chunks;
  if (blocks > uint64_t(sm_count()) * 32) blocks = uint64_t(sm_count()) * 32;
  k_mutate<<<unsigned(blocks), 256, 0, cudaStream_t(stream)>>>(
      d_spans, d_ids, d_chunk_first, n_spans, chunk_bytes, total_chunks, seed, epoch, threshold);
  return int(cudaGetLastError());
}

}  // extern "C"
