/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the thing measured or
 * shipped.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * / --impl reference legs may load this library.
 *
 * Plain-C restatement of the checksum the reference stores after every image
 * section.  The reference calls zlib (image.cpp:16-26 `crc32_of`, used at
 * image.cpp:301 and :396); zlib is not vendored in /root/reference
 * (find_package(ZLIB) at proj/CMakeLists.txt:16), the container's is zlib 1.3
 * (Ubuntu 1:1.3.dfsg-3.1ubuntu2.2).  CRC-32/IEEE-802.3 is a fixed standard,
 * restated here from its published definition:
 *   reflected polynomial 0xEDB88320, init 0xFFFFFFFF, final xor 0xFFFFFFFF,
 *   crc32(0, NULL, 0) == 0, crc32("123456789") == 0xCBF43926.
 * crc32_combine restates zlib's published combine (multmodp / x2nmodp):
 *   crc(A||B) = (x^(8|B|) mod P) * crc(A)  xor  crc(B).
 *
 * Pinned against: Python's zlib.crc32 (same system zlib the reference links)
 * and the reference library itself (tests/test_oracle.py).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define POLY 0xEDB88320u

static uint32_t table[8][256];
static int table_ready = 0;
static pthread_once_t table_once = PTHREAD_ONCE_INIT;

static void build_tables(void) {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ POLY : (c >> 1);
    table[0][i] = c;
  }
  for (uint32_t i = 0; i < 256; ++i)
    for (int t = 1; t < 8; ++t) table[t][i] = (table[t - 1][i] >> 8) ^ table[0][table[t - 1][i] & 0xff];
  table_ready = 1;
}

/* Bit-at-a-time definition: the slowest, most literal restatement. */
uint32_t oracle_crc32_bitwise(uint32_t crc, const uint8_t* p, uint64_t n) {
  crc = ~crc;
  for (uint64_t i = 0; i < n; ++i) {
    crc ^= p[i];
    for (int k = 0; k < 8; ++k) crc = (crc & 1) ? (crc >> 1) ^ POLY : (crc >> 1);
  }
  return ~crc;
}

/* Slicing-by-8 over the same tables; equal to the bitwise form. */
uint32_t oracle_crc32(uint32_t crc, const uint8_t* p, uint64_t n) {
  pthread_once(&table_once, build_tables);
  crc = ~crc;
  while (n >= 8) {
    uint32_t lo, hi;
    memcpy(&lo, p, 4);
    memcpy(&hi, p + 4, 4);
    lo ^= crc;
    crc = table[7][lo & 0xff] ^ table[6][(lo >> 8) & 0xff] ^ table[5][(lo >> 16) & 0xff] ^
          table[4][lo >> 24] ^ table[3][hi & 0xff] ^ table[2][(hi >> 8) & 0xff] ^
          table[1][(hi >> 16) & 0xff] ^ table[0][hi >> 24];
    p += 8;
    n -= 8;
  }
  while (n--) crc = table[0][(crc ^ *p++) & 0xff] ^ (crc >> 8);
  return ~crc;
}

/* GF(2) polynomial product a*b mod P in the reflected representation. */
static uint32_t multmodp(uint32_t a, uint32_t b) {
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ POLY : b >> 1;
  }
  return p;
}

/* x^(n * 2^k) mod P. */
static uint32_t x2nmodp(uint64_t n, unsigned k) {
  uint32_t p = 1u << 31; /* x^0 */
  uint32_t x2[64];
  x2[0] = 1u << 30; /* x^1 */
  for (int i = 1; i < 64; ++i) x2[i] = multmodp(x2[i - 1], x2[i - 1]);
  while (n) {
    if (n & 1) p = multmodp(x2[k & 63], p);
    n >>= 1;
    k++;
  }
  return p;
}

uint32_t oracle_crc32_combine(uint32_t crc1, uint32_t crc2, uint64_t len2) {
  return multmodp(x2nmodp(len2, 3), crc1) ^ crc2;
}

/* Per-chunk CRCs over a buffer on `threads` host threads: the CPU
 * counterpart of the GPU chunk hash (fair hashing baseline). */
struct chunk_job {
  const uint8_t* p;
  uint64_t n, chunk, first, last;
  uint32_t* out;
};

static void* chunk_worker(void* arg) {
  struct chunk_job* j = (struct chunk_job*)arg;
  for (uint64_t c = j->first; c < j->last; ++c) {
    uint64_t off = c * j->chunk;
    uint64_t len = j->n - off < j->chunk ? j->n - off : j->chunk;
    j->out[c] = oracle_crc32(0, j->p + off, len);
  }
  return NULL;
}

void oracle_chunk_crc32(const uint8_t* p, uint64_t n, uint64_t chunk, uint32_t* out, int threads) {
  uint64_t nchunks = (n + chunk - 1) / chunk;
  if (threads < 1) threads = 1;
  pthread_t tid[256];
  struct chunk_job jobs[256];
  if (threads > 256) threads = 256;
  for (int t = 0; t < threads; ++t) {
    jobs[t].p = p;
    jobs[t].n = n;
    jobs[t].chunk = chunk;
    jobs[t].first = nchunks * (uint64_t)t / (uint64_t)threads;
    jobs[t].last = nchunks * (uint64_t)(t + 1) / (uint64_t)threads;
    jobs[t].out = out;
    pthread_create(&tid[t], NULL, chunk_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* splitmix64, common.hpp:55-60. */
uint64_t oracle_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* Synthetic allocation content shared with the GPU fill kernel: word k of
 * allocation `id` is mix64(k + 0x1000003*id + (seed << 56)), little-endian,
 * trailing partial word truncated. */
void oracle_synth_bytes(uint64_t seed, uint64_t id, uint64_t offset_words, uint64_t size,
                        uint8_t* out) {
  uint64_t words = size / 8;
  for (uint64_t k = 0; k < words; ++k) {
    uint64_t w = oracle_mix64(offset_words + k + 0x1000003ull * id + (seed << 56));
    memcpy(out + 8 * k, &w, 8);
  }
  if (size % 8) {
    uint64_t w = oracle_mix64(offset_words + words + 0x1000003ull * id + (seed << 56));
    memcpy(out + 8 * words, &w, size % 8);
  }
}
