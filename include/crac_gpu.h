/* crac_gpu.h — C-ABI kernel layer of the B200 checkpoint drain / restart
 * refill (sm_100a).  Plain pointers and sizes only; `stream` is a
 * cudaStream_t passed as void* so this header needs no CUDA includes.
 *
 * Conventions:
 *   - every function returns 0 or a cudaError_t value and never throws;
 *   - buffers are caller-owned device (or UVA-visible pinned/managed)
 *     pointers; nothing here allocates;
 *   - work is enqueued asynchronously on `stream`; re-entrant per stream;
 *   - one process per GPU; crac_gpu_init() once per process/device.
 *
 * Each kernel replaces a CPU step of the reference (/root/reference/proj):
 *   crac_chunk_crc32     K1   crc32_of per section payload, src/image.cpp:16-26,
 *                             used by encode_image :396 and decode_inner :301
 *   crac_pack_records    K2a  encode_payloads / encode_uvm framing + the
 *                             read_raw drain, src/image.cpp:53-77,
 *                             src/ckpt_engine.cpp:38-56, device_core.cpp:442-447
 *   crac_diff_compact /  K2b  new (incremental drain; the reference has none,
 *   crac_gather_chunks        SPEC.md:336) — emits the same bytes as a full drain
 *   crac_scatter_records K3   restart refill via write_raw,
 *                             src/ckpt_engine.cpp:147-164, device_core.cpp:449-454
 */
#ifndef CRAC_GPU_H
#define CRAC_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A device-visible byte range (16-byte aligned `ptr` for the hash kernel). */
typedef struct crac_span {
  uint64_t ptr;
  uint64_t len;
} crac_span_t;

/* One framed record of a section stream (ALLOC_PAYLOADS / UVM_PAGES):
 * `frame_len` literal bytes at stream offset `out_off`, followed by `len`
 * payload bytes that live at device-visible address `ptr`.
 * Refill writes `ext` >= len bytes at `ptr`; bytes past `len` are zeroed
 * (the allocator's 256-byte padding, ref: device_core.cpp:48,65).
 * ptr == 0 with len > 0 marks host-filled content: pack emits zeros for it
 * and scatter skips it (host-resident managed pages are copied by the host). */
typedef struct crac_record {
  uint64_t out_off;
  uint64_t ptr;
  uint64_t len;
  uint64_t ext;
  uint32_t frame_len; /* 0..24 */
  uint32_t reserved;
  uint8_t frame[24];
} crac_record_t; /* 64 bytes */

/* Stream tile size used by pack/scatter: the host supplies, per tile of the
 * window, the index of the first record overlapping it (tile_rec). */
#define CRAC_TILE_BYTES 65536u

/* Uploads the CRC tables to the current device.  Idempotent. */
int crac_gpu_init(void);

/* K1: zlib-identical CRC-32 of every `chunk_bytes` piece of every span.
 * chunk_bytes: multiple of 512.  d_chunk_first[i] = index of span i's first
 * chunk (exclusive prefix sum of ceil(len/chunk_bytes)), n_spans+1 entries.
 * d_crc receives total_chunks values. */
int crac_chunk_crc32(const crac_span_t* d_spans, const uint64_t* d_chunk_first, uint32_t n_spans,
                     uint32_t chunk_bytes, uint64_t total_chunks, uint32_t* d_crc, void* stream);

/* K1 over the absolute chunk range [c_lo, c_hi) of the same span table,
 * writing d_crc[c]; at most max_ctas CTAs (0 = one per SM) so the kernel can
 * leave SMs to work running beside it. */
int crac_chunk_crc32_range(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                           uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                           uint32_t* d_crc, uint32_t max_ctas, void* stream);

/* K1 plus the chunk key: the same pass also writes d_key[c], a second,
 * independent 32-bit lane (integer multiply-add over the chunk's 32-bit
 * words with position-dependent offsets, not GF(2)-linear; definition in
 * kernels.cu "Key2").  (d_crc[c], d_key[c]) is the 64-bit dirty key of the
 * incremental and pre-copy drains: a change that preserves the CRC-32 (four
 * compensating bytes suffice) still changes the key.  d_key may be null
 * (= crac_chunk_crc32_range). */
int crac_chunk_key_range(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                         uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                         uint32_t* d_crc, uint32_t* d_key, uint32_t max_ctas, void* stream);

/* Fused incremental drain (K1 + K2b in one pass): hashes chunks [c_lo, c_hi)
 * into d_crc (and d_key); every chunk whose dirty key (d_crc, d_key) differs
 * from (d_crc_prev, d_key_prev) is written by the hashing warp straight into
 * host_image + d_dst_off[span] + chunk offset (pinned, UVA-mapped) and its
 * previous-key entries updated.  d_key / d_key_prev: both null (CRC-only
 * comparison) or both set.  d_counters[0] += dirty chunks, d_counters[1] +=
 * dirty bytes (caller zeroes them). */
int crac_hash_drain_range(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                          uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                          uint32_t* d_crc, uint32_t* d_crc_prev, uint32_t* d_key,
                          uint32_t* d_key_prev, const uint64_t* d_dst_off,
                          uint8_t* host_image, unsigned long long* d_counters, void* stream);
/* Split form of crac_hash_drain_range: the first n_writers CTAs only write
 * dirty chunks to the image, the others hash and hand each dirty chunk over
 * through d_queue (>= c_hi - c_lo + 16 * n_writers + 1 u64, zeroed here), so
 * the hashing never waits on PCIe.  d_counters needs 5 u64 ([0] dirty chunks,
 * [1] dirty bytes, [2..4] queue control; zeroed by the caller).  n_writers
 * <= SMs / 4. */
int crac_hash_drain_split(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                          uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                          uint32_t* d_crc, uint32_t* d_crc_prev, uint32_t* d_key,
                          uint32_t* d_key_prev, const uint64_t* d_dst_off,
                          uint8_t* host_image, unsigned long long* d_counters,
                          unsigned long long* d_queue, uint32_t n_writers, void* stream);

/* Incremental drain straight to the host image: dirty chunk k (index
 * d_dirty_idx[first + k]) of payload span s is written by the SMs to
 * host_image + d_dst_off[s] + chunk offset (pinned, UVA-mapped memory). */
int crac_gather_chunks_to_host(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                               uint32_t n_spans, uint32_t chunk_bytes,
                               const uint64_t* d_dirty_idx, uint64_t first, uint64_t count,
                               const uint64_t* d_dst_off, uint8_t* host_image, void* stream);

/* Same as crac_gather_chunks_to_host over d_dirty_idx[0 .. *d_count) where
 * the count is read on the device (no host round trip after the diff);
 * max_count bounds it, max_ctas caps the grid (0 = 8 per SM). */
int crac_gather_chunks_to_host_dev(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                                   uint32_t n_spans, uint32_t chunk_bytes,
                                   const uint64_t* d_dirty_idx, const uint64_t* d_count,
                                   uint64_t max_count, uint32_t max_ctas,
                                   const uint64_t* d_dst_off, uint8_t* host_image, void* stream);

/* K4: the linear parts of the ALLOC_PAYLOADS and UVM_PAGES CRCs from chunk
 * and page CRCs plus the frame bytes (d_out[0], d_out[1]; the caller xors in
 * K(section length) = crc32 of that many zero bytes' affine term).  Records
 * as for crac_pack_records, sec3 first (record i <-> payload span i), the
 * 20-byte gap record at len3, then sec4 with page records carrying their page
 * CRC index in `reserved`. */
int crac_fold_sections(const crac_record_t* d_recs, uint32_t n_recs, const uint64_t* d_pay_first,
                       const uint32_t* d_pay_crc, uint32_t n_pay, const uint32_t* d_page_crc,
                       uint64_t len3, uint64_t total_pay_chunks, uint32_t* d_out, void* stream);

/* Hash + copy (stall-reduced snapshot): hashes chunks [c_lo, c_hi) into
 * d_crc (and the chunk key into d_key, unless null) and writes every chunk to d_dst + d_dst_off[span] + chunk offset
 * from the registers it was hashed from (one HBM read; d_dst is device or
 * UVA memory).  dst_aligned = 1 promises every d_dst + d_dst_off[span] is
 * 16-byte aligned (faster kernel); 0 accepts any alignment. */
int crac_hash_copy_range(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                         uint32_t n_spans, uint32_t chunk_bytes, uint64_t c_lo, uint64_t c_hi,
                         uint32_t* d_crc, uint32_t* d_key, const uint64_t* d_dst_off,
                         uint8_t* d_dst, int dst_aligned, void* stream);

/* The frame bytes (frame_len <= 24) of records [0, n_recs) at
 * d_stream + out_off, with byte stores only, so a concurrent
 * crac_hash_drain_range copy of the payloads may share their 16-byte words. */
int crac_write_frames(const crac_record_t* d_recs, uint32_t n_recs, uint8_t* d_stream,
                      void* stream);

/* K2a: writes stream bytes [win_off, win_off + win_len) into d_out (16-byte
 * aligned; win_off multiple of 16).  Records sorted by out_off; bytes not
 * covered by any record are written as zero.  d_tile_rec[t] = first record
 * overlapping stream tile (win_off / CRAC_TILE_BYTES + t). */
int crac_pack_records(const crac_record_t* d_recs, uint32_t n_recs, const uint32_t* d_tile_rec,
                      uint64_t win_off, uint64_t win_len, uint8_t* d_out, void* stream);

/* K3: inverse of pack.  d_win holds stream bytes [win_off, win_off+win_len+16)
 * (16 bytes of look-ahead past the window).  Every destination 16-byte word
 * whose first stream byte lies in the window is written; the padding words
 * (len..ext) of a record are zero-filled by the window holding its last
 * payload byte (or by window 0 for len == 0). */
int crac_scatter_records(const crac_record_t* d_recs, uint32_t n_recs,
                         const uint32_t* d_tile_rec, const uint8_t* d_win, uint64_t win_off,
                         uint64_t win_len, void* stream);

/* K2b: dirty-chunk detection.  d_dirty_idx receives, in ascending order, the
 * indices c with d_crc_new[c] != d_crc_prev[c]; *d_dirty_count their number.
 * d_block_counts: scratch of ceil(n_chunks / 4096) uint32.  d_crc_prev is
 * then overwritten with d_crc_new. */
int crac_diff_compact(const uint32_t* d_crc_new, uint32_t* d_crc_prev, uint64_t n_chunks,
                      uint32_t* d_block_counts, uint64_t* d_dirty_idx, uint64_t* d_dirty_count,
                      void* stream);

/* crac_diff_compact over the chunk range [c_lo, c_hi): indices written are
 * absolute; d_block_counts needs ceil((c_hi - c_lo) / 4096) entries. */
int crac_diff_compact_range(const uint32_t* d_crc_new, uint32_t* d_crc_prev, uint64_t c_lo,
                            uint64_t c_hi, uint32_t* d_block_counts, uint64_t* d_dirty_idx,
                            uint64_t* d_dirty_count, void* stream);

/* Copies dirty chunks d_dirty_idx[first .. first+count) (chunk numbering as in
 * crac_chunk_crc32) to d_staging + k * chunk_bytes, k = 0..count-1. */
int crac_gather_chunks(const crac_span_t* d_spans, const uint64_t* d_chunk_first,
                       uint32_t n_spans, uint32_t chunk_bytes, const uint64_t* d_dirty_idx,
                       uint64_t first, uint64_t count, uint8_t* d_staging, void* stream);

/* Test/bench fixtures: synthetic content and epoch mutation.
 * Word k of allocation `id`: mix64(k + 0x1000003*id + (seed << 56)), LE. */
int crac_fill_synth(uint8_t* d_dst, uint64_t len, uint64_t seed, uint64_t id,
                    uint64_t word_offset, void* stream);
/* K5, GPU deflate (deflate.cu): [d_in, +n) in CRAC_DEFLATE_SEGMENT-byte
 * segments, one deflate piece each (fixed Huffman LZ77, or a stored block if
 * that would not shrink it), every piece byte-aligned at both ends (sync
 * flush), written to its CRAC_DEFLATE_SLOT-byte slot of d_slots; d_len[s] =
 * its byte length (bit 31 set: a stored piece, built by the gather from the
 * input), d_adler[s] = the Adler-32 of segment s alone.  With last_is_final
 * the last piece carries BFINAL.  crac_gather_segments writes the pieces to
 * d_out at the (host-computed) d_offset. */
#define CRAC_DEFLATE_SEGMENT 32768u
#define CRAC_DEFLATE_SLOT (CRAC_DEFLATE_SEGMENT + CRAC_DEFLATE_SEGMENT / 8 + 64u)
int crac_deflate_segments(const uint8_t* d_in, uint64_t n, uint8_t* d_slots, uint32_t* d_len,
                          uint32_t* d_adler, int last_is_final, void* stream);
int crac_gather_segments(const uint8_t* d_in, uint64_t n, const uint8_t* d_slots,
                         const uint32_t* d_len, const uint64_t* d_offset, uint8_t* d_out,
                         int last_is_final, void* stream);

/* First touch on the GPU of the even `run`-byte runs of [d_managed, +len)
 * (the managed-populate ceiling probe). */
int crac_touch_even_runs(uint8_t* d_managed, uint64_t len, uint64_t run, void* stream);
/* Sets *d_flag = 1 if any byte of [d_src, +len) differs from the synthetic
 * content of crac_fill_synth(seed, id, word offset 0); leaves it otherwise. */
int crac_verify_synth(const uint8_t* d_src, uint64_t len, uint64_t seed, uint64_t id,
                      uint32_t* d_flag, void* stream);

/* Rewrites chunk c of span s iff mix64(seed ^ (epoch << 40) ^ (chunk_first[s]+c)) <
 * threshold, with synth content of seed' = seed + epoch (ids from d_ids). */
int crac_mutate_chunks(const crac_span_t* d_spans, const uint64_t* d_ids,
                       const uint64_t* d_chunk_first, uint32_t n_spans, uint32_t chunk_bytes,
                       uint64_t total_chunks, uint64_t seed, uint64_t epoch, uint64_t threshold,
                       void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CRAC_GPU_H */
