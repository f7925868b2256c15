/* crac_engine.h — C-ABI of the B200 checkpoint engine (libcrac_b200.so).
 *
 * This is the boundary a non-C++ caller binds (ctypes / cgo / JNI; see
 * INTEGRATION.md).  Every entry point wraps one reference C++ interface
 * (/root/reference/proj, cited per function) with the B200 implementation
 * behind it; handles are opaque, all sizes are bytes, `stream` < 0 means
 * "synchronous" (std::nullopt in the reference API).
 *
 * Return convention: 0 on success, otherwise 1 + the cracsim::Errc code of the
 * failure (ImageCorrupt = 14, ReplayDivergence = 13, QuiesceTimeout = 12,
 * DeviceFault = 17, ...); crac_last_error() returns the message of the last
 * failure on the calling thread.  Nothing here falls back to a CPU path: with
 * no usable GPU every call that needs one returns DeviceFault.
 */
#ifndef CRAC_ENGINE_H
#define CRAC_ENGINE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct crac_session crac_session_t; /* cracsim::Session */
typedef struct crac_image crac_image_t;     /* cracsim::PinnedImage */

/* Device-timed phases of the last drain/refill (cracsim::DrainStats). */
typedef struct crac_stats {
  double total_ms, hash_ms, pack_ms, copy_ms;
  uint64_t hash_bytes, hash_launches, pack_launches, pack_bytes;
  uint64_t d2h_bytes, h2d_bytes, image_bytes, dirty_chunks, total_chunks;
  int32_t incremental;
  int32_t reserved;
  double stall_ms;       /* quiesce -> the app may resume */
  uint64_t shadow_bytes; /* stream bytes staged in the HBM shadow */
  double barrier_ms;     /* host wait in the global-checkpoint hook (ABI 2) */
  double host_pre_ms;    /* refill: parse + set-up before the first device event,
                            included in total_ms (ABI 2) */
} crac_stats_t;

const char* crac_last_error(void);
int crac_abi_version(void); /* 2: crac_stats_t grew barrier_ms/host_pre_ms; barrier API */

/* Session — ref: include/cracsim/ckpt_engine.hpp:18-55 (SessionConfig, Session) */
int crac_session_create(uint64_t seed, uint64_t arena_bytes, int mode, uint32_t quiesce_timeout_ms,
                        crac_session_t** out);
void crac_session_destroy(crac_session_t* s);
int crac_session_fixed_va(crac_session_t* s); /* 1 if the arena sits at kArenaBase */

/* RuntimeApi — ref: include/cracsim/shim.hpp:159-184 (the interposed calls) */
int crac_alloc(crac_session_t* s, uint8_t kind, uint64_t size, uint64_t* id, uint64_t* address);
int crac_free(crac_session_t* s, uint64_t id);
int crac_stream_create(crac_session_t* s, uint64_t* id);
int crac_stream_destroy(crac_session_t* s, uint64_t id);
/* Kernel bodies resolve by name from the standard catalog; other names get
 * an empty body (ref: include/cracsim/kernels.hpp:16-21). */
int crac_register_fat_binary(crac_session_t* s, uint32_t n, const char* const* names,
                             const uint32_t* buffer_arity, const uint32_t* scalar_arity,
                             uint64_t* handle);
int crac_unregister_fat_binary(crac_session_t* s, uint64_t handle);
int crac_launch(crac_session_t* s, uint64_t stream, const char* kernel, uint32_t nbuf,
                const uint64_t* buf_ids, const uint64_t* buf_offsets, uint32_t nscalar,
                const uint64_t* scalars);
int crac_copy_h2d(crac_session_t* s, uint64_t id, uint64_t offset, const void* src, uint64_t n,
                  int64_t stream);
int crac_copy_d2h(crac_session_t* s, void* dst, uint64_t id, uint64_t offset, uint64_t n,
                  int64_t stream);
int crac_copy_d2d(crac_session_t* s, uint64_t dst_id, uint64_t dst_off, uint64_t src_id,
                  uint64_t src_off, uint64_t n, int64_t stream);
int crac_synchronize(crac_session_t* s);
int crac_page_read(crac_session_t* s, uint64_t id, uint64_t offset, uint64_t n, uint8_t side,
                   void* out);
int crac_page_write(crac_session_t* s, uint64_t id, uint64_t offset, const void* src, uint64_t n,
                    uint8_t side);
int crac_set_app_state(crac_session_t* s, const void* src, uint64_t n);

/* Checkpoint drain — ref: src/ckpt_engine.cpp:29-61 + src/image.cpp:383-399.
 * The image lives in `img` (page-locked, reused across calls). */
int crac_image_create(crac_image_t** out);
void crac_image_destroy(crac_image_t* img);
int crac_image_view(crac_image_t* img, const uint8_t** data, uint64_t* size);
/* Capacity of the page-locked buffer and how much of it is 2 MiB-page backed. */
int crac_image_pages(crac_image_t* img, uint64_t* capacity, uint64_t* huge_bytes);
int crac_checkpoint(crac_session_t* s, crac_image_t* img, crac_stats_t* stats);
int crac_checkpoint_incremental(crac_session_t* s, crac_image_t* img, crac_stats_t* stats);
/* Stall-reduced drain (new): the app is quiesced only while the
 * state is snapshotted into HBM reserved with crac_reserve_shadow; the D2H
 * into `img` continues after crac_checkpoint_begin returns and
 * crac_checkpoint_finish completes it.  Bytes equal crac_checkpoint's at the
 * instant of begin.  crac_reserve_shadow(s, 0) releases the reservation;
 * OutOfArena (1 + 1) if the HBM is not available. */
/* Global checkpoint across the per-GPU processes of a job (the
 * reference is single-process, ckpt_engine.cpp:29-61 quiesces one table).
 * With a hook set, every checkpoint entry point calls fn(ctx, phase) at
 *   CRAC_PHASE_QUIESCED        inside the quiesce, before any state is read;
 *   CRAC_PHASE_IMAGE_COMPLETE  once this rank's image is complete (for
 *                              crac_checkpoint_begin: in crac_checkpoint_finish);
 *   CRAC_PHASE_PERSISTED       crac_checkpoint_to_file, after the fdatasync.
 * fn returns 0 when every rank arrived; nonzero fails the checkpoint with
 * QuiesceTimeout (the application is resumed).  fn = NULL removes the hook. */
#define CRAC_PHASE_QUIESCED 0
#define CRAC_PHASE_IMAGE_COMPLETE 1
#define CRAC_PHASE_PERSISTED 2
typedef int (*crac_barrier_fn)(void* ctx, int phase);
int crac_session_set_barrier(crac_session_t* s, crac_barrier_fn fn, void* ctx);
/* Built-in hook for the ranks of one node: a barrier in POSIX shared memory
 * (name "/x", created by the first opener; every rank passes the same world).
 * crac_barrier_wait returns QuiesceTimeout (12) after timeout_ms, with its
 * arrival withdrawn.  Install with crac_session_set_barrier(s, crac_barrier_hook, b). */
typedef struct crac_barrier crac_barrier_t;
int crac_barrier_open(const char* name, uint32_t world, uint32_t rank, uint32_t timeout_ms,
                      crac_barrier_t** out);
int crac_barrier_wait(crac_barrier_t* b);
int crac_barrier_hook(void* b, int phase); /* a crac_barrier_fn; b = crac_barrier_t* */
uint64_t crac_barrier_generation(crac_barrier_t* b);
void crac_barrier_close(crac_barrier_t* b, int unlink);

/* Independent host check of an image (no GPU, no code shared with the drain):
 * strict parse, every section CRC recomputed on `threads` host cores (0 = all),
 * and with check_synth every Device payload compared byte for byte with the
 * synthetic content f(synth_seed, id, offset) of crac_fill_synthetic.  Returns
 * 0 with the findings in *out (a failed check is a finding, not an error);
 * ImageCorrupt when the framing itself is invalid. */
typedef struct crac_verify {
  uint64_t sections_checked, crc_bytes;
  uint64_t payloads_compared, payload_bytes_compared, mismatched_payloads, first_bad_id;
  uint32_t bad_sections; /* bit s: recomputed CRC of section s+1 differs */
  uint32_t threads;
  double ms;
} crac_verify_t;
int crac_image_verify(const void* image, uint64_t size, uint32_t threads, uint64_t synth_seed,
                      int check_synth, crac_verify_t* out);
/* Compares every live Device allocation of `s` on the GPU with
 * f(seed, id, offset); *bad_allocations = allocations with any differing word. */
int crac_session_verify_synthetic(crac_session_t* s, uint64_t seed, uint64_t* bad_allocations,
                                  uint64_t* bytes_checked);

/* The ceiling of a managed-memory refill on this box (C3): fresh
 * cudaMallocManaged memory of `bytes`, alternating `run`-byte runs first
 * touched on the GPU (even runs, one kernel) and by `threads` host threads
 * (odd runs, memcpy from page-locked memory) at the same time, as the refill
 * restores split residence.  *ms = wall time of both; the memory is freed. */
int crac_probe_managed_populate(uint64_t bytes, uint64_t run, uint32_t threads, double* ms);

int crac_reserve_shadow(crac_session_t* s, uint64_t bytes);
/* The shadow in another GPU's HBM (SURVEY §8f.3 buddy copy): reachable by
 * peer access (InvalidArgument otherwise); `device` = this session's GPU is
 * crac_reserve_shadow. */
int crac_reserve_shadow_on(crac_session_t* s, uint64_t bytes, int device);
int crac_checkpoint_begin(crac_session_t* s, crac_image_t* img, crac_stats_t* stats);
int crac_checkpoint_finish(crac_session_t* s, crac_stats_t* stats);
/* Pre-copy drain (new): begin copies the state into `img`
 * while the application runs; finish quiesces it and re-sends only the chunks
 * that changed since (stats.stall_ms = the quiesced phase).  Bytes equal
 * crac_checkpoint's at the instant of finish.  Device-only sessions; others
 * drain synchronously in begin. */
int crac_checkpoint_precopy_begin(crac_session_t* s, crac_image_t* img, crac_stats_t* stats);
int crac_checkpoint_precopy_finish(crac_session_t* s, crac_stats_t* stats);
/* checkpoint(Session&) -> Snapshot -> encode_image, into a malloc'd buffer
 * released with crac_buffer_free (the reference-shaped value API). */
int crac_checkpoint_value(crac_session_t* s, uint8_t** image, uint64_t* size);

/* Image persistence — ref: src/ckpt_engine.cpp:63-65,173-177
 * (checkpoint_to_file / restart_from_file) and src/image.cpp:432-451 (the
 * whole-buffer ofstream / ifstream they use).  The drain lands in `img`; the
 * file is written from it by parallel positional writes (O_DIRECT when the
 * filesystem accepts it) and fdatasync'd; restart reads the file back into
 * `img` the same way and refills from it.  Files are byte-identical to the
 * reference's.  Write errors: InvalidArgument (1 + 0); unreadable file:
 * ImageCorrupt (1 + 13). */
typedef struct crac_io_stats {
  double ms;          /* open .. fdatasync / close */
  uint64_t bytes;     /* file bytes */
  uint32_t threads;   /* I/O threads */
  int32_t direct;     /* 1 if O_DIRECT */
  uint64_t bounced;   /* bytes moved through an aligned bounce buffer */
  uint64_t streamed;  /* checkpoint_to_file: bytes written while the drain still ran */
} crac_io_stats_t;
/* compress: 0 none; 1 the reference's CRACSIMZ bytes (zlib compress2 level 6,
 * host, image.cpp:419-430); 2 the GPU deflate (K5): a different, valid zlib
 * stream in the same wrapper, which the reference's maybe_decompress inflates
 * to the exact image. */
int crac_checkpoint_to_file(crac_session_t* s, crac_image_t* img, const char* path, int compress,
                            crac_stats_t* drain, crac_io_stats_t* io);
/* The GPU deflate of any image into a CRACSIMZ wrapper (free with
 * crac_buffer_free); *ms = wall time. */
int crac_compress_image_gpu(const void* image, uint64_t n, uint8_t** out, uint64_t* out_n,
                            double* ms);
int crac_restart_from_file(const char* path, crac_image_t* img, int mode, crac_session_t** out,
                           crac_stats_t* refill, crac_io_stats_t* io);
/* The parallel file transfer alone, on any host buffer (no GPU needed):
 * threads / chunk_bytes 0 = defaults; flags bit 0 = O_DIRECT, bit 1 = fdatasync. */
int crac_file_write(const char* path, const void* data, uint64_t n, uint32_t threads,
                    uint64_t chunk_bytes, uint32_t flags, crac_io_stats_t* io);
int crac_file_size(const char* path, uint64_t* n);
int crac_file_read(const char* path, void* dst, uint64_t capacity, uint32_t threads,
                   uint64_t chunk_bytes, uint32_t flags, uint64_t* n, crac_io_stats_t* io);

/* Restart refill — ref: src/ckpt_engine.cpp:120-171 + src/image.cpp:280-345. */
int crac_restart(const void* image, uint64_t size, int mode, crac_session_t** out,
                 crac_stats_t* stats);
/* decode_image validation only — ref: src/image.cpp:401-404. */
int crac_decode_check(const void* image, uint64_t size);
/* summarize_image — ref: src/image.cpp:406-413; lengths/crcs: 7 each;
 * totals: log_entries, active, payload_bytes, uvm_bytes, file_bytes. */
int crac_summarize(const void* image, uint64_t size, uint64_t* lengths, uint32_t* crcs,
                   uint64_t* totals);

/* Introspection (tests) — ref: include/cracsim/device_core.hpp:117-140 */
int crac_debug_dump(crac_session_t* s, char** out);
void crac_buffer_free(void* p);
int crac_log_size(crac_session_t* s, uint64_t* n);
int crac_live_records(crac_session_t* s, uint64_t cap, uint64_t* ids, uint8_t* kinds,
                      uint64_t* sizes, uint64_t* addresses, uint64_t* n);
int crac_managed_pages(crac_session_t* s, uint64_t id, uint64_t cap, uint8_t* flags, uint64_t* n);
int crac_read_raw(crac_session_t* s, uint64_t address, uint64_t n, void* out);
int crac_backing_ptr(crac_session_t* s, uint64_t id, uint64_t* ptr);

/* Interposition support (libcrac_preload.so, crac_preload.h).
 * The reference's shim has no real cudart underneath (ref: src/shim.cpp:
 * 204-253 is the call path an LD_PRELOAD interposer feeds):
 *   crac_stream_handle   the cudaStream_t behind app stream `id`;
 *   crac_live_streams    live app stream ids (restart: rebuild the handle map);
 *   crac_gate_enter/leave  admit a call forwarded to the real runtime through
 *                        the dispatch gate (DispatchTable::admit / release);
 *   crac_set_device_wide_drain  quiesce = cudaDeviceSynchronize;
 *   crac_get_app_state   the APPSTATE bytes (a view, valid until the next
 *                        crac_set_app_state / destroy). */
int crac_stream_handle(crac_session_t* s, uint64_t id, void** cuda_stream);
int crac_live_streams(crac_session_t* s, uint64_t cap, uint64_t* ids, uint64_t* n);
int crac_gate_enter(crac_session_t* s);
int crac_gate_leave(crac_session_t* s);
int crac_set_device_wide_drain(crac_session_t* s, int on);
int crac_get_app_state(crac_session_t* s, const uint8_t** data, uint64_t* n);

/* Workload fixtures (bench / tests): synthetic content (see crac_gpu.h) and
 * the C5 epoch mutation over every live Device allocation. */
int crac_fill_synthetic(crac_session_t* s, uint64_t id, uint64_t seed, uint8_t managed_side);
int crac_mutate_device(crac_session_t* s, uint64_t seed, uint64_t epoch, uint64_t threshold,
                       uint64_t* mutated_chunks);

/* Hash-only pass (C5 "hash-only"): K1 over every live allocation of the
 * session, chunk CRCs left on the device; stats.hash_ms / hash_bytes. */
int crac_hash_session(crac_session_t* s, crac_stats_t* stats);

/* Diagnostics: the CUDA runtime's pending (non-sticky) error of this library,
 * without clearing it (cudaPeekAtLastError); 0 when none. */
int crac_peek_cuda_error(void);

/* Frees the mapped arena a closed session left on `device` (-1: the current
 * one) for the next session of the same size to adopt.  The next restart
 * then maps its physical memory afresh, as in a new process (a cold restart). */
int crac_drop_arena_cache(int device);

/* As crac_drop_arena_cache, but only the VA is freed before returning: the
 * physical memory is released on a background thread, and a restart that
 * needs it (its arena map) waits for that release, so the release overlaps
 * the restart's first H2D copies.  crac_drop_arena_cache on the device waits
 * for releases in flight. */
int crac_drop_arena_cache_async(int device);

/* Host CRC-32 the engine uses for host-resident pages and small sections
 * (zlib's crc32, bit-identical; PCLMUL folding).  No GPU needed. */
uint32_t crac_crc32_host(const void* data, uint64_t n, uint32_t crc);
/* The drain's host-page move: copies n bytes src -> dst (non-temporal stores
 * when dst is 16-byte aligned) and returns crac_crc32_host(src, n, crc) from
 * the same single read of src.  No GPU needed. */
uint32_t crac_crc32_copy_host(void* dst, const void* src, uint64_t n, uint32_t crc);

/* Kernel-level entry for parity tests: CRC of every 64 KiB (chunk_bytes)
 * chunk of a host buffer, computed by K1 on the GPU. */
int crac_hash_host_buffer(const void* data, uint64_t n, uint32_t chunk_bytes, uint32_t* crc_out);

#ifdef __cplusplus
}
#endif

#endif /* CRAC_ENGINE_H */
