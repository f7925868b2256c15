// Per-session state of the B200 drain/refill pipeline (internal).
//
// HBM layout owned here (allocated once, grown geometrically, reused by every
// checkpoint; engines are pooled across sessions so restarts reuse them):
//   ring      kSlots x (kWindow + 64) bytes  staging for the section stream
//   recs      crac_record_t per framed record of ALLOC_PAYLOADS + UVM_PAGES
//   tile_rec  u32 per 64 KiB stream tile: first record overlapping it
//   spans/first/crc  K1 inputs/outputs: payload spans (64 KiB chunks) and
//             managed spans (4 KiB chunks = one CRC per page)
//   prev_crc / dirty_idx / block_counts / pay_dst   incremental state (K2b)
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>
#include <memory>
#include <new>
#include <utility>
#include <vector>

#include "crac_gpu.h"
#include "cracsim/ckpt_engine.hpp"

namespace cracsim {

struct LandSink;  // cracsim/image_io.hpp
// The streamed file write that follows the next full drain on this thread
// (checkpoint_to_file); null = none.  The drain reports the landed image
// prefix to it when the whole stream goes through the ring windows with no
// host-written pages; otherwise it reports nothing and the writer writes the
// finished image.
void set_land_sink(LandSink* sink);

// Phase tracing for diagnosis: CRAC_TRACE=1 prints host-side phase times of
// every drain / refill to stderr.
struct PhaseTrace {
  const char* op;
  double t0, last;
  bool on;
  explicit PhaseTrace(const char* name);
  void mark(const char* phase);
  ~PhaseTrace();
};

template <typename T>
struct DevArray {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  void ensure(size_t n);
  void release();
};

template <typename T>
struct HostArray {  // pinned
  T* ptr = nullptr;
  size_t cap = 0;
  void ensure(size_t n);
  void release();
};

// Page-locked storage for big host tables that are uploaded every drain (the
// record table: 268 MB for C3's 4 M pages), so the upload is a real async DMA
// rather than a staged pageable copy; elements are default-initialised (a
// resize does not zero memory the plan overwrites anyway).
template <typename T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <typename U>
  PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      throw std::bad_alloc();
    }
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) { cudaFreeHost(p); }
  template <typename U, typename... A>
  void construct(U* p, A&&... a) {
    if constexpr (sizeof...(A) == 0)
      ::new (static_cast<void*>(p)) U;
    else
      ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
  }
  bool operator==(const PinnedAlloc&) const { return true; }
};

// Layout of the last image this session drained (enables incremental drains).
// A host-resident managed page: its content is copied by host threads
// between the managed allocation and the image (never crosses PCIe).
// Its CRC is computed by the host thread that moves it (h_host_crc[k] for
// host_pages[k]); K1 hashes device-resident pages only.
struct HostPage {
  uint64_t stream_off;  // content offset in the bulk stream
  uint64_t ptr;         // managed address of the page
  uint32_t len, ext;    // content bytes; bytes to write on refill (zero tail)
  uint64_t rec;         // its record in ImagePlan::recs (ptr zeroed there)
  bool own_frame = false;  // in a skipped host run: the host writes its frame too
};

struct ImagePlan {
  uint64_t image_bytes = 0;
  uint64_t image_ptr = 0;   // where that image lives (host)
  uint64_t s3 = 0;          // file offset of the ALLOC_PAYLOADS payload (= stream start)
  uint64_t len3 = 0, len4 = 0;
  uint64_t stream_len = 0;  // len3 + 20 + len4
  std::vector<crac_record_t, PinnedAlloc<crac_record_t>> recs;
  // the arrays upload_plan copies to the device are page-locked, so those
  // copies are plain DMA (no staging through the driver's pageable path)
  std::vector<uint32_t, PinnedAlloc<uint32_t>> tile_rec;
  std::vector<crac_span_t, PinnedAlloc<crac_span_t>> pay_spans, page_spans;  // page_spans: device-resident runs
  std::vector<uint64_t, PinnedAlloc<uint64_t>> pay_first, page_first;
  // page-CRC index space (record.reserved): device-resident pages [0, n_dev),
  // in page_spans order; host-resident pages n_dev + k for host_pages[k]
  uint64_t n_dev_pages = 0;
  std::vector<uint64_t> pay_rec_off;  // stream offset of each payload's first byte
  std::vector<uint64_t> log_sizes;    // signature: (id, size) of every bulk record
  std::vector<HostPage> host_pages;   // host-resident managed pages
  // stream ranges of host-resident pages only (frames + content), long
  // enough that the window copies skip them (plan_host_runs)
  std::vector<std::pair<uint64_t, uint64_t>> host_runs;
  // Direct runs (plan_direct_runs): tile-aligned interiors of big Device
  // payloads, copied by the copy engine straight between the allocation and
  // the image -- no pack / scatter, no HBM staging.  `dev` = device address
  // of stream byte `lo`.
  struct DirectRun {
    uint64_t lo, hi, dev;
    bool exact_end = false;  // hi is the payload's last byte + 1 (no padding): no straddle
  };
  std::vector<DirectRun> direct_runs;
  std::vector<std::pair<uint64_t, uint64_t>> skip_runs;  // host ∪ direct, sorted
  // Pinned-host payload contents of at least kSkipMin (plan_host_runs): they
  // live in host memory, so host threads copy them between the allocation and
  // the image; no window copy, pack or scatter touches them (their records
  // carry ptr 0) and they never cross PCIe for the move.  Also in host_runs.
  struct PinnedRun {
    uint64_t lo, hi;  // stream range of the content
    uint64_t host;    // the allocation's host address of stream byte lo
    uint64_t pay;     // payload index (its chunks: pay_first[pay] .. pay_first[pay + 1])
    uint64_t pin0;    // first slot of its chunks in h_pin_crc / h_pin_key
  };
  std::vector<PinnedRun> pinned_runs;
  uint64_t pinned_chunks = 0;  // chunks of all pinned runs
  std::vector<uint8_t> pay_kind;  // AllocationKind of each payload record
  uint64_t log_len = 0;
  uint64_t tail_bytes = 0;  // STREAMS + APPSTATE + KERNEL_REGISTRY, framed
  bool valid = false;
};

struct DrainEngine {
  static constexpr int kSlots = 4;
  static constexpr uint64_t kWindow = 64ull << 20;     // pack/scatter launch (multiple of 64 KiB)
  static constexpr uint64_t kCopyChunk = 16ull << 20;  // D2H/H2D piece (tools/ab_piece.sh: box-dependent, 16 MiB never the outlier)
  static constexpr uint32_t kChunk = 65536;         // payload hash chunk
  static constexpr uint32_t kPageChunk = 4096;      // managed hash chunk (= page)
  static constexpr int kPackSMs = 16;               // SMs K1 leaves to the pack during a drain
  static constexpr int kPackSMsDirect = 4;          // ... when direct copies carry the payloads

  int device = 0;
  int sm_count = 148;
  cudaStream_t s_pack = nullptr, s_copy = nullptr, s_hash = nullptr;
  cudaEvent_t ev_ready[kSlots] = {}, ev_free[kSlots] = {};
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr, ev_h0 = nullptr, ev_h1 = nullptr;
  cudaEvent_t ev_c0 = nullptr, ev_c1 = nullptr;
  std::vector<cudaEvent_t> ev_w0, ev_w1;  // per-window kernel timing (stats only)
  std::vector<cudaEvent_t> ev_v0, ev_v1;  // per refill-verify K1 launch (stats only)
  uint8_t* d_ring = nullptr;

  DevArray<crac_record_t> d_recs;
  DevArray<uint32_t> d_tile_rec;
  DevArray<crac_span_t> d_pay_spans, d_page_spans;
  DevArray<uint64_t> d_pay_first, d_page_first, d_pay_dst, d_pay_soff;
  DevArray<uint32_t> d_pay_crc, d_page_crc, d_prev_crc, d_block_counts;
  // second dirty-key lane of every payload chunk (crac_chunk_key_range): the
  // incremental / pre-copy drains compare (crc, key), a 64-bit dirty key
  DevArray<uint32_t> d_pay_key, d_prev_key;
  DevArray<uint64_t> d_dirty_idx, d_dirty_count;
  DevArray<unsigned long long> d_counters;
  DevArray<uint32_t> d_fold;   // linear parts of crc3 / crc4 (K4)
  HostArray<uint32_t> h_fold;
  HostArray<uint32_t> h_host_crc;          // CRCs of host-resident pages (host threads)
  // chunk CRCs / keys of the pinned-host payloads the host threads move
  // (ImagePlan::pinned_runs), uploaded into d_pay_crc / d_pay_key
  HostArray<uint32_t> h_pin_crc, h_pin_key;
  std::vector<cudaEvent_t> ev_land;        // window w's D2H has landed (host-page copies)
  HostArray<uint64_t> h_count, h_dirty_idx;

  // Stall-reduced drain (checkpoint_begin/finish): the tail of the bulk
  // stream is packed into this HBM shadow while the app is quiesced and copied
  // out after it resumes.  Reserved explicitly (reserve_shadow), never inside
  // a drain.
  cudaStream_t s_shadow = nullptr;
  cudaEvent_t ev_s1 = nullptr, ev_join[3] = {};
  uint8_t* d_shadow = nullptr;
  uint64_t shadow_cap = 0;
  // Buddy shadow: the shadow may live in a peer GPU's HBM,
  // written over NVLink by this GPU's kernels (peer access) and drained to
  // the host by the peer's own copy engine on the peer's PCIe link.
  int shadow_device = -1;           // -1: this device
  cudaStream_t s_peer = nullptr;    // on shadow_device
  cudaEvent_t ev_peer = nullptr;    // on shadow_device: the shadow D2H is done
  struct Pending {
    bool active = false;
    PinnedImage* out = nullptr;
    uint64_t head = 0;       // stream bytes drained through the ring (stall)
    uint32_t crc3 = 0, crc4 = 0;
    uint64_t windows = 0;    // ring windows (stats)
    uint64_t packed = 0;     // stream bytes the ring windows' pack kernels produced
    uint64_t launches = 0, ring_launches = 0;  // pack launches: all / of the ring windows
    bool timed = false;      // the ring windows recorded ev_w0 / ev_w1 (drain_locked had stats)
    double stall_ms = 0;
    // host-resident pages of short runs in the shadow part, copied while the
    // app was stopped; written into the image after the shadow D2H lands
    std::vector<uint8_t> stash;
    std::vector<std::pair<uint64_t, uint32_t>> stash_at;  // (stream_off, len)
    bool precopy = false;  // a pre-copy pass (checkpoint_precopy_begin) is in flight
  } pending;

  ImagePlan plan;
  // host scratch of the drain prologue, reused (no page faults on fresh
  // megabyte-sized vectors: C2's 40 k-entry log)
  std::vector<AllocationRecord> scratch_active;
  std::vector<uint8_t> scratch_alive;
  bool prev_valid = false;      // d_prev_crc holds the chunk CRCs of `plan`'s image
  uint64_t dst_for_image = 0;   // image the d_pay_dst table was built for

  explicit DrainEngine(int dev);
  ~DrainEngine();
  DrainEngine(const DrainEngine&) = delete;
  DrainEngine& operator=(const DrainEngine&) = delete;
  void ensure_window_events(size_t n);
  void ensure_verify_events(size_t n);
  void ensure_land_events(size_t n);
};

// Frees the (possibly buddy-GPU) shadow of an engine.
void free_shadow(DrainEngine& E);

// Process-wide engine pool (Session construction / destruction).
std::unique_ptr<DrainEngine> acquire_engine(int device);
void release_engine(std::unique_ptr<DrainEngine> e);

}  // namespace cracsim
