// cracsim B200 build — the checkpoint engine.
//
// Drop-in surface of the reference engine (ref: include/cracsim/ckpt_engine.hpp:16-84):
// Session / SessionConfig / checkpoint / checkpoint_to_file / replay_log /
// restart / restart_from_file, with the same semantics (non-destructive
// checkpoint, replay verified address-by-address, ReplayDivergence fatal).
//
// B200 fast path (the timed hot path):
//   checkpoint_image   quiesce -> K1 chunk CRCs (HBM) || pack kernel -> staging
//                      ring -> D2H into a pinned image; host writes the small
//                      sections and folds chunk CRCs into section CRCs.
//                      Bytes equal encode_image(checkpoint(session)).
//   checkpoint_incremental  same bytes; only chunks whose CRC changed since
//                      the previous image of this session cross PCIe.
//   restart_image      strict host parse of the framing -> log replay (same
//                      first-fit, real backing only for allocations live at
//                      the end) -> H2D ring -> scatter kernel -> K1 over the
//                      refilled regions verifies the stored CRCs -> managed
//                      residence restored with cudaMemPrefetchAsync.
// checkpoint()/restart() on Snapshot values are adapters over these.
#pragma once

#include <chrono>
#include <memory>

#include "cracsim/global_barrier.hpp"
#include "cracsim/image.hpp"
#include "cracsim/image_io.hpp"

namespace cracsim {

using KernelCatalog = std::map<std::string, KernelBody, std::less<>>;

struct SessionConfig {
  uint64_t seed = 0;
  uint64_t arena_bytes = 1ull << 24;
  TableMode mode = TableMode::Direct;
  std::chrono::milliseconds quiesce_timeout{30000};
};

struct DrainEngine;  // staging ring, device tables, streams (drain.cu)

class Session {
 public:
  explicit Session(const SessionConfig& cfg);
  ~Session();
  Session(Session&&) noexcept;
  Session& operator=(Session&&) noexcept;

  RuntimeApi& api() { return *table_; }
  DispatchTable& table() { return *table_; }
  DeviceContext& device() { return *ctx_; }
  CallLog& log() { return *log_; }
  RegionMap& regions() { return *regions_; }
  std::vector<uint8_t>& app_state() { return app_state_; }
  const SessionConfig& config() const { return cfg_; }
  DrainEngine& drain_engine();
  // true once drain_engine() has been acquired (its acquisition allocates
  // device and pinned memory, which must not happen before a quiesce: a
  // pinned allocation waits for a kernel stuck on the device)
  bool has_drain_engine() const { return drain_ != nullptr; }
  // Global-checkpoint hook (global_barrier.hpp); called by every checkpoint
  // entry point at kPhaseQuiesced and kPhaseImageComplete.
  void set_barrier(GlobalBarrier b) { barrier_ = b; }
  const GlobalBarrier& barrier() const { return barrier_; }
  // Runs the hook (no-op without one); a nonzero return raises QuiesceTimeout.
  // The wait is added to barrier_ms.
  void global_barrier(int phase);
  double barrier_ms = 0;     // host time in the hook during the last checkpoint
  bool commit_armed = false; // a checkpoint_begin awaits its kPhaseImageComplete

 private:
  SessionConfig cfg_;
  std::unique_ptr<DeviceContext> ctx_;
  std::unique_ptr<CallLog> log_;
  std::unique_ptr<RegionMap> regions_;
  std::unique_ptr<DispatchTable> table_;
  std::vector<uint8_t> app_state_;
  std::unique_ptr<DrainEngine> drain_;
  GlobalBarrier barrier_;
};

// Page-locked host buffer holding one image; reused across checkpoints.  The
// drain places the image so the bulk sections start 4 KiB-aligned.
class PinnedImage {
 public:
  PinnedImage() = default;
  ~PinnedImage();
  PinnedImage(const PinnedImage&) = delete;
  PinnedImage& operator=(const PinnedImage&) = delete;
  PinnedImage(PinnedImage&& o) noexcept;
  PinnedImage& operator=(PinnedImage&& o) noexcept;

  const uint8_t* data() const { return base_ + off_; }
  uint8_t* mutable_data() { return base_ + off_; }
  uint64_t size() const { return size_; }
  std::span<const uint8_t> bytes() const { return {data(), size_}; }
  // Ensures capacity for `size` bytes with (data() + align_at) % 4096 == 0.
  void prepare(uint64_t size, uint64_t align_at);
  void set_size(uint64_t n) { size_ = n; }
  uint64_t capacity() const { return cap_; }
  uint64_t room() const { return cap_ - off_; }  // bytes writable from data()
  // Bytes of the buffer backed by 2 MiB pages (D2H into 4 KiB-backed memory
  // is slower on the B200 box); from /proc/self/smaps.
  uint64_t huge_page_bytes() const;

 private:
  uint8_t* base_ = nullptr;
  uint64_t cap_ = 0;
  uint64_t off_ = 0;
  uint64_t size_ = 0;
};

// Device-timed phase breakdown of the last drain / refill (CUDA events on the
// engine streams; milliseconds).
struct DrainStats {
  double total_ms = 0;       // first to last event of the operation
  double hash_ms = 0;        // K1 span (all launches)
  double pack_ms = 0;        // pack (drain) or scatter (refill) device time per launch
  double copy_ms = 0;        // D2H (drain) or H2D (refill) span
  uint64_t hash_bytes = 0;   // bytes K1 read
  uint64_t hash_launches = 0;
  uint64_t pack_launches = 0;
  uint64_t pack_bytes = 0;   // stream bytes packed / scattered
  uint64_t d2h_bytes = 0;
  uint64_t h2d_bytes = 0;
  uint64_t image_bytes = 0;
  uint64_t dirty_chunks = 0;
  uint64_t total_chunks = 0;
  bool incremental = false;
  double stall_ms = 0;       // quiesce -> app may resume (device events)
  uint64_t shadow_bytes = 0; // stream bytes staged in the HBM shadow
  double barrier_ms = 0;     // host wait in the global-checkpoint hook
  double host_pre_ms = 0;    // refill: parse + session set-up before the first
                             // device event (included in total_ms)
};

// ---- reference surface ----
Snapshot checkpoint(Session& session);
void checkpoint_to_file(Session& session, const std::filesystem::path& path, bool compress = false);
std::map<uint64_t, uint64_t> replay_log(
    DeviceContext& ctx, std::span<const CallLogEntry> log,
    const std::map<uint64_t, std::vector<KernelDescriptor>>* binaries = nullptr);
// replay_log without building the returned map (placed_out may be null).
void replay_log_into(DeviceContext& ctx, std::span<const CallLogEntry> log,
                     const std::map<uint64_t, std::vector<KernelDescriptor>>* binaries,
                     std::map<uint64_t, uint64_t>* placed_out);
Session restart(const Snapshot& snapshot, const KernelCatalog& catalog,
                TableMode mode = TableMode::Direct,
                std::chrono::milliseconds quiesce_timeout = std::chrono::milliseconds{30000});
Session restart_from_file(const std::filesystem::path& path, const KernelCatalog& catalog,
                          TableMode mode = TableMode::Direct);

// ---- B200 fast path ----
// Persistence: the drain into a caller-owned pinned image, then
// parallel O_DIRECT writes of it (image_io.hpp); restart reads the file into
// the caller's pinned staging image in parallel and refills from it.  Same
// files as the reference's checkpoint_to_file / restart_from_file.
void checkpoint_to_file(Session& session, PinnedImage& image, const std::filesystem::path& path,
                        bool compress, DrainStats* drain = nullptr, FileIoStats* io = nullptr);
// Compression of checkpoint_to_file: none, the reference's bytes (zlib
// compress2 level 6 on the host, compress_image), or the GPU deflate
// (compress_image_gpu: a different, valid zlib stream that the reference's
// maybe_decompress inflates to the exact image).
enum class Compression { None = 0, Zlib6 = 1, Gpu = 2 };
void checkpoint_to_file(Session& session, PinnedImage& image, const std::filesystem::path& path,
                        Compression compression, DrainStats* drain = nullptr,
                        FileIoStats* io = nullptr, double* compress_ms = nullptr);
// GPU deflate of an image into a CRACSIMZ wrapper (SURVEY §8f.4, K5 in
// deflate.cu): segments of 32 KiB compressed independently with fixed
// Huffman codes and joined by sync flushes, Adler-32 folded on the host.
std::vector<uint8_t> compress_image_gpu(std::span<const uint8_t> image, double* ms = nullptr);
// The same into caller memory of at least compressed_bound_gpu(n) bytes;
// returns the bytes written.
uint64_t compressed_bound_gpu(uint64_t n);
uint8_t* alloc_compressed_host(uint64_t bytes);  // 2 MiB-aligned, THP; std::free
uint64_t compress_image_gpu_into(std::span<const uint8_t> image, uint8_t* out, uint64_t cap,
                                 double* ms = nullptr);
Session restart_from_file(const std::filesystem::path& path, PinnedImage& staging,
                          const KernelCatalog& catalog, TableMode mode = TableMode::Direct,
                          DrainStats* refill = nullptr, FileIoStats* io = nullptr);
// Reads an image file into `staging` (4 KiB-aligned, page-locked).
void read_image_into(const std::filesystem::path& path, PinnedImage& staging,
                     FileIoStats* io = nullptr);
void checkpoint_image(Session& session, PinnedImage& out, DrainStats* stats = nullptr);
void checkpoint_incremental(Session& session, PinnedImage& image, DrainStats* stats = nullptr);
// Stall-reduced drain.  checkpoint_begin quiesces, drains the
// head of the bulk stream through the ring and packs the rest into the HBM
// shadow reserved with reserve_shadow (K1 and K4 run meanwhile), then resumes
// the app and starts the shadow -> image D2H.  checkpoint_finish waits for it
// and completes `out`: the bytes equal checkpoint_image's at the instant of
// checkpoint_begin, whatever the app does in between.  With no shadow this is
// checkpoint_image.  Any other drain first finishes a pending one.
// `device` >= 0 places the shadow in that GPU's HBM (a buddy GPU reachable by
// peer access): the snapshot crosses NVLink during the stall and
// the buddy's copy engine drains it over the buddy's PCIe link afterwards.
void reserve_shadow(Session& session, uint64_t bytes, int device = -1);
void checkpoint_begin(Session& session, PinnedImage& out, DrainStats* stats = nullptr);
void checkpoint_finish(Session& session, DrainStats* stats = nullptr);
// Pre-copy drain (no spare HBM needed): begin copies the whole
// state into `out` while the application keeps running (K1 hashes each chunk
// and writes the bytes it hashed); finish stops the application and re-sends
// only the chunks that changed since (an incremental drain), so the stall is
// one hash pass plus the changed bytes.  The bytes equal checkpoint_image's at
// the instant of finish.  Device-only sessions; others drain synchronously in
// begin.  finish's stats: stall_ms = the gated phase, total_ms = both phases.
void checkpoint_precopy_begin(Session& session, PinnedImage& out, DrainStats* stats = nullptr);
void checkpoint_precopy_finish(Session& session, DrainStats* stats = nullptr);
// K1 over every live allocation (hash-only timing; no drain).
void hash_only(Session& session, DrainStats* stats);
Session restart_image(std::span<const uint8_t> image, const KernelCatalog& catalog,
                      TableMode mode = TableMode::Direct,
                      std::chrono::milliseconds quiesce_timeout = std::chrono::milliseconds{30000},
                      DrainStats* stats = nullptr);

}  // namespace cracsim
