// Session lifecycle, log replay, and the value-type (Snapshot) adapters over
// the B200 drain/refill (drain.cu).
#include <cstdlib>
#include <cstring>

#include "cracsim/image_io.hpp"
#include "drain_engine.hpp"
#include "image_codec.hpp"

namespace cracsim {

Session::Session(const SessionConfig& cfg)
    : cfg_(cfg),
      ctx_(std::make_unique<DeviceContext>(cfg.seed, cfg.arena_bytes)),
      log_(std::make_unique<CallLog>()),
      regions_(std::make_unique<RegionMap>()),
      table_(std::make_unique<DispatchTable>(*ctx_, *log_, *regions_, cfg.mode)) {}

Session::~Session() {
  PhaseTrace tr("close");
  release_engine(std::move(drain_));  // pooled for the next session on this device
  tr.mark("engine");
  // the members in their default destruction order, timed under CRAC_TRACE
  table_.reset();
  regions_.reset();
  tr.mark("table+regions");
  log_.reset();
  tr.mark("log");
  ctx_.reset();
  tr.mark("context");
}
Session::Session(Session&&) noexcept = default;
Session& Session::operator=(Session&&) noexcept = default;

void Session::global_barrier(int phase) {
  if (!barrier_) return;
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = barrier_.fn(barrier_.ctx, phase);
  barrier_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (rc != 0)
    raise(Errc::QuiesceTimeout, "global checkpoint barrier failed at phase " + std::to_string(phase) +
                                    " (hook returned " + std::to_string(rc) + ")");
}

DrainEngine& Session::drain_engine() {
  if (!drain_) drain_ = acquire_engine(ctx_->device());
  return *drain_;
}

// ref: ckpt_engine.cpp:29-61.  The snapshot is decoded from the image the
// GPU drain produced, so both APIs share one hot path.
Snapshot checkpoint(Session& session) {
  PinnedImage img;
  checkpoint_image(session, img);
  std::vector<uint8_t> bytes(img.data(), img.data() + img.size());
  return decode_image(bytes);
}

// ref: ckpt_engine.cpp:63-65 (the drain itself is the GPU path; the file is
// written from the pinned image by the parallel writer, compressed on request).
void checkpoint_to_file(Session& session, const std::filesystem::path& path, bool compress) {
  PinnedImage img;
  checkpoint_to_file(session, img, path, compress);
}

void checkpoint_to_file(Session& session, PinnedImage& image, const std::filesystem::path& path,
                        bool compress, DrainStats* drain, FileIoStats* io) {
  checkpoint_to_file(session, image, path, compress ? Compression::Zlib6 : Compression::None, drain,
                     io);
}

void checkpoint_to_file(Session& session, PinnedImage& image, const std::filesystem::path& path,
                        Compression compression, DrainStats* drain, FileIoStats* io,
                        double* compress_ms) {
  if (compress_ms) *compress_ms = 0;
  // CRAC_FILE_STREAM=1: the file write runs under the drain: each piece is
  // written once the windows covering it have landed in the image
  // (StreamWriter), the bytes the host completes afterwards are written again
  // at the end.  Off by default: on the box's virtio disk it measured 1-4 %
  // slower than drain-then-write (profiles/r02/file_stream.txt) -- the disk
  // binds, and its 16 write streams start staggered behind the landing
  // windows instead of together
  const char* stream_env = std::getenv("CRAC_FILE_STREAM");
  const bool stream = stream_env && !std::strcmp(stream_env, "1");
  if (compression == Compression::None && stream) {
    StreamWriter w(path);
    struct Scope {
      explicit Scope(LandSink* s) { set_land_sink(s); }
      ~Scope() { set_land_sink(nullptr); }
    } scope(&w);
    checkpoint_image(session, image, drain);
    set_land_sink(nullptr);
    w.finish(image.bytes().data(), image.size(), io);
    if (io) io->streamed = w.early_bytes();
    session.global_barrier(kPhasePersisted);
    if (drain) drain->barrier_ms = session.barrier_ms;
    return;
  }
  checkpoint_image(session, image, drain);
  if (compression == Compression::Zlib6) {
    const auto t0 = std::chrono::steady_clock::now();
    const std::vector<uint8_t> z = compress_image(image.bytes());
    if (compress_ms)
      *compress_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    write_file_parallel(path, z, io);
  } else if (compression == Compression::Gpu) {
    const uint64_t cap = compressed_bound_gpu(image.size());
    std::unique_ptr<uint8_t, decltype(&std::free)> z(alloc_compressed_host(cap), &std::free);
    const uint64_t zn = compress_image_gpu_into(image.bytes(), z.get(), cap, compress_ms);
    write_file_parallel(path, {z.get(), zn}, io);
  } else {
    write_file_parallel(path, image.bytes(), io);
  }
  // every rank's file is durable (write_file_parallel ends with fdatasync)
  session.global_barrier(kPhasePersisted);
  if (drain) drain->barrier_ms = session.barrier_ms;
}

void read_image_into(const std::filesystem::path& path, PinnedImage& staging, FileIoStats* io) {
  const uint64_t n = file_bytes(path);
  staging.prepare(n, 0);  // data() 4 KiB-aligned: O_DIRECT lands in place
  staging.set_size(read_file_parallel(path, staging.mutable_data(), staging.room(), io));
}

// ref: ckpt_engine.cpp:67-118 — re-execute in seq order, verify every result.
std::map<uint64_t, uint64_t> replay_log(
    DeviceContext& ctx, std::span<const CallLogEntry> log,
    const std::map<uint64_t, std::vector<KernelDescriptor>>* binaries) {
  std::map<uint64_t, uint64_t> placed;
  replay_log_into(ctx, log, binaries, &placed);
  return placed;
}

// The restart path does not need the seq -> address map (C2: 28 k inserts).
void replay_log_into(DeviceContext& ctx, std::span<const CallLogEntry> log,
                     const std::map<uint64_t, std::vector<KernelDescriptor>>* binaries,
                     std::map<uint64_t, uint64_t>* placed_out) {
  auto diverged = [](const CallLogEntry& e, const std::string& what) {
    raise(Errc::ReplayDivergence, "seq " + std::to_string(e.seq) + ": " + what);
  };
  for (const CallLogEntry& e : log) {
    switch (e.op) {
      case LogOp::Alloc: {
        const AllocationRecord rec = ctx.alloc(static_cast<AllocationKind>(e.kind), e.size);
        if (rec.id != e.id)
          diverged(e, "id " + std::to_string(rec.id) + " != logged " + std::to_string(e.id));
        if (rec.address != e.address)
          diverged(e, "address mismatch for allocation " + std::to_string(e.id));
        if (placed_out) placed_out->emplace_hint(placed_out->end(), e.seq, rec.address);  // seq ascends
        break;
      }
      case LogOp::Free: ctx.free(e.id); break;
      case LogOp::StreamCreate:
        if (ctx.stream_create() != e.id) diverged(e, "stream id mismatch");
        break;
      case LogOp::StreamDestroy: ctx.stream_destroy(e.id); break;
      case LogOp::RegisterBinary: {
        // binaries unregistered before the checkpoint replay as empty
        // placeholders so later handles line up (ref: ckpt_engine.cpp:98-110)
        std::vector<KernelDescriptor> kernels;
        if (binaries)
          if (auto it = binaries->find(e.id); it != binaries->end()) kernels = it->second;
        if (ctx.register_fat_binary(std::move(kernels)) != e.id) diverged(e, "handle mismatch");
        break;
      }
      case LogOp::UnregisterBinary: ctx.unregister_fat_binary(e.id); break;
    }
  }
}

// ref: ckpt_engine.cpp:120-171, via the GPU refill.
Session restart(const Snapshot& snapshot, const KernelCatalog& catalog, TableMode mode,
                std::chrono::milliseconds quiesce_timeout) {
  for (const BinaryInfo& b : snapshot.binaries)
    for (const KernelInfo& k : b.kernels)
      if (!catalog.count(k.name))
        raise(Errc::UnknownKernelBody, "no body registered for kernel '" + k.name + "'");
  const std::vector<uint8_t> image = encode_image(snapshot);
  try {
    return restart_image(image, catalog, mode, quiesce_timeout);
  } catch (const Error& e) {
    // a snapshot that does not frame consistently is a replay mismatch here
    // (the reference checks payload/record agreement during restart)
    if (e.code() == Errc::ImageCorrupt) raise(Errc::ReplayDivergence, e.what());
    throw;
  }
}

Session restart_from_file(const std::filesystem::path& path, const KernelCatalog& catalog,
                          TableMode mode) {
  PinnedImage staging;
  return restart_from_file(path, staging, catalog, mode);
}

Session restart_from_file(const std::filesystem::path& path, PinnedImage& staging,
                          const KernelCatalog& catalog, TableMode mode, DrainStats* refill,
                          FileIoStats* io) {
  read_image_into(path, staging, io);
  return restart_image(staging.bytes(), catalog, mode, std::chrono::milliseconds{30000}, refill);
}

}  // namespace cracsim
