// cracsim B200 build — image persistence.
//
// Replaces the reference's whole-buffer ofstream/ifstream file I/O
// (ref: src/image.cpp:432-451 write_image_file / read_file_bytes) on the
// checkpoint_to_file / restart_from_file path with parallel positional I/O:
//   * the file is cut into `chunk` byte pieces written / read by a pool of
//     host threads with pwrite / pread, each thread one contiguous run of
//     pieces (CRAC_IO_LAYOUT=interleave hands them out round-robin instead);
//   * an existing file is overwritten in place (no O_TRUNC) and cut to the
//     image size at the end: overwriting mapped blocks is ext4's concurrent
//     O_DIRECT path, and freeing them first queues discards under the writes;
//   * O_DIRECT when the filesystem accepts it (no page-cache copy; the image
//     is already in page-locked memory).  O_DIRECT needs 4 KiB-aligned memory,
//     offsets and lengths: aligned pieces are written straight from the
//     image, the others through a per-thread aligned bounce buffer; reads
//     always land in the bounce buffer and are copied out (a reused buffer
//     reads 1.4x faster than a large image on the box's disk); the last piece
//     is zero-padded to 4 KiB and the file truncated to its true length;
//   * the write ends with fdatasync (a checkpoint is durable when the call
//     returns; the reference only flushes the stream).
// The bytes on disk are exactly the image bytes, so files interoperate with
// the reference reader and writer.
#pragma once

#include <cstdint>
#include <filesystem>
#include <span>

namespace cracsim {

struct FileIoStats {
  double ms = 0;          // wall time of the transfer (open .. fdatasync/close)
  uint64_t bytes = 0;     // file bytes moved
  uint32_t threads = 0;   // I/O threads used
  bool direct = false;    // O_DIRECT was in effect
  uint64_t bounced = 0;   // bytes that went through a bounce buffer
  uint64_t streamed = 0;  // streamed writes: bytes written while the drain still ran
};

struct FileIoOptions {
  uint32_t threads = 0;         // 0 = CRAC_IO_THREADS or min(16, hardware threads)
  uint64_t chunk = 0;           // 0 = CRAC_IO_CHUNK_MIB or 64 MiB (multiple of 4 KiB)
  bool direct = true;           // try O_DIRECT, fall back to buffered I/O if refused
  bool sync = true;             // fdatasync before returning (writes)
};

// Writes `bytes` to `path` (created, or overwritten and cut to size).  InvalidArgument on an I/O
// error (the reference's "cannot write").
void write_file_parallel(const std::filesystem::path& path, std::span<const uint8_t> bytes,
                         FileIoStats* stats = nullptr, const FileIoOptions& opt = {});

// Size of the file at `path`; ImageCorrupt if it cannot be opened (the
// reference's "cannot read").
uint64_t file_bytes(const std::filesystem::path& path);

// Reads the whole file into dst[0, size).  `capacity` must be at least the
// file size; with O_DIRECT, pieces land in place when dst is 4 KiB-aligned
// and capacity >= size rounded up to 4 KiB.  Returns the file size.
uint64_t read_file_parallel(const std::filesystem::path& path, uint8_t* dst, uint64_t capacity,
                            FileIoStats* stats = nullptr, const FileIoOptions& opt = {});

// Producer side of a streamed image write: the drain reports the image
// prefix that has landed in host memory while the D2H is still running, so
// the file write starts under the drain (checkpoint_to_file).
struct LandSink {
  virtual ~LandSink() = default;
  // the image is [base, base + n); called once, before any other call
  virtual void start(const uint8_t* base, uint64_t n) = 0;
  // bytes the producer completes only after the stream has landed (section
  // headers, folded CRCs): written again once every byte is final
  virtual void rewrite(uint64_t a, uint64_t b) = 0;
  // bytes [0, end) hold their final values, except the rewrite ranges
  virtual void landed(uint64_t end) = 0;
};

// A parallel positional writer (the layout and O_DIRECT rules of
// write_file_parallel) that writes each piece as soon as the producer has
// landed it.  finish() is called once the whole image is final: the pieces
// still waiting are written, the rewrite ranges written again (whole 4 KiB
// blocks), the file cut to size and fdatasync'd.  Destroying an unfinished
// writer stops its threads (the file is then incomplete).
class StreamWriter final : public LandSink {
 public:
  explicit StreamWriter(const std::filesystem::path& path, const FileIoOptions& opt = {});
  ~StreamWriter() override;
  StreamWriter(const StreamWriter&) = delete;
  StreamWriter& operator=(const StreamWriter&) = delete;

  void start(const uint8_t* base, uint64_t n) override;
  void rewrite(uint64_t a, uint64_t b) override;
  void landed(uint64_t end) override;
  // `base`/`n` must match start()'s when it was called (else it starts here)
  void finish(const uint8_t* base, uint64_t n, FileIoStats* stats = nullptr);
  // bytes the pieces wrote before finish() was called (streamed under the drain)
  uint64_t early_bytes() const;

 private:
  struct State;
  State* st_;
};

}  // namespace cracsim
