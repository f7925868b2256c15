// Parallel positional file I/O for checkpoint images.
// Replaces ref: src/image.cpp:432-451 (write_image_file / read_file_bytes:
// one ofstream/ifstream over the whole buffer).  See cracsim/image_io.hpp.
#include "cracsim/image_io.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "cracsim/base.hpp"

namespace cracsim {
namespace {

constexpr uint64_t kBlock = 4096;

uint64_t round_block(uint64_t n) { return (n + kBlock - 1) / kBlock * kBlock; }

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

uint32_t io_threads(const FileIoOptions& o) {
  if (o.threads) return o.threads;
  if (const char* e = std::getenv("CRAC_IO_THREADS")) {
    const long v = std::atol(e);
    if (v > 0) return static_cast<uint32_t>(std::min(v, 256L));
  }
  return std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
}

uint64_t io_chunk(const FileIoOptions& o) {
  uint64_t c = o.chunk;
  if (!c)
    if (const char* e = std::getenv("CRAC_IO_CHUNK_MIB")) c = uint64_t(std::max(1L, std::atol(e))) << 20;
  if (!c) c = 64ull << 20;  // measured best on the box's virtio disk (profiles/r01d)
  return std::max(kBlock, c / kBlock * kBlock);
}

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

// Opens with O_DIRECT when asked and the filesystem accepts it.
int open_maybe_direct(const std::filesystem::path& path, int flags, bool want_direct, bool* direct) {
  *direct = false;
  if (want_direct) {
    const int fd = ::open(path.c_str(), flags | O_DIRECT | O_CLOEXEC, 0644);
    if (fd >= 0) {
      *direct = true;
      return fd;
    }
    if (errno != EINVAL) return -1;  // a real error, not "no O_DIRECT here"
  }
  return ::open(path.c_str(), flags | O_CLOEXEC, 0644);
}

struct AlignedBuf {
  uint8_t* p = nullptr;
  explicit AlignedBuf(uint64_t n) { p = static_cast<uint8_t*>(std::aligned_alloc(kBlock, round_block(n))); }
  ~AlignedBuf() { std::free(p); }
};

// Runs fn(piece_index) for every piece on `threads` workers; the first error
// (errno) stops the others.  Each worker owns one bounce buffer.
// Piece order: "striped" gives each thread one contiguous run of pieces (a
// sequential stream per thread, what the virtio disk of the B200 box serves
// best); "interleave" hands out pieces from a shared counter.
bool striped_layout() {
  const char* e = std::getenv("CRAC_IO_LAYOUT");
  return !(e && std::strcmp(e, "interleave") == 0);
}

template <typename Fn>
int run_pieces(uint64_t pieces, uint32_t threads, uint64_t bounce_bytes, Fn&& fn) {
  std::atomic<uint64_t> next{0};
  std::atomic<int> err{0};
  threads = static_cast<uint32_t>(std::min<uint64_t>(threads, std::max<uint64_t>(pieces, 1)));
  const bool striped = striped_layout();
  auto worker = [&](uint32_t t) {
    std::unique_ptr<AlignedBuf> bounce;
    uint64_t k = striped ? pieces * t / threads : 0;
    const uint64_t end = striped ? pieces * (t + 1) / threads : pieces;
    for (;; ++k) {
      if (err.load(std::memory_order_relaxed)) return;
      if (!striped) k = next.fetch_add(1);
      if (k >= end) return;
      const int e = fn(k, t, bounce, bounce_bytes);
      if (e) {
        int expected = 0;
        err.compare_exchange_strong(expected, e);
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (uint32_t t = 1; t < threads; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& t : pool) t.join();
  return err.load();
}

int full_pwrite(int fd, const uint8_t* p, uint64_t n, uint64_t off) {
  while (n) {
    const ssize_t r = ::pwrite(fd, p, n, static_cast<off_t>(off));
    if (r < 0) {
      if (errno == EINTR) continue;
      return errno;
    }
    if (r == 0) return EIO;
    p += r;
    n -= uint64_t(r);
    off += uint64_t(r);
  }
  return 0;
}

// Reads until `want` bytes or EOF; stores the count in *got.
int full_pread(int fd, uint8_t* p, uint64_t n, uint64_t off, uint64_t want, uint64_t* got) {
  uint64_t done = 0;
  while (done < want) {
    const ssize_t r = ::pread(fd, p + done, n - done, static_cast<off_t>(off + done));
    if (r < 0) {
      if (errno == EINTR) continue;
      return errno;
    }
    if (r == 0) break;
    done += uint64_t(r);
  }
  *got = done;
  return 0;
}

}  // namespace

void write_file_parallel(const std::filesystem::path& path, std::span<const uint8_t> bytes,
                         FileIoStats* stats, const FileIoOptions& opt) {
  const double t0 = now_ms();
  const uint64_t n = bytes.size();
  const uint64_t chunk = io_chunk(opt);
  const uint32_t threads = io_threads(opt);
  bool direct = false;
  // No O_TRUNC: an existing image is overwritten in place and cut to size at
  // the end.  Overwriting mapped blocks is ext4's concurrent O_DIRECT path
  // (4.3-4.9 GB/s on the box against 3.6-4.1 for a fresh file), and freeing
  // the old blocks first would also queue discards on the (discard-mounted)
  // disk under the new writes (2.5 GB/s measured; profiles/r01d).
  Fd f{open_maybe_direct(path, O_WRONLY | O_CREAT, opt.direct, &direct)};
  if (f.fd < 0) raise(Errc::InvalidArgument, "cannot write " + path.string() + ": " + std::strerror(errno));
  // Experiment knob CRAC_IO_PREALLOC = fallocate | truncate | none (default):
  // size the file before the writes (no measurable gain, tools/io_variants.py).
  const char* pre = std::getenv("CRAC_IO_PREALLOC");
  const std::string prealloc = pre ? pre : "none";
  int prc = 0;
  if (n && prealloc == "fallocate") {
    prc = ::fallocate(f.fd, 0, 0, static_cast<off_t>(n));
    if (prc != 0) prc = ::ftruncate(f.fd, static_cast<off_t>(n));
  } else if (n && prealloc == "truncate") {
    prc = ::ftruncate(f.fd, static_cast<off_t>(n));
  }
  if (prc != 0)
    raise(Errc::InvalidArgument, "cannot write " + path.string() + ": " + std::strerror(errno));
  // experiment knob: one open file description per thread
  const bool fd_per_thread = std::getenv("CRAC_IO_FD_PER_THREAD") != nullptr;
  const uint8_t* src = bytes.data();
  const bool src_aligned = reinterpret_cast<uintptr_t>(src) % kBlock == 0;
  const uint64_t pieces = (n + chunk - 1) / chunk;
  std::atomic<uint64_t> bounced{0};
  std::vector<Fd> fds(fd_per_thread ? threads : 0);
  for (Fd& x : fds)
    if ((x.fd = ::open(path.c_str(), O_WRONLY | O_CLOEXEC | (direct ? O_DIRECT : 0))) < 0)
      raise(Errc::InvalidArgument, "cannot write " + path.string() + ": " + std::strerror(errno));
  const int err = run_pieces(pieces, threads, chunk, [&](uint64_t k, uint32_t t,
                                                          std::unique_ptr<AlignedBuf>& b,
                                                          uint64_t bb) -> int {
    const int fd = fd_per_thread ? fds[t].fd : f.fd;
    const uint64_t off = k * chunk, len = std::min(chunk, n - off);
    if (!direct) return full_pwrite(fd, src + off, len, off);
    const uint64_t padded = round_block(len);
    if (src_aligned && padded == len) return full_pwrite(fd, src + off, len, off);
    if (!b) b = std::make_unique<AlignedBuf>(bb);
    if (!b->p) return ENOMEM;
    std::memcpy(b->p, src + off, len);
    std::memset(b->p + len, 0, padded - len);
    bounced.fetch_add(len, std::memory_order_relaxed);
    return full_pwrite(fd, b->p, padded, off);
  });
  if (err) raise(Errc::InvalidArgument, "cannot write " + path.string() + ": " + std::strerror(err));
  if (::ftruncate(f.fd, static_cast<off_t>(n)) != 0)  // padded tail, or a longer old image
    raise(Errc::InvalidArgument, "cannot write " + path.string() + ": " + std::strerror(errno));
  if (opt.sync && ::fdatasync(f.fd) != 0 && errno != EINVAL)
    raise(Errc::InvalidArgument, "cannot write " + path.string() + ": " + std::strerror(errno));
  if (::close(f.fd) != 0) {
    f.fd = -1;
    raise(Errc::InvalidArgument, "cannot write " + path.string() + ": " + std::strerror(errno));
  }
  f.fd = -1;
  if (stats) *stats = FileIoStats{now_ms() - t0, n, std::min<uint32_t>(threads, uint32_t(std::max<uint64_t>(pieces, 1))), direct, bounced.load()};
}

// ---------------------------------------------------------------------------
// streamed write (checkpoint_to_file under the drain)
// ---------------------------------------------------------------------------
struct StreamWriter::State {
  std::filesystem::path path;
  FileIoOptions opt;
  Fd f;
  bool direct = false;
  uint64_t chunk = 0;
  uint32_t threads = 0;
  const uint8_t* base = nullptr;
  uint64_t n = 0;
  std::mutex mu;
  std::condition_variable cv;
  uint64_t landed = 0;   // [0, landed) final except the rewrite ranges
  bool final_all = false, stop = false, started = false;
  std::vector<std::pair<uint64_t, uint64_t>> rewrites;
  std::vector<std::thread> pool;
  std::atomic<int> err{0};
  std::atomic<uint64_t> bounced{0}, early{0};
  double t0 = 0;

  int write_range(uint64_t off, uint64_t len, std::unique_ptr<AlignedBuf>& b) {
    if (!direct) return full_pwrite(f.fd, base + off, len, off);
    const uint64_t padded = round_block(len);
    if (reinterpret_cast<uintptr_t>(base + off) % kBlock == 0 && padded == len)
      return full_pwrite(f.fd, base + off, len, off);
    if (!b) b = std::make_unique<AlignedBuf>(chunk);
    if (!b->p) return ENOMEM;
    std::memcpy(b->p, base + off, len);
    std::memset(b->p + len, 0, padded - len);
    bounced.fetch_add(len, std::memory_order_relaxed);
    return full_pwrite(f.fd, b->p, padded, off);
  }

  // thread t: its contiguous run of pieces, each once the producer has landed it
  void worker(uint32_t t) {
    const uint64_t pieces = (n + chunk - 1) / chunk;
    std::unique_ptr<AlignedBuf> b;
    for (uint64_t k = pieces * t / threads; k < pieces * (t + 1) / threads; ++k) {
      const uint64_t off = k * chunk, len = std::min(chunk, n - off);
      bool early_piece;
      {
        std::unique_lock lk(mu);
        cv.wait(lk, [&] { return stop || final_all || landed >= off + len; });
        if (stop) return;
        early_piece = !final_all;
      }
      if (err.load(std::memory_order_relaxed)) return;
      if (const int e = write_range(off, len, b)) {
        int expected = 0;
        err.compare_exchange_strong(expected, e);
        return;
      }
      if (early_piece) early.fetch_add(len, std::memory_order_relaxed);
    }
  }

  void halt() {
    {
      std::lock_guard lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& th : pool)
      if (th.joinable()) th.join();
    pool.clear();
  }
};

StreamWriter::StreamWriter(const std::filesystem::path& path, const FileIoOptions& opt)
    : st_(new State) {
  State& S = *st_;
  S.path = path;
  S.opt = opt;
  S.t0 = now_ms();
  S.chunk = io_chunk(opt);
  S.threads = io_threads(opt);
  // in place, as write_file_parallel (no O_TRUNC; cut to size at the end)
  S.f.fd = open_maybe_direct(path, O_WRONLY | O_CREAT, opt.direct, &S.direct);
  if (S.f.fd < 0) {
    const std::string why = std::strerror(errno);
    delete st_;
    raise(Errc::InvalidArgument, "cannot write " + path.string() + ": " + why);
  }
}

StreamWriter::~StreamWriter() {
  st_->halt();
  delete st_;
}

void StreamWriter::start(const uint8_t* base, uint64_t n) {
  State& S = *st_;
  if (S.started) return;
  S.started = true;
  S.base = base;
  S.n = n;
  const uint64_t pieces = (n + S.chunk - 1) / S.chunk;
  S.threads = uint32_t(std::min<uint64_t>(S.threads, std::max<uint64_t>(pieces, 1)));
  for (uint32_t t = 0; t < S.threads && pieces; ++t) S.pool.emplace_back([&S, t] { S.worker(t); });
}

void StreamWriter::rewrite(uint64_t a, uint64_t b) {
  std::lock_guard lk(st_->mu);
  if (b > a) st_->rewrites.emplace_back(a, b);
}

void StreamWriter::landed(uint64_t end) {
  {
    std::lock_guard lk(st_->mu);
    if (end <= st_->landed) return;
    st_->landed = end;
  }
  st_->cv.notify_all();
}

uint64_t StreamWriter::early_bytes() const { return st_->early.load(); }

void StreamWriter::finish(const uint8_t* base, uint64_t n, FileIoStats* stats) {
  State& S = *st_;
  if (S.started && (base != S.base || n != S.n)) {
    S.halt();  // the producer's buffer moved: nothing written so far counts
    S.started = false;
    S.rewrites.clear();
    S.early = 0;
    S.threads = io_threads(S.opt);
  }
  if (!S.started) start(base, n);
  {
    std::lock_guard lk(S.mu);
    S.final_all = true;
    S.landed = n;
  }
  S.cv.notify_all();
  for (auto& th : S.pool) th.join();
  S.pool.clear();
  auto fail = [&](int e) { raise(Errc::InvalidArgument, "cannot write " + S.path.string() + ": " + std::strerror(e)); };
  if (const int e = S.err.load()) fail(e);
  // the ranges the producer completed after they streamed, as whole blocks
  std::sort(S.rewrites.begin(), S.rewrites.end());
  std::unique_ptr<AlignedBuf> b;
  uint64_t done = 0;  // blocks below this are written again already
  for (auto [a, e] : S.rewrites) {
    a = std::max(a / kBlock * kBlock, done);
    e = std::min(round_block(std::min(e, n)), round_block(n));
    if (a >= e) continue;
    for (uint64_t off = a; off < e; off += S.chunk) {
      const uint64_t len = std::min({S.chunk, e - off, n - off});
      if (const int er = S.write_range(off, len, b)) fail(er);
    }
    done = e;
  }
  if (::ftruncate(S.f.fd, static_cast<off_t>(n)) != 0) fail(errno);
  if (S.opt.sync && ::fdatasync(S.f.fd) != 0 && errno != EINVAL) fail(errno);
  const int fd = S.f.fd;
  S.f.fd = -1;
  if (::close(fd) != 0) fail(errno);
  if (stats)
    *stats = FileIoStats{now_ms() - S.t0, n, S.threads, S.direct, S.bounced.load()};
}

uint64_t file_bytes(const std::filesystem::path& path) {
  Fd f{::open(path.c_str(), O_RDONLY | O_CLOEXEC)};
  struct stat st {};
  if (f.fd < 0 || ::fstat(f.fd, &st) != 0 || !S_ISREG(st.st_mode))
    raise(Errc::ImageCorrupt, "cannot read " + path.string());
  return static_cast<uint64_t>(st.st_size);
}

uint64_t read_file_parallel(const std::filesystem::path& path, uint8_t* dst, uint64_t capacity,
                            FileIoStats* stats, const FileIoOptions& opt) {
  const double t0 = now_ms();
  bool direct = false;
  Fd f{open_maybe_direct(path, O_RDONLY, opt.direct, &direct)};
  struct stat st {};
  if (f.fd < 0 || ::fstat(f.fd, &st) != 0 || !S_ISREG(st.st_mode))
    raise(Errc::ImageCorrupt, "cannot read " + path.string());
  const uint64_t n = static_cast<uint64_t>(st.st_size);
  if (n > capacity) raise(Errc::InvalidArgument, "buffer too small for " + path.string());
  const uint64_t chunk = io_chunk(opt);
  const uint32_t threads = io_threads(opt);
  // O_DIRECT reads land in a reused per-thread bounce buffer and are copied
  // out: 4.1-4.3 GB/s on the box's disk against 2.9 straight into a large
  // image (dd's 4.0-4.4 reads into one reused buffer too; io_read_variants.py).
  // CRAC_IO_BOUNCE_READ=0 reads in place when the destination allows it.
  const char* bounce_env = std::getenv("CRAC_IO_BOUNCE_READ");
  const bool in_place = reinterpret_cast<uintptr_t>(dst) % kBlock == 0 && capacity >= round_block(n) &&
                        bounce_env && !std::strcmp(bounce_env, "0");
  const uint64_t pieces = (n + chunk - 1) / chunk;
  // experiment knob: one open file description per thread (as dd runs)
  const bool fd_per_thread = std::getenv("CRAC_IO_FD_PER_THREAD") != nullptr;
  std::vector<Fd> fds(fd_per_thread ? std::min<uint64_t>(threads, std::max<uint64_t>(pieces, 1)) : 0);
  for (Fd& x : fds)
    if ((x.fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC | (direct ? O_DIRECT : 0))) < 0)
      raise(Errc::ImageCorrupt, "cannot read " + path.string());
  std::atomic<uint64_t> bounced{0};
  std::atomic<bool> short_read{false};
  const int err = run_pieces(pieces, threads, chunk, [&](uint64_t k, uint32_t t,
                                                          std::unique_ptr<AlignedBuf>& b,
                                                          uint64_t bb) -> int {
    const int fd = fd_per_thread ? fds[t].fd : f.fd;
    const uint64_t off = k * chunk, len = std::min(chunk, n - off);
    uint64_t got = 0;
    int e;
    if (!direct || in_place) {
      e = full_pread(fd, dst + off, direct ? round_block(len) : len, off, len, &got);
    } else {
      if (!b) b = std::make_unique<AlignedBuf>(bb);
      if (!b->p) return ENOMEM;
      e = full_pread(fd, b->p, round_block(len), off, len, &got);
      if (!e) std::memcpy(dst + off, b->p, std::min(got, len));
      bounced.fetch_add(len, std::memory_order_relaxed);
    }
    if (!e && got < len) short_read = true;  // the file shrank underneath us
    return e;
  });
  if (err || short_read) raise(Errc::ImageCorrupt, "cannot read " + path.string());
  if (stats) *stats = FileIoStats{now_ms() - t0, n, std::min<uint32_t>(threads, uint32_t(std::max<uint64_t>(pieces, 1))), direct, bounced.load()};
  return n;
}

}  // namespace cracsim
