// Host barrier of the global checkpoint (cracsim/global_barrier.hpp).
//
// One 64-bit word in a POSIX shared-memory segment: generation in the high
// half, arrivals in the low half.  An arrival CASes (g, c) -> (g, c + 1), or
// -> (g + 1, 0) when it is the last one, which releases every waiter of
// generation g.  A waiter that times out withdraws its arrival with a CAS
// (g, c) -> (g, c - 1) that only succeeds while generation g is still open, so
// a timed-out rank never leaves a phantom arrival behind.
#include "cracsim/global_barrier.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <thread>

#include "cracsim/base.hpp"

namespace cracsim {
namespace {

constexpr uint32_t kMagicReady = 2;

inline void relax(uint32_t spins) {
  if (spins < 2048) {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  } else if (spins < 4096) {
    std::this_thread::yield();
  } else {
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

}  // namespace

ShmBarrier::ShmBarrier(const std::string& name, uint32_t world, uint32_t rank,
                       std::chrono::milliseconds timeout)
    : name_(name), world_(world), rank_(rank), timeout_(timeout) {
  if (name.size() < 2 || name[0] != '/' || name.find('/', 1) != std::string::npos)
    raise(Errc::InvalidArgument, "barrier name must look like \"/name\": " + name);
  if (world == 0 || rank >= world)
    raise(Errc::InvalidArgument, "barrier rank " + std::to_string(rank) + " outside world " +
                                     std::to_string(world));
  const int fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) raise(Errc::InvalidArgument, "shm_open " + name + ": " + std::strerror(errno));
  // ftruncate only grows a fresh (zero-length) segment: zero-filled = state 0
  struct stat st {};
  if (fstat(fd, &st) != 0 || (st.st_size < off_t(sizeof(Shared)) &&
                              ftruncate(fd, sizeof(Shared)) != 0)) {
    const int e = errno;
    close(fd);
    raise(Errc::InvalidArgument, "sizing barrier segment " + name + ": " + std::strerror(e));
  }
  void* p = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) raise(Errc::InvalidArgument, "mmap barrier segment " + name);
  sh_ = static_cast<Shared*>(p);
  uint32_t s = 0;
  if (sh_->state.compare_exchange_strong(s, 1, std::memory_order_acq_rel)) {
    sh_->world = world;
    sh_->word.store(0, std::memory_order_relaxed);
    sh_->waits.store(0, std::memory_order_relaxed);
    sh_->state.store(kMagicReady, std::memory_order_release);
  } else {
    const auto until = std::chrono::steady_clock::now() + std::chrono::seconds(10);
    for (uint32_t k = 0; sh_->state.load(std::memory_order_acquire) != kMagicReady; ++k) {
      if (std::chrono::steady_clock::now() > until) {
        munmap(sh_, sizeof(Shared));
        sh_ = nullptr;
        raise(Errc::QuiesceTimeout, "barrier segment " + name + " never became ready");
      }
      relax(k);
    }
  }
  if (sh_->world != world) {
    const uint32_t other = sh_->world;
    munmap(sh_, sizeof(Shared));
    sh_ = nullptr;
    raise(Errc::InvalidArgument, "barrier " + name + " was opened for " + std::to_string(other) +
                                     " ranks, not " + std::to_string(world));
  }
}

ShmBarrier::~ShmBarrier() {
  if (sh_) munmap(sh_, sizeof(Shared));
  if (unlink_) shm_unlink(name_.c_str());
}

uint64_t ShmBarrier::generation() const {
  return sh_->word.load(std::memory_order_acquire) >> 32;
}

bool ShmBarrier::wait() {
  std::atomic<uint64_t>& w = sh_->word;
  uint64_t cur = w.load(std::memory_order_acquire);
  uint64_t gen;
  for (;;) {
    gen = cur >> 32;
    const uint64_t arrived = (cur & 0xffffffffull) + 1;
    const uint64_t next = arrived == world_ ? ((gen + 1) << 32) : ((gen << 32) | arrived);
    if (w.compare_exchange_weak(cur, next, std::memory_order_acq_rel, std::memory_order_acquire)) {
      if (arrived == world_) {
        sh_->waits.fetch_add(1, std::memory_order_relaxed);
        return true;
      }
      break;
    }
  }
  const auto until = std::chrono::steady_clock::now() + timeout_;
  for (uint32_t k = 0;; ++k) {
    cur = w.load(std::memory_order_acquire);
    if ((cur >> 32) != gen) return true;
    if ((k & 255) == 255 && std::chrono::steady_clock::now() > until) {
      // withdraw the arrival while generation `gen` is still open
      while ((cur >> 32) == gen) {
        if (w.compare_exchange_weak(cur, cur - 1, std::memory_order_acq_rel,
                                    std::memory_order_acquire))
          return false;
      }
      return true;  // released while withdrawing
    }
    relax(k);
  }
}

int ShmBarrier::hook(void* ctx, int /*phase*/) {
  return static_cast<ShmBarrier*>(ctx)->wait() ? 0 : 1;
}

}  // namespace cracsim
