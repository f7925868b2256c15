// Storage probe for image persistence: parallel pwrite/pread of
// a large buffer to a directory, buffered and O_DIRECT.
//   probe_io <dir> <GiB> [threads] [chunk_MiB]
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>
static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static double run(const std::string& path, char* buf, size_t n, unsigned th, size_t chunk, bool write,
                  bool direct) {
  int flags = write ? (O_WRONLY | O_CREAT) : O_RDONLY;
  if (direct) flags |= O_DIRECT;
  int fd = open(path.c_str(), flags, 0644);
  if (fd < 0) { perror("open"); return -1; }
  if (write) ftruncate(fd, n);
  std::atomic<size_t> next{0};
  std::atomic<int> err{0};
  double t = now();
  std::vector<std::thread> pool;
  for (unsigned i = 0; i < th; ++i)
    pool.emplace_back([&] {
      for (;;) {
        size_t o = next.fetch_add(chunk);
        if (o >= n) break;
        size_t len = chunk < n - o ? chunk : n - o;
        size_t done = 0;
        while (done < len) {
          ssize_t r = write ? pwrite(fd, buf + o + done, len - done, o + done)
                            : pread(fd, buf + o + done, len - done, o + done);
          if (r <= 0) { err = errno ? errno : -1; return; }
          done += r;
        }
      }
    });
  for (auto& x : pool) x.join();
  if (write) fdatasync(fd);
  double dt = now() - t;
  close(fd);
  if (err) { printf("  error %d (%s)\n", err.load(), strerror(err.load())); return -1; }
  return n / dt / 1e9;
}
int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : "/tmp";
  size_t n = (size_t)(argc > 2 ? atof(argv[2]) : 8) << 30;
  unsigned th = argc > 3 ? atoi(argv[3]) : 8;
  size_t chunk = (size_t)(argc > 4 ? atol(argv[4]) : 16) << 20;
  char* buf = (char*)mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  madvise(buf, n, MADV_HUGEPAGE);
  for (size_t o = 0; o < n; o += 4096) buf[o] = (char)(o >> 12);
  std::string path = dir + "/crac_probe_io.bin";
  for (int direct = 0; direct < 2; ++direct) {
    double w = run(path, buf, n, th, chunk, true, direct);
    // drop the page cache copy of this file so the read hits the device
    int fd = open(path.c_str(), O_RDONLY);
    if (fd >= 0) { posix_fadvise(fd, 0, 0, POSIX_FADV_DONTNEED); close(fd); }
    double r = run(path, buf, n, th, chunk, false, direct);
    printf("%s %s: write %.2f GB/s (incl fdatasync), read %.2f GB/s, %u threads, %zu MiB chunks\n",
           dir.c_str(), direct ? "O_DIRECT" : "buffered", w, r, th, chunk >> 20);
    fflush(stdout);
  }
  unlink(path.c_str());
  return 0;
}
