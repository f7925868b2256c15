// The B200 hot path: checkpoint drain and restart refill.
//
// Drain  (replaces ref: src/ckpt_engine.cpp:29-61 checkpoint + src/image.cpp:383-399
//         encode_image; the read_raw copies at ckpt_engine.cpp:49,54):
//   host  : quiesce, small sections (META/LOG/STREAMS/APPSTATE/REGISTRY),
//           record table of the bulk stream ALLOC_PAYLOADS||crc3||hdr4||UVM_PAGES
//   GPU   : s_hash  K1 over every payload (64 KiB chunks) and every run of
//                   device-resident managed pages, on all but kPackSMs SMs so
//                   the pack never waits for it; K4 folds the section CRCs
//           s_pack  pack kernel builds the exact stream bytes window by window
//                   into a 4 x 64 MiB staging ring
//           s_copy  D2H of each window into the pinned image (4 KiB aligned),
//                   skipping host runs (plan_host_runs)
//   host  : threads hash (PCLMUL CRC) and copy host-resident managed pages
//           beside the window loop, then crc3/crc4 are patched.
// Refill (replaces ref: src/image.cpp:280-345 decode + src/ckpt_engine.cpp:120-171):
//   host  : strict parse of the framing, replay of the log (real backing only
//           for allocations live at the end, pre-mapped in coalesced runs);
//           Device-only images at the fixed VA start the data path first
//   GPU   : s_copy H2D windows (+16 B look-ahead) -> ring, and direct H2D of
//           big payload interiors straight into their allocations
//           (plan_direct_runs); s_pack scatter kernel writes the rest (padding
//           zero-filled), then K1 re-hashes regions in 2 GiB batches as their
//           last window lands
//   host  : threads write and hash host-resident managed pages (first touch
//           restores residence), then fold + compare -> ImageCorrupt.
// Incremental drain (new; the reference has none): K1 compares every chunk's
//   CRC with the previous image's; writer CTAs copy the dirty chunks straight
//   into the pinned image (crac_hash_drain_split).
// Stall reduction (new): the HBM shadow (checkpoint_begin/finish) and the
//   pre-copy drain (checkpoint_precopy_begin/finish).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <optional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <atomic>
#include <climits>
#include <exception>
#include <mutex>
#include <set>
#include <thread>

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <cctype>
#include <string>

#include "crc_math.hpp"
#include "cracsim/image_io.hpp"
#include "drain_engine.hpp"
#include "image_codec.hpp"

namespace cracsim {

namespace {
thread_local LandSink* t_land_sink = nullptr;
}  // namespace

void set_land_sink(LandSink* sink) { t_land_sink = sink; }

// ---------------------------------------------------------------------------
// tracing
// ---------------------------------------------------------------------------
namespace {
double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
bool trace_on() {
  static const bool on = std::getenv("CRAC_TRACE") != nullptr;
  return on;
}
}  // namespace

PhaseTrace::PhaseTrace(const char* name) : op(name), t0(now_ms()), last(t0), on(trace_on()) {}
void PhaseTrace::mark(const char* phase) {
  if (!on) return;
  const double t = now_ms();
  std::fprintf(stderr, "[crac] %s %-14s %9.3f ms\n", op, phase, t - last);
  last = t;
}
PhaseTrace::~PhaseTrace() {
  if (on) std::fprintf(stderr, "[crac] %s %-14s %9.3f ms\n", op, "TOTAL", now_ms() - t0);
}

// ---------------------------------------------------------------------------
// buffers
// ---------------------------------------------------------------------------
// cudaMalloc that, when the device is out of memory, first frees a closed
// session's cached arena (and waits for arena releases in flight) and retries
static cudaError_t engine_malloc(void** p, size_t n) {
  cudaError_t e = cudaMalloc(p, n);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
      drop_arena_cache(dev);
      e = cudaMalloc(p, n);
    }
  }
  return e;
}

template <typename T>
void DevArray<T>::ensure(size_t n) {
  if (n <= cap) return;
  release();
  const size_t c = std::max<size_t>(n + n / 2, 64);
  check_cuda(engine_malloc(reinterpret_cast<void**>(&ptr), c * sizeof(T)), "cudaMalloc engine array");
  cap = c;
}
template <typename T>
void DevArray<T>::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  cap = 0;
}
template <typename T>
void HostArray<T>::ensure(size_t n) {
  if (n <= cap) return;
  release();
  const size_t c = std::max<size_t>(n + n / 2, 64);
  check_cuda(cudaHostAlloc(reinterpret_cast<void**>(&ptr), c * sizeof(T), cudaHostAllocDefault),
             "cudaHostAlloc engine array");
  cap = c;
}
template <typename T>
void HostArray<T>::release() {
  if (ptr) cudaFreeHost(ptr);
  ptr = nullptr;
  cap = 0;
}

DrainEngine::DrainEngine(int dev) : device(dev) {
  int lo = 0, hi = 0;
  check_cuda(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities");
  check_cuda(cudaStreamCreateWithPriority(&s_pack, cudaStreamNonBlocking, hi), "pack stream");
  check_cuda(cudaStreamCreateWithPriority(&s_copy, cudaStreamNonBlocking, hi), "copy stream");
  check_cuda(cudaStreamCreateWithPriority(&s_hash, cudaStreamNonBlocking, lo), "hash stream");
  check_cuda(cudaStreamCreateWithPriority(&s_shadow, cudaStreamNonBlocking, hi), "shadow stream");
  check_cuda(cudaEventCreate(&ev_s1), "event");
  for (cudaEvent_t& e : ev_join) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  for (int i = 0; i < kSlots; ++i) {
    check_cuda(cudaEventCreateWithFlags(&ev_ready[i], cudaEventDisableTiming), "event");
    check_cuda(cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming), "event");
  }
  for (cudaEvent_t* e : {&ev_t0, &ev_t1, &ev_h0, &ev_h1, &ev_c0, &ev_c1})
    check_cuda(cudaEventCreate(e), "event");
  check_cuda(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev), "sm count");
  check_cuda(engine_malloc(reinterpret_cast<void**>(&d_ring), kSlots * (kWindow + 64)), "staging ring");
  if (int rc = crac_gpu_init()) check_cuda(cudaError_t(rc), "crac_gpu_init");
}

DrainEngine::~DrainEngine() {
  cudaDeviceSynchronize();
  for (int i = 0; i < kSlots; ++i) {
    cudaEventDestroy(ev_ready[i]);
    cudaEventDestroy(ev_free[i]);
  }
  for (cudaEvent_t e : ev_w0) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_w1) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_v0) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_v1) cudaEventDestroy(e);
  for (cudaEvent_t e : {ev_t0, ev_t1, ev_h0, ev_h1, ev_c0, ev_c1}) cudaEventDestroy(e);
  cudaFree(d_ring);
  free_shadow(*this);
  if (s_peer) cudaStreamDestroy(s_peer);
  if (ev_peer) cudaEventDestroy(ev_peer);
  cudaEventDestroy(ev_s1);
  for (cudaEvent_t e : ev_join) cudaEventDestroy(e);
  cudaStreamDestroy(s_shadow);
  d_recs.release();
  d_tile_rec.release();
  d_pay_spans.release();
  d_page_spans.release();
  d_pay_first.release();
  d_page_first.release();
  d_pay_dst.release();
  d_pay_soff.release();
  d_pay_crc.release();
  d_page_crc.release();
  d_prev_crc.release();
  d_pay_key.release();
  d_prev_key.release();
  d_block_counts.release();
  d_dirty_idx.release();
  d_dirty_count.release();
  d_counters.release();
  d_fold.release();
  h_fold.release();
  h_count.release();
  h_dirty_idx.release();
  cudaStreamDestroy(s_pack);
  cudaStreamDestroy(s_copy);
  cudaStreamDestroy(s_hash);
}

void DrainEngine::ensure_verify_events(size_t n) {
  while (ev_v0.size() < n) {
    cudaEvent_t a, b;
    check_cuda(cudaEventCreate(&a), "event");
    check_cuda(cudaEventCreate(&b), "event");
    ev_v0.push_back(a);
    ev_v1.push_back(b);
  }
}

void DrainEngine::ensure_land_events(size_t n) {
  while (ev_land.size() < n) {
    cudaEvent_t a;
    check_cuda(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "event");
    ev_land.push_back(a);
  }
}

void DrainEngine::ensure_window_events(size_t n) {
  while (ev_w0.size() < n) {
    cudaEvent_t a, b;
    check_cuda(cudaEventCreate(&a), "event");
    check_cuda(cudaEventCreate(&b), "event");
    ev_w0.push_back(a);
    ev_w1.push_back(b);
  }
}

// Engines (streams, events, staging ring, device tables) outlive sessions:
// a restart reuses the engine of the session it replaces, so no timed step
// pays for cudaMalloc / stream creation.  Deliberately never freed at exit.
namespace {
std::mutex g_pool_mu;
std::vector<DrainEngine*>* g_pool = new std::vector<DrainEngine*>();
}  // namespace

std::unique_ptr<DrainEngine> acquire_engine(int device) {
  {
    std::lock_guard lk(g_pool_mu);
    for (auto it = g_pool->begin(); it != g_pool->end(); ++it)
      if ((*it)->device == device) {
        DrainEngine* e = *it;
        g_pool->erase(it);
        return std::unique_ptr<DrainEngine>(e);
      }
  }
  return std::make_unique<DrainEngine>(device);
}

// Frees the shadow on the device that holds it.
void free_shadow(DrainEngine& E) {
  if (E.d_shadow) {
    if (E.shadow_device >= 0) {
      cudaStreamSynchronize(E.s_peer);
      cudaSetDevice(E.shadow_device);
      cudaFree(E.d_shadow);
      cudaSetDevice(E.device);
    } else {
      cudaFree(E.d_shadow);
    }
  }
  E.d_shadow = nullptr;
  E.shadow_cap = 0;
  E.shadow_device = -1;
}

void release_engine(std::unique_ptr<DrainEngine> e) {
  if (!e) return;
  if (cudaStreamSynchronize(e->s_pack) != cudaSuccess ||
      cudaStreamSynchronize(e->s_copy) != cudaSuccess ||
      cudaStreamSynchronize(e->s_hash) != cudaSuccess ||
      cudaStreamSynchronize(e->s_shadow) != cudaSuccess)
    return;  // a broken engine is dropped (and leaked), never pooled
  e->pending = DrainEngine::Pending{};  // an unfinished async drain is abandoned
  free_shadow(*e);  // the shadow belongs to its session
  e->plan.valid = false;  // keep the vectors' capacity for the next session
  e->plan.image_ptr = 0;
  e->prev_valid = false;
  e->dst_for_image = 0;
  std::lock_guard lk(g_pool_mu);
  if (g_pool->size() < 4) g_pool->push_back(e.release());
}

// ---------------------------------------------------------------------------
// pinned image
// ---------------------------------------------------------------------------
// Page-locked host memory for images.  cudaHostAlloc faults and pins 4 KiB
// pages one by one (~2.3 GB/s measured on the B200 box); instead map
// anonymous memory with transparent huge pages, first-touch it from all
// cores, then register it with the driver (~28 GB/s measured, and the same
// 55.9 GB/s D2H into it).
namespace {
constexpr int kMadvCollapse = 25;  // MADV_COLLAPSE (Linux 6.1); older kernels return EINVAL

}  // namespace

// AnonHugePages of the mapping that contains `p` (/proc/self/smaps), in bytes.
uint64_t mapping_huge_bytes(const void* p) {
  FILE* f = std::fopen("/proc/self/smaps", "r");
  if (!f) return 0;
  const uint64_t a = reinterpret_cast<uint64_t>(p);
  char line[512];
  bool in = false;
  uint64_t huge = 0;
  while (std::fgets(line, sizeof line, f)) {
    uint64_t lo, hi;
    if (std::sscanf(line, "%lx-%lx ", &lo, &hi) == 2 && std::strchr(line, '-') < std::strchr(line, ' ')) {
      if (in) break;
      in = a >= lo && a < hi;
    } else if (in && !std::strncmp(line, "AnonHugePages:", 14)) {
      huge = std::strtoull(line + 14, nullptr, 10) << 10;
    }
  }
  std::fclose(f);
  return huge;
}

namespace {
// NUMA node the current GPU hangs off (sysfs numa_node of its PCI function),
// or -1 on single-node hosts, unknown topology, or CRAC_NUMA=off.
int device_numa_node() {
  if (const char* e = std::getenv("CRAC_NUMA"); e && !std::strcmp(e, "off")) return -1;
  char online[64] = {};
  if (FILE* f = std::fopen("/sys/devices/system/node/online", "r")) {
    if (!std::fgets(online, sizeof online, f)) online[0] = 0;
    std::fclose(f);
  }
  if (!std::strchr(online, '-') && !std::strchr(online, ',')) return -1;  // one node
  int dev = 0;
  char bus[32] = {};
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  for (char* c = bus; *c; ++c) *c = char(std::tolower(*c));
  int node = -1;
  if (FILE* f = std::fopen((std::string("/sys/bus/pci/devices/") + bus + "/numa_node").c_str(), "r")) {
    if (std::fscanf(f, "%d", &node) != 1) node = -1;
    std::fclose(f);
  }
  return node >= 0 && node < 64 ? node : -1;
}

uint8_t* pinned_alloc(uint64_t bytes) {
  void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE,
                 -1, 0);
  if (m == MAP_FAILED) raise(Errc::DeviceFault, "mmap of the image buffer failed");
  madvise(m, bytes, MADV_HUGEPAGE);
  // On multi-socket hosts put the image on the GPU's own node, so the DMA of
  // every GPU of the box stays off the socket interconnect (MPOL_PREFERRED:
  // spills rather than fails when the node is full).
  if (const int node = device_numa_node(); node >= 0) {
    constexpr int kMpolPreferred = 1;
    unsigned long mask = 1ul << node;
    syscall(SYS_mbind, m, bytes, kMpolPreferred, &mask, 64ul, 0u);
  }
  const unsigned threads = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([=] {
      const uint64_t a = bytes * t / threads / 4096 * 4096, b = bytes * (t + 1) / threads;
      for (uint64_t o = a; o < b; o += 4096) static_cast<volatile uint8_t*>(m)[o] = 0;
    });
  for (auto& th : pool) th.join();
  // Fault-time THP can fall back to 4 KiB pages when free memory is
  // fragmented; every measured fast drain had the image fully on 2 MiB pages
  // (the bench reports the coverage).  Collapse whatever the fault path
  // missed (best effort).
  if (mapping_huge_bytes(m) + (4ull << 20) < bytes) madvise(m, bytes, kMadvCollapse);
  const cudaError_t e = cudaHostRegister(m, bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    munmap(m, bytes);
    check_cuda(e, "cudaHostRegister image");
  }
  return static_cast<uint8_t*>(m);
}

void pinned_free(uint8_t* p, uint64_t bytes) {
  if (!p) return;
  cudaHostUnregister(p);
  munmap(p, bytes);
}
}  // namespace

PinnedImage::~PinnedImage() { pinned_free(base_, cap_); }
uint64_t PinnedImage::huge_page_bytes() const { return base_ ? mapping_huge_bytes(base_) : 0; }
PinnedImage::PinnedImage(PinnedImage&& o) noexcept
    : base_(o.base_), cap_(o.cap_), off_(o.off_), size_(o.size_) {
  o.base_ = nullptr;
  o.cap_ = o.off_ = o.size_ = 0;
}
PinnedImage& PinnedImage::operator=(PinnedImage&& o) noexcept {
  if (this != &o) {
    pinned_free(base_, cap_);
    base_ = o.base_;
    cap_ = o.cap_;
    off_ = o.off_;
    size_ = o.size_;
    o.base_ = nullptr;
    o.cap_ = o.off_ = o.size_ = 0;
  }
  return *this;
}

void PinnedImage::prepare(uint64_t size, uint64_t align_at) {
  const uint64_t need = (size + 4096 + (2ull << 20) - 1) / (2ull << 20) * (2ull << 20);
  if (need > cap_) {
    pinned_free(base_, cap_);
    base_ = nullptr;
    cap_ = 0;
    base_ = pinned_alloc(need);
    cap_ = need;
  }
  const uint64_t b = reinterpret_cast<uint64_t>(base_);
  off_ = (4096 - (b + align_at) % 4096) % 4096;
  size_ = size;
}

// ---------------------------------------------------------------------------
// CRC helpers
// ---------------------------------------------------------------------------
namespace {

using namespace codec;

const uint32_t* pow2_table() {
  static const std::vector<uint32_t> t = [] {
    std::vector<uint32_t> v(64);
    v[0] = 0x00800000u;
    for (int k = 1; k < 64; ++k) v[k] = crac::gf_mul(v[k - 1], v[k - 1]);
    return v;
  }();
  return t.data();
}

// fn(0..n-1) on up to 16 host threads (only worth it for big plans).
template <typename Fn>
void parallel_for(uint64_t n, Fn&& fn, uint64_t min_parallel = 4096) {
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  if (n < min_parallel || hw == 1) {
    for (uint64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  // blocks small enough that a few big items (managed allocations) spread
  const uint64_t blk = std::max<uint64_t>(1, std::min<uint64_t>(1024, n / (4 * hw)));
  std::atomic<uint64_t> next{0};
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < hw; ++t)
    pool.emplace_back([&] {
      for (uint64_t b; (b = next.fetch_add(blk)) < n;)
        for (uint64_t i = b; i < std::min(n, b + blk); ++i) fn(i);
    });
  for (auto& th : pool) th.join();
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float v = 0;
  cudaEventElapsedTime(&v, a, b);
  return v;
}

// Median duration of the first n window kernels (robust to the windows that
// ran beside K1 at the start of a drain).
// device time of the ring windows' pack launches, per launch
double mean_pack_launch_ms(DrainEngine& E, size_t windows, uint64_t launches) {
  if (!launches) return 0;
  double t = 0;
  for (size_t i = 0; i < windows; ++i) t += elapsed(E.ev_w0[i], E.ev_w1[i]);
  return t / double(launches);
}

// Bulk-stream plan shared by drain and refill.  `ptr` = device-visible
// address of the region (drain: source; refill: destination).
struct BulkItem {
  uint64_t id = 0;
  AllocationKind kind = AllocationKind::Device;
  uint64_t size = 0;
  uint64_t ptr = 0;
  const std::vector<uint8_t>* flags = nullptr;  // managed page flags
};

void build_plan(const std::vector<BulkItem>& items, ImagePlan& P) {
  PhaseTrace tr("  plan");
  P.page_spans.clear();
  P.page_first.assign(1, 0);
  // every payload array sized once and filled by index (C2: 16 k payloads)
  uint64_t n_pay = 0, n_recs = 1;
  for (const BulkItem& it : items) {
    const bool managed = it.kind == AllocationKind::Managed;
    n_pay += !managed;
    n_recs += managed ? 1 + page_count_for(it.size) : 1;
  }
  P.recs.reserve(n_recs);  // one allocation for the whole record table
  P.recs.resize(n_pay);
  P.pay_spans.resize(n_pay);
  P.pay_first.resize(n_pay + 1);
  P.pay_first[0] = 0;
  P.pay_rec_off.resize(n_pay);
  P.pay_kind.resize(n_pay);
  P.log_sizes.resize(2 * items.size());
  uint64_t pos = 0, len4 = 0, k = 0, first = 0;
  for (size_t j = 0; j < items.size(); ++j) {
    const BulkItem& it = items[j];
    P.log_sizes[2 * j] = it.id;
    P.log_sizes[2 * j + 1] = it.size;
    if (it.kind == AllocationKind::Managed) {
      len4 += 16 + 16 * page_count_for(it.size) + it.size;
      continue;
    }
    crac_record_t& r = P.recs[k];
    r = crac_record_t{};
    r.out_off = pos;
    r.ptr = it.ptr;
    r.len = it.size;
    r.ext = round_up_align(it.size);
    r.frame_len = 16;
    std::memcpy(r.frame, &it.id, 8);
    std::memcpy(r.frame + 8, &it.size, 8);
    P.pay_spans[k] = crac_span_t{it.ptr, it.size};
    first += (it.size + DrainEngine::kChunk - 1) / DrainEngine::kChunk;
    P.pay_first[k + 1] = first;
    P.pay_rec_off[k] = pos + 16;
    P.pay_kind[k] = uint8_t(it.kind);
    pos += 16 + it.size;
    ++k;
  }
  P.len3 = pos;
  P.len4 = len4;
  {  // crc3 placeholder + the UVM_PAGES section header, as one frame-only record
    crac_record_t g{};
    g.out_off = pos;
    g.frame_len = 20;
    const uint32_t tag = 4, zero = 0;
    std::memcpy(g.frame + 4, &tag, 4);
    std::memcpy(g.frame + 8, &zero, 4);
    std::memcpy(g.frame + 12, &len4, 8);
    P.recs.push_back(g);
    pos += 20;
  }
  tr.mark("payloads");
  // managed allocations: lay out offsets and page-CRC indices first, then
  // fill the page records of every allocation in parallel (C3 has millions of
  // pages).  Device-resident pages are hashed by K1 as runs (page_spans);
  // host-resident ones (flag bit0 clear) are moved and hashed by host
  // threads, never by the SMs: pack emits zeros for them, scatter skips them.
  struct Slot {
    const BulkItem* it;
    size_t rec0;
    uint64_t pos0, dev0, host0;
  };
  std::vector<const BulkItem*> managed;
  for (const BulkItem& it : items)
    if (it.kind == AllocationKind::Managed) managed.push_back(&it);
  // per allocation (in parallel): its device-resident runs and host count
  std::vector<std::vector<crac_span_t>> runs(managed.size());
  std::vector<uint64_t> host_n(managed.size(), 0);
  parallel_for(managed.size(), [&](uint64_t k) {
    const BulkItem& it = *managed[k];
    const uint64_t pages = page_count_for(it.size);
    const uint8_t* f = it.flags ? it.flags->data() : nullptr;
    for (uint64_t p = 0; p < pages;) {
      if (f && !(f[p] & 1)) {
        ++host_n[k];
        ++p;
        continue;
      }
      uint64_t q = p + 1;
      while (q < pages && !(f && !(f[q] & 1))) ++q;
      const uint64_t lo = p * kPageSize, hi = std::min(it.size, q * kPageSize);
      runs[k].push_back(crac_span_t{it.ptr + lo, hi - lo});
      p = q;
    }
  }, /*min_parallel=*/2);
  std::vector<Slot> slots;
  uint64_t n_dev = 0, n_host = 0;
  for (size_t k = 0; k < managed.size(); ++k) {
    const BulkItem& it = *managed[k];
    const uint64_t pages = page_count_for(it.size);
    slots.push_back(Slot{&it, P.recs.size(), pos, n_dev, n_host});
    P.recs.resize(P.recs.size() + 1 + pages);
    pos += 16 + 16 * pages + it.size;
    n_dev += pages - host_n[k];
    n_host += host_n[k];
    for (const crac_span_t& r : runs[k]) {  // device-resident runs, in page-index order
      P.page_spans.push_back(r);
      P.page_first.push_back(P.page_first.back() + (r.len + kPageSize - 1) / kPageSize);
    }
  }
  P.n_dev_pages = n_dev;
  tr.mark("layout");
  P.host_pages.assign(n_host, HostPage{});
  parallel_for(slots.size(), [&](uint64_t k) {
    const Slot& sl = slots[k];
    const BulkItem& it = *sl.it;
    const uint64_t pages = page_count_for(it.size), padded = round_up_align(it.size);
    crac_record_t& h = P.recs[sl.rec0];
    h = crac_record_t{};
    h.out_off = sl.pos0;
    h.frame_len = 16;
    std::memcpy(h.frame, &it.id, 8);
    std::memcpy(h.frame + 8, &pages, 8);
    uint64_t at = sl.pos0 + 16;
    uint64_t dp = sl.dev0, hp = sl.host0;
    for (uint64_t p = 0; p < pages; ++p) {
      const uint64_t off = p * kPageSize;
      const uint32_t len = uint32_t(std::min<uint64_t>(kPageSize, it.size - off));
      const uint32_t fl = it.flags ? (*it.flags)[p] : 0;
      const bool host = it.flags && !(fl & 1);
      crac_record_t& r = P.recs[sl.rec0 + 1 + p];
      r = crac_record_t{};
      r.out_off = at;
      r.ptr = host ? 0 : it.ptr + off;
      r.len = len;
      r.ext = p + 1 == pages ? padded - off : len;
      r.frame_len = 16;
      r.reserved = uint32_t(host ? n_dev + hp : dp);  // its page-CRC index
      std::memcpy(r.frame, &p, 8);
      std::memcpy(r.frame + 8, &fl, 4);
      std::memcpy(r.frame + 12, &len, 4);
      if (host)
        P.host_pages[hp++] = HostPage{at + 16, it.ptr + off, len, uint32_t(r.ext), sl.rec0 + 1 + p};
      else
        ++dp;
      at += 16 + len;
    }
  }, /*min_parallel=*/2);
  tr.mark("pages");
  P.stream_len = pos;
  const uint64_t tiles = (pos + CRAC_TILE_BYTES - 1) / CRAC_TILE_BYTES;
  P.tile_rec.resize(tiles);
  // last record starting at or before each tile: one sequential merge of the
  // two sorted lists for small streams (C2), a parallel binary search per
  // tile for big ones (C3's 4 M page records, C4's 2 M tiles)
  if (tiles < 65536) {
    size_t r = 0;
    const size_t nr = P.recs.size();
    for (uint64_t t = 0; t < tiles; ++t) {
      const uint64_t start = t * CRAC_TILE_BYTES;
      while (r + 1 < nr && P.recs[r + 1].out_off <= start) ++r;
      P.tile_rec[t] = uint32_t(r);
    }
  } else {
    parallel_for(tiles, [&](uint64_t t) {
      const uint64_t start = t * CRAC_TILE_BYTES;
      const auto it = std::upper_bound(P.recs.begin(), P.recs.end(), start,
                                       [](uint64_t v, const crac_record_t& r) { return v < r.out_off; });
      P.tile_rec[t] = uint32_t((it - P.recs.begin()) - 1);
    });
  }
}

template <typename D, typename H>
void upload(D& dev, const H& host, cudaStream_t st) {
  if (host.empty()) return;
  dev.ensure(host.size());
  check_cuda(cudaMemcpyAsync(dev.ptr, host.data(), host.size() * sizeof(host[0]),
                             cudaMemcpyHostToDevice, st),
             "plan upload");
}

void upload_plan(DrainEngine& E, const ImagePlan& P, cudaStream_t st) {
  upload(E.d_recs, P.recs, st);
  upload(E.d_tile_rec, P.tile_rec, st);
  upload(E.d_pay_spans, P.pay_spans, st);
  upload(E.d_pay_first, P.pay_first, st);
  upload(E.d_page_spans, P.page_spans, st);
  upload(E.d_page_first, P.page_first, st);
  const uint64_t n_pay = P.pay_first.back(), n_page = P.n_dev_pages + P.host_pages.size();
  E.d_pay_crc.ensure(std::max<uint64_t>(n_pay, 1));
  E.d_pay_key.ensure(std::max<uint64_t>(n_pay, 1));
  E.d_page_crc.ensure(std::max<uint64_t>(n_page, 1));
}

// with_key: also the chunks' second dirty-key lane (drains and hash-only,
// whose chunk keys seed the next incremental drain; not the refill verify)
void hash_payloads(DrainEngine& E, const ImagePlan& P, uint64_t c_lo, uint64_t c_hi,
                   uint32_t max_ctas, cudaStream_t st, bool with_key = true) {
  check_cuda(cudaError_t(crac_chunk_key_range(E.d_pay_spans.ptr, E.d_pay_first.ptr,
                                              uint32_t(P.pay_spans.size()), DrainEngine::kChunk,
                                              c_lo, c_hi, E.d_pay_crc.ptr,
                                              with_key ? E.d_pay_key.ptr : nullptr, max_ctas, st)),
             "K1 payloads");
}

// The previous image's dirty keys := this pass's (CRC and key lanes).
void seed_prev_keys(DrainEngine& E, uint64_t n_pay, cudaStream_t st) {
  E.d_prev_crc.ensure(n_pay);
  E.d_prev_key.ensure(n_pay);
  check_cuda(cudaMemcpyAsync(E.d_prev_crc.ptr, E.d_pay_crc.ptr, n_pay * 4,
                             cudaMemcpyDeviceToDevice, st),
             "seed prev crc");
  check_cuda(cudaMemcpyAsync(E.d_prev_key.ptr, E.d_pay_key.ptr, n_pay * 4,
                             cudaMemcpyDeviceToDevice, st),
             "seed prev key");
}

void hash_pages(DrainEngine& E, const ImagePlan& P, uint32_t max_ctas, cudaStream_t st) {
  check_cuda(cudaError_t(crac_chunk_crc32_range(E.d_page_spans.ptr, E.d_page_first.ptr,
                                                uint32_t(P.page_spans.size()),
                                                DrainEngine::kPageChunk, 0, P.page_first.back(),
                                                E.d_page_crc.ptr, max_ctas, st)),
             "K1 pages");
}

uint64_t hashed_bytes(const ImagePlan& P) {
  uint64_t b = 0;
  for (const auto& s : P.pay_spans) b += s.len;
  for (const auto& s : P.page_spans) b += s.len;
  return b;
}

// Section CRCs on the device (K4): enqueues the fold and the 8-byte readback
// on `st`; finish_fold() applies K(section length) once `st` has completed.
void enqueue_fold(DrainEngine& E, const ImagePlan& P, cudaStream_t st) {
  E.d_fold.ensure(2);
  E.h_fold.ensure(2);
  check_cuda(cudaError_t(crac_fold_sections(E.d_recs.ptr, uint32_t(P.recs.size()), E.d_pay_first.ptr,
                                            E.d_pay_crc.ptr, uint32_t(P.pay_spans.size()),
                                            E.d_page_crc.ptr, P.len3, P.pay_first.back(),
                                            E.d_fold.ptr, st)),
             "fold");
  check_cuda(cudaMemcpyAsync(E.h_fold.ptr, E.d_fold.ptr, 8, cudaMemcpyDeviceToHost, st), "fold out");
}

void finish_fold(const DrainEngine& E, const ImagePlan& P, uint32_t& crc3, uint32_t& crc4) {
  crc3 = E.h_fold.ptr[0] ^ crac::crc_affine(P.len3, pow2_table());
  crc4 = E.h_fold.ptr[1] ^ crac::crc_affine(P.len4, pow2_table());
}

// Host runs: maximal stream ranges made only of host-resident pages (frame +
// content of consecutive pages), at least kSkipMin long and wholly below
// `limit`.  The window D2H / H2D skips them -- they never cross PCIe -- and
// the host threads write those pages' frames as well as their content.
// Shorter runs travel as the pack's zeros and are overwritten after landing.
constexpr uint64_t kSkipMin = 256ull << 10;

void plan_host_runs(ImagePlan& P, uint64_t limit) {
  P.host_runs.clear();
  const size_t n = P.host_pages.size();
  for (size_t i = 0; i < n;) {
    const uint64_t lo = P.host_pages[i].stream_off - 16;
    uint64_t hi = P.host_pages[i].stream_off + P.host_pages[i].len;
    size_t j = i + 1;
    while (j < n && P.host_pages[j].stream_off - 16 == hi) {
      hi = P.host_pages[j].stream_off + P.host_pages[j].len;
      ++j;
    }
    const bool skip = hi - lo >= kSkipMin && hi <= limit;
    if (skip) P.host_runs.emplace_back(lo, hi);
    for (size_t k = i; k < j; ++k) P.host_pages[k].own_frame = skip;
    i = j;
  }
  // pinned-host payloads: content moved by host threads (pinned_runs), the
  // frame stays in the window stream
  P.pinned_runs.clear();
  P.pinned_chunks = 0;
  for (size_t k = 0; k < P.pay_spans.size(); ++k) {
    if (P.pay_kind[k] != uint8_t(AllocationKind::PinnedHost)) continue;
    const uint64_t lo = P.pay_rec_off[k], hi = lo + P.pay_spans[k].len;
    if (hi - lo < kSkipMin || hi > limit) continue;
    P.pinned_runs.push_back(ImagePlan::PinnedRun{lo, hi, P.pay_spans[k].ptr, k, P.pinned_chunks});
    P.pinned_chunks += P.pay_first[k + 1] - P.pay_first[k];
    P.recs[k].ptr = 0;  // pack emits zeros / scatter skips: host-filled content
  }
  if (!P.pinned_runs.empty()) {
    std::vector<std::pair<uint64_t, uint64_t>> runs;
    runs.reserve(P.pinned_runs.size() + P.host_runs.size());
    for (const auto& r : P.pinned_runs) runs.emplace_back(r.lo, r.hi);
    runs.insert(runs.end(), P.host_runs.begin(), P.host_runs.end());  // UVM part: after
    P.host_runs = std::move(runs);
  }
  P.direct_runs.clear();
  P.skip_runs = P.host_runs;
}

// The second dirty-key lane of one chunk on the host: Key2 of kernels.cu
// (16-byte word j = lane j % 32 of row j / 32; a partial last word
// zero-padded; the same 64-bit finalizer).
uint32_t chunk_key_host(const uint8_t* p, uint32_t len) {
  uint64_t sum = 0;
  for (uint32_t j = 0; 16ull * j < len; ++j) {
    uint32_t w[4] = {0, 0, 0, 0};
    std::memcpy(w, p + 16ull * j, std::min<uint64_t>(16, len - 16ull * j));
    const uint32_t k = ((j & 31u) + 1) * 0x27D4EB2Fu + (j >> 5) * 0x9E3779B9u;
    sum += uint64_t(w[0] + k) * (w[1] + 0x85EBCA6Bu) +
           uint64_t(w[2] + (k ^ 0xC2B2AE35u)) * (w[3] + 0x165667B1u);
  }
  uint64_t x = sum ^ (uint64_t(len) * 0x9E3779B97F4A7C15ull);
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return uint32_t(x) ^ uint32_t(x >> 32);
}

// Host threads move the pinned-host payload contents: allocation -> image
// (drain) or image -> allocation (refill), in 64 KiB-chunk-aligned 4 MiB
// pieces, and hash what they moved: every chunk's CRC (and, draining, its
// dirty key) into h_pin_crc / h_pin_key, so no SM reads host memory for them.
// CRAC_HOST_NT=1: the drain's host threads hash and copy host-run pages and
// pinned payloads in one read, streaming them into the image with
// non-temporal stores (crc32_copy_stream).  Off by default: neutral on one
// box, ~4 % slower C3 checkpoints on another (profiles/r02/host_nt.txt).
bool host_nt_copy() {
  static const bool on = [] {
    const char* e = std::getenv("CRAC_HOST_NT");
    return e && e[0] == '1';
  }();
  return on;
}

void copy_pinned_runs(DrainEngine& E, const ImagePlan& P, uint8_t* stream, bool drain) {
  if (P.pinned_runs.empty()) return;
  constexpr uint64_t kPiece = 4ull << 20;  // a multiple of the 64 KiB chunk
  static_assert(kPiece % DrainEngine::kChunk == 0);
  E.h_pin_crc.ensure(P.pinned_chunks);
  E.h_pin_key.ensure(P.pinned_chunks);
  std::vector<std::pair<size_t, uint64_t>> pieces;  // (run, offset in run)
  for (size_t r = 0; r < P.pinned_runs.size(); ++r)
    for (uint64_t o = 0; o < P.pinned_runs[r].hi - P.pinned_runs[r].lo; o += kPiece)
      pieces.emplace_back(r, o);
  parallel_for(pieces.size(), [&](uint64_t i) {
    const auto& run = P.pinned_runs[pieces[i].first];
    const uint64_t o = pieces[i].second, n = std::min(kPiece, run.hi - run.lo - o);
    uint8_t* host = reinterpret_cast<uint8_t*>(run.host) + o;
    uint8_t* img = stream + run.lo + o;
    const bool nt = drain && host_nt_copy();
    if (drain && !nt) std::memcpy(img, host, n);
    if (!drain) std::memcpy(host, img, n);
    for (uint64_t c = 0; c < n; c += DrainEngine::kChunk) {
      const uint32_t len = uint32_t(std::min<uint64_t>(DrainEngine::kChunk, n - c));
      const uint64_t slot = run.pin0 + (o + c) / DrainEngine::kChunk;
      // (nt: each chunk read once, hashed and streamed into the image)
      E.h_pin_crc.ptr[slot] = nt ? crc32_copy_stream(img + c, host + c, len) : crc32_fast(host + c, len);
      if (drain) E.h_pin_key.ptr[slot] = chunk_key_host(host + c, len);
    }
    if (nt) stream_fence();
  }, /*min_parallel=*/2);
}

// Uploads the host-computed chunk CRCs (and keys) of the pinned runs into the
// payload chunk tables, on `st` (before the fold that reads them).
void upload_pinned_hashes(DrainEngine& E, const ImagePlan& P, bool keys, cudaStream_t st) {
  for (const auto& run : P.pinned_runs) {
    const uint64_t c0 = P.pay_first[run.pay], n = P.pay_first[run.pay + 1] - c0;
    check_cuda(cudaMemcpyAsync(E.d_pay_crc.ptr + c0, E.h_pin_crc.ptr + run.pin0, n * 4,
                               cudaMemcpyHostToDevice, st),
               "pinned crcs");
    if (keys)
      check_cuda(cudaMemcpyAsync(E.d_pay_key.ptr + c0, E.h_pin_key.ptr + run.pin0, n * 4,
                                 cudaMemcpyHostToDevice, st),
                 "pinned keys");
  }
}

// K1 over payload chunks [c_lo, c_hi) minus the chunks of the pinned runs
// (hashed by the host threads that move them).
void hash_payloads_skip_pinned(DrainEngine& E, const ImagePlan& P, uint64_t c_lo, uint64_t c_hi,
                               uint32_t max_ctas, cudaStream_t st, bool with_key) {
  uint64_t at = c_lo;
  for (const auto& run : P.pinned_runs) {
    const uint64_t r0 = P.pay_first[run.pay], r1 = P.pay_first[run.pay + 1];
    if (r1 <= at || r0 >= c_hi) continue;
    if (r0 > at) hash_payloads(E, P, at, r0, max_ctas, st, with_key);
    at = std::max(at, r1);
  }
  if (at < c_hi) hash_payloads(E, P, at, c_hi, max_ctas, st, with_key);
}

// Whether the stream range [g0, g1) (a kernel range, outside every direct
// run) holds any byte the scatter writes: content of a record with a device
// destination (frames and host-filled content need no kernel).  `rec` walks
// P.recs forward across calls (ranges ascend).
bool range_needs_scatter(const ImagePlan& P, size_t& rec, uint64_t g0, uint64_t g1) {
  const auto& R = P.recs;
  while (rec < R.size() && R[rec].out_off + R[rec].frame_len + R[rec].len <= g0) ++rec;
  for (size_t r = rec; r < R.size() && R[r].out_off < g1; ++r) {
    const uint64_t c0 = R[r].out_off + R[r].frame_len, c1 = c0 + R[r].len;
    if (R[r].ptr && R[r].len && c0 < g1 && c1 > g0) return true;
  }
  return false;
}

// Direct runs: the interior of every Device payload of at least
// kDirectMinTiles + 2 tiles, cut to whole stream tiles 64 bytes clear of the
// payload's ends, wholly below `limit`.  The copy engines move them straight
// between the allocation and the image (a D2H from a misaligned device
// address into a 4 KiB-aligned host address runs at full PCIe speed,
// profiles/r01d/direct_copy2.txt); the pack / scatter kernels only handle
// the tiles around them (frames, payload edges, small payloads, pages).
// Host runs and direct runs are disjoint (UVM_PAGES vs ALLOC_PAYLOADS).
constexpr uint64_t kTile = CRAC_TILE_BYTES;
constexpr uint64_t kDirectMinTiles = 4;

void plan_direct_runs(ImagePlan& P, uint64_t limit, bool drain, uint64_t from = 0) {
  P.direct_runs.clear();
  struct Exact {
    size_t k;
    uint64_t a, len;  // the payload's content [a, a + len) in the stream
  };
  std::vector<Exact> exact;  // per direct run (refill)
  // CRAC_DIRECT = 0 | drain | refill | both (default).  Measured on C4: the
  // refill gains with direct H2D (55.0 against 54.3 GB/s through the ring,
  // round 1); the drain's direct D2H runs at the ring's speed (checkpoint
  // 2281-2287 ms either way, profiles/r02/direct_drain.txt; round 1 measured
  // it 2 % slower) and halves the drain's HBM traffic (no pack read + write
  // of the payloads), so both use them.
  static const int enabled = [] {
    const char* e = std::getenv("CRAC_DIRECT");
    if (!e) return 3;
    if (!std::strcmp(e, "0")) return 0;
    if (!std::strcmp(e, "drain")) return 1;
    if (!std::strcmp(e, "refill")) return 2;
    return 3;
  }();
  if (enabled & (drain ? 1 : 2))
    for (size_t k = 0; k < P.pay_spans.size(); ++k) {
      if (P.pay_kind[k] != uint8_t(AllocationKind::Device)) continue;
      const uint64_t a = P.pay_rec_off[k], len = P.pay_spans[k].len,
                     b = std::min(a + len, limit);
      if (b < a + 64 + (kDirectMinTiles + 2) * kTile) continue;
      uint64_t lo = std::max(from, (a + 64 + kTile - 1) / kTile * kTile),
               hi = (b - 64) / kTile * kTile;
      if (hi < lo + kDirectMinTiles * kTile) continue;
      P.direct_runs.push_back(ImagePlan::DirectRun{lo, hi, P.pay_spans[k].ptr + (lo - a), false});
      if (!drain) exact.push_back({k, a, len});
    }
  static const bool exact_runs = [] {
    const char* e = std::getenv("CRAC_EXACT_DIRECT");
    return !(e && e[0] == '0');
  }();
  if (!drain && exact_runs && !P.direct_runs.empty()) {
    // Refill: a run may reach its payload's exact head, and its exact end when
    // the extent has no padding (the scatter zero-fills padding), wherever the
    // stream between it and its neighbour holds nothing the scatter writes
    // (only frames): then no scatter is launched there at all (C4: the
    // windows of big payloads need none).  Gaps the scatter does handle keep
    // tile-aligned boundaries (the scatter's window offsets are tile-aligned).
    auto& D = P.direct_runs;
    for (size_t i = 0; i < D.size(); ++i)  // heads: the gap before ends at a frame
      if (exact[i].a >= from) {
        D[i].dev -= D[i].lo - exact[i].a;
        D[i].lo = exact[i].a;
      }
    size_t rec = 0;
    for (size_t i = 0; i < D.size(); ++i) {  // ends: only before a frame-only gap
      const uint64_t end = exact[i].a + exact[i].len;
      if (round_up_align(exact[i].len) != exact[i].len || end > limit) continue;
      const uint64_t next = i + 1 < D.size() ? D[i + 1].lo : P.stream_len;
      if (end <= next && !range_needs_scatter(P, rec, end, next)) {
        D[i].hi = end;
        D[i].exact_end = true;
      }
    }
  }
  P.skip_runs.clear();
  P.skip_runs.reserve(P.host_runs.size() + P.direct_runs.size());
  for (const auto& d : P.direct_runs) P.skip_runs.emplace_back(d.lo, d.hi);
  P.skip_runs.insert(P.skip_runs.end(), P.host_runs.begin(), P.host_runs.end());
  std::sort(P.skip_runs.begin(), P.skip_runs.end());
}

uint64_t direct_run_bytes(const ImagePlan& P) {
  uint64_t b = 0;
  for (const auto& d : P.direct_runs) b += d.hi - d.lo;
  return b;
}

// The kernel (pack / scatter) ranges of window [off, end): the window minus
// its direct runs, each starting on a tile boundary.  `run` walks
// P.direct_runs across calls.
void kernel_ranges(const ImagePlan& P, size_t& run, uint64_t off, uint64_t end,
                   std::vector<std::pair<uint64_t, uint64_t>>& out) {
  out.clear();
  const auto& D = P.direct_runs;
  for (uint64_t a = off; a < end;) {
    while (run < D.size() && D[run].hi <= a) ++run;
    uint64_t b = end;
    if (run < D.size() && D[run].lo < end) {
      if (D[run].lo <= a) {
        a = std::min(end, D[run].hi);
        continue;
      }
      b = D[run].lo;
    }
    out.emplace_back(a, b);
    a = b;
  }
}

// Enqueues the direct copies of every direct run starting in [off, end).
void copy_direct(const ImagePlan& P, size_t& run, uint64_t off, uint64_t end, uint8_t* stream,
                 bool d2h, cudaStream_t st) {
  static const uint64_t kPiece = [] {  // the copy engine's best piece (direct_copy2.txt)
    const char* e = std::getenv("CRAC_DIRECT_PIECE_MIB");
    return uint64_t(e ? std::max(1, std::atoi(e)) : 64) << 20;
  }();
  const auto& D = P.direct_runs;
  while (run < D.size() && D[run].lo < off) ++run;
  for (; run < D.size() && D[run].lo < end; ++run) {
    const auto& d = D[run];
    // refill: through the end of the destination word straddling `hi` (the
    // scatter writes only words that start outside the run), unless `hi` is
    // the payload's exact end
    const uint64_t hi = d2h || d.exact_end ? d.hi : d.hi + 15;
    for (uint64_t c = d.lo, n = 0; c < hi; c += n) {
      // an exact (unaligned) head goes first on its own, so the big pieces
      // read / write page-aligned image addresses
      n = c % kTile ? std::min(hi, (c / kTile + 1) * kTile) - c : std::min(kPiece, hi - c);
      uint8_t* dev = reinterpret_cast<uint8_t*>(d.dev + (c - d.lo));
      const cudaError_t e = d2h ? cudaMemcpyAsync(stream + c, dev, n, cudaMemcpyDeviceToHost, st)
                                : cudaMemcpyAsync(dev, stream + c, n, cudaMemcpyHostToDevice, st);
      if (e != cudaSuccess)
        check_cuda(e, (std::string(d2h ? "D2H direct" : "H2D direct") + " [" + std::to_string(d.lo) +
                       ", " + std::to_string(d.hi) + ") piece " + std::to_string(c) + "+" +
                       std::to_string(n) + " dev " + std::to_string(uint64_t(dev)))
                          .c_str());
    }
  }
}

uint64_t host_run_bytes(const ImagePlan& P) {
  uint64_t b = 0;
  for (const auto& r : P.host_runs) b += r.second - r.first;
  return b;
}

// Enqueues the copy of stream bytes [off, end) between a window buffer
// (`buf` holds stream offset `off`) and the image stream, minus the host runs,
// in pieces of at most kCopyChunk.  `run` walks P.host_runs across calls.
uint64_t copy_window(const ImagePlan& P, size_t& run, uint64_t off, uint64_t end, uint8_t* buf,
                     uint8_t* stream, bool d2h, cudaStream_t st, bool dry = false) {
  uint64_t bytes = 0;
  const auto& R = P.skip_runs;
  // ring window pieces (CRAC_COPY_CHUNK_MIB, default DrainEngine::kCopyChunk)
  static const uint64_t piece = [] {
    const char* e = std::getenv("CRAC_COPY_CHUNK_MIB");
    return e ? uint64_t(std::max(1, std::atoi(e))) << 20 : DrainEngine::kCopyChunk;
  }();
  // one cudaMemcpyAsync per piece (host runs cut C3 windows into ~32 pieces)
  const cudaMemcpyKind kind = d2h ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
  for (uint64_t a = off; a < end;) {
    while (run < R.size() && R[run].second <= a) ++run;
    uint64_t b = end;
    if (run < R.size() && R[run].first < end) {
      if (R[run].first <= a) {
        a = std::min(end, R[run].second);
        continue;
      }
      b = R[run].first;
    }
    // H2D: 16 bytes past a gap that a skip run ends, for the scatter's
    // straddling last word (ring bytes under a skip run are never read else)
    const uint64_t bc = d2h ? b : std::min(end, b + 16);
    bytes += b - a;
    for (uint64_t c = a; c < bc && !dry; c += piece) {
      const uint64_t n = std::min(piece, bc - c);
      void* dst = d2h ? static_cast<void*>(stream + c) : static_cast<void*>(buf + (c - off));
      const void* src = d2h ? static_cast<const void*>(buf + (c - off))
                            : static_cast<const void*>(stream + c);
      check_cuda(cudaMemcpyAsync(dst, src, n, kind, st), d2h ? "D2H" : "H2D");
    }
    a = b;
  }
  return bytes;
}

// Host-resident managed pages of a drain.  Each host thread takes a block of
// pages in stream order, hashes every page (zlib CRC, into h_host_crc) and,
// for pages of the ring part [0, head), copies it into the image once the
// D2H of the window holding its last byte has landed (the windows carry
// zeros there; windows land in order on s_copy).  The CPU reads pages that
// live on its side: nothing migrates and no device mapping is needed.
void host_pages_drain(DrainEngine& E, const ImagePlan& P, uint8_t* stream, uint64_t head,
                      const std::atomic<int64_t>& recorded) {
  const uint64_t n = P.host_pages.size();
  if (!n) return;
  // short-run pages of the shadow part: stashed now (the app may change them
  // once it resumes), written after the shadow D2H (drain_finish)
  DrainEngine::Pending& Q = E.pending;
  Q.stash_at.clear();
  std::vector<uint64_t> stash_of(n, ~0ull);
  uint64_t stash_bytes = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const HostPage& h = P.host_pages[i];
    if (!h.own_frame && h.stream_off + h.len > head) {
      stash_of[i] = stash_bytes;
      Q.stash_at.emplace_back(h.stream_off, h.len);
      stash_bytes += h.len;
    }
  }
  Q.stash.resize(stash_bytes);
  E.h_host_crc.ensure(n);
  uint32_t* crc = E.h_host_crc.ptr;
  constexpr uint64_t W = DrainEngine::kWindow;
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const bool nt_copy = host_nt_copy();
  std::atomic<uint64_t> next{0};
  std::atomic<int> failed{0};
  auto worker = [&] {
    int64_t landed = -1;
    for (uint64_t b; (b = next.fetch_add(512)) < n;)
      for (uint64_t i = b; i < std::min(n, b + 512); ++i) {
        const HostPage& h = P.host_pages[i];
        const auto* src = reinterpret_cast<const uint8_t*>(h.ptr);
        if (h.own_frame) {  // in a host run: no window copy touches these bytes
          std::memcpy(stream + h.stream_off - 16, P.recs[h.rec].frame, 16);
          if (nt_copy) {  // one read of the page, streamed into the image
            crc[i] = crc32_copy_stream(stream + h.stream_off, src, h.len);
          } else {
            crc[i] = crc32_fast(src, h.len);
            std::memcpy(stream + h.stream_off, src, h.len);
          }
          continue;
        }
        crc[i] = crc32_fast(src, h.len);
        if (stash_of[i] != ~0ull) {
          std::memcpy(Q.stash.data() + stash_of[i], src, h.len);
          continue;
        }
        const int64_t w = int64_t((h.stream_off + h.len - 1) / W);
        if (w > landed) {
          // the window loop runs beside this pass: an event not yet recorded
          // would read as complete
          while (recorded.load(std::memory_order_acquire) < w) std::this_thread::yield();
          if (cudaEventSynchronize(E.ev_land[w]) != cudaSuccess) failed = 1;
          landed = w;
        }
        std::memcpy(stream + h.stream_off, src, h.len);
      }
    if (nt_copy) stream_fence();  // the streamed image bytes are visible before the join
  };
  std::vector<std::thread> pool;
  for (unsigned t = 1; t < hw; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  if (failed) raise(Errc::DeviceFault, "D2H window failed under a host-page copy");
}

// Host-resident managed pages of a refill: image -> managed memory, then the
// CRC of what landed (zero tail up to ext).
void host_pages_refill(DrainEngine& E, const ImagePlan& P, const uint8_t* stream) {
  const uint64_t n = P.host_pages.size();
  if (!n) return;
  E.h_host_crc.ensure(n);
  uint32_t* crc = E.h_host_crc.ptr;
  parallel_for(n, [&](uint64_t i) {
    const HostPage& h = P.host_pages[i];
    uint8_t* dst = reinterpret_cast<uint8_t*>(h.ptr);
    std::memcpy(dst, stream + h.stream_off, h.len);
    if (h.ext > h.len) std::memset(dst + h.len, 0, h.ext - h.len);
    crc[i] = crc32_fast(dst, h.len);
  });
}

template <typename T>
void put_at(uint8_t* p, T v) {
  std::memcpy(p, &v, sizeof(T));
}

// Writes one complete small section (header, payload, crc) at `p`.
uint64_t write_section(uint8_t* p, uint32_t tag, const std::vector<uint8_t>& payload) {
  put_at<uint32_t>(p, tag);
  put_at<uint32_t>(p + 4, 0);
  put_at<uint64_t>(p + 8, payload.size());
  if (!payload.empty()) std::memcpy(p + 16, payload.data(), payload.size());
  put_at<uint32_t>(p + 16 + payload.size(), crc32_host(payload.data(), payload.size()));
  return 20 + payload.size();
}

struct QuiesceScope {
  DispatchTable& t;
  QuiesceScope(DispatchTable& table, std::chrono::milliseconds to) : t(table) { t.quiesce(to); }
  ~QuiesceScope() { t.resume(); }
};

std::vector<BulkItem> live_items(DeviceContext& ctx, const std::vector<AllocationRecord>& active,
                                 std::vector<std::vector<uint8_t>>& flags, bool with_flags) {
  std::vector<BulkItem> items;
  flags.clear();
  flags.reserve(active.size());
  items.reserve(active.size());
  std::vector<uint64_t> ptrs;
  if (!ctx.match_records(active, ptrs))
    raise(Errc::InvalidArgument, "the log's active set does not match the live allocations");
  for (size_t k = 0; k < active.size(); ++k) {
    const AllocationRecord& rec = active[k];
    BulkItem it{rec.id, rec.kind, rec.size, ptrs[k], nullptr};
    if (with_flags && rec.kind == AllocationKind::Managed) {
      const auto pages = ctx.managed_pages(rec.id);
      std::vector<uint8_t> f(pages.size());
      for (size_t i = 0; i < pages.size(); ++i)
        f[i] = uint8_t((pages[i].device_resident ? 1 : 0) | (pages[i].dirty ? 2 : 0));
      flags.push_back(std::move(f));
      it.flags = &flags.back();
    }
    items.push_back(it);
  }
  return items;
}

// The bulk items of a drain straight from the live table (id order, their
// records in `recs`), with managed page flags; drain_locked checks the
// records against the log's active set.
std::vector<BulkItem> table_items(DeviceContext& ctx, std::vector<AllocationRecord>& recs,
                                  std::vector<std::vector<uint8_t>>& flags) {
  thread_local std::vector<uint64_t> ptrs;
  if (!ctx.live_backed(recs, ptrs))
    raise(Errc::InvalidArgument, "the log's active set does not match the live allocations");
  std::vector<BulkItem> items(recs.size());
  size_t n_managed = 0;
  for (const auto& r : recs) n_managed += r.kind == AllocationKind::Managed;
  flags.clear();
  flags.reserve(n_managed);
  for (size_t k = 0; k < recs.size(); ++k) {
    const AllocationRecord& rec = recs[k];
    items[k] = BulkItem{rec.id, rec.kind, rec.size, ptrs[k], nullptr};
    if (rec.kind == AllocationKind::Managed) {
      const auto pages = ctx.managed_pages(rec.id);
      std::vector<uint8_t> f(pages.size());
      for (size_t i = 0; i < pages.size(); ++i)
        f[i] = uint8_t((pages[i].device_resident ? 1 : 0) | (pages[i].dirty ? 2 : 0));
      flags.push_back(std::move(f));
      items[k].flags = &flags.back();
    }
  }
  return items;
}

uint64_t tail_bytes(Session& session) {
  DeviceContext& ctx = session.device();
  return (20 + 8 * ctx.live_stream_ids().size()) + (20 + session.app_state().size()) +
         (20 + registry_bytes(ctx.registered_binaries()).size());
}

}  // namespace

// ---------------------------------------------------------------------------
// drain
// ---------------------------------------------------------------------------
namespace {

// Everything of a full drain that needs the app stopped: the plan, K1 + K4
// over the live state, the ring windows [0, head) drained to the image and
// the shadow windows [head, stream_len) packed into HBM.  Returns with every
// kernel that reads app memory complete; the shadow D2H (if any) is enqueued
// on s_copy and finished by drain_finish.  Runs with the gate held.
void drain_locked(Session& session, PinnedImage& out, bool use_shadow, DrainStats* stats) {
  PhaseTrace tr("drain");
  DeviceContext& ctx = session.device();
  DrainEngine& E = session.drain_engine();
  if (stats) *stats = DrainStats{};
  check_cuda(cudaEventRecord(E.ev_t0, E.s_pack), "event");

  const SnapshotMeta meta{ctx.seed(), ctx.arena_bytes(), kEngineVersion};
  // the gate is held: the log cannot move, read it in place
  const std::span<const CallLogEntry> log = session.log().quiesced_view();
  tr.mark("log-snapshot");
  // The log side runs on a helper thread beside the plan: the active set of
  // the log (the reference's definition of what the image holds, checked
  // below against the live table the bulk items come from), then, once the
  // image exists, the LOG section encoded into it with its CRC.  Neither is
  // needed before the first D2H (C2: ~0.6 ms off the drain's critical path).
  std::atomic<int> log_stage{0};  // 1: active set ready, 2: image ready, 3: LOG written
  uint8_t* log_dst = nullptr;
  std::exception_ptr log_err;
  std::thread log_side([&] {
    try {
      active_set_into(log, E.scratch_active, E.scratch_alive);
      log_stage.store(1, std::memory_order_release);
      while (log_stage.load(std::memory_order_acquire) < 2) std::this_thread::yield();
      if (log_dst) {
        const uint64_t n = log.size() * kLogRecordBytes;
        encode_log_into(log_dst + 16, log);
        put_at<uint32_t>(log_dst + 16 + n, crc32_host(log_dst + 16, n));
      }
    } catch (...) {
      log_err = std::current_exception();
    }
    log_stage.store(3, std::memory_order_release);
  });
  struct LogJoin {
    std::thread& t;
    std::atomic<int>& st;
    ~LogJoin() {
      if (st.load() < 2) st.store(2);  // unblock on an early exit
      if (t.joinable()) t.join();
    }
  } log_join{log_side, log_stage};
  const std::vector<uint8_t> sec1 = meta_bytes(meta);
  const uint64_t sec2_len = log.size() * kLogRecordBytes;
  const std::vector<uint8_t> sec5 = streams_bytes(ctx.live_stream_ids());
  const std::vector<uint8_t>& sec6 = session.app_state();
  const std::vector<uint8_t> sec7 = registry_bytes(ctx.registered_binaries());
  tr.mark("sections");

  std::vector<std::vector<uint8_t>> flags;
  ImagePlan& P = E.plan;
  thread_local std::vector<AllocationRecord> table;
  std::vector<BulkItem> items = table_items(ctx, table, flags);
  tr.mark("live-items");
  build_plan(items, P);
  P.log_len = log.size();
  tr.mark("plan");
  // the log's active set must be exactly the live table (what live_items
  // used to check record by record), before any device work is queued
  while (log_stage.load(std::memory_order_acquire) < 1) std::this_thread::yield();
  if (log_err) std::rethrow_exception(log_err);
  {
    const std::vector<AllocationRecord>& active = E.scratch_active;
    bool same = active.size() == table.size();
    for (size_t k = 0; same && k < table.size(); ++k)
      same = active[k].id == table[k].id && active[k].kind == table[k].kind &&
             active[k].size == table[k].size && active[k].address == table[k].address;
    if (!same) raise(Errc::InvalidArgument, "the log's active set does not match the live allocations");
  }
  tr.mark("active-set-check");

  // file layout: header | META | LOG | ALLOC hdr | stream | crc4 | STREAMS | APPSTATE | REGISTRY
  const uint64_t s3 = 16 + (20 + sec1.size()) + (20 + sec2_len) + 16;
  const uint64_t total = s3 + P.stream_len + 4 + (20 + sec5.size()) + (20 + sec6.size()) +
                         (20 + sec7.size());
  out.prepare(total, s3);
  tr.mark("image-alloc");
  P.s3 = s3;
  P.image_bytes = total;
  uint8_t* img = out.mutable_data();
  std::memcpy(img, kImageMagic, 8);
  put_at<uint32_t>(img + 8, kImageVersion);
  put_at<uint32_t>(img + 12, kSectionCount);
  uint64_t at = 16;
  at += write_section(img + at, 1, sec1);
  {  // LOG: header here, records + CRC by the log-side thread
    put_at<uint32_t>(img + at, 2);
    put_at<uint32_t>(img + at + 4, 0);
    put_at<uint64_t>(img + at + 8, sec2_len);
    log_dst = img + at;
    log_stage.store(2, std::memory_order_release);
    at += 20 + sec2_len;
  }
  put_at<uint32_t>(img + at, 3);
  put_at<uint32_t>(img + at + 4, 0);
  put_at<uint64_t>(img + at + 8, P.len3);
  // the tail lies past the stream: no D2H touches it
  at = s3 + P.stream_len + 4;
  at += write_section(img + at, 5, sec5);
  at += write_section(img + at, 6, sec6);
  at += write_section(img + at, 7, sec7);
  if (at != total) raise(Errc::DeviceFault, "image layout mismatch");
  P.tail_bytes = (20 + sec5.size()) + (20 + sec6.size()) + (20 + sec7.size());

  DrainEngine::Pending& Q = E.pending;
  Q = DrainEngine::Pending{};
  Q.out = &out;
  const bool bulk = P.len3 + P.len4 > 0;
  if (!bulk) {
    // no bulk bytes: the stream is just crc3 (0) and the UVM_PAGES header
    put_at<uint32_t>(img + s3, 0);
    put_at<uint32_t>(img + s3 + 4, 4);
    put_at<uint32_t>(img + s3 + 8, 0);
    put_at<uint64_t>(img + s3 + 12, 0);
    log_side.join();
    if (log_err) std::rethrow_exception(log_err);
    Q.active = true;
    check_cuda(cudaEventRecord(E.ev_s1, E.s_pack), "event");
    return;
  }

  // split: ring windows [0, head) during the stall, shadow [head, end) after
  constexpr uint64_t W = DrainEngine::kWindow;
  uint64_t head = P.stream_len;
  if (use_shadow && E.shadow_cap) {
    const uint64_t want = P.stream_len > E.shadow_cap ? P.stream_len - E.shadow_cap : 0;
    head = std::min(P.stream_len, (want + W - 1) / W * W);
  }
  Q.head = head;
  // host-resident pages reaching into the shadow part are read by the pack
  // kernels over the link (the app may touch them once it resumes); pages
  // wholly in the ring part are copied by host threads after their D2H.
  // Either way their CRCs come from the host threads.
  // host-resident pages never go through the SMs (no device mapping of them
  // is needed, nothing migrates): long runs are skipped by every window copy,
  // ring and shadow alike, and written by host threads during the stall
  plan_host_runs(P, P.stream_len);
  plan_direct_runs(P, head, true);  // only where the app stays stopped until they land

  const uint64_t windows = (head + W - 1) / W;
  Q.windows = windows;
  Q.timed = stats != nullptr;
  if (stats) E.ensure_window_events(windows);
  // a streamed file write follows the windows as they land (the image is
  // final there except for what the host writes after the stream: the
  // leading sections, crc3 inside the stream, crc4 and the tail)
  LandSink* const sink = (t_land_sink && head == P.stream_len && P.host_pages.empty() &&
                          P.pinned_runs.empty() && windows)
                             ? t_land_sink
                             : nullptr;
  const bool land_events = !P.host_pages.empty() || sink;
  if (land_events) E.ensure_land_events(windows);
  // host-resident pages: hashed (all) and copied by host threads from now
  // on, beside the plan upload, K1 and the window loop (long runs at once;
  // short ring-part runs after their window has landed)
  std::atomic<int64_t> recorded{-1};
  std::exception_ptr host_err;
  std::thread host_pass;
  if (!P.host_pages.empty() || !P.pinned_runs.empty())
    host_pass = std::thread([&] {
      try {
        cudaSetDevice(E.device);  // (its event waits must not touch device 0's context)
        copy_pinned_runs(E, P, img + s3, true);  // before the app resumes (join below)
        host_pages_drain(E, P, img + s3, head, recorded);
      } catch (...) {
        host_err = std::current_exception();
      }
    });
  struct Joiner {
    std::thread& t;
    std::atomic<int64_t>& r;
    ~Joiner() {
      r.store(INT64_MAX);  // unblock waiters if the loop throws
      if (t.joinable()) t.join();
    }
  } join_host{host_pass, recorded};
  std::atomic<bool> sink_stop{false};
  std::thread sink_pass;
  if (sink) {
    sink->start(img, total);
    sink->rewrite(0, s3);
    sink->rewrite(s3 + P.len3, s3 + P.len3 + 4);
    sink->rewrite(s3 + P.stream_len, total);
    sink_pass = std::thread([&, sink, img, s3, head, windows] {
      cudaSetDevice(E.device);
      for (uint64_t w = 0; w < windows; ++w) {
        while (recorded.load(std::memory_order_acquire) < int64_t(w)) {
          if (sink_stop.load(std::memory_order_relaxed)) return;
          std::this_thread::yield();
        }
        if (sink_stop.load(std::memory_order_relaxed) ||
            cudaEventSynchronize(E.ev_land[w]) != cudaSuccess)
          return;
        sink->landed(s3 + std::min((w + 1) * W, head));
      }
    });
  }
  struct SinkJoiner {  // (declared after join_host: runs first on unwinding)
    std::thread& t;
    std::atomic<bool>& stop;
    ~SinkJoiner() {
      if (t.joinable()) {
        stop.store(true);
        t.join();
      }
    }
  } join_sink{sink_pass, sink_stop};

  // With the whole stream in the shadow, K1 copies every payload chunk to
  // its stream position right after hashing it: one HBM read of the state
  // instead of two; frames and the UVM_PAGES part are written beside it.
  const bool fused = use_shadow && head == 0 && !P.pay_spans.empty();
  tr.mark("host-pass-start");
  upload_plan(E, P, E.s_pack);
  if (fused) upload(E.d_pay_soff, P.pay_rec_off, E.s_pack);
  tr.mark("upload");
  check_cuda(cudaEventRecord(E.ev_ready[0], E.s_pack), "event");
  check_cuda(cudaStreamWaitEvent(E.s_hash, E.ev_ready[0], 0), "wait");
  check_cuda(cudaStreamWaitEvent(E.s_shadow, E.ev_ready[0], 0), "wait");
  // K1 on all but kPackSMs SMs: the pack kernels never queue behind it
  // CRAC_K1_WAVES=n: K1 on every SM in n waves of CTAs (the high-priority
  // pack takes SMs as K1 CTAs retire) instead of all but kPackSMs SMs in one
  // persistent wave.  4 waves: K1 in situ 0.93 of HBM against 0.82-0.85, but
  // the drain 0.5 % slower (profiles/r02/k1_waves.txt): off by default
  static const int k1_waves = [] {
    const char* e = std::getenv("CRAC_K1_WAVES");
    return e ? std::atoi(e) : 0;
  }();
  // When the direct D2H copies carry nearly all of the ring part, the pack
  // only writes frames and payload edges: K1 leaves it kPackSMsDirect SMs
  // (CRAC_K1_SPARE_SMS overrides either count).
  static const int spare_env = [] {
    const char* e = std::getenv("CRAC_K1_SPARE_SMS");
    return e ? std::atoi(e) : -1;
  }();
  const bool mostly_direct = head && direct_run_bytes(P) >= head - head / 32;
  const int spare = spare_env >= 0 ? spare_env
                                   : (mostly_direct ? DrainEngine::kPackSMsDirect : DrainEngine::kPackSMs);
  const uint32_t k1_ctas = k1_waves > 0 ? uint32_t(k1_waves * E.sm_count)
                                        : uint32_t(std::max(1, E.sm_count - spare));
  check_cuda(cudaEventRecord(E.ev_h0, E.s_hash), "event");
  if (fused) {
    const bool aligned = std::all_of(P.pay_rec_off.begin(), P.pay_rec_off.end(),
                                     [](uint64_t o) { return o % 16 == 0; });
    check_cuda(cudaError_t(crac_hash_copy_range(
                   E.d_pay_spans.ptr, E.d_pay_first.ptr, uint32_t(P.pay_spans.size()),
                   DrainEngine::kChunk, 0, P.pay_first.back(), E.d_pay_crc.ptr, E.d_pay_key.ptr,
                   E.d_pay_soff.ptr, E.d_shadow, aligned ? 1 : 0, E.s_hash)),
               "K1 hash+copy");
    check_cuda(cudaError_t(crac_write_frames(E.d_recs.ptr, uint32_t(P.pay_spans.size()),
                                             E.d_shadow, E.s_shadow)),
               "frames");
  } else if (P.pay_first.back()) {
    hash_payloads_skip_pinned(E, P, 0, P.pay_first.back(), k1_ctas, E.s_hash, true);
  }
  // pages: the device-resident runs (the host-resident ones are hashed by
  // the host threads that move them)
  if (P.n_dev_pages) hash_pages(E, P, k1_ctas, E.s_hash);
  check_cuda(cudaEventRecord(E.ev_h1, E.s_hash), "event");
  tr.mark("k1-launch");

  // shadow windows: pack at HBM speed on their own stream, beside the ring
  // (fused: only from the 16-byte word holding crc3 on; the payload bytes
  // that word shares are rewritten with the same values)
  for (uint64_t off = fused ? (P.len3 & ~uint64_t(15)) : head; off < P.stream_len; off += W) {
    const uint64_t len = std::min(W, P.stream_len - off);
    check_cuda(cudaError_t(crac_pack_records(E.d_recs.ptr, uint32_t(P.recs.size()),
                                             E.d_tile_rec.ptr + off / CRAC_TILE_BYTES, off, len,
                                             E.d_shadow + (off - head), E.s_shadow)),
               "pack shadow");
    ++Q.launches;
  }

  check_cuda(cudaEventRecord(E.ev_c0, E.s_pack), "event");
  size_t run_i = 0, krun_i = 0, drun_i = 0;
  std::vector<std::pair<uint64_t, uint64_t>> kr;
  for (uint64_t w = 0; w < windows; ++w) {
    const int slot = int(w % DrainEngine::kSlots);
    uint8_t* buf = E.d_ring + slot * (W + 64);
    const uint64_t off = w * W;
    const uint64_t len = std::min(W, head - off);
    if (w >= uint64_t(DrainEngine::kSlots))
      check_cuda(cudaStreamWaitEvent(E.s_pack, E.ev_free[slot], 0), "wait");
    if (stats) cudaEventRecord(E.ev_w0[w], E.s_pack);
    kernel_ranges(P, krun_i, off, off + len, kr);
    for (const auto& [g0, g1] : kr) {
      check_cuda(cudaError_t(crac_pack_records(E.d_recs.ptr, uint32_t(P.recs.size()),
                                               E.d_tile_rec.ptr + g0 / CRAC_TILE_BYTES, g0, g1 - g0,
                                               buf + (g0 - off), E.s_pack)),
                 "pack");
      Q.packed += g1 - g0;
      ++Q.launches;
      ++Q.ring_launches;
    }
    if (stats) cudaEventRecord(E.ev_w1[w], E.s_pack);
    check_cuda(cudaEventRecord(E.ev_ready[slot], E.s_pack), "event");
    check_cuda(cudaStreamWaitEvent(E.s_copy, E.ev_ready[slot], 0), "wait");
    // the copy engine runs best on 16 MiB pieces; the pack on bigger windows
    copy_window(P, run_i, off, off + len, buf, img + s3, true, E.s_copy);
    copy_direct(P, drun_i, off, off + len, img + s3, true, E.s_copy);
    check_cuda(cudaEventRecord(E.ev_free[slot], E.s_copy), "event");
    if (land_events) check_cuda(cudaEventRecord(E.ev_land[w], E.s_copy), "event");
    recorded.store(int64_t(w), std::memory_order_release);
  }
  tr.mark("enqueue");
  if (host_pass.joinable()) host_pass.join();
  if (sink_pass.joinable()) sink_pass.join();  // every window has landed
  if (host_err) std::rethrow_exception(host_err);
  log_side.join();
  if (log_err) std::rethrow_exception(log_err);
  // (fused: K1 hashed the pinned runs too, in place over the link)
  if (!fused) upload_pinned_hashes(E, P, true, E.s_hash);
  // then K4 folds every CRC
  if (!P.host_pages.empty())
    check_cuda(cudaMemcpyAsync(E.d_page_crc.ptr + P.n_dev_pages, E.h_host_crc.ptr,
                               P.host_pages.size() * 4, cudaMemcpyHostToDevice, E.s_hash),
               "host page crcs");
  enqueue_fold(E, P, E.s_hash);
  tr.mark("host-pages");
  // snapshot complete = K1/K4, the shadow packs and the ring D2H have landed
  check_cuda(cudaEventRecord(E.ev_join[0], E.s_hash), "event");
  check_cuda(cudaEventRecord(E.ev_join[1], E.s_shadow), "event");
  check_cuda(cudaEventRecord(E.ev_join[2], E.s_copy), "event");
  for (cudaEvent_t e : E.ev_join) check_cuda(cudaStreamWaitEvent(E.s_pack, e, 0), "wait");
  check_cuda(cudaEventRecord(E.ev_s1, E.s_pack), "event");
  // the section CRCs are ready long before the D2H finishes
  check_cuda(cudaStreamSynchronize(E.s_hash), "hash sync");
  tr.mark("hash+fold");
  finish_fold(E, P, Q.crc3, Q.crc4);
  // seed the incremental table with this image's payload chunk CRCs
  const uint64_t n_pay = P.pay_first.back();
  if (n_pay) seed_prev_keys(E, n_pay, E.s_hash);
  check_cuda(cudaEventSynchronize(E.ev_s1), "snapshot sync");
  tr.mark("d2h-wait");

  // the app may run from here on: the shadow -> image D2H reads only HBM
  // that belongs to the engine
  if (head < P.stream_len) {
    if (E.shadow_device >= 0) {  // the buddy GPU drains its copy over its own link
      check_cuda(cudaStreamWaitEvent(E.s_peer, E.ev_s1, 0), "wait");
      copy_window(P, run_i, head, P.stream_len, E.d_shadow, img + s3, true, E.s_peer);
      check_cuda(cudaEventRecord(E.ev_peer, E.s_peer), "event");
      check_cuda(cudaStreamWaitEvent(E.s_copy, E.ev_peer, 0), "wait");
    } else {
      copy_window(P, run_i, head, P.stream_len, E.d_shadow, img + s3, true, E.s_copy);
    }
  }
  check_cuda(cudaEventRecord(E.ev_c1, E.s_copy), "event");
  Q.active = true;
}

// Waits for the shadow D2H and completes the image.  No gate needed.
void drain_finish(Session& session, DrainStats* stats) {
  DrainEngine& E = session.drain_engine();
  DrainEngine::Pending& Q = E.pending;
  if (!Q.active) return;
  ImagePlan& P = E.plan;
  uint8_t* img = Q.out->mutable_data();
  check_cuda(cudaStreamWaitEvent(E.s_pack, E.ev_c1, 0), "wait");
  check_cuda(cudaEventRecord(E.ev_t1, E.s_pack), "event");
  check_cuda(cudaEventSynchronize(E.ev_t1), "drain sync");
  uint64_t at = 0;
  for (const auto& [off, len] : Q.stash_at) {
    std::memcpy(img + P.s3 + off, Q.stash.data() + at, len);
    at += len;
  }
  // crc3 lies inside the stream (the windows carried zeros there)
  put_at<uint32_t>(img + P.s3 + P.len3, Q.crc3);
  put_at<uint32_t>(img + P.s3 + P.stream_len, Q.crc4);
  P.valid = true;
  P.image_ptr = reinterpret_cast<uint64_t>(img);
  E.prev_valid = P.pay_first.back() > 0;
  const bool bulk = P.len3 + P.len4 > 0;
  if (stats) {
    *stats = DrainStats{};
    stats->total_ms = elapsed(E.ev_t0, E.ev_t1);
    stats->stall_ms = elapsed(E.ev_t0, E.ev_s1);
    if (bulk) {
      stats->hash_ms = elapsed(E.ev_h0, E.ev_h1);
      stats->copy_ms = elapsed(E.ev_c0, E.ev_c1);
      stats->hash_launches = (P.pay_first.back() ? 1 : 0) + (P.n_dev_pages ? 1 : 0);
      stats->hash_bytes = hashed_bytes(P);
      stats->pack_launches = Q.launches;  // ring + shadow
      stats->pack_bytes = Q.packed + (P.stream_len - Q.head);  // ring windows + shadow
      // per ring launch; a split drain begun without stats (checkpoint_begin)
      // recorded no window events
      stats->pack_ms = Q.timed ? mean_pack_launch_ms(E, Q.windows, Q.ring_launches) : 0.0;
      stats->d2h_bytes = P.stream_len - host_run_bytes(P);
      stats->shadow_bytes = P.stream_len - Q.head;
    }
    stats->image_bytes = P.image_bytes;
    stats->total_chunks = P.pay_first.back() + P.n_dev_pages + P.host_pages.size();
    stats->dirty_chunks = stats->total_chunks;
  }
  Q = DrainEngine::Pending{};
}

void precopy_wait(Session& session, double* phase1_ms);

// The global-checkpoint hook (global_barrier.hpp) of a split drain whose
// image completes in a later call: checkpoint_begin arms it, whichever call
// completes the image (checkpoint_finish or any drain that finishes the
// pending one first) runs the kPhaseImageComplete arrival, so every rank's
// barrier sequence stays quiesced -> image-complete.
void commit_pending(Session& session) {
  if (!session.commit_armed) return;
  session.commit_armed = false;
  session.global_barrier(kPhaseImageComplete);
}

void finish_pending(Session& session) {
  if (!session.has_drain_engine()) return;  // nothing pending; acquired under the gate
  if (session.drain_engine().pending.precopy) {
    precopy_wait(session, nullptr);
    return;
  }
  if (session.drain_engine().pending.active) drain_finish(session, nullptr);
  commit_pending(session);
}

// A full drain; `global` runs the global-checkpoint hook around it (the
// internal fallbacks of the incremental / pre-copy drains pass false when
// their caller already owns the barrier sequence).
void full_drain(Session& session, PinnedImage& out, DrainStats* stats, bool global) {
  finish_pending(session);
  if (global) session.barrier_ms = 0;
  {
    QuiesceScope q(session.table(), session.config().quiesce_timeout);
    if (global) session.global_barrier(kPhaseQuiesced);
    drain_locked(session, out, false, stats);
  }
  drain_finish(session, stats);
  if (global) session.global_barrier(kPhaseImageComplete);
  if (stats) stats->barrier_ms = session.barrier_ms;
}

}  // namespace

void checkpoint_image(Session& session, PinnedImage& out, DrainStats* stats) {
  full_drain(session, out, stats, true);
}

void reserve_shadow(Session& session, uint64_t bytes, int device) {
  finish_pending(session);
  DrainEngine& E = session.drain_engine();
  const int own = E.device;
  if (device < 0) device = own;
  bytes = (bytes + DrainEngine::kWindow - 1) / DrainEngine::kWindow * DrainEngine::kWindow;
  if (bytes == E.shadow_cap && device == (E.shadow_device < 0 ? own : E.shadow_device)) return;
  if (bytes && device != own) {
    int n = 0, can = 0;
    check_cuda(cudaGetDeviceCount(&n), "device count");
    if (device >= n) raise(Errc::InvalidArgument, "reserve_shadow: no device " + std::to_string(device));
    check_cuda(cudaDeviceCanAccessPeer(&can, own, device), "peer query");
    if (!can)
      raise(Errc::InvalidArgument, "reserve_shadow: device " + std::to_string(device) +
                                       " is not reachable from device " + std::to_string(own) +
                                       " by peer access");
    const cudaError_t pe = cudaDeviceEnablePeerAccess(device, 0);
    if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) check_cuda(pe, "peer access");
    cudaGetLastError();
  }
  free_shadow(E);
  if (!bytes) return;
  // +64: the pack of the last window writes whole 16-byte words
  check_cuda(cudaSetDevice(device), "set device");
  cudaError_t e = cudaMalloc(&E.d_shadow, bytes + 64);
  if (e == cudaErrorMemoryAllocation) {
    // a closed session's cached arena may hold the memory (device_core.cu)
    cudaGetLastError();
    drop_arena_cache(device);
    e = cudaMalloc(&E.d_shadow, bytes + 64);
  }
  if (e == cudaSuccess && device != own && !E.s_peer) {
    check_cuda(cudaStreamCreateWithFlags(&E.s_peer, cudaStreamNonBlocking), "peer stream");
    check_cuda(cudaEventCreateWithFlags(&E.ev_peer, cudaEventDisableTiming), "peer event");
  }
  check_cuda(cudaSetDevice(own), "set device");
  if (e != cudaSuccess) {
    cudaGetLastError();
    E.d_shadow = nullptr;
    raise(Errc::OutOfArena, "reserve_shadow: " + std::to_string(bytes) + " bytes of HBM unavailable");
  }
  E.shadow_cap = bytes;
  E.shadow_device = device == own ? -1 : device;
}

void checkpoint_begin(Session& session, PinnedImage& out, DrainStats* stats) {
  finish_pending(session);
  session.barrier_ms = 0;
  QuiesceScope q(session.table(), session.config().quiesce_timeout);
  session.global_barrier(kPhaseQuiesced);
  drain_locked(session, out, true, nullptr);
  DrainEngine& E = session.drain_engine();
  session.commit_armed = true;
  if (stats) {
    *stats = DrainStats{};
    stats->stall_ms = elapsed(E.ev_t0, E.ev_s1);
    stats->shadow_bytes = E.plan.stream_len - E.pending.head;
    stats->barrier_ms = session.barrier_ms;
  }
}

void checkpoint_finish(Session& session, DrainStats* stats) {
  drain_finish(session, stats);
  commit_pending(session);
  if (stats) stats->barrier_ms = session.barrier_ms;
}

void hash_only(Session& session, DrainStats* stats) {
  finish_pending(session);
  QuiesceScope q(session.table(), session.config().quiesce_timeout);
  DeviceContext& ctx = session.device();
  DrainEngine& E = session.drain_engine();
  if (stats) *stats = DrainStats{};
  std::vector<std::vector<uint8_t>> flags;
  ImagePlan P;
  build_plan(live_items(ctx, active_set(session.log().snapshot()), flags, false), P);
  upload_plan(E, P, E.s_hash);
  check_cuda(cudaEventRecord(E.ev_h0, E.s_hash), "event");
  if (P.pay_first.back()) hash_payloads(E, P, 0, P.pay_first.back(), 0, E.s_hash);
  if (P.n_dev_pages) hash_pages(E, P, 0, E.s_hash);
  check_cuda(cudaEventRecord(E.ev_h1, E.s_hash), "event");
  check_cuda(cudaStreamSynchronize(E.s_hash), "hash sync");
  if (stats) {
    stats->hash_ms = stats->total_ms = elapsed(E.ev_h0, E.ev_h1);
    stats->hash_bytes = hashed_bytes(P);
    stats->hash_launches = (P.pay_first.back() ? 1 : 0) + (P.n_dev_pages ? 1 : 0);
    stats->total_chunks = P.pay_first.back() + P.n_dev_pages + P.host_pages.size();
  }
  E.plan.valid = false;  // the device tables now describe this pass, not an image
  E.prev_valid = false;
}

// ---------------------------------------------------------------------------
// refill
// ---------------------------------------------------------------------------
namespace {

// META and the bulk stream's place, read from the first section headers
// without any validation beyond bounds (the early start of restart_image).
struct StreamPeek {
  bool ok = false;
  uint64_t seed = 0, arena_bytes = 0, s3 = 0, stream_len = 0, len4 = 0;
  uint64_t arena_hi = 0;  // end of the highest Device extent in the LOG (2 MiB rounded)
  bool pinned_big = false;
};

StreamPeek peek_stream(std::span<const uint8_t> raw) {
  StreamPeek k;
  auto u64 = [&](uint64_t at, uint64_t& v) {
    if (at > raw.size() || raw.size() - at < 8) return false;
    std::memcpy(&v, raw.data() + at, 8);
    return true;
  };
  uint64_t len1 = 0, len2 = 0, len3 = 0, len4 = 0;
  if (raw.size() < 16 || std::memcmp(raw.data(), kImageMagic, 8) != 0) return k;
  if (!u64(24, len1) || len1 != 24 || !u64(32, k.seed) || !u64(40, k.arena_bytes)) return k;
  uint32_t crc1 = 0;  // META is used before the parse: only with its CRC intact
  if (raw.size() < 60) return k;
  std::memcpy(&crc1, raw.data() + 56, 4);
  if (crc32_host(raw.data() + 32, 24) != crc1) return k;
  const uint64_t h2 = 16 + 20 + len1;
  if (!u64(h2 + 8, len2) || len2 > raw.size() || h2 + 16 + len2 > raw.size()) return k;
  k.s3 = h2 + 20 + len2 + 16;
  if (!u64(k.s3 - 8, len3) || len3 > raw.size() || k.s3 + len3 + 20 > raw.size()) return k;
  if (!u64(k.s3 + len3 + 4 + 8, len4) || len4 > raw.size() - (k.s3 + len3 + 20)) return k;
  k.stream_len = len3 + 20 + len4;
  k.len4 = len4;
  // big pinned-host payloads stay off the link (host threads move them):
  // the early windows would carry them, so such an image goes without
  // (LOG records: seq u64, op u8, kind u8, u16, size u64, id u64, addr u64)
  for (uint64_t at = h2 + 16; at + kLogRecordBytes <= h2 + 16 + len2; at += kLogRecordBytes) {
    const uint8_t op = raw[at + 8], kind = raw[at + 9];
    if (op != uint8_t(LogOp::Alloc)) continue;
    uint64_t size = 0, addr = 0;
    std::memcpy(&size, raw.data() + at + 12, 8);
    std::memcpy(&addr, raw.data() + at + 28, 8);
    if (kind == uint8_t(AllocationKind::PinnedHost) && size >= kSkipMin) k.pinned_big = true;
    // the highest extent any allocation ever took (the cold arena's whole map)
    if (kind == uint8_t(AllocationKind::Device) && addr >= kArenaBase && size < (1ull << 62))
      k.arena_hi = std::max(k.arena_hi, addr - kArenaBase + round_up_align(size));
  }
  k.arena_hi = std::min<uint64_t>(k.arena_bytes, (k.arena_hi + (2ull << 20) - 1) & ~((2ull << 20) - 1));
  // a session must be constructible from META (DeviceContext's own checks)
  k.ok = k.arena_bytes > 0 && k.arena_bytes % kAlign == 0 && k.stream_len > 20;
  return k;
}

}  // namespace

Session restart_image(std::span<const uint8_t> image, const KernelCatalog& catalog, TableMode mode,
                      std::chrono::milliseconds quiesce_timeout, DrainStats* stats) {
  if (stats) *stats = DrainStats{};
  // the refill's time starts here: the host parse and the session set-up
  // before the first device event count (host clock, added to total_ms)
  const auto t_entry = std::chrono::steady_clock::now();
  PhaseTrace tr("refill");
  std::vector<uint8_t> storage;
  const std::span<const uint8_t> raw = unwrap(image, storage, nullptr);
  constexpr uint64_t W = DrainEngine::kWindow;

  // Early start: META and the position of the bulk stream need only the first
  // section headers, so the refill session is set up and the first ring
  // windows' H2D is queued before the full parse and the plan (C2: ~1 ms of
  // host work that used to precede the first copy).  The speculative windows
  // carry every byte of their range; the scatter handles them whole (no
  // direct runs start below them).  Nothing is trusted from the peek: the
  // full parse below decides validity, and an image it refuses unwinds the
  // session after the copies (which only write the engine's ring) complete.
  const StreamPeek pk = peek_stream(raw);
  std::optional<Session> holder;
  SessionConfig cfg;
  cfg.mode = mode;
  cfg.quiesce_timeout = quiesce_timeout;
  uint64_t n_spec = 0;
  double host_pre_ms = 0;  // entry -> the first device event (ev_t0)
  auto open_session = [&](uint64_t seed, uint64_t arena) {
    cfg.seed = seed;
    cfg.arena_bytes = arena;
    holder.emplace(cfg);
    DrainEngine& e = holder->drain_engine();
    check_cuda(cudaEventRecord(e.ev_t0, e.s_pack), "event");
    host_pre_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_entry).count();
  };
  constexpr uint64_t kColdHeadDefault = 8ull << 30;
  // (only without managed pages: the early windows would carry the host
  // runs the H2D otherwise skips, and a UVM refill is not link-bound)
  if (pk.ok && pk.len4 == 0 && !pk.pinned_big) {
    try {
      open_session(pk.seed, pk.arena_bytes);
    } catch (const Error&) {
      holder.reset();  // whatever failed is reported in order, after the parse
    }
  }
  // ... and only into an arena whose map is under way before the parse: the
  // premap from the parsed log behind early windows was slow (C2 cold
  // restart 17.9 ms, r02j; it mapped 16 k extents in many runs, and many
  // small handles cost far more than one, profiles/r02/probe_vmm.txt).  A
  // cold arena is mapped right here,
  // before the parse, up to the highest extent the LOG ever placed (a scan
  // of its records, no parse) when that is at most ~4x the stream; a sparser
  // one keeps the premap from the active set and goes without early windows.
  static const bool cold_fullmap = [] {
    const char* e = std::getenv("CRAC_COLD_FULLMAP");
    return !(e && e[0] == '0');
  }();
  // The cold map runs on a thread while the early windows are queued and the
  // image parsed, for arenas up to 16 GiB (C2: cold restart 11.5-12.8 ->
  // 10.6 ms); a bigger map beside the copies measured ~20 ms slower than
  // before them (C4, profiles/r02/map_beside.txt).  CRAC_MAP_BESIDE=0|1 forces.
  static const int map_beside_env = [] {
    const char* e = std::getenv("CRAC_MAP_BESIDE");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  const bool map_beside = map_beside_env >= 0 ? map_beside_env == 1 : pk.arena_hi <= (16ull << 30);
  // A bigger cold arena is mapped as two handles: its first `head` bytes
  // before the copies, the rest on a thread while the windows bound for the
  // head stream in (the enqueue joins it before the first window whose
  // destinations lie beyond; VMM calls do not wait for copies in flight,
  // profiles/r02/probe_vmm.txt).  CRAC_COLD_HEAD_MIB sets the head (0: one
  // handle, mapped before the copies).
  static const uint64_t cold_head_env = [] {
    const char* e = std::getenv("CRAC_COLD_HEAD_MIB");
    return e ? uint64_t(std::strtoull(e, nullptr, 10)) << 20 : kColdHeadDefault;
  }();
  const uint64_t cold_head = (cold_head_env & ~((2ull << 20) - 1));
  // the first ring windows' H2D, queued before the parse (they land in the
  // engine's ring, not the arena, so they need no mapping)
  auto enqueue_early = [&] {
    DrainEngine& e = holder->drain_engine();
    n_spec = std::min<uint64_t>(DrainEngine::kSlots, (pk.stream_len + W - 1) / W);
    check_cuda(cudaEventRecord(e.ev_c0, e.s_copy), "event");
    for (uint64_t w = 0; w < n_spec; ++w) {
      const uint64_t off = w * W, n = std::min(W + 16, pk.stream_len - off);
      uint8_t* buf = e.d_ring + w * (W + 64);
      for (uint64_t c = 0; c < n; c += DrainEngine::kCopyChunk)
        check_cuda(cudaMemcpyAsync(buf + c, raw.data() + pk.s3 + off + c,
                                   std::min(DrainEngine::kCopyChunk, n - c), cudaMemcpyHostToDevice,
                                   e.s_copy),
                   "H2D (early)");
      check_cuda(cudaEventRecord(e.ev_ready[w], e.s_copy), "event");
    }
  };
  // CRAC_EARLY_FIRST=0: a big cold arena's head is mapped before the early
  // windows are queued (the copy engine idles during that map)
  static const bool early_first = [] {
    const char* e = std::getenv("CRAC_EARLY_FIRST");
    return !(e && e[0] == '0');
  }();
  std::thread map_thread;
  std::exception_ptr map_err;
  bool mapping = false;
  bool deferred_map = false;  // the tail of the arena is being mapped by map_thread
  uint64_t map_head = 0;      // bytes of the arena mapped before the copies when deferred
  if (holder && !holder->device().arena_premapped() && cold_fullmap && pk.arena_hi &&
      pk.arena_hi <= 4 * pk.stream_len + (1ull << 30)) {
    if (map_beside) {
      mapping = true;
      map_thread = std::thread([&, dev = holder->drain_engine().device] {
        try {
          cudaSetDevice(dev);
          holder->device().premap(kArenaBase, pk.arena_hi);
        } catch (...) {
          map_err = std::current_exception();
        }
      });
    } else {
      try {
        const bool split = cold_head && pk.arena_hi >= 2 * cold_head;
        map_head = split ? cold_head : pk.arena_hi;
        if (early_first) enqueue_early();  // the link works while the head maps
        holder->device().premap(kArenaBase, map_head);
        if (split) {
          deferred_map = true;
          map_thread = std::thread([&, dev = holder->drain_engine().device] {
            try {
              cudaSetDevice(dev);
              holder->device().premap(kArenaBase + map_head, pk.arena_hi - map_head);
            } catch (...) {
              map_err = std::current_exception();
            }
          });
        }
      } catch (const Error&) {
        if (n_spec) cudaStreamSynchronize(holder->drain_engine().s_copy);  // early copies in flight
        n_spec = 0;
        holder.reset();  // reported in order after the parse, if at all
      }
    }
    tr.mark("fullmap");
  }
  // joins the deferred tail map; the engine streams drain before an error
  // unwinds the session (the arena they write into is unmapped with it)
  auto join_tail_map = [&] {
    if (!deferred_map) return;
    map_thread.join();
    deferred_map = false;
    tr.mark("tail-map-join");
    if (map_err) {
      cudaStreamSynchronize(holder->drain_engine().s_copy);
      cudaStreamSynchronize(holder->drain_engine().s_pack);
      std::rethrow_exception(map_err);
    }
  };
  struct MapJoin {
    std::thread& t;
    ~MapJoin() {
      if (t.joinable()) t.join();
    }
  } map_join{map_thread};
  if (holder && !mapping && !deferred_map && !holder->device().arena_premapped()) {
    // keep the session; no early windows
  } else if (holder && !n_spec) {
    enqueue_early();
  }
  tr.mark("early");
  ParsedImage p;
  try {
    p = parse_image(raw, /*verify_bulk=*/false);
  } catch (...) {
    if (map_thread.joinable()) map_thread.join();
    if (holder) cudaStreamSynchronize(holder->drain_engine().s_copy);
    throw;
  }
  if (map_thread.joinable() && !deferred_map) {
    map_thread.join();
    tr.mark("map-join");
    if (map_err) {  // reported in order below, if at all
      cudaStreamSynchronize(holder->drain_engine().s_copy);
      holder.reset();
      n_spec = 0;
    }
  }
  tr.mark("parse");
  if (holder && (p.meta.seed != pk.seed || p.meta.arena_bytes != pk.arena_bytes ||
                 p.sec[2].payload_off != pk.s3)) {
    // (cannot happen for an image the parse accepts; kept as a guard)
    if (deferred_map) {
      map_thread.join();
      deferred_map = false;
    }
    cudaStreamSynchronize(holder->drain_engine().s_copy);
    holder.reset();
    n_spec = 0;
  }
  if (!holder) open_session(p.meta.seed, p.meta.arena_bytes);
  Session& session = *holder;
  DeviceContext& ctx = session.device();
  DrainEngine& E = session.drain_engine();
  tr.mark("session");

  std::map<uint64_t, std::vector<KernelDescriptor>> binaries;
  for (const BinaryInfo& b : p.binaries) {
    std::vector<KernelDescriptor> ks;
    for (const KernelInfo& k : b.kernels) {
      auto it = catalog.find(k.name);
      if (it == catalog.end())
        raise(Errc::UnknownKernelBody, "no body registered for kernel '" + k.name + "'");
      ks.push_back(KernelDescriptor{k.name, k.buffer_arity, k.scalar_arity, it->second});
    }
    binaries.emplace(b.handle, std::move(ks));
  }

  // With the arena at its logged VA and only Device allocations live, every
  // destination is the logged address itself: the H2D / scatter / verify
  // pipeline starts before the replay and the replay (host bookkeeping only,
  // the extents are pre-mapped) runs beside it, then vouches for the
  // addresses.  Otherwise the data path waits for the replayed backings.
  const bool early = ctx.fixed_va() && !p.facts.active.empty() &&
                     std::all_of(p.facts.active.begin(), p.facts.active.end(),
                                 [](const AllocationRecord& r) {
                                   return r.kind == AllocationKind::Device;
                                 });
  ImagePlan& P = E.plan;
  const uint64_t s3 = p.sec[2].payload_off;
  auto plan = [&](const std::vector<BulkItem>& items) {
    build_plan(items, P);
    plan_host_runs(P, P.stream_len);
    plan_direct_runs(P, P.stream_len, false, n_spec * W);  // none inside the early windows
    P.log_len = p.log.size();
    if (P.len3 != p.sec[2].length || P.len4 != p.sec[3].length ||
        s3 + P.stream_len != p.sec[3].payload_off + p.sec[3].length)
      raise(Errc::ImageCorrupt, "bulk sections do not match the log's active set");
  };
  // early: the plan (host work only) is built on a thread beside the premap
  // (driver work only); the data path is enqueued once both are done
  std::vector<BulkItem> early_items;
  std::exception_ptr plan_err;
  std::thread early_plan;
  struct PlanJoiner {
    std::thread& t;
    ~PlanJoiner() {
      if (t.joinable()) t.join();
    }
  } plan_joiner{early_plan};
  if (early) {
    early_items.reserve(p.facts.active.size());
    for (const AllocationRecord& rec : p.facts.active)
      early_items.push_back(BulkItem{rec.id, rec.kind, rec.size, rec.address, nullptr});
    early_plan = std::thread([&, dev = E.device] {
      try {
        cudaSetDevice(dev);  // the record table may grow (pinned)
        plan(early_items);
      } catch (...) {
        plan_err = std::current_exception();
      }
    });
  }

  std::vector<uint64_t> live;
  live.reserve(p.facts.active.size());
  // map every live Device extent up front in coalesced runs, so the replay
  // itself makes no driver calls (and the early data path below has its
  // destinations).  The runs come from a bitmap of the 2 MiB blocks the
  // extents touch, in address order (first fit hands out low addresses
  // again after frees, so id order is not address order), without
  // sorting the extents (C2: 16 k); one-block gaps are bridged.  Mapping in
  // 1 GiB pieces interleaved with the windows' H2D was measured slower (C4
  // cold restart 2681 vs 2462 ms, profiles/r02/lazy_premap.txt): 120 handles
  // cost far more than one (profiles/r02/probe_vmm.txt), and the enqueue
  // loop waited on them.
  {
    constexpr uint64_t kBlock = 2ull << 20;
    std::vector<uint8_t> need((cfg.arena_bytes + kBlock - 1) / kBlock, 0);
    for (const AllocationRecord& r : p.facts.active) {
      live.push_back(r.id);
      if (r.kind != AllocationKind::Device) continue;
      const uint64_t off = r.address - kArenaBase;  // parse_log checked it lies in the arena
      // parse_log's arena check is the reference's (image.cpp:133-135), whose
      // round_up_align wraps to 0 for sizes near 2^64; such an extent cannot
      // lie in the arena, and its payload frame cannot exist (the reference
      // rejects the image in decode_payloads/decode_uvm): ImageCorrupt here,
      // before anything is indexed by it
      if (r.size > cfg.arena_bytes - off)
        raise(Errc::ImageCorrupt, "Alloc extent outside arena");
      const uint64_t b1 = (off + round_up_align(r.size) - 1) / kBlock;
      for (uint64_t b = off / kBlock; b <= b1; ++b) need[b] = 1;
    }
    const uint64_t nb = need.size();
    std::vector<std::pair<uint64_t, uint64_t>> runs;  // block ranges
    uint64_t touched = 0;
    for (uint64_t b = 0; b < nb;) {
      if (!need[b]) {
        ++b;
        continue;
      }
      uint64_t e = b + 1;
      while (e < nb && (need[e] || (e + 1 < nb && need[e + 1]))) ++e;
      runs.emplace_back(b, e);
      touched += e - b;
      b = e;
    }
    // a cold arena pays ~3 driver calls per run (create, map, access): many
    // runs over a mostly touched span (C2: 16 k small extents) are mapped as
    // one run instead (the holes get memory too, at most 1/4 of the span)
    static const bool single = [] {
      const char* e = std::getenv("CRAC_PREMAP_SINGLE");
      return !(e && e[0] == '0');
    }();
    // the deferred tail map covers every extent up to pk.arena_hi (the
    // highest the log placed); anything beyond waits for it
    if (deferred_map && !runs.empty() && runs.back().second * kBlock > pk.arena_hi) join_tail_map();
    if (deferred_map) runs.clear();
    if (single && !ctx.arena_premapped() && runs.size() > 8 &&
        4 * touched >= 3 * (runs.back().second - runs.front().first))
      runs = {{runs.front().first, runs.back().second}};
    for (const auto& [b, e] : runs) {
      const uint64_t hi = std::min(e * kBlock, cfg.arena_bytes);
      ctx.premap(kArenaBase + b * kBlock, hi - b * kBlock);
    }
  }
  tr.mark("premap");

  uint64_t windows = 0, verifies = 0, scattered = 0, scatter_launches = 0, ring_skipped = 0;
  // enqueues H2D windows -> scatter -> K1 verify (payloads as their regions
  // complete, then the device-resident pages); nothing here waits
  auto enqueue_data_path = [&] {
    if (P.stream_len <= 20) return;
    upload_plan(E, P, E.s_pack);
    check_cuda(cudaEventRecord(E.ev_join[0], E.s_pack), "event");
    check_cuda(cudaStreamWaitEvent(E.s_copy, E.ev_join[0], 0), "wait");
    windows = (P.stream_len + DrainEngine::kWindow - 1) / DrainEngine::kWindow;
    if (stats) E.ensure_window_events(windows);
    if (!n_spec) check_cuda(cudaEventRecord(E.ev_c0, E.s_copy), "event");
    // while the tail map runs: the stream prefix whose records all land in
    // the mapped head (the first record with arena bytes beyond it ends it)
    uint64_t head_safe_end = ~0ull;
    if (deferred_map) {
      const uint64_t lo = kArenaBase, hi = kArenaBase + cfg.arena_bytes;
      for (const crac_record_t& r : P.recs)
        if (r.ptr >= lo && r.ptr < hi && r.ptr + std::max(r.len, r.ext) > kArenaBase + map_head) {
          head_safe_end = r.out_off;
          break;
        }
    }
    size_t spans_done = 0, run_i = 0, krun_i = 0, drun_i = 0, srec_i = 0;
    std::vector<std::pair<uint64_t, uint64_t>> kr, scatter_kr;
    // CRAC_RING_SKIP=0: every window's ring part crosses the link, read or not
    static const bool ring_skip = [] {
      const char* e = std::getenv("CRAC_RING_SKIP");
      return !(e && e[0] == '0');
    }();
    constexpr uint64_t kVerifyBatch = 32768;  // 2 GiB of 64 KiB chunks: big enough to keep
                                              // K1 efficient beside the H2D; the tail
                                              // batch after the last window is < 0.5 ms
    // a stream of fewer chunks (C2: 15.8 k small payloads) is verified in
    // `verify_split` batches as its windows land, so only the last one
    // follows the last H2D (CRAC_VERIFY_SPLIT, default 4; 1 = one batch)
    static const uint64_t verify_split = [] {
      const char* e = std::getenv("CRAC_VERIFY_SPLIT");
      return uint64_t(e ? std::max(1, std::atoi(e)) : 4);
    }();
    const uint64_t verify_batch =
        std::min<uint64_t>(kVerifyBatch, std::max<uint64_t>(1024, P.pay_first.back() / verify_split));
    for (uint64_t w = 0; w < windows; ++w) {
      const int slot = int(w % DrainEngine::kSlots);
      uint8_t* buf = E.d_ring + slot * (DrainEngine::kWindow + 64);
      const uint64_t off = w * DrainEngine::kWindow;
      const uint64_t len = std::min(DrainEngine::kWindow, P.stream_len - off);
      const uint64_t with_ahead = std::min(len + 16, P.stream_len - off);
      if (deferred_map && off + with_ahead > head_safe_end) join_tail_map();
      // the window's kernel ranges, and which of them hold device-bound bytes
      kernel_ranges(P, krun_i, off, off + len, kr);
      scatter_kr.clear();
      for (const auto& [g0, g1] : kr)
        if (range_needs_scatter(P, srec_i, g0, g1)) scatter_kr.emplace_back(g0, g1);
      if (w >= n_spec) {  // (the early windows are in their slots already)
        // a window no scatter reads (C4: only frames between direct runs)
        // needs no ring copy, so the copy stream carries no slot wait there
        // and its direct copies follow each other back to back
        if (scatter_kr.empty() && ring_skip) {
          ring_skipped += copy_window(P, run_i, off, off + len, buf, nullptr, false, E.s_copy, true);
        } else {
          if (w >= uint64_t(DrainEngine::kSlots))
            check_cuda(cudaStreamWaitEvent(E.s_copy, E.ev_free[slot], 0), "wait");
          copy_window(P, run_i, off, off + with_ahead, buf, const_cast<uint8_t*>(raw.data() + s3),
                      false, E.s_copy);
        }
        copy_direct(P, drun_i, off, off + len, const_cast<uint8_t*>(raw.data() + s3), false,
                    E.s_copy);
        check_cuda(cudaEventRecord(E.ev_ready[slot], E.s_copy), "event");
      }
      check_cuda(cudaStreamWaitEvent(E.s_pack, E.ev_ready[slot], 0), "wait");
      if (stats) cudaEventRecord(E.ev_w0[w], E.s_pack);
      for (const auto& [g0, g1] : scatter_kr) {
        ++scatter_launches;
        check_cuda(cudaError_t(crac_scatter_records(E.d_recs.ptr, uint32_t(P.recs.size()),
                                                    E.d_tile_rec.ptr + g0 / CRAC_TILE_BYTES,
                                                    buf + (g0 - off), g0, g1 - g0, E.s_pack)),
                   "scatter");
        scattered += g1 - g0;
      }
      if (stats) cudaEventRecord(E.ev_w1[w], E.s_pack);
      check_cuda(cudaEventRecord(E.ev_free[slot], E.s_pack), "event");
      // verify as we go: re-hash the regions whose last byte has landed, in
      // batches big enough to fill every SM (one 64 MiB region is only 64
      // K1 CTAs, and a warp hashing a single chunk never reaches its stride)
      size_t done = spans_done;
      while (done < P.pay_spans.size() &&
             P.pay_rec_off[done] + P.pay_spans[done].len <= off + len)
        ++done;
      if (done > spans_done && (P.pay_first[done] - P.pay_first[spans_done] >= verify_batch ||
                                w + 1 == windows)) {
        if (stats) {
          E.ensure_verify_events(verifies + 1);
          cudaEventRecord(E.ev_v0[verifies], E.s_pack);
        }
        hash_payloads_skip_pinned(E, P, P.pay_first[spans_done], P.pay_first[done], 0, E.s_pack,
                                  false);
        if (stats) cudaEventRecord(E.ev_v1[verifies], E.s_pack);
        ++verifies;
        spans_done = done;
      }
    }
    check_cuda(cudaEventRecord(E.ev_c1, E.s_copy), "event");
    join_tail_map();  // (every record fit in the head)
    if (P.n_dev_pages) {
      if (stats) {
        E.ensure_verify_events(verifies + 1);
        cudaEventRecord(E.ev_v0[verifies], E.s_pack);
      }
      hash_pages(E, P, 0, E.s_pack);
      if (stats) cudaEventRecord(E.ev_v1[verifies], E.s_pack);
      ++verifies;
    }
    tr.mark("windows");
  };
  // the engine streams must be idle before an error unwinds the session
  // (the arena they write into is unmapped with it)
  auto quiet = [&] {
    cudaStreamSynchronize(E.s_copy);
    cudaStreamSynchronize(E.s_pack);
  };

  // the replay (host bookkeeping; the extents are premapped) runs on its own
  // thread beside the plan join and the data path's enqueue when early
  std::exception_ptr replay_err;
  auto do_replay = [&] {
    ctx.begin_replay(live);
    try {
      replay_log_into(ctx, p.log, &binaries, nullptr);
    } catch (...) {
      replay_err = std::current_exception();
    }
    ctx.end_replay();
  };
  std::thread replay_thread;
  struct ReplayJoin {
    std::thread& t;
    ~ReplayJoin() {
      if (t.joinable()) t.join();
    }
  } replay_join{replay_thread};
  if (early) {
    replay_thread = std::thread([&, dev = E.device] {
      cudaSetDevice(dev);  // stream creates of the replay land on this device
      do_replay();
    });
    early_plan.join();
    if (plan_err) std::rethrow_exception(plan_err);
    tr.mark("plan");
    enqueue_data_path();
    replay_thread.join();
  } else {
    do_replay();
  }
  if (replay_err) {
    quiet();
    std::rethrow_exception(replay_err);
  }
  tr.mark("replay");
  join_tail_map();  // (when the data path had nothing to wait for it)
  if (ctx.live_stream_ids() != p.streams) {
    quiet();
    raise(Errc::ReplayDivergence, "live streams after replay do not match the snapshot");
  }

  // destinations of every framed record, in image order
  std::vector<BulkItem> items;
  std::vector<uint64_t> ptrs;
  bool match = ctx.match_records(p.facts.active, ptrs);
  for (size_t k = 0; match && early && k < ptrs.size(); ++k)
    match = ptrs[k] == p.facts.active[k].address;
  if (!match) {
    quiet();
    raise(Errc::ReplayDivergence, "the active set does not match the replayed allocations");
  }
  size_t mi = 0;
  items.reserve(ptrs.size());
  for (size_t k = 0; k < ptrs.size(); ++k) {
    const AllocationRecord& rec = p.facts.active[k];
    BulkItem it{rec.id, rec.kind, rec.size, ptrs[k], nullptr};
    if (rec.kind == AllocationKind::Managed) it.flags = &p.managed[mi++].flags;
    items.push_back(it);
  }
  tr.mark("items");
  if (!early) {
    plan(items);
    tr.mark("plan");
  }

  // managed pages land where they were: device-resident ones are first
  // touched by the scatter kernel (and verified by K1), host-resident ones
  // are written and hashed by the host threads below, so nothing migrates
  // and no prefetch or device mapping is needed to restore residence
  mi = 0;
  for (const AllocationRecord& rec : p.facts.active)
    if (rec.kind == AllocationKind::Managed) ctx.set_managed_flags(rec.id, p.managed[mi++].flags);
  std::exception_ptr fill_err;
  std::thread host_fill([&, dev = E.device] {
    try {
      cudaSetDevice(dev);  // the host-CRC buffer is pinned: no context on device 0
      host_pages_refill(E, P, raw.data() + s3);
    } catch (...) {
      fill_err = std::current_exception();
    }
  });
  struct Joiner {
    std::thread& t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } joiner{host_fill};
  tr.mark("place");

  // pinned-host payload contents: moved and hashed by host threads (the
  // verify launches skip their chunks; their CRCs join the fold below)
  copy_pinned_runs(E, P, const_cast<uint8_t*>(raw.data() + s3), false);
  if (!early) enqueue_data_path();
  if (P.stream_len > 20) {
    host_fill.join();  // the host-resident pages' CRCs
    if (fill_err) {
      cudaStreamSynchronize(E.s_copy);  // the enqueued data path reads the image
      cudaStreamSynchronize(E.s_pack);
      std::rethrow_exception(fill_err);
    }
    tr.mark("host-fill-join");
    if (!P.host_pages.empty())
      check_cuda(cudaMemcpyAsync(E.d_page_crc.ptr + P.n_dev_pages, E.h_host_crc.ptr,
                                 P.host_pages.size() * 4, cudaMemcpyHostToDevice, E.s_pack),
                 "host page crcs");
    upload_pinned_hashes(E, P, false, E.s_pack);
    enqueue_fold(E, P, E.s_pack);
    tr.mark("enqueue");
    check_cuda(cudaStreamSynchronize(E.s_pack), "refill sync");
    tr.mark("h2d+verify");
    uint32_t crc3 = 0, crc4 = 0;
    finish_fold(E, P, crc3, crc4);
    if (crc3 != p.sec[2].crc) raise(Errc::ImageCorrupt, "crc mismatch in ALLOC_PAYLOADS");
    if (crc4 != p.sec[3].crc) raise(Errc::ImageCorrupt, "crc mismatch in UVM_PAGES");
  } else if (p.sec[2].crc != 0 || p.sec[3].crc != 0) {
    raise(Errc::ImageCorrupt, "crc mismatch in empty bulk section");
  }
  check_cuda(cudaEventRecord(E.ev_t1, E.s_pack), "event");
  check_cuda(cudaEventSynchronize(E.ev_t1), "event sync");
  E.prev_valid = false;  // no pinned image of this session exists yet
  P.valid = false;

  session.log().reset(std::move(p.log));
  session.app_state() = std::move(p.app_state);
  if (stats) {
    stats->host_pre_ms = host_pre_ms;
    stats->total_ms = host_pre_ms + elapsed(E.ev_t0, E.ev_t1);
    if (windows) {
      stats->copy_ms = elapsed(E.ev_c0, E.ev_c1);
      stats->pack_launches = scatter_launches;
      stats->pack_bytes = scattered;
      // mean per scatter launch (windows of direct runs only launch none)
      double win_ms = 0;
      for (uint64_t w = 0; w < windows; ++w) win_ms += elapsed(E.ev_w0[w], E.ev_w1[w]);
      stats->pack_ms = scatter_launches ? win_ms / double(scatter_launches) : 0.0;
      // the early windows carried the host-run bytes of their range too
      uint64_t early_host = 0;
      for (const auto& [lo, hi] : P.host_runs)
        if (lo < n_spec * W) early_host += std::min(hi, n_spec * W) - lo;
      stats->h2d_bytes = P.stream_len - host_run_bytes(P) + early_host - ring_skipped;
      stats->hash_bytes = hashed_bytes(P);
      stats->hash_launches = verifies;
      for (uint64_t v = 0; v < verifies; ++v) stats->hash_ms += elapsed(E.ev_v0[v], E.ev_v1[v]);
    }
    stats->image_bytes = raw.size();
    stats->total_chunks = P.pay_first.back() + P.n_dev_pages + P.host_pages.size();
  }
  return std::move(session);
}

// ---------------------------------------------------------------------------
// incremental drain
// ---------------------------------------------------------------------------
namespace {

// Runs with the dispatch gate held; the layout of `image` is E.plan's.
void incremental_locked(Session& session, PinnedImage& image, DrainStats* stats) {
  PhaseTrace tr("incr");
  DrainEngine& E = session.drain_engine();
  const ImagePlan& P = E.plan;
  DeviceContext& ctx = session.device();
  if (stats) {
    *stats = DrainStats{};
    stats->incremental = true;
  }
  check_cuda(cudaEventRecord(E.ev_t0, E.s_pack), "event");
  uint8_t* img = image.mutable_data();
  const uint64_t s3 = P.s3;

  // One fused pass (K1 + K2b): every warp hashes its chunks and, where the
  // CRC differs from the previous image's, writes the chunk straight into the
  // pinned image; the PCIe writes of dirty chunks overlap the hashing.
  const uint64_t n = P.pay_first.back();
  E.d_counters.ensure(2);
  E.h_count.ensure(2);
  if (E.dst_for_image != P.image_ptr) {
    std::vector<uint64_t> dst(P.pay_rec_off.size());
    for (size_t s = 0; s < dst.size(); ++s) dst[s] = s3 + P.pay_rec_off[s];
    upload(E.d_pay_dst, dst, E.s_pack);
    E.dst_for_image = P.image_ptr;
  }
  // Split by default: writer CTAs stream the dirty chunks over PCIe while the
  // other SMs hash at HBM speed (CRAC_INCR_SPLIT=0: every hashing warp writes
  // its own dirty chunks, the fused form)
  static const bool split = [] {
    const char* e = std::getenv("CRAC_INCR_SPLIT");
    return !(e && !std::strcmp(e, "0"));
  }();
  static const int writers_env = [] {
    const char* e = std::getenv("CRAC_INCR_WRITERS");
    return e ? std::atoi(e) : 0;
  }();
  const uint32_t writers =
      uint32_t(writers_env > 0 ? writers_env : std::max(1, std::min(16, E.sm_count / 8)));
  E.d_counters.ensure(5);
  check_cuda(cudaMemsetAsync(E.d_counters.ptr, 0, 40, E.s_pack), "counters");
  if (split) E.d_dirty_idx.ensure(n + uint64_t(writers) * 16 + 1);
  check_cuda(cudaEventRecord(E.ev_h0, E.s_pack), "event");
  if (split)
    check_cuda(cudaError_t(crac_hash_drain_split(
                   E.d_pay_spans.ptr, E.d_pay_first.ptr, uint32_t(P.pay_spans.size()),
                   DrainEngine::kChunk, 0, n, E.d_pay_crc.ptr, E.d_prev_crc.ptr, E.d_pay_key.ptr,
                   E.d_prev_key.ptr, E.d_pay_dst.ptr, img, E.d_counters.ptr,
                   reinterpret_cast<unsigned long long*>(E.d_dirty_idx.ptr), writers, E.s_pack)),
               "hash+drain split");
  else
    check_cuda(cudaError_t(crac_hash_drain_range(
                   E.d_pay_spans.ptr, E.d_pay_first.ptr, uint32_t(P.pay_spans.size()),
                   DrainEngine::kChunk, 0, n, E.d_pay_crc.ptr, E.d_prev_crc.ptr, E.d_pay_key.ptr,
                   E.d_prev_key.ptr, E.d_pay_dst.ptr, img, E.d_counters.ptr, E.s_pack)),
               "hash+drain");
  check_cuda(cudaEventRecord(E.ev_h1, E.s_pack), "event");
  check_cuda(cudaMemcpyAsync(E.h_count.ptr, E.d_counters.ptr, 16, cudaMemcpyDeviceToHost, E.s_pack),
             "counters");
  enqueue_fold(E, P, E.s_pack);
  check_cuda(cudaStreamSynchronize(E.s_pack), "hash sync");
  tr.mark("hash+drain+fold");
  const uint64_t dirty = E.h_count.ptr[0], dirty_bytes = E.h_count.ptr[1];
  uint32_t crc3 = 0, crc4 = 0;
  finish_fold(E, P, crc3, crc4);
  put_at<uint32_t>(img + s3 + P.len3, crc3);
  put_at<uint32_t>(img + s3 + P.stream_len, crc4);

  // the tail sections may change without a layout change (app_state bytes)
  const std::vector<uint8_t> sec5 = streams_bytes(ctx.live_stream_ids());
  const std::vector<uint8_t>& sec6 = session.app_state();
  const std::vector<uint8_t> sec7 = registry_bytes(ctx.registered_binaries());
  uint64_t at = s3 + P.stream_len + 4;
  at += write_section(img + at, 5, sec5);
  at += write_section(img + at, 6, sec6);
  at += write_section(img + at, 7, sec7);

  check_cuda(cudaEventRecord(E.ev_t1, E.s_pack), "event");
  check_cuda(cudaEventSynchronize(E.ev_t1), "event sync");
  if (stats) {
    stats->total_ms = elapsed(E.ev_t0, E.ev_t1);
    stats->hash_ms = elapsed(E.ev_h0, E.ev_h1);
    stats->hash_launches = 1;
    stats->hash_bytes = hashed_bytes(P);
    stats->copy_ms = stats->hash_ms;  // the drain writes ride inside the hash pass
    stats->pack_launches = 0;
    stats->pack_bytes = dirty_bytes;
    stats->d2h_bytes = dirty_bytes;
    stats->image_bytes = P.image_bytes;
    stats->dirty_chunks = dirty;
    stats->total_chunks = n;
  }
}

}  // namespace

void checkpoint_incremental(Session& session, PinnedImage& image, DrainStats* stats) {
  // Emits exactly the bytes of a full drain.  Valid while the layout of the
  // previous image of this session is unchanged (same log, same bulk
  // records, no managed allocations, same tail size) and `image` is that
  // image; otherwise this is a full drain.
  if (!session.has_drain_engine()) {  // no previous image: a full drain
    full_drain(session, image, stats, true);
    return;
  }
  finish_pending(session);
  DrainEngine& E = session.drain_engine();
  const ImagePlan& P = E.plan;
  auto layout_unchanged = [&] {
    if (!P.valid || !E.prev_valid || image.size() != P.image_bytes ||
        reinterpret_cast<uint64_t>(image.data()) != P.image_ptr ||
        session.log().size() != P.log_len || tail_bytes(session) != P.tail_bytes)
      return false;
    std::vector<uint64_t> sig;
    for (const auto& r : active_set(session.log().snapshot())) {
      if (r.kind == AllocationKind::Managed) return false;
      sig.push_back(r.id);
      sig.push_back(r.size);
    }
    return sig == P.log_sizes;
  };
  if (!layout_unchanged()) {
    full_drain(session, image, stats, true);
    return;
  }
  bool raced = false;
  session.barrier_ms = 0;
  {
    QuiesceScope q(session.table(), session.config().quiesce_timeout);
    raced = !layout_unchanged();  // re-check under the gate: the log cannot move now
    if (!raced) {
      session.global_barrier(kPhaseQuiesced);
      incremental_locked(session, image, stats);
    }
  }
  if (raced) {
    full_drain(session, image, stats, true);
    return;
  }
  session.global_barrier(kPhaseImageComplete);
  if (stats) stats->barrier_ms = session.barrier_ms;
}

}  // namespace cracsim

// ---------------------------------------------------------------------------
// pre-copy drain (SURVEY §8f.3 stall reduction without spare HBM)
// ---------------------------------------------------------------------------
// Phase 1 runs while the application keeps running: K1 hashes every payload
// chunk and writes the very bytes it hashed (from its registers) straight into
// the pinned image, so every chunk's CRC describes exactly the bytes the image
// holds, however the application changes the memory meanwhile.  Phase 2 is an
// ordinary incremental drain under the gate: every chunk whose content moved
// since phase 1 hashed it is written again, so the image is the state at the
// instant of phase 2 and the application stops only for a hash pass plus the
// changed bytes.  Device-only sessions (a freed Device extent stays mapped,
// so reading it mid-free is harmless; pinned / managed backings are released
// on free) with at least one payload; anything else is a synchronous drain.
namespace cracsim {
namespace {

void precopy_wait(Session& session, double* phase1_ms) {
  DrainEngine& E = session.drain_engine();
  DrainEngine::Pending& Q = E.pending;
  if (!Q.precopy) return;
  check_cuda(cudaStreamSynchronize(E.s_hash), "pre-copy sync");
  if (phase1_ms) *phase1_ms = elapsed(E.ev_t0, E.ev_h1);
  ImagePlan& P = E.plan;
  // the image now holds, chunk by chunk, the bytes whose CRCs K1 left in
  // d_pay_crc: they seed the incremental pass
  const uint64_t n_pay = P.pay_first.back();
  seed_prev_keys(E, n_pay, E.s_hash);
  check_cuda(cudaStreamSynchronize(E.s_hash), "pre-copy seed");
  P.valid = true;
  P.image_ptr = reinterpret_cast<uint64_t>(Q.out->data());
  E.prev_valid = true;
  E.dst_for_image = 0;  // rebuild the image-offset table for this image
  Q = DrainEngine::Pending{};
}

}  // namespace

void checkpoint_precopy_begin(Session& session, PinnedImage& out, DrainStats* stats) {
  finish_pending(session);
  DeviceContext& ctx = session.device();
  DrainEngine& E = session.drain_engine();
  ImagePlan& P = E.plan;
  bool eligible = true;
  uint8_t* img = nullptr;
  {
    QuiesceScope q(session.table(), session.config().quiesce_timeout);
    if (stats) *stats = DrainStats{};
    const SnapshotMeta meta{ctx.seed(), ctx.arena_bytes(), kEngineVersion};
    const std::vector<CallLogEntry> log = session.log().snapshot();
    const std::vector<AllocationRecord> active = active_set(log);
    eligible = !active.empty() && std::all_of(active.begin(), active.end(), [](const AllocationRecord& r) {
      return r.kind == AllocationKind::Device;
    });
    if (eligible) {
      const std::vector<uint8_t> sec1 = meta_bytes(meta);
      const std::vector<uint8_t> sec2 = log_bytes(log);
      const std::vector<uint8_t> sec5 = streams_bytes(ctx.live_stream_ids());
      const std::vector<uint8_t>& sec6 = session.app_state();
      const std::vector<uint8_t> sec7 = registry_bytes(ctx.registered_binaries());
      std::vector<std::vector<uint8_t>> flags;
      build_plan(live_items(ctx, active, flags, false), P);
      P.log_len = log.size();
      const uint64_t s3 = 16 + (20 + sec1.size()) + (20 + sec2.size()) + 16;
      const uint64_t total = s3 + P.stream_len + 4 + (20 + sec5.size()) + (20 + sec6.size()) +
                             (20 + sec7.size());
      out.prepare(total, s3);
      P.s3 = s3;
      P.image_bytes = total;
      P.tail_bytes = (20 + sec5.size()) + (20 + sec6.size()) + (20 + sec7.size());
      P.valid = false;
      E.prev_valid = false;
      img = out.mutable_data();
      std::memcpy(img, kImageMagic, 8);
      put_at<uint32_t>(img + 8, kImageVersion);
      put_at<uint32_t>(img + 12, kSectionCount);
      uint64_t at = 16;
      at += write_section(img + at, 1, sec1);
      at += write_section(img + at, 2, sec2);
      put_at<uint32_t>(img + at, 3);
      put_at<uint32_t>(img + at + 4, 0);
      put_at<uint64_t>(img + at + 8, P.len3);
      // crc3 (patched by phase 2) and the empty UVM_PAGES header
      put_at<uint32_t>(img + s3 + P.len3, 0);
      put_at<uint32_t>(img + s3 + P.len3 + 4, 4);
      put_at<uint32_t>(img + s3 + P.len3 + 8, 0);
      put_at<uint64_t>(img + s3 + P.len3 + 12, 0);
      at = s3 + P.stream_len + 4;
      at += write_section(img + at, 5, sec5);
      at += write_section(img + at, 6, sec6);
      at += write_section(img + at, 7, sec7);
      if (at != total) raise(Errc::DeviceFault, "image layout mismatch");
      upload_plan(E, P, E.s_hash);
      upload(E.d_pay_soff, P.pay_rec_off, E.s_hash);
      check_cuda(cudaEventRecord(E.ev_t0, E.s_hash), "event");
    }
  }  // the application runs from here on
  if (!eligible) {
    full_drain(session, out, stats, true);
    return;
  }
  const bool aligned = std::all_of(P.pay_rec_off.begin(), P.pay_rec_off.end(),
                                   [](uint64_t o) { return o % 16 == 0; });
  uint8_t* stream = img + P.s3;  // page-locked host memory, written by the SMs over PCIe
  check_cuda(cudaError_t(crac_hash_copy_range(E.d_pay_spans.ptr, E.d_pay_first.ptr,
                                              uint32_t(P.pay_spans.size()), DrainEngine::kChunk, 0,
                                              P.pay_first.back(), E.d_pay_crc.ptr, E.d_pay_key.ptr,
                                              E.d_pay_soff.ptr,
                                              stream, aligned ? 1 : 0, E.s_hash)),
             "pre-copy hash+copy");
  check_cuda(cudaError_t(crac_write_frames(E.d_recs.ptr, uint32_t(P.pay_spans.size()), stream,
                                           E.s_hash)),
             "pre-copy frames");
  check_cuda(cudaEventRecord(E.ev_h1, E.s_hash), "event");
  DrainEngine::Pending& Q = E.pending;
  Q = DrainEngine::Pending{};
  Q.precopy = true;
  Q.out = &out;
}

void checkpoint_precopy_finish(Session& session, DrainStats* stats) {
  DrainEngine& E = session.drain_engine();
  if (!E.pending.precopy) {  // nothing in flight (or a synchronous fallback ran)
    if (stats && E.pending.active) drain_finish(session, stats);
    return;
  }
  PinnedImage& out = *E.pending.out;
  double phase1 = 0;
  precopy_wait(session, &phase1);
  checkpoint_incremental(session, out, stats);
  if (stats) {
    stats->stall_ms = stats->total_ms;  // phase 2 runs with the gate held
    stats->total_ms += phase1;
    stats->shadow_bytes = 0;
  }
}

}  // namespace cracsim
