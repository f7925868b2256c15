// libcrac_preload.so — cudart interposition onto the logged dispatch table
// (API and environment in include/crac_preload.h).
//
// The reference's shim (ref: src/shim.cpp:204-253) is the logged call path;
// its harness drives it directly because there is no real runtime below it
// (SPEC.md:17).  Here the application's own CUDA runtime calls land on it:
// allocation-family calls become logged session calls, everything that
// touches device state and is forwarded to the real runtime is admitted
// through the session's dispatch gate.  Only this file sees the application's
// libcudart (through dlsym(RTLD_NEXT)); libcrac_b200.so carries its own
// statically linked runtime and does not export cuda* symbols, so the
// engine's internal calls never come back through these interposers.
#include <cuda_runtime_api.h>
#include <dlfcn.h>
#include <semaphore.h>
#include <signal.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "crac_engine.h"
#include "crac_preload.h"

namespace {

constexpr int kDevice = 1, kPinned = 2, kManaged = 3;
constexpr char kWrapMagic[8] = {'C', 'R', 'A', 'C', 'P', 'R', 'L', '1'};

template <typename Fn>
Fn real(const char* name) {
  void* p = dlsym(RTLD_NEXT, name);
  if (!p) {
    std::fprintf(stderr, "crac_preload: %s not found in the application's runtime "
                         "(link it with -cudart shared)\n", name);
    std::abort();
  }
  return reinterpret_cast<Fn>(p);
}

struct Alloc {
  uint64_t id;
  int kind;
  uint64_t logical;  // arena address from the log: stable across restarts
};

struct State {
  std::once_flag once;
  int init_rc = 0;
  crac_session_t* s = nullptr;
  crac_image_t* img = nullptr;
  bool restarted = false;
  std::mutex mu;
  std::unordered_map<uintptr_t, Alloc> allocs;              // pointer -> allocation
  std::unordered_map<cudaStream_t, uint64_t> streams;       // handle -> stream id
  std::unordered_map<uint64_t, uintptr_t> by_logical;       // logical -> pointer now
  std::unordered_map<uintptr_t, uint64_t> old_to_logical;   // pointer before restart
  std::vector<uint8_t> app;                                 // the application's bytes
  std::atomic<uint64_t> n_alloc{0}, n_free{0}, n_gated{0}, n_ckpt{0};
  sem_t ckpt_sem;
};

State& st() {
  static State* g = new State();  // never destroyed: calls may arrive during exit
  return *g;
}

cudaError_t to_cuda(int rc) {
  switch (rc) {
    case 0: return cudaSuccess;
    case 1: return cudaErrorInvalidValue;          // InvalidArgument
    case 2: return cudaErrorMemoryAllocation;      // OutOfArena
    case 5: return cudaErrorInvalidResourceHandle;  // StreamLimitExceeded
    default: return cudaErrorUnknown;
  }
}

void note(const char* what, int rc) {
  std::fprintf(stderr, "crac_preload: %s failed (%d): %s\n", what, rc, crac_last_error());
}

// APPSTATE = "CRACPRL1" | u64 n | n x (pointer u64, logical u64) | app bytes:
// the pointer table lets crac_preload_translate map pre-restart pointers.
std::vector<uint8_t> wrap_app_state(State& g) {
  std::vector<uint8_t> out(kWrapMagic, kWrapMagic + 8);
  auto put = [&](uint64_t v) {
    for (int i = 0; i < 8; ++i) out.push_back(uint8_t(v >> (8 * i)));
  };
  put(g.allocs.size());
  for (const auto& [ptr, a] : g.allocs) {
    put(ptr);
    put(a.logical);
  }
  out.insert(out.end(), g.app.begin(), g.app.end());
  return out;
}

void unwrap_app_state(State& g, const uint8_t* p, uint64_t n) {
  auto get = [&](uint64_t at) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= uint64_t(p[at + i]) << (8 * i);
    return v;
  };
  if (n >= 16 && std::memcmp(p, kWrapMagic, 8) == 0) {
    const uint64_t k = get(8);
    if (16 + 16 * k <= n) {
      for (uint64_t i = 0; i < k; ++i) g.old_to_logical[get(16 + 16 * i)] = get(24 + 16 * i);
      g.app.assign(p + 16 + 16 * k, p + n);
      return;
    }
  }
  g.app.assign(p, p + n);
}

void rebuild_maps(State& g) {
  uint64_t n = 0;
  crac_live_records(g.s, 0, nullptr, nullptr, nullptr, nullptr, &n);
  std::vector<uint64_t> ids(n), sizes(n), addrs(n);
  std::vector<uint8_t> kinds(n);
  crac_live_records(g.s, n, ids.data(), kinds.data(), sizes.data(), addrs.data(), &n);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t ptr = 0;
    crac_backing_ptr(g.s, ids[i], &ptr);
    g.allocs[ptr] = Alloc{ids[i], kinds[i], addrs[i]};
    g.by_logical[addrs[i]] = ptr;
  }
  crac_live_streams(g.s, 0, nullptr, &n);
  std::vector<uint64_t> sids(n);
  crac_live_streams(g.s, n, sids.data(), &n);
  for (uint64_t id : sids) {
    void* h = nullptr;
    if (crac_stream_handle(g.s, id, &h) == 0) g.streams[static_cast<cudaStream_t>(h)] = id;
  }
}

// The application is stopped only for the drain's gated phase: a pre-copy
// (the state is copied while the application runs, then only what changed is
// re-sent under the gate; sessions with pinned / managed memory drain
// synchronously instead), then the file is written from the pinned image
// while the application runs again.  CRAC_PRECOPY=0: a plain drain.
int checkpoint_locked(State& g, const char* path) {
  const std::vector<uint8_t> wrapped = wrap_app_state(g);
  int rc = crac_set_app_state(g.s, wrapped.data(), wrapped.size());
  const char* pc = std::getenv("CRAC_PRECOPY");
  if (pc && !std::strcmp(pc, "0")) {
    if (rc == 0) rc = crac_checkpoint_to_file(g.s, g.img, path, 0, nullptr, nullptr);
  } else {
    if (rc == 0) rc = crac_checkpoint_precopy_begin(g.s, g.img, nullptr);
    if (rc == 0) rc = crac_checkpoint_precopy_finish(g.s, nullptr);
    const uint8_t* data = nullptr;
    uint64_t n = 0;
    if (rc == 0) rc = crac_image_view(g.img, &data, &n);
    if (rc == 0) rc = crac_file_write(path, data, n, 0, 0, 3, nullptr);  // O_DIRECT + fdatasync
  }
  if (rc == 0) ++g.n_ckpt;
  return rc;
}

void ckpt_thread() {
  State& g = st();
  for (;;) {
    while (sem_wait(&g.ckpt_sem) != 0) {
    }
    const char* path = std::getenv("CRAC_CKPT_PATH");
    if (!path) {
      std::fprintf(stderr, "crac_preload: SIGUSR2 without CRAC_CKPT_PATH\n");
      continue;
    }
    std::lock_guard lk(g.mu);
    const int rc = checkpoint_locked(g, path);
    if (rc) note("checkpoint (SIGUSR2)", rc);
  }
}

void on_sigusr2(int) { sem_post(&st().ckpt_sem); }  // async-signal-safe

void report_at_exit() {
  State& g = st();
  std::fprintf(stderr, "crac_preload: allocs %lu frees %lu gated %lu checkpoints %lu%s\n",
               (unsigned long)g.n_alloc.load(), (unsigned long)g.n_free.load(),
               (unsigned long)g.n_gated.load(), (unsigned long)g.n_ckpt.load(),
               g.restarted ? " (restarted)" : "");
}

void init() {
  State& g = st();
  int rc = crac_image_create(&g.img);
  if (const char* from = std::getenv("CRAC_RESTART_FROM"); rc == 0 && from && *from) {
    rc = crac_restart_from_file(from, g.img, 0, &g.s, nullptr, nullptr);
    if (rc == 0) {
      g.restarted = true;
      const uint8_t* p = nullptr;
      uint64_t n = 0;
      crac_get_app_state(g.s, &p, &n);
      unwrap_app_state(g, p, n);
      rebuild_maps(g);
    } else {
      note("restart_from_file", rc);
    }
  } else if (rc == 0) {
    const char* a = std::getenv("CRAC_ARENA_BYTES");
    const char* sd = std::getenv("CRAC_SEED");
    const uint64_t arena = a ? std::strtoull(a, nullptr, 0) : (16ull << 30);
    rc = crac_session_create(sd ? std::strtoull(sd, nullptr, 0) : 0, arena, 0, 30000, &g.s);
    if (rc) note("session create", rc);
  }
  if (rc == 0) rc = crac_set_device_wide_drain(g.s, 1);
  g.init_rc = rc;
  if (rc) return;
  sem_init(&g.ckpt_sem, 0, 0);
  std::thread(ckpt_thread).detach();
  struct sigaction sa {};
  sa.sa_handler = on_sigusr2;
  sa.sa_flags = SA_RESTART;
  sigaction(SIGUSR2, &sa, nullptr);
  if (const char* v = std::getenv("CRAC_PRELOAD_VERBOSE"); v && *v == '1') std::atexit(report_at_exit);
}

State* session() {
  State& g = st();
  std::call_once(g.once, init);
  return g.init_rc == 0 ? &g : nullptr;
}

cudaError_t intercept_alloc(void** out, size_t n, int kind) {
  if (!out) return cudaErrorInvalidValue;
  if (n == 0) {
    *out = nullptr;
    return cudaSuccess;
  }
  State* g = session();
  if (!g) return cudaErrorInitializationError;
  uint64_t id = 0, logical = 0, ptr = 0;
  int rc = crac_alloc(g->s, uint8_t(kind), n, &id, &logical);
  if (rc == 0) rc = crac_backing_ptr(g->s, id, &ptr);
  if (rc) return to_cuda(rc);
  {
    std::lock_guard lk(g->mu);
    g->allocs[ptr] = Alloc{id, kind, logical};
    g->by_logical[logical] = ptr;
  }
  ++g->n_alloc;
  *out = reinterpret_cast<void*>(ptr);
  return cudaSuccess;
}

// 1: not ours (forward); otherwise the cudaError_t of the session free.
int intercept_free(void* p, bool host_api) {
  if (!p) return cudaSuccess;
  State* g = session();
  if (!g) return 1;
  Alloc a;
  {
    std::lock_guard lk(g->mu);
    auto it = g->allocs.find(reinterpret_cast<uintptr_t>(p));
    if (it == g->allocs.end() || (it->second.kind == kPinned) != host_api) return 1;
    a = it->second;
    g->allocs.erase(it);
    g->by_logical.erase(a.logical);
  }
  // cudaFree synchronises the device before releasing memory; the session
  // unmaps the extent, so in-flight kernels must be done with it
  static auto sync = real<cudaError_t (*)()>("cudaDeviceSynchronize");
  sync();
  ++g->n_free;
  return to_cuda(crac_free(g->s, a.id));
}

cudaError_t intercept_stream(cudaStream_t* out) {
  if (!out) return cudaErrorInvalidValue;
  State* g = session();
  if (!g) return cudaErrorInitializationError;
  uint64_t id = 0;
  void* h = nullptr;
  int rc = crac_stream_create(g->s, &id);
  if (rc == 0) rc = crac_stream_handle(g->s, id, &h);
  if (rc) return to_cuda(rc);
  std::lock_guard lk(g->mu);
  g->streams[static_cast<cudaStream_t>(h)] = id;
  *out = static_cast<cudaStream_t>(h);
  return cudaSuccess;
}

// Holds the dispatch gate shared around a forwarded call.
struct Admitted {
  State* g;
  Admitted() : g(session()) {
    if (g) {
      crac_gate_enter(g->s);
      ++g->n_gated;
    }
  }
  ~Admitted() {
    if (g) crac_gate_leave(g->s);
  }
};

}  // namespace

extern "C" {

// ---- allocation family: logged session calls -------------------------------
cudaError_t cudaMalloc(void** devPtr, size_t size) { return intercept_alloc(devPtr, size, kDevice); }

cudaError_t cudaMallocManaged(void** devPtr, size_t size, unsigned int) {
  return intercept_alloc(devPtr, size, kManaged);
}

cudaError_t cudaMallocHost(void** ptr, size_t size) { return intercept_alloc(ptr, size, kPinned); }

cudaError_t cudaHostAlloc(void** pHost, size_t size, unsigned int) {
  return intercept_alloc(pHost, size, kPinned);
}

cudaError_t cudaFree(void* devPtr) {
  const int rc = intercept_free(devPtr, false);
  if (rc != 1) return static_cast<cudaError_t>(rc);
  static auto f = real<cudaError_t (*)(void*)>("cudaFree");
  return f(devPtr);
}

cudaError_t cudaFreeHost(void* ptr) {
  const int rc = intercept_free(ptr, true);
  if (rc != 1) return static_cast<cudaError_t>(rc);
  static auto f = real<cudaError_t (*)(void*)>("cudaFreeHost");
  return f(ptr);
}

cudaError_t cudaStreamCreate(cudaStream_t* pStream) { return intercept_stream(pStream); }

cudaError_t cudaStreamCreateWithFlags(cudaStream_t* pStream, unsigned int) {
  return intercept_stream(pStream);  // session streams are non-blocking
}

cudaError_t cudaStreamCreateWithPriority(cudaStream_t* pStream, unsigned int, int) {
  return intercept_stream(pStream);
}

cudaError_t cudaStreamDestroy(cudaStream_t stream) {
  State* g = session();
  uint64_t id = 0;
  bool ours = false;
  if (g) {
    std::lock_guard lk(g->mu);
    auto it = g->streams.find(stream);
    if (it != g->streams.end()) {
      id = it->second;
      ours = true;
      g->streams.erase(it);
    }
  }
  if (ours) return to_cuda(crac_stream_destroy(g->s, id));
  static auto f = real<cudaError_t (*)(cudaStream_t)>("cudaStreamDestroy");
  return f(stream);
}

// ---- forwarded through the gate ------------------------------------------------
cudaError_t cudaLaunchKernel(const void* func, dim3 grid, dim3 block, void** args, size_t shmem,
                             cudaStream_t stream) {
  static auto f = real<cudaError_t (*)(const void*, dim3, dim3, void**, size_t, cudaStream_t)>(
      "cudaLaunchKernel");
  Admitted a;
  return f(func, grid, block, args, shmem, stream);
}

cudaError_t cudaMemcpy(void* dst, const void* src, size_t count, cudaMemcpyKind kind) {
  static auto f = real<cudaError_t (*)(void*, const void*, size_t, cudaMemcpyKind)>("cudaMemcpy");
  Admitted a;
  return f(dst, src, count, kind);
}

cudaError_t cudaMemcpyAsync(void* dst, const void* src, size_t count, cudaMemcpyKind kind,
                            cudaStream_t stream) {
  static auto f = real<cudaError_t (*)(void*, const void*, size_t, cudaMemcpyKind, cudaStream_t)>(
      "cudaMemcpyAsync");
  Admitted a;
  return f(dst, src, count, kind, stream);
}

cudaError_t cudaMemset(void* devPtr, int value, size_t count) {
  static auto f = real<cudaError_t (*)(void*, int, size_t)>("cudaMemset");
  Admitted a;
  return f(devPtr, value, count);
}

cudaError_t cudaMemsetAsync(void* devPtr, int value, size_t count, cudaStream_t stream) {
  static auto f = real<cudaError_t (*)(void*, int, size_t, cudaStream_t)>("cudaMemsetAsync");
  Admitted a;
  return f(devPtr, value, count, stream);
}

// The rest of the runtime's device-state-changing calls: same gate.  (Driver
// API launches a library obtains through cuGetProcAddress -- cuBLAS under
// the runtime, for example -- never reach an LD_PRELOAD symbol; they are
// quiesced by the drain's device-wide synchronize.)
#define CRAC_GATED(ret, name, params, args)                              \
  ret name params {                                                      \
    static auto f = real<ret(*) params>(#name);                          \
    Admitted a;                                                          \
    return f args;                                                       \
  }

CRAC_GATED(cudaError_t, cudaMemcpy2D,
           (void* d, size_t dp, const void* s, size_t sp, size_t w, size_t h, cudaMemcpyKind k),
           (d, dp, s, sp, w, h, k))
CRAC_GATED(cudaError_t, cudaMemcpy2DAsync,
           (void* d, size_t dp, const void* s, size_t sp, size_t w, size_t h, cudaMemcpyKind k,
            cudaStream_t st),
           (d, dp, s, sp, w, h, k, st))
CRAC_GATED(cudaError_t, cudaMemcpy3D, (const cudaMemcpy3DParms* p), (p))
CRAC_GATED(cudaError_t, cudaMemcpy3DAsync, (const cudaMemcpy3DParms* p, cudaStream_t st), (p, st))
CRAC_GATED(cudaError_t, cudaMemcpyPeer, (void* d, int dd, const void* s, int sd, size_t n),
           (d, dd, s, sd, n))
CRAC_GATED(cudaError_t, cudaMemcpyPeerAsync,
           (void* d, int dd, const void* s, int sd, size_t n, cudaStream_t st), (d, dd, s, sd, n, st))
CRAC_GATED(cudaError_t, cudaMemcpyToSymbol,
           (const void* sym, const void* s, size_t n, size_t off, cudaMemcpyKind k), (sym, s, n, off, k))
CRAC_GATED(cudaError_t, cudaMemcpyToSymbolAsync,
           (const void* sym, const void* s, size_t n, size_t off, cudaMemcpyKind k, cudaStream_t st),
           (sym, s, n, off, k, st))
CRAC_GATED(cudaError_t, cudaMemcpyFromSymbol,
           (void* d, const void* sym, size_t n, size_t off, cudaMemcpyKind k), (d, sym, n, off, k))
CRAC_GATED(cudaError_t, cudaMemcpyFromSymbolAsync,
           (void* d, const void* sym, size_t n, size_t off, cudaMemcpyKind k, cudaStream_t st),
           (d, sym, n, off, k, st))
CRAC_GATED(cudaError_t, cudaMemset2D, (void* d, size_t p, int v, size_t w, size_t h), (d, p, v, w, h))
CRAC_GATED(cudaError_t, cudaMemset2DAsync,
           (void* d, size_t p, int v, size_t w, size_t h, cudaStream_t st), (d, p, v, w, h, st))
CRAC_GATED(cudaError_t, cudaMemset3D, (cudaPitchedPtr p, int v, cudaExtent e), (p, v, e))
CRAC_GATED(cudaError_t, cudaMemset3DAsync, (cudaPitchedPtr p, int v, cudaExtent e, cudaStream_t st),
           (p, v, e, st))
CRAC_GATED(cudaError_t, cudaLaunchKernelExC,
           (const cudaLaunchConfig_t* c, const void* fn, void** args), (c, fn, args))
CRAC_GATED(cudaError_t, cudaLaunchCooperativeKernel,
           (const void* fn, dim3 g, dim3 b, void** args, size_t sh, cudaStream_t st),
           (fn, g, b, args, sh, st))
CRAC_GATED(cudaError_t, cudaGraphLaunch, (cudaGraphExec_t e, cudaStream_t st), (e, st))
#undef CRAC_GATED

// ---- application API (crac_preload.h) -------------------------------------------
int crac_preload_checkpoint(const char* path) {
  State* g = session();
  if (!g) return st().init_rc;
  std::lock_guard lk(g->mu);
  const int rc = checkpoint_locked(*g, path);
  if (rc) note("checkpoint", rc);
  return rc;
}

int crac_preload_set_app_state(const void* data, uint64_t n) {
  State* g = session();
  if (!g) return st().init_rc;
  std::lock_guard lk(g->mu);
  const auto* p = static_cast<const uint8_t*>(data);
  g->app.assign(p, p + n);
  return 0;
}

int crac_preload_app_state(const void** data, uint64_t* n) {
  State* g = session();
  if (!g) return st().init_rc;
  std::lock_guard lk(g->mu);
  *data = g->app.data();
  *n = g->app.size();
  return 0;
}

int crac_preload_restarted(void) {
  State* g = session();
  return g && g->restarted ? 1 : 0;
}

void* crac_preload_translate(const void* old_ptr) {
  State* g = session();
  if (!g) return nullptr;
  std::lock_guard lk(g->mu);
  const auto key = reinterpret_cast<uintptr_t>(old_ptr);
  auto it = g->old_to_logical.find(key);
  if (it == g->old_to_logical.end()) return g->allocs.count(key) ? const_cast<void*>(old_ptr) : nullptr;
  auto p = g->by_logical.find(it->second);
  return p == g->by_logical.end() ? nullptr : reinterpret_cast<void*>(p->second);
}

void* crac_preload_session(void) {
  State* g = session();
  return g ? g->s : nullptr;
}

}  // extern "C"
