// extern "C" boundary of libcrac_b200.so (declared in include/crac_engine.h).
#include <cuda_runtime.h>

#include <cstdlib>
#include <algorithm>
#include <vector>
#include <chrono>
#include <atomic>
#include <thread>
#include <cstring>
#include <memory>

#include "crac_engine.h"
#include "crac_gpu.h"
#include "cracsim/kernels.hpp"
#include "image_codec.hpp"

using namespace cracsim;

namespace cracsim {
void verify_image(const void* image, uint64_t size, uint32_t threads, uint64_t synth_seed,
                  int check_synth, crac_verify_t* out);  // verify.cpp
}

struct crac_session {
  Session s;
  explicit crac_session(Session&& x) : s(std::move(x)) {}
};
struct crac_image {
  PinnedImage img;
};

namespace {

thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

std::optional<uint64_t> opt(int64_t stream) {
  if (stream < 0) return std::nullopt;
  return static_cast<uint64_t>(stream);
}

void to_c(const DrainStats& d, crac_stats_t* o) {
  if (!o) return;
  *o = crac_stats_t{};
  o->total_ms = d.total_ms;
  o->hash_ms = d.hash_ms;
  o->pack_ms = d.pack_ms;
  o->copy_ms = d.copy_ms;
  o->hash_bytes = d.hash_bytes;
  o->hash_launches = d.hash_launches;
  o->pack_launches = d.pack_launches;
  o->pack_bytes = d.pack_bytes;
  o->d2h_bytes = d.d2h_bytes;
  o->h2d_bytes = d.h2d_bytes;
  o->image_bytes = d.image_bytes;
  o->dirty_chunks = d.dirty_chunks;
  o->total_chunks = d.total_chunks;
  o->incremental = d.incremental ? 1 : 0;
  o->stall_ms = d.stall_ms;
  o->shadow_bytes = d.shadow_bytes;
  o->barrier_ms = d.barrier_ms;
  o->host_pre_ms = d.host_pre_ms;
}

void to_c(const FileIoStats& f, crac_io_stats_t* o) {
  if (!o) return;
  *o = crac_io_stats_t{f.ms, f.bytes, f.threads, f.direct ? 1 : 0, f.bounced, f.streamed};
}

template <typename T>
T* heap_copy(const T* p, size_t n) {
  T* out = static_cast<T*>(std::malloc(n ? n * sizeof(T) : 1));
  if (n) std::memcpy(out, p, n * sizeof(T));
  return out;
}

}  // namespace

extern "C" {

const char* crac_last_error(void) { return g_err.c_str(); }
int crac_abi_version(void) { return 2; }

int crac_session_create(uint64_t seed, uint64_t arena_bytes, int mode, uint32_t timeout_ms,
                        crac_session_t** out) {
  return guard([&] {
    SessionConfig cfg;
    cfg.seed = seed;
    cfg.arena_bytes = arena_bytes;
    cfg.mode = mode ? TableMode::Proxy : TableMode::Direct;
    cfg.quiesce_timeout = std::chrono::milliseconds(timeout_ms);
    *out = new crac_session(Session(cfg));
  });
}

void crac_session_destroy(crac_session_t* s) { delete s; }

int crac_session_fixed_va(crac_session_t* s) { return s->s.device().fixed_va() ? 1 : 0; }

int crac_alloc(crac_session_t* s, uint8_t kind, uint64_t size, uint64_t* id, uint64_t* address) {
  return guard([&] {
    const auto rec = s->s.api().alloc(static_cast<AllocationKind>(kind), size);
    *id = rec.id;
    *address = rec.address;
  });
}

int crac_free(crac_session_t* s, uint64_t id) {
  return guard([&] { s->s.api().free(id); });
}

int crac_stream_create(crac_session_t* s, uint64_t* id) {
  return guard([&] { *id = s->s.api().stream_create(); });
}

int crac_stream_destroy(crac_session_t* s, uint64_t id) {
  return guard([&] { s->s.api().stream_destroy(id); });
}

int crac_register_fat_binary(crac_session_t* s, uint32_t n, const char* const* names,
                             const uint32_t* buffer_arity, const uint32_t* scalar_arity,
                             uint64_t* handle) {
  return guard([&] {
    const KernelCatalog& cat = standard_catalog();
    std::vector<KernelDescriptor> ks;
    for (uint32_t i = 0; i < n; ++i) {
      auto it = cat.find(names[i]);
      KernelBody body = it != cat.end() ? it->second : KernelBody([](KernelArgs&) {});
      ks.push_back(KernelDescriptor{names[i], buffer_arity[i], scalar_arity[i], body});
    }
    *handle = s->s.api().register_fat_binary(std::move(ks));
  });
}

int crac_unregister_fat_binary(crac_session_t* s, uint64_t handle) {
  return guard([&] { s->s.api().unregister_fat_binary(handle); });
}

int crac_launch(crac_session_t* s, uint64_t stream, const char* kernel, uint32_t nbuf,
                const uint64_t* ids, const uint64_t* offs, uint32_t nsc, const uint64_t* scalars) {
  return guard([&] {
    std::vector<BufferRef> b;
    for (uint32_t i = 0; i < nbuf; ++i) b.push_back(BufferRef{ids[i], offs[i]});
    s->s.api().launch(stream, kernel, std::move(b), std::vector<uint64_t>(scalars, scalars + nsc));
  });
}

int crac_copy_h2d(crac_session_t* s, uint64_t id, uint64_t off, const void* src, uint64_t n,
                  int64_t stream) {
  return guard([&] {
    s->s.api().copy_h2d({id, off}, {static_cast<const uint8_t*>(src), n}, opt(stream));
  });
}

int crac_copy_d2h(crac_session_t* s, void* dst, uint64_t id, uint64_t off, uint64_t n,
                  int64_t stream) {
  return guard([&] {
    s->s.api().copy_d2h({static_cast<uint8_t*>(dst), n}, {id, off}, opt(stream));
  });
}

int crac_copy_d2d(crac_session_t* s, uint64_t did, uint64_t doff, uint64_t sid, uint64_t soff,
                  uint64_t n, int64_t stream) {
  return guard([&] { s->s.api().copy_d2d({did, doff}, {sid, soff}, n, opt(stream)); });
}

int crac_synchronize(crac_session_t* s) {
  return guard([&] { s->s.api().synchronize(); });
}

int crac_page_read(crac_session_t* s, uint64_t id, uint64_t off, uint64_t n, uint8_t side,
                   void* out) {
  return guard([&] {
    const auto v = s->s.api().page_read(id, off, n, static_cast<PageSide>(side));
    if (!v.empty()) std::memcpy(out, v.data(), v.size());
  });
}

int crac_page_write(crac_session_t* s, uint64_t id, uint64_t off, const void* src, uint64_t n,
                    uint8_t side) {
  return guard([&] {
    s->s.api().page_write(id, off, {static_cast<const uint8_t*>(src), n},
                          static_cast<PageSide>(side));
  });
}

int crac_set_app_state(crac_session_t* s, const void* src, uint64_t n) {
  return guard([&] {
    const uint8_t* p = static_cast<const uint8_t*>(src);
    s->s.app_state().assign(p, p + n);
  });
}

int crac_stream_handle(crac_session_t* s, uint64_t id, void** cuda_stream) {
  return guard([&] { *cuda_stream = s->s.device().stream_handle(id); });
}

int crac_live_streams(crac_session_t* s, uint64_t cap, uint64_t* ids, uint64_t* n) {
  return guard([&] {
    const auto v = s->s.device().live_stream_ids();
    *n = v.size();
    for (size_t i = 0; i < v.size() && i < cap; ++i) ids[i] = v[i];
  });
}

int crac_gate_enter(crac_session_t* s) {
  return guard([&] { s->s.table().admit(); });
}

int crac_gate_leave(crac_session_t* s) {
  return guard([&] { s->s.table().release(); });
}

int crac_set_device_wide_drain(crac_session_t* s, int on) {
  return guard([&] { s->s.table().set_device_wide_drain(on != 0); });
}

int crac_get_app_state(crac_session_t* s, const uint8_t** data, uint64_t* n) {
  return guard([&] {
    *data = s->s.app_state().data();
    *n = s->s.app_state().size();
  });
}

int crac_image_create(crac_image_t** out) {
  return guard([&] { *out = new crac_image(); });
}

void crac_image_destroy(crac_image_t* img) { delete img; }

int crac_image_view(crac_image_t* img, const uint8_t** data, uint64_t* size) {
  return guard([&] {
    *data = img->img.data();
    *size = img->img.size();
  });
}

int crac_image_pages(crac_image_t* img, uint64_t* capacity, uint64_t* huge_bytes) {
  return guard([&] {
    *capacity = img->img.capacity();
    *huge_bytes = img->img.huge_page_bytes();
  });
}

int crac_checkpoint(crac_session_t* s, crac_image_t* img, crac_stats_t* stats) {
  return guard([&] {
    DrainStats d;
    checkpoint_image(s->s, img->img, stats ? &d : nullptr);
    to_c(d, stats);
  });
}

int crac_image_verify(const void* image, uint64_t size, uint32_t threads, uint64_t synth_seed,
                      int check_synth, crac_verify_t* out) {
  return guard([&] { verify_image(image, size, threads, synth_seed, check_synth, out); });
}

int crac_session_verify_synthetic(crac_session_t* s, uint64_t seed, uint64_t* bad_allocations,
                                  uint64_t* bytes_checked) {
  return guard([&] {
    DeviceContext& ctx = s->s.device();
    std::vector<AllocationRecord> dev;
    for (const auto& r : ctx.live_records())
      if (r.kind == AllocationKind::Device) dev.push_back(r);
    uint32_t* d_flags = nullptr;
    check_cuda(cudaMalloc(&d_flags, 4 * (dev.size() + 1)), "verify flags");
    std::unique_ptr<uint32_t, decltype(&cudaFree)> keep(d_flags, &cudaFree);
    check_cuda(cudaMemset(d_flags, 0, 4 * (dev.size() + 1)), "verify memset");
    uint64_t bytes = 0;
    for (size_t k = 0; k < dev.size(); ++k) {
      const uint64_t p = ctx.backing_ptr(dev[k].id);
      check_cuda(cudaError_t(crac_verify_synth(reinterpret_cast<const uint8_t*>(p), dev[k].size,
                                               seed, dev[k].id, d_flags + k, nullptr)),
                 "verify synth");
      bytes += dev[k].size;
    }
    std::vector<uint32_t> h(dev.size() + 1);
    check_cuda(cudaMemcpy(h.data(), d_flags, 4 * h.size(), cudaMemcpyDeviceToHost), "verify readback");
    uint64_t bad = 0;
    for (size_t k = 0; k < dev.size(); ++k) bad += h[k] != 0;
    *bad_allocations = bad;
    *bytes_checked = bytes;
  });
}

int crac_probe_managed_populate(uint64_t bytes, uint64_t run, uint32_t threads, double* ms) {
  return guard([&] {
    if (!bytes || !run || run % 16 || !ms) raise(Errc::InvalidArgument, "populate probe arguments");
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    uint8_t* m = nullptr;
    check_cuda(cudaMallocManaged(&m, bytes, cudaMemAttachGlobal), "probe managed");
    std::unique_ptr<uint8_t, decltype(&cudaFree)> keep_m(m, &cudaFree);
    uint8_t* src = nullptr;
    check_cuda(cudaHostAlloc(&src, run, cudaHostAllocDefault), "probe pinned");
    std::unique_ptr<uint8_t, decltype(&cudaFreeHost)> keep_s(src, &cudaFreeHost);
    std::memset(src, 3, run);
    cudaStream_t st = nullptr;
    check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "probe stream");
    const auto t0 = std::chrono::steady_clock::now();
    check_cuda(cudaError_t(crac_touch_even_runs(m, bytes, run, st)), "probe kernel");
    std::atomic<uint64_t> next{1};
    std::vector<std::thread> pool;
    const uint64_t runs = (bytes + run - 1) / run;
    for (uint32_t t = 0; t < threads; ++t)
      pool.emplace_back([&] {
        for (uint64_t r; (r = next.fetch_add(2)) < runs;)
          std::memcpy(m + r * run, src, std::min(run, bytes - r * run));
      });
    for (auto& t : pool) t.join();
    const cudaError_t e = cudaStreamSynchronize(st);
    *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    cudaStreamDestroy(st);
    check_cuda(e, "probe sync");
  });
}

int crac_session_set_barrier(crac_session_t* s, crac_barrier_fn fn, void* ctx) {
  return guard([&] { s->s.set_barrier(GlobalBarrier{fn, ctx}); });
}

int crac_barrier_open(const char* name, uint32_t world, uint32_t rank, uint32_t timeout_ms,
                      crac_barrier_t** out) {
  return guard([&] {
    if (!name || !out) raise(Errc::InvalidArgument, "crac_barrier_open: null argument");
    *out = reinterpret_cast<crac_barrier_t*>(
        new ShmBarrier(name, world, rank, std::chrono::milliseconds(timeout_ms)));
  });
}

int crac_barrier_wait(crac_barrier_t* b) {
  return guard([&] {
    if (!reinterpret_cast<ShmBarrier*>(b)->wait())
      raise(Errc::QuiesceTimeout, "barrier wait timed out");
  });
}

int crac_barrier_hook(void* b, int phase) { return ShmBarrier::hook(b, phase); }

uint64_t crac_barrier_generation(crac_barrier_t* b) {
  return reinterpret_cast<ShmBarrier*>(b)->generation();
}

void crac_barrier_close(crac_barrier_t* b, int unlink) {
  auto* p = reinterpret_cast<ShmBarrier*>(b);
  if (!p) return;
  if (unlink) p->unlink_on_close();
  delete p;
}

int crac_reserve_shadow(crac_session_t* s, uint64_t bytes) {
  return guard([&] { reserve_shadow(s->s, bytes); });
}

int crac_reserve_shadow_on(crac_session_t* s, uint64_t bytes, int device) {
  return guard([&] { reserve_shadow(s->s, bytes, device); });
}

int crac_checkpoint_precopy_begin(crac_session_t* s, crac_image_t* img, crac_stats_t* stats) {
  return guard([&] {
    DrainStats d;
    checkpoint_precopy_begin(s->s, img->img, stats ? &d : nullptr);
    to_c(d, stats);
  });
}

int crac_checkpoint_precopy_finish(crac_session_t* s, crac_stats_t* stats) {
  return guard([&] {
    DrainStats d;
    checkpoint_precopy_finish(s->s, stats ? &d : nullptr);
    to_c(d, stats);
  });
}

int crac_checkpoint_begin(crac_session_t* s, crac_image_t* img, crac_stats_t* stats) {
  return guard([&] {
    DrainStats d;
    checkpoint_begin(s->s, img->img, stats ? &d : nullptr);
    to_c(d, stats);
  });
}

int crac_checkpoint_finish(crac_session_t* s, crac_stats_t* stats) {
  return guard([&] {
    DrainStats d;
    checkpoint_finish(s->s, stats ? &d : nullptr);
    to_c(d, stats);
  });
}

int crac_checkpoint_incremental(crac_session_t* s, crac_image_t* img, crac_stats_t* stats) {
  return guard([&] {
    DrainStats d;
    checkpoint_incremental(s->s, img->img, stats ? &d : nullptr);
    to_c(d, stats);
  });
}

int crac_checkpoint_value(crac_session_t* s, uint8_t** image, uint64_t* size) {
  return guard([&] {
    const auto bytes = encode_image(checkpoint(s->s));
    *size = bytes.size();
    *image = heap_copy(bytes.data(), bytes.size());
  });
}

int crac_restart(const void* image, uint64_t size, int mode, crac_session_t** out,
                 crac_stats_t* stats) {
  return guard([&] {
    DrainStats d;
    Session r = restart_image({static_cast<const uint8_t*>(image), size}, standard_catalog(),
                              mode ? TableMode::Proxy : TableMode::Direct,
                              std::chrono::milliseconds{30000}, stats ? &d : nullptr);
    to_c(d, stats);
    *out = new crac_session(std::move(r));
  });
}

int crac_checkpoint_to_file(crac_session_t* s, crac_image_t* img, const char* path, int compress,
                            crac_stats_t* drain, crac_io_stats_t* io) {
  return guard([&] {
    DrainStats d;
    FileIoStats f;
    if (compress < 0 || compress > 2) raise(Errc::InvalidArgument, "compress must be 0, 1 or 2");
    checkpoint_to_file(s->s, img->img, path, static_cast<Compression>(compress),
                       drain ? &d : nullptr, &f);
    to_c(d, drain);
    to_c(f, io);
  });
}

int crac_compress_image_gpu(const void* image, uint64_t n, uint8_t** out, uint64_t* out_n,
                            double* ms) {
  return guard([&] {
    const uint64_t cap = compressed_bound_gpu(n);
    std::unique_ptr<uint8_t, decltype(&std::free)> buf(alloc_compressed_host(cap), &std::free);
    *out_n = compress_image_gpu_into({static_cast<const uint8_t*>(image), n}, buf.get(), cap, ms);
    *out = buf.release();  // (no copy: the caller frees it with crac_buffer_free)
  });
}

int crac_restart_from_file(const char* path, crac_image_t* img, int mode, crac_session_t** out,
                           crac_stats_t* refill, crac_io_stats_t* io) {
  return guard([&] {
    DrainStats d;
    FileIoStats f;
    Session r = restart_from_file(path, img->img, standard_catalog(),
                                  mode ? TableMode::Proxy : TableMode::Direct,
                                  refill ? &d : nullptr, &f);
    to_c(d, refill);
    to_c(f, io);
    *out = new crac_session(std::move(r));
  });
}

int crac_file_write(const char* path, const void* data, uint64_t n, uint32_t threads,
                    uint64_t chunk_bytes, uint32_t flags, crac_io_stats_t* io) {
  return guard([&] {
    FileIoStats f;
    write_file_parallel(path, {static_cast<const uint8_t*>(data), n}, &f,
                        FileIoOptions{threads, chunk_bytes, (flags & 1) != 0, (flags & 2) != 0});
    to_c(f, io);
  });
}

int crac_file_size(const char* path, uint64_t* n) {
  return guard([&] { *n = file_bytes(path); });
}

int crac_file_read(const char* path, void* dst, uint64_t capacity, uint32_t threads,
                   uint64_t chunk_bytes, uint32_t flags, uint64_t* n, crac_io_stats_t* io) {
  return guard([&] {
    FileIoStats f;
    *n = read_file_parallel(path, static_cast<uint8_t*>(dst), capacity, &f,
                            FileIoOptions{threads, chunk_bytes, (flags & 1) != 0, false});
    to_c(f, io);
  });
}

int crac_peek_cuda_error(void) { return int(cudaPeekAtLastError()); }

int crac_drop_arena_cache(int device) {
  return guard([&] {
    int dev = device;
    if (dev < 0) check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    drop_arena_cache(dev);
  });
}

int crac_drop_arena_cache_async(int device) {
  return guard([&] {
    int dev = device;
    if (dev < 0) check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
    drop_arena_cache(dev, /*release_later=*/true);
  });
}

uint32_t crac_crc32_host(const void* data, uint64_t n, uint32_t crc) {
  return codec::crc32_fast(static_cast<const uint8_t*>(data), n, crc);
}

uint32_t crac_crc32_copy_host(void* dst, const void* src, uint64_t n, uint32_t crc) {
  const uint32_t r = codec::crc32_copy_stream(static_cast<uint8_t*>(dst), static_cast<const uint8_t*>(src), n, crc);
  codec::stream_fence();
  return r;
}

int crac_decode_check(const void* image, uint64_t size) {
  return guard([&] { (void)decode_image({static_cast<const uint8_t*>(image), size}); });
}

int crac_summarize(const void* image, uint64_t size, uint64_t* lengths, uint32_t* crcs,
                   uint64_t* totals) {
  return guard([&] {
    const auto sum = summarize_image({static_cast<const uint8_t*>(image), size});
    for (size_t i = 0; i < sum.sections.size() && i < 7; ++i) {
      lengths[i] = sum.sections[i].length;
      crcs[i] = sum.sections[i].crc;
    }
    totals[0] = sum.log_entries;
    totals[1] = sum.active_allocations;
    totals[2] = sum.payload_bytes;
    totals[3] = sum.uvm_page_bytes;
    totals[4] = sum.file_bytes;
  });
}

int crac_debug_dump(crac_session_t* s, char** out) {
  return guard([&] {
    const std::string d = s->s.device().debug_dump();
    *out = heap_copy(d.c_str(), d.size() + 1);
  });
}

void crac_buffer_free(void* p) { std::free(p); }

int crac_log_size(crac_session_t* s, uint64_t* n) {
  return guard([&] { *n = s->s.log().size(); });
}

int crac_live_records(crac_session_t* s, uint64_t cap, uint64_t* ids, uint8_t* kinds,
                      uint64_t* sizes, uint64_t* addresses, uint64_t* n) {
  return guard([&] {
    const auto recs = s->s.device().live_records();
    *n = recs.size();
    for (size_t i = 0; i < recs.size() && i < cap; ++i) {
      ids[i] = recs[i].id;
      kinds[i] = static_cast<uint8_t>(recs[i].kind);
      sizes[i] = recs[i].size;
      addresses[i] = recs[i].address;
    }
  });
}

int crac_managed_pages(crac_session_t* s, uint64_t id, uint64_t cap, uint8_t* flags, uint64_t* n) {
  return guard([&] {
    const auto pages = s->s.device().managed_pages(id);
    *n = pages.size();
    for (size_t i = 0; i < pages.size() && i < cap; ++i)
      flags[i] = uint8_t((pages[i].device_resident ? 1 : 0) | (pages[i].dirty ? 2 : 0));
  });
}

int crac_read_raw(crac_session_t* s, uint64_t address, uint64_t n, void* out) {
  return guard([&] {
    const auto v = s->s.device().read_raw(address, n);
    if (n) std::memcpy(out, v.data(), n);
  });
}

int crac_backing_ptr(crac_session_t* s, uint64_t id, uint64_t* ptr) {
  return guard([&] { *ptr = s->s.device().backing_ptr(id); });
}

int crac_fill_synthetic(crac_session_t* s, uint64_t id, uint64_t seed, uint8_t managed_side) {
  return guard([&] {
    DeviceContext& ctx = s->s.device();
    const auto rec = ctx.find_record(id);
    if (!rec) raise(Errc::UnknownId, "allocation " + std::to_string(id));
    if (rec->kind == AllocationKind::Managed && managed_side == uint8_t(PageSide::Host)) {
      // host-side write: generate on the host, page_write from the Host side
      std::vector<uint8_t> bytes(rec->size);
      for (uint64_t k = 0; k * 8 < rec->size; ++k) {
        const uint64_t w = mix64(k + 0x1000003ull * id + (seed << 56));
        std::memcpy(bytes.data() + 8 * k, &w, std::min<uint64_t>(8, rec->size - 8 * k));
      }
      s->s.api().page_write(id, 0, bytes, PageSide::Host);
      return;
    }
    ctx.device_fill(id, [&](void* p, uint64_t len, cudaStream_t st) {
      check_cuda(cudaError_t(crac_fill_synth(static_cast<uint8_t*>(p), len, seed, id, 0, st)),
                 "fill");
    });
  });
}

int crac_mutate_device(crac_session_t* s, uint64_t seed, uint64_t epoch, uint64_t threshold,
                       uint64_t* mutated) {
  return guard([&] {
    DeviceContext& ctx = s->s.device();
    std::vector<crac_span_t> spans;
    std::vector<uint64_t> ids, first{0};
    const uint64_t chunk = 65536;
    for (const auto& r : ctx.live_records()) {
      if (r.kind != AllocationKind::Device) continue;
      spans.push_back(crac_span_t{ctx.backing_ptr(r.id), r.size});
      ids.push_back(r.id);
      first.push_back(first.back() + (r.size + chunk - 1) / chunk);
    }
    uint64_t count = 0;
    for (uint64_t c = 0; c < first.back(); ++c)
      if (mix64(seed ^ (epoch << 40) ^ c) < threshold) ++count;
    if (mutated) *mutated = count;
    if (spans.empty()) return;
    cudaStream_t st = ctx.engine_stream();
    crac_span_t* d_spans = nullptr;
    uint64_t *d_ids = nullptr, *d_first = nullptr;
    check_cuda(cudaMallocAsync(&d_spans, spans.size() * sizeof(crac_span_t), st), "alloc");
    check_cuda(cudaMallocAsync(&d_ids, ids.size() * 8, st), "alloc");
    check_cuda(cudaMallocAsync(&d_first, first.size() * 8, st), "alloc");
    check_cuda(cudaMemcpyAsync(d_spans, spans.data(), spans.size() * sizeof(crac_span_t),
                               cudaMemcpyHostToDevice, st), "upload");
    check_cuda(cudaMemcpyAsync(d_ids, ids.data(), ids.size() * 8, cudaMemcpyHostToDevice, st), "upload");
    check_cuda(cudaMemcpyAsync(d_first, first.data(), first.size() * 8, cudaMemcpyHostToDevice, st),
               "upload");
    check_cuda(cudaError_t(crac_mutate_chunks(d_spans, d_ids, d_first, uint32_t(spans.size()),
                                              uint32_t(chunk), first.back(), seed, epoch,
                                              threshold, st)),
               "mutate");
    cudaFreeAsync(d_spans, st);
    cudaFreeAsync(d_ids, st);
    cudaFreeAsync(d_first, st);
    check_cuda(cudaStreamSynchronize(st), "mutate sync");
  });
}

int crac_hash_session(crac_session_t* s, crac_stats_t* stats) {
  return guard([&] {
    DrainStats d;
    hash_only(s->s, &d);
    to_c(d, stats);
  });
}

int crac_hash_host_buffer(const void* data, uint64_t n, uint32_t chunk_bytes, uint32_t* crc_out) {
  return guard([&] {
    if (n == 0) return;
    const uint64_t chunks = (n + chunk_bytes - 1) / chunk_bytes;
    uint8_t* d = nullptr;
    uint32_t* d_crc = nullptr;
    crac_span_t* d_span = nullptr;
    uint64_t* d_first = nullptr;
    check_cuda(cudaMalloc(&d, n + 64), "alloc");
    check_cuda(cudaMalloc(&d_crc, chunks * 4), "alloc");
    check_cuda(cudaMalloc(&d_span, sizeof(crac_span_t)), "alloc");
    check_cuda(cudaMalloc(&d_first, 16), "alloc");
    const crac_span_t span{reinterpret_cast<uint64_t>(d), n};
    const uint64_t first[2] = {0, chunks};
    check_cuda(cudaMemcpy(d, data, n, cudaMemcpyHostToDevice), "upload");
    check_cuda(cudaMemcpy(d_span, &span, sizeof(span), cudaMemcpyHostToDevice), "upload");
    check_cuda(cudaMemcpy(d_first, first, 16, cudaMemcpyHostToDevice), "upload");
    const int rc = crac_chunk_crc32(d_span, d_first, 1, chunk_bytes, chunks, d_crc, nullptr);
    cudaError_t e = cudaError_t(rc);
    if (!e) e = cudaMemcpy(crc_out, d_crc, chunks * 4, cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaFree(d_crc);
    cudaFree(d_span);
    cudaFree(d_first);
    check_cuda(e, "K1");
  });
}

}  // extern "C"
