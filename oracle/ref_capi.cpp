// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI over the *unmodified* reference library (cracsim, compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libcracsim_ref.so).  Every entry point mirrors one entry point
// of include/crac_engine.h with a `ref_` prefix instead of `crac_`, so the
// parity tests drive the reference and the B200 engine with the same call
// sequence and byte-compare the images.
//
// Reference interfaces wrapped (file:line under /root/reference/proj):
//   Session / SessionConfig          include/cracsim/ckpt_engine.hpp:18-55
//   RuntimeApi (DispatchTable)        include/cracsim/shim.hpp:159-184
//   checkpoint / restart              src/ckpt_engine.cpp:29-61, 120-171
//   encode_image / decode_image       src/image.cpp:383-404
//   summarize_image                   src/image.cpp:406-413
//   standard_kernels / catalog        src/kernels.cpp:108-117
//
// Error convention: 0 = ok, 1 + Errc index on cracsim::Error, 100 on any
// other exception; ref_last_error() returns the message of the last failure
// on the calling thread.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cracsim/ckpt_engine.hpp"
#include "cracsim/image.hpp"
#include "cracsim/kernels.hpp"

using namespace cracsim;

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

struct RefSession {
  Session s;
  explicit RefSession(Session&& x) : s(std::move(x)) {}
};

std::optional<uint64_t> opt_stream(int64_t s) {
  if (s < 0) return std::nullopt;
  return static_cast<uint64_t>(s);
}

double secs_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// The synthetic content function shared with the B200 engine's fill kernel
// (paper_2008_10596_b200/csrc/kernels.cu:synth_word): the 64-bit word at
// byte offset 8k of allocation `id` is mix64(k + 0x1000003*id + (seed<<56)),
// stored little-endian; a trailing partial word is truncated.
void synth_bytes(uint64_t seed, uint64_t id, uint64_t size, uint8_t* out) {
  const uint64_t words = size / 8;
  for (uint64_t k = 0; k < words; ++k) {
    const uint64_t w = mix64(k + 0x1000003ull * id + (seed << 56));
    std::memcpy(out + 8 * k, &w, 8);
  }
  if (size % 8) {
    const uint64_t w = mix64(words + 0x1000003ull * id + (seed << 56));
    std::memcpy(out + 8 * words, &w, size % 8);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_session_create(uint64_t seed, uint64_t arena_bytes, int mode, uint32_t timeout_ms,
                       void** out) {
  return guard([&] {
    SessionConfig cfg;
    cfg.seed = seed;
    cfg.arena_bytes = arena_bytes;
    cfg.mode = mode ? TableMode::Proxy : TableMode::Direct;
    cfg.quiesce_timeout = std::chrono::milliseconds(timeout_ms);
    *out = new RefSession(Session(cfg));
  });
}

void ref_session_destroy(void* h) { delete static_cast<RefSession*>(h); }

int ref_alloc(void* h, uint8_t kind, uint64_t size, uint64_t* id, uint64_t* address) {
  return guard([&] {
    auto rec = static_cast<RefSession*>(h)->s.api().alloc(static_cast<AllocationKind>(kind), size);
    *id = rec.id;
    *address = rec.address;
  });
}

int ref_free(void* h, uint64_t id) {
  return guard([&] { static_cast<RefSession*>(h)->s.api().free(id); });
}

int ref_stream_create(void* h, uint64_t* id) {
  return guard([&] { *id = static_cast<RefSession*>(h)->s.api().stream_create(); });
}

int ref_stream_destroy(void* h, uint64_t id) {
  return guard([&] { static_cast<RefSession*>(h)->s.api().stream_destroy(id); });
}

// Names found in the standard catalog get their real bodies; other names get
// an empty body (the reference tests register such placeholder kernels).
int ref_register_fat_binary(void* h, uint32_t n, const char* const* names,
                            const uint32_t* buffer_arity, const uint32_t* scalar_arity,
                            uint64_t* handle) {
  return guard([&] {
    std::vector<KernelDescriptor> ks;
    const auto& cat = standard_catalog();
    for (uint32_t i = 0; i < n; ++i) {
      KernelBody body = [](KernelArgs&) {};
      auto it = cat.find(names[i]);
      if (it != cat.end()) body = it->second;
      ks.push_back(KernelDescriptor{names[i], buffer_arity[i], scalar_arity[i], body});
    }
    *handle = static_cast<RefSession*>(h)->s.api().register_fat_binary(std::move(ks));
  });
}

int ref_unregister_fat_binary(void* h, uint64_t handle) {
  return guard([&] { static_cast<RefSession*>(h)->s.api().unregister_fat_binary(handle); });
}

int ref_launch(void* h, uint64_t stream, const char* kernel, uint32_t nbuf, const uint64_t* ids,
               const uint64_t* offs, uint32_t nsc, const uint64_t* scalars) {
  return guard([&] {
    std::vector<BufferRef> b;
    for (uint32_t i = 0; i < nbuf; ++i) b.push_back(BufferRef{ids[i], offs[i]});
    std::vector<uint64_t> sc(scalars, scalars + nsc);
    static_cast<RefSession*>(h)->s.api().launch(stream, kernel, std::move(b), std::move(sc));
  });
}

int ref_copy_h2d(void* h, uint64_t id, uint64_t off, const uint8_t* src, uint64_t n,
                 int64_t stream) {
  return guard([&] {
    static_cast<RefSession*>(h)->s.api().copy_h2d({id, off}, {src, n}, opt_stream(stream));
  });
}

int ref_copy_d2h(void* h, uint8_t* dst, uint64_t id, uint64_t off, uint64_t n, int64_t stream) {
  return guard([&] {
    static_cast<RefSession*>(h)->s.api().copy_d2h({dst, n}, {id, off}, opt_stream(stream));
  });
}

int ref_copy_d2d(void* h, uint64_t did, uint64_t doff, uint64_t sid, uint64_t soff, uint64_t n,
                 int64_t stream) {
  return guard([&] {
    static_cast<RefSession*>(h)->s.api().copy_d2d({did, doff}, {sid, soff}, n,
                                                  opt_stream(stream));
  });
}

int ref_synchronize(void* h) {
  return guard([&] { static_cast<RefSession*>(h)->s.api().synchronize(); });
}

int ref_page_read(void* h, uint64_t id, uint64_t off, uint64_t n, uint8_t side, uint8_t* out) {
  return guard([&] {
    auto v = static_cast<RefSession*>(h)->s.api().page_read(id, off, n,
                                                            static_cast<PageSide>(side));
    std::memcpy(out, v.data(), v.size());
  });
}

int ref_page_write(void* h, uint64_t id, uint64_t off, const uint8_t* src, uint64_t n,
                   uint8_t side) {
  return guard([&] {
    static_cast<RefSession*>(h)->s.api().page_write(id, off, {src, n},
                                                    static_cast<PageSide>(side));
  });
}

int ref_set_app_state(void* h, const uint8_t* src, uint64_t n) {
  return guard([&] { static_cast<RefSession*>(h)->s.app_state().assign(src, src + n); });
}

// Writes synth content (see synth_bytes) into a Device/PinnedHost allocation
// with one copy_h2d, or into a managed one with page_write from `side`.
int ref_fill_synthetic(void* h, uint64_t id, uint64_t seed, uint8_t managed_side) {
  return guard([&] {
    auto& s = static_cast<RefSession*>(h)->s;
    auto rec = s.device().find_record(id);
    if (!rec) raise(Errc::UnknownId, "fill_synthetic");
    std::vector<uint8_t> bytes(rec->size);
    synth_bytes(seed, id, rec->size, bytes.data());
    if (rec->kind == AllocationKind::Managed)
      s.api().page_write(id, 0, bytes, static_cast<PageSide>(managed_side));
    else
      s.api().copy_h2d({id, 0}, bytes, std::nullopt);
  });
}

void ref_synth_bytes(uint64_t seed, uint64_t id, uint64_t size, uint8_t* out) {
  synth_bytes(seed, id, size, out);
}

// checkpoint(session) + encode_image; the image is heap memory released by
// ref_buffer_free.  Optional phase timings in seconds.
int ref_checkpoint_image(void* h, uint8_t** image, uint64_t* size, double* t_ckpt,
                         double* t_encode) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    Snapshot snap = checkpoint(static_cast<RefSession*>(h)->s);
    if (t_ckpt) *t_ckpt = secs_since(t0);
    t0 = std::chrono::steady_clock::now();
    auto bytes = encode_image(snap);
    if (t_encode) *t_encode = secs_since(t0);
    *size = bytes.size();
    *image = static_cast<uint8_t*>(std::malloc(bytes.size() ? bytes.size() : 1));
    std::memcpy(*image, bytes.data(), bytes.size());
  });
}

void ref_buffer_free(void* p) { std::free(p); }

// decode_image + restart(standard_catalog) from an in-memory image.
int ref_restart_image(const uint8_t* image, uint64_t size, int mode, void** out, double* t_decode,
                      double* t_restart) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    Snapshot snap = decode_image({image, size});
    if (t_decode) *t_decode = secs_since(t0);
    t0 = std::chrono::steady_clock::now();
    Session s = restart(snap, standard_catalog(), mode ? TableMode::Proxy : TableMode::Direct);
    if (t_restart) *t_restart = secs_since(t0);
    *out = new RefSession(std::move(s));
  });
}

// checkpoint_to_file / restart_from_file (ref: ckpt_engine.hpp:63-84), the
// reference's own file path: whole-buffer ofstream / ifstream.
int ref_checkpoint_to_file(void* h, const char* path, int compress, double* t_total) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    checkpoint_to_file(static_cast<RefSession*>(h)->s, path, compress != 0);
    if (t_total) *t_total = secs_since(t0);
  });
}

int ref_restart_from_file(const char* path, int mode, void** out, double* t_total) {
  return guard([&] {
    auto t0 = std::chrono::steady_clock::now();
    Session s = restart_from_file(path, standard_catalog(),
                                  mode ? TableMode::Proxy : TableMode::Direct);
    if (t_total) *t_total = secs_since(t0);
    *out = new RefSession(std::move(s));
  });
}

int ref_decode_check(const uint8_t* image, uint64_t size) {
  return guard([&] { (void)decode_image({image, size}); });
}

// summarize_image: section tags/lengths/crcs (7 each) plus the totals.
int ref_summarize(const uint8_t* image, uint64_t size, uint64_t* lengths, uint32_t* crcs,
                  uint64_t* totals /* log_entries, active, payload_bytes, uvm_bytes, file */) {
  return guard([&] {
    auto sum = summarize_image({image, size});
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

// Encodes the reference test fixture snapshots (test_image.cpp:14-52):
// which = 0 empty_snapshot, 1 rich_snapshot.  Restated here because the
// doctest suites cannot be built (doctest.h is not vendored).
int ref_fixture_image(int which, uint8_t** image, uint64_t* size) {
  return guard([&] {
    Snapshot s;
    if (which == 0) {
      s.meta.seed = 0;
      s.meta.arena_bytes = 1ull << 24;
    } else {
      s.meta.seed = 5;
      s.meta.arena_bytes = 1ull << 20;
      auto alloc = [&](uint64_t id, AllocationKind kind, uint64_t sz, uint64_t address) {
        s.log.push_back(
            {s.log.size() + 1, LogOp::Alloc, static_cast<uint8_t>(kind), sz, id, address});
      };
      auto op = [&](LogOp o, uint64_t id) { s.log.push_back({s.log.size() + 1, o, 0, 0, id, 0}); };
      alloc(1, AllocationKind::Device, 1000, kArenaBase);
      alloc(2, AllocationKind::Managed, 4196, kArenaBase + 1024);
      op(LogOp::StreamCreate, 1);
      alloc(3, AllocationKind::PinnedHost, 10, kArenaBase + 1024 + 4352);
      op(LogOp::RegisterBinary, 1);
      op(LogOp::StreamCreate, 2);
      op(LogOp::StreamDestroy, 1);
      alloc(4, AllocationKind::Device, 5, kArenaBase + 1024 + 4352 + 256);
      op(LogOp::Free, 4);
      s.payloads.push_back({1, std::vector<uint8_t>(1000, 0xA1)});
      s.payloads.push_back({3, std::vector<uint8_t>(10, 0xA3)});
      ManagedRecord m{2, {}};
      m.pages.push_back({0, true, false, std::vector<uint8_t>(4096, 0xB0)});
      m.pages.push_back({1, false, true, std::vector<uint8_t>(100, 0xB1)});
      s.managed.push_back(std::move(m));
      s.streams = {2};
      s.app_state.assign(33, 0x5A);
      s.binaries.push_back({1, {{"scale", 2, 1}, {"probe", 1, 0}}});
    }
    auto bytes = encode_image(s);
    *size = bytes.size();
    *image = static_cast<uint8_t*>(std::malloc(bytes.size()));
    std::memcpy(*image, bytes.data(), bytes.size());
  });
}

int ref_debug_dump(void* h, char** out) {
  return guard([&] {
    auto d = static_cast<RefSession*>(h)->s.device().debug_dump();
    *out = static_cast<char*>(std::malloc(d.size() + 1));
    std::memcpy(*out, d.c_str(), d.size() + 1);
  });
}

// Log as 36-byte records exactly as the image stores them (image.cpp:39-51
// layout), into a caller buffer of 36*log_size bytes.
int ref_log_size(void* h, uint64_t* n) {
  return guard([&] { *n = static_cast<RefSession*>(h)->s.log().size(); });
}

int ref_live_records(void* h, uint64_t cap, uint64_t* ids, uint8_t* kinds, uint64_t* sizes,
                     uint64_t* addresses, uint64_t* n) {
  return guard([&] {
    auto recs = static_cast<RefSession*>(h)->s.device().live_records();
    *n = recs.size();
    for (size_t i = 0; i < recs.size() && i < cap; ++i) {
      ids[i] = recs[i].id;
      kinds[i] = static_cast<uint8_t>(recs[i].kind);
      sizes[i] = recs[i].size;
      addresses[i] = recs[i].address;
    }
  });
}

// Managed page flags: bit0 device_resident, bit1 dirty, one byte per page.
int ref_managed_pages(void* h, uint64_t id, uint64_t cap, uint8_t* flags, uint64_t* n) {
  return guard([&] {
    auto pages = static_cast<RefSession*>(h)->s.device().managed_pages(id);
    *n = pages.size();
    for (size_t i = 0; i < pages.size() && i < cap; ++i)
      flags[i] = (pages[i].device_resident ? 1 : 0) | (pages[i].dirty ? 2 : 0);
  });
}

int ref_read_raw(void* h, uint64_t address, uint64_t n, uint8_t* out) {
  return guard([&] {
    auto v = static_cast<RefSession*>(h)->s.device().read_raw(address, n);
    std::memcpy(out, v.data(), v.size());
  });
}

}  // extern "C"
