// Source-compatibility check of the C++ drop-in surface: a client written
// against the reference API (/root/reference/proj/include/cracsim/*.hpp, the
// shapes of proj/tests/test_ckpt_engine.cpp and test_image.cpp) compiles
// unchanged against include/cracsim and runs on the B200 engine.
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <string>
#include <thread>
#include <vector>

#include "cracsim/ckpt_engine.hpp"
#include "cracsim/common.hpp"
#include "cracsim/errors.hpp"
#include "cracsim/image.hpp"
#include "cracsim/kernels.hpp"
#include "cracsim/shim.hpp"

using namespace cracsim;

static int failures = 0;
#define CHECK(cond)                                                    \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

template <typename Fn>
static void expect_errc(Errc code, Fn&& fn) {
  try {
    fn();
    std::printf("FAIL: expected %s, got none\n", errc_name(code));
    ++failures;
  } catch (const Error& e) {
    CHECK(e.code() == code);
  }
}

static std::vector<uint8_t> patterned(uint64_t n, uint8_t salt) {
  std::vector<uint8_t> v(n);
  for (uint64_t i = 0; i < n; ++i) v[i] = static_cast<uint8_t>(mix64(i + salt));
  return v;
}

int main() {
  SessionConfig cfg;
  cfg.seed = 4;
  cfg.arena_bytes = 1ull << 20;

  {  // checkpoint captures exactly the bytes the app wrote (test_ckpt_engine.cpp:75-87)
    Session s(cfg);
    const auto rec = s.api().alloc(AllocationKind::Device, 1024);
    s.api().copy_h2d({rec.id, 0}, std::vector<uint8_t>(1024, 0xAB), std::nullopt);
    const Snapshot snap = checkpoint(s);
    CHECK(snap.payloads.size() == 1);
    CHECK(snap.payloads[0].bytes == std::vector<uint8_t>(1024, 0xAB));
    CHECK(encode_image(snap).size() == 188 + 36 + 16 + 1024);
  }
  {  // restart rebuilds structure, bytes, streams and registry (test_ckpt_engine.cpp:162-210)
    Session s(cfg);
    auto& api = s.api();
    api.register_fat_binary(standard_kernels());
    const uint64_t s1 = api.stream_create();
    api.stream_create();
    api.stream_destroy(2);
    const auto dev = api.alloc(AllocationKind::Device, 3000);
    const auto man = api.alloc(AllocationKind::Managed, 2 * kPageSize + 100);
    api.copy_h2d({dev.id, 0}, patterned(3000, 1), std::nullopt);
    api.page_write(man.id, 0, patterned(2 * kPageSize + 100, 3), PageSide::Host);
    api.launch(s1, "add8", {{man.id, 0}}, {7, 100});
    api.synchronize();
    s.app_state() = {1, 2, 3};
    const Snapshot snap = checkpoint(s);
    Session r = restart(snap, standard_catalog());
    CHECK(r.device().live_records() == s.device().live_records());
    CHECK(r.device().free_holes() == s.device().free_holes());
    CHECK(r.device().live_stream_ids() == s.device().live_stream_ids());
    CHECK(r.device().registered_binaries() == s.device().registered_binaries());
    CHECK(r.app_state() == s.app_state());
    for (const auto& rec : s.device().live_records())
      CHECK(r.device().read_raw(rec.address, rec.size) == s.device().read_raw(rec.address, rec.size));
    CHECK(r.device().managed_pages(man.id) == s.device().managed_pages(man.id));
    // restart of a restart is lossless, image bytes included
    CHECK(encode_image(checkpoint(r)) == encode_image(snap));
  }
  {  // the fast path emits the same bytes as the value path
    Session s(cfg);
    for (int i = 0; i < 5; ++i) {
      const auto rec = s.api().alloc(AllocationKind::Device, 5000 + 17 * i);
      s.api().copy_h2d({rec.id, 0}, patterned(5000 + 17 * i, uint8_t(i)), std::nullopt);
    }
    PinnedImage img;
    DrainStats st;
    checkpoint_image(s, img, &st);
    CHECK(std::vector<uint8_t>(img.data(), img.data() + img.size()) == encode_image(checkpoint(s)));
    CHECK(st.hash_launches >= 1 && st.d2h_bytes > 0);
    Session r = restart_image(img.bytes(), standard_catalog());
    CHECK(r.device().live_records() == s.device().live_records());
  }
  {  // replay divergence and unknown kernel bodies (test_ckpt_engine.cpp:132-141, 226-240)
    Session s(cfg);
    s.api().alloc(AllocationKind::Device, 512);
    s.api().alloc(AllocationKind::Device, 512);
    auto log = s.log().snapshot();
    log[1].address += kAlign;
    DeviceContext fresh(3, 1ull << 20);
    expect_errc(Errc::ReplayDivergence, [&] { replay_log(fresh, log); });
    Session t(cfg);
    t.api().register_fat_binary(standard_kernels());
    expect_errc(Errc::UnknownKernelBody, [&] { restart(checkpoint(t), KernelCatalog{}); });
  }
  {  // image files, compressed included (test_ckpt_engine.cpp:257-278)
    Session s(cfg);
    const auto rec = s.api().alloc(AllocationKind::PinnedHost, 777);
    s.api().copy_h2d({rec.id, 0}, patterned(777, 9), std::nullopt);
    const auto path = std::filesystem::temp_directory_path() / "dropin_roundtrip.ckpt";
    for (bool compress : {false, true}) {
      checkpoint_to_file(s, path, compress);
      CHECK(is_compressed_image(read_file_bytes(path)) == compress);
      Session r = restart_from_file(path, standard_catalog());
      CHECK(r.device().read_raw(rec.address, rec.size) == s.device().read_raw(rec.address, rec.size));
    }
    std::filesystem::remove(path);
  }
  {  // log text and active set (test_shim.cpp:32-49, 84-111)
    Session s(cfg);
    const auto a = s.api().alloc(AllocationKind::Device, 1024);
    s.api().alloc(AllocationKind::Managed, 50);
    s.api().free(a.id);
    const auto entries = s.log().snapshot();
    CHECK(format_log_entry(entries[0]) == "1 Alloc device 1024 1 0xd0000000000");
    CHECK(format_log_entry(entries[1]) == "2 Alloc managed 50 2 0xd0000000400");
    CHECK(format_log_entry(entries[2]) == "3 Free - 0 1 0x0");
    CHECK(active_set(entries).size() == 1);
  }
  {  // checkpoints interleaved with live traffic stay consistent (test_ckpt_engine.cpp:310-330)
    Session s(cfg);
    std::thread worker([&] {
      for (int i = 0; i < 300; ++i) {
        const auto rec = s.api().alloc(AllocationKind::Device, 256 + 16 * (i % 7));
        s.api().copy_h2d({rec.id, 0}, patterned(64, uint8_t(i)), std::nullopt);
        if (i % 3 == 2) s.api().free(rec.id);
      }
    });
    for (int i = 0; i < 20; ++i) {
      const Snapshot snap = checkpoint(s);
      CHECK(decode_image(encode_image(snap)) == snap);
    }
    worker.join();
  }
  std::printf(failures ? "FAILED %d\n" : "ok\n", failures);
  return failures ? 1 : 0;
}
