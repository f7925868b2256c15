// Independent host check of a drained image (crac_image_verify, crac_engine.h).
//
// The refill's own check is K1 at refill against K1 at drain: a defect shared
// by the two (a 64-bit offset bug in K1 or the K4 fold at >4 GiB stream
// offsets) would pass it.  This check shares no code with the GPU path: every
// section CRC is recomputed on the host cores (PCLMUL CRC over 1 MiB blocks,
// combined in GF(2)), and, for the synthetic workloads of BASELINE.json
// (every Device payload filled with fill_synthetic(id, seed)), every payload
// byte is compared with the content regenerated from f(seed, id, offset)
// (the reference harness's synthetic pattern, common.hpp:55-60 mix64).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "crac_engine.h"
#include "crc_math.hpp"
#include "image_codec.hpp"

using namespace cracsim;

namespace {

constexpr uint64_t kBlock = 1ull << 20;

// Compares image bytes [p, p + n) with synthetic allocation content starting
// at byte `off` of allocation `id`.  Returns true when equal.
bool synth_equal(const uint8_t* p, uint64_t n, uint64_t seed, uint64_t id, uint64_t off) {
  const uint64_t salt = 0x1000003ull * id + (seed << 56);
  uint64_t k = off / 8;
  uint64_t i = 0;
  // leading partial word
  if (off % 8) {
    const uint64_t w = mix64(k + salt);
    const uint32_t b0 = uint32_t(off % 8);
    for (uint32_t b = b0; b < 8 && i < n; ++b, ++i)
      if (p[i] != uint8_t(w >> (8 * b))) return false;
    ++k;
  }
  uint64_t diff = 0;
  for (; i + 8 <= n; i += 8, ++k) {
    uint64_t v;
    std::memcpy(&v, p + i, 8);
    diff |= v ^ mix64(k + salt);
  }
  if (diff) return false;
  if (i < n) {
    const uint64_t w = mix64(k + salt);
    for (uint32_t b = 0; i < n; ++b, ++i)
      if (p[i] != uint8_t(w >> (8 * b))) return false;
  }
  return true;
}

}  // namespace

namespace cracsim {

// Body of crac_image_verify (capi.cpp); throws cracsim::Error.
void verify_image(const void* image, uint64_t size, uint32_t threads, uint64_t synth_seed,
                  int check_synth, crac_verify_t* out) {
  {
    if (!image || !out) raise(Errc::InvalidArgument, "crac_image_verify: null argument");
    const auto t0 = std::chrono::steady_clock::now();
    *out = crac_verify_t{};
    std::vector<uint8_t> storage;
    const std::span<const uint8_t> raw =
        codec::unwrap({static_cast<const uint8_t*>(image), size}, storage, nullptr);
    // framing, log and small sections (strict rules of the reference decode);
    // the bulk sections' CRCs are recomputed below, not trusted
    const codec::ParsedImage p = codec::parse_image(raw, /*verify_bulk=*/false);
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());

    // work list: every section in 1 MiB blocks
    struct Block {
      uint32_t sec;
      uint64_t off, len;  // absolute offset in raw
    };
    std::vector<Block> blocks;
    for (uint32_t s = 0; s < kSectionCount; ++s) {
      const auto& v = p.sec[s];
      for (uint64_t a = 0; a < v.length || (a == 0 && v.length == 0); a += kBlock) {
        blocks.push_back({s, v.payload_off + a, std::min(kBlock, v.length - a)});
        if (v.length == 0) break;
      }
    }
    // payload frames of ALLOC_PAYLOADS, ascending frame_off, with their kind
    std::vector<uint8_t> is_device(p.payloads.size(), 0);
    if (check_synth) {
      for (size_t k = 0; k < p.payloads.size(); ++k) {
        const auto it = std::lower_bound(
            p.facts.active.begin(), p.facts.active.end(), p.payloads[k].id,
            [](const AllocationRecord& r, uint64_t id) { return r.id < id; });
        is_device[k] = it != p.facts.active.end() && it->id == p.payloads[k].id &&
                       it->kind == AllocationKind::Device;
      }
    }
    const uint64_t s3 = p.sec[2].payload_off;
    std::vector<uint32_t> crc(blocks.size());
    std::unique_ptr<std::atomic<uint8_t>[]> bad_payload(new std::atomic<uint8_t>[p.payloads.size() + 1]());
    std::atomic<uint64_t> next{0}, compared{0};
    std::exception_ptr err;
    std::mutex mu;
    auto worker = [&] {
      try {
        for (;;) {
          const uint64_t b = next.fetch_add(1, std::memory_order_relaxed);
          if (b >= blocks.size()) return;
          const Block& B = blocks[b];
          const uint8_t* q = raw.data() + B.off;
          crc[b] = codec::crc32_fast(q, B.len, 0);
          if (!check_synth || B.sec != 2 || p.payloads.empty()) continue;
          // payload bytes of this block: frames whose data intersects it
          const uint64_t lo = B.off - s3, hi = lo + B.len;  // section-relative
          auto it = std::upper_bound(p.payloads.begin(), p.payloads.end(), lo,
                                     [](uint64_t x, const codec::PayloadFrame& f) {
                                       return x < f.frame_off;
                                     });
          if (it != p.payloads.begin()) --it;
          uint64_t cmp = 0;
          for (; it != p.payloads.end() && it->frame_off < hi; ++it) {
            const size_t k = size_t(it - p.payloads.begin());
            if (!is_device[k]) continue;
            const uint64_t d0 = it->frame_off + 16, d1 = d0 + it->len;
            const uint64_t a = std::max(lo, d0), e = std::min(hi, d1);
            if (a >= e) continue;
            if (!synth_equal(raw.data() + s3 + a, e - a, synth_seed, it->id, a - d0))
              bad_payload[k].store(1, std::memory_order_relaxed);
            cmp += e - a;
          }
          compared.fetch_add(cmp, std::memory_order_relaxed);
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
      }
    };
    std::vector<std::thread> pool;
    for (uint32_t t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    if (err) std::rethrow_exception(err);

    // combine block CRCs per section (crc32_combine) and compare
    uint32_t pow2[64];
    pow2[0] = 0x00800000u;
    for (int k = 1; k < 64; ++k) pow2[k] = crac::gf_mul(pow2[k - 1], pow2[k - 1]);
    const uint32_t shift_block = crac::x8n(kBlock, pow2);
    size_t b = 0;
    for (uint32_t s = 0; s < kSectionCount; ++s) {
      uint32_t c = 0;
      bool first = true;
      for (; b < blocks.size() && blocks[b].sec == s; ++b) {
        if (first) {
          c = crc[b];
          first = false;
        } else {
          c = (blocks[b].len == kBlock ? crac::gf_mul(shift_block, c)
                                       : crac::advance(c, blocks[b].len, pow2)) ^ crc[b];
        }
        out->crc_bytes += blocks[b].len;
      }
      if (c != p.sec[s].crc) out->bad_sections |= 1u << s;
      ++out->sections_checked;
    }
    out->first_bad_id = ~0ull;
    for (size_t k = 0; k < p.payloads.size(); ++k) {
      if (!is_device[k]) continue;
      ++out->payloads_compared;
      if (bad_payload[k].load()) {
        ++out->mismatched_payloads;
        if (out->first_bad_id == ~0ull) out->first_bad_id = p.payloads[k].id;
      }
    }
    out->payload_bytes_compared = compared.load();
    out->threads = threads;
    out->ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
}

}  // namespace cracsim
