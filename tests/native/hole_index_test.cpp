// CPU check: the HoleIndex allocator (include/cracsim/hole_index.hpp, as
// driven by DeviceContext::alloc/free) places and coalesces exactly like the
// reference allocator (linear first fit over an address-ordered std::map,
// ref: /root/reference/proj/src/device_core.cpp:45-103, restated below).
#include <cstdio>
#include <cstdlib>
#include <map>
#include <random>
#include <vector>

#include "cracsim/hole_index.hpp"

namespace {

struct RefAlloc {  // the reference's hole map
  std::map<uint64_t, uint64_t> holes;
  bool alloc(uint64_t need, uint64_t& addr) {
    auto it = holes.begin();
    for (; it != holes.end(); ++it)
      if (it->second >= need) break;
    if (it == holes.end()) return false;
    addr = it->first;
    const uint64_t len = it->second;
    holes.erase(it);
    if (len > need) holes.emplace(addr + need, len - need);
    return true;
  }
  void free(uint64_t addr, uint64_t len) {
    auto next = holes.lower_bound(addr);
    if (next != holes.end() && addr + len == next->first) {
      len += next->second;
      next = holes.erase(next);
    }
    if (next != holes.begin()) {
      auto prev = std::prev(next);
      if (prev->first + prev->second == addr) {
        addr = prev->first;
        len += prev->second;
        holes.erase(prev);
      }
    }
    holes.emplace(addr, len);
  }
};

struct IdxAlloc {  // DeviceContext's logic over HoleIndex
  cracsim::HoleIndex holes;
  bool alloc(uint64_t need, uint64_t& addr) {
    uint64_t len = 0;
    if (!holes.first_fit(need, addr, len)) return false;
    if (len > need)
      holes.update(addr, addr + need, len - need);
    else
      holes.erase(addr);
    return true;
  }
  void free(uint64_t addr, uint64_t len) {
    uint64_t next_len = 0, ps = 0, pl = 0;
    const bool next = holes.at(addr + len, next_len);
    const bool prev = holes.before(addr, ps, pl) && ps + pl == addr;
    if (prev && next) {
      holes.erase(addr + len);
      holes.update(ps, ps, pl + len + next_len);
    } else if (prev) {
      holes.update(ps, ps, pl + len);
    } else if (next) {
      holes.update(addr + len, addr, len + next_len);
    } else {
      holes.insert(addr, len);
    }
  }
};

struct FusedAlloc {  // the one-search forms DeviceContext uses since round 2
  cracsim::HoleIndex holes;
  bool alloc(uint64_t need, uint64_t& addr) {
    uint64_t len = 0;
    return holes.take_first_fit(need, addr, len);
  }
  void free(uint64_t addr, uint64_t len) { holes.release(addr, len); }
};

}  // namespace

int main(int argc, char** argv) {
  const int rounds = argc > 1 ? std::atoi(argv[1]) : 100;
  std::mt19937_64 rng(12345);
  for (int round = 0; round < rounds; ++round) {
    const uint64_t base = 0x0D0000000000ull, arena = 1ull << (20 + round % 6);
    RefAlloc ref;
    IdxAlloc idx;
    FusedAlloc fused;
    ref.holes.emplace(base, arena);
    idx.holes.insert(base, arena);
    fused.holes.insert(base, arena);
    std::vector<std::pair<uint64_t, uint64_t>> live;
    for (int op = 0; op < 4000; ++op) {
      if (!live.empty() && rng() % 100 < 40) {
        const size_t i = rng() % live.size();
        const auto [addr, len] = live[i];
        live.erase(live.begin() + long(i));
        ref.free(addr, len);
        idx.free(addr, len);
        fused.free(addr, len);
      } else {
        const uint64_t need = ((1 + rng() % 30000) + 255) / 256 * 256;
        uint64_t a = 0, b = 0, c = 0;
        const bool ra = ref.alloc(need, a), ib = idx.alloc(need, b), fc = fused.alloc(need, c);
        if (ra != ib || (ra && a != b) || ra != fc || (ra && a != c)) {
          std::printf("FAIL alloc round %d op %d\n", round, op);
          return 1;
        }
        if (ra) live.emplace_back(a, need);
      }
      std::vector<std::pair<uint64_t, uint64_t>> want(ref.holes.begin(), ref.holes.end()), got;
      idx.holes.for_each([&](uint64_t k, uint64_t v) { got.emplace_back(k, v); });
      std::vector<std::pair<uint64_t, uint64_t>> got2;
      fused.holes.for_each([&](uint64_t k, uint64_t v) { got2.emplace_back(k, v); });
      if (want != got || idx.holes.size() != want.size() || want != got2 ||
          fused.holes.size() != want.size()) {
        std::printf("FAIL holes round %d op %d\n", round, op);
        return 1;
      }
    }
  }
  std::printf("ok\n");
  return 0;
}
