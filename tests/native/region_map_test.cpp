// CPU check: RegionMap (csrc/shim.cpp, a start-sorted vector) keeps the
// reference's region-table contract (ref: /root/reference/proj/src/shim.cpp:
// 42-88): the reference's own cases (tests/test_shim.cpp:214-263) restated,
// then random register / classify sequences against a restatement of its
// algorithm (an address-keyed std::map swept from the region before `start`)
// — same regions, same Errc, same classification after every call.
#include <cstdio>
#include <cstdlib>
#include <map>
#include <optional>
#include <random>
#include <vector>

#include "cracsim/shim.hpp"

using namespace cracsim;

namespace {

int failures = 0;
#define EXPECT(c)                                               \
  do {                                                          \
    if (!(c)) {                                                 \
      std::printf("FAIL %s at line %d\n", #c, __LINE__);        \
      ++failures;                                               \
    }                                                           \
  } while (0)

template <typename Fn>
std::optional<Errc> errc_of(Fn&& fn) {
  try {
    fn();
  } catch (const Error& e) {
    return e.code();
  }
  return std::nullopt;
}

struct RefRegions {  // the reference's table, restated
  std::map<uint64_t, Region> m;
  std::optional<Errc> add(uint64_t start, uint64_t length, Half half, uint8_t perms) {
    if (length == 0) return Errc::InvalidArgument;
    const uint64_t end = start + length;
    uint64_t lo = start, hi = end;
    std::vector<uint64_t> gone;
    auto it = m.lower_bound(start);
    if (it != m.begin()) --it;
    for (; it != m.end() && it->first <= end; ++it) {
      const Region& r = it->second;
      const uint64_t r_end = r.start + r.length;
      const bool overlap = r.start < end && start < r_end;
      const bool touch = r_end == start || r.start == end;
      if (overlap && r.half != half) return Errc::HalfConflict;
      if (overlap && r.perms != perms) return Errc::InvalidArgument;
      if ((overlap || touch) && r.half == half && r.perms == perms) {
        lo = std::min(lo, r.start);
        hi = std::max(hi, r_end);
        gone.push_back(r.start);
      }
    }
    for (uint64_t k : gone) m.erase(k);
    m.emplace(lo, Region{lo, hi - lo, half, perms});
    return std::nullopt;
  }
  Classification classify(uint64_t a) const {
    auto it = m.upper_bound(a);
    if (it == m.begin()) return Classification::Unmapped;
    const Region& r = std::prev(it)->second;
    if (a >= r.start + r.length) return Classification::Unmapped;
    return r.half == Half::Upper ? Classification::Upper : Classification::Lower;
  }
  std::vector<Region> regions() const {
    std::vector<Region> v;
    for (const auto& kv : m) v.push_back(kv.second);
    return v;
  }
};

void reference_cases() {
  constexpr uint8_t RW = kPermRead | kPermWrite;
  auto base = [&](RegionMap& map) {
    map.register_range(0x1000, 0x1000, Half::Upper, RW);
    map.register_range(0x2000, 0x1000, Half::Upper, RW);
  };
  {
    RegionMap map;
    base(map);
    const auto r = map.regions();
    EXPECT(r.size() == 1 && r[0] == (Region{0x1000, 0x2000, Half::Upper, RW}));
  }
  {  // overlap with identical permissions merges to the union
    RegionMap map;
    base(map);
    map.register_range(0x1800, 0x2000, Half::Upper, RW);
    const auto r = map.regions();
    EXPECT(r.size() == 1 && r[0].start == 0x1000 && r[0].length == 0x2800);
  }
  {  // different permissions stay separate when disjoint
    RegionMap map;
    base(map);
    map.register_range(0x4000, 0x1000, Half::Upper, kPermRead);
    EXPECT(map.regions().size() == 2);
  }
  {  // different permissions may not overlap
    RegionMap map;
    base(map);
    EXPECT(errc_of([&] { map.register_range(0x2800, 0x1000, Half::Upper, kPermRead); }) ==
           Errc::InvalidArgument);
  }
  {  // the other half may not overlap
    RegionMap map;
    base(map);
    EXPECT(errc_of([&] { map.register_range(0x2f00, 0x1000, Half::Lower, RW); }) ==
           Errc::HalfConflict);
  }
  {  // classification
    RegionMap map;
    map.register_range(0x10000, 0x1000, Half::Upper, RW);
    EXPECT(map.classify(0x10000) == Classification::Upper);
    EXPECT(map.classify(0x10fff) == Classification::Upper);
    EXPECT(map.classify(0x11000) == Classification::Unmapped);
    EXPECT(map.classify(0x500) == Classification::Unmapped);
    EXPECT(errc_of([&] { map.register_range(0x20000, 0, Half::Upper, RW); }) ==
           Errc::InvalidArgument);
  }
  {  // a differing neighbour on each side survives a bridging merge
    RegionMap map;
    map.register_range(0x1000, 0x1000, Half::Lower, RW);
    map.register_range(0x2000, 0x1000, Half::Upper, RW);
    map.register_range(0x4000, 0x1000, Half::Upper, RW);
    map.register_range(0x5000, 0x1000, Half::Upper, kPermRead);
    map.register_range(0x3000, 0x1000, Half::Upper, RW);
    const auto r = map.regions();
    EXPECT(r.size() == 3 && r[1] == (Region{0x2000, 0x3000, Half::Upper, RW}));
  }
}

void random_against_reference(int rounds) {
  std::mt19937_64 rng(11);
  for (int round = 0; round < rounds; ++round) {
    RegionMap map;
    RefRegions ref;
    const uint64_t space = 64 + rng() % 512;  // small: many overlaps and touches
    for (int op = 0; op < 400; ++op) {
      const uint64_t start = rng() % space, length = rng() % 24 == 0 ? 0 : 1 + rng() % 24;
      const Half half = rng() % 5 == 0 ? Half::Lower : Half::Upper;
      const uint8_t perms = rng() % 4 == 0 ? kPermRead : uint8_t(kPermRead | kPermWrite);
      const auto want = ref.add(start, length, half, perms);
      const auto got = errc_of([&] { map.register_range(start, length, half, perms); });
      EXPECT(got == want);
      EXPECT(map.regions() == ref.regions());
      for (int q = 0; q < 4; ++q) {
        const uint64_t a = rng() % (space + 32);
        EXPECT(map.classify(a) == ref.classify(a));
      }
      if (failures) {
        std::printf("round %d op %d: [%llu, +%llu) half %d perms %d\n", round, op,
                    (unsigned long long)start, (unsigned long long)length, int(half), int(perms));
        for (const Region& r : map.regions())
          std::printf("  got  [%llu, %llu) %d %d\n", (unsigned long long)r.start,
                      (unsigned long long)(r.start + r.length), int(r.half), int(r.perms));
        for (const Region& r : ref.regions())
          std::printf("  want [%llu, %llu) %d %d\n", (unsigned long long)r.start,
                      (unsigned long long)(r.start + r.length), int(r.half), int(r.perms));
        return;
      }
    }
  }
}

}  // namespace

int main(int argc, char** argv) {
  reference_cases();
  random_against_reference(argc > 1 ? std::atoi(argv[1]) : 200);
  if (failures) return 1;
  std::printf("ok\n");
  return 0;
}
