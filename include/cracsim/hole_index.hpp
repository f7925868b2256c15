// Free-hole index of the arena allocator.
//
// The reference keeps holes in an address-ordered std::map and takes the
// first hole that fits by scanning it front to back (ref: src/device_core.cpp:
// 49-54), O(holes) per allocation — the cost that makes malloc-heavy restarts
// slow (3.6 s replay for 40 k calls).  This index answers the
// same question — the LOWEST-ADDRESS hole with length >= need — over
// address-ordered blocks of at most 128 holes that each keep their longest
// hole: first fit skips every block that cannot fit and scans one.  Lookups
// by address are two binary searches, updates touch one small contiguous
// block (a pointer-chasing treap did the same in ~675 ns per allocator call;
// this layout is cache-resident).  Placement is bit-identical to the
// reference; only the search is faster.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <iterator>
#include <vector>

namespace cracsim {

class HoleIndex {
 public:
  void insert(uint64_t addr, uint64_t len) {
    ++count_;
    if (first_.empty()) {
      first_.push_back(addr);
      max_.push_back(len);
      blocks_.emplace_back(1, Hole{addr, len});
      return;
    }
    const size_t b = block_at_or_before(addr);
    auto& h = blocks_[b];
    h.insert(std::upper_bound(h.begin(), h.end(), addr,
                              [](uint64_t a, const Hole& x) { return a < x.key; }),
             Hole{addr, len});
    first_[b] = h.front().key;
    if (len > max_[b]) max_[b] = len;
    if (h.size() > kMaxBlock) split(b);
  }

  void erase(uint64_t addr) {
    size_t b, i;
    if (!find(addr, b, i)) return;
    auto& h = blocks_[b];
    const uint64_t len = h[i].len;
    h.erase(h.begin() + ptrdiff_t(i));
    --count_;
    if (h.empty()) {
      blocks_.erase(blocks_.begin() + ptrdiff_t(b));
      first_.erase(first_.begin() + ptrdiff_t(b));
      max_.erase(max_.begin() + ptrdiff_t(b));
      return;
    }
    first_[b] = h.front().key;
    if (len == max_[b]) recompute(b);
  }

  // Re-keys / resizes the hole starting at `addr` in place.  The caller
  // guarantees ordering is preserved (no other hole between the old and the
  // new start) — true for the allocator's split and merge steps, which only
  // move a hole's boundary inside the gap it already occupies.
  void update(uint64_t addr, uint64_t new_addr, uint64_t new_len) {
    size_t b, i;
    if (!find(addr, b, i)) return;
    Hole& x = blocks_[b][i];
    const uint64_t old = x.len;
    x.key = new_addr;
    x.len = new_len;
    if (i == 0) first_[b] = new_addr;
    if (new_len > max_[b])
      max_[b] = new_len;
    else if (old == max_[b] && new_len < old)
      recompute(b);
  }

  // Lowest-address hole whose length is at least `need`.
  bool first_fit(uint64_t need, uint64_t& addr, uint64_t& len) const {
    for (size_t b = 0; b < max_.size(); ++b) {
      if (max_[b] < need) continue;
      for (const Hole& x : blocks_[b])
        if (x.len >= need) {
          addr = x.key;
          len = x.len;
          return true;
        }
    }
    return false;
  }

  // Hole starting exactly at `addr`.
  bool at(uint64_t addr, uint64_t& len) const {
    size_t b, i;
    if (!find(addr, b, i)) return false;
    len = blocks_[b][i].len;
    return true;
  }

  // Hole with the greatest start strictly below `addr`.
  bool before(uint64_t addr, uint64_t& start, uint64_t& len) const {
    if (first_.empty() || first_[0] >= addr) return false;
    // last block whose first key < addr
    const size_t b = size_t(std::lower_bound(first_.begin(), first_.end(), addr) - first_.begin()) - 1;
    const auto& h = blocks_[b];
    const auto it = std::lower_bound(h.begin(), h.end(), addr,
                                     [](const Hole& x, uint64_t a) { return x.key < a; });
    start = std::prev(it)->key;
    len = std::prev(it)->len;
    return true;
  }

  // In-order (ascending address) visit.
  template <typename Fn>
  void for_each(Fn&& fn) const {
    for (const auto& h : blocks_)
      for (const Hole& x : h) fn(x.key, x.len);
  }

  size_t size() const { return count_; }

 private:
  struct Hole {
    uint64_t key, len;
  };
  static constexpr size_t kMaxBlock = 128;

  // Block whose range holds `addr`: the last block with first key <= addr
  // (block 0 when addr precedes every hole).
  size_t block_at_or_before(uint64_t addr) const {
    const size_t b = size_t(std::upper_bound(first_.begin(), first_.end(), addr) - first_.begin());
    return b ? b - 1 : 0;
  }

  bool find(uint64_t addr, size_t& b, size_t& i) const {
    if (first_.empty()) return false;
    b = block_at_or_before(addr);
    const auto& h = blocks_[b];
    const auto it = std::lower_bound(h.begin(), h.end(), addr,
                                     [](const Hole& x, uint64_t a) { return x.key < a; });
    if (it == h.end() || it->key != addr) return false;
    i = size_t(it - h.begin());
    return true;
  }

  void recompute(size_t b) {
    uint64_t m = 0;
    for (const Hole& x : blocks_[b]) m = x.len > m ? x.len : m;
    max_[b] = m;
  }

  void split(size_t b) {
    auto& h = blocks_[b];
    std::vector<Hole> tail(h.begin() + ptrdiff_t(h.size() / 2), h.end());
    h.resize(h.size() / 2);
    blocks_.insert(blocks_.begin() + ptrdiff_t(b + 1), std::move(tail));
    first_.insert(first_.begin() + ptrdiff_t(b + 1), blocks_[b + 1].front().key);
    max_.insert(max_.begin() + ptrdiff_t(b + 1), 0);
    recompute(b);
    recompute(b + 1);
  }

  // Address-ordered holes in blocks of at most kMaxBlock; per block its first
  // key (binary search) and its longest hole (first-fit skips whole blocks).
  std::vector<std::vector<Hole>> blocks_;
  std::vector<uint64_t> first_, max_;
  size_t count_ = 0;
};

}  // namespace cracsim
