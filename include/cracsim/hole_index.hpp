// Free-hole index of the arena allocator.
//
// The reference keeps holes in an address-ordered std::map and takes the
// first hole that fits by scanning it front to back (ref: src/device_core.cpp:
// 49-54), O(holes) per allocation — the cost that makes malloc-heavy restarts
// slow (3.6 s replay for 40 k calls).  This index answers the
// same question — the LOWEST-ADDRESS hole with length >= need — over
// address-ordered blocks of at most 16 holes that each keep their longest
// hole, and groups of 16 blocks that keep theirs: first fit skips every group
// and block that cannot fit and scans one block.  Lookups
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
      rebuild_groups();
      return;
    }
    const size_t b = block_at_or_before(addr);
    auto& h = blocks_[b];
    h.insert(std::upper_bound(h.begin(), h.end(), addr,
                              [](uint64_t a, const Hole& x) { return a < x.key; }),
             Hole{addr, len});
    first_[b] = h.front().key;
    if (len > max_[b]) set_max(b, len);
    if (h.size() > kMaxBlock) split(b);
  }

  void erase(uint64_t addr) {
    size_t b, i;
    if (!find(addr, b, i)) return;
    erase_at(b, i);
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
      set_max(b, new_len);
    else if (old == max_[b] && new_len < old)
      recompute(b);
  }

  // Lowest-address hole whose length is at least `need`.
  bool first_fit(uint64_t need, uint64_t& addr, uint64_t& len) const {
    for (size_t g = 0; g < gmax_.size(); ++g) {
      if (gmax_[g] < need) continue;
      const size_t end = std::min(max_.size(), (g + 1) * kGroup);
      for (size_t b = g * kGroup; b < end; ++b) {
        if (max_[b] < need) continue;
        for (const Hole& x : blocks_[b])
          if (x.len >= need) {
            addr = x.key;
            len = x.len;
            return true;
          }
      }
    }
    return false;
  }

  // First fit and its split in one pass (DeviceContext::alloc): the lowest-
  // address hole of length >= need gives its first `need` bytes; returns its
  // address (the rest stays a hole, or the hole goes).  One search, no
  // re-lookup by address.
  bool take_first_fit(uint64_t need, uint64_t& addr, uint64_t& hole_len) {
    for (size_t g = 0; g < gmax_.size(); ++g) {
      if (gmax_[g] < need) continue;
      const size_t end = std::min(max_.size(), (g + 1) * kGroup);
      for (size_t b = g * kGroup; b < end; ++b) {
        if (max_[b] < need) continue;
        auto& h = blocks_[b];
        for (size_t i = 0; i < h.size(); ++i) {
          if (h[i].len < need) continue;
          addr = h[i].key;
          hole_len = h[i].len;
          if (hole_len > need) {  // shrink in place: order is kept
            h[i].key += need;
            h[i].len -= need;
            if (i == 0) first_[b] = h[i].key;
            if (hole_len == max_[b]) recompute(b);
          } else {
            erase_at(b, i);
          }
          return true;
        }
      }
    }
    return false;
  }

  // Returns [addr, addr + len) with the two-sided coalesce of the reference
  // (ref: src/device_core.cpp:88-101) in one search (DeviceContext::free).
  void release(uint64_t addr, uint64_t len) {
    if (first_.empty()) {
      insert(addr, len);
      return;
    }
    const size_t b = block_at_or_before(addr);
    auto& h = blocks_[b];
    const size_t p = size_t(std::upper_bound(h.begin(), h.end(), addr,
                                             [](uint64_t a, const Hole& x) { return a < x.key; }) -
                            h.begin());
    // neighbours: (block, index) of the holes before and after addr
    const bool has_prev = p > 0 || b > 0;
    const size_t pb = p > 0 ? b : b - 1, pi = p > 0 ? p - 1 : (has_prev ? blocks_[pb].size() - 1 : 0);
    const bool has_next = p < h.size() || b + 1 < blocks_.size();
    const size_t nb = p < h.size() ? b : b + 1, ni = p < h.size() ? p : 0;
    const bool prev = has_prev && blocks_[pb][pi].key + blocks_[pb][pi].len == addr;
    const bool next = has_next && addr + len == blocks_[nb][ni].key;
    if (prev && next) {  // bridge: prev absorbs this extent and next
      Hole& x = blocks_[pb][pi];
      x.len += len + blocks_[nb][ni].len;
      const uint64_t grown = x.len;
      erase_at(nb, ni);  // (may remove block nb; pb < nb or pb == nb with pi < ni)
      if (grown > max_[pb]) set_max(pb, grown);
    } else if (prev) {
      Hole& x = blocks_[pb][pi];
      x.len += len;
      if (x.len > max_[pb]) set_max(pb, x.len);
    } else if (next) {
      Hole& x = blocks_[nb][ni];
      x.key = addr;
      x.len += len;
      if (ni == 0) first_[nb] = addr;
      if (x.len > max_[nb]) set_max(nb, x.len);
    } else {
      ++count_;
      h.insert(h.begin() + ptrdiff_t(p), Hole{addr, len});
      first_[b] = h.front().key;
      if (len > max_[b]) set_max(b, len);
      if (h.size() > kMaxBlock) split(b);
    }
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
  static constexpr size_t kMaxBlock = 16;  // holes per block
  static constexpr size_t kGroup = 16;     // blocks per group (a second level of maxima)

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

  void erase_at(size_t b, size_t i) {
    auto& h = blocks_[b];
    const uint64_t len = h[i].len;
    h.erase(h.begin() + ptrdiff_t(i));
    --count_;
    if (h.empty()) {
      blocks_.erase(blocks_.begin() + ptrdiff_t(b));
      first_.erase(first_.begin() + ptrdiff_t(b));
      max_.erase(max_.begin() + ptrdiff_t(b));
      rebuild_groups();
      return;
    }
    first_[b] = h.front().key;
    if (len == max_[b]) recompute(b);
  }

  void recompute(size_t b) {
    uint64_t m = 0;
    for (const Hole& x : blocks_[b]) m = x.len > m ? x.len : m;
    max_[b] = m;
    regroup(b / kGroup);
  }

  // a block's maximum grew: its group's can only grow with it
  void set_max(size_t b, uint64_t m) {
    max_[b] = m;
    if (m > gmax_[b / kGroup]) gmax_[b / kGroup] = m;
  }

  void regroup(size_t g) {
    uint64_t m = 0;
    const size_t end = std::min(max_.size(), (g + 1) * kGroup);
    for (size_t b = g * kGroup; b < end; ++b) m = max_[b] > m ? max_[b] : m;
    gmax_[g] = m;
  }

  // blocks were inserted or removed: group boundaries moved
  void rebuild_groups() {
    gmax_.assign((max_.size() + kGroup - 1) / kGroup, 0);
    for (size_t g = 0; g < gmax_.size(); ++g) regroup(g);
  }

  void split(size_t b) {
    auto& h = blocks_[b];
    std::vector<Hole> tail(h.begin() + ptrdiff_t(h.size() / 2), h.end());
    h.resize(h.size() / 2);
    blocks_.insert(blocks_.begin() + ptrdiff_t(b + 1), std::move(tail));
    first_.insert(first_.begin() + ptrdiff_t(b + 1), blocks_[b + 1].front().key);
    max_.insert(max_.begin() + ptrdiff_t(b + 1), 0);
    uint64_t m0 = 0, m1 = 0;
    for (const Hole& x : blocks_[b]) m0 = x.len > m0 ? x.len : m0;
    for (const Hole& x : blocks_[b + 1]) m1 = x.len > m1 ? x.len : m1;
    max_[b] = m0;
    max_[b + 1] = m1;
    rebuild_groups();
  }

  // Address-ordered holes in blocks of at most kMaxBlock; per block its first
  // key (binary search) and its longest hole (first-fit skips whole blocks).
  std::vector<std::vector<Hole>> blocks_;
  std::vector<uint64_t> first_, max_;
  std::vector<uint64_t> gmax_;  // per group of kGroup blocks: their longest hole
  size_t count_ = 0;
};

}  // namespace cracsim
