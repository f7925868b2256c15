// Free-hole index of the arena allocator.
//
// The reference keeps holes in an address-ordered std::map and takes the
// first hole that fits by scanning it front to back (ref: src/device_core.cpp:
// 49-54), O(holes) per allocation — the cost that makes malloc-heavy restarts
// slow (3.6 s replay for 40 k calls).  This index answers the
// same question — the LOWEST-ADDRESS hole with length >= need — in O(log n):
// a treap keyed by address where every node also stores the largest hole
// length in its subtree.  Placement is therefore bit-identical to the
// reference; only the search is faster.
#pragma once

#include <cstdint>
#include <vector>

namespace cracsim {

class HoleIndex {
 public:
  void insert(uint64_t addr, uint64_t len) {
    int a, b;
    split(root_, addr, a, b);
    root_ = merge(merge(a, make(addr, len)), b);
  }

  void erase(uint64_t addr) {
    int a, b, m, c;
    split(root_, addr, a, b);
    split(b, addr + 1, m, c);
    if (m >= 0) release(m);
    root_ = merge(a, c);
  }

  // Re-keys / resizes the hole starting at `addr` in place.  The caller
  // guarantees ordering is preserved (no other hole between the old and the
  // new start) — true for the allocator's split and merge steps, which only
  // move a hole's boundary inside the gap it already occupies.
  void update(uint64_t addr, uint64_t new_addr, uint64_t new_len) {
    int path[128];
    int depth = 0;
    for (int t = root_; t >= 0;) {
      if (depth == 128) {  // pathological depth: fall back to erase + insert
        erase(addr);
        insert(new_addr, new_len);
        return;
      }
      path[depth++] = t;
      Node& n = nodes_[t];
      if (n.key == addr) {
        n.key = new_addr;
        n.len = new_len;
        while (depth) pull(path[--depth]);
        return;
      }
      t = addr < n.key ? n.l : n.r;
    }
  }

  // Lowest-address hole whose length is at least `need`.
  bool first_fit(uint64_t need, uint64_t& addr, uint64_t& len) const {
    int t = root_;
    if (t < 0 || nodes_[t].maxlen < need) return false;
    for (;;) {
      const Node& n = nodes_[t];
      if (n.l >= 0 && nodes_[n.l].maxlen >= need) {
        t = n.l;
      } else if (n.len >= need) {
        addr = n.key;
        len = n.len;
        return true;
      } else {
        t = n.r;
      }
    }
  }

  // Hole starting exactly at `addr`.
  bool at(uint64_t addr, uint64_t& len) const {
    for (int t = root_; t >= 0;) {
      const Node& n = nodes_[t];
      if (n.key == addr) {
        len = n.len;
        return true;
      }
      t = addr < n.key ? n.l : n.r;
    }
    return false;
  }

  // Hole with the greatest start strictly below `addr`.
  bool before(uint64_t addr, uint64_t& start, uint64_t& len) const {
    bool found = false;
    for (int t = root_; t >= 0;) {
      const Node& n = nodes_[t];
      if (n.key < addr) {
        start = n.key;
        len = n.len;
        found = true;
        t = n.r;
      } else {
        t = n.l;
      }
    }
    return found;
  }

  // In-order (ascending address) visit.
  template <typename Fn>
  void for_each(Fn&& fn) const {
    std::vector<int> stack;
    for (int t = root_; t >= 0 || !stack.empty();) {
      while (t >= 0) {
        stack.push_back(t);
        t = nodes_[t].l;
      }
      t = stack.back();
      stack.pop_back();
      fn(nodes_[t].key, nodes_[t].len);
      t = nodes_[t].r;
    }
  }

  size_t size() const { return nodes_.size() - free_.size(); }

 private:
  struct Node {
    uint64_t key, len, maxlen;
    uint32_t pri;
    int l, r;
  };

  int make(uint64_t key, uint64_t len) {
    rng_ ^= rng_ << 13;
    rng_ ^= rng_ >> 7;
    rng_ ^= rng_ << 17;
    const Node n{key, len, len, uint32_t(rng_ >> 32), -1, -1};
    if (!free_.empty()) {
      const int i = free_.back();
      free_.pop_back();
      nodes_[i] = n;
      return i;
    }
    nodes_.push_back(n);
    return int(nodes_.size() - 1);
  }

  void release(int t) {
    if (t < 0) return;
    release(nodes_[t].l);
    release(nodes_[t].r);
    free_.push_back(t);
  }

  void pull(int t) {
    Node& n = nodes_[t];
    n.maxlen = n.len;
    if (n.l >= 0 && nodes_[n.l].maxlen > n.maxlen) n.maxlen = nodes_[n.l].maxlen;
    if (n.r >= 0 && nodes_[n.r].maxlen > n.maxlen) n.maxlen = nodes_[n.r].maxlen;
  }

  // a: keys < key, b: keys >= key
  void split(int t, uint64_t key, int& a, int& b) {
    if (t < 0) {
      a = b = -1;
      return;
    }
    if (nodes_[t].key < key) {
      split(nodes_[t].r, key, nodes_[t].r, b);
      a = t;
    } else {
      split(nodes_[t].l, key, a, nodes_[t].l);
      b = t;
    }
    pull(t);
  }

  int merge(int a, int b) {
    if (a < 0) return b;
    if (b < 0) return a;
    if (nodes_[a].pri > nodes_[b].pri) {
      nodes_[a].r = merge(nodes_[a].r, b);
      pull(a);
      return a;
    }
    nodes_[b].l = merge(a, nodes_[b].l);
    pull(b);
    return b;
  }

  std::vector<Node> nodes_;
  std::vector<int> free_;
  int root_ = -1;
  uint64_t rng_ = 0x9E3779B97F4A7C15ull;
};

}  // namespace cracsim
