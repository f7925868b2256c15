// cracsim B200 build — foundation types shared by every layer.
//
// Drop-in for the reference's L0 headers (one file here, three there):
//   constants / kinds / records / mix64   ref: proj/include/cracsim/common.hpp:9-60
//   Errc / Error / raise                  ref: proj/include/cracsim/errors.hpp:8-60
//   ByteWriter / ByteReader (LE codec)    ref: proj/include/cracsim/bytes.hpp:16-84
// The forwarding headers common.hpp / errors.hpp / bytes.hpp include this one,
// so reference-side `#include "cracsim/common.hpp"` keeps compiling.
//
// B200 notes: addresses remain *logical* arena addresses (kArenaBase + offset);
// DeviceContext maps them onto a VMM reservation that sits at exactly that VA
// when the driver grants it (device_core.hpp), so the logged address is the
// device pointer the application dereferences.
#pragma once

#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace cracsim {

// ---- address-space and placement constants (common.hpp:9-12) --------------
inline constexpr uint64_t kArenaBase = 0x0D00'0000'0000ULL;
inline constexpr uint64_t kAlign = 256;
inline constexpr uint64_t kPageSize = 4096;
inline constexpr uint32_t kMaxStreams = 128;

enum class AllocationKind : uint8_t { Device = 1, PinnedHost = 2, Managed = 3 };
enum class PageSide : uint8_t { Host = 0, Device = 1 };
enum class AccessMode : uint8_t { Read = 0, Write = 1 };

constexpr const char* allocation_kind_name(AllocationKind k) {
  return k == AllocationKind::Device       ? "device"
         : k == AllocationKind::PinnedHost ? "pinned"
         : k == AllocationKind::Managed    ? "managed"
                                           : "?";
}

struct BufferRef {
  uint64_t id = 0;      // allocation id
  uint64_t offset = 0;  // byte offset into it
};

struct AllocationRecord {
  uint64_t id = 0;
  AllocationKind kind = AllocationKind::Device;
  uint64_t size = 0;     // requested bytes (the image stores exactly these)
  uint64_t address = 0;  // logical arena address; extent = round_up_align(size)
  bool freed = false;
  bool operator==(const AllocationRecord&) const = default;
};

inline constexpr uint64_t round_up_align(uint64_t n) { return (n + kAlign - 1) & ~(kAlign - 1); }
inline constexpr uint64_t page_count_for(uint64_t n) { return (n + kPageSize - 1) / kPageSize; }

// splitmix64 finalizer (common.hpp:55-60); also the synthetic-content source.
inline constexpr uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// ---- error model (errors.hpp:8-60) ------------------------------------------
// Codes 0..15 keep the reference's order (the C-ABI returns 1 + code).
// DeviceFault is new: a CUDA runtime/driver failure underneath the engine.
enum class Errc {
  InvalidArgument,
  OutOfArena,
  DoubleFree,
  UnknownId,
  StreamLimitExceeded,
  BusyStream,
  UnregisteredKernel,
  DuplicateKernelId,
  OutOfRange,
  NotManaged,
  HalfConflict,
  QuiesceTimeout,
  ReplayDivergence,
  ImageCorrupt,
  UnknownKernelBody,
  DivisionByZero,
  DeviceFault,
};

constexpr const char* errc_name(Errc c) {
  constexpr const char* names[] = {
      "InvalidArgument",  "OutOfArena",        "DoubleFree",   "UnknownId",
      "StreamLimitExceeded", "BusyStream",     "UnregisteredKernel", "DuplicateKernelId",
      "OutOfRange",       "NotManaged",        "HalfConflict", "QuiesceTimeout",
      "ReplayDivergence", "ImageCorrupt",      "UnknownKernelBody", "DivisionByZero",
      "DeviceFault"};
  const auto i = static_cast<unsigned>(c);
  return i < sizeof(names) / sizeof(names[0]) ? names[i] : "Unknown";
}

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what)
      : std::runtime_error(std::string(errc_name(code)) + ": " + what), code_(code) {}
  Errc code() const noexcept { return code_; }

 private:
  Errc code_;
};

[[noreturn]] inline void raise(Errc code, const std::string& what) { throw Error(code, what); }

// ---- little-endian codec (bytes.hpp:16-84) ----------------------------------
// Host byte order is asserted little-endian at build time (x86-64 / aarch64),
// so fixed-width fields are written with one memcpy instead of byte loops.
static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "little-endian host required");

class ByteWriter {
 public:
  void u8(uint8_t v) { put(&v, 1); }
  void u16(uint16_t v) { put(&v, 2); }
  void u32(uint32_t v) { put(&v, 4); }
  void u64(uint64_t v) { put(&v, 8); }
  void bytes(std::span<const uint8_t> b) { put(b.data(), b.size()); }
  void str(const std::string& s) {
    u32(static_cast<uint32_t>(s.size()));
    put(s.data(), s.size());
  }
  const std::vector<uint8_t>& data() const { return out_; }
  std::vector<uint8_t> take() { return std::move(out_); }
  size_t size() const { return out_.size(); }

 private:
  void put(const void* p, size_t n) {
    const size_t at = out_.size();
    out_.resize(at + n);
    if (n) std::memcpy(out_.data() + at, p, n);
  }
  std::vector<uint8_t> out_;
};

class ByteReader {
 public:
  ByteReader(std::span<const uint8_t> in, Errc on_underrun) : in_(in), err_(on_underrun) {}
  uint8_t u8() { return get<uint8_t>(); }
  uint16_t u16() { return get<uint16_t>(); }
  uint32_t u32() { return get<uint32_t>(); }
  uint64_t u64() { return get<uint64_t>(); }
  std::span<const uint8_t> bytes(size_t n) {
    require(n);
    auto s = in_.subspan(at_, n);
    at_ += n;
    return s;
  }
  std::string str() {
    const uint32_t n = u32();
    auto b = bytes(n);
    return std::string(reinterpret_cast<const char*>(b.data()), b.size());
  }
  size_t remaining() const { return in_.size() - at_; }
  size_t position() const { return at_; }
  bool done() const { return at_ == in_.size(); }

 private:
  template <typename T>
  T get() {
    require(sizeof(T));
    T v;
    std::memcpy(&v, in_.data() + at_, sizeof(T));
    at_ += sizeof(T);
    return v;
  }
  void require(size_t n) {
    if (in_.size() - at_ < n) raise(err_, "truncated input");
  }
  std::span<const uint8_t> in_;
  size_t at_ = 0;
  Errc err_;
};

}  // namespace cracsim
