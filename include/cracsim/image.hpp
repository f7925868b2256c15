// cracsim B200 build — the CRACSIM1 checkpoint image (format contract).
//
// Byte-identical to the reference format (ref: include/cracsim/image.hpp:11-91,
// docs/image_format.md): LE integers, magic "CRACSIM1", version 1, seven
// sections tag 1..7 each framed {tag u32, reserved u32 = 0, length u64,
// payload, crc32 u32}; file size = 16 + sum(16 + length + 4).
// decode is strict and all-or-nothing (ImageCorrupt).
#pragma once

#include <filesystem>

#include "cracsim/snapshot.hpp"

namespace cracsim {

inline constexpr char kImageMagic[8] = {'C', 'R', 'A', 'C', 'S', 'I', 'M', '1'};
inline constexpr char kCompressedMagic[8] = {'C', 'R', 'A', 'C', 'S', 'I', 'M', 'Z'};
inline constexpr uint32_t kImageVersion = 1;
inline constexpr uint32_t kSectionCount = 7;
inline constexpr size_t kLogRecordBytes = 36;  // seq u64 op u8 kind u8 pad u16 size u64 id u64 addr u64

enum class SectionTag : uint32_t {
  Meta = 1,
  Log = 2,
  AllocPayloads = 3,
  UvmPages = 4,
  Streams = 5,
  AppState = 6,
  KernelRegistry = 7,
};

constexpr const char* section_tag_name(SectionTag t) {
  constexpr const char* names[] = {"?",         "META",    "LOG",     "ALLOC_PAYLOADS",
                                   "UVM_PAGES", "STREAMS", "APPSTATE", "KERNEL_REGISTRY"};
  const auto i = static_cast<uint32_t>(t);
  return i < 8 ? names[i] : "?";
}

std::vector<uint8_t> encode_image(const Snapshot& snapshot);
Snapshot decode_image(std::span<const uint8_t> bytes);

std::vector<uint8_t> compress_image(std::span<const uint8_t> image);
bool is_compressed_image(std::span<const uint8_t> bytes);

struct SectionSummary {
  SectionTag tag;
  uint64_t length = 0;
  uint32_t crc = 0;
};

struct ImageSummary {
  uint32_t version = 0;
  bool was_compressed = false;
  std::vector<SectionSummary> sections;
  uint64_t log_entries = 0;
  uint64_t active_allocations = 0;
  uint64_t payload_bytes = 0;
  uint64_t uvm_page_bytes = 0;
  uint64_t file_bytes = 0;
};

ImageSummary summarize_image(std::span<const uint8_t> bytes);

void write_image_file(const std::filesystem::path& path, const Snapshot& snapshot,
                      bool compress = false);
Snapshot read_image_file(const std::filesystem::path& path);
std::vector<uint8_t> read_file_bytes(const std::filesystem::path& path);

}  // namespace cracsim
