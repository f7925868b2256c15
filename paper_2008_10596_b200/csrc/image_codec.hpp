// Internal image codec shared by the value-type API (encode_image /
// decode_image) and the B200 fast paths (checkpoint_image / restart_image).
// The strict parse restates the reference's validation rules
// (ref: src/image.cpp:108-345) and additionally returns byte offsets of every
// framed record so the refill can stream payloads straight from the image.
#pragma once

#include <array>

#include "cracsim/image.hpp"

namespace cracsim::codec {

// CRC-32/IEEE of a host buffer (small sections only; bulk sections are
// hashed on the GPU).
uint32_t crc32_host(const uint8_t* p, size_t n, uint32_t crc = 0);
// zlib-identical CRC-32 by carry-less multiplication (crc_host.cpp), ~12 GB/s
// per core against zlib's 2.6; zlib below 64 bytes or without PCLMUL.
uint32_t crc32_fast(const uint8_t* p, size_t n, uint32_t crc = 0);
// crc32_fast of src that also copies src to dst (non-temporal stores when dst
// is 16-byte aligned: no read-for-ownership of the destination); the caller
// runs stream_fence() before another agent may read dst
uint32_t crc32_copy_stream(uint8_t* dst, const uint8_t* src, size_t n, uint32_t crc = 0);
void stream_fence();

std::vector<uint8_t> meta_bytes(const SnapshotMeta& m);
std::vector<uint8_t> log_bytes(std::span<const CallLogEntry> log);
// The LOG payload encoded straight into `dst` (kLogRecordBytes per entry).
void encode_log_into(uint8_t* dst, std::span<const CallLogEntry> log);
std::vector<uint8_t> streams_bytes(std::span<const uint64_t> streams);
std::vector<uint8_t> registry_bytes(std::span<const BinaryInfo> binaries);

struct LogFacts {
  std::vector<AllocationRecord> active;  // ascending id
  std::vector<uint64_t> live_streams;    // ascending
  std::vector<uint64_t> live_handles;    // ascending
};

struct SectionView {
  uint64_t payload_off = 0;  // file offset of the payload
  uint64_t length = 0;
  uint32_t crc = 0;          // stored value
};

struct PayloadFrame {
  uint64_t id = 0;
  uint64_t len = 0;
  uint64_t frame_off = 0;  // offset of the 16-byte frame inside the section payload
};

struct ManagedFrame {
  uint64_t id = 0;
  uint64_t size = 0;
  uint64_t frame_off = 0;       // offset of the 16-byte (id, pages) header
  std::vector<uint8_t> flags;   // per page: bit0 device_resident, bit1 dirty
};

struct ParsedImage {
  uint32_t version = 0;
  std::array<SectionView, kSectionCount> sec{};
  SnapshotMeta meta;
  std::vector<CallLogEntry> log;
  LogFacts facts;
  std::vector<uint64_t> streams;
  std::vector<uint8_t> app_state;
  std::vector<BinaryInfo> binaries;
  std::vector<PayloadFrame> payloads;
  std::vector<ManagedFrame> managed;
  uint64_t payload_bytes = 0;
  uint64_t uvm_page_bytes = 0;
  uint64_t file_bytes = 0;
};

// Strict parse of an uncompressed image.  verify_bulk = false defers the CRC
// of sections 3 and 4 to the caller (the GPU refill verifies them).
ParsedImage parse_image(std::span<const uint8_t> raw, bool verify_bulk);

// Returns the raw image (inflating a CRACSIMZ wrapper into `storage`).
std::span<const uint8_t> unwrap(std::span<const uint8_t> bytes, std::vector<uint8_t>& storage,
                                bool* was_compressed);

}  // namespace cracsim::codec
