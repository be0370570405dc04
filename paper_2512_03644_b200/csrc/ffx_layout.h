// ffx_layout.h -- HBM layout of a neighbour replica (host + device).
//
// A replica is one cudaMalloc'd (IPC-exportable) allocation on the holder GPU
// holding `versions` slots for one origin rank (reference NeighborBuffer keeps
// two: ckpt.cpp:86-92).  Slot layout, all offsets from the slot base:
//
//   [0, 256)                 SlotMeta (state, iteration, role, sizes, region table)
//   [256, 256 + 8*S)         per-slice FNV-1a-64 table, S = table capacity
//   [P - 32, P)              SNP1 header (storage.hpp:12-25), P = payload offset
//   [P, P + payload_cap)     payload: unique regions at 256-byte aligned offsets
//
// P is 4096-aligned, so header+payload of a single-region slot is byte-for-byte
// the reference's framed blob (pack_blob, storage.cpp:45-66) once the header's
// whole-payload checksum is filled in on export.
#pragma once

#include <cstdint>

namespace ffx {

constexpr uint32_t kSlotMagic = 0x52584646u;  // "FFXR"
constexpr uint32_t kSlotEmpty = 0, kSlotWriting = 1, kSlotCommitted = 2;
constexpr uint32_t kMaxRegions = 16;
constexpr uint64_t kRegionAlign = 256;
constexpr uint64_t kMetaBytes = 256;

struct SlotMeta {  // exactly 256 bytes
  uint32_t magic;
  uint32_t state;
  uint64_t iteration;
  uint64_t seq;          // write sequence, larger = newer
  uint64_t payload_len;  // logical bytes (regions concatenated)
  uint64_t slice_bytes;
  uint64_t num_slices;
  uint64_t whole_checksum;
  uint16_t dp, pp, tp;
  uint8_t kind;
  uint8_t whole_checksum_valid;
  uint32_t num_regions;
  uint32_t reserved0;
  uint64_t region_bytes[kMaxRegions];  // 128 bytes
  uint8_t region_kinds[kMaxRegions];   // ffx_region_kind of each region (a replacement allocates from these)
  uint64_t reserved[5];
};
static_assert(sizeof(SlotMeta) == kMetaBytes, "SlotMeta must be 256 bytes");

struct SlotLayout {
  uint64_t payload_cap;  // bytes reserved for the payload (incl. region padding)
  uint64_t table_cap;    // checksum table entries
  uint64_t payload_off;  // P
  uint64_t slot_stride;  // bytes per slot
};

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

inline SlotLayout make_layout(uint64_t capacity, uint64_t slice_bytes) {
  SlotLayout L;
  L.payload_cap = align_up(capacity, kRegionAlign) + kMaxRegions * kRegionAlign;
  L.table_cap = (capacity + slice_bytes - 1) / slice_bytes + kMaxRegions;
  L.payload_off = align_up(kMetaBytes + 8 * L.table_cap + 32, 4096);
  L.slot_stride = align_up(L.payload_off + L.payload_cap, 1 << 21);
  return L;
}

}  // namespace ffx
