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
#include <cstdlib>

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

// ---- slice runs: which slice size covers which bytes --------------------------
// A snapshot claims its warp tasks last task first, so the tasks it runs LAST
// are the first ones of the payload.  The head of the first region is cut
// into quarter-size slices: the final round of warp tasks is then 4x shorter
// and the launch's tail shrinks (N=1, 2.34 GB: 3024 -> 3112 GB/s,
// profiles/r2_head_split_1gpu.jsonl; a further 8-16 MiB of S/16 slices
// measured no gain, profiles/r2_fine_head_ab_1gpu.jsonl).  Everything that builds a job over a
// slot (snapshot, recovery, verify, plan) cuts the regions the same way, so
// the checksum table is entries of the head slices, then the rest of region
// 0 at the context's slice size, then the other regions.
constexpr uint64_t kHeadBytes = 48ull << 20;
constexpr int kRegionRuns = 2;  // runs per region, at most (head + rest)
inline uint64_t head_slice_bytes(uint64_t S) { return (S % 1024 == 0 && S >= 1024) ? S / 4 : 0; }
#ifdef FFX_DEV
// development builds: FFX_HEAD_MIB overrides the head size (every process of
// a run must agree -- the layout is not recorded in the slot)
inline uint64_t head_size() {
  static const uint64_t h = [] {
    const char* e = std::getenv("FFX_HEAD_MIB");
    return e ? static_cast<uint64_t>(std::strtoull(e, nullptr, 10)) << 20 : kHeadBytes;
  }();
  return h;
}
#else
inline uint64_t head_size() { return kHeadBytes; }
#endif
inline uint64_t head_bytes(uint64_t region0_bytes, uint64_t S) {
  const uint64_t h = head_size();
  return h && head_slice_bytes(S) && region0_bytes >= 4 * h ? h : 0;
}
struct SliceRun {
  uint64_t offset;  // within its region
  uint64_t bytes;
  uint64_t slice;   // slice size of this run
};
// The runs of one region (first = the first region of the payload); returns 1..kRegionRuns.
inline int region_runs(uint64_t bytes, uint64_t S, bool first, SliceRun out[kRegionRuns]) {
  const uint64_t h = first ? head_bytes(bytes, S) : 0;
  if (!h) {
    out[0] = SliceRun{0, bytes, S};
    return 1;
  }
  out[0] = SliceRun{0, h, head_slice_bytes(S)};
  out[1] = SliceRun{h, bytes - h, S};
  return 2;
}
inline uint64_t run_slices(const SliceRun& r) { return (r.bytes + r.slice - 1) / r.slice; }
// Region i of n gets the head when it is the first and a job region is left
// for it (a job holds at most kMaxRegions).
inline bool head_region(uint32_t i, uint32_t n) { return i == 0 && n + kRegionRuns - 1 <= kMaxRegions; }
// Checksum-table entries of a payload of n regions.
inline uint64_t table_entries(const uint64_t* region_bytes, uint32_t n, uint64_t S) {
  uint64_t e = 0;
  for (uint32_t i = 0; i < n; ++i) {
    SliceRun r[kRegionRuns];
    const int k = region_runs(region_bytes[i], S, head_region(i, n), r);
    for (int j = 0; j < k; ++j) e += run_slices(r[j]);
  }
  return e;
}

inline SlotLayout make_layout(uint64_t capacity, uint64_t slice_bytes) {
  SlotLayout L;
  L.payload_cap = align_up(capacity, kRegionAlign) + kMaxRegions * kRegionAlign;
  // a capacity-sized first region: its head runs' extra entries
  SliceRun r[kRegionRuns];
  const int k = region_runs(capacity, slice_bytes, true, r);
  uint64_t extra = 0;
  for (int j = 0; j + 1 < k; ++j) extra += r[j].bytes / r[j].slice - r[j].bytes / slice_bytes;
  L.table_cap = (capacity + slice_bytes - 1) / slice_bytes + kMaxRegions + extra;
  L.payload_off = align_up(kMetaBytes + 8 * L.table_cap + 32, 4096);
  L.slot_stride = align_up(L.payload_off + L.payload_cap, 1 << 21);
  return L;
}

}  // namespace ffx
