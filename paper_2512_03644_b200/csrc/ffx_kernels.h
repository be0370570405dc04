// ffx_kernels.h -- host-side launchers for the sm_100a kernels in
// ffx_kernels.cu.  Internal to libffx.so; the public boundary is include/ffx.h.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "ffx_layout.h"

namespace ffx {

// One contiguous range moved and/or hashed slice by slice.  Slices restart at
// every region: slice s of region r covers [s*S, min((s+1)*S, bytes)).
struct SliceRegion {
  const uint8_t* src;
  uint8_t* dst;          // null in hash-only mode
  uint64_t bytes;
  uint64_t slice_base;   // first checksum-table index of this region
  uint64_t group_base;   // first 32-slice warp task of this region
  int32_t tmap;          // index of this region's src/dst tensor-map pair, -1 = none
  uint32_t slice_bytes;  // this region's slice size (0 = the job's)
  uint64_t nfull;        // full-length slices (the tensor maps' outer extent)
  uint8_t* dst2;         // second replica (double-neighbour), null = none
  const uint64_t* expected;  // verify: this region's own table (region-local index), else the job's
};

// regions that get TMA tensor maps per launch (the largest ones): a Llama-3
// ZeRO-3 shard is 4 large regions + the first one's head run, a two-source
// gather twice that; 8 x 3 maps make the job a 5 KB kernel parameter
// (CUDA >= 12.1 allows 32 KB)
constexpr int kTmaRegions = 8;

// Optional slot commit fused into the snapshot kernel: every CTA marks the
// slot WRITING before its first payload store; the last CTA to finish writes
// the final meta + SNP1 header and flips the state to COMMITTED.
struct SlotCommit {
  uint8_t* slot;             // slot base (peer-mapped or local); null = no commit
  unsigned int* done;        // local completion counter (zero between launches)
  uint32_t finalize;         // this launch is the last batch of the snapshot
  uint32_t mcast;            // slot is written through a multicast range (multimem.st metadata)
  uint64_t payload_off;      // SNP1 header lives at slot + payload_off - 32
  uint64_t iteration, seq;
  uint4 meta[kMetaBytes / 16];  // final SlotMeta image (state field = COMMITTED)
  uint4 snp1[2];                // SNP1 header image
  uint64_t* ack;                // pull mode: origin's word set to ack_value after commit
  uint64_t ack_value;
};

struct SliceJob {
  // [3*i] = source, [3*i+1] = destination of tensor-mapped region i: a 2-D
  // view {slice_bytes, nfull} with row pitch slice_bytes, 128 x 32 boxes,
  // 128-byte swizzle (conflict-free per-lane row reads).
  // [3*i+2] = second destination (double-neighbour replication).
  CUtensorMap maps[3 * kTmaRegions];
  SliceRegion reg[kMaxRegions];
  uint32_t nregions;
  uint32_t rows;                  // slices per warp task (32 or 64; set by finalize_job)
  uint64_t total_groups;
  uint64_t group_lo, group_hi;  // warp tasks this launch covers (a scheduler batch)
  uint64_t slice_bytes;
  uint64_t* sums_out;             // may be null
  uint64_t* sums_out2;            // second replica's table (double-neighbour), may be null
  const uint64_t* sums_expected;  // verify mode
  const uint64_t* init_state;     // per-slice FNV start (null = offset basis)
  unsigned long long* result;     // verify mode: [first bad slice, bad count]
  unsigned int* sched;            // [next task, CTAs done]: dynamic scheduling
                                  // (zero between launches; null = static)
  uint32_t proxy_fence;           // tensor path: generic->async proxy fence before each refill
  uint32_t stagger_ns;            // start-up de-phasing: warp w sleeps (w % 8) * stagger_ns first
  uint32_t claim_order;           // 0: last task first, then backwards; 1: last task first, then forwards
  uint32_t store_hint;            // tensor stores with an L2 evict_first hint (experiment)
  uint32_t prefetch_next;         // tensor path: claim the next task S steps early and load its
                                  // first S steps into the stages this task frees (no per-task drain)
  uint32_t one_shot;              // one task per warp, no claim loop (task-granular batches)
  uint32_t l2_stream;             // TMA loads / stores with an L2 evict_first policy
  uint32_t static_first;          // each warp's first task is blockIdx*W+warp (no atomic), then dynamic
  uint32_t skip_begin;            // the slot was marked WRITING by a preceding mark launch
  SlotCommit commit;
  SlotCommit commit2;             // second replica's slot (slot null = none)
};

enum class SliceMode { Hash, Copy, CopyVerify, HashVerify };

// ---- copy-only TMA batches (split scheduling policy, ffx_copy.cu) ----------

struct CopyRegion {
  const uint8_t* src;
  uint8_t* dst;
  uint64_t bytes;
  uint32_t aligned;  // all pointers 16-byte aligned (set by finalize_copy_job)
  uint32_t pad_;
  uint8_t* dst2;     // second replica (double-neighbour), null = none
};

struct SlotMark {  // every copy CTA marks the slot WRITING first
  uint8_t* slot;   // null = no mark
  uint64_t iteration, seq;
  uint32_t mcast;  // through a multicast range (multimem.st)
  uint32_t pad_;
};

struct CopyJob {
  CopyRegion reg[kMaxRegions];
  uint64_t chunk_base[kMaxRegions];
  uint32_t nregions;
  uint32_t pad_;
  uint64_t total_chunks;
  uint64_t chunk_lo, chunk_hi;  // this launch's 32 KB chunks
  SlotMark mark;
  SlotMark mark2;
};

void finalize_copy_job(CopyJob& job);
cudaError_t launch_copy(const CopyJob& job, uint32_t ctas, cudaStream_t stream);
// One-thread kernel writing the final meta + SNP1 header, then COMMITTED.
cudaError_t launch_commit(const SlotCommit& c, cudaStream_t stream);
// One-warp kernel marking the slot(s) of c (and c2) WRITING.
cudaError_t launch_mark(const SlotCommit& c, const SlotCommit* c2, cudaStream_t stream);

// Slices per warp task.  Two kernel configurations ship (ffx_slice.cu):
// kBulkRows (32 slices, one chain per lane: the full-GPU, HBM/NVLink-bound
// launches) and kCappedRows (64 slices, two chains per lane, 8 warps per
// CTA: CTA-capped scheduler batches, where SM time per byte is the cost).
constexpr uint32_t kBulkRows = 32, kCappedRows = 64;
// Default rows for a launch with at most max_ctas CTAs (0 = whole GPU).
uint32_t rows_for_cap(uint32_t max_ctas);

// Fill job.reg[*].group_base / slice_base, job.total_groups and the group
// range [0, total_groups) for `rows` slices per task (0 = kBulkRows).
void finalize_job(SliceJob& job, uint32_t rows = 0);
// Launch with at most max_ctas CTAs (0 = occupancy-sized full grid).
cudaError_t launch_slices(const SliceJob& job, SliceMode mode, bool commit, uint32_t max_ctas,
                          cudaStream_t stream);

cudaError_t launch_expand(uint8_t* dst, uint64_t fold, uint64_t bytes, const uint8_t* prefix32,
                          cudaStream_t stream);
// result[0] <- min offset of a byte != materialize(prefix, bytes); must be
// initialised to UINT64_MAX by the caller.
cudaError_t launch_blob_check(const uint8_t* blob, uint64_t bytes, unsigned long long* result,
                              cudaStream_t stream);

// Whole-buffer FNV-1a-64 continuing from `h0` (kFnvBasis for checksum64).
// Uses a scratch allocation internally; synchronises `stream`.
cudaError_t whole_fnv(const uint8_t* data, uint64_t len, uint64_t h0, uint64_t* out,
                      cudaStream_t stream);

// Keep up to 256 MB cached in the current device's default memory pool.
void retain_pool();

// The data loader's device side (ffx_preload.cu): `count` synthetic samples
// of `sample_bytes` each, sample i = expand(digest_i) given its fold64
// (DataServerStub::fetch, dataloader.cpp:104-127, evolution.cpp:71-120), and
// fold_of_blob (dataloader.cpp:150-164) accumulated into *out (wrapping).
cudaError_t launch_items(uint8_t* dst, const uint64_t* folds, uint32_t count, uint32_t sample_bytes,
                         cudaStream_t stream);
cudaError_t launch_fold_blob(const uint8_t* blob, uint64_t bytes, uint32_t bytes_per_sample,
                             unsigned long long* out, cudaStream_t stream);

cudaError_t launch_fill(uint8_t* dst, uint64_t bytes, uint32_t pattern, cudaStream_t stream);
cudaError_t launch_xor_byte(uint8_t* dst, uint8_t mask, cudaStream_t stream);

int sm_count();

}  // namespace ffx
