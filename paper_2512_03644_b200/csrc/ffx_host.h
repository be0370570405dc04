// ffx_host.h -- internal to libffx.so: the objects behind the C ABI's opaque
// handles (ffx_ctx, ffx_replica) and the helpers the host-side files share:
//   ffx_api.cu       status, domain, planning, sizing, framing, primitives,
//                    buffer plumbing, contexts + the state registry
//   ffx_replica.cu   neighbour replica manager + SNP1 export
//   ffx_snapshot.cu  snapshot issue, pull mode, slice scheduler batches
//   ffx_recover.cu   recovery gather/verify, CUDA IPC, failure injection
//   ffx_mcast.cu     shareable replicas + NVSwitch multicast
//   ffx_sched.cu     the slice scheduler (gap-driven batches)
// No CPU compute path exists for any payload byte: every copy, checksum and
// verification runs on the GPU; the host only sizes, chooses slots and
// launches.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/ffx.h"
#include "ffx_device.cuh"
#include "ffx_kernels.h"
#include "ffx_layout.h"
#include "ffx_share.h"

namespace ffx::host {

// Last error message of the calling thread (ffx_last_error).
extern thread_local std::string g_err;
int fail(int status, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {  // dev < 0: leave the current device alone
    cudaGetDevice(&prev);
    if (dev >= 0 && prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline void le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}
inline uint64_t rd(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

// ctx scratch words (ctx->done, 64 x u32): 0 commit counter, 4 second-replica
// commit counter, 8-9 snapshot task counter, 12-13 verify task counter,
// 16-17 split hash-batch task counter, 20-21 hybrid fused-share task
// counter, 24-25 pull-mode ack (u64).
constexpr uint32_t kAckWord = 24;
// No pulled iteration pending (the ack word's value at open, after every
// consumed wait and after a rollback / recovery).
constexpr uint64_t kAckNone = ~0ull;

inline bool valid_spec(const ffx_cluster_spec* s) {
  return s && s->data_parallel && s->pipeline_parallel && s->tensor_parallel && s->gpus_per_node;
}

// Device a context-free primitive runs on: the stream's device when a
// stream is given, else the device that owns `p` (host / unknown: -1 = the
// current device).  One process may drive several GPUs.
inline int pick_device(void* stream, const void* p) {
  int d = -1;
  if (stream && cudaStreamGetDevice(static_cast<cudaStream_t>(stream), &d) == cudaSuccess) return d;
  cudaGetLastError();
  cudaPointerAttributes a{};
  if (p && cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeDevice) return a.device;
  cudaGetLastError();
  return -1;
}

inline bool slice_ok(uint64_t s) { return s >= 256 && s % 256 == 0; }
inline uint64_t slices_of(uint64_t bytes, uint64_t s) { return (bytes + s - 1) / s; }

// Driver entry points through the runtime (no -lcuda: the library must load
// on hosts without a driver for the CPU-side ABI checks).
template <typename Fn>
Fn driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<Fn>(p);
}

}  // namespace ffx::host

#define FFX_CUDA(call)                                                \
  do {                                                                \
    cudaError_t e_ = (call);                                          \
    if (e_ != cudaSuccess) return ffx::host::cuda_fail(e_, #call);    \
  } while (0)

using namespace ffx;


struct Region {
  int kind;
  uint8_t* dev;
  uint64_t bytes;
  bool unique;
};

struct SlotCache {
  bool known = false;
  uint32_t state = kSlotEmpty;
  uint64_t iteration = 0;
  uint64_t seq = 0;
};

struct ffx_replica {
  int device = 0;          // device the memory lives on
  int owner_pid = 0;
  bool owned = false;      // cudaMalloc'd here
  bool ipc_opened = false; // cudaIpcOpenMemHandle'd here
  uint8_t* base = nullptr;
  ffx_role origin{};
  uint64_t capacity = 0;
  uint64_t slice_bytes = 0;
  uint32_t versions = 0;
  SlotLayout layout{};
  std::vector<SlotCache> cache;  // writer-side view of the slots
  ffx_ctx* ctx = nullptr;        // context that created/opened it
  // Shareable (VMM) replicas, the NVSwitch-multicast path: the allocation
  // handle, its size, and the fd it is exported through (owner only).
  bool vmm = false;
  bool vmm_mapped = false;       // imported + mapped here (not the owner)
  unsigned long long vmm_handle = 0;
  uint64_t vmm_bytes = 0;
  int vmm_fd = -1;
  // Tiered replicas (a replica larger than the holder's free HBM, configs[4]):
  // one VA range whose first tier_hbm bytes are device memory and the rest
  // pinned host memory on the device's NUMA node (vmm_handle2 / vmm_fd2).
  // Kernels address it as one buffer; the host tier moves over PCIe.
  uint64_t tier_hbm = 0;
  unsigned long long vmm_handle2 = 0;
  int vmm_fd2 = -1;
  // Multicast target: kernels WRITE through wbase (the multicast range every
  // holder's replica is bound to) and the host READS slot metadata through
  // base (one holder's unicast mapping).  Null = write through base.
  uint8_t* wbase = nullptr;

  uint8_t* slot(uint32_t v) const { return base + v * layout.slot_stride; }
  uint8_t* payload(uint32_t v) const { return slot(v) + layout.payload_off; }
  uint64_t* sums(uint32_t v) const { return reinterpret_cast<uint64_t*>(slot(v) + kMetaBytes); }
  uint8_t* wslot(uint32_t v) const { return (wbase ? wbase : base) + v * layout.slot_stride; }
  uint8_t* wpayload(uint32_t v) const { return wslot(v) + layout.payload_off; }
  uint64_t* wsums(uint32_t v) const { return reinterpret_cast<uint64_t*>(wslot(v) + kMetaBytes); }
};

// A snapshot split by the slice scheduler into batches still to be issued.
struct PendingSnapshot {
  bool active = false;
  SliceJob job{};  // fused: copy + hash (+ commit); split: the hash-only job
  uint32_t batches = 1, next = 0, max_ctas = 0, slot = 0, slot2 = 0;
  uint64_t iteration = 0, seq = 0, seq2 = 0, nslices = 0, logical = 0;
  bool verify = false;
  bool one_shot = false;  // task-granular fused batches (opts.task_ctas)
  // split policy: copy batches and hash batches drain independently
  bool split = false, copy_engine = false;
  CopyJob copy{};
  ffx_replica* tgt = nullptr;   // destination replica(s) of this snapshot
  ffx_replica* tgt2 = nullptr;
  uint32_t hbatches = 0, hnext = 0, hash_ctas = 0;
  // hybrid (split + copy engines + fused_permille): warp tasks [0, gcut) are
  // copied + hashed by the fused kernel (fjob), the copy engines move the rest
  uint64_t gcut = 0;
  SliceJob fjob{};
  uint64_t logical_of[kMaxRegions] = {};  // logical payload offset of each job region (batch spans)
  std::vector<double> frac;  // cumulative batch boundaries in [0, 1] (measured-gap weights)
  uint64_t cut(uint64_t total, uint32_t b) const {
    return b >= batches ? total : static_cast<uint64_t>(static_cast<double>(total) * frac[b]);
  }
};

struct ffx_ctx {
  PendingSnapshot pending;
  int device = 0;
  ffx_cluster_spec spec{};
  ffx_role self{};
  uint64_t slice_bytes = 4096;
  std::vector<Region> regions;
  ffx_replica* target = nullptr;
  ffx_replica* target2 = nullptr;  // second holder (double-neighbour), optional
  unsigned int* done = nullptr;            // commit counter (device)
  unsigned long long* result = nullptr;    // verify result (device, 2 words)
  unsigned long long* result_host = nullptr;  // pinned mirror
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t copy_done = nullptr, hash_done = nullptr;  // split-policy joins
  // Recorded after each snapshot's last launch; the next snapshot's first
  // launch of each kind waits on it, so two snapshots of one ctx never run
  // concurrently (they share the task / commit counter words) even when the
  // caller issues them on different streams.
  cudaEvent_t snap_done = nullptr;
  uint64_t seq = 0;
  uint32_t last_slot = 0;
  ffx_replica* last_target = nullptr;
  uint64_t last_nslices = 0;
  ffx_stats stats{};
  // ffx_snapshot_from_host: the H2D copy stream and one event per batch
  cudaStream_t h2d = nullptr;
  std::vector<cudaEvent_t> h2d_ev;
};

namespace ffx::host {

struct HandleBlob {  // FFX_HANDLE_BYTES on the wire
  uint32_t magic;    // "FFXH"
  uint32_t abi;
  int32_t pid;
  int32_t device;
  uint64_t raw;      // device pointer (valid in the exporting process)
  uint64_t capacity, slice_bytes;
  uint32_t versions;
  uint16_t dp, pp, tp, pad_;
  SlotLayout layout;
  cudaIpcMemHandle_t ipc;
  uint32_t kind;         // 0 = cudaMalloc + CUDA IPC, 1 = shareable VMM allocation, 2 = tiered VMM
  int32_t fd;            // kind 1/2: the exporter's fd (fetched through its fd server)
  uint64_t alloc_bytes;  // kind 1/2: size of the whole range
  int32_t fd2;           // kind 2: the host-memory tier's fd
  uint32_t pad2_;
  uint64_t tier_hbm;     // kind 2: bytes of the range backed by device memory (the rest: host memory)
};
static_assert(sizeof(HandleBlob) <= FFX_HANDLE_BYTES, "handle too large");
constexpr uint32_t kHandleMagic = 0x48584646u;

// Unique regions in registration order and their offsets in a slot payload.
struct PayloadMap {
  std::vector<const Region*> regs;
  std::vector<uint64_t> offs;
  uint64_t logical = 0;
  uint64_t physical = 0;
};
PayloadMap payload_map(const ffx_ctx* c);
// The slice runs of a payload map in table order (ffx_layout.h).
struct RunRef {
  uint32_t region;  // index into PayloadMap::regs
  SliceRun run;
};
inline std::vector<RunRef> payload_runs(const PayloadMap& pm, uint64_t S) {
  std::vector<RunRef> out;
  const uint32_t n = static_cast<uint32_t>(pm.regs.size());
  for (uint32_t r = 0; r < n; ++r) {
    SliceRun runs[kRegionRuns];
    const int k = region_runs(pm.regs[r]->bytes, S, head_region(r, n), runs);
    for (int j = 0; j < k; ++j) out.push_back(RunRef{r, runs[j]});
  }
  return out;
}

int read_meta(ffx_replica* r, uint32_t v, SlotMeta* m);
int refresh_cache(ffx_replica* r);
// A one-region slice job over [src, src+len) (dst null = hash only).
SliceJob single_job(const void* src, void* dst, uint64_t len, uint64_t slice_bytes);
// Slot holding `iteration` (-1 none, -2 metadata unreadable).
int find_slot(ffx_replica* r, uint64_t iteration, SlotMeta* meta);
// Shareable (VMM) replicas: open an exported one / release (ffx_mcast.cu).
int open_shared(ffx_ctx* c, const HandleBlob& h, ffx_replica* r);
void release_shared(ffx_replica* r);
// ffx_preload.cu: one fetch into the preload buffer (host bytes or synthetic
// samples) on stream s after gate.
int preload_fetch(ffx_preload* p, uint64_t iteration, const void* host_src, const uint8_t* digests, uint32_t count,
                  uint32_t sample_bytes, uint64_t bytes, cudaStream_t s, cudaEvent_t gate);

}  // namespace ffx::host

namespace ffx::host {
// Set ctx's pull-mode ack word to kAckNone on stream s (stream-ordered).
int reset_ack(ffx_ctx* c, cudaStream_t s);
// Slot metadata sanity: regions, payload length, slice size and table length
// agree with each other and with r's layout (FFX_ECORRUPT otherwise).
int check_meta(const ffx_replica* r, const SlotMeta& m);
}  // namespace ffx::host

using namespace ffx::host;
