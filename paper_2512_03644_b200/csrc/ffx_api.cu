// ffx_api.cu -- the C ABI (include/ffx.h): state registry / partitioner,
// neighbour replica manager, snapshot issue + slice scheduler, recovery
// gather/verify, SNP1 export, failure injection.
//
// Host code over the sm_100a kernels in ffx_kernels.cu.  No CPU compute
// path exists for any payload byte: every copy, checksum and verification
// runs on the GPU; the host only sizes, chooses slots and launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <numeric>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ffx.h"
#include "ffx_device.cuh"
#include "ffx_kernels.h"
#include "ffx_layout.h"
#include "ffx_share.h"

using namespace ffx;

// ---------------------------------------------------------------------------
// errors

namespace {

thread_local std::string g_err;

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return status;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(FFX_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define FFX_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

void le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}
uint64_t rd(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

// ctx scratch words (ctx->done, 64 x u32): 0 commit counter, 4 second-replica
// commit counter, 8-9 snapshot task counter, 12-13 verify task counter,
// 16-17 split hash-batch task counter, 24-25 pull-mode ack (u64).
constexpr uint32_t kAckWord = 24;

bool valid_spec(const ffx_cluster_spec* s) {
  return s && s->data_parallel && s->pipeline_parallel && s->tensor_parallel && s->gpus_per_node;
}

}  // namespace

// ---------------------------------------------------------------------------
// objects

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
  uint64_t iteration = 0, seq = 0, nslices = 0, logical = 0;
  bool verify = false;
  // split policy: copy batches and hash batches drain independently
  bool split = false, copy_engine = false;
  CopyJob copy{};
  ffx_replica* tgt = nullptr;   // destination replica(s) of this snapshot
  ffx_replica* tgt2 = nullptr;
  uint32_t hbatches = 0, hnext = 0, hash_ctas = 0;
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
  uint64_t seq = 0;
  uint32_t last_slot = 0;
  ffx_replica* last_target = nullptr;
  uint64_t last_nslices = 0;
  ffx_stats stats{};
};

namespace {

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
  uint32_t kind;         // 0 = cudaMalloc + CUDA IPC, 1 = shareable VMM allocation
  int32_t fd;            // kind 1: the exporter's fd (fetched through its fd server)
  uint64_t alloc_bytes;  // kind 1: allocation size
};
static_assert(sizeof(HandleBlob) <= FFX_HANDLE_BYTES, "handle too large");
// Shareable replicas (defined with the multicast section below).
int open_shared(ffx_ctx* c, const HandleBlob& h, ffx_replica* r);
void release_shared(ffx_replica* r);
constexpr uint32_t kHandleMagic = 0x48584646u;

int read_meta(ffx_replica* r, uint32_t v, SlotMeta* m) {
  DeviceGuard g(r->ctx ? r->ctx->device : r->device);
  FFX_CUDA(cudaMemcpy(m, r->slot(v), sizeof(SlotMeta), cudaMemcpyDefault));
  return FFX_OK;
}

// Unique regions in registration order and their offsets in a slot payload.
struct PayloadMap {
  std::vector<const Region*> regs;
  std::vector<uint64_t> offs;
  uint64_t logical = 0;
  uint64_t physical = 0;
};

PayloadMap payload_map(const ffx_ctx* c) {
  PayloadMap m;
  for (const auto& r : c->regions)
    if (r.unique) {
      m.regs.push_back(&r);
      m.offs.push_back(m.physical);
      m.logical += r.bytes;
      m.physical = align_up(m.physical + r.bytes, kRegionAlign);
    }
  return m;
}

uint64_t slices_of(uint64_t bytes, uint64_t s) { return (bytes + s - 1) / s; }

int refresh_cache(ffx_replica* r) {
  for (uint32_t v = 0; v < r->versions; ++v) {
    SlotMeta m;
    int st = read_meta(r, v, &m);
    if (st) return st;
    SlotCache& c = r->cache[v];
    c.known = true;
    if (m.magic == kSlotMagic) {
      c.state = m.state;
      c.iteration = m.iteration;
      c.seq = m.seq;
    } else {
      c.state = kSlotEmpty;
      c.iteration = 0;
      c.seq = 0;
    }
  }
  return FFX_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// status

extern "C" const char* ffx_status_str(int s) {
  switch (s) {
    case FFX_OK: return "ok";
    case FFX_ECONFIG: return "config error";
    case FFX_EVERSION: return "version error";
    case FFX_ERESTORE: return "restore error";
    case FFX_ECORRUPT: return "corrupt snapshot";
    case FFX_EINVAL: return "invalid argument";
    case FFX_ERANGE: return "out of range";
    case FFX_ECUDA: return "cuda error";
    case FFX_ENOMEM: return "out of device memory";
    case FFX_ESTATE: return "invalid state";
  }
  return "unknown";
}
extern "C" const char* ffx_last_error(void) { return g_err.c_str(); }
extern "C" int ffx_abi_version(void) { return FFX_ABI_VERSION; }

// ---------------------------------------------------------------------------
// domain (domain.cpp:18-62)

extern "C" int ffx_role_of(const ffx_cluster_spec* s, uint32_t idx, ffx_role* out) {
  if (!valid_spec(s) || !out) return fail(FFX_EINVAL, "role_of: bad spec");
  const uint64_t world = uint64_t{s->num_nodes} * s->gpus_per_node;
  if (idx >= world) return fail(FFX_ERANGE, "role_of: index %u outside world of %llu", idx,
                                (unsigned long long)world);
  out->tp = static_cast<uint16_t>(idx % s->tensor_parallel);
  out->pp = static_cast<uint16_t>((idx / s->tensor_parallel) % s->pipeline_parallel);
  out->dp = static_cast<uint16_t>(idx / (s->tensor_parallel * s->pipeline_parallel));
  return FFX_OK;
}

extern "C" int ffx_index_of(const ffx_cluster_spec* s, ffx_role r, uint32_t* out) {
  if (!valid_spec(s) || !out) return fail(FFX_EINVAL, "index_of: bad spec");
  if (r.tp >= s->tensor_parallel || r.pp >= s->pipeline_parallel || r.dp >= s->data_parallel)
    return fail(FFX_ERANGE, "index_of: role d%up%ut%u outside layout", r.dp, r.pp, r.tp);
  *out = (uint32_t{r.dp} * s->pipeline_parallel + r.pp) * s->tensor_parallel + r.tp;
  return FFX_OK;
}

extern "C" int ffx_node_of(const ffx_cluster_spec* s, ffx_role r, uint32_t* out) {
  uint32_t idx = 0;
  int st = ffx_index_of(s, r, &idx);
  if (st) return st;
  *out = idx / s->gpus_per_node;
  return FFX_OK;
}

extern "C" int ffx_dp_neighbor(const ffx_cluster_spec* s, ffx_role r, ffx_role* out) {
  if (!valid_spec(s) || !out) return fail(FFX_EINVAL, "dp_neighbor: bad spec");
  *out = r;
  out->dp = static_cast<uint16_t>((r.dp + 1u) % s->data_parallel);
  return FFX_OK;
}

extern "C" int ffx_dp_predecessor(const ffx_cluster_spec* s, ffx_role r, ffx_role* out) {
  if (!valid_spec(s) || !out) return fail(FFX_EINVAL, "dp_predecessor: bad spec");
  *out = r;
  out->dp = static_cast<uint16_t>((r.dp + s->data_parallel - 1u) % s->data_parallel);
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// recovery planning (controller.cpp:144-209)

extern "C" int ffx_plan_recovery(const ffx_cluster_spec* s, const uint32_t* pods, uint32_t n_pods,
                                 const ffx_role* roles, uint32_t n_roles, uint64_t global_consistent,
                                 uint64_t latest_fallback, uint32_t replicas, ffx_recovery_plan* out) {
  if (!valid_spec(s) || !out) return fail(FFX_EINVAL, "plan_recovery: bad arguments");
  if ((n_pods && !pods) || (n_roles && !roles)) return fail(FFX_EINVAL, "plan_recovery: null list");
  if (replicas < 1) replicas = 1;
  auto key = [](const ffx_role& r) {
    return (uint64_t{r.dp} << 32) | (uint64_t{r.pp} << 16) | r.tp;
  };
  std::vector<uint32_t> fp(pods, pods + n_pods);
  std::sort(fp.begin(), fp.end());
  fp.erase(std::unique(fp.begin(), fp.end()), fp.end());
  std::vector<ffx_role> lost(roles, roles + n_roles);
  for (uint32_t pod : fp)
    for (uint32_t lr = 0; lr < s->gpus_per_node; ++lr) {
      ffx_role r;
      int st = ffx_role_of(s, pod * s->gpus_per_node + lr, &r);
      if (st) return st;
      lost.push_back(r);
    }
  // std::set<Role> ordering: (dp, pp, tp) lexicographic.
  std::sort(lost.begin(), lost.end(), [&](const ffx_role& a, const ffx_role& b) { return key(a) < key(b); });
  lost.erase(std::unique(lost.begin(), lost.end(),
                         [&](const ffx_role& a, const ffx_role& b) { return key(a) == key(b); }),
             lost.end());
  auto is_lost = [&](const ffx_role& r) {
    return std::binary_search(lost.begin(), lost.end(), r,
                              [&](const ffx_role& a, const ffx_role& b) { return key(a) < key(b); });
  };
  const uint32_t cap = out->capacity;
  if (fp.size() > cap || lost.size() > cap) return fail(FFX_ECONFIG, "plan_recovery: capacity %u too small", cap);
  out->n_failed_pods = static_cast<uint32_t>(fp.size());
  out->n_failed_roles = static_cast<uint32_t>(lost.size());
  out->n_lazy = out->n_forwards = out->n_redundant = 0;
  if (out->failed_pods) std::copy(fp.begin(), fp.end(), out->failed_pods);
  if (out->failed_roles) std::copy(lost.begin(), lost.end(), out->failed_roles);

  // Serving holder per lost role: first survivor among dp+1 .. dp+replicas.
  const uint32_t d = s->data_parallel;
  const uint32_t k = std::min<uint32_t>(replicas, d > 1 ? d - 1 : 1);
  bool neighbor_ok = d > 1;
  std::vector<uint32_t> holder(lost.size(), 0);
  for (size_t i = 0; i < lost.size() && neighbor_ok; ++i) {
    bool found = false;
    for (uint32_t j = 1; j <= k; ++j) {
      ffx_role h = lost[i];
      h.dp = static_cast<uint16_t>((lost[i].dp + j) % d);
      if (!is_lost(h)) {
        holder[i] = h.dp;
        found = true;
        break;
      }
    }
    if (!found) neighbor_ok = false;
  }
  ffx_uniqueness_plan up;
  ffx_razor(s, &up);
  if (!neighbor_ok) {
    out->kind = 1;
    out->resume_iteration = latest_fallback;
    return FFX_OK;
  }
  out->kind = 0;
  out->resume_iteration = global_consistent;
  if (global_consistent == 0) return FFX_OK;  // rebuilt from the seed (controller.cpp:172-174)
  for (size_t i = 0; i < lost.size(); ++i) {
    const ffx_role f = lost[i];
    if (up.unique_bytes_per_device > 0) {
      ffx_role h = f;
      h.dp = static_cast<uint16_t>(holder[i]);
      ffx_forward fw{};
      fw.origin = f;
      fw.holder_dp = holder[i];
      int st = ffx_node_of(s, h, &fw.holder_node);
      if (!st) st = ffx_node_of(s, f, &fw.dest_node);
      if (st) return st;
      if (out->forwards) out->forwards[out->n_forwards] = fw;
      out->n_forwards++;
    }
    if (up.weights_redundant || up.optimizer_redundant) {
      for (uint32_t dp = 0; dp < d; ++dp) {
        ffx_role cand{static_cast<uint16_t>(dp), f.pp, f.tp};
        if (!is_lost(cand)) {
          if (out->redundant_from) out->redundant_from[out->n_redundant] = ffx_redundant_source{f, cand};
          out->n_redundant++;
          break;
        }
      }
    }
  }
  if (up.weights_redundant || up.optimizer_redundant) {
    for (uint32_t pp = 0; pp < s->pipeline_parallel; ++pp)
      for (uint32_t tp = 0; tp < s->tensor_parallel; ++tp)
        for (uint32_t dp = 0; dp < d; ++dp) {
          ffx_role cand{static_cast<uint16_t>(dp), static_cast<uint16_t>(pp), static_cast<uint16_t>(tp)};
          if (!is_lost(cand)) {
            if (out->n_lazy >= cap) return fail(FFX_ECONFIG, "plan_recovery: capacity %u too small", cap);
            if (out->lazy_backup_targets) out->lazy_backup_targets[out->n_lazy] = cand;
            out->n_lazy++;
            break;
          }
        }
  }
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// sizing (ckpt.cpp:13-33, evolution.cpp:11-19)

extern "C" uint64_t ffx_weights_bytes(const ffx_cluster_spec* s) {
  return s ? 2 * s->params_per_device : 0;
}

extern "C" uint64_t ffx_optimizer_bytes(const ffx_cluster_spec* s) {
  if (!s) return 0;
  const uint64_t full = 12 * s->params_per_device;
  if (!s->distributed_optimizer || s->data_parallel <= 1) return full;
  return (full + s->data_parallel - 1) / s->data_parallel;
}

extern "C" int ffx_razor(const ffx_cluster_spec* s, ffx_uniqueness_plan* out) {
  if (!s || !out) return fail(FFX_EINVAL, "razor: null argument");
  out->weights_redundant = s->data_parallel > 1;
  out->optimizer_redundant = s->data_parallel > 1 && !s->distributed_optimizer;
  out->unique_bytes_per_device = out->optimizer_redundant ? 0 : ffx_optimizer_bytes(s);
  return FFX_OK;
}

extern "C" int ffx_version_for_target(uint64_t held, uint64_t target, int* out) {
  if (!out) return fail(FFX_EINVAL, "version_for_target: null out");
  if (held == target) {
    *out = 0;
    return FFX_OK;
  }
  if (held == target + 1) {
    *out = 1;
    return FFX_OK;
  }
  return fail(FFX_EVERSION, "backup target %llu outside the retained window ending at %llu",
              (unsigned long long)target, (unsigned long long)held);
}

// ---------------------------------------------------------------------------
// SNP1 framing (storage.cpp:45-101)

extern "C" int ffx_pack_header(ffx_role role, uint64_t iteration, uint8_t kind, uint64_t len,
                               uint64_t checksum, uint8_t out[32]) {
  if (!out) return fail(FFX_EINVAL, "pack_header: null out");
  if (len > 0xffffffffull) return fail(FFX_EINVAL, "snapshot payload exceeds 4 GiB framing limit");
  std::memset(out, 0, 32);
  le(out + 0, 0x31504E53u, 4);
  out[4] = 1;
  out[5] = kind;
  le(out + 6, role.dp, 2);
  le(out + 8, role.pp, 2);
  le(out + 10, role.tp, 2);
  le(out + 12, iteration, 8);
  le(out + 20, len, 4);
  le(out + 24, checksum, 8);
  return FFX_OK;
}

extern "C" int ffx_parse_header(const uint8_t* h, uint64_t framed_len, ffx_blob_info* out) {
  if (!h || !out) return fail(FFX_EINVAL, "parse_header: null argument");
  if (framed_len != 0 && framed_len < 32) return fail(FFX_ECORRUPT, "snapshot shorter than header");
  if (rd(h, 4) != 0x31504E53u) return fail(FFX_ECORRUPT, "bad snapshot magic");
  if (h[4] != 1) return fail(FFX_ECORRUPT, "unsupported snapshot format version");
  if (h[5] > 1) return fail(FFX_ECORRUPT, "unknown blob kind");
  out->kind = h[5];
  out->role.dp = static_cast<uint16_t>(rd(h + 6, 2));
  out->role.pp = static_cast<uint16_t>(rd(h + 8, 2));
  out->role.tp = static_cast<uint16_t>(rd(h + 10, 2));
  out->iteration = rd(h + 12, 8);
  out->payload_len = static_cast<uint32_t>(rd(h + 20, 4));
  out->checksum = rd(h + 24, 8);
  if (framed_len != 0 && framed_len != 32 + uint64_t{out->payload_len})
    return fail(FFX_ECORRUPT, "snapshot length disagrees with header");
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// device primitives

namespace {

SliceJob single_job(const void* src, void* dst, uint64_t len, uint64_t slice_bytes) {
  SliceJob job{};
  job.nregions = 1;
  job.reg[0] = SliceRegion{static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), len, 0, 0};
  job.slice_bytes = slice_bytes;
  finalize_job(job);
  return job;
}

bool slice_ok(uint64_t s) { return s >= 256 && s % 256 == 0; }

}  // namespace

extern "C" int ffx_checksum64(const void* dev, uint64_t len, uint64_t* host_out, void* stream) {
  if (!host_out || (len && !dev)) return fail(FFX_EINVAL, "checksum64: null argument");
  cudaError_t e = whole_fnv(static_cast<const uint8_t*>(dev), len, kFnvBasis, host_out,
                            as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "whole_fnv");
  return FFX_OK;
}

extern "C" int ffx_slice_checksums(const void* dev, uint64_t len, uint64_t slice_bytes,
                                   uint64_t* dev_out, void* stream) {
  if (!slice_ok(slice_bytes)) return fail(FFX_EINVAL, "slice_bytes must be a multiple of 256");
  if (len == 0) return FFX_OK;
  if (!dev || !dev_out) return fail(FFX_EINVAL, "slice_checksums: null argument");
  SliceJob job = single_job(dev, nullptr, len, slice_bytes);
  job.sums_out = dev_out;
  FFX_CUDA(launch_slices(job, SliceMode::Hash, false, 0, as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_copy_checksums(void* dst, const void* src, uint64_t len, uint64_t slice_bytes,
                                  uint64_t* dev_out, void* stream) {
  if (!slice_ok(slice_bytes)) return fail(FFX_EINVAL, "slice_bytes must be a multiple of 256");
  if (len == 0) return FFX_OK;
  if (!dst || !src) return fail(FFX_EINVAL, "copy_checksums: null argument");
  SliceJob job = single_job(src, dst, len, slice_bytes);
  job.sums_out = dev_out;
  FFX_CUDA(launch_slices(job, SliceMode::Copy, false, 0, as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_copy_verify(void* dst, const void* src, uint64_t len, uint64_t slice_bytes,
                               const uint64_t* dev_expected, uint64_t* dev_result, void* stream) {
  if (!slice_ok(slice_bytes)) return fail(FFX_EINVAL, "slice_bytes must be a multiple of 256");
  if (!dev_result || !dev_expected) return fail(FFX_EINVAL, "copy_verify: null argument");
  const unsigned long long init[2] = {~0ull, 0ull};
  FFX_CUDA(cudaMemcpyAsync(dev_result, init, sizeof init, cudaMemcpyHostToDevice, as_stream(stream)));
  if (len == 0) return FFX_OK;
  SliceJob job = single_job(src, dst, len, slice_bytes);
  job.sums_expected = dev_expected;
  job.result = reinterpret_cast<unsigned long long*>(dev_result);
  FFX_CUDA(launch_slices(job, dst ? SliceMode::CopyVerify : SliceMode::HashVerify, false, 0,
                         as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_copy(void* dst, const void* src, uint64_t len, uint32_t ctas, void* stream) {
  if (len == 0) return FFX_OK;
  if (!dst || !src) return fail(FFX_EINVAL, "copy: null argument");
  CopyJob job{};
  job.nregions = 1;
  job.reg[0] = CopyRegion{static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), len, 0, 0};
  finalize_copy_job(job);
  FFX_CUDA(launch_copy(job, ctas, as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_expand(void* dst, const uint8_t digest[32], uint64_t bytes, void* stream) {
  if (!digest || (bytes && !dst)) return fail(FFX_EINVAL, "expand: null argument");
  uint64_t fold = rd(digest, 8);
  FFX_CUDA(launch_expand(static_cast<uint8_t*>(dst), fold, bytes, nullptr, as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_materialize(void* dst, const uint8_t digest[32], uint64_t bytes, void* stream) {
  if (!digest) return fail(FFX_EINVAL, "materialize: null digest");
  if (bytes < 32) return fail(FFX_EINVAL, "state blob smaller than its digest prefix");
  if (!dst) return fail(FFX_EINVAL, "materialize: null dst");
  FFX_CUDA(launch_expand(static_cast<uint8_t*>(dst), rd(digest, 8), bytes, digest,
                         as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_blob_check(const void* dev, uint64_t bytes, uint64_t* host_first_bad,
                              void* stream) {
  if (!host_first_bad) return fail(FFX_EINVAL, "blob_check: null out");
  if (bytes < 32) {  // evolution.cpp:107: shorter than the digest is never sound
    *host_first_bad = 0;
    return FFX_OK;
  }
  unsigned long long* d = nullptr;
  cudaStream_t s = as_stream(stream);
  retain_pool();
  FFX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 8, s));
  const unsigned long long init = ~0ull;
  FFX_CUDA(cudaMemcpyAsync(d, &init, 8, cudaMemcpyHostToDevice, s));
  FFX_CUDA(launch_blob_check(static_cast<const uint8_t*>(dev), bytes, d, s));
  unsigned long long r = 0;
  FFX_CUDA(cudaMemcpyAsync(&r, d, 8, cudaMemcpyDeviceToHost, s));
  FFX_CUDA(cudaFreeAsync(d, s));
  FFX_CUDA(cudaStreamSynchronize(s));
  *host_first_bad = r;
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// buffer plumbing

extern "C" int ffx_device_alloc(int device, uint64_t bytes, void** dev) {
  if (!dev) return fail(FFX_EINVAL, "device_alloc: null out");
  DeviceGuard g(device);
  cudaError_t e = cudaMalloc(dev, bytes ? bytes : 1);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FFX_ENOMEM, "device_alloc(%llu): %s", (unsigned long long)bytes, cudaGetErrorString(e));
  }
  return FFX_OK;
}

extern "C" int ffx_device_free(int device, void* dev) {
  if (!dev) return FFX_OK;
  DeviceGuard g(device);
  FFX_CUDA(cudaFree(dev));
  return FFX_OK;
}

extern "C" int ffx_memcpy(void* dst, const void* src, uint64_t bytes, void* stream, int sync) {
  if (!bytes) return FFX_OK;
  if (!dst || !src) return fail(FFX_EINVAL, "memcpy: null pointer");
  FFX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, as_stream(stream)));
  if (sync) FFX_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_pointer_is_device(const void* p, int* is_device) {
  if (!is_device) return fail(FFX_EINVAL, "pointer_is_device: null out");
  *is_device = 0;
  if (!p) return FFX_OK;
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return FFX_OK;
  }
  *is_device = (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) ? 1 : 0;
  return FFX_OK;
}

extern "C" int ffx_stream_sync(void* stream) {
  FFX_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// context + registry

extern "C" int ffx_open(int device, const ffx_cluster_spec* spec, ffx_role self,
                        uint64_t slice_bytes, ffx_ctx** out) {
  if (!out || !valid_spec(spec)) return fail(FFX_EINVAL, "open: bad arguments");
  if (slice_bytes == 0) slice_bytes = 4096;
  if (!slice_ok(slice_bytes)) return fail(FFX_EINVAL, "slice_bytes must be a multiple of 256");
  int ndev = 0;
  FFX_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(FFX_EINVAL, "open: no device %d", device);
  DeviceGuard g(device);
  auto* c = new ffx_ctx;
  c->device = device;
  c->spec = *spec;
  c->self = self;
  c->slice_bytes = slice_bytes;
  cudaError_t e = cudaMalloc(&c->done, 256);
  if (e == cudaSuccess) e = cudaMemset(c->done, 0, 256);
  if (e == cudaSuccess) e = cudaMalloc(&c->result, 16);
  if (e == cudaSuccess) e = cudaMallocHost(&c->result_host, 16);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->copy_done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->hash_done, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    ffx_close(c);
    return cuda_fail(e, "open");
  }
  *out = c;
  return FFX_OK;
}

extern "C" int ffx_close(ffx_ctx* c) {
  if (!c) return FFX_OK;
  DeviceGuard g(c->device);
  if (c->done) cudaFree(c->done);
  if (c->result) cudaFree(c->result);
  if (c->result_host) cudaFreeHost(c->result_host);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->copy_done) cudaEventDestroy(c->copy_done);
  if (c->hash_done) cudaEventDestroy(c->hash_done);
  delete c;
  return FFX_OK;
}

extern "C" int ffx_register_region(ffx_ctx* c, int kind, void* dev, uint64_t bytes, int unique) {
  if (!c) return fail(FFX_EINVAL, "register_region: null ctx");
  if (c->regions.size() >= kMaxRegions)
    return fail(FFX_ECONFIG, "state registry holds at most %u regions", kMaxRegions);
  if (bytes && !dev) return fail(FFX_EINVAL, "register_region: null pointer");
  if (reinterpret_cast<uintptr_t>(dev) % 16)
    return fail(FFX_EINVAL, "register_region: device pointer must be 16-byte aligned");
  if (kind < FFX_REGION_MASTER || kind > FFX_REGION_BLOB)
    return fail(FFX_EINVAL, "register_region: unknown kind %d", kind);
  c->regions.push_back(Region{kind, static_cast<uint8_t*>(dev), bytes, unique != 0});
  return FFX_OK;
}

extern "C" int ffx_clear_regions(ffx_ctx* c) {
  if (!c) return fail(FFX_EINVAL, "clear_regions: null ctx");
  c->regions.clear();
  return FFX_OK;
}

extern "C" int ffx_plan(ffx_ctx* c, ffx_plan_info* out) {
  if (!c || !out) return fail(FFX_EINVAL, "plan: null argument");
  std::memset(out, 0, sizeof *out);
  ffx_razor(&c->spec, &out->razor);
  out->slice_bytes = c->slice_bytes;
  out->num_regions = static_cast<uint32_t>(c->regions.size());
  for (const auto& r : c->regions) {
    if (r.unique) {
      out->registered_unique_bytes += r.bytes;
      out->num_slices += slices_of(r.bytes, c->slice_bytes);
      out->num_unique_regions++;
    } else {
      out->registered_redundant_bytes += r.bytes;
    }
  }
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// replicas

extern "C" int ffx_replica_create(ffx_ctx* c, ffx_role origin, uint64_t capacity, uint32_t versions,
                                  ffx_replica** out) {
  if (!c || !out) return fail(FFX_EINVAL, "replica_create: null argument");
  if (versions < 1 || versions > 8) return fail(FFX_EINVAL, "replica_create: 1..8 versions");
  DeviceGuard g(c->device);
  auto* r = new ffx_replica;
  r->device = c->device;
  r->owner_pid = getpid();
  r->owned = true;
  r->origin = origin;
  r->capacity = capacity;
  r->slice_bytes = c->slice_bytes;
  r->versions = versions;
  r->layout = make_layout(capacity, c->slice_bytes);
  r->cache.assign(versions, SlotCache{});
  r->ctx = c;
  const uint64_t total = r->layout.slot_stride * versions;
  cudaError_t e = cudaMalloc(&r->base, total);
  if (e != cudaSuccess) {
    delete r;
    cudaGetLastError();
    return fail(FFX_ENOMEM, "replica_create: cudaMalloc(%llu): %s", (unsigned long long)total,
                cudaGetErrorString(e));
  }
  for (uint32_t v = 0; v < versions; ++v) {
    e = cudaMemset(r->slot(v), 0, kMetaBytes);
    if (e != cudaSuccess) break;
    r->cache[v].known = true;
  }
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(r->base);
    delete r;
    return cuda_fail(e, "replica_create");
  }
  *out = r;
  return FFX_OK;
}

extern "C" int ffx_replica_export(const ffx_replica* r, uint8_t handle[FFX_HANDLE_BYTES]) {
  if (!r || !handle) return fail(FFX_EINVAL, "replica_export: null argument");
  HandleBlob h{};
  h.magic = kHandleMagic;
  h.abi = FFX_ABI_VERSION;
  h.pid = r->owner_pid;
  h.device = r->device;
  h.raw = reinterpret_cast<uint64_t>(r->base);
  h.capacity = r->capacity;
  h.slice_bytes = r->slice_bytes;
  h.versions = r->versions;
  h.dp = r->origin.dp;
  h.pp = r->origin.pp;
  h.tp = r->origin.tp;
  h.layout = r->layout;
  if (r->vmm) {
    h.kind = 1;
    h.fd = r->vmm_fd;
    h.alloc_bytes = r->vmm_bytes;
    if (r->vmm_fd < 0) return fail(FFX_EINVAL, "replica_export: an imported shared replica cannot be re-exported");
  } else if (r->owned) {
    DeviceGuard g(r->device);
    FFX_CUDA(cudaIpcGetMemHandle(&h.ipc, r->base));
  }
  std::memset(handle, 0, FFX_HANDLE_BYTES);
  std::memcpy(handle, &h, sizeof h);
  return FFX_OK;
}

extern "C" int ffx_replica_open(ffx_ctx* c, const uint8_t handle[FFX_HANDLE_BYTES],
                                ffx_replica** out) {
  if (!c || !handle || !out) return fail(FFX_EINVAL, "replica_open: null argument");
  HandleBlob h;
  std::memcpy(&h, handle, sizeof h);
  if (h.magic != kHandleMagic || h.abi != FFX_ABI_VERSION)
    return fail(FFX_EINVAL, "replica_open: not an ffx replica handle");
  DeviceGuard g(c->device);
  auto* r = new ffx_replica;
  r->device = h.device;
  r->owner_pid = h.pid;
  r->origin = ffx_role{h.dp, h.pp, h.tp};
  r->capacity = h.capacity;
  r->slice_bytes = h.slice_bytes;
  r->versions = h.versions;
  r->layout = h.layout;
  r->cache.assign(h.versions, SlotCache{});
  r->ctx = c;
  if (h.kind == 1) {
    int st = open_shared(c, h, r);
    if (st) {
      delete r;
      return st;
    }
  } else if (h.pid == getpid()) {
    r->base = reinterpret_cast<uint8_t*>(h.raw);
    if (h.device != c->device) {
      int can = 0;
      FFX_CUDA(cudaDeviceCanAccessPeer(&can, c->device, h.device));
      if (!can) {
        delete r;
        return fail(FFX_ECONFIG, "device %d cannot access peer %d", c->device, h.device);
      }
      cudaError_t e = cudaDeviceEnablePeerAccess(h.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) {
        delete r;
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
    }
  } else {
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      delete r;
      return cuda_fail(e, "cudaIpcOpenMemHandle");
    }
    r->base = static_cast<uint8_t*>(p);
    r->ipc_opened = true;
  }
  int st = refresh_cache(r);
  if (st) {
    ffx_replica_destroy(r);
    return st;
  }
  *out = r;
  return FFX_OK;
}

extern "C" int ffx_replica_destroy(ffx_replica* r) {
  if (!r) return FFX_OK;
  if (r->ctx && r->ctx->target == r) r->ctx->target = nullptr;
  if (r->ctx && r->ctx->target2 == r) r->ctx->target2 = nullptr;
  if (r->ctx && r->ctx->last_target == r) r->ctx->last_target = nullptr;
  DeviceGuard g(r->ctx ? r->ctx->device : r->device);
  if (r->vmm) {
    cudaDeviceSynchronize();
    release_shared(r);
  } else {
    if (r->owned && r->base) cudaFree(r->base);
    if (r->ipc_opened && r->base) cudaIpcCloseMemHandle(r->base);
  }
  delete r;
  return FFX_OK;
}

extern "C" int ffx_replica_slots(const ffx_replica* r, uint32_t* versions) {
  if (!r || !versions) return fail(FFX_EINVAL, "replica_slots: null argument");
  *versions = r->versions;
  return FFX_OK;
}

extern "C" int ffx_replica_slot_info(ffx_replica* r, uint32_t slot, ffx_slot_info* out) {
  if (!r || !out) return fail(FFX_EINVAL, "slot_info: null argument");
  if (slot >= r->versions) return fail(FFX_ERANGE, "slot_info: slot %u of %u", slot, r->versions);
  SlotMeta m;
  int st = read_meta(r, slot, &m);
  if (st) return st;
  std::memset(out, 0, sizeof *out);
  if (m.magic != kSlotMagic) return FFX_OK;  // never written: empty
  out->state = m.state;
  out->num_regions = m.num_regions;
  out->role = ffx_role{m.dp, m.pp, m.tp};
  out->kind = m.kind;
  out->whole_checksum_valid = m.whole_checksum_valid;
  out->iteration = m.iteration;
  out->payload_len = m.payload_len;
  out->slice_bytes = m.slice_bytes;
  out->num_slices = m.num_slices;
  out->whole_checksum = m.whole_checksum;
  out->seq = m.seq;
  return FFX_OK;
}

extern "C" int ffx_replica_newest(ffx_replica* r, uint64_t* iteration) {
  if (!r || !iteration) return fail(FFX_EINVAL, "replica_newest: null argument");
  uint64_t best_seq = 0;
  bool any = false;
  for (uint32_t v = 0; v < r->versions; ++v) {
    SlotMeta m;
    int st = read_meta(r, v, &m);
    if (st) return st;
    if (m.magic == kSlotMagic && m.state == kSlotCommitted && (!any || m.seq > best_seq)) {
      any = true;
      best_seq = m.seq;
      *iteration = m.iteration;
    }
  }
  if (!any) return fail(FFX_ERESTORE, "replica holds no committed snapshot");
  return FFX_OK;
}

extern "C" int ffx_replica_slot_ptrs(ffx_replica* r, uint32_t slot, void** payload, uint64_t** sums) {
  if (!r) return fail(FFX_EINVAL, "slot_ptrs: null replica");
  if (slot >= r->versions) return fail(FFX_ERANGE, "slot_ptrs: slot %u of %u", slot, r->versions);
  if (payload) *payload = r->payload(slot);
  if (sums) *sums = r->sums(slot);
  return FFX_OK;
}

extern "C" int ffx_replica_clear(ffx_replica* r) {
  if (!r) return fail(FFX_EINVAL, "replica_clear: null replica");
  DeviceGuard g(r->ctx ? r->ctx->device : r->device);
  for (uint32_t v = 0; v < r->versions; ++v) {
    FFX_CUDA(cudaMemset(r->slot(v), 0, kMetaBytes));
    r->cache[v] = SlotCache{true, kSlotEmpty, 0, 0};
  }
  FFX_CUDA(cudaDeviceSynchronize());
  return FFX_OK;
}

namespace {

// Locate the slot holding `iteration` in any state.  -1 when absent.
int find_slot(ffx_replica* r, uint64_t iteration, SlotMeta* meta) {
  int found = -1;
  uint64_t best_seq = 0;
  for (uint32_t v = 0; v < r->versions; ++v) {
    SlotMeta m;
    if (read_meta(r, v, &m)) return -2;
    if (m.magic != kSlotMagic || m.state == kSlotEmpty || m.iteration != iteration) continue;
    // Prefer a committed copy; among equals the newest write.
    const bool better = found < 0 || (m.state == kSlotCommitted && meta->state != kSlotCommitted) ||
                        (m.state == meta->state && m.seq > best_seq);
    if (better) {
      found = static_cast<int>(v);
      best_seq = m.seq;
      *meta = m;
    }
  }
  return found;
}

}  // namespace

extern "C" int ffx_replica_export_frame(ffx_replica* r, uint64_t iteration, void* host_dst,
                                        uint64_t cap, uint64_t* framed_len, void* stream) {
  if (!r || !framed_len) return fail(FFX_EINVAL, "export_frame: null argument");
  DeviceGuard g(r->ctx ? r->ctx->device : r->device);
  SlotMeta m;
  const int v = find_slot(r, iteration, &m);
  if (v == -2) return fail(FFX_ECUDA, "export_frame: cannot read slot metadata: %s", g_err.c_str());
  if (v < 0 || m.state != kSlotCommitted)
    return fail(FFX_ERESTORE, "no committed snapshot at iteration %llu", (unsigned long long)iteration);
  if (m.payload_len > 0xffffffffull)
    return fail(FFX_EINVAL, "snapshot payload exceeds 4 GiB framing limit");
  *framed_len = 32 + m.payload_len;
  if (!host_dst) return FFX_OK;  // size query
  if (cap < *framed_len) return fail(FFX_ECONFIG, "export_frame: buffer of %llu < %llu bytes",
                                     (unsigned long long)cap, (unsigned long long)*framed_len);
  cudaStream_t s = as_stream(stream);
  uint8_t* pay = r->payload(static_cast<uint32_t>(v));
  // Region offsets inside the slot payload (256-byte aligned, registration order).
  std::vector<uint64_t> offs, lens;
  uint64_t phys = 0;
  for (uint32_t i = 0; i < m.num_regions; ++i) {
    offs.push_back(phys);
    lens.push_back(m.region_bytes[i]);
    phys = align_up(phys + m.region_bytes[i], kRegionAlign);
  }
  if (!m.whole_checksum_valid) {
    uint64_t h = kFnvBasis;
    for (size_t i = 0; i < offs.size(); ++i) {
      cudaError_t e = whole_fnv(pay + offs[i], lens[i], h, &h, s);
      if (e != cudaSuccess) return cuda_fail(e, "whole_fnv");
    }
    m.whole_checksum = h;
    m.whole_checksum_valid = 1;
    // Persist into the slot meta and the SNP1 header so later exports are free.
    uint8_t hdr[32];
    int st = ffx_pack_header(ffx_role{m.dp, m.pp, m.tp}, m.iteration, m.kind, m.payload_len, h, hdr);
    if (st) return st;
    FFX_CUDA(cudaMemcpyAsync(r->slot(v) + offsetof(SlotMeta, whole_checksum), &m.whole_checksum, 8,
                             cudaMemcpyHostToDevice, s));
    FFX_CUDA(cudaMemcpyAsync(r->slot(v) + offsetof(SlotMeta, whole_checksum_valid),
                             &m.whole_checksum_valid, 1, cudaMemcpyHostToDevice, s));
    FFX_CUDA(cudaMemcpyAsync(pay - 32, hdr, 32, cudaMemcpyHostToDevice, s));
    FFX_CUDA(cudaStreamSynchronize(s));
  }
  uint8_t* dst = static_cast<uint8_t*>(host_dst);
  FFX_CUDA(cudaMemcpyAsync(dst, pay - 32, 32, cudaMemcpyDeviceToHost, s));
  uint64_t o = 32;
  for (size_t i = 0; i < offs.size(); ++i) {
    if (lens[i]) FFX_CUDA(cudaMemcpyAsync(dst + o, pay + offs[i], lens[i], cudaMemcpyDeviceToHost, s));
    o += lens[i];
  }
  FFX_CUDA(cudaStreamSynchronize(s));
  return FFX_OK;
}

// Payloads above the SNP1 length field (storage.cpp:48-49 throws) leave as
// several frames: part i carries logical payload bytes
// [i*FFX_FRAME_PART_BYTES, ...) of the concatenated regions, with its own
// header (same role / iteration / kind, the part's length and FNV).
extern "C" int ffx_replica_export_frame_part(ffx_replica* r, uint64_t iteration, uint32_t part, void* host_dst,
                                             uint64_t cap, uint64_t* framed_len, uint32_t* parts, void* stream) {
  if (!r || !framed_len) return fail(FFX_EINVAL, "export_frame_part: null argument");
  DeviceGuard g(r->ctx ? r->ctx->device : r->device);
  SlotMeta m;
  const int v = find_slot(r, iteration, &m);
  if (v == -2) return fail(FFX_ECUDA, "export_frame_part: cannot read slot metadata: %s", g_err.c_str());
  if (v < 0 || m.state != kSlotCommitted)
    return fail(FFX_ERESTORE, "no committed snapshot at iteration %llu", (unsigned long long)iteration);
  const uint64_t F = FFX_FRAME_PART_BYTES;
  const uint32_t n_parts = m.payload_len ? static_cast<uint32_t>((m.payload_len + F - 1) / F) : 1;
  if (parts) *parts = n_parts;
  if (part >= n_parts) return fail(FFX_ERANGE, "export_frame_part: part %u of %u", part, n_parts);
  const uint64_t a = static_cast<uint64_t>(part) * F;
  const uint64_t b = std::min<uint64_t>(m.payload_len, a + F);
  *framed_len = 32 + (b - a);
  if (!host_dst) return FFX_OK;  // size query
  if (cap < *framed_len) return fail(FFX_ECONFIG, "export_frame_part: buffer of %llu < %llu bytes",
                                     (unsigned long long)cap, (unsigned long long)*framed_len);
  cudaStream_t s = as_stream(stream);
  const uint8_t* pay = r->payload(static_cast<uint32_t>(v));
  // the logical range [a, b) as pieces of the (256-byte aligned) regions
  struct Piece { const uint8_t* p; uint64_t n; };
  std::vector<Piece> pieces;
  uint64_t phys = 0, logical = 0;
  for (uint32_t i = 0; i < m.num_regions; ++i) {
    const uint64_t lo = std::max(a, logical), hi = std::min(b, logical + m.region_bytes[i]);
    if (lo < hi) pieces.push_back(Piece{pay + phys + (lo - logical), hi - lo});
    logical += m.region_bytes[i];
    phys = align_up(phys + m.region_bytes[i], kRegionAlign);
  }
  uint64_t h = kFnvBasis;
  for (const Piece& pc : pieces) {
    cudaError_t e = whole_fnv(pc.p, pc.n, h, &h, s);
    if (e != cudaSuccess) return cuda_fail(e, "whole_fnv");
  }
  uint8_t* dst = static_cast<uint8_t*>(host_dst);
  int st = ffx_pack_header(ffx_role{m.dp, m.pp, m.tp}, m.iteration, m.kind, b - a, h, dst);
  if (st) return st;
  uint64_t o = 32;
  for (const Piece& pc : pieces) {
    FFX_CUDA(cudaMemcpyAsync(dst + o, pc.p, pc.n, cudaMemcpyDeviceToHost, s));
    o += pc.n;
  }
  FFX_CUDA(cudaStreamSynchronize(s));
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// snapshot

extern "C" int ffx_snapshot_target(ffx_ctx* c, ffx_replica* t) {
  if (!c) return fail(FFX_EINVAL, "snapshot_target: null ctx");
  c->target = t;
  if (t) {
    int st = refresh_cache(t);
    if (st) return st;
    for (const auto& sc : t->cache) c->seq = std::max(c->seq, sc.seq);
  }
  return FFX_OK;
}

extern "C" int ffx_snapshot_target2(ffx_ctx* c, ffx_replica* t) {
  if (!c) return fail(FFX_EINVAL, "snapshot_target2: null ctx");
  c->target2 = t;
  if (t) {
    int st = refresh_cache(t);
    if (st) return st;
    for (const auto& sc : t->cache) c->seq = std::max(c->seq, sc.seq);
  }
  return FFX_OK;
}

namespace {

// Two-version rule (ckpt.cpp:46-52, :86-92): replace the slot holding this
// iteration, else an empty slot, else the oldest.
uint32_t pick_slot(const ffx_replica* t, uint64_t iteration) {
  int v = -1;
  for (uint32_t i = 0; i < t->versions; ++i)
    if (t->cache[i].state != kSlotEmpty && t->cache[i].iteration == iteration) v = static_cast<int>(i);
  if (v < 0)
    for (uint32_t i = 0; i < t->versions && v < 0; ++i)
      if (t->cache[i].state == kSlotEmpty) v = static_cast<int>(i);
  if (v < 0) {
    v = 0;
    for (uint32_t i = 1; i < t->versions; ++i)
      if (t->cache[i].seq < t->cache[static_cast<uint32_t>(v)].seq) v = static_cast<int>(i);
  }
  return static_cast<uint32_t>(v);
}

}  // namespace

namespace {

struct SrcRegion {
  const uint8_t* dev;  // local or peer-mapped
  uint64_t bytes;
};

// Shared by push (sources = this rank's registered regions, destination = the
// successor's replica) and pull (sources = the predecessor's regions mapped
// over NVLink, destination = the replica this rank holds).
int begin_impl(ffx_ctx* c, ffx_replica* t, ffx_replica* t2, const std::vector<SrcRegion>& srcs, ffx_role role,
               uint64_t* ack, uint64_t iteration, const ffx_snapshot_opts* o, uint32_t* batches_out) {
  if (c->pending.active)
    return fail(FFX_ESTATE, "snapshot of iteration %llu still has %u batches to issue",
                (unsigned long long)c->pending.iteration, c->pending.batches - c->pending.next);
  if (srcs.size() > kMaxRegions) return fail(FFX_ECONFIG, "at most %u regions", kMaxRegions);
  ffx_snapshot_opts opts{};
  if (o) opts = *o;
  uint64_t logical = 0, physical = 0, nslices = 0;
  std::vector<uint64_t> offs;
  for (const SrcRegion& r : srcs) {
    offs.push_back(physical);
    logical += r.bytes;
    physical = align_up(physical + r.bytes, kRegionAlign);
    nslices += slices_of(r.bytes, c->slice_bytes);
  }
  for (ffx_replica* rr : {t, t2}) {
    if (!rr) continue;
    if (logical > rr->capacity)
      return fail(FFX_ECONFIG, "snapshot payload %llu exceeds the replica buffer of %llu bytes",
                  (unsigned long long)logical, (unsigned long long)rr->capacity);
    if (physical > rr->layout.payload_cap)
      return fail(FFX_ECONFIG, "snapshot regions need %llu payload bytes, slot has %llu",
                  (unsigned long long)physical, (unsigned long long)rr->layout.payload_cap);
    if (nslices > rr->layout.table_cap)
      return fail(FFX_ECONFIG, "snapshot needs %llu checksum entries, slot has %llu",
                  (unsigned long long)nslices, (unsigned long long)rr->layout.table_cap);
  }
  const uint32_t slot = pick_slot(t, iteration);
  const uint32_t slot2 = t2 ? pick_slot(t2, iteration) : 0;
  uint64_t seq = ++c->seq;
  for (ffx_replica* rr : {t, t2})
    if (rr)
      for (const auto& sc : rr->cache) seq = std::max(seq, sc.seq + 1);
  c->seq = seq;

  PendingSnapshot& P = c->pending;
  P = PendingSnapshot{};
  P.tgt = t;
  P.tgt2 = t2;
  SliceJob& job = P.job;
  job.nregions = static_cast<uint32_t>(srcs.size());
  for (size_t i = 0; i < srcs.size(); ++i)
    job.reg[i] = SliceRegion{srcs[i].dev, t->wpayload(slot) + offs[i], srcs[i].bytes, 0, 0};
  job.slice_bytes = c->slice_bytes;
  job.sums_out = t->wsums(slot);
  job.sched = c->done + 8;  // dynamic task counter (words 8-9 of the ctx scratch)
  finalize_job(job);

  SlotMeta m{};
  m.magic = kSlotMagic;
  m.state = kSlotCommitted;
  m.iteration = iteration;
  m.seq = seq;
  m.payload_len = logical;
  m.slice_bytes = c->slice_bytes;
  m.num_slices = nslices;
  m.dp = role.dp;
  m.pp = role.pp;
  m.tp = role.tp;
  m.kind = opts.weights_kind ? 0 : 1;
  m.num_regions = job.nregions;
  for (size_t i = 0; i < srcs.size(); ++i) m.region_bytes[i] = srcs[i].bytes;
  uint8_t hdr[32];
  ffx_pack_header(role, iteration, m.kind, logical > 0xffffffffull ? 0 : logical, 0, hdr);

  SlotCommit& cm = job.commit;
  cm.slot = t->wslot(slot);
  cm.done = c->done;
  cm.payload_off = t->layout.payload_off;
  cm.iteration = iteration;
  cm.seq = seq;
  std::memcpy(cm.meta, &m, sizeof m);
  std::memcpy(cm.snp1, hdr, 32);
  cm.ack = ack;
  cm.ack_value = iteration;
  if (t2) {
    // Double-neighbour replication: the same tiles stored twice, one table
    // per replica, each slot committed by its own counter.
    for (size_t i = 0; i < srcs.size(); ++i) job.reg[i].dst2 = t2->wpayload(slot2) + offs[i];
    job.sums_out2 = t2->wsums(slot2);
    job.commit2 = cm;
    job.commit2.slot = t2->wslot(slot2);
    job.commit2.done = c->done + 4;
    job.commit2.payload_off = t2->layout.payload_off;
    P.slot2 = slot2;
  }

  P.active = true;
  P.batches = std::max<uint32_t>(1, opts.batches);
  P.frac.assign(P.batches + 1, 0.0);
  {
    double sum = 0;
    for (uint32_t b = 0; b < P.batches; ++b) {
      const double w = opts.batch_weights ? opts.batch_weights[b] : 1.0;
      sum += (w > 0 ? w : 0);
      P.frac[b + 1] = sum;
    }
    for (uint32_t b = 0; b <= P.batches; ++b) P.frac[b] = sum > 0 ? P.frac[b] / sum : double(b) / P.batches;
    P.frac[P.batches] = 1.0;
  }
  P.max_ctas = opts.max_ctas;
  P.slot = slot;
  P.iteration = iteration;
  P.seq = seq;
  P.nslices = nslices;
  P.logical = logical;
  P.verify = opts.verify_on_store != 0;
  P.split = opts.split != 0;
  if (P.split && ack) {
    P.active = false;
    return fail(FFX_EINVAL, "pull snapshots are fused (the split policy is push-only)");
  }
  if (P.split) {
    // Copy batches: TMA copy-only (or copy engines) into the slot payload.
    P.copy_engine = opts.copy_engine != 0;
    if (P.copy_engine && t->wbase) {
      P.active = false;
      return fail(FFX_EINVAL, "copy-engine batches cannot target a multicast range (TMA copy batches can)");
    }
    CopyJob& cj = P.copy;
    cj.nregions = job.nregions;
    for (uint32_t i = 0; i < job.nregions; ++i)
      cj.reg[i] = CopyRegion{job.reg[i].src, job.reg[i].dst, job.reg[i].bytes, 0, 0, job.reg[i].dst2};
    finalize_copy_job(cj);
    cj.mark = SlotMark{t->wslot(slot), iteration, seq};
    if (t2) cj.mark2 = SlotMark{t2->wslot(slot2), iteration, seq};
    // Hash batches: the local state hashed straight into the slot's table.
    for (uint32_t i = 0; i < job.nregions; ++i) job.reg[i].dst = nullptr;
    P.hbatches = std::max<uint32_t>(1, opts.hash_batches ? opts.hash_batches : P.batches);
    P.hash_ctas = opts.hash_ctas;
  }
  if (batches_out) *batches_out = P.batches;
  return FFX_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// pull mode: the holder reads the origin's registered regions over NVLink

struct ffx_remote {
  ffx_ctx* ctx = nullptr;  // holder context that opened it
  ffx_role role{};
  std::vector<SrcRegion> regs;
  uint64_t* ack = nullptr;      // origin's ack word (peer-mapped)
  std::vector<void*> opened;    // IPC mappings to close
};

namespace {

constexpr uint32_t kRegionsMagic = 0x47524646u;  // "FFRG"

struct RegionsBlob {
  uint32_t magic, abi;
  int32_t pid, device;
  uint16_t dp, pp, tp, pad_;
  uint32_t nregions;
  cudaIpcMemHandle_t ack_ipc;
  uint64_t ack_off, ack_raw;
  struct Entry {
    cudaIpcMemHandle_t ipc;
    uint64_t off, raw, bytes;
  } r[kMaxRegions];
};
static_assert(sizeof(RegionsBlob) <= FFX_REGIONS_HANDLE_BYTES, "regions handle too large");

template <typename Fn>
Fn driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<Fn>(p);
}

// Allocation base of a device pointer (IPC handles name whole allocations).
int alloc_base(const void* p, uint8_t** base) {
  using Fn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static Fn fn = driver_fn<Fn>("cuMemGetAddressRange");
  if (!fn) return fail(FFX_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
    return fail(FFX_EINVAL, "pointer %p is not device memory", p);
  *base = reinterpret_cast<uint8_t*>(b);
  return FFX_OK;
}

}  // namespace

extern "C" int ffx_regions_export(ffx_ctx* c, uint8_t handle[FFX_REGIONS_HANDLE_BYTES]) {
  if (!c || !handle) return fail(FFX_EINVAL, "regions_export: null argument");
  DeviceGuard g(c->device);
  RegionsBlob b{};
  b.magic = kRegionsMagic;
  b.abi = FFX_ABI_VERSION;
  b.pid = getpid();
  b.device = c->device;
  b.dp = c->self.dp;
  b.pp = c->self.pp;
  b.tp = c->self.tp;
  uint8_t* base = nullptr;
  uint8_t* ack = reinterpret_cast<uint8_t*>(c->done + kAckWord);
  int st = alloc_base(ack, &base);
  if (st) return st;
  FFX_CUDA(cudaIpcGetMemHandle(&b.ack_ipc, base));
  b.ack_off = static_cast<uint64_t>(ack - base);
  b.ack_raw = reinterpret_cast<uint64_t>(ack);
  for (const auto& r : c->regions) {
    if (!r.unique) continue;
    auto& e = b.r[b.nregions++];
    e.bytes = r.bytes;
    e.raw = reinterpret_cast<uint64_t>(r.dev);
    if (r.bytes == 0) continue;
    st = alloc_base(r.dev, &base);
    if (st) return st;
    FFX_CUDA(cudaIpcGetMemHandle(&e.ipc, base));
    e.off = static_cast<uint64_t>(r.dev - base);
  }
  std::memset(handle, 0, FFX_REGIONS_HANDLE_BYTES);
  std::memcpy(handle, &b, sizeof b);
  return FFX_OK;
}

extern "C" int ffx_remote_open(ffx_ctx* c, const uint8_t handle[FFX_REGIONS_HANDLE_BYTES], ffx_remote** out) {
  if (!c || !handle || !out) return fail(FFX_EINVAL, "remote_open: null argument");
  RegionsBlob b;
  std::memcpy(&b, handle, sizeof b);
  if (b.magic != kRegionsMagic || b.abi != FFX_ABI_VERSION)
    return fail(FFX_EINVAL, "remote_open: not an ffx regions handle");
  DeviceGuard g(c->device);
  auto* r = new ffx_remote;
  r->ctx = c;
  r->role = ffx_role{b.dp, b.pp, b.tp};
  const bool local = b.pid == getpid();
  std::vector<std::pair<std::string, uint8_t*>> seen;  // one mapping per exported allocation
  auto map = [&](const cudaIpcMemHandle_t& h, uint8_t** base) -> int {
    const std::string key(reinterpret_cast<const char*>(&h), sizeof h);
    for (const auto& kv : seen)
      if (kv.first == key) {
        *base = kv.second;
        return FFX_OK;
      }
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    r->opened.push_back(p);
    seen.emplace_back(key, static_cast<uint8_t*>(p));
    *base = static_cast<uint8_t*>(p);
    return FFX_OK;
  };
  if (local && b.device != c->device) {
    cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) {
      delete r;
      return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    }
  }
  int st = FFX_OK;
  uint8_t* base = nullptr;
  if (local) {
    r->ack = reinterpret_cast<uint64_t*>(b.ack_raw);
  } else if (!(st = map(b.ack_ipc, &base))) {
    r->ack = reinterpret_cast<uint64_t*>(base + b.ack_off);
  }
  for (uint32_t i = 0; i < b.nregions && !st; ++i) {
    const auto& e = b.r[i];
    if (local || e.bytes == 0) {
      r->regs.push_back(SrcRegion{reinterpret_cast<const uint8_t*>(e.raw), e.bytes});
    } else if (!(st = map(e.ipc, &base))) {
      r->regs.push_back(SrcRegion{base + e.off, e.bytes});
    }
  }
  if (st) {
    ffx_remote_close(r);
    return st;
  }
  *out = r;
  return FFX_OK;
}

extern "C" int ffx_remote_close(ffx_remote* r) {
  if (!r) return FFX_OK;
  DeviceGuard g(r->ctx ? r->ctx->device : 0);
  for (void* p : r->opened) cudaIpcCloseMemHandle(p);
  delete r;
  return FFX_OK;
}

extern "C" int ffx_snapshot_begin_pull(ffx_ctx* c, ffx_remote* origin, ffx_replica* held, uint64_t iteration,
                                       const ffx_snapshot_opts* o, uint32_t* batches_out) {
  if (!c || !origin || !held) return fail(FFX_EINVAL, "snapshot_pull: null argument");
  if (held->origin.dp != origin->role.dp || held->origin.pp != origin->role.pp ||
      held->origin.tp != origin->role.tp)
    return fail(FFX_ECONFIG, "replica is for d%up%ut%u, origin is d%up%ut%u", held->origin.dp, held->origin.pp,
                held->origin.tp, origin->role.dp, origin->role.pp, origin->role.tp);
  return begin_impl(c, held, nullptr, origin->regs, origin->role, origin->ack, iteration, o, batches_out);
}

extern "C" int ffx_snapshot_pull(ffx_ctx* c, ffx_remote* origin, ffx_replica* held, uint64_t iteration,
                                 void* stream, const ffx_snapshot_opts* o) {
  uint32_t batches = 1;
  int st = ffx_snapshot_begin_pull(c, origin, held, iteration, o, &batches);
  if (st) return st;
  auto* gates = o ? static_cast<void**>(o->gate_events) : nullptr;
  for (uint32_t b = 0; b < batches; ++b) {
    uint32_t left = 0;
    st = ffx_snapshot_next_kind(c, FFX_BATCH_COPY, stream, gates ? gates[b] : nullptr, &left);
    if (st) {
      c->pending.active = false;
      return st;
    }
  }
  return FFX_OK;
}

extern "C" int ffx_snapshot_wait_pulled(ffx_ctx* c, uint64_t iteration, void* stream) {
  if (!c) return fail(FFX_EINVAL, "wait_pulled: null ctx");
  using Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
  static Fn fn = driver_fn<Fn>("cuStreamWaitValue64");
  if (!fn) return fail(FFX_ECUDA, "cuStreamWaitValue64 unavailable");
  DeviceGuard g(c->device);
  if (fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(c->done + kAckWord), iteration,
         CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    return fail(FFX_ECUDA, "cuStreamWaitValue64 failed");
  return FFX_OK;
}

extern "C" int ffx_snapshot_begin(ffx_ctx* c, uint64_t iteration, const ffx_snapshot_opts* o,
                                  uint32_t* batches_out) {
  if (!c) return fail(FFX_EINVAL, "snapshot: null ctx");
  if (!c->target) return fail(FFX_ESTATE, "snapshot: no target replica (ffx_snapshot_target)");
  std::vector<SrcRegion> srcs;
  for (const auto& r : c->regions)
    if (r.unique) srcs.push_back(SrcRegion{r.dev, r.bytes});
  return begin_impl(c, c->target, c->target2, srcs, c->self, nullptr, iteration, o, batches_out);
}

namespace {

// Holder-side re-verification of a landed slot (NeighborBuffer::store
// validates before accepting, ckpt.cpp:78): one HBM read of the replica.
int verify_landed(ffx_ctx* c, const PendingSnapshot& P, cudaStream_t s) {
  const unsigned long long init[2] = {~0ull, 0ull};
  FFX_CUDA(cudaMemcpyAsync(c->result, init, sizeof init, cudaMemcpyHostToDevice, s));
  SliceJob vj = P.job;
  // A multicast target is written through its multicast range but read back
  // through one holder's unicast mapping.
  const ffx_replica* t = P.tgt;
  auto readable = [t](const uint8_t* p) { return t->wbase ? t->base + (p - t->wbase) : p; };
  for (uint32_t i = 0; i < vj.nregions; ++i) {
    vj.reg[i].src = readable(P.split ? P.copy.reg[i].dst : vj.reg[i].dst);  // the landed payload
    vj.reg[i].dst = nullptr;
    vj.reg[i].dst2 = nullptr;
  }
  vj.sums_out = nullptr;
  vj.sums_out2 = nullptr;
  vj.sums_expected = reinterpret_cast<const uint64_t*>(readable(reinterpret_cast<const uint8_t*>(P.job.sums_out)));
  vj.result = c->result;
  vj.sched = c->done + 12;
  vj.commit = SlotCommit{};
  vj.group_lo = 0;
  vj.group_hi = vj.total_groups;
  FFX_CUDA(launch_slices(vj, SliceMode::HashVerify, false, P.max_ctas, s));
  c->stats.kernel_launches++;
  FFX_CUDA(cudaMemcpyAsync(c->result_host, c->result, 16, cudaMemcpyDeviceToHost, s));
  FFX_CUDA(cudaStreamSynchronize(s));
  if (c->result_host[1]) {
    c->stats.verify_failures++;
    return fail(FFX_ECORRUPT, "snapshot verify-on-store: %llu bad slices (first %llu)",
                c->result_host[1], c->result_host[0]);
  }
  return FFX_OK;
}

}  // namespace

namespace {

// Split policy: one copy batch (TMA copy-only kernel, or copy engines).
int issue_copy_batch(ffx_ctx* c, PendingSnapshot& P, uint32_t b, cudaStream_t s) {
  CopyJob bj = P.copy;
  const uint64_t n = P.copy.total_chunks;
  bj.chunk_lo = P.cut(n, b);
  bj.chunk_hi = P.cut(n, b + 1);
  if (bj.chunk_lo == bj.chunk_hi) return FFX_OK;
  if (!P.copy_engine) {
    FFX_CUDA(launch_copy(bj, P.max_ctas, s));
    c->stats.kernel_launches++;
    return FFX_OK;
  }
  // Copy engines: no SMs at all.  Mark WRITING first with a (tiny) copy
  // kernel over zero chunks, then one cudaMemcpyAsync per region piece.
  CopyJob mark = bj;
  mark.chunk_lo = mark.chunk_hi = 0;
  FFX_CUDA(launch_copy(mark, 1, s));
  for (uint32_t r = 0; r < bj.nregions; ++r) {
    const uint64_t c0 = std::max(bj.chunk_lo, bj.chunk_base[r]);
    const uint64_t cend = (r + 1 < bj.nregions) ? bj.chunk_base[r + 1] : bj.total_chunks;
    const uint64_t c1 = std::min(bj.chunk_hi, cend);
    if (c0 >= c1) continue;
    const uint64_t off = (c0 - bj.chunk_base[r]) * (32 * 1024);
    const uint64_t end = std::min(bj.reg[r].bytes, (c1 - bj.chunk_base[r]) * (32 * 1024));
    FFX_CUDA(cudaMemcpyAsync(bj.reg[r].dst + off, bj.reg[r].src + off, end - off, cudaMemcpyDefault, s));
    if (bj.reg[r].dst2)
      FFX_CUDA(cudaMemcpyAsync(bj.reg[r].dst2 + off, bj.reg[r].src + off, end - off, cudaMemcpyDefault, s));
  }
  return FFX_OK;
}

// Split policy: one hash batch (local state -> checksum table in the slot).
int issue_hash_batch(ffx_ctx* c, PendingSnapshot& P, uint32_t b, cudaStream_t s) {
  SliceJob hj = P.job;
  const uint64_t G = P.job.total_groups;
  hj.group_lo = G * b / P.hbatches;
  hj.group_hi = G * (b + 1) / P.hbatches;
  hj.commit.finalize = 0;
  hj.sched = c->done + 16;
  if (hj.group_lo == hj.group_hi) return FFX_OK;
  FFX_CUDA(launch_slices(hj, SliceMode::Hash, true, P.hash_ctas, s));
  c->stats.kernel_launches++;
  return FFX_OK;
}

int finish_snapshot(ffx_ctx* c, PendingSnapshot& P, cudaStream_t s) {
  P.active = false;
  ffx_replica* t = P.tgt;
  t->cache[P.slot] = SlotCache{true, kSlotCommitted, P.iteration, P.seq};
  if (P.tgt2) P.tgt2->cache[P.slot2] = SlotCache{true, kSlotCommitted, P.iteration, P.seq};
  c->last_target = t;
  c->last_slot = P.slot;
  c->last_nslices = P.nslices;
  c->stats.snapshots++;
  c->stats.snapshot_bytes += P.logical;
  return P.verify ? verify_landed(c, P, s) : FFX_OK;
}

}  // namespace

extern "C" int ffx_snapshot_next_kind(ffx_ctx* c, int kind, void* stream, void* gate_event,
                                      uint32_t* remaining) {
  if (!c) return fail(FFX_EINVAL, "snapshot_next: null ctx");
  PendingSnapshot& P = c->pending;
  if (!P.active) return fail(FFX_ESTATE, "snapshot_next: no snapshot in progress (ffx_snapshot_begin)");
  if (kind != FFX_BATCH_COPY && kind != FFX_BATCH_HASH) return fail(FFX_EINVAL, "snapshot_next: kind %d", kind);
  if (kind == FFX_BATCH_HASH && !P.split) return fail(FFX_ESTATE, "snapshot_next: hash batches need opts.split");
  DeviceGuard g(c->device);
  cudaStream_t s = as_stream(stream);
  uint32_t* next = kind == FFX_BATCH_COPY ? &P.next : &P.hnext;
  const uint32_t total = kind == FFX_BATCH_COPY ? P.batches : P.hbatches;
  if (*next >= total) return fail(FFX_ESTATE, "snapshot_next: no %s batches left", kind ? "hash" : "copy");
  if (gate_event) FFX_CUDA(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(gate_event), 0));
  const uint32_t b = (*next)++;

  if (!P.split) {
    // Fused: batch b covers warp tasks [G*b/B, G*(b+1)/B); the last commits.
    const uint64_t G = P.job.total_groups;
    SliceJob bj = P.job;
    bj.group_lo = P.cut(G, b);
    bj.group_hi = P.cut(G, b + 1);
    bj.commit.finalize = (b + 1 == P.batches);
    bj.commit2.finalize = bj.commit.finalize;
    if (bj.group_lo != bj.group_hi || bj.commit.finalize) {
      FFX_CUDA(launch_slices(bj, SliceMode::Copy, true, P.max_ctas, s));
      c->stats.kernel_launches++;
    }
    if (remaining) *remaining = P.batches - P.next;
    return P.next < P.batches ? FFX_OK : finish_snapshot(c, P, s);
  }

  int st = kind == FFX_BATCH_COPY ? issue_copy_batch(c, P, b, s) : issue_hash_batch(c, P, b, s);
  if (st) return st;
  if (remaining) *remaining = total - *next;
  if (*next == total) FFX_CUDA(cudaEventRecord(kind == FFX_BATCH_COPY ? c->copy_done : c->hash_done, s));
  if (P.next < P.batches || P.hnext < P.hbatches) return FFX_OK;
  // Both queues drained: join the other queue's stream, then commit.
  FFX_CUDA(cudaStreamWaitEvent(s, kind == FFX_BATCH_COPY ? c->hash_done : c->copy_done, 0));
  FFX_CUDA(launch_commit(P.job.commit, s));
  if (P.job.commit2.slot) FFX_CUDA(launch_commit(P.job.commit2, s));
  c->stats.kernel_launches++;
  return finish_snapshot(c, P, s);
}

extern "C" int ffx_snapshot_next(ffx_ctx* c, void* stream, void* gate_event, uint32_t* remaining) {
  if (!c) return fail(FFX_EINVAL, "snapshot_next: null ctx");
  PendingSnapshot& P = c->pending;
  if (!P.active) return fail(FFX_ESTATE, "snapshot_next: no snapshot in progress (ffx_snapshot_begin)");
  // Split mode: copy batches first, then hash batches.
  const int kind = (P.split && P.next >= P.batches) ? FFX_BATCH_HASH : FFX_BATCH_COPY;
  uint32_t left = 0;
  int st = ffx_snapshot_next_kind(c, kind, stream, gate_event, &left);
  if (remaining) *remaining = (P.batches - P.next) + (P.split ? P.hbatches - P.hnext : 0);
  return st;
}

extern "C" int ffx_snapshot(ffx_ctx* c, uint64_t iteration, void* stream, const ffx_snapshot_opts* o) {
  uint32_t batches = 1;
  int st = ffx_snapshot_begin(c, iteration, o, &batches);
  if (st) return st;
  auto* gates = o ? static_cast<void**>(o->gate_events) : nullptr;
  // Copy (or fused) batches on their gates, then -- split policy -- the hash
  // batches on the same stream.
  const uint32_t hb = c->pending.split ? c->pending.hbatches : 0;
  for (uint32_t b = 0; b < batches + hb; ++b) {
    uint32_t left = 0;
    st = ffx_snapshot_next_kind(c, b < batches ? FFX_BATCH_COPY : FFX_BATCH_HASH, stream,
                                (gates && b < batches) ? gates[b] : nullptr, &left);
    if (st) {
      c->pending.active = false;
      return st;
    }
  }
  return FFX_OK;
}

extern "C" int ffx_snapshot_read_sums(ffx_ctx* c, uint64_t* host_dst, uint64_t max_entries,
                                      uint64_t* n_out, void* stream) {
  if (!c || !n_out) return fail(FFX_EINVAL, "snapshot_read_sums: null argument");
  if (!c->last_target || !c->stats.snapshots) return fail(FFX_ESTATE, "snapshot_read_sums: no snapshot taken");
  const uint64_t n = std::min(max_entries, c->last_nslices);
  *n_out = n;
  if (n && host_dst) {
    DeviceGuard g(c->device);
    FFX_CUDA(cudaMemcpyAsync(host_dst, c->last_target->sums(c->last_slot), n * 8, cudaMemcpyDefault,
                             as_stream(stream)));
  }
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// recovery

namespace {

// ckpt.cpp:111-136 (checked): missing, invalid, wrong kind, stale, wrong role,
// plus the B200 layout checks (region count / sizes match the registry).
int check_source(ffx_ctx* c, ffx_replica* src, uint64_t target, SlotMeta* m, uint32_t* slot) {
  const int v = find_slot(src, target, m);
  if (v == -2) return fail(FFX_ECUDA, "recover: cannot read replica metadata: %s", g_err.c_str());
  if (v < 0) return fail(FFX_ERESTORE, "unique-state source missing: no snapshot at iteration %llu",
                         (unsigned long long)target);
  *slot = static_cast<uint32_t>(v);
  if (m->state != kSlotCommitted)
    return fail(FFX_ERESTORE, "unique-state source invalid: slot %d torn (write never committed)", v);
  if (m->kind != 1) return fail(FFX_ERESTORE, "unique-state source has the wrong kind");
  if (m->iteration != target)
    return fail(FFX_ERESTORE, "unique-state source is at iteration %llu, want %llu",
                (unsigned long long)m->iteration, (unsigned long long)target);
  if (m->dp != c->self.dp || m->pp != c->self.pp || m->tp != c->self.tp)
    return fail(FFX_ERESTORE, "unique-state source is for d%up%ut%u, want d%up%ut%u", m->dp, m->pp,
                m->tp, c->self.dp, c->self.pp, c->self.tp);
  const PayloadMap pm = payload_map(c);
  if (m->num_regions != pm.regs.size())
    return fail(FFX_ERESTORE, "snapshot has %u regions, %zu registered", m->num_regions, pm.regs.size());
  for (size_t i = 0; i < pm.regs.size(); ++i)
    if (m->region_bytes[i] != pm.regs[i]->bytes)
      return fail(FFX_ERESTORE, "region %zu: snapshot %llu bytes, registered %llu", i,
                  (unsigned long long)m->region_bytes[i], (unsigned long long)pm.regs[i]->bytes);
  return FFX_OK;
}

}  // namespace

extern "C" int ffx_recover_from(ffx_ctx* c, ffx_replica* const* srcs, uint32_t nsrc, uint64_t target,
                                void* stream, ffx_recover_report* rep) {
  if (!c || !srcs || nsrc == 0 || nsrc > 4) return fail(FFX_EINVAL, "recover: 1..4 sources");
  DeviceGuard g(c->device);
  ffx_recover_report local{};
  ffx_recover_report& R = rep ? *rep : local;
  std::memset(&R, 0, sizeof R);
  R.first_bad_slice = ~0ull;
  SlotMeta m[4];
  uint32_t slot[4];
  for (uint32_t i = 0; i < nsrc; ++i) {
    if (!srcs[i]) return fail(FFX_EINVAL, "recover: null source %u", i);
    int st = check_source(c, srcs[i], target, &m[i], &slot[i]);
    if (st) return st;
    if (m[i].slice_bytes != m[0].slice_bytes)
      return fail(FFX_ERESTORE, "sources disagree on the slice size");
  }
  R.slot = slot[0];
  const PayloadMap pm = payload_map(c);
  if (pm.regs.size() * nsrc > kMaxRegions) nsrc = 1;  // not enough region entries to split
  const uint64_t S = m[0].slice_bytes;

  // Parallel peer gathers: region r's slices are cut into nsrc consecutive
  // parts, part i pulled from source i.  Sub-regions keep registration
  // order, so the global slice numbering (and the checksum table) is that
  // of the whole snapshot; every part verifies against source 0's table.
  cudaStream_t s = as_stream(stream);
  SliceJob job{};
  for (size_t r = 0; r < pm.regs.size(); ++r) {
    const uint64_t ns = slices_of(pm.regs[r]->bytes, S);
    for (uint32_t i = 0; i < nsrc; ++i) {
      const uint64_t a = ns * i / nsrc, b = ns * (i + 1) / nsrc;
      const uint64_t lo = a * S, hi = std::min(b * S, pm.regs[r]->bytes);
      if (hi <= lo && !(nsrc == 1)) continue;
      job.reg[job.nregions++] =
          SliceRegion{srcs[i]->payload(slot[i]) + pm.offs[r] + lo, pm.regs[r]->dev + lo, hi - lo, 0, 0};
    }
  }
  job.slice_bytes = S;
  job.sums_expected = srcs[0]->sums(slot[0]);
  job.result = c->result;
  job.sched = c->done + 12;
  finalize_job(job);
  const unsigned long long init[2] = {~0ull, 0ull};
  FFX_CUDA(cudaMemcpyAsync(c->result, init, sizeof init, cudaMemcpyHostToDevice, s));
  FFX_CUDA(cudaEventRecord(c->ev0, s));
  FFX_CUDA(launch_slices(job, SliceMode::CopyVerify, false, 0, s));
  FFX_CUDA(cudaEventRecord(c->ev1, s));
  c->stats.kernel_launches++;
  FFX_CUDA(cudaMemcpyAsync(c->result_host, c->result, 16, cudaMemcpyDeviceToHost, s));
  FFX_CUDA(cudaStreamSynchronize(s));
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  R.seconds = ms * 1e-3;
  R.bytes = pm.logical;
  R.first_bad_slice = c->result_host[0];
  R.bad_slices = c->result_host[1];
  c->stats.recoveries++;
  c->stats.recovered_bytes += pm.logical;
  if (R.bad_slices) {
    c->stats.verify_failures++;
    return fail(FFX_ERESTORE, "unique-state source invalid: snapshot checksum mismatch in %llu "
                "slices (first slice %llu)", (unsigned long long)R.bad_slices,
                (unsigned long long)R.first_bad_slice);
  }
  return FFX_OK;
}

extern "C" int ffx_recover_full(ffx_ctx* c, ffx_replica* const* srcs, uint32_t nsrc, uint64_t target,
                                const ffx_peer_region* redundant, uint32_t nred, void* stream,
                                ffx_recover_report* rep) {
  if (!c || (nsrc && !srcs) || (nred && !redundant) || nsrc > 4) return fail(FFX_EINVAL, "recover_full: bad arguments");
  DeviceGuard g(c->device);
  ffx_recover_report local{};
  ffx_recover_report& R = rep ? *rep : local;
  std::memset(&R, 0, sizeof R);
  R.first_bad_slice = ~0ull;
  SlotMeta m[4];
  uint32_t slot[4];
  for (uint32_t i = 0; i < nsrc; ++i) {
    int st = check_source(c, srcs[i], target, &m[i], &slot[i]);
    if (st) return st;
    if (m[i].slice_bytes != c->slice_bytes)
      return fail(FFX_ERESTORE, "snapshot slice size %llu, context %llu", (unsigned long long)m[i].slice_bytes,
                  (unsigned long long)c->slice_bytes);
  }
  const PayloadMap pm = payload_map(c);
  if (nsrc == 0 && !pm.regs.empty()) return fail(FFX_ERESTORE, "unique-state source missing");
  const uint64_t S = c->slice_bytes;
  // One kernel, every source at once: the unique regions split across the
  // replica holders, each redundant region from its live DP peer (weights,
  // ckpt.cpp:150-152), each part verified against its own source's table.
  SliceJob job{};
  auto add = [&](const uint8_t* src, uint8_t* dst, uint64_t bytes, const uint64_t* expected) -> int {
    if (job.nregions >= kMaxRegions) return fail(FFX_ECONFIG, "recover_full: more than %u parts", kMaxRegions);
    SliceRegion sr{src, dst, bytes, 0, 0};
    sr.expected = expected;
    job.reg[job.nregions++] = sr;
    return FFX_OK;
  };
  uint64_t total = 0;
  for (size_t r = 0; r < pm.regs.size(); ++r) {
    const uint64_t ns = slices_of(pm.regs[r]->bytes, S);
    const uint64_t base = std::accumulate(pm.regs.begin(), pm.regs.begin() + r, uint64_t{0},
                                          [&](uint64_t a, const Region* q) { return a + slices_of(q->bytes, S); });
    for (uint32_t i = 0; i < nsrc; ++i) {
      const uint64_t a = ns * i / nsrc, b = ns * (i + 1) / nsrc;
      const uint64_t lo = a * S, hi = std::min(b * S, pm.regs[r]->bytes);
      if (hi <= lo) continue;
      int st = add(srcs[i]->payload(slot[i]) + pm.offs[r] + lo, pm.regs[r]->dev + lo, hi - lo,
                   srcs[i]->sums(slot[i]) + base + a);
      if (st) return st;
    }
    total += pm.regs[r]->bytes;
  }
  for (uint32_t j = 0; j < nred; ++j) {
    const ffx_peer_region& pr = redundant[j];
    if (pr.region_index >= c->regions.size() || c->regions[pr.region_index].unique)
      return fail(FFX_ERANGE, "recover_full: region %u is not a registered redundant region", pr.region_index);
    if (!pr.src || !pr.sums) return fail(FFX_EINVAL, "recover_full: null peer pointer");
    const Region& reg = c->regions[pr.region_index];
    int st = add(static_cast<const uint8_t*>(pr.src), reg.dev, reg.bytes, pr.sums);
    if (st) return st;
    total += reg.bytes;
  }
  cudaStream_t s = as_stream(stream);
  job.slice_bytes = S;
  job.result = c->result;
  job.sched = c->done + 12;
  finalize_job(job);
  const unsigned long long init[2] = {~0ull, 0ull};
  FFX_CUDA(cudaMemcpyAsync(c->result, init, sizeof init, cudaMemcpyHostToDevice, s));
  FFX_CUDA(cudaEventRecord(c->ev0, s));
  FFX_CUDA(launch_slices(job, SliceMode::CopyVerify, false, 0, s));
  FFX_CUDA(cudaEventRecord(c->ev1, s));
  c->stats.kernel_launches++;
  FFX_CUDA(cudaMemcpyAsync(c->result_host, c->result, 16, cudaMemcpyDeviceToHost, s));
  FFX_CUDA(cudaStreamSynchronize(s));
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  R.seconds = ms * 1e-3;
  R.bytes = total;
  R.slot = nsrc ? slot[0] : 0;
  R.first_bad_slice = c->result_host[0];
  R.bad_slices = c->result_host[1];
  c->stats.recoveries++;
  c->stats.recovered_bytes += total;
  if (R.bad_slices) {
    c->stats.verify_failures++;
    return fail(FFX_ERESTORE, "restore source invalid: checksum mismatch in %llu slices (first %llu)",
                (unsigned long long)R.bad_slices, (unsigned long long)R.first_bad_slice);
  }
  return FFX_OK;
}

extern "C" int ffx_recover(ffx_ctx* c, ffx_replica* src, uint64_t target, void* stream,
                           ffx_recover_report* rep) {
  if (!c || !src) return fail(FFX_EINVAL, "recover: null argument");
  return ffx_recover_from(c, &src, 1, target, stream, rep);
}

extern "C" int ffx_recover_region(ffx_ctx* c, uint32_t idx, const void* peer_src,
                                  const uint64_t* peer_sums, void* stream, ffx_recover_report* rep) {
  if (!c || !peer_src || !peer_sums) return fail(FFX_EINVAL, "recover_region: null argument");
  if (idx >= c->regions.size()) return fail(FFX_ERANGE, "recover_region: no region %u", idx);
  DeviceGuard g(c->device);
  ffx_recover_report local{};
  ffx_recover_report& R = rep ? *rep : local;
  std::memset(&R, 0, sizeof R);
  const Region& reg = c->regions[idx];
  cudaStream_t s = as_stream(stream);
  SliceJob job = single_job(peer_src, reg.dev, reg.bytes, c->slice_bytes);
  job.sums_expected = peer_sums;
  job.result = c->result;
  job.sched = c->done + 12;
  const unsigned long long init[2] = {~0ull, 0ull};
  FFX_CUDA(cudaMemcpyAsync(c->result, init, sizeof init, cudaMemcpyHostToDevice, s));
  FFX_CUDA(cudaEventRecord(c->ev0, s));
  if (reg.bytes) FFX_CUDA(launch_slices(job, SliceMode::CopyVerify, false, 0, s));
  FFX_CUDA(cudaEventRecord(c->ev1, s));
  FFX_CUDA(cudaMemcpyAsync(c->result_host, c->result, 16, cudaMemcpyDeviceToHost, s));
  FFX_CUDA(cudaStreamSynchronize(s));
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  R.seconds = ms * 1e-3;
  R.bytes = reg.bytes;
  R.first_bad_slice = c->result_host[0];
  R.bad_slices = c->result_host[1];
  c->stats.recovered_bytes += reg.bytes;
  if (R.bad_slices)
    return fail(FFX_ERESTORE, "weights source invalid: checksum mismatch in %llu slices",
                (unsigned long long)R.bad_slices);
  return FFX_OK;
}

extern "C" int ffx_ipc_export(void* dev_base, uint8_t handle[64]) {
  if (!dev_base || !handle) return fail(FFX_EINVAL, "ipc_export: null argument");
  cudaIpcMemHandle_t h;
  FFX_CUDA(cudaIpcGetMemHandle(&h, dev_base));
  std::memcpy(handle, &h, 64);
  return FFX_OK;
}

extern "C" int ffx_ipc_open(const uint8_t handle[64], void** dev_base) {
  if (!handle || !dev_base) return fail(FFX_EINVAL, "ipc_open: null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  FFX_CUDA(cudaIpcOpenMemHandle(dev_base, h, cudaIpcMemLazyEnablePeerAccess));
  return FFX_OK;
}

extern "C" int ffx_ipc_close(void* dev_base) {
  if (!dev_base) return FFX_OK;
  FFX_CUDA(cudaIpcCloseMemHandle(dev_base));
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// failure injection + stats

extern "C" int ffx_inject(ffx_ctx* c, int fault, ffx_replica* r, uint64_t arg) {
  if (!c) return fail(FFX_EINVAL, "inject: null ctx");
  DeviceGuard g(c->device);
  switch (fault) {
    case FFX_FAULT_POISON_STATE:
      for (const auto& reg : c->regions)
        if (reg.unique) FFX_CUDA(launch_fill(reg.dev, reg.bytes, 0xDEADBEEFu, nullptr));
      FFX_CUDA(cudaDeviceSynchronize());
      return FFX_OK;
    case FFX_FAULT_CORRUPT_REPLICA: {
      if (!r) return fail(FFX_EINVAL, "inject: replica required");
      const uint32_t slot = static_cast<uint32_t>(arg >> 48);
      const uint64_t off = arg & ((1ull << 48) - 1);
      if (slot >= r->versions) return fail(FFX_ERANGE, "inject: slot %u", slot);
      SlotMeta m;
      int st = read_meta(r, slot, &m);
      if (st) return st;
      // logical offset -> physical (regions are 256-byte aligned in the slot)
      uint64_t phys = 0, logical = off;
      uint32_t i = 0;
      for (; i < m.num_regions; ++i) {
        if (logical < m.region_bytes[i]) break;
        logical -= m.region_bytes[i];
        phys = align_up(phys + m.region_bytes[i], kRegionAlign);
      }
      if (i >= m.num_regions) return fail(FFX_ERANGE, "inject: offset %llu beyond payload",
                                          (unsigned long long)off);
      FFX_CUDA(launch_xor_byte(r->payload(slot) + phys + logical, 0x01, nullptr));
      FFX_CUDA(cudaDeviceSynchronize());
      return FFX_OK;
    }
    case FFX_FAULT_TEAR_SLOT: {
      if (!r) return fail(FFX_EINVAL, "inject: replica required");
      if (arg >= r->versions) return fail(FFX_ERANGE, "inject: slot %llu", (unsigned long long)arg);
      const uint32_t st = kSlotWriting;
      FFX_CUDA(cudaMemcpy(r->slot(static_cast<uint32_t>(arg)) + offsetof(SlotMeta, state), &st, 4,
                          cudaMemcpyHostToDevice));
      r->cache[arg].state = kSlotWriting;
      return FFX_OK;
    }
    case FFX_FAULT_CORRUPT_SUMS: {
      if (!r) return fail(FFX_EINVAL, "inject: replica required");
      const uint32_t slot = static_cast<uint32_t>(arg >> 48);
      const uint64_t idx = arg & ((1ull << 48) - 1);
      if (slot >= r->versions || idx >= r->layout.table_cap)
        return fail(FFX_ERANGE, "inject: slot/index out of range");
      FFX_CUDA(launch_xor_byte(reinterpret_cast<uint8_t*>(r->sums(slot) + idx), 0x80, nullptr));
      FFX_CUDA(cudaDeviceSynchronize());
      return FFX_OK;
    }
  }
  return fail(FFX_EINVAL, "inject: unknown fault %d", fault);
}

extern "C" int ffx_get_stats(ffx_ctx* c, ffx_stats* out) {
  if (!c || !out) return fail(FFX_EINVAL, "stats: null argument");
  *out = c->stats;
  return FFX_OK;
}

// ---------------------------------------------------------------------------
// shareable replicas + NVSwitch multicast: the double neighbour with one
// egress per tile (measured feasible on the box first,
// profiles/r1_multicast_probe_4gpu.jsonl: TMA bulk stores into a multicast
// range reach every bound member, 564 GB/s for two replicas vs 355 GB/s per
// copy for two unicast stores).

namespace {

struct Drv {
  decltype(&cuMemCreate) memCreate;
  decltype(&cuMemRelease) memRelease;
  decltype(&cuMemAddressReserve) addressReserve;
  decltype(&cuMemAddressFree) addressFree;
  decltype(&cuMemMap) memMap;
  decltype(&cuMemUnmap) memUnmap;
  decltype(&cuMemSetAccess) setAccess;
  decltype(&cuMemExportToShareableHandle) exportHandle;
  decltype(&cuMemImportFromShareableHandle) importHandle;
  decltype(&cuMemGetAllocationGranularity) allocGran;
  decltype(&cuMulticastCreate) mcCreate;
  decltype(&cuMulticastAddDevice) mcAddDevice;
  decltype(&cuMulticastBindMem) mcBindMem;
  decltype(&cuMulticastUnbind) mcUnbind;
  decltype(&cuMulticastGetGranularity) mcGran;
  decltype(&cuDeviceGet) deviceGet;
  decltype(&cuDeviceGetAttribute) deviceAttr;
  decltype(&cuGetErrorString) errorString;
  bool ok;
};

const Drv& drv() {
  static const Drv d = [] {
    Drv x{};
    x.memCreate = driver_fn<decltype(&cuMemCreate)>("cuMemCreate");
    x.memRelease = driver_fn<decltype(&cuMemRelease)>("cuMemRelease");
    x.addressReserve = driver_fn<decltype(&cuMemAddressReserve)>("cuMemAddressReserve");
    x.addressFree = driver_fn<decltype(&cuMemAddressFree)>("cuMemAddressFree");
    x.memMap = driver_fn<decltype(&cuMemMap)>("cuMemMap");
    x.memUnmap = driver_fn<decltype(&cuMemUnmap)>("cuMemUnmap");
    x.setAccess = driver_fn<decltype(&cuMemSetAccess)>("cuMemSetAccess");
    x.exportHandle = driver_fn<decltype(&cuMemExportToShareableHandle)>("cuMemExportToShareableHandle");
    x.importHandle = driver_fn<decltype(&cuMemImportFromShareableHandle)>("cuMemImportFromShareableHandle");
    x.allocGran = driver_fn<decltype(&cuMemGetAllocationGranularity)>("cuMemGetAllocationGranularity");
    x.mcCreate = driver_fn<decltype(&cuMulticastCreate)>("cuMulticastCreate");
    x.mcAddDevice = driver_fn<decltype(&cuMulticastAddDevice)>("cuMulticastAddDevice");
    x.mcBindMem = driver_fn<decltype(&cuMulticastBindMem)>("cuMulticastBindMem");
    x.mcUnbind = driver_fn<decltype(&cuMulticastUnbind)>("cuMulticastUnbind");
    x.mcGran = driver_fn<decltype(&cuMulticastGetGranularity)>("cuMulticastGetGranularity");
    x.deviceGet = driver_fn<decltype(&cuDeviceGet)>("cuDeviceGet");
    x.deviceAttr = driver_fn<decltype(&cuDeviceGetAttribute)>("cuDeviceGetAttribute");
    x.errorString = driver_fn<decltype(&cuGetErrorString)>("cuGetErrorString");
    x.ok = x.memCreate && x.memRelease && x.addressReserve && x.addressFree && x.memMap && x.memUnmap &&
           x.setAccess && x.exportHandle && x.importHandle && x.allocGran && x.mcCreate && x.mcAddDevice &&
           x.mcBindMem && x.mcUnbind && x.mcGran && x.deviceGet && x.deviceAttr && x.errorString;
    return x;
  }();
  return d;
}

int drv_fail(CUresult r, const char* what) {
  const char* s = nullptr;
  if (drv().errorString) drv().errorString(r, &s);
  return fail(r == CUDA_ERROR_OUT_OF_MEMORY ? FFX_ENOMEM : FFX_ECUDA, "%s: %s", what, s ? s : "CUDA driver error");
}

#define FFX_DRV(call)                                     \
  do {                                                    \
    CUresult r_ = (call);                                 \
    if (r_ != CUDA_SUCCESS) return drv_fail(r_, #call);   \
  } while (0)

constexpr CUmemAllocationHandleType kShareType = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
constexpr uint32_t kMcastMagic = 0x4d584646u;  // "FFXM"
constexpr uint64_t kSinkMax = 256ull << 20;    // origin's alias sink (see target_mcast)

CUmemAllocationProp share_prop(int device) {
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  ap.requestedHandleTypes = kShareType;
  return ap;
}

// Size unit of shareable replicas and multicast ranges: both the VMM and the
// multicast minimum granularity (2 MiB on B200).
int share_gran(int device, uint64_t* gran) {
  if (!drv().ok) return fail(FFX_ECUDA, "CUDA driver lacks the VMM / multicast entry points");
  CUmemAllocationProp ap = share_prop(device);
  size_t g1 = 0, g2 = 0;
  FFX_DRV(drv().allocGran(&g1, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  CUmulticastObjectProp mp{};
  mp.numDevices = 2;
  mp.handleTypes = kShareType;
  mp.size = g1;
  FFX_DRV(drv().mcGran(&g2, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  *gran = std::max<uint64_t>(g1, g2);
  return FFX_OK;
}

int map_range(CUmemGenericAllocationHandle h, uint64_t bytes, uint64_t align, int device, uint8_t** va) {
  CUdeviceptr p = 0;
  FFX_DRV(drv().addressReserve(&p, bytes, align, 0, 0));
  CUresult r = drv().memMap(p, bytes, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    drv().addressFree(p, bytes);
    return drv_fail(r, "cuMemMap");
  }
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = drv().setAccess(p, bytes, &acc, 1);
  if (r != CUDA_SUCCESS) {
    drv().memUnmap(p, bytes);
    drv().addressFree(p, bytes);
    return drv_fail(r, "cuMemSetAccess");
  }
  *va = reinterpret_cast<uint8_t*>(p);
  return FFX_OK;
}

int grant_access(uint8_t* va, uint64_t bytes, int owner_dev, int other_dev) {
  CUmemAccessDesc acc[2] = {};
  for (int i = 0; i < 2; ++i) {
    acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[i].location.id = i ? other_dev : owner_dev;
    acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  FFX_DRV(drv().setAccess(reinterpret_cast<CUdeviceptr>(va), bytes, acc, 2));
  return FFX_OK;
}

int fetch_or_fail(int pid, int fd, int* out) {
  const int e = fetch_fd(pid, fd, out);
  if (e) return fail(FFX_ECUDA, "cannot fetch fd %d of process %d: %s", fd, pid, std::strerror(e));
  return FFX_OK;
}

}  // namespace

namespace {

int open_shared(ffx_ctx* c, const HandleBlob& h, ffx_replica* r) {
  if (!drv().ok) return fail(FFX_ECUDA, "CUDA driver lacks the VMM entry points");
  r->vmm = true;
  r->vmm_bytes = h.alloc_bytes;
  if (h.pid == getpid()) {  // the owner's own mapping; grant this ctx's device access
    r->base = reinterpret_cast<uint8_t*>(h.raw);
    if (h.device != c->device) return grant_access(r->base, h.alloc_bytes, h.device, c->device);
    return FFX_OK;
  }
  int fd = -1;
  int st = fetch_or_fail(h.pid, h.fd, &fd);
  if (st) return st;
  CUmemGenericAllocationHandle mh = 0;
  CUresult cr = drv().importHandle(&mh, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)), kShareType);
  close(fd);
  if (cr != CUDA_SUCCESS) return drv_fail(cr, "cuMemImportFromShareableHandle");
  uint64_t gran = 0;
  st = share_gran(c->device, &gran);
  if (!st) st = map_range(mh, h.alloc_bytes, gran, c->device, &r->base);
  if (st) {
    drv().memRelease(mh);
    return st;
  }
  r->vmm_handle = mh;
  r->vmm_mapped = true;
  return FFX_OK;
}

void release_shared(ffx_replica* r) {
  if ((r->owned || r->vmm_mapped) && r->base) {
    drv().memUnmap(reinterpret_cast<CUdeviceptr>(r->base), r->vmm_bytes);
    drv().addressFree(reinterpret_cast<CUdeviceptr>(r->base), r->vmm_bytes);
    drv().memRelease(r->vmm_handle);
  }
  if (r->owned && r->vmm_fd >= 0) {
    unshare_fd(r->vmm_fd);
    close(r->vmm_fd);
  }
}

}  // namespace

extern "C" int ffx_mcast_supported(int device, int* supported) {
  if (!supported) return fail(FFX_EINVAL, "mcast_supported: null out");
  *supported = 0;
  if (!drv().ok) return FFX_OK;
  DeviceGuard g(device);
  CUdevice d;
  FFX_DRV(drv().deviceGet(&d, device));
  int v = 0;
  FFX_DRV(drv().deviceAttr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d));
  *supported = v;
  return FFX_OK;
}

extern "C" int ffx_replica_create_shared(ffx_ctx* c, ffx_role origin, uint64_t capacity, uint32_t versions,
                                         ffx_replica** out) {
  if (!c || !out) return fail(FFX_EINVAL, "replica_create_shared: null argument");
  if (versions < 1 || versions > 8) return fail(FFX_EINVAL, "replica_create_shared: 1..8 versions");
  DeviceGuard g(c->device);
  uint64_t gran = 0;
  int st = share_gran(c->device, &gran);
  if (st) return st;
  const SlotLayout L = make_layout(capacity, c->slice_bytes);
  const uint64_t bytes = align_up(L.slot_stride * versions, gran);
  CUmemAllocationProp ap = share_prop(c->device);
  CUmemGenericAllocationHandle h = 0;
  FFX_DRV(drv().memCreate(&h, bytes, &ap, 0));
  auto* r = new ffx_replica;
  r->device = c->device;
  r->owner_pid = getpid();
  r->owned = true;
  r->vmm = true;
  r->vmm_handle = h;
  r->vmm_bytes = bytes;
  r->origin = origin;
  r->capacity = capacity;
  r->slice_bytes = c->slice_bytes;
  r->versions = versions;
  r->layout = L;
  r->cache.assign(versions, SlotCache{});
  r->ctx = c;
  st = map_range(h, bytes, gran, c->device, &r->base);
  if (st) {
    drv().memRelease(h);
    delete r;
    return st;
  }
  int fd = -1;
  CUresult cr = drv().exportHandle(&fd, h, kShareType, 0);
  int e = cr == CUDA_SUCCESS ? share_fd(fd) : 0;
  if (cr != CUDA_SUCCESS || e) {
    if (fd >= 0) close(fd);
    release_shared(r);
    delete r;
    return cr != CUDA_SUCCESS ? drv_fail(cr, "cuMemExportToShareableHandle")
                              : fail(FFX_ECUDA, "fd server: %s", std::strerror(e));
  }
  r->vmm_fd = fd;
  cudaError_t ce = cudaSuccess;
  for (uint32_t v = 0; v < versions && ce == cudaSuccess; ++v) {
    ce = cudaMemset(r->slot(v), 0, kMetaBytes);
    r->cache[v].known = true;
  }
  if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
  if (ce != cudaSuccess) {
    release_shared(r);
    delete r;
    return cuda_fail(ce, "replica_create_shared");
  }
  *out = r;
  return FFX_OK;
}

struct ffx_mcast {
  ffx_ctx* ctx = nullptr;
  int device = 0;
  CUmemGenericAllocationHandle handle = 0;
  uint64_t bytes = 0, gran = 0, capacity = 0, slice_bytes = 0;
  uint32_t versions = 0, members = 0;
  int owner_pid = 0;
  int fd = -1;           // owner: the exported fd
  bool owner = false;
  bool joined = false;
  bool bound = false;    // holder: its replica is bound at offset 0
  uint8_t* va = nullptr; // origin: the multicast range mapped here
  CUmemGenericAllocationHandle sink = 0;  // origin: alias sink (kSinkMax or less)
  uint64_t sink_bytes = 0;
  ffx_replica* target = nullptr;          // origin: view + write-through-range
};

namespace {

struct McastBlob {  // FFX_MCAST_HANDLE_BYTES on the wire
  uint32_t magic, abi;
  int32_t pid, fd;
  uint64_t bytes, capacity, slice_bytes;
  uint32_t versions, members;
};
static_assert(sizeof(McastBlob) <= FFX_MCAST_HANDLE_BYTES, "mcast handle too large");

}  // namespace

extern "C" int ffx_mcast_create(ffx_ctx* c, uint64_t capacity, uint32_t versions, uint32_t members,
                                ffx_mcast** out) {
  if (!c || !out) return fail(FFX_EINVAL, "mcast_create: null argument");
  if (members < 2 || members > 8) return fail(FFX_EINVAL, "mcast_create: 2..8 members");
  if (versions < 1 || versions > 8) return fail(FFX_EINVAL, "mcast_create: 1..8 versions");
  DeviceGuard g(c->device);
  uint64_t gran = 0;
  int st = share_gran(c->device, &gran);
  if (st) return st;
  const SlotLayout L = make_layout(capacity, c->slice_bytes);
  CUmulticastObjectProp mp{};
  mp.numDevices = members;
  mp.handleTypes = kShareType;
  mp.size = align_up(L.slot_stride * versions, gran);
  CUmemGenericAllocationHandle h = 0;
  FFX_DRV(drv().mcCreate(&h, &mp));
  int fd = -1;
  CUresult cr = drv().exportHandle(&fd, h, kShareType, 0);
  const int e = cr == CUDA_SUCCESS ? share_fd(fd) : 0;
  if (cr != CUDA_SUCCESS || e) {
    if (fd >= 0) close(fd);
    drv().memRelease(h);
    return cr != CUDA_SUCCESS ? drv_fail(cr, "cuMemExportToShareableHandle")
                              : fail(FFX_ECUDA, "fd server: %s", std::strerror(e));
  }
  auto* m = new ffx_mcast;
  m->ctx = c;
  m->device = c->device;
  m->handle = h;
  m->bytes = mp.size;
  m->gran = gran;
  m->capacity = capacity;
  m->slice_bytes = c->slice_bytes;
  m->versions = versions;
  m->members = members;
  m->owner_pid = getpid();
  m->fd = fd;
  m->owner = true;
  *out = m;
  return FFX_OK;
}

extern "C" int ffx_mcast_export(const ffx_mcast* m, uint8_t handle[FFX_MCAST_HANDLE_BYTES]) {
  if (!m || !handle) return fail(FFX_EINVAL, "mcast_export: null argument");
  if (!m->owner) return fail(FFX_EINVAL, "mcast_export: only the creating process exports");
  McastBlob b{kMcastMagic, FFX_ABI_VERSION, m->owner_pid, m->fd, m->bytes, m->capacity, m->slice_bytes,
              m->versions, m->members};
  std::memset(handle, 0, FFX_MCAST_HANDLE_BYTES);
  std::memcpy(handle, &b, sizeof b);
  return FFX_OK;
}

extern "C" int ffx_mcast_open(ffx_ctx* c, const uint8_t handle[FFX_MCAST_HANDLE_BYTES], ffx_mcast** out) {
  if (!c || !handle || !out) return fail(FFX_EINVAL, "mcast_open: null argument");
  McastBlob b;
  std::memcpy(&b, handle, sizeof b);
  if (b.magic != kMcastMagic || b.abi != FFX_ABI_VERSION) return fail(FFX_EINVAL, "mcast_open: not an ffx multicast handle");
  if (!drv().ok) return fail(FFX_ECUDA, "CUDA driver lacks the multicast entry points");
  DeviceGuard g(c->device);
  uint64_t gran = 0;
  int st = share_gran(c->device, &gran);
  if (st) return st;
  int fd = -1;
  st = fetch_or_fail(b.pid, b.fd, &fd);
  if (st) return st;
  CUmemGenericAllocationHandle h = 0;
  CUresult cr = drv().importHandle(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)), kShareType);
  close(fd);
  if (cr != CUDA_SUCCESS) return drv_fail(cr, "cuMemImportFromShareableHandle (multicast)");
  auto* m = new ffx_mcast;
  m->ctx = c;
  m->device = c->device;
  m->handle = h;
  m->bytes = b.bytes;
  m->gran = gran;
  m->capacity = b.capacity;
  m->slice_bytes = b.slice_bytes;
  m->versions = b.versions;
  m->members = b.members;
  m->owner_pid = b.pid;
  *out = m;
  return FFX_OK;
}

extern "C" int ffx_mcast_join(ffx_mcast* m) {
  if (!m) return fail(FFX_EINVAL, "mcast_join: null argument");
  if (m->joined) return FFX_OK;
  DeviceGuard g(m->device);
  CUdevice d;
  FFX_DRV(drv().deviceGet(&d, m->device));
  FFX_DRV(drv().mcAddDevice(m->handle, d));
  m->joined = true;
  return FFX_OK;
}

extern "C" int ffx_mcast_bind(ffx_mcast* m, ffx_replica* held) {
  if (!m || !held) return fail(FFX_EINVAL, "mcast_bind: null argument");
  if (!m->joined) return fail(FFX_ESTATE, "mcast_bind: join the team first (ffx_mcast_join)");
  if (!held->vmm || !held->owned) return fail(FFX_EINVAL, "mcast_bind: needs a replica from ffx_replica_create_shared");
  if (held->device != m->device) return fail(FFX_EINVAL, "mcast_bind: replica lives on another device");
  if (held->capacity != m->capacity || held->versions != m->versions || held->slice_bytes != m->slice_bytes ||
      held->vmm_bytes != m->bytes)
    return fail(FFX_ECONFIG, "mcast_bind: replica layout differs from the multicast range");
  if (m->bound) return FFX_OK;
  DeviceGuard g(m->device);
  FFX_DRV(drv().mcBindMem(m->handle, 0, held->vmm_handle, 0, m->bytes, 0));
  m->bound = true;
  return FFX_OK;
}

extern "C" int ffx_snapshot_target_mcast(ffx_ctx* c, ffx_mcast* m, ffx_replica* view) {
  if (!c || !m || !view) return fail(FFX_EINVAL, "snapshot_target_mcast: null argument");
  if (!m->joined) return fail(FFX_ESTATE, "snapshot_target_mcast: join the team first (ffx_mcast_join)");
  if (m->device != c->device) return fail(FFX_EINVAL, "snapshot_target_mcast: multicast object of another device");
  if (view->capacity != m->capacity || view->versions != m->versions || view->slice_bytes != m->slice_bytes ||
      view->slice_bytes != c->slice_bytes)
    return fail(FFX_ECONFIG, "snapshot_target_mcast: view layout differs from the multicast range");
  DeviceGuard g(c->device);
  if (!m->va) {
    // Every member of a team must back the range: the origin binds one small
    // sink repeatedly (aliased) instead of a replica-sized buffer -- without
    // any binding here the stores crawl at ~50 GB/s (measured).
    m->sink_bytes = std::min<uint64_t>(m->bytes, kSinkMax);
    m->sink_bytes = align_up(m->sink_bytes, m->gran);
    while (m->bytes % m->sink_bytes) m->sink_bytes -= m->gran;
    CUmemAllocationProp ap = share_prop(c->device);
    FFX_DRV(drv().memCreate(&m->sink, m->sink_bytes, &ap, 0));
    for (uint64_t o = 0; o < m->bytes; o += m->sink_bytes)
      FFX_DRV(drv().mcBindMem(m->handle, o, m->sink, 0, m->sink_bytes, 0));
    int st = map_range(m->handle, m->bytes, m->gran, c->device, &m->va);
    if (st) return st;
  }
  if (!m->target) {
    auto* t = new ffx_replica;
    t->device = view->device;
    t->owner_pid = view->owner_pid;
    t->origin = view->origin;
    t->capacity = view->capacity;
    t->slice_bytes = view->slice_bytes;
    t->versions = view->versions;
    t->layout = view->layout;
    t->cache.assign(view->versions, SlotCache{});
    t->ctx = c;
    t->base = view->base;
    t->wbase = m->va;
    m->target = t;
  }
  c->target2 = nullptr;
  return ffx_snapshot_target(c, m->target);
}

extern "C" int ffx_mcast_destroy(ffx_mcast* m) {
  if (!m) return FFX_OK;
  DeviceGuard g(m->device);
  cudaDeviceSynchronize();
  if (m->target) {
    if (m->ctx && m->ctx->target == m->target) m->ctx->target = nullptr;
    if (m->ctx && m->ctx->last_target == m->target) m->ctx->last_target = nullptr;
    delete m->target;
  }
  CUdevice d;
  if (drv().ok && drv().deviceGet(&d, m->device) == CUDA_SUCCESS) {
    if (m->va) {
      drv().memUnmap(reinterpret_cast<CUdeviceptr>(m->va), m->bytes);
      drv().addressFree(reinterpret_cast<CUdeviceptr>(m->va), m->bytes);
    }
    if (m->bound || m->sink) drv().mcUnbind(m->handle, d, 0, m->bytes);
    if (m->sink) drv().memRelease(m->sink);
    drv().memRelease(m->handle);
  }
  if (m->owner && m->fd >= 0) {
    unshare_fd(m->fd);
    close(m->fd);
  }
  delete m;
  return FFX_OK;
}
