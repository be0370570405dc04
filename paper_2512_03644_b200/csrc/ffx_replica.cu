// ffx_replica.cu -- the C ABI, part 2: the neighbour replica manager
// (NeighborBuffer, ckpt.hpp:105-120) -- HBM slots, CUDA-IPC export / open,
// slot metadata -- and SNP1 frame export.
#include "ffx_host.h"

namespace ffx::host {

int read_meta(ffx_replica* r, uint32_t v, SlotMeta* m) {
  DeviceGuard g(r->ctx ? r->ctx->device : r->device);
  FFX_CUDA(cudaMemcpy(m, r->slot(v), sizeof(SlotMeta), cudaMemcpyDefault));
  return FFX_OK;
}

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

}  // namespace ffx::host

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
    h.kind = r->vmm_handle2 || r->vmm_fd2 >= 0 ? 2 : 1;
    h.fd = r->vmm_fd;
    h.fd2 = r->vmm_fd2;
    h.tier_hbm = r->tier_hbm;
    h.alloc_bytes = r->vmm_bytes;
    if (!r->owned) return fail(FFX_EINVAL, "replica_export: an imported shared replica cannot be re-exported");
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
  // a damaged handle must not become out-of-bounds slot addressing
  const SlotLayout want = make_layout(h.capacity, h.slice_bytes ? h.slice_bytes : 1);
  if (h.versions < 1 || h.versions > 8 || !slice_ok(h.slice_bytes) || h.kind > 2 ||
      std::memcmp(&want, &h.layout, sizeof want) != 0)
    return fail(FFX_EINVAL, "replica_open: inconsistent replica handle");
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
  if (h.kind == 1 || h.kind == 2) {
    int st = open_shared(c, h, r);
    if (st) {
      delete r;
      return st;
    }
  } else if (h.pid == getpid()) {
    r->base = reinterpret_cast<uint8_t*>(h.raw);
    if (h.device != c->device) {
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, c->device, h.device) != cudaSuccess) {
        cudaGetLastError();
        can = 0;
      }
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

extern "C" int ffx_replica_slot_regions(ffx_replica* r, uint32_t slot, uint32_t* n, int32_t* kinds,
                                        uint64_t* bytes) {
  if (!r || !n) return fail(FFX_EINVAL, "slot_regions: null argument");
  if (slot >= r->versions) return fail(FFX_ERANGE, "slot_regions: slot %u of %u", slot, r->versions);
  SlotMeta m;
  int st = read_meta(r, slot, &m);
  if (st) return st;
  *n = 0;
  if (m.magic != kSlotMagic || m.state != kSlotCommitted)
    return fail(FFX_ERESTORE, "slot_regions: slot %u holds no committed snapshot", slot);
  if (int cst = check_meta(r, m)) return cst;
  *n = m.num_regions;
  for (uint32_t i = 0; i < m.num_regions; ++i) {
    if (kinds) kinds[i] = m.region_kinds[i];
    if (bytes) bytes[i] = m.region_bytes[i];
  }
  return FFX_OK;
}

extern "C" int ffx_replica_rollback(ffx_replica* r, uint64_t iteration, uint32_t* dropped) {
  if (!r) return fail(FFX_EINVAL, "replica_rollback: null argument");
  DeviceGuard g(r->device);
  uint32_t n = 0;
  for (uint32_t v = 0; v < r->versions; ++v) {
    SlotMeta m;
    int st = read_meta(r, v, &m);
    if (st) return st;
    if (m.magic != kSlotMagic || m.state == kSlotEmpty || m.iteration <= iteration) continue;
    const uint32_t empty = kSlotEmpty;
    FFX_CUDA(cudaMemcpy(r->slot(v) + offsetof(SlotMeta, state), &empty, 4, cudaMemcpyHostToDevice));
    if (v < r->cache.size()) r->cache[v] = SlotCache{true, kSlotEmpty, 0, 0};
    ++n;
  }
  if (dropped) *dropped = n;
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

namespace ffx::host {

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
  if (int st = check_meta(r, m)) return st;
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
  if (int st = check_meta(r, m)) return st;
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

