// ffx_mcast.cu -- the C ABI, part 5: shareable (VMM) replicas and the
// NVSwitch-multicast double neighbour.
#include "ffx_host.h"

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

// A pinned host-memory allocation on the NUMA node closest to `device`
// (the tier below HBM of a tiered replica), shareable by fd like the rest.
CUmemAllocationProp host_prop(int device) {
  CUmemAllocationProp ap{};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  int numa = -1;
  CUdevice d;
  if (drv().deviceGet(&d, device) == CUDA_SUCCESS) drv().deviceAttr(&numa, CU_DEVICE_ATTRIBUTE_HOST_NUMA_ID, d);
  ap.location.id = numa < 0 ? 0 : numa;
  ap.requestedHandleTypes = kShareType;
  return ap;
}

// One VA range [0, dev_bytes + host_bytes): device memory first, host memory
// after; `device` gets read/write access to all of it.
int map_tiered(CUmemGenericAllocationHandle hd, uint64_t dev_bytes, CUmemGenericAllocationHandle hh,
               uint64_t host_bytes, uint64_t align, int device, uint8_t** va) {
  const uint64_t total = dev_bytes + host_bytes;
  CUdeviceptr p = 0;
  FFX_DRV(drv().addressReserve(&p, total, align, 0, 0));
  CUresult r = CUDA_SUCCESS;
  if (dev_bytes) r = drv().memMap(p, dev_bytes, 0, hd, 0);
  if (r == CUDA_SUCCESS && host_bytes) {
    r = drv().memMap(p + dev_bytes, host_bytes, 0, hh, 0);
    if (r != CUDA_SUCCESS && dev_bytes) drv().memUnmap(p, dev_bytes);
  }
  if (r != CUDA_SUCCESS) {
    drv().addressFree(p, total);
    return drv_fail(r, "cuMemMap (tiered)");
  }
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = drv().setAccess(p, total, &acc, 1);
  if (r != CUDA_SUCCESS) {
    drv().memUnmap(p, total);
    drv().addressFree(p, total);
    return drv_fail(r, "cuMemSetAccess (tiered)");
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

namespace ffx::host {

int open_shared(ffx_ctx* c, const HandleBlob& h, ffx_replica* r) {
  if (!drv().ok) return fail(FFX_ECUDA, "CUDA driver lacks the VMM entry points");
  r->vmm = true;
  r->vmm_bytes = h.alloc_bytes;
  if (h.pid == getpid()) {  // the owner's own mapping; grant this ctx's device access
    r->base = reinterpret_cast<uint8_t*>(h.raw);
    if (h.device != c->device) return grant_access(r->base, h.alloc_bytes, h.device, c->device);
    return FFX_OK;
  }
  auto import_fd = [&](int remote_fd, CUmemGenericAllocationHandle* out) -> int {
    int fd = -1;
    int st = fetch_or_fail(h.pid, remote_fd, &fd);
    if (st) return st;
    CUresult cr = drv().importHandle(out, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)), kShareType);
    close(fd);
    return cr != CUDA_SUCCESS ? drv_fail(cr, "cuMemImportFromShareableHandle") : FFX_OK;
  };
  CUmemGenericAllocationHandle mh = 0, mh2 = 0;
  const bool tiered = h.kind == 2;
  const uint64_t dev_bytes = tiered ? h.tier_hbm : h.alloc_bytes;
  int st = dev_bytes ? import_fd(h.fd, &mh) : FFX_OK;
  if (!st && tiered && h.alloc_bytes > dev_bytes) st = import_fd(h.fd2, &mh2);
  uint64_t gran = 0;
  if (!st) st = share_gran(c->device, &gran);
  if (!st) st = tiered ? map_tiered(mh, dev_bytes, mh2, h.alloc_bytes - dev_bytes, gran, c->device, &r->base)
                       : map_range(mh, h.alloc_bytes, gran, c->device, &r->base);
  if (st) {
    if (mh) drv().memRelease(mh);
    if (mh2) drv().memRelease(mh2);
    return st;
  }
  r->vmm_handle = mh;
  r->vmm_handle2 = mh2;
  r->tier_hbm = tiered ? dev_bytes : 0;
  r->vmm_mapped = true;
  return FFX_OK;
}

void release_shared(ffx_replica* r) {
  if ((r->owned || r->vmm_mapped) && r->base) {
    drv().memUnmap(reinterpret_cast<CUdeviceptr>(r->base), r->vmm_bytes);
    drv().addressFree(reinterpret_cast<CUdeviceptr>(r->base), r->vmm_bytes);
    if (r->vmm_handle) drv().memRelease(r->vmm_handle);
    if (r->vmm_handle2) drv().memRelease(r->vmm_handle2);
  }
  for (int fd : {r->vmm_fd, r->vmm_fd2}) {
    if (r->owned && fd >= 0) {
      unshare_fd(fd);
      close(fd);
    }
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

extern "C" int ffx_replica_create_tiered(ffx_ctx* c, ffx_role origin, uint64_t capacity, uint32_t versions,
                                         uint64_t hbm_bytes, ffx_replica** out) {
  if (!c || !out) return fail(FFX_EINVAL, "replica_create_tiered: null argument");
  if (versions < 1 || versions > 8) return fail(FFX_EINVAL, "replica_create_tiered: 1..8 versions");
  DeviceGuard g(c->device);
  uint64_t gran = 0;
  int st = share_gran(c->device, &gran);
  if (st) return st;
  CUmemAllocationProp hp = host_prop(c->device);
  size_t hg = 0;
  FFX_DRV(drv().allocGran(&hg, &hp, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
  gran = std::max<uint64_t>(gran, hg);
  const SlotLayout L = make_layout(capacity, c->slice_bytes);
  const uint64_t total = align_up(L.slot_stride * versions, gran);
  const uint64_t dev_bytes = std::min(total, align_up(hbm_bytes, gran));
  const uint64_t host_bytes = total - dev_bytes;
  CUmemAllocationProp dp = share_prop(c->device);
  CUmemGenericAllocationHandle hd = 0, hh = 0;
  if (dev_bytes) FFX_DRV(drv().memCreate(&hd, dev_bytes, &dp, 0));
  if (host_bytes) {
    CUresult cr = drv().memCreate(&hh, host_bytes, &hp, 0);
    if (cr != CUDA_SUCCESS) {
      if (hd) drv().memRelease(hd);
      return drv_fail(cr, "cuMemCreate (host tier)");
    }
  }
  auto* r = new ffx_replica;
  r->device = c->device;
  r->owner_pid = getpid();
  r->owned = true;
  r->vmm = true;
  r->vmm_handle = hd;
  r->vmm_handle2 = hh;
  r->vmm_bytes = total;
  r->tier_hbm = dev_bytes;
  r->origin = origin;
  r->capacity = capacity;
  r->slice_bytes = c->slice_bytes;
  r->versions = versions;
  r->layout = L;
  r->cache.assign(versions, SlotCache{});
  r->ctx = c;
  st = map_tiered(hd, dev_bytes, hh, host_bytes, gran, c->device, &r->base);
  if (st) {
    if (hd) drv().memRelease(hd);
    if (hh) drv().memRelease(hh);
    delete r;
    return st;
  }
  auto export_fd = [&](CUmemGenericAllocationHandle h, int* fd_out) -> int {
    if (!h) return FFX_OK;
    int fd = -1;
    CUresult cr = drv().exportHandle(&fd, h, kShareType, 0);
    const int e = cr == CUDA_SUCCESS ? share_fd(fd) : 0;
    if (cr != CUDA_SUCCESS || e) {
      if (fd >= 0) close(fd);
      return cr != CUDA_SUCCESS ? drv_fail(cr, "cuMemExportToShareableHandle (tiered)")
                                : fail(FFX_ECUDA, "fd server: %s", std::strerror(e));
    }
    *fd_out = fd;
    return FFX_OK;
  };
  st = export_fd(hd, &r->vmm_fd);
  if (!st) st = export_fd(hh, &r->vmm_fd2);
  cudaError_t ce = cudaSuccess;
  for (uint32_t v = 0; !st && v < versions && ce == cudaSuccess; ++v) {
    ce = cudaMemset(r->slot(v), 0, kMetaBytes);
    r->cache[v].known = true;
  }
  if (!st && ce == cudaSuccess) ce = cudaDeviceSynchronize();
  if (st || ce != cudaSuccess) {
    release_shared(r);
    delete r;
    return st ? st : cuda_fail(ce, "replica_create_tiered");
  }
  *out = r;
  return FFX_OK;
}

extern "C" int ffx_replica_tiers(const ffx_replica* r, uint64_t* hbm_bytes, uint64_t* host_bytes) {
  if (!r) return fail(FFX_EINVAL, "replica_tiers: null argument");
  const uint64_t total = r->vmm ? r->vmm_bytes : r->layout.slot_stride * r->versions;
  const uint64_t dev = (r->vmm_handle2 || r->tier_hbm) ? r->tier_hbm : total;
  if (hbm_bytes) *hbm_bytes = dev;
  if (host_bytes) *host_bytes = total - dev;
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
  if (members < 1 || members > 8) return fail(FFX_EINVAL, "mcast_create: 1..8 members");
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
    // any binding here the stores crawl at ~50 GB/s (measured).  When the
    // origin's own device already backs it with a holder's replica (a holder
    // on the writer's GPU, e.g. a one-GPU team), that binding is the backing.
    if (!m->bound) {
      m->sink_bytes = std::min<uint64_t>(m->bytes, kSinkMax);
      m->sink_bytes = align_up(m->sink_bytes, m->gran);
      while (m->bytes % m->sink_bytes) m->sink_bytes -= m->gran;
      CUmemAllocationProp ap = share_prop(c->device);
      FFX_DRV(drv().memCreate(&m->sink, m->sink_bytes, &ap, 0));
      for (uint64_t o = 0; o < m->bytes; o += m->sink_bytes)
        FFX_DRV(drv().mcBindMem(m->handle, o, m->sink, 0, m->sink_bytes, 0));
    }
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

