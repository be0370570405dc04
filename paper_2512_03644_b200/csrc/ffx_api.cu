// ffx_api.cu -- the C ABI (include/ffx.h), part 1: status, domain,
// recovery planning, sizing, SNP1 framing, device primitives, buffer
// plumbing, contexts and the state registry.  Objects and shared helpers:
// ffx_host.h.
#include "ffx_host.h"

namespace ffx::host {

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

}  // namespace ffx::host

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

  // Serving holder per lost role among the survivors of dp+1 .. dp+replicas.
  // replicas = 1: the ring successor (the reference rule).  replicas > 1:
  // spread the gathers over the surviving holders -- roles with the fewest
  // candidates first, each to its least-loaded candidate (ties: the nearest)
  // -- so an adjacent pair does not share one holder's NVLink egress.
  const uint32_t d = s->data_parallel;
  const uint32_t k = std::min<uint32_t>(replicas, d > 1 ? d - 1 : 1);
  bool neighbor_ok = d > 1;
  std::vector<uint32_t> holder(lost.size(), 0);
  std::vector<std::vector<uint32_t>> cand(lost.size());
  for (size_t i = 0; i < lost.size() && neighbor_ok; ++i) {
    for (uint32_t j = 1; j <= k; ++j) {
      ffx_role h = lost[i];
      h.dp = static_cast<uint16_t>((lost[i].dp + j) % d);
      if (!is_lost(h)) cand[i].push_back(h.dp);
    }
    if (cand[i].empty()) neighbor_ok = false;
  }
  if (neighbor_ok) {
    std::vector<size_t> order(lost.size());
    std::iota(order.begin(), order.end(), size_t{0});
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t b) { return cand[a].size() < cand[b].size(); });
    std::vector<uint32_t> load;  // per (holder dp, pp, tp) key, linear scan (small)
    std::vector<uint64_t> load_key;
    auto load_of = [&](uint64_t kk) -> uint32_t& {
      for (size_t x = 0; x < load_key.size(); ++x)
        if (load_key[x] == kk) return load[x];
      load_key.push_back(kk);
      load.push_back(0);
      return load.back();
    };
    for (size_t i : order) {
      uint32_t best = cand[i][0];
      for (uint32_t c : cand[i]) {
        ffx_role hc = lost[i], hb = lost[i];
        hc.dp = static_cast<uint16_t>(c);
        hb.dp = static_cast<uint16_t>(best);
        if (load_of(key(hc)) < load_of(key(hb))) best = c;
      }
      ffx_role h = lost[i];
      h.dp = static_cast<uint16_t>(best);
      load_of(key(h))++;
      holder[i] = best;
    }
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

namespace ffx::host {

SliceJob single_job(const void* src, void* dst, uint64_t len, uint64_t slice_bytes) {
  SliceJob job{};
  job.nregions = 1;
  job.reg[0] = SliceRegion{static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), len, 0, 0};
  job.slice_bytes = slice_bytes;
  finalize_job(job);
  return job;
}

}  // namespace

extern "C" int ffx_checksum64(const void* dev, uint64_t len, uint64_t* host_out, void* stream) {
  if (!host_out || (len && !dev)) return fail(FFX_EINVAL, "checksum64: null argument");
  DeviceGuard g(pick_device(stream, dev));
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
  DeviceGuard g(pick_device(stream, dev));
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
  DeviceGuard g(pick_device(stream, src));
  SliceJob job = single_job(src, dst, len, slice_bytes);
  job.sums_out = dev_out;
  FFX_CUDA(launch_slices(job, SliceMode::Copy, false, 0, as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_copy_verify(void* dst, const void* src, uint64_t len, uint64_t slice_bytes,
                               const uint64_t* dev_expected, uint64_t* dev_result, void* stream) {
  if (!slice_ok(slice_bytes)) return fail(FFX_EINVAL, "slice_bytes must be a multiple of 256");
  if (!dev_result || !dev_expected) return fail(FFX_EINVAL, "copy_verify: null argument");
  DeviceGuard g(pick_device(stream, dev_result));
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
  DeviceGuard g(pick_device(stream, src));
  CopyJob job{};
  job.nregions = 1;
  job.reg[0] = CopyRegion{static_cast<const uint8_t*>(src), static_cast<uint8_t*>(dst), len, 0, 0};
  finalize_copy_job(job);
  FFX_CUDA(launch_copy(job, ctas, as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_expand(void* dst, const uint8_t digest[32], uint64_t bytes, void* stream) {
  if (!digest || (bytes && !dst)) return fail(FFX_EINVAL, "expand: null argument");
  DeviceGuard g(pick_device(stream, dst));
  uint64_t fold = rd(digest, 8);
  FFX_CUDA(launch_expand(static_cast<uint8_t*>(dst), fold, bytes, nullptr, as_stream(stream)));
  return FFX_OK;
}

extern "C" int ffx_materialize(void* dst, const uint8_t digest[32], uint64_t bytes, void* stream) {
  if (!digest) return fail(FFX_EINVAL, "materialize: null digest");
  if (bytes < 32) return fail(FFX_EINVAL, "state blob smaller than its digest prefix");
  if (!dst) return fail(FFX_EINVAL, "materialize: null dst");
  DeviceGuard g(pick_device(stream, dst));
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
  DeviceGuard g(pick_device(stream, dev));
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

extern "C" int ffx_prepare_peers(int device, uint32_t* enabled) {
  DeviceGuard g(device);
  int n = 0;
  FFX_CUDA(cudaGetDeviceCount(&n));
  uint32_t k = 0;
  for (int p = 0; p < n; ++p) {
    if (p == device) continue;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, device, p) != cudaSuccess || !can) {
      cudaGetLastError();
      continue;
    }
    const cudaError_t e = cudaDeviceEnablePeerAccess(p, 0);
    if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) ++k;
    cudaGetLastError();
  }
  if (enabled) *enabled = k;
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
  if (e == cudaSuccess) e = cudaMemset(c->done + kAckWord, 0xff, 8);  // kAckNone
  if (e == cudaSuccess) e = cudaMalloc(&c->result, 16);
  if (e == cudaSuccess) e = cudaMallocHost(&c->result_host, 16);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->copy_done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->hash_done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->snap_done, cudaEventDisableTiming);
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
  if (c->snap_done) cudaEventDestroy(c->snap_done);
  for (cudaEvent_t e : c->h2d_ev) cudaEventDestroy(e);
  if (c->h2d) cudaStreamDestroy(c->h2d);
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

extern "C" int ffx_slice_runs(const uint64_t* region_bytes, uint32_t n, uint64_t slice_bytes, ffx_slice_run* out,
                              uint32_t cap, uint32_t* count) {
  if ((n && !region_bytes) || !count || (cap && !out)) return fail(FFX_EINVAL, "slice_runs: null argument");
  if (!slice_ok(slice_bytes)) return fail(FFX_EINVAL, "slice_runs: bad slice size %llu", (unsigned long long)slice_bytes);
  uint32_t k = 0;
  uint64_t first = 0;
  for (uint32_t i = 0; i < n; ++i) {
    SliceRun runs[kRegionRuns];
    const int m = region_runs(region_bytes[i], slice_bytes, head_region(i, n), runs);
    for (int j = 0; j < m; ++j, ++k) {
      if (k < cap)
        out[k] = ffx_slice_run{i, static_cast<uint32_t>(runs[j].slice), runs[j].offset, runs[j].bytes, first};
      first += run_slices(runs[j]);
    }
  }
  *count = k;
  return k <= cap ? FFX_OK : fail(FFX_EINVAL, "slice_runs: %u runs, room for %u", k, cap);
}

extern "C" int ffx_plan(ffx_ctx* c, ffx_plan_info* out) {
  if (!c || !out) return fail(FFX_EINVAL, "plan: null argument");
  std::memset(out, 0, sizeof *out);
  ffx_razor(&c->spec, &out->razor);
  out->slice_bytes = c->slice_bytes;
  out->num_regions = static_cast<uint32_t>(c->regions.size());
  std::vector<uint64_t> unique;  // payload regions, in payload order
  for (const auto& r : c->regions) {
    if (r.unique) {
      out->registered_unique_bytes += r.bytes;
      unique.push_back(r.bytes);
      out->num_unique_regions++;
    } else {
      out->registered_redundant_bytes += r.bytes;
    }
  }
  out->num_slices = table_entries(unique.data(), static_cast<uint32_t>(unique.size()), c->slice_bytes);
  return FFX_OK;
}

