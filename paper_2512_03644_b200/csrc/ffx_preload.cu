// ffx_preload.cu -- the C ABI, part 8: the data loader's preload buffer in
// HBM (the preload stream under the same TRAIN > STATE
// arbitration as the snapshot).
//
// Reference semantics (dataloader.hpp:45-73, dataloader.cpp:59-82, SPEC
// preload_loop): a byte-capped, TID-ordered buffer; insert fails on
// overflow or a duplicate TID (std::logic_error; callers gate on fits());
// take() removes an entry and returns its blob; the preloader fetches a
// worker-iteration's window only when the buffer has room and the link is
// idle.  On a B200 an entry is a stream-ordered allocation from the device
// memory pool: a fetch lands it by an H2D copy (copy engines, host or file
// data) or generates it on the device (the synthetic DataServerStub), on the
// stream the caller (or the slice scheduler, ffx_sched_preload) chooses,
// gated on an event; take() hands the consumer a device pointer its stream
// waits for, and ffx_preload_free returns the memory after the consumer's
// last use, stream-ordered.
#include <map>

#include "ffx_host.h"

struct ffx_preload {
  struct Entry {
    uint8_t* dev = nullptr;
    uint64_t bytes = 0;
    cudaEvent_t ready = nullptr;  // the fetch has landed
  };
  ffx_ctx* ctx = nullptr;
  uint64_t capacity = 0;
  uint64_t bytes = 0;
  std::map<uint64_t, Entry> entries;  // TID order (this rank's role, by iteration)
  uint64_t fetched = 0, taken = 0;
};

namespace ffx::host {

// insert(): FFX_ECONFIG on overflow, FFX_ESTATE on a duplicate TID.
int preload_reserve(ffx_preload* p, uint64_t iteration, uint64_t bytes, cudaStream_t s,
                    ffx_preload::Entry** out) {
  if (p->entries.count(iteration))
    return fail(FFX_ESTATE, "duplicate preload entry for iteration %llu", (unsigned long long)iteration);
  if (p->bytes + bytes > p->capacity)
    return fail(FFX_ECONFIG, "preload buffer overflow at iteration %llu (%llu + %llu > %llu)",
                (unsigned long long)iteration, (unsigned long long)p->bytes, (unsigned long long)bytes,
                (unsigned long long)p->capacity);
  ffx_preload::Entry e;
  e.bytes = bytes;
  retain_pool();
  cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&e.dev), bytes ? bytes : 1, s);
  if (err != cudaSuccess) {
    cudaGetLastError();
    return fail(FFX_ENOMEM, "preload: cudaMallocAsync(%llu): %s", (unsigned long long)bytes,
                cudaGetErrorString(err));
  }
  err = cudaEventCreateWithFlags(&e.ready, cudaEventDisableTiming);
  if (err != cudaSuccess) {
    cudaFreeAsync(e.dev, s);
    return cuda_fail(err, "preload: event");
  }
  p->bytes += bytes;
  *out = &(p->entries[iteration] = e);
  return FFX_OK;
}

int preload_fetch(ffx_preload* p, uint64_t iteration, const void* host_src, const uint8_t* digests, uint32_t count,
                  uint32_t sample_bytes, uint64_t bytes, cudaStream_t s, cudaEvent_t gate) {
  DeviceGuard g(p->ctx->device);
  if (gate) FFX_CUDA(cudaStreamWaitEvent(s, gate, 0));
  ffx_preload::Entry* e = nullptr;
  int rc = preload_reserve(p, iteration, bytes, s, &e);
  if (rc) return rc;
  cudaError_t err = cudaSuccess;
  if (host_src) {
    if (bytes) err = cudaMemcpyAsync(e->dev, host_src, bytes, cudaMemcpyHostToDevice, s);
  } else if (count) {
    // DataServerStub::sample in synthetic mode: expand(data_item_digest(seed,
    // index), bytes) depends on each digest's fold64 only (evolution.cpp:71-120)
    std::vector<uint64_t> folds(count);
    for (uint32_t i = 0; i < count; ++i) folds[i] = rd(digests + 32 * size_t(i), 8);
    uint64_t* dfolds = nullptr;
    err = cudaMallocAsync(reinterpret_cast<void**>(&dfolds), 8ull * count, s);
    if (err == cudaSuccess) err = cudaMemcpyAsync(dfolds, folds.data(), 8ull * count, cudaMemcpyHostToDevice, s);
    if (err == cudaSuccess) err = launch_items(e->dev, dfolds, count, sample_bytes, s);
    if (dfolds) cudaFreeAsync(dfolds, s);
    // the pageable `folds` copy is staged before cudaMemcpyAsync returns
  }
  if (err == cudaSuccess) err = cudaEventRecord(e->ready, s);
  if (err != cudaSuccess) {
    cudaEventDestroy(e->ready);
    cudaFreeAsync(e->dev, s);
    p->bytes -= e->bytes;
    p->entries.erase(iteration);
    return cuda_fail(err, "preload fetch");
  }
  ++p->fetched;
  return FFX_OK;
}

}  // namespace ffx::host

extern "C" int ffx_preload_create(ffx_ctx* c, uint64_t capacity_bytes, ffx_preload** out) {
  if (!c || !out) return fail(FFX_EINVAL, "preload_create: null argument");
  auto* p = new ffx_preload;
  p->ctx = c;
  p->capacity = capacity_bytes;
  *out = p;
  return FFX_OK;
}

extern "C" int ffx_preload_destroy(ffx_preload* p) {
  if (!p) return FFX_OK;
  DeviceGuard g(p->ctx->device);
  for (auto& kv : p->entries) {
    cudaEventSynchronize(kv.second.ready);
    cudaEventDestroy(kv.second.ready);
    cudaFree(kv.second.dev);
  }
  delete p;
  return FFX_OK;
}

extern "C" int ffx_preload_fits(ffx_preload* p, uint64_t bytes, int* fits) {
  if (!p || !fits) return fail(FFX_EINVAL, "preload_fits: null argument");
  *fits = p->bytes + bytes <= p->capacity;
  return FFX_OK;
}

extern "C" int ffx_preload_fetch_host(ffx_preload* p, uint64_t iteration, const void* host_src, uint64_t bytes,
                                      void* stream, void* gate_event) {
  if (!p || (bytes && !host_src)) return fail(FFX_EINVAL, "preload_fetch_host: null argument");
  return preload_fetch(p, iteration, host_src, nullptr, 0, 0, bytes, as_stream(stream),
                       static_cast<cudaEvent_t>(gate_event));
}

extern "C" int ffx_preload_fetch_synthetic(ffx_preload* p, uint64_t iteration, const uint8_t* item_digests,
                                           uint32_t count, uint32_t sample_bytes, void* stream, void* gate_event) {
  if (!p || (count && !item_digests)) return fail(FFX_EINVAL, "preload_fetch_synthetic: null argument");
  return preload_fetch(p, iteration, nullptr, item_digests, count, sample_bytes, uint64_t(count) * sample_bytes,
                       as_stream(stream), static_cast<cudaEvent_t>(gate_event));
}

extern "C" int ffx_preload_take(ffx_preload* p, uint64_t iteration, void* consumer_stream, void** dev,
                                uint64_t* bytes) {
  if (!p || !dev) return fail(FFX_EINVAL, "preload_take: null argument");
  auto it = p->entries.find(iteration);
  if (it == p->entries.end())  // take() -> nullopt
    return fail(FFX_ESTATE, "iteration %llu is not in the preload buffer", (unsigned long long)iteration);
  DeviceGuard g(p->ctx->device);
  FFX_CUDA(cudaStreamWaitEvent(as_stream(consumer_stream), it->second.ready, 0));
  *dev = it->second.dev;
  if (bytes) *bytes = it->second.bytes;
  cudaEventDestroy(it->second.ready);  // safe: destruction defers until the event completes
  p->bytes -= it->second.bytes;
  p->entries.erase(it);
  ++p->taken;
  return FFX_OK;
}

extern "C" int ffx_preload_free(ffx_preload* p, void* dev, void* consumer_stream) {
  if (!p) return fail(FFX_EINVAL, "preload_free: null argument");
  if (!dev) return FFX_OK;
  DeviceGuard g(p->ctx->device);
  FFX_CUDA(cudaFreeAsync(dev, as_stream(consumer_stream)));
  return FFX_OK;
}

extern "C" int ffx_preload_info(ffx_preload* p, ffx_preload_state* out) {
  if (!p || !out) return fail(FFX_EINVAL, "preload_info: null argument");
  out->capacity = p->capacity;
  out->bytes = p->bytes;
  out->entries = p->entries.size();
  out->oldest = p->entries.empty() ? UINT64_MAX : p->entries.begin()->first;
  out->fetched = p->fetched;
  out->taken = p->taken;
  return FFX_OK;
}

extern "C" int ffx_fold_of_blob(const void* dev, uint64_t bytes, uint32_t bytes_per_sample, uint64_t* host_out,
                                void* stream) {
  if (!host_out || (bytes && !dev)) return fail(FFX_EINVAL, "fold_of_blob: null argument");
  if (bytes_per_sample == 0 || bytes % bytes_per_sample != 0)  // dataloader.cpp:152-153
    return fail(FFX_EINVAL, "blob is not a whole number of samples");
  DeviceGuard g(pick_device(stream, dev));
  cudaStream_t s = as_stream(stream);
  unsigned long long* d = nullptr;
  retain_pool();
  FFX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 8, s));
  cudaError_t e = cudaMemsetAsync(d, 0, 8, s);
  if (e == cudaSuccess) e = launch_fold_blob(static_cast<const uint8_t*>(dev), bytes, bytes_per_sample, d, s);
  unsigned long long r = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&r, d, 8, cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(d, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "fold_of_blob");
  *host_out = r;
  return FFX_OK;
}
