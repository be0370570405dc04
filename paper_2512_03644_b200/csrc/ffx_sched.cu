// ffx_sched.cu -- the C ABI, part 6: the slice scheduler as a native object
// (include/ffx.h "the slice scheduler as a native object").
//
// Reference semantics (sim_net.cpp:401-454, test_transport.cpp:173-197):
// STATE traffic moves only when no TRAIN chunk is queued and a chunk in
// flight is never cut, so TRAIN is delayed by at most one chunk.  On a B200
// the step reports its gaps; each report records an event on the step's
// stream and issues the next snapshot batch on a low-priority stream gated
// on that event, with a CTA cap bounding what a batch can hold while TRAIN
// kernels arrive.  Copy batches go into link-idle gaps (after a collective),
// checksum batches (split policies) into SM-idle gaps (before a collective).
#include <deque>

#include "ffx_host.h"

struct ffx_sched {
  struct Fetch {  // a queued preload (ffx_sched_preload_*)
    ffx_preload* p;
    uint64_t iteration;
    const void* host_src;        // null: synthetic
    std::vector<uint8_t> digests;
    uint32_t count, sample_bytes;
    uint64_t bytes;
  };
  ffx_ctx* ctx = nullptr;
  std::deque<Fetch> fetches;
  ffx_sched_opts opts{};
  std::vector<double> weights;        // link-gap durations (copy-batch sizes)
  cudaStream_t copy_stream = nullptr; // low priority
  cudaStream_t hash_stream = nullptr; // low priority
  std::vector<cudaEvent_t> gates;     // one per report, reused every step
  cudaEvent_t done = nullptr;         // recorded after the commit
  uint32_t copies_left = 0, hashes_left = 0, next_gate = 0;
  bool active = false;
};

namespace {

bool split_policy(const ffx_sched* s) { return s->opts.policy != FFX_SCHED_FUSED; }

// Record a gate on the step's stream and issue the next batch of `kind`.
int issue(ffx_sched* s, int kind, cudaStream_t train) {
  cudaEvent_t gate = nullptr;
  if (train) {
    gate = s->gates[s->next_gate++ % s->gates.size()];
    FFX_CUDA(cudaEventRecord(gate, train));
  }
  cudaStream_t st = kind == FFX_BATCH_COPY ? s->copy_stream : s->hash_stream;
  uint32_t left = 0;
  const int rc = split_policy(s) ? ffx_snapshot_next_kind(s->ctx, kind, st, gate, &left)
                                 : ffx_snapshot_next(s->ctx, st, gate, &left);
  if (rc) return rc;
  if (kind == FFX_BATCH_COPY) s->copies_left = left;
  else s->hashes_left = left;
  if (s->copies_left == 0 && s->hashes_left == 0) FFX_CUDA(cudaEventRecord(s->done, st));  // carried the commit
  return FFX_OK;
}

// Issue the queued preloads in iteration order on the copy stream after
// `gate`, stopping at the first that does not fit (buffer full: no fetch).
int issue_fetches(ffx_sched* s, cudaEvent_t gate) {
  while (!s->fetches.empty()) {
    auto& f = s->fetches.front();
    int fits = 0;
    int rc = ffx_preload_fits(f.p, f.bytes, &fits);
    if (rc) return rc;
    if (!fits) break;
    rc = preload_fetch(f.p, f.iteration, f.host_src, f.digests.empty() ? nullptr : f.digests.data(), f.count,
                       f.sample_bytes, f.bytes, s->copy_stream, gate);
    if (rc) return rc;
    s->fetches.pop_front();
  }
  return FFX_OK;
}

}  // namespace

extern "C" int ffx_sched_create(ffx_ctx* c, const ffx_sched_opts* o, ffx_sched** out) {
  if (!c || !o || !out) return fail(FFX_EINVAL, "sched_create: null argument");
  if (o->policy > FFX_SCHED_SPLIT_CE) return fail(FFX_EINVAL, "sched_create: policy %u", o->policy);
  if (o->link_gaps == 0) return fail(FFX_EINVAL, "sched_create: link_gaps must be > 0");
  if (o->policy != FFX_SCHED_FUSED && o->sm_gaps == 0) return fail(FFX_EINVAL, "sched_create: sm_gaps must be > 0");
  DeviceGuard g(c->device);
  auto* s = new ffx_sched;
  s->ctx = c;
  s->opts = *o;
  s->opts.gap_ms = nullptr;
  if (!s->opts.copy_ctas) s->opts.copy_ctas = o->policy == FFX_SCHED_FUSED ? 32 : 8;
  if (!s->opts.hash_ctas) s->opts.hash_ctas = 96;  // uncapped, the checksum starves NCCL and the DMA engines
  if (o->gap_ms) s->weights.assign(o->gap_ms, o->gap_ms + o->link_gaps);
  int lo = 0, hi = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);  // lo = least urgent
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&s->copy_stream, cudaStreamNonBlocking, lo);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&s->hash_stream, cudaStreamNonBlocking, lo);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->done, cudaEventDisableTiming);
  s->gates.assign(o->link_gaps + o->sm_gaps + 2, nullptr);
  for (auto& ev : s->gates)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    ffx_sched_destroy(s);
    return cuda_fail(e, "sched_create");
  }
  *out = s;
  return FFX_OK;
}

extern "C" int ffx_sched_begin(ffx_sched* s, uint64_t iteration) {
  if (!s) return fail(FFX_EINVAL, "sched_begin: null argument");
  if (s->active) return fail(FFX_ESTATE, "sched_begin: the previous step was not finished (ffx_sched_finish)");
  ffx_snapshot_opts o{};
  o.batches = s->opts.link_gaps;
  o.max_ctas = s->opts.copy_ctas;
  o.task_ctas = s->opts.policy == FFX_SCHED_FUSED ? s->opts.task_ctas : 0;
  o.batch_weights = s->weights.empty() ? nullptr : s->weights.data();
  if (split_policy(s)) {
    o.split = 1;
    o.hash_batches = s->opts.sm_gaps;
    o.hash_ctas = s->opts.hash_ctas;
    o.copy_engine = s->opts.policy == FFX_SCHED_SPLIT_CE;
  }
  uint32_t n = 0;
  int rc = ffx_snapshot_begin(s->ctx, iteration, &o, &n);
  if (rc) return rc;
  s->copies_left = n;
  s->hashes_left = split_policy(s) ? s->opts.sm_gaps : 0;
  s->next_gate = 0;
  s->active = true;
  return FFX_OK;
}

extern "C" int ffx_sched_gap(ffx_sched* s, int kind, void* train_stream) {
  if (!s) return fail(FFX_EINVAL, "sched_gap: null argument");
  DeviceGuard g(s->ctx->device);
  if (kind == FFX_GAP_LINK_IDLE && !s->fetches.empty()) {  // the loader's preloads ride the same gaps
    cudaEvent_t gate = nullptr;
    if (train_stream) {
      gate = s->gates[s->next_gate++ % s->gates.size()];
      FFX_CUDA(cudaEventRecord(gate, as_stream(train_stream)));
    }
    const int rc = issue_fetches(s, gate);
    if (rc) return rc;
  }
  if (!s->active) return FFX_OK;  // no snapshot this step
  if (kind == FFX_GAP_LINK_IDLE && s->copies_left) return issue(s, FFX_BATCH_COPY, as_stream(train_stream));
  if (kind == FFX_GAP_SM_IDLE && s->hashes_left) return issue(s, FFX_BATCH_HASH, as_stream(train_stream));
  if (kind != FFX_GAP_LINK_IDLE && kind != FFX_GAP_SM_IDLE) return fail(FFX_EINVAL, "sched_gap: kind %d", kind);
  return FFX_OK;
}

extern "C" int ffx_sched_finish(ffx_sched* s, void* train_stream) {
  if (!s) return fail(FFX_EINVAL, "sched_finish: null argument");
  if (!s->active) return FFX_OK;
  DeviceGuard g(s->ctx->device);
  while (s->copies_left) {  // more batches than gaps this step: flush now
    int rc = issue(s, FFX_BATCH_COPY, nullptr);
    if (rc) return rc;
  }
  while (s->hashes_left) {
    int rc = issue(s, FFX_BATCH_HASH, nullptr);
    if (rc) return rc;
  }
  s->active = false;
  // the optimizer may only mutate the snapshotted state after the commit
  FFX_CUDA(cudaStreamWaitEvent(as_stream(train_stream), s->done, 0));
  return FFX_OK;
}

extern "C" int ffx_sched_preload_host(ffx_sched* s, ffx_preload* p, uint64_t iteration, const void* host_src,
                                      uint64_t bytes) {
  if (!s || !p || (bytes && !host_src)) return fail(FFX_EINVAL, "sched_preload_host: null argument");
  s->fetches.push_back(ffx_sched::Fetch{p, iteration, host_src, {}, 0, 0, bytes});
  return FFX_OK;
}

extern "C" int ffx_sched_preload_synthetic(ffx_sched* s, ffx_preload* p, uint64_t iteration,
                                           const uint8_t* item_digests, uint32_t count, uint32_t sample_bytes) {
  if (!s || !p || (count && !item_digests)) return fail(FFX_EINVAL, "sched_preload_synthetic: null argument");
  ffx_sched::Fetch f{p, iteration, nullptr, std::vector<uint8_t>(item_digests, item_digests + 32 * size_t(count)),
                     count, sample_bytes, uint64_t(count) * sample_bytes};
  s->fetches.push_back(std::move(f));
  return FFX_OK;
}

extern "C" int ffx_sched_preload_pending(ffx_sched* s, uint32_t* pending) {
  if (!s || !pending) return fail(FFX_EINVAL, "sched_preload_pending: null argument");
  *pending = static_cast<uint32_t>(s->fetches.size());
  return FFX_OK;
}

extern "C" int ffx_sched_destroy(ffx_sched* s) {
  if (!s) return FFX_OK;
  DeviceGuard g(s->ctx ? s->ctx->device : -1);
  if (s->copy_stream) cudaStreamSynchronize(s->copy_stream);
  if (s->hash_stream) cudaStreamSynchronize(s->hash_stream);
  for (auto ev : s->gates)
    if (ev) cudaEventDestroy(ev);
  if (s->done) cudaEventDestroy(s->done);
  if (s->copy_stream) cudaStreamDestroy(s->copy_stream);
  if (s->hash_stream) cudaStreamDestroy(s->hash_stream);
  delete s;
  return FFX_OK;
}
