// ffx_snapshot.cu -- the C ABI, part 3: snapshot issue (HostSnapshots::take
// + the ring stream, ckpt.cpp:38-53), pull mode (the holder drives it,
// NeighborBuffer::store), the slice scheduler's batches, and snapshots from
// host memory with the H2D copy pipelined under those batches.
#include "ffx_host.h"

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
// iteration, else a free slot -- empty, or torn (WRITING at rest: a writer
// that died, or a slot the holder dropped after a failed verify) -- else the
// oldest committed one.
uint32_t pick_slot(const ffx_replica* t, uint64_t iteration) {
  int v = -1;
  for (uint32_t i = 0; i < t->versions; ++i)
    if (t->cache[i].state != kSlotEmpty && t->cache[i].iteration == iteration) v = static_cast<int>(i);
  if (v < 0)
    for (uint32_t i = 0; i < t->versions && v < 0; ++i)
      if (t->cache[i].state == kSlotEmpty) v = static_cast<int>(i);
  if (v < 0)
    for (uint32_t i = 0; i < t->versions && v < 0; ++i)
      if (t->cache[i].state != kSlotCommitted) v = static_cast<int>(i);
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
  int kind;            // ffx_region_kind (recorded in the slot meta)
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
  uint64_t logical = 0, physical = 0;
  std::vector<uint64_t> offs, sizes;
  for (const SrcRegion& r : srcs) {
    offs.push_back(physical);
    sizes.push_back(r.bytes);
    logical += r.bytes;
    physical = align_up(physical + r.bytes, kRegionAlign);
  }
  const uint64_t nslices = table_entries(sizes.data(), static_cast<uint32_t>(sizes.size()), c->slice_bytes);
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
  // Insertion order: a fresh iteration gets the next sequence number; a
  // replace-in-place keeps its slot's (ckpt.cpp:46-50 swaps the bytes but
  // leaves the entry where it is in the deque), so eviction and newest()
  // still follow the first insertion.
  uint64_t fresh = ++c->seq;
  for (ffx_replica* rr : {t, t2})
    if (rr)
      for (const auto& sc : rr->cache) fresh = std::max(fresh, sc.seq + 1);
  c->seq = fresh;
  auto seq_for = [&](const ffx_replica* rr, uint32_t v) {
    const SlotCache& sc = rr->cache[v];
    return (sc.state != kSlotEmpty && sc.iteration == iteration && sc.seq) ? sc.seq : fresh;
  };
  const uint64_t seq = seq_for(t, slot);
  const uint64_t seq2 = t2 ? seq_for(t2, slot2) : seq;

  PendingSnapshot& P = c->pending;
  P = PendingSnapshot{};
  P.tgt = t;
  P.tgt2 = t2;
  SliceJob& job = P.job;
  // one job region per slice run (ffx_layout.h): the first region's head in
  // quarter-size slices, everything else at the context's slice size
  std::vector<std::pair<uint32_t, uint64_t>> run_of;  // (registered region, offset within it) per job region
  job.nregions = 0;
  uint64_t logical_at = 0;  // logical payload offset of srcs[i]
  for (size_t i = 0; i < srcs.size(); ++i) {
    SliceRun runs[kRegionRuns];
    const int k = region_runs(srcs[i].bytes, c->slice_bytes,
                              head_region(static_cast<uint32_t>(i), static_cast<uint32_t>(srcs.size())), runs);
    for (int j = 0; j < k; ++j) {
      P.logical_of[job.nregions] = logical_at + runs[j].offset;
      SliceRegion R{srcs[i].dev + runs[j].offset, t->wpayload(slot) + offs[i] + runs[j].offset, runs[j].bytes, 0, 0};
      R.slice_bytes = static_cast<uint32_t>(runs[j].slice);
      job.reg[job.nregions++] = R;
      run_of.emplace_back(static_cast<uint32_t>(i), runs[j].offset);
    }
    logical_at += srcs[i].bytes;
  }
  job.slice_bytes = c->slice_bytes;
  job.sums_out = t->wsums(slot);
  job.sched = c->done + 8;  // dynamic task counter (words 8-9 of the ctx scratch)
  // CTA-capped snapshots (scheduler batches inside a step) use the SM-lean
  // configuration (two chains per lane); split hash batches follow hash_ctas
  finalize_job(job, rows_for_cap(opts.split ? opts.hash_ctas : opts.max_ctas));

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
  m.num_regions = static_cast<uint32_t>(srcs.size());
  for (size_t i = 0; i < srcs.size(); ++i) {
    m.region_bytes[i] = srcs[i].bytes;
    m.region_kinds[i] = static_cast<uint8_t>(srcs[i].kind);
  }
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
  cm.mcast = t->wbase != nullptr ? 1u : 0u;
  if (t2) {
    // Double-neighbour replication: the same tiles stored twice, one table
    // per replica, each slot committed by its own counter.
    for (uint32_t q = 0; q < job.nregions; ++q)
      job.reg[q].dst2 = t2->wpayload(slot2) + offs[run_of[q].first] + run_of[q].second;
    job.sums_out2 = t2->wsums(slot2);
    job.commit2 = cm;
    job.commit2.slot = t2->wslot(slot2);
    job.commit2.seq = seq2;
    reinterpret_cast<SlotMeta*>(job.commit2.meta)->seq = seq2;
    job.commit2.done = c->done + 4;
    job.commit2.payload_off = t2->layout.payload_off;
    job.commit2.mcast = t2->wbase != nullptr ? 1u : 0u;
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
  P.seq2 = seq2;
  P.nslices = nslices;
  P.logical = logical;
  P.verify = opts.verify_on_store != 0;
  P.one_shot = opts.task_ctas != 0 && !opts.split;
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
    cj.mark = SlotMark{t->wslot(slot), iteration, seq, t->wbase != nullptr ? 1u : 0u, 0};
    if (t2) cj.mark2 = SlotMark{t2->wslot(slot2), iteration, seq2, t2->wbase != nullptr ? 1u : 0u, 0};
    if (opts.fused_permille) {
      if (!P.copy_engine) {
        P.active = false;
        return fail(FFX_EINVAL, "fused_permille needs copy_engine (the fused kernel shares NVLink with the DMA)");
      }
      // Warp tasks [0, gcut) go through the fused kernel; each region's CE
      // range starts where its fused slices end.
      const uint64_t G = job.total_groups;
      P.gcut = G * std::min<uint32_t>(opts.fused_permille, 1000) / 1000;
      const uint64_t rows = job.rows;
      for (uint32_t i = 0; i < job.nregions; ++i) {
        const SliceRegion& R = job.reg[i];
        const uint64_t S = R.slice_bytes ? R.slice_bytes : job.slice_bytes;
        const uint64_t ns = slices_of(R.bytes, S);
        const uint64_t fs = P.gcut > R.group_base ? std::min(ns, (P.gcut - R.group_base) * rows) : 0;
        const uint64_t fb = std::min(R.bytes, fs * S);
        CopyRegion& C = cj.reg[i];
        C.src += fb;
        C.dst += fb;
        if (C.dst2) C.dst2 += fb;
        C.bytes -= fb;
      }
      finalize_copy_job(cj);
      P.fjob = job;  // copy + hash of the fused share, destinations kept
    }
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
    int32_t kind, pad_;
  } r[kMaxRegions];
};
static_assert(sizeof(RegionsBlob) <= FFX_REGIONS_HANDLE_BYTES, "regions handle too large");

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
    e.kind = r.kind;
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
      r->regs.push_back(SrcRegion{reinterpret_cast<const uint8_t*>(e.raw), e.bytes, e.kind});
    } else if (!(st = map(e.ipc, &base))) {
      r->regs.push_back(SrcRegion{base + e.off, e.bytes, e.kind});
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

// The ack word is a one-shot token: the holder's commit writes the pulled
// iteration, the origin's wait matches it EXACTLY and then consumes it
// (writes kAckNone back, stream-ordered).  A ">= iteration" test on a
// monotone word would let a replayed iteration after a rollback pass on the
// pre-failure maximum while the holder is still reading the live buffers.
extern "C" int ffx_snapshot_wait_pulled(ffx_ctx* c, uint64_t iteration, void* stream) {
  if (!c) return fail(FFX_EINVAL, "wait_pulled: null ctx");
  if (iteration == kAckNone) return fail(FFX_EINVAL, "wait_pulled: iteration %llu is reserved",
                                         (unsigned long long)iteration);
  using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
  using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
  static WaitFn wait = driver_fn<WaitFn>("cuStreamWaitValue64");
  static WriteFn write = driver_fn<WriteFn>("cuStreamWriteValue64");
  if (!wait || !write) return fail(FFX_ECUDA, "cuStreamWaitValue64 / cuStreamWriteValue64 unavailable");
  DeviceGuard g(c->device);
  const CUdeviceptr ack = reinterpret_cast<CUdeviceptr>(c->done + kAckWord);
  if (wait(static_cast<CUstream>(stream), ack, iteration, CU_STREAM_WAIT_VALUE_EQ) != CUDA_SUCCESS)
    return fail(FFX_ECUDA, "cuStreamWaitValue64 failed");
  if (write(static_cast<CUstream>(stream), ack, kAckNone, 0) != CUDA_SUCCESS)
    return fail(FFX_ECUDA, "cuStreamWriteValue64 failed");
  return FFX_OK;
}

extern "C" int ffx_snapshot_ack_reset(ffx_ctx* c, void* stream) {
  if (!c) return fail(FFX_EINVAL, "ack_reset: null ctx");
  DeviceGuard g(c->device);
  return reset_ack(c, as_stream(stream));
}

extern "C" int ffx_snapshot_begin(ffx_ctx* c, uint64_t iteration, const ffx_snapshot_opts* o,
                                  uint32_t* batches_out) {
  if (!c) return fail(FFX_EINVAL, "snapshot: null ctx");
  if (!c->target) return fail(FFX_ESTATE, "snapshot: no target replica (ffx_snapshot_target)");
  std::vector<SrcRegion> srcs;
  for (const auto& r : c->regions)
    if (r.unique) srcs.push_back(SrcRegion{r.dev, r.bytes, r.kind});
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
    vj.reg[i].src = readable(P.gcut ? P.fjob.reg[i].dst : P.split ? P.copy.reg[i].dst : vj.reg[i].dst);  // landed payload
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
  if (b == 0 && P.gcut) {
    // hybrid: the fused share (marks the slot WRITING; the commit waits for both queues)
    SliceJob fj = P.fjob;
    fj.group_lo = 0;
    fj.group_hi = P.gcut;
    fj.commit.finalize = 0;
    fj.commit2.finalize = 0;
    fj.sched = c->done + 20;
    FFX_CUDA(launch_slices(fj, SliceMode::Copy, true, P.hash_ctas, s));
    c->stats.kernel_launches++;
  }
  SliceJob hj = P.job;
  const uint64_t G0 = P.gcut, G = P.job.total_groups - P.gcut;
  hj.group_lo = G0 + G * b / P.hbatches;
  hj.group_hi = G0 + G * (b + 1) / P.hbatches;
  hj.commit.finalize = 0;
  hj.sched = c->done + 16;
  if (hj.group_lo == hj.group_hi) return FFX_OK;
  FFX_CUDA(launch_slices(hj, SliceMode::Hash, true, P.hash_ctas, s));
  c->stats.kernel_launches++;
  return FFX_OK;
}

int finish_snapshot(ffx_ctx* c, PendingSnapshot& P, cudaStream_t s) {
  P.active = false;
  FFX_CUDA(cudaEventRecord(c->snap_done, s));
  ffx_replica* t = P.tgt;
  t->cache[P.slot] = SlotCache{true, kSlotCommitted, P.iteration, P.seq};
  if (P.tgt2) P.tgt2->cache[P.slot2] = SlotCache{true, kSlotCommitted, P.iteration, P.seq2};
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
  if (*next == 0) FFX_CUDA(cudaStreamWaitEvent(s, c->snap_done, 0));  // the previous snapshot has drained
  const uint32_t b = (*next)++;

  if (!P.split) {
    // Fused: batch b covers warp tasks [G*b/B, G*(b+1)/B); the last commits.
    const uint64_t G = P.job.total_groups;
    SliceJob bj = P.job;
    bj.group_lo = P.cut(G, b);
    bj.group_hi = P.cut(G, b + 1);
    bj.commit.finalize = (b + 1 == P.batches);
    bj.commit2.finalize = bj.commit.finalize;
    if (P.one_shot) {
      // thousands of short CTAs: mark the slot WRITING once, stream-ordered
      // ahead of every payload store, instead of in each CTA
      if (b == 0) {
        FFX_CUDA(launch_mark(P.job.commit, P.job.commit2.slot ? &P.job.commit2 : nullptr, s));
        c->stats.kernel_launches++;
      }
      bj.one_shot = 1;
      bj.skip_begin = 1;
    }
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

extern "C" int ffx_snapshot_batch_span(ffx_ctx* c, uint32_t batch, uint64_t* lo, uint64_t* hi) {
  if (!c || !lo || !hi) return fail(FFX_EINVAL, "snapshot_batch_span: null argument");
  const PendingSnapshot& P = c->pending;
  if (!P.active || P.split) return fail(FFX_ESTATE, "snapshot_batch_span: no fused snapshot pending");
  if (batch >= P.batches) return fail(FFX_ERANGE, "snapshot_batch_span: batch %u of %u", batch, P.batches);
  const SliceJob& J = P.job;
  const uint64_t G = J.total_groups;
  const uint64_t g0 = P.cut(G, batch), g1 = P.cut(G, batch + 1);
  // job region of warp task g, and the logical bytes [first, end) the task reads
  auto span_of = [&](uint64_t g, uint64_t* first, uint64_t* end) {
    uint32_t r = 0;
    for (uint32_t i = 1; i < J.nregions; ++i)
      if (J.reg[i].group_base <= g) r = i;
    const SliceRegion& R = J.reg[r];
    const uint64_t S = R.slice_bytes ? R.slice_bytes : J.slice_bytes;
    const uint64_t a = std::min(R.bytes, (g - R.group_base) * J.rows * S);
    const uint64_t b = std::min(R.bytes, a + static_cast<uint64_t>(J.rows) * S);
    *first = P.logical_of[r] + a;
    *end = P.logical_of[r] + b;
  };
  if (g0 >= g1) {  // an empty batch reads nothing
    uint64_t f = 0, e = 0;
    if (g0 < G) span_of(g0, &f, &e);
    else f = P.logical;
    *lo = *hi = f;
    return FFX_OK;
  }
  uint64_t f0, e0, f1, e1;
  span_of(g0, &f0, &e0);
  span_of(g1 - 1, &f1, &e1);
  *lo = f0;
  *hi = e1;
  return FFX_OK;
}

extern "C" int ffx_snapshot_from_host(ffx_ctx* c, uint64_t iteration, const void* host, uint64_t len,
                                      uint32_t batches, void* stream) {
  if (!c) return fail(FFX_EINVAL, "snapshot_from_host: null ctx");
  if (len && !host) return fail(FFX_EINVAL, "snapshot_from_host: null host pointer");
  const PayloadMap pm = payload_map(c);
  if (len != pm.logical)
    return fail(FFX_ECONFIG, "snapshot_from_host: %llu host bytes, the registered regions hold %llu",
                (unsigned long long)len, (unsigned long long)pm.logical);
  DeviceGuard g(c->device);
  if (!c->h2d) FFX_CUDA(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
  ffx_snapshot_opts o{};
  // ~8 batches for large payloads: each batch's kernel runs under the next
  // chunk's copy, only the last one (~1/8 of the kernel) is exposed
  o.batches = batches ? batches : (len >= (64ull << 20) ? 8u : 1u);
  uint32_t nb = 1;
  if (int st = ffx_snapshot_begin(c, iteration, &o, &nb)) return st;
  cudaStream_t s = as_stream(stream);
  // A failure after begin abandons the snapshot: its slot is left torn
  // (never restored from) and the next snapshot still waits for whatever
  // batches of this one were issued.
  auto abandon = [&](int st) {
    PendingSnapshot& P = c->pending;
    if (P.active) {
      P.active = false;
      P.tgt->cache[P.slot].state = kSlotWriting;
      if (P.tgt2) P.tgt2->cache[P.slot2].state = kSlotWriting;
      cudaEventRecord(c->snap_done, s);
    }
    return st;
  };
  while (c->h2d_ev.size() < nb + 1) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return abandon(fail(FFX_ECUDA, "snapshot_from_host: event creation failed"));
    c->h2d_ev.push_back(e);
  }
  // the copies overwrite the registered regions: after earlier work on `stream`
  if (cudaEventRecord(c->h2d_ev[nb], s) != cudaSuccess || cudaStreamWaitEvent(c->h2d, c->h2d_ev[nb], 0) != cudaSuccess)
    return abandon(fail(FFX_ECUDA, "snapshot_from_host: cannot order the copy stream"));
  const uint8_t* src = static_cast<const uint8_t*>(host);
  uint64_t copied = 0;  // logical bytes already queued
  for (uint32_t b = 0; b < nb; ++b) {
    uint64_t lo = 0, hi = 0;
    if (int st = ffx_snapshot_batch_span(c, b, &lo, &hi)) return abandon(st);
    hi = b + 1 == nb ? pm.logical : std::max(hi, copied);
    // queue [copied, hi): region by region (the payload is the regions concatenated)
    uint64_t at = 0;
    for (size_t r = 0; r < pm.regs.size() && copied < hi; ++r) {
      const uint64_t rb = pm.regs[r]->bytes;
      if (copied < at + rb) {
        const uint64_t n = std::min(hi, at + rb) - copied;
        const cudaError_t e =
            cudaMemcpyAsync(pm.regs[r]->dev + (copied - at), src + copied, n, cudaMemcpyHostToDevice, c->h2d);
        if (e != cudaSuccess) return abandon(cuda_fail(e, "snapshot_from_host: H2D"));
        copied += n;
      }
      at += rb;
    }
    if (cudaEventRecord(c->h2d_ev[b], c->h2d) != cudaSuccess)
      return abandon(fail(FFX_ECUDA, "snapshot_from_host: event record failed"));
    uint32_t left = 0;
    if (int st = ffx_snapshot_next(c, stream, c->h2d_ev[b], &left)) return abandon(st);
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

