// ffx_recover.cu -- the C ABI, part 4: recovery gather + verify
// (assemble_restore, ckpt.cpp:111-167), CUDA IPC helpers, failure injection
// and statistics.
#include "ffx_host.h"

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
  if (int st = check_meta(src, *m)) return st;
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

// The slot's regions, payload and slicing agree with each other and with the
// replica's layout: a corrupt meta must not steer a job (or an export) past
// the payload or the table.
int ffx::host::check_meta(const ffx_replica* r, const SlotMeta& m) {
  if (m.num_regions > kMaxRegions) return fail(FFX_ECORRUPT, "slot metadata: %u regions", m.num_regions);
  uint64_t logical = 0, physical = 0;
  for (uint32_t i = 0; i < m.num_regions; ++i) {
    if (m.region_bytes[i] > r->capacity)
      return fail(FFX_ECORRUPT, "slot metadata: region %u of %llu bytes", i, (unsigned long long)m.region_bytes[i]);
    logical += m.region_bytes[i];
    physical = align_up(physical + m.region_bytes[i], kRegionAlign);
  }
  if (logical != m.payload_len || m.payload_len > r->capacity || physical > r->layout.payload_cap)
    return fail(FFX_ECORRUPT, "slot metadata: payload %llu bytes, regions %llu, capacity %llu",
                (unsigned long long)m.payload_len, (unsigned long long)logical, (unsigned long long)r->capacity);
  if (!slice_ok(m.slice_bytes))
    return fail(FFX_ECORRUPT, "slot metadata: slice size %llu", (unsigned long long)m.slice_bytes);
  const uint64_t want = table_entries(m.region_bytes, m.num_regions, m.slice_bytes);
  if (m.num_slices != want || want > r->layout.table_cap)
    return fail(FFX_ECORRUPT, "slot metadata: %llu table entries, the regions need %llu",
                (unsigned long long)m.num_slices, (unsigned long long)want);
  return FFX_OK;
}

int ffx::host::reset_ack(ffx_ctx* c, cudaStream_t s) {
  FFX_CUDA(cudaMemsetAsync(c->done + kAckWord, 0xff, 8, s));
  return FFX_OK;
}

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
  const uint64_t S = m[0].slice_bytes;
  const std::vector<RunRef> runs = payload_runs(pm, S);
  if (runs.size() * nsrc > kMaxRegions) nsrc = 1;  // not enough region entries to split

  // Parallel peer gathers: every slice run (ffx_layout.h) is cut into nsrc
  // consecutive parts, part i pulled from source i.  Parts keep payload
  // order, so the global slice numbering (and the checksum table) is that
  // of the whole snapshot; every part verifies against source 0's table.
  cudaStream_t s = as_stream(stream);
  SliceJob job{};
  for (const RunRef& q : runs) {
    const uint64_t ns = run_slices(q.run);
    for (uint32_t i = 0; i < nsrc; ++i) {
      const uint64_t a = ns * i / nsrc, b = ns * (i + 1) / nsrc;
      const uint64_t lo = q.run.offset + a * q.run.slice;
      const uint64_t hi = std::min(q.run.offset + b * q.run.slice, q.run.offset + q.run.bytes);
      if (hi <= lo && !(nsrc == 1)) continue;
      SliceRegion part{srcs[i]->payload(slot[i]) + pm.offs[q.region] + lo, pm.regs[q.region]->dev + lo, hi - lo, 0, 0};
      part.slice_bytes = static_cast<uint32_t>(q.run.slice);
      job.reg[job.nregions++] = part;
    }
  }
  job.slice_bytes = S;
  job.sums_expected = srcs[0]->sums(slot[0]);
  job.result = c->result;
  job.sched = c->done + 12;
  finalize_job(job);
  // restored state = a rollback: an ack left over from before the failure
  // must not release a replayed iteration's optimizer update
  if (int ast = reset_ack(c, s)) return ast;
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
  auto add = [&](const uint8_t* src, uint8_t* dst, uint64_t bytes, const uint64_t* expected, uint64_t slice) -> int {
    if (job.nregions >= kMaxRegions) return fail(FFX_ECONFIG, "recover_full: more than %u parts", kMaxRegions);
    SliceRegion sr{src, dst, bytes, 0, 0};
    sr.expected = expected;
    sr.slice_bytes = static_cast<uint32_t>(slice);
    job.reg[job.nregions++] = sr;
    return FFX_OK;
  };
  uint64_t total = 0, base = 0;  // base: table entries of the runs before this one
  for (const RunRef& q : payload_runs(pm, S)) {
    const uint64_t ns = run_slices(q.run);
    for (uint32_t i = 0; i < nsrc; ++i) {
      const uint64_t a = ns * i / nsrc, b = ns * (i + 1) / nsrc;
      const uint64_t lo = q.run.offset + a * q.run.slice;
      const uint64_t hi = std::min(q.run.offset + b * q.run.slice, q.run.offset + q.run.bytes);
      if (hi <= lo) continue;
      int st = add(srcs[i]->payload(slot[i]) + pm.offs[q.region] + lo, pm.regs[q.region]->dev + lo, hi - lo,
                   srcs[i]->sums(slot[i]) + base + a, q.run.slice);
      if (st) return st;
    }
    base += ns;
    total += q.run.bytes;
  }
  for (uint32_t j = 0; j < nred; ++j) {
    const ffx_peer_region& pr = redundant[j];
    if (pr.region_index >= c->regions.size() || c->regions[pr.region_index].unique)
      return fail(FFX_ERANGE, "recover_full: region %u is not a registered redundant region", pr.region_index);
    if (!pr.src || !pr.sums) return fail(FFX_EINVAL, "recover_full: null peer pointer");
    if (pr.slice_bytes && pr.slice_bytes != c->slice_bytes)
      return fail(FFX_ECONFIG, "recover_full: region %u's peer table has %u-byte slices, the context %llu",
                  pr.region_index, pr.slice_bytes, (unsigned long long)c->slice_bytes);
    const Region& reg = c->regions[pr.region_index];
    int st = add(static_cast<const uint8_t*>(pr.src), reg.dev, reg.bytes, pr.sums, S);  // peer tables: uniform
    if (st) return st;
    total += reg.bytes;
  }
  cudaStream_t s = as_stream(stream);
  job.slice_bytes = S;
  job.result = c->result;
  job.sched = c->done + 12;
  finalize_job(job);
  // restored state = a rollback: an ack left over from before the failure
  // must not release a replayed iteration's optimizer update
  if (int ast = reset_ack(c, s)) return ast;
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

// NeighborBuffer::store validates a frame before accepting it (ckpt.cpp:78,
// storage.cpp:98-99).  On the B200 the bytes land first; the holder then
// re-hashes the committed slot from its own HBM against the slot's table
// (computed by the origin from its source bytes) -- checksum-as-landed, one
// local HBM read, no NVLink traffic.  A mismatch drops the slot to WRITING
// (torn: never restored from) and returns FFX_ECORRUPT with the first slice.
extern "C" int ffx_replica_verify(ffx_ctx* c, ffx_replica* held, uint64_t iteration, uint32_t max_ctas,
                                  void* stream, ffx_recover_report* rep) {
  if (!c || !held) return fail(FFX_EINVAL, "replica_verify: null argument");
  if (!held->owned) return fail(FFX_EINVAL, "replica_verify: only the holder verifies (its local HBM)");
  DeviceGuard g(c->device);
  ffx_recover_report local{};
  ffx_recover_report& R = rep ? *rep : local;
  std::memset(&R, 0, sizeof R);
  R.first_bad_slice = ~0ull;
  SlotMeta m;
  const int v = find_slot(held, iteration, &m);
  if (v == -2) return fail(FFX_ECUDA, "replica_verify: cannot read slot metadata: %s", g_err.c_str());
  if (v < 0 || m.state != kSlotCommitted)
    return fail(FFX_ERESTORE, "replica_verify: no committed snapshot at iteration %llu", (unsigned long long)iteration);
  if (int st = check_meta(held, m)) return st;
  SliceJob job{};
  uint64_t phys = 0;
  for (uint32_t i = 0; i < m.num_regions; ++i) {
    SliceRun runs[kRegionRuns];
    const int k = region_runs(m.region_bytes[i], m.slice_bytes, head_region(i, m.num_regions), runs);
    for (int j = 0; j < k; ++j) {
      SliceRegion part{held->payload(v) + phys + runs[j].offset, nullptr, runs[j].bytes, 0, 0};
      part.slice_bytes = static_cast<uint32_t>(runs[j].slice);
      job.reg[job.nregions++] = part;
    }
    phys = align_up(phys + m.region_bytes[i], kRegionAlign);
  }
  job.slice_bytes = m.slice_bytes;
  job.sums_expected = held->sums(v);
  job.result = c->result;
  job.sched = c->done + 12;
  finalize_job(job, rows_for_cap(max_ctas));
  cudaStream_t s = as_stream(stream);
  const unsigned long long init[2] = {~0ull, 0ull};
  FFX_CUDA(cudaMemcpyAsync(c->result, init, sizeof init, cudaMemcpyHostToDevice, s));
  FFX_CUDA(cudaEventRecord(c->ev0, s));
  FFX_CUDA(launch_slices(job, SliceMode::HashVerify, false, max_ctas, s));
  FFX_CUDA(cudaEventRecord(c->ev1, s));
  c->stats.kernel_launches++;
  FFX_CUDA(cudaMemcpyAsync(c->result_host, c->result, 16, cudaMemcpyDeviceToHost, s));
  FFX_CUDA(cudaStreamSynchronize(s));
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev0, c->ev1);
  R.seconds = ms * 1e-3;
  R.bytes = m.payload_len;
  R.slot = static_cast<uint32_t>(v);
  R.first_bad_slice = c->result_host[0];
  R.bad_slices = c->result_host[1];
  if (R.bad_slices) {
    c->stats.verify_failures++;
    const uint32_t torn = kSlotWriting;
    FFX_CUDA(cudaMemcpy(held->slot(static_cast<uint32_t>(v)) + offsetof(SlotMeta, state), &torn, 4,
                        cudaMemcpyHostToDevice));
    held->cache[v].state = kSlotWriting;
    return fail(FFX_ECORRUPT, "replica_verify: %llu slices differ from the origin's table (first %llu); "
                "slot %d dropped", (unsigned long long)R.bad_slices, (unsigned long long)R.first_bad_slice, v);
  }
  return FFX_OK;
}

extern "C" int ffx_recover(ffx_ctx* c, ffx_replica* src, uint64_t target, void* stream,
                           ffx_recover_report* rep) {
  if (!c || !src) return fail(FFX_EINVAL, "recover: null argument");
  return ffx_recover_from(c, &src, 1, target, stream, rep);
}

extern "C" int ffx_recover_region(ffx_ctx* c, const ffx_peer_region* peer, void* stream, ffx_recover_report* rep) {
  if (!c || !peer || !peer->src || !peer->sums) return fail(FFX_EINVAL, "recover_region: null argument");
  const uint32_t idx = peer->region_index;
  const void* peer_src = peer->src;
  const uint64_t* peer_sums = peer->sums;
  if (idx >= c->regions.size()) return fail(FFX_ERANGE, "recover_region: no region %u", idx);
  if (peer->slice_bytes && peer->slice_bytes != c->slice_bytes)
    return fail(FFX_ECONFIG, "recover_region: the peer table has %u-byte slices, the context %llu",
                peer->slice_bytes, (unsigned long long)c->slice_bytes);
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
  // restored state = a rollback: an ack left over from before the failure
  // must not release a replayed iteration's optimizer update
  if (int ast = reset_ack(c, s)) return ast;
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

