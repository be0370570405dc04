// ffx_control.cpp -- the C ABI, part 7: the controller state that drives the
// hot path, host-only.
//
//   ffx_heartbeats  ctl::HeartbeatTable (controller.hpp:56-101,
//                   controller.cpp:16-77): one slot per pod, O(1) reports,
//                   a sweep declares pods silent for > interval * threshold.
//   ffx_ledger      ctl::IterationLedger (controller.hpp:106-130,
//                   controller.cpp:81-121): per-worker latest recoverable
//                   iteration; the global consistent iteration is the minimum
//                   over the whole grid, absent workers counting as zero.
//                   ffx_ledger_record_replica is the CkptRecord the holder's
//                   agent sends after each committed replica (wire.hpp:85-90),
//                   read straight from the replica's slot headers.
//
// The reference keeps the ledger in a std::map<Role, u64>; here it is a
// dense array indexed by the role's global index (domain.cpp:32-40) with a
// presence count, so record / worker_latest are O(1) and global_consistent is
// one linear scan with no allocation.  Both objects take a mutex: heartbeat
// receivers and the recovery driver may sit on different host threads (the
// reference runs everything on one SimLoop thread, runtime.hpp:5-10).
// Timestamps are caller-supplied nanoseconds (rt::Nanos), so simulated and
// wall clocks both work; ffx_now_ns gives CLOCK_MONOTONIC.
// Plain host C++ (g++, no CUDA headers), so it also builds under
// -fsanitize=thread for tests/cpp/test_control_threads.cpp.
#include <time.h>

#include <algorithm>
#include <cstdint>
#include <mutex>
#include <new>
#include <vector>

#include "ffx.h"

namespace ffx::host {
int fail(int status, const char* fmt, ...);  // ffx_api.cu: sets ffx_last_error()
}
using ffx::host::fail;

struct ffx_heartbeats {
  struct Slot {
    bool enrolled = false;
    bool failed = false;
    int64_t last_seen = 0;
    uint64_t last_iteration = 0;
  };
  std::mutex mu;
  std::vector<Slot> slots;
  int64_t interval_ns = 0;
  uint32_t miss_threshold = 0;
  uint64_t unknown = 0, late = 0, regressed = 0;
};

struct ffx_ledger {
  std::mutex mu;
  ffx_cluster_spec spec{};
  std::vector<uint64_t> latest;  // by global index
  std::vector<uint8_t> present;
  uint64_t n_present = 0;
};

namespace {

uint64_t world_of(const ffx_cluster_spec& s) {
  return uint64_t(s.data_parallel) * s.pipeline_parallel * s.tensor_parallel;
}

// ClusterSpec::world_size() = num_nodes * gpus_per_node, a u32 product
// (domain.hpp:72); the reference's global_consistent compares the number of
// recorded workers against it.
uint32_t world_u32(const ffx_cluster_spec& s) { return s.num_nodes * s.gpus_per_node; }

uint64_t index_in(const ffx_cluster_spec& s, ffx_role r) {
  return (uint64_t(r.dp) * s.pipeline_parallel + r.pp) * s.tensor_parallel + r.tp;
}

bool in_grid(const ffx_cluster_spec& s, ffx_role r) {
  return r.dp < s.data_parallel && r.pp < s.pipeline_parallel && r.tp < s.tensor_parallel;
}

}  // namespace

extern "C" int64_t ffx_now_ns(void) {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return int64_t(ts.tv_sec) * 1000000000LL + ts.tv_nsec;
}

// ---- heartbeats (controller.cpp:16-77) ---------------------------------------

extern "C" int ffx_heartbeats_create(uint32_t pods, int64_t interval_ns, uint32_t miss_threshold,
                                     ffx_heartbeats** out) {
  if (!out) return fail(FFX_EINVAL, "heartbeats_create: null argument");
  auto* h = new (std::nothrow) ffx_heartbeats;
  if (!h) return fail(FFX_ENOMEM, "heartbeats_create");
  h->slots.resize(pods);
  h->interval_ns = interval_ns;
  h->miss_threshold = miss_threshold;
  *out = h;
  return FFX_OK;
}

extern "C" int ffx_heartbeats_destroy(ffx_heartbeats* h) {
  delete h;
  return FFX_OK;
}

// controller.cpp:21-28 (slots_.at: std::out_of_range -> FFX_ERANGE)
extern "C" int ffx_heartbeats_enroll(ffx_heartbeats* h, uint32_t node, uint64_t iteration, int64_t now_ns) {
  if (!h) return fail(FFX_EINVAL, "heartbeats_enroll: null argument");
  std::lock_guard<std::mutex> l(h->mu);
  if (node >= h->slots.size()) return fail(FFX_ERANGE, "heartbeats_enroll: node %u of %zu", node, h->slots.size());
  auto& s = h->slots[node];
  s.enrolled = true;
  s.failed = false;
  s.last_seen = now_ns;
  s.last_iteration = iteration;
  return FFX_OK;
}

// controller.cpp:30-44: oddities are counted, never an error
extern "C" int ffx_heartbeats_observe(ffx_heartbeats* h, uint32_t node, uint64_t iteration, int64_t now_ns) {
  if (!h) return fail(FFX_EINVAL, "heartbeats_observe: null argument");
  std::lock_guard<std::mutex> l(h->mu);
  if (node >= h->slots.size() || !h->slots[node].enrolled) {
    ++h->unknown;
    return FFX_OK;
  }
  auto& s = h->slots[node];
  if (s.failed) {
    ++h->late;
    return FFX_OK;
  }
  if (iteration < s.last_iteration) ++h->regressed;
  s.last_iteration = iteration;
  s.last_seen = now_ns;
  return FFX_OK;
}

// controller.cpp:46-58.  Newly dead pods in node order; at most `cap` are
// written to `dead` (n_dead is the full count -- every one is marked failed
// either way, so size `dead` for the pod count).
extern "C" int ffx_heartbeats_sweep(ffx_heartbeats* h, int64_t now_ns, uint32_t* dead, uint32_t cap,
                                    uint32_t* n_dead) {
  if (!h || !n_dead || (cap && !dead)) return fail(FFX_EINVAL, "heartbeats_sweep: null argument");
  std::lock_guard<std::mutex> l(h->mu);
  const int64_t limit = h->interval_ns * int64_t(h->miss_threshold);
  uint32_t n = 0;
  for (uint32_t i = 0; i < h->slots.size(); ++i) {
    auto& s = h->slots[i];
    if (!s.enrolled || s.failed) continue;
    if (now_ns - s.last_seen > limit) {
      s.failed = true;
      if (n < cap) dead[n] = i;
      ++n;
    }
  }
  *n_dead = n;
  return FFX_OK;
}

// controller.cpp:60-62
extern "C" int ffx_heartbeats_mark_failed(ffx_heartbeats* h, uint32_t node) {
  if (!h) return fail(FFX_EINVAL, "heartbeats_mark_failed: null argument");
  std::lock_guard<std::mutex> l(h->mu);
  if (node >= h->slots.size()) return fail(FFX_ERANGE, "heartbeats_mark_failed: node %u", node);
  h->slots[node].failed = true;
  return FFX_OK;
}

// controller.cpp:64-77: enrolled/failed are false for unknown nodes; the
// last_* accessors throw (FFX_ERANGE) there, as slots_.at does.
extern "C" int ffx_heartbeats_query(ffx_heartbeats* h, uint32_t node, ffx_heartbeat_slot* out) {
  if (!h || !out) return fail(FFX_EINVAL, "heartbeats_query: null argument");
  std::lock_guard<std::mutex> l(h->mu);
  if (node >= h->slots.size()) return fail(FFX_ERANGE, "heartbeats_query: node %u", node);
  const auto& s = h->slots[node];
  out->enrolled = s.enrolled;
  out->failed = s.failed;
  out->last_seen_ns = s.last_seen;
  out->last_iteration = s.last_iteration;
  return FFX_OK;
}

extern "C" int ffx_heartbeats_counters(ffx_heartbeats* h, uint64_t* unknown, uint64_t* late, uint64_t* regressed) {
  if (!h) return fail(FFX_EINVAL, "heartbeats_counters: null argument");
  std::lock_guard<std::mutex> l(h->mu);
  if (unknown) *unknown = h->unknown;
  if (late) *late = h->late;
  if (regressed) *regressed = h->regressed;
  return FFX_OK;
}

// ---- iteration ledger (controller.cpp:81-121) --------------------------------

extern "C" int ffx_ledger_create(const ffx_cluster_spec* spec, ffx_ledger** out) {
  if (!spec || !out) return fail(FFX_EINVAL, "ledger_create: null argument");
  const uint64_t w = world_of(*spec);
  if (w > (1ull << 32)) return fail(FFX_EINVAL, "ledger_create: grid of %llu workers", (unsigned long long)w);
  auto* g = new (std::nothrow) ffx_ledger;
  if (!g) return fail(FFX_ENOMEM, "ledger_create");
  g->spec = *spec;
  g->latest.assign(w, 0);
  g->present.assign(w, 0);
  *out = g;
  return FFX_OK;
}

extern "C" int ffx_ledger_destroy(ffx_ledger* g) {
  delete g;
  return FFX_OK;
}

// controller.cpp:83-90: a role outside the grid is a protocol error
// (net::ProtocolError -> FFX_ERANGE); an older record is a no-op.
extern "C" int ffx_ledger_record(ffx_ledger* g, ffx_role role, uint64_t iteration) {
  if (!g) return fail(FFX_EINVAL, "ledger_record: null argument");
  if (!in_grid(g->spec, role))
    return fail(FFX_ERANGE, "ledger_record: role d%up%ut%u outside the grid", role.dp, role.pp, role.tp);
  std::lock_guard<std::mutex> l(g->mu);
  const uint64_t i = index_in(g->spec, role);
  if (!g->present[i]) {
    g->present[i] = 1;
    ++g->n_present;
  }
  if (iteration > g->latest[i]) g->latest[i] = iteration;
  return FFX_OK;
}

// controller.cpp:92-97
extern "C" uint64_t ffx_ledger_global_consistent(ffx_ledger* g) {
  if (!g) return 0;
  std::lock_guard<std::mutex> l(g->mu);
  if (g->n_present < world_u32(g->spec)) return 0;
  uint64_t low = UINT64_MAX;
  for (uint64_t i = 0; i < g->latest.size(); ++i)
    if (g->present[i] && g->latest[i] < low) low = g->latest[i];
  return low;
}

// controller.cpp:99-110: dp_group = pp * tensor_parallel + tp (the u16
// narrowing of the reference kept); members never recorded count as 0.
extern "C" uint64_t ffx_ledger_group_latest(ffx_ledger* g, uint32_t dp_group) {
  if (!g) return 0;
  std::lock_guard<std::mutex> l(g->mu);
  const auto& s = g->spec;
  if (s.tensor_parallel == 0 || s.data_parallel == 0) return 0;
  const ffx_role base{0, uint16_t(dp_group / s.tensor_parallel), uint16_t(dp_group % s.tensor_parallel)};
  if (!in_grid(s, ffx_role{0, base.pp, base.tp})) return 0;
  uint64_t low = UINT64_MAX;
  for (uint32_t dp = 0; dp < s.data_parallel && dp <= 0xFFFF; ++dp) {
    const uint64_t i = index_in(s, ffx_role{uint16_t(dp), base.pp, base.tp});
    low = std::min(low, g->present[i] ? g->latest[i] : 0);
  }
  return low == UINT64_MAX ? 0 : low;
}

// controller.cpp:112-115
extern "C" uint64_t ffx_ledger_worker_latest(ffx_ledger* g, ffx_role role) {
  if (!g || !in_grid(g->spec, role)) return 0;
  std::lock_guard<std::mutex> l(g->mu);
  const uint64_t i = index_in(g->spec, role);
  return g->present[i] ? g->latest[i] : 0;
}

// controller.cpp:117-121: every worker's recoverable state is `iteration`
extern "C" int ffx_ledger_rebase(ffx_ledger* g, uint64_t iteration) {
  if (!g) return fail(FFX_EINVAL, "ledger_rebase: null argument");
  std::lock_guard<std::mutex> l(g->mu);
  std::fill(g->latest.begin(), g->latest.end(), iteration);
  std::fill(g->present.begin(), g->present.end(), uint8_t(1));
  g->n_present = g->latest.size();
  return FFX_OK;
}

// The CkptRecord of a completed replica (wire.hpp:85-90): the holder records
// its origin at the newest COMMITTED iteration of the replica it holds (a
// slot still WRITING never counts -- the reference sends the record only
// after NeighborBuffer::store returned, ckpt.cpp:77-105).  *recorded = the
// iteration recorded, 0 when the replica holds nothing committed yet.
extern "C" int ffx_ledger_record_replica(ffx_ledger* g, ffx_replica* held, uint64_t* recorded) {
  if (!g || !held) return fail(FFX_EINVAL, "ledger_record_replica: null argument");
  uint32_t versions = 0;
  int rc = ffx_replica_slots(held, &versions);
  if (rc) return rc;
  ffx_slot_info best{};
  bool any = false;
  for (uint32_t s = 0; s < versions; ++s) {  // newest committed = largest write sequence
    ffx_slot_info si{};
    if ((rc = ffx_replica_slot_info(held, s, &si))) return rc;
    if (si.state == 2 && (!any || si.seq > best.seq)) {
      best = si;
      any = true;
    }
  }
  if (recorded) *recorded = 0;
  if (!any) return FFX_OK;  // nothing committed yet: no record
  if ((rc = ffx_ledger_record(g, best.role, best.iteration))) return rc;
  if (recorded) *recorded = best.iteration;
  return FFX_OK;
}
