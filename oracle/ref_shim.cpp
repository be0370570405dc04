// ref_shim.cpp -- extern "C" entry points onto the UNMODIFIED reference
// library (proj/src/{hash,storage,ckpt,evolution,domain,dataloader,
// controller + its network-stack deps}.cpp), compiled by
// oracle/Makefile into oracle/_ref/libftsim_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by oracle/gen_golden.py to produce the golden
// fixtures, by tests/ to cross-check the C restatement, and by bench.py's
// reference arm / cpu_baseline leg to time the reference's own CPU path.
// Nothing here is linked into libffx.so.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "ftsim/ckpt.hpp"
#include "ftsim/controller.hpp"
#include "ftsim/transport.hpp"
#include "ftsim/dataloader.hpp"
#include "ftsim/evolution.hpp"
#include "ftsim/hash.hpp"
#include "ftsim/storage.hpp"

using namespace ftsim;

extern "C" {

std::uint64_t ref_checksum64(const void* p, std::uint64_t n) { return checksum64(p, n); }

void ref_optimizer_init(std::uint64_t seed, std::uint16_t dp, std::uint16_t pp,
                        std::uint16_t tp, int distributed, std::uint8_t* out) {
  const auto d = evo::optimizer_init(seed, Role{dp, pp, tp}, distributed != 0);
  std::memcpy(out, d.data(), 32);
}

// The rank's optimizer digest after n iterations, through the reference's
// own evolution + data-window functions (evolution.cpp:26-69,
// dataloader.cpp:36-49, :166-171); the assignment restates
// controller.cpp:127-140 (that file drags in the network stack).
int ref_optimizer_at(std::uint64_t seed, std::uint16_t dp, std::uint16_t pp, std::uint16_t tp, std::uint32_t d,
                     std::uint32_t p, std::uint32_t t, std::uint32_t batch, std::uint64_t n, int distributed,
                     std::uint8_t* out) {
  const std::uint32_t world = d * p * t;
  if (world == 0 || batch % world != 0) return -1;
  wire::IndexAssign a;
  a.start_iteration = 0;
  a.per_column = batch / world;
  a.columns = world;
  a.base_index = 0;
  const Role r{dp, pp, tp};
  const std::uint32_t column = (static_cast<std::uint32_t>(dp) * p + pp) * t + tp;
  auto dig = evo::optimizer_init(seed, r, distributed != 0);
  for (std::uint64_t it = 1; it <= n; ++it) {
    const auto w = data::window_of(a, column, it);
    const auto lanes = evo::grad_contribution(seed, r, it, data::window_fold(seed, w));
    dig = evo::optimizer_next(dig, evo::grad_digest(lanes));
  }
  std::memcpy(out, dig.data(), 32);
  return 0;
}

void ref_weights_init(std::uint64_t seed, std::uint16_t pp, std::uint16_t tp, std::uint8_t* out) {
  const auto d = evo::weights_init(seed, Role{0, pp, tp});
  std::memcpy(out, d.data(), 32);
}

int ref_materialize(const std::uint8_t* digest, std::uint64_t bytes, std::uint8_t* out) {
  Digest d;
  std::memcpy(d.data(), digest, 32);
  try {
    const auto v = evo::materialize(d, bytes);
    std::memcpy(out, v.data(), v.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

void ref_expand(const std::uint8_t* digest, std::uint64_t bytes, std::uint8_t* out) {
  Digest d;
  std::memcpy(d.data(), digest, 32);
  const auto v = evo::expand(d, bytes);
  if (!v.empty()) std::memcpy(out, v.data(), v.size());
}

int ref_blob_is_sound(const std::uint8_t* p, std::uint64_t n) {
  return evo::blob_is_sound(std::vector<std::uint8_t>(p, p + n)) ? 1 : 0;
}

std::uint64_t ref_optimizer_bytes(std::uint64_t phi, std::uint32_t d, int distributed) {
  ClusterSpec cs;
  cs.params_per_device = phi;
  cs.data_parallel = d;
  cs.distributed_optimizer = distributed != 0;
  return evo::optimizer_bytes(cs);
}

std::uint64_t ref_razor(std::uint64_t phi, std::uint32_t d, int distributed, int* flags) {
  ClusterSpec cs;
  cs.params_per_device = phi;
  cs.data_parallel = d;
  cs.distributed_optimizer = distributed != 0;
  const auto p = ckpt::razor(cs);
  flags[0] = p.weights_redundant;
  flags[1] = p.optimizer_redundant;
  return p.unique_bytes_per_device;
}

int ref_version_for_target(std::uint64_t held, std::uint64_t target) {
  try {
    return ckpt::version_for_target(held, target);
  } catch (const ckpt::VersionError&) {
    return -1;
  }
}

// Frame into `out` (32 + len bytes).  -1 where pack_blob throws.
int ref_pack_blob(std::uint16_t dp, std::uint16_t pp, std::uint16_t tp, std::uint64_t it,
                  int kind, const void* payload, std::uint64_t len, std::uint8_t* out) {
  try {
    const auto f = store::pack_blob(Role{dp, pp, tp}, it, static_cast<store::BlobKind>(kind),
                                    payload, len);
    std::memcpy(out, f.data(), f.size());
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

// 0 valid, 1 CorruptSnapshot.
int ref_unpack_ok(const std::uint8_t* f, std::uint64_t n) {
  try {
    store::unpack_blob(std::vector<std::uint8_t>(f, f + n));
    return 0;
  } catch (const store::CorruptSnapshot&) {
    return 1;
  }
}

// The reference's per-iteration CPU hot path, timed.  One std::thread per
// ring rank: HostSnapshots::take (pack + FNV) ->
// NeighborBuffer::store at the holder (by-value copy + unpack + FNV verify)
// -> assemble_restore of the unique piece (unpack + FNV).  Payloads are
// evo::materialize(optimizer_init(42, role, true), bytes), built once by
// ref_ring_setup outside any timed region.
struct RefRing {
  int threads;
  std::uint64_t bytes;
  std::vector<std::vector<std::uint8_t>> blobs;
};

void* ref_ring_setup(int threads, std::uint64_t bytes) {
  auto* r = new RefRing{threads, bytes, std::vector<std::vector<std::uint8_t>>(threads)};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([r, t] {
      r->blobs[t] = evo::materialize(
          evo::optimizer_init(42, Role{static_cast<std::uint16_t>(t), 0, 0}, true), r->bytes);
    });
  for (auto& th : pool) th.join();
  return r;
}

void ref_ring_free(void* h) { delete static_cast<RefRing*>(h); }

// Per-stage seconds (max over threads) into secs[0..2] (take, store,
// restore), the wall time of the whole parallel iteration into secs[3], and
// the snapshot time of the slowest thread -- max over threads of that
// thread's own take + store -- into secs[4].
// Returns 0, or -1 if any stage threw or restored the wrong size.
int ref_ring_run(void* h, std::uint64_t iteration, double* secs) {
  auto* r = static_cast<RefRing*>(h);
  const int threads = r->threads;
  const std::uint64_t bytes = r->bytes;
  std::vector<double> st(3 * threads, 0.0);
  std::vector<int> ok(threads, 0);
  std::vector<std::thread> pool;
  using clk = std::chrono::steady_clock;
  const auto w0 = clk::now();
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        const Role me{static_cast<std::uint16_t>(t), 0, 0};
        ckpt::HostSnapshots hs(me, bytes);
        ckpt::NeighborBuffer nb(me);  // the ring successor's buffer for `me`
        auto t0 = clk::now();
        hs.take(iteration, r->blobs[t].data(), r->blobs[t].size());
        auto t1 = clk::now();
        nb.store(*hs.framed(iteration));
        auto t2 = clk::now();
        ckpt::UniquenessPlan plan;
        plan.weights_redundant = true;
        plan.unique_bytes_per_device = bytes;
        const auto w = store::pack_blob(me, iteration, store::BlobKind::Weights, nullptr, 0);
        ckpt::RestorePieces pieces;
        pieces.unique = nb.framed_at(iteration);
        pieces.weights = &w;
        auto t3 = clk::now();
        const auto bundle = ckpt::assemble_restore(me, iteration, plan, pieces);
        auto t4 = clk::now();
        ok[t] = bundle.optimizer_current.blob.size() == bytes;
        st[3 * t + 0] = std::chrono::duration<double>(t1 - t0).count();
        st[3 * t + 1] = std::chrono::duration<double>(t2 - t1).count();
        st[3 * t + 2] = std::chrono::duration<double>(t4 - t3).count();
      } catch (...) {
        ok[t] = 0;
      }
    });
  for (auto& th : pool) th.join();
  secs[3] = std::chrono::duration<double>(clk::now() - w0).count();
  for (int k = 0; k < 3; ++k) {
    secs[k] = 0;
    for (int t = 0; t < threads; ++t) secs[k] = st[3 * t + k] > secs[k] ? st[3 * t + k] : secs[k];
  }
  secs[4] = 0;
  for (int t = 0; t < threads; ++t) {
    const double snap = st[3 * t + 0] + st[3 * t + 1];
    secs[4] = snap > secs[4] ? snap : secs[4];
  }
  for (int t = 0; t < threads; ++t)
    if (!ok[t]) return -1;
  return 0;
}


// ---- ckpt::HostSnapshots / ckpt::NeighborBuffer (ckpt.cpp:35-105) ----------
// Handles onto the reference's two-version containers, for the differential
// fuzz of the B200 replica semantics (tests/test_gpu_replica_fuzz.py).
// Return codes: 0 ok, 1 ConfigError, 2 CorruptSnapshot, 3 not held, -1 other.

void* ref_hs_create(std::uint16_t dp, std::uint16_t pp, std::uint16_t tp, std::uint64_t capacity) {
  return new ckpt::HostSnapshots(Role{dp, pp, tp}, capacity);
}
void ref_hs_free(void* h) { delete static_cast<ckpt::HostSnapshots*>(h); }
int ref_hs_take(void* h, std::uint64_t it, const void* p, std::uint64_t n) {
  try {
    static_cast<ckpt::HostSnapshots*>(h)->take(it, p, n);
    return 0;
  } catch (const ckpt::ConfigError&) {
    return 1;
  } catch (...) {
    return -1;
  }
}
// newest / previous: 1 and *it set, or 0 when absent
int ref_hs_newest(void* h, std::uint64_t* it) {
  const auto v = static_cast<ckpt::HostSnapshots*>(h)->newest();
  if (v) *it = *v;
  return v ? 1 : 0;
}
int ref_hs_previous(void* h, std::uint64_t* it) {
  const auto v = static_cast<ckpt::HostSnapshots*>(h)->previous();
  if (v) *it = *v;
  return v ? 1 : 0;
}
// framed(it): its length (0 when not held); copies up to cap bytes
std::uint64_t ref_hs_framed(void* h, std::uint64_t it, std::uint8_t* out, std::uint64_t cap) {
  const auto* f = static_cast<ckpt::HostSnapshots*>(h)->framed(it);
  if (!f) return 0;
  std::memcpy(out, f->data(), f->size() < cap ? f->size() : cap);
  return f->size();
}

void* ref_nb_create(std::uint16_t dp, std::uint16_t pp, std::uint16_t tp) {
  return new ckpt::NeighborBuffer(Role{dp, pp, tp});
}
void ref_nb_free(void* h) { delete static_cast<ckpt::NeighborBuffer*>(h); }
int ref_nb_store(void* h, const std::uint8_t* frame, std::uint64_t n) {
  try {
    static_cast<ckpt::NeighborBuffer*>(h)->store(std::vector<std::uint8_t>(frame, frame + n));
    return 0;
  } catch (const store::CorruptSnapshot&) {
    return 2;
  } catch (...) {
    return -1;
  }
}
int ref_nb_newest(void* h, std::uint64_t* it) {
  const auto v = static_cast<ckpt::NeighborBuffer*>(h)->newest();
  if (v) *it = *v;
  return v ? 1 : 0;
}
std::uint64_t ref_nb_framed_at(void* h, std::uint64_t it, std::uint8_t* out, std::uint64_t cap) {
  const auto* f = static_cast<ckpt::NeighborBuffer*>(h)->framed_at(it);
  if (!f) return 0;
  std::memcpy(out, f->data(), f->size() < cap ? f->size() : cap);
  return f->size();
}

// ---- the controller's state machines (controller.cpp:16-121, :144-209) -----
// Thin handles onto ctl::HeartbeatTable / ctl::IterationLedger / plan_recovery
// for the parity tests of libffx's ffx_heartbeats / ffx_ledger / plan.

void* ref_hb_create(std::uint32_t pods, std::int64_t interval_ns, std::uint32_t miss) {
  ctl::ControllerConfig cfg;
  cfg.heartbeat_interval = interval_ns;
  cfg.miss_threshold = miss;
  return new ctl::HeartbeatTable(pods, cfg);
}
void ref_hb_free(void* h) { delete static_cast<ctl::HeartbeatTable*>(h); }
int ref_hb_enroll(void* h, std::uint32_t node, std::uint64_t it, std::int64_t now) {
  try {
    static_cast<ctl::HeartbeatTable*>(h)->enroll(node, it, now);
    return 0;
  } catch (const std::out_of_range&) {
    return -1;
  }
}
void ref_hb_observe(void* h, std::uint32_t node, std::uint64_t it, std::int64_t now) {
  static_cast<ctl::HeartbeatTable*>(h)->observe(node, it, now);
}
std::uint32_t ref_hb_sweep(void* h, std::int64_t now, std::uint32_t* dead, std::uint32_t cap) {
  const auto v = static_cast<ctl::HeartbeatTable*>(h)->sweep(now);
  for (std::uint32_t i = 0; i < v.size() && i < cap; ++i) dead[i] = v[i];
  return static_cast<std::uint32_t>(v.size());
}
int ref_hb_mark_failed(void* h, std::uint32_t node) {
  try {
    static_cast<ctl::HeartbeatTable*>(h)->mark_failed(node);
    return 0;
  } catch (const std::out_of_range&) {
    return -1;
  }
}
// out = {enrolled, failed, last_seen, last_iteration}; -1 where the last_*
// accessors throw (enrolled/failed are still written).
int ref_hb_query(void* h, std::uint32_t node, std::int64_t* out) {
  auto* t = static_cast<ctl::HeartbeatTable*>(h);
  out[0] = t->enrolled(node);
  out[1] = t->failed(node);
  try {
    out[2] = t->last_seen(node);
    out[3] = static_cast<std::int64_t>(t->last_iteration(node));
    return 0;
  } catch (const std::out_of_range&) {
    return -1;
  }
}
void ref_hb_counters(void* h, std::uint64_t* out) {
  auto* t = static_cast<ctl::HeartbeatTable*>(h);
  out[0] = t->unknown_reports();
  out[1] = t->late_reports();
  out[2] = t->regressions();
}

static ClusterSpec ref_spec(std::uint32_t nodes, std::uint32_t gpn, std::uint32_t d, std::uint32_t p,
                            std::uint32_t t, int distributed, std::uint64_t phi) {
  ClusterSpec s;
  s.num_nodes = nodes;
  s.gpus_per_node = gpn;
  s.data_parallel = d;
  s.pipeline_parallel = p;
  s.tensor_parallel = t;
  s.distributed_optimizer = distributed != 0;
  s.params_per_device = phi;
  return s;
}

void* ref_ledger_create(std::uint32_t nodes, std::uint32_t gpn, std::uint32_t d, std::uint32_t p, std::uint32_t t) {
  return new ctl::IterationLedger(ref_spec(nodes, gpn, d, p, t, 1, 1));
}
void ref_ledger_free(void* g) { delete static_cast<ctl::IterationLedger*>(g); }
int ref_ledger_record(void* g, std::uint16_t dp, std::uint16_t pp, std::uint16_t tp, std::uint64_t it) {
  try {
    static_cast<ctl::IterationLedger*>(g)->record(Role{dp, pp, tp}, it);
    return 0;
  } catch (const net::ProtocolError&) {
    return -1;
  }
}
std::uint64_t ref_ledger_global(void* g) { return static_cast<ctl::IterationLedger*>(g)->global_consistent(); }
std::uint64_t ref_ledger_group(void* g, std::uint32_t group) {
  return static_cast<ctl::IterationLedger*>(g)->group_latest(group);
}
std::uint64_t ref_ledger_worker(void* g, std::uint16_t dp, std::uint16_t pp, std::uint16_t tp) {
  return static_cast<ctl::IterationLedger*>(g)->worker_latest(Role{dp, pp, tp});
}
void ref_ledger_rebase(void* g, std::uint64_t it) { static_cast<ctl::IterationLedger*>(g)->rebase(it); }

// plan_recovery (controller.cpp:144-209) flattened into `out` (int64 words):
// kind, resume, then each list as a count followed by its entries -- pods;
// roles (dp,pp,tp); lazy (dp,pp,tp); forwards (dp,pp,tp,holder,dest);
// redundant (target dp,pp,tp, source dp,pp,tp).  Returns the words written,
// or -1 when the plan does not fit / the call throws.
long ref_plan_recovery(std::uint32_t nodes, std::uint32_t gpn, std::uint32_t d, std::uint32_t p, std::uint32_t t,
                       int distributed, std::uint64_t phi, const std::uint32_t* pods, std::uint32_t npods,
                       const std::uint16_t* roles, std::uint32_t nroles, std::uint64_t global_consistent,
                       std::uint64_t latest_fallback, std::int64_t* out, long cap) {
  try {
    std::vector<std::uint32_t> fp(pods, pods + npods);
    std::vector<Role> fr;
    for (std::uint32_t i = 0; i < nroles; ++i) fr.push_back(Role{roles[3 * i], roles[3 * i + 1], roles[3 * i + 2]});
    const auto plan = ctl::plan_recovery(ref_spec(nodes, gpn, d, p, t, distributed, phi), fp, fr,
                                         global_consistent, latest_fallback);
    std::vector<std::int64_t> w;
    w.push_back(plan.kind == ctl::RestoreKind::Fallback ? 1 : 0);
    w.push_back(static_cast<std::int64_t>(plan.resume_iteration));
    auto role = [&](const Role& r) {
      w.push_back(r.dp);
      w.push_back(r.pp);
      w.push_back(r.tp);
    };
    w.push_back(static_cast<std::int64_t>(plan.failed_pods.size()));
    for (auto x : plan.failed_pods) w.push_back(x);
    w.push_back(static_cast<std::int64_t>(plan.failed_roles.size()));
    for (auto& r : plan.failed_roles) role(r);
    w.push_back(static_cast<std::int64_t>(plan.lazy_backup_targets.size()));
    for (auto& r : plan.lazy_backup_targets) role(r);
    w.push_back(static_cast<std::int64_t>(plan.forwards.size()));
    for (auto& f : plan.forwards) {
      role(f.origin);
      w.push_back(f.holder_node);
      w.push_back(f.dest_node);
    }
    w.push_back(static_cast<std::int64_t>(plan.redundant_from.size()));
    for (auto& r : plan.redundant_from) {
      role(r.target);
      role(r.source);
    }
    if (static_cast<long>(w.size()) > cap) return -1;
    std::memcpy(out, w.data(), w.size() * sizeof(std::int64_t));
    return static_cast<long>(w.size());
  } catch (const std::exception&) {
    return -1;
  }
}

// ---- the data loader (dataloader.cpp:104-164) --------------------------------
void ref_fetch(std::uint64_t seed, std::uint64_t first, std::uint32_t count, std::uint32_t bps, std::uint8_t* out) {
  const data::DataServerStub server(seed);
  const auto v = server.fetch(data::IndexWindow{first, count}, bps);
  if (!v.empty()) std::memcpy(out, v.data(), v.size());
}

int ref_fold_of_blob(const std::uint8_t* p, std::uint64_t n, std::uint32_t bps, std::uint64_t* out) {
  try {
    *out = data::fold_of_blob(std::vector<std::uint8_t>(p, p + n), bps);
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}
}  // extern "C"
