// controller.cpp -- facade: ftsim::ctl's controller state over libffx
// (ffx_heartbeats_*, ffx_ledger_*, ffx_plan_recovery; include/ffx.h).
#include "ftsim/controller.hpp"

#include "device.hpp"

namespace ftsim::ctl {
namespace {

ffx_heartbeats* H(void* p) { return static_cast<ffx_heartbeats*>(p); }
ffx_ledger* G(void* p) { return static_cast<ffx_ledger*>(p); }
ffx_role R(const Role& r) { return ffx_role{r.dp, r.pp, r.tp}; }
Role R(const ffx_role& r) { return Role{r.dp, r.pp, r.tp}; }

ffx_cluster_spec C(const ClusterSpec& s) {
  ffx_cluster_spec c{};
  c.num_nodes = s.num_nodes;
  c.gpus_per_node = s.gpus_per_node;
  c.data_parallel = s.data_parallel;
  c.pipeline_parallel = s.pipeline_parallel;
  c.tensor_parallel = s.tensor_parallel;
  c.distributed_optimizer = s.distributed_optimizer;
  c.params_per_device = s.params_per_device;
  return c;
}

ffx_heartbeat_slot slot(void* h, std::uint32_t node) {
  ffx_heartbeat_slot s{};
  b200::check(ffx_heartbeats_query(H(h), node, &s), "HeartbeatTable");  // out_of_range past the pods
  return s;
}

}  // namespace

HeartbeatTable::HeartbeatTable(std::uint32_t pods, const ControllerConfig& cfg) : pods_(pods) {
  ffx_heartbeats* h = nullptr;
  b200::check(ffx_heartbeats_create(pods, cfg.heartbeat_interval, cfg.miss_threshold, &h), "HeartbeatTable");
  h_ = h;
}

HeartbeatTable::~HeartbeatTable() {
  if (h_) ffx_heartbeats_destroy(H(h_));
}

void HeartbeatTable::enroll(std::uint32_t node, std::uint64_t iteration, rt::Nanos now) {
  b200::check(ffx_heartbeats_enroll(H(h_), node, iteration, now), "HeartbeatTable::enroll");
}

void HeartbeatTable::observe(std::uint32_t node, std::uint64_t iteration, rt::Nanos now) {
  b200::check(ffx_heartbeats_observe(H(h_), node, iteration, now), "HeartbeatTable::observe");
}

std::vector<std::uint32_t> HeartbeatTable::sweep(rt::Nanos now) {
  std::vector<std::uint32_t> dead(pods_);
  std::uint32_t n = 0;
  b200::check(ffx_heartbeats_sweep(H(h_), now, dead.data(), pods_, &n), "HeartbeatTable::sweep");
  dead.resize(n);
  return dead;
}

void HeartbeatTable::mark_failed(std::uint32_t node) {
  b200::check(ffx_heartbeats_mark_failed(H(h_), node), "HeartbeatTable::mark_failed");
}

bool HeartbeatTable::enrolled(std::uint32_t node) const { return node < pods_ && slot(h_, node).enrolled; }
bool HeartbeatTable::failed(std::uint32_t node) const { return node < pods_ && slot(h_, node).failed; }
std::uint64_t HeartbeatTable::last_iteration(std::uint32_t node) const { return slot(h_, node).last_iteration; }
rt::Nanos HeartbeatTable::last_seen(std::uint32_t node) const { return slot(h_, node).last_seen_ns; }

std::uint64_t HeartbeatTable::unknown_reports() const {
  std::uint64_t v = 0;
  ffx_heartbeats_counters(H(h_), &v, nullptr, nullptr);
  return v;
}
std::uint64_t HeartbeatTable::late_reports() const {
  std::uint64_t v = 0;
  ffx_heartbeats_counters(H(h_), nullptr, &v, nullptr);
  return v;
}
std::uint64_t HeartbeatTable::regressions() const {
  std::uint64_t v = 0;
  ffx_heartbeats_counters(H(h_), nullptr, nullptr, &v);
  return v;
}

IterationLedger::IterationLedger(const ClusterSpec& spec) {
  const ffx_cluster_spec c = C(spec);
  ffx_ledger* g = nullptr;
  b200::check(ffx_ledger_create(&c, &g), "IterationLedger");
  g_ = g;
}

IterationLedger::~IterationLedger() {
  if (g_) ffx_ledger_destroy(G(g_));
}

void IterationLedger::record(const Role& role, std::uint64_t iteration) {
  const int st = ffx_ledger_record(G(g_), R(role), iteration);
  if (st == FFX_ERANGE)  // controller.cpp:85-87
    throw net::ProtocolError("checkpoint record for a role outside the grid: " + role.str());
  b200::check(st, "IterationLedger::record");
}

std::uint64_t IterationLedger::global_consistent() const { return ffx_ledger_global_consistent(G(g_)); }
std::uint64_t IterationLedger::group_latest(std::uint32_t g) const { return ffx_ledger_group_latest(G(g_), g); }
std::uint64_t IterationLedger::worker_latest(const Role& r) const { return ffx_ledger_worker_latest(G(g_), R(r)); }
void IterationLedger::rebase(std::uint64_t it) { b200::check(ffx_ledger_rebase(G(g_), it), "IterationLedger::rebase"); }

RecoveryPlan plan_recovery(const ClusterSpec& spec, const std::vector<std::uint32_t>& failed_pods,
                           const std::vector<Role>& failed_roles, std::uint64_t global_consistent,
                           std::uint64_t latest_fallback_round) {
  const ffx_cluster_spec c = C(spec);
  const std::size_t cap = static_cast<std::size_t>(spec.num_nodes) * spec.gpus_per_node + failed_roles.size() +
                          failed_pods.size() * spec.gpus_per_node + 1;
  std::vector<std::uint32_t> pods(cap);
  std::vector<ffx_role> roles(cap), lazy(cap);
  std::vector<ffx_forward> fwd(cap);
  std::vector<ffx_redundant_source> red(cap);
  std::vector<ffx_role> in_roles;
  for (const auto& r : failed_roles) in_roles.push_back(R(r));
  ffx_recovery_plan p{};
  p.capacity = static_cast<std::uint32_t>(cap);
  p.failed_pods = pods.data();
  p.failed_roles = roles.data();
  p.lazy_backup_targets = lazy.data();
  p.forwards = fwd.data();
  p.redundant_from = red.data();
  b200::check(ffx_plan_recovery(&c, failed_pods.data(), static_cast<std::uint32_t>(failed_pods.size()),
                                in_roles.data(), static_cast<std::uint32_t>(in_roles.size()), global_consistent,
                                latest_fallback_round, 1, &p),
              "plan_recovery");
  RecoveryPlan out;
  out.kind = p.kind == FFX_PLAN_FALLBACK ? RestoreKind::Fallback : RestoreKind::Neighbor;
  out.resume_iteration = p.resume_iteration;
  out.failed_pods.assign(pods.begin(), pods.begin() + p.n_failed_pods);
  for (std::uint32_t i = 0; i < p.n_failed_roles; ++i) out.failed_roles.push_back(R(roles[i]));
  for (std::uint32_t i = 0; i < p.n_lazy; ++i) out.lazy_backup_targets.push_back(R(lazy[i]));
  for (std::uint32_t i = 0; i < p.n_forwards; ++i)
    out.forwards.push_back(ForwardInstruction{R(fwd[i].origin), fwd[i].holder_node, fwd[i].dest_node});
  for (std::uint32_t i = 0; i < p.n_redundant; ++i)
    out.redundant_from.push_back(RedundantSource{R(red[i].target), R(red[i].source)});
  return out;
}

}  // namespace ftsim::ctl
