// ftsim/controller.hpp -- B200 facade: the controller STATE the recovery path
// reads (heartbeat table, iteration ledger, recovery plan).
//
// Drop-in for that subset of the reference's proj/include/ftsim/controller.hpp
// (:31-34, :56-130, :136-179), implemented over libffx's ffx_heartbeats_*,
// ffx_ledger_* and ffx_plan_recovery (include/ffx.h).  The Controller actor
// (:183-) and the wire / transport stack it drives are not part of the
// B200 path; a host keeps its own and calls these.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "ftsim/domain.hpp"

namespace ftsim {

namespace rt {  // runtime.hpp:36-37 (the time type only)
using Nanos = std::int64_t;
constexpr Nanos kSecond = 1'000'000'000;
}  // namespace rt

namespace net {  // transport.hpp: the error the ledger raises
struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
}  // namespace net

namespace ctl {

struct ControllerConfig {
  rt::Nanos heartbeat_interval = rt::kSecond;
  std::uint32_t miss_threshold = 3;
};

// controller.hpp:56-101 over ffx_heartbeats_*.
class HeartbeatTable {
 public:
  HeartbeatTable(std::uint32_t pods, const ControllerConfig& cfg);
  ~HeartbeatTable();
  HeartbeatTable(HeartbeatTable&& o) noexcept : h_(o.h_), pods_(o.pods_) { o.h_ = nullptr; }
  HeartbeatTable& operator=(HeartbeatTable&&) = delete;
  HeartbeatTable(const HeartbeatTable&) = delete;
  HeartbeatTable& operator=(const HeartbeatTable&) = delete;

  void enroll(std::uint32_t node, std::uint64_t iteration, rt::Nanos now);
  void observe(std::uint32_t node, std::uint64_t iteration, rt::Nanos now);
  std::vector<std::uint32_t> sweep(rt::Nanos now);
  void mark_failed(std::uint32_t node);

  bool enrolled(std::uint32_t node) const;
  bool failed(std::uint32_t node) const;
  std::uint64_t last_iteration(std::uint32_t node) const;
  rt::Nanos last_seen(std::uint32_t node) const;

  std::uint64_t unknown_reports() const;
  std::uint64_t late_reports() const;
  std::uint64_t regressions() const;

 private:
  void* h_ = nullptr;  // ffx_heartbeats*
  std::uint32_t pods_ = 0;
};

// controller.hpp:106-130 over ffx_ledger_*.
class IterationLedger {
 public:
  explicit IterationLedger(const ClusterSpec& spec);
  ~IterationLedger();
  IterationLedger(IterationLedger&& o) noexcept : g_(o.g_) { o.g_ = nullptr; }
  IterationLedger& operator=(IterationLedger&&) = delete;
  IterationLedger(const IterationLedger&) = delete;
  IterationLedger& operator=(const IterationLedger&) = delete;

  void record(const Role& role, std::uint64_t iteration);
  std::uint64_t global_consistent() const;
  std::uint64_t group_latest(std::uint32_t dp_group) const;
  std::uint64_t worker_latest(const Role& role) const;
  void rebase(std::uint64_t iteration);

 private:
  void* g_ = nullptr;  // ffx_ledger*
};

enum class RestoreKind : std::uint8_t { Neighbor, Fallback };

struct ForwardInstruction {
  Role origin;
  std::uint32_t holder_node = 0;
  std::uint32_t dest_node = 0;
};

struct RedundantSource {
  Role target;
  Role source;
};

struct RecoveryPlan {
  RestoreKind kind = RestoreKind::Neighbor;
  std::uint64_t notice_id = 0;
  std::uint64_t new_epoch = 0;
  std::uint64_t resume_iteration = 0;
  std::vector<std::uint32_t> failed_pods;
  std::vector<Role> failed_roles;
  std::vector<Role> lazy_backup_targets;
  std::vector<ForwardInstruction> forwards;
  std::vector<RedundantSource> redundant_from;
};

// controller.hpp:175-179 over ffx_plan_recovery (replicas = 1, the
// reference rule).
RecoveryPlan plan_recovery(const ClusterSpec& spec, const std::vector<std::uint32_t>& failed_pods,
                           const std::vector<Role>& failed_roles, std::uint64_t global_consistent,
                           std::uint64_t latest_fallback_round);

}  // namespace ctl
}  // namespace ftsim
