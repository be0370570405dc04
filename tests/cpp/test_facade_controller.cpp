// test_facade_controller.cpp -- the facade's ftsim::ctl controller state
// (HeartbeatTable, IterationLedger, plan_recovery over libffx), checked with
// the expectations of the reference's proj/tests/test_controller.cpp:37-276
// (restated; the Controller-actor cases after :277 are not on the B200 path).
// Host-only: runs without a GPU (tests/test_control.py).
#include <doctest.h>

#include <vector>

#include "ftsim/controller.hpp"

using namespace ftsim;
using namespace ftsim::ctl;

namespace {

ClusterSpec grid(std::uint32_t d, std::uint32_t p, std::uint32_t t, std::uint32_t per_node) {
  ClusterSpec s;
  s.data_parallel = d;
  s.pipeline_parallel = p;
  s.tensor_parallel = t;
  s.gpus_per_node = per_node;
  s.num_nodes = d * p * t / per_node;
  return s;
}

constexpr rt::Nanos sec = rt::kSecond;

}  // namespace

TEST_CASE("liveness slots: refresh, unknown senders, regressions, late reports, revival") {
  HeartbeatTable hb(4, ControllerConfig{});
  hb.enroll(0, 0, 0);
  hb.enroll(1, 0, 0);
  hb.observe(0, 5, 2 * sec);
  CHECK(hb.last_iteration(0) == 5);
  CHECK(hb.last_seen(0) == 2 * sec);
  hb.observe(2, 1, sec);   // never enrolled
  hb.observe(99, 1, sec);  // no slot at all
  CHECK(hb.unknown_reports() == 2);
  CHECK_FALSE(hb.enrolled(99));
  hb.observe(0, 3, 3 * sec);  // went backwards: stored, flagged
  CHECK(hb.regressions() == 1);
  CHECK(hb.last_iteration(0) == 3);
  hb.mark_failed(1);
  hb.observe(1, 9, 5 * sec);
  CHECK(hb.late_reports() == 1);
  CHECK(hb.last_iteration(1) == 0);
  CHECK(hb.failed(1));
  hb.enroll(1, 42, 9 * sec);  // the substitute registers
  CHECK_FALSE(hb.failed(1));
  hb.observe(1, 43, 10 * sec);
  CHECK(hb.last_iteration(1) == 43);
  CHECK_THROWS_AS(hb.last_iteration(7), std::out_of_range);
}

TEST_CASE("a pod is declared after more than threshold silent intervals, once") {
  HeartbeatTable hb(2, ControllerConfig{});
  hb.enroll(0, 0, 0);
  hb.enroll(1, 0, 0);
  hb.observe(0, 10, 10 * sec);
  for (int s = 10; s <= 15; ++s) hb.observe(1, 10 + s, s * sec);
  std::vector<std::vector<std::uint32_t>> seen;
  for (int s = 11; s <= 15; ++s) seen.push_back(hb.sweep(s * sec));
  CHECK(seen[2].empty());  // exactly 3 s: not yet
  CHECK(seen[3] == std::vector<std::uint32_t>{0});
  CHECK(seen[4].empty());
  CHECK(hb.failed(0));
  CHECK_FALSE(hb.failed(1));
}

TEST_CASE("32768 senders, a few silent") {
  const std::uint32_t pods = 32768;
  HeartbeatTable hb(pods, ControllerConfig{});
  for (std::uint32_t n = 0; n < pods; ++n) hb.enroll(n, 0, 0);
  for (int b = 1; b <= 5; ++b) {
    for (std::uint32_t n = 0; n < pods; ++n)
      if (b < 3 || n % 4096 != 7) hb.observe(n, static_cast<std::uint64_t>(b), b * sec);
    CHECK(hb.sweep(b * sec).empty());
  }
  std::vector<std::uint32_t> want;
  for (std::uint32_t n = 7; n < pods; n += 4096) want.push_back(n);
  CHECK(hb.sweep(6 * sec) == want);
}

TEST_CASE("the ledger's consistent iteration is the grid minimum") {
  IterationLedger led(grid(2, 2, 1, 2));
  CHECK(led.global_consistent() == 0);
  led.record(Role{0, 0, 0}, 3);
  led.record(Role{0, 1, 0}, 3);
  led.record(Role{1, 0, 0}, 3);
  CHECK(led.global_consistent() == 0);
  led.record(Role{1, 1, 0}, 2);
  CHECK(led.global_consistent() == 2);
  led.record(Role{1, 1, 0}, 1);  // monotone
  CHECK(led.worker_latest(Role{1, 1, 0}) == 2);
  led.record(Role{1, 1, 0}, 3);
  led.record(Role{0, 0, 0}, 4);
  led.record(Role{1, 0, 0}, 4);
  CHECK(led.group_latest(0) == 4);
  CHECK(led.group_latest(1) == 3);
  CHECK(led.global_consistent() == 3);
  CHECK_THROWS_AS(led.record(Role{5, 0, 0}, 1), net::ProtocolError);
  led.rebase(7);
  led.record(Role{0, 0, 0}, 8);
  CHECK(led.global_consistent() == 7);
  CHECK(led.group_latest(0) == 7);
}

TEST_CASE("neighbour path iff no two lost ring members are adjacent (6-ring)") {
  auto spec = grid(6, 1, 1, 1);
  spec.distributed_optimizer = true;
  for (unsigned mask = 1; mask < 64; ++mask) {
    std::vector<std::uint32_t> pods;
    bool adjacent = false;
    for (unsigned i = 0; i < 6; ++i) {
      if (mask >> i & 1) pods.push_back(i);
      if ((mask >> i & 1) && (mask >> ((i + 1) % 6) & 1)) adjacent = true;
    }
    const auto plan = plan_recovery(spec, pods, {}, 40, 35);
    CHECK((plan.kind == RestoreKind::Fallback) == adjacent);
    CHECK(plan.resume_iteration == (adjacent ? 35u : 40u));
    CHECK(plan.forwards.size() == (adjacent ? 0 : pods.size()));
  }
}

TEST_CASE("plans name holders, redundant sources and lazy-backup targets") {
  auto spec = grid(4, 2, 1, 2);
  spec.distributed_optimizer = true;
  const auto plan = plan_recovery(spec, {1}, {}, 17, 10);
  REQUIRE(plan.kind == RestoreKind::Neighbor);
  CHECK(plan.failed_pods == std::vector<std::uint32_t>{1});
  REQUIRE(plan.failed_roles.size() == 2);
  CHECK(plan.failed_roles[1] == Role{1, 1, 0});
  REQUIRE(plan.forwards.size() == 2);
  for (const auto& f : plan.forwards) CHECK((f.holder_node == 2 && f.dest_node == 1));
  REQUIRE(plan.redundant_from.size() == 2);
  for (const auto& r : plan.redundant_from) CHECK(r.source.dp == 0);
  REQUIRE(plan.lazy_backup_targets.size() == 2);
  spec.distributed_optimizer = false;  // replicated optimizer: nothing forwarded
  const auto p2 = plan_recovery(spec, {1}, {}, 17, 10);
  CHECK(p2.forwards.empty());
  CHECK(p2.redundant_from.size() == 2);
  CHECK(plan_recovery(grid(2, 2, 1, 2), {0, 1}, {}, 17, 10).kind == RestoreKind::Fallback);
  CHECK(plan_recovery(grid(1, 4, 2, 2), {1}, {}, 17, 10).kind == RestoreKind::Fallback);
  spec.distributed_optimizer = true;
  const auto p3 = plan_recovery(spec, {1}, {}, 0, 0);  // before any record
  CHECK(p3.kind == RestoreKind::Neighbor);
  CHECK((p3.forwards.empty() && p3.redundant_from.empty() && p3.lazy_backup_targets.empty()));
  CHECK(p3.failed_roles.size() == 2);
}
