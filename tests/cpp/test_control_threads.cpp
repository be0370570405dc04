// test_control_threads.cpp -- the controller state under concurrent host
// threads, built with -fsanitize=thread together with
// paper_2512_03644_b200/csrc/ffx_control.cpp (tests/test_control.py).
//
// The reference's HeartbeatTable / IterationLedger are single-threaded (one
// SimLoop, runtime.hpp:5-10); ffx's are documented thread-safe per object so
// heartbeat receivers, holders' CkptRecords and the recovery driver can run
// on different threads.  This drives all of them at once; TSan fails the run
// on any data race, and the final state is checked against what the threads
// wrote.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <chrono>
#include <thread>
#include <vector>

#include "ffx.h"

// The error reporter and the replica accessors live in the CUDA part of
// libffx; this host-only build stubs them (record_replica is covered on the
// GPU by tests/test_gpu_replica.py).
namespace ffx::host {
int fail(int status, const char*, ...) { return status; }
}  // namespace ffx::host
extern "C" int ffx_replica_slots(const ffx_replica*, uint32_t*) { return FFX_EINVAL; }
extern "C" int ffx_replica_slot_info(ffx_replica*, uint32_t, ffx_slot_info*) { return FFX_EINVAL; }

#define REQUIRE(c)                                                     \
  do {                                                                 \
    if (!(c)) {                                                        \
      std::fprintf(stderr, "%s:%d: REQUIRE(%s)\n", __FILE__, __LINE__, #c); \
      return 1;                                                        \
    }                                                                  \
  } while (0)

int main() {
  // ---- heartbeats: 4 reporters, a sweeper, an enroller -------------------
  const uint32_t pods = 256;
  ffx_heartbeats* hb = nullptr;
  REQUIRE(ffx_heartbeats_create(pods, 10, 3, &hb) == FFX_OK);
  for (uint32_t n = 0; n < pods; ++n) REQUIRE(ffx_heartbeats_enroll(hb, n, 0, 0) == FFX_OK);
  std::atomic<int64_t> clock{0};
  std::atomic<bool> stop{false};
  std::atomic<uint64_t> declared{0};
  std::vector<std::thread> th;
  for (int r = 0; r < 4; ++r)
    th.emplace_back([&, r] {
      for (uint64_t it = 1; it <= 120; ++it)
        for (uint32_t n = r; n < pods; n += 4)
          if (n % 97 != 5 || it < 10) ffx_heartbeats_observe(hb, n, it, clock.fetch_add(1) / 256);
    });
  th.emplace_back([&] {
    uint32_t dead[pods], nd = 0;
    // Bounded and paced: an unthrottled sweeper holds the table's mutex
    // back to back and starves the reporters under TSan's slow locks.
    for (int k = 0; k < 4000 && !stop.load(); ++k) {
      ffx_heartbeats_sweep(hb, clock.load() / 256, dead, pods, &nd);
      declared += nd;
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  });
  th.emplace_back([&] {
    ffx_heartbeat_slot s{};
    for (int k = 0; k < 5000; ++k) ffx_heartbeats_query(hb, k % pods, &s);
  });
  for (int i = 0; i < 4; ++i) th[i].join();
  stop = true;
  for (size_t i = 4; i < th.size(); ++i) th[i].join();
  th.clear();
  uint32_t dead[pods], nd = 0;
  REQUIRE(ffx_heartbeats_sweep(hb, clock.load() / 256 + 1000, dead, pods, &nd) == FFX_OK);
  declared += nd;
  REQUIRE(declared.load() == pods);  // every pod declared exactly once in the end
  uint64_t unknown = 0, late = 0, regressed = 0;
  REQUIRE(ffx_heartbeats_counters(hb, &unknown, &late, &regressed) == FFX_OK);
  REQUIRE(unknown == 0 && regressed == 0);
  ffx_heartbeats_destroy(hb);

  // ---- ledger: 8 recorders (monotone per worker), 2 readers ---------------
  ffx_cluster_spec spec{};
  spec.num_nodes = 8;
  spec.gpus_per_node = 8;
  spec.data_parallel = 16;
  spec.pipeline_parallel = 2;
  spec.tensor_parallel = 2;
  ffx_ledger* led = nullptr;
  REQUIRE(ffx_ledger_create(&spec, &led) == FFX_OK);
  std::atomic<bool> regress{false};
  for (int r = 0; r < 8; ++r)
    th.emplace_back([&, r] {
      for (uint64_t it = 1; it <= 300; ++it)
        for (uint16_t dp = static_cast<uint16_t>(2 * r); dp < 2 * r + 2; ++dp)
          for (uint16_t pp = 0; pp < 2; ++pp)
            for (uint16_t tp = 0; tp < 2; ++tp) ffx_ledger_record(led, ffx_role{dp, pp, tp}, it + r);
    });
  for (int r = 0; r < 2; ++r)
    th.emplace_back([&] {
      uint64_t last = 0;
      for (int k = 0; k < 5000; ++k) {
        const uint64_t g = ffx_ledger_global_consistent(led);
        if (g < last) regress = true;  // records only grow: so must the minimum
        last = g;
        ffx_ledger_group_latest(led, k % 4);
      }
    });
  for (auto& t : th) t.join();
  REQUIRE(!regress.load());
  REQUIRE(ffx_ledger_global_consistent(led) == 300);  // worker group r ends at 300 + r
  REQUIRE(ffx_ledger_worker_latest(led, ffx_role{15, 1, 1}) == 307);
  ffx_ledger_destroy(led);
  std::printf("control threads ok\n");
  return 0;
}
