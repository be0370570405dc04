/*
 * c_snapshot.c -- the C ABI from plain C (no C++, no Python, no torch):
 * the whole backup / failure / recovery path of one rank through
 * include/ffx.h, the way a Go (cgo), Java (JNI) or Rust host would drive it.
 *
 *   gcc -std=c99 -O2 -Iinclude examples/c_snapshot.c -Lpaper_2512_03644_b200 -lffx \
 *       -Wl,-rpath,$PWD/paper_2512_03644_b200 -o examples/c_snapshot && examples/c_snapshot
 *
 * One GPU, two contexts: rank d1 snapshots into the replica rank d0 holds
 * for it (ckpt.cpp:77-105), three iterations with an evolving state; each
 * committed replica is recorded in the iteration ledger (the CkptRecord,
 * wire.hpp:85-90) while both pods heartbeat.  Then d1's pod goes silent: the
 * heartbeat sweep declares it (controller.cpp:46-58), plan_recovery names the
 * holder (controller.cpp:144-209), and d1 restores the ledger's consistent
 * iteration from d0's replica (assemble_restore, ckpt.cpp:140-167), verified
 * on the device.
 */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "ffx.h"

#define CHECK(call)                                                              \
  do {                                                                           \
    int st_ = (call);                                                            \
    if (st_ != FFX_OK) {                                                         \
      fprintf(stderr, "%s failed: %s: %s\n", #call, ffx_status_str(st_), ffx_last_error()); \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

int main(void) {
  const uint64_t n = (64ull << 20) + 12345; /* a ragged 64 MiB state */
  ffx_cluster_spec spec = {2, 1, 2, 1, 1, 1, 1000000}; /* 2 pods x 1 GPU, d=2 */
  ffx_role d0 = {0, 0, 0}, d1 = {1, 0, 0};
  ffx_ctx *holder = NULL, *me = NULL;
  CHECK(ffx_open(0, &spec, d0, 4096, &holder));
  CHECK(ffx_open(0, &spec, d1, 4096, &me));

  void* state = NULL;
  CHECK(ffx_device_alloc(0, n, &state));
  CHECK(ffx_register_region(me, FFX_REGION_BLOB, state, n, 1));

  ffx_replica* held = NULL; /* d0 holds d1's replica: two versions */
  CHECK(ffx_replica_create(holder, d1, n, 2, &held));
  uint8_t handle[FFX_HANDLE_BYTES];
  CHECK(ffx_replica_export(held, handle)); /* would travel to d1's process */
  ffx_replica* target = NULL;
  CHECK(ffx_replica_open(me, handle, &target));
  CHECK(ffx_snapshot_target(me, target));

  /* the controller state: 1 s heartbeat interval, 3 misses */
  const int64_t sec = 1000000000;
  ffx_heartbeats* hb = NULL;
  ffx_ledger* led = NULL;
  CHECK(ffx_heartbeats_create(2, sec, 3, &hb));
  CHECK(ffx_ledger_create(&spec, &led));
  CHECK(ffx_heartbeats_enroll(hb, 0, 0, 0));
  CHECK(ffx_heartbeats_enroll(hb, 1, 0, 0));

  uint8_t digest[32];
  for (uint64_t it = 1; it <= 3; ++it) {
    memset(digest, 0, sizeof digest);
    digest[0] = (uint8_t)it; /* a new optimizer state every iteration */
    CHECK(ffx_materialize(state, digest, n, NULL));
    CHECK(ffx_snapshot(me, it, NULL, NULL));
    CHECK(ffx_stream_sync(NULL));
    uint64_t rec = 0;
    CHECK(ffx_ledger_record_replica(led, held, &rec)); /* holder: d1 is safe at `it` */
    CHECK(ffx_ledger_record(led, d0, it));             /* d0's own record (its holder is d1) */
    CHECK(ffx_heartbeats_observe(hb, 0, it, (int64_t)it * sec));
    CHECK(ffx_heartbeats_observe(hb, 1, it, (int64_t)it * sec));
  }
  uint64_t newest = ffx_ledger_global_consistent(led);

  /* d1's pod goes silent after iteration 3; d0 keeps reporting */
  uint32_t dead[2], ndead = 0;
  for (int64_t t = 4; t <= 8 && ndead == 0; ++t) {
    CHECK(ffx_heartbeats_observe(hb, 0, 3, t * sec));
    CHECK(ffx_heartbeats_sweep(hb, t * sec, dead, 2, &ndead));
  }
  ffx_role lost[2], lazy[2];
  uint32_t pods[2];
  ffx_forward fwd[2];
  ffx_redundant_source red[2];
  ffx_recovery_plan plan = {0};
  plan.capacity = 2;
  plan.failed_pods = pods;
  plan.failed_roles = lost;
  plan.lazy_backup_targets = lazy;
  plan.forwards = fwd;
  plan.redundant_from = red;
  CHECK(ffx_plan_recovery(&spec, dead, ndead, NULL, 0, newest, 0, 1, &plan));
  if (ndead != 1 || dead[0] != 1 || plan.kind != FFX_PLAN_NEIGHBOR || plan.n_forwards != 1 ||
      plan.forwards[0].holder_node != 0) {
    fprintf(stderr, "detection / plan mismatch (ndead %u)\n", ndead);
    return 1;
  }

  /* the failure: every byte of the state is gone */
  CHECK(ffx_inject(me, FFX_FAULT_POISON_STATE, NULL, 0));
  uint64_t bad = 0;
  CHECK(ffx_blob_check(state, n, &bad, NULL));
  if (bad == UINT64_MAX) {
    fprintf(stderr, "poisoning did not take\n");
    return 1;
  }

  /* recovery: pull + verify every slice against the checksum table */
  ffx_recover_report rep;
  CHECK(ffx_recover(me, target, newest, NULL, &rep));
  CHECK(ffx_blob_check(state, n, &bad, NULL));
  uint8_t head[32];
  CHECK(ffx_memcpy(head, state, 32, NULL, 1));
  const int ok = rep.bad_slices == 0 && bad == UINT64_MAX && head[0] == 3 && newest == 3;
  printf("{\"newest\": %llu, \"restored_bytes\": %llu, \"bad_slices\": %llu, \"seconds\": %.6f, \"ok\": %s}\n",
         (unsigned long long)newest, (unsigned long long)rep.bytes, (unsigned long long)rep.bad_slices,
         rep.seconds, ok ? "true" : "false");

  CHECK(ffx_ledger_rebase(led, newest)); /* every worker resumes at `newest` */
  CHECK(ffx_ledger_destroy(led));
  CHECK(ffx_heartbeats_destroy(hb));
  CHECK(ffx_replica_destroy(target));
  CHECK(ffx_replica_destroy(held));
  CHECK(ffx_device_free(0, state));
  CHECK(ffx_close(me));
  CHECK(ffx_close(holder));
  return ok ? 0 : 1;
}
