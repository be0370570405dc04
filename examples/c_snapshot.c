/*
 * c_snapshot.c -- the C ABI from plain C (no C++, no Python, no torch):
 * the whole backup / failure / recovery path of one rank through
 * include/ffx.h, the way a Go (cgo), Java (JNI) or Rust host would drive it.
 *
 *   gcc -std=c99 -O2 -Iinclude examples/c_snapshot.c -Lpaper_2512_03644_b200 -lffx \
 *       -Wl,-rpath,$PWD/paper_2512_03644_b200 -o examples/c_snapshot && examples/c_snapshot
 *
 * One GPU, two contexts: rank d1 snapshots into the replica rank d0 holds
 * for it (ckpt.cpp:77-105), three iterations with an evolving state, then
 * d1 loses its state and restores the newest snapshot from d0's replica
 * (assemble_restore, ckpt.cpp:140-167), verified on the device.
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
  ffx_cluster_spec spec = {1, 1, 2, 1, 1, 1, 1000000};
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

  uint8_t digest[32];
  for (uint64_t it = 1; it <= 3; ++it) {
    memset(digest, 0, sizeof digest);
    digest[0] = (uint8_t)it; /* a new optimizer state every iteration */
    CHECK(ffx_materialize(state, digest, n, NULL));
    CHECK(ffx_snapshot(me, it, NULL, NULL));
  }
  CHECK(ffx_stream_sync(NULL));
  uint64_t newest = 0;
  CHECK(ffx_replica_newest(held, &newest));

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

  CHECK(ffx_replica_destroy(target));
  CHECK(ffx_replica_destroy(held));
  CHECK(ffx_device_free(0, state));
  CHECK(ffx_close(me));
  CHECK(ffx_close(holder));
  return ok ? 0 : 1;
}
