/*
 * sanitize_paths.c -- every libffx kernel on a small ragged payload, for
 * compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
 *   slice_kernel<Copy, commit>    fused snapshot (TMA + register path)
 *   slice_kernel<Copy>            batched snapshot (2 gated batches)
 *   slice_kernel<Hash> + copy_kernel + commit_kernel   split policy
 *   slice_kernel<HashVerify>      verify-on-store
 *   slice_kernel<CopyVerify>      recovery (+ a corrupted-byte failure)
 *   fnv_* kernels                 whole-payload FNV (SNP1 export)
 *   expand / check / fill / xor   synthetic state, poisoning, fault injection
 * Exit 0 when every result is as expected; the sanitizer's own report is the
 * evidence (profiles/r2_sanitizer_*.log, tools/run_sanitizers.sh).
 *
 *   gcc -std=c99 -O2 -Iinclude tools/sanitize_paths.c -Lpaper_2512_03644_b200 -lffx \
 *       -Wl,-rpath,$PWD/paper_2512_03644_b200 -o tools/sanitize_paths
 */
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "ffx.h"

#define CHECK(call)                                                                          \
  do {                                                                                       \
    int st_ = (call);                                                                        \
    if (st_ != FFX_OK) {                                                                     \
      fprintf(stderr, "%s failed: %s: %s\n", #call, ffx_status_str(st_), ffx_last_error()); \
      return 1;                                                                              \
    }                                                                                        \
  } while (0)
#define EXPECT(c)                                              \
  do {                                                         \
    if (!(c)) {                                                \
      fprintf(stderr, "%s:%d: FAILED %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                \
    }                                                          \
  } while (0)

int main(void) {
  /* two regions, one ragged and one 16-byte word, ~3 MB: every warp task
   * kind (full TMA tasks, ragged register-path tails, a tiny region) */
  const uint64_t n0 = (3ull << 20) + 4099, n1 = 16;
  ffx_cluster_spec spec = {1, 2, 2, 1, 1, 1, 1000000};
  ffx_role d0 = {0, 0, 0}, d1 = {1, 0, 0};
  ffx_ctx *holder = NULL, *me = NULL;
  CHECK(ffx_open(0, &spec, d0, 4096, &holder));
  CHECK(ffx_open(0, &spec, d1, 4096, &me));
  void *a = NULL, *b = NULL, *sums = NULL;
  CHECK(ffx_device_alloc(0, n0, &a));
  CHECK(ffx_device_alloc(0, n1, &b));
  uint8_t digest[32] = {7};
  CHECK(ffx_materialize(a, digest, n0, NULL));
  uint8_t word[16] = {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 16};
  CHECK(ffx_memcpy(b, word, n1, NULL, 1));
  CHECK(ffx_register_region(me, FFX_REGION_MASTER, a, n0, 1));
  CHECK(ffx_register_region(me, FFX_REGION_CURSOR, b, n1, 1));
  ffx_replica *held = NULL, *view = NULL;
  CHECK(ffx_replica_create(holder, d1, n0 + n1, 2, &held));
  uint8_t h[FFX_HANDLE_BYTES];
  CHECK(ffx_replica_export(held, h));
  CHECK(ffx_replica_open(me, h, &view));
  CHECK(ffx_snapshot_target(me, view));

  /* fused, whole GPU */
  CHECK(ffx_snapshot(me, 1, NULL, NULL));
  /* two batches */
  ffx_snapshot_opts o;
  memset(&o, 0, sizeof o);
  o.batches = 2;
  o.max_ctas = 8;
  CHECK(ffx_snapshot(me, 2, NULL, &o));
  /* split: TMA copy batches + hash batches, and with verify-on-store */
  memset(&o, 0, sizeof o);
  o.split = 1;
  o.batches = 2;
  o.hash_batches = 2;
  o.verify_on_store = 1;
  CHECK(ffx_snapshot(me, 3, NULL, &o));
  CHECK(ffx_stream_sync(NULL));

  /* whole-payload FNV (SNP1 export) */
  uint64_t len = 0;
  static uint8_t frame[(3u << 20) + 8192];
  CHECK(ffx_replica_export_frame(held, 3, frame, sizeof frame, &len, NULL));
  EXPECT(len == 32 + n0 + n1);
  uint64_t whole = 0;
  CHECK(ffx_checksum64(a, n0, &whole, NULL));

  /* per-slice checksums and a fused copy + checksums */
  const uint64_t ns = (n0 + 4095) / 4096;
  CHECK(ffx_device_alloc(0, ns * 8, &sums));
  CHECK(ffx_slice_checksums(a, n0, 4096, (uint64_t*)sums, NULL));
  CHECK(ffx_stream_sync(NULL));

  /* failure + recovery, then a corrupted replica byte must be caught */
  CHECK(ffx_inject(me, FFX_FAULT_POISON_STATE, NULL, 0));
  ffx_recover_report rep;
  CHECK(ffx_recover(me, view, 3, NULL, &rep));
  EXPECT(rep.bad_slices == 0);
  uint64_t bad = 0;
  CHECK(ffx_blob_check(a, n0, &bad, NULL));
  EXPECT(bad == UINT64_MAX);
  uint32_t slot = 0;
  for (uint32_t v = 0; v < 2; ++v) {
    ffx_slot_info si;
    CHECK(ffx_replica_slot_info(held, v, &si));
    if (si.state == 2 && si.iteration == 3) slot = v;
  }
  CHECK(ffx_inject(me, FFX_FAULT_CORRUPT_REPLICA, view, ((uint64_t)slot << 48) | 123457));
  EXPECT(ffx_recover(me, view, 3, NULL, &rep) == FFX_ERESTORE);
  EXPECT(rep.first_bad_slice == 123457 / 4096);

  CHECK(ffx_replica_destroy(view));
  CHECK(ffx_replica_destroy(held));
  CHECK(ffx_device_free(0, a));
  CHECK(ffx_device_free(0, b));
  CHECK(ffx_device_free(0, sums));
  CHECK(ffx_close(me));
  CHECK(ffx_close(holder));
  printf("sanitize paths ok\n");
  return 0;
}
