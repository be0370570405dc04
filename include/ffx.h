/*
 * ffx.h -- C ABI of the B200-native state-backup / failover-recovery path.
 *
 * This is the drop-in boundary for FFTrainer's per-iteration snapshot ->
 * neighbour replica -> failure -> recover/verify path.  The reference exposes
 * that path as a C++ API (proj/include/ftsim/{ckpt,storage,hash,evolution,
 * domain}.hpp); it has no C ABI of its own.  Every entry point below names the
 * reference interface it replaces (file:line, relative to the reference's
 * proj/ directory).  The C++ facade in paper_2512_03644_b200/facade/ re-exposes
 * the reference's exact class/function names on top of these calls, mapping
 * status codes back to the reference's exception types 1:1.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or CUDA types in signatures.
 *    `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - "dev" pointers are device (or peer-mapped) global memory on the context's
 *    device.  Region and replica pointers must be 16-byte aligned.
 *  - Context calls run on the context's device.  The context-free device
 *    primitives run on the device of `stream` when one is given, else on the
 *    device owning their source pointer (one process may drive several GPUs).
 *  - Every call returns an ffx_status; ffx_last_error() gives the detail
 *    message of the last failure on the calling thread.
 *  - One ffx_ctx per rank (one process per GPU, or one thread per GPU).  Calls
 *    on one context are not internally locked.
 */
#ifndef FFX_H_
#define FFX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFX_ABI_VERSION 2
#define FFX_MAX_REGIONS 16
#define FFX_HANDLE_BYTES 256

typedef enum ffx_status {
  FFX_OK = 0,
  FFX_ECONFIG = 1,  /* ckpt::ConfigError         ckpt.hpp:58-60 */
  FFX_EVERSION = 2, /* ckpt::VersionError        ckpt.hpp:62-64 */
  FFX_ERESTORE = 3, /* ckpt::RestoreError        ckpt.hpp:66-68 */
  FFX_ECORRUPT = 4, /* store::CorruptSnapshot    storage.hpp:55-57 */
  FFX_EINVAL = 5,   /* std::invalid_argument     storage.cpp:49, evolution.cpp:90 */
  FFX_ERANGE = 6,   /* std::out_of_range         domain.cpp:22, :36 */
  FFX_ECUDA = 7,    /* CUDA runtime / driver failure */
  FFX_ENOMEM = 8,   /* device allocation failed */
  FFX_ESTATE = 9    /* call out of order (e.g. snapshot with no target) */
} ffx_status;

const char* ffx_status_str(int status);
const char* ffx_last_error(void);
int ffx_abi_version(void);

/* ---- domain (domain.hpp:15-110) ------------------------------------------ */

typedef struct ffx_role {
  uint16_t dp, pp, tp;
} ffx_role;

/* The sizing subset of ftsim::ClusterSpec (domain.hpp:49-73). */
typedef struct ffx_cluster_spec {
  uint32_t num_nodes;
  uint32_t gpus_per_node;
  uint32_t data_parallel;
  uint32_t pipeline_parallel;
  uint32_t tensor_parallel;
  uint32_t distributed_optimizer; /* bool */
  uint64_t params_per_device;
} ffx_cluster_spec;

/* ckpt::UniquenessPlan (ckpt.hpp:38-42) */
typedef struct ffx_uniqueness_plan {
  uint32_t weights_redundant;
  uint32_t optimizer_redundant;
  uint64_t unique_bytes_per_device;
} ffx_uniqueness_plan;

int ffx_role_of(const ffx_cluster_spec* spec, uint32_t global_index, ffx_role* out); /* domain.cpp:18-30 */
int ffx_index_of(const ffx_cluster_spec* spec, ffx_role role, uint32_t* out);        /* domain.cpp:32-40 */
int ffx_node_of(const ffx_cluster_spec* spec, ffx_role role, uint32_t* out);         /* domain.cpp:47-49 */
int ffx_dp_neighbor(const ffx_cluster_spec* spec, ffx_role role, ffx_role* out);     /* domain.cpp:51-55 */
int ffx_dp_predecessor(const ffx_cluster_spec* spec, ffx_role role, ffx_role* out);  /* domain.cpp:57-62 */

/* ---- recovery planning (ctl::plan_recovery, controller.cpp:144-209) ------ */

typedef struct ffx_forward { /* ForwardInstruction, controller.hpp:143-147 */
  ffx_role origin;
  uint16_t pad_;
  uint32_t holder_node;
  uint32_t dest_node;
  uint32_t holder_dp; /* which replica holder serves it (dp+1 .. dp+replicas) */
} ffx_forward;

typedef struct ffx_redundant_source { /* RedundantSource, controller.hpp:151-154 */
  ffx_role target;
  ffx_role source;
} ffx_redundant_source;

/* RecoveryPlan (controller.hpp:156-169).  The caller provides the arrays,
 * each with room for `capacity` entries (world size suffices). */
enum ffx_plan_kind { FFX_PLAN_NEIGHBOR = 0, FFX_PLAN_FALLBACK = 1 }; /* ctl::RestoreKind */

typedef struct ffx_recovery_plan {
  uint32_t kind; /* ffx_plan_kind */
  uint32_t capacity;
  uint64_t resume_iteration;
  uint32_t* failed_pods;
  ffx_role* failed_roles;
  ffx_role* lazy_backup_targets;
  ffx_forward* forwards;
  ffx_redundant_source* redundant_from;
  uint32_t n_failed_pods, n_failed_roles, n_lazy, n_forwards, n_redundant;
} ffx_recovery_plan;

/* replicas = 1 is the reference rule (neighbour path iff no lost role's ring
 * successor is lost).  replicas = 2 is the double-neighbour extension: a lost
 * role is served by a surviving holder among dp+1, dp+2 -- roles with the
 * fewest surviving holders first, each to its least-loaded one (ties: the
 * nearest), so concurrent recoveries spread over the holders' NVLink. */
int ffx_plan_recovery(const ffx_cluster_spec* spec, const uint32_t* failed_pods, uint32_t n_pods,
                      const ffx_role* failed_roles, uint32_t n_roles, uint64_t global_consistent,
                      uint64_t latest_fallback_round, uint32_t replicas, ffx_recovery_plan* out);

/* ---- controller state that drives recovery -----------
 * Host-only (no GPU needed), thread-safe per object.  Timestamps are
 * caller-supplied nanoseconds (rt::Nanos): simulated or ffx_now_ns(). */

int64_t ffx_now_ns(void); /* CLOCK_MONOTONIC */

/* ctl::HeartbeatTable (controller.hpp:56-101, controller.cpp:16-77). */
typedef struct ffx_heartbeats ffx_heartbeats;
typedef struct ffx_heartbeat_slot {
  uint32_t enrolled, failed;
  int64_t last_seen_ns;
  uint64_t last_iteration;
} ffx_heartbeat_slot;
/* ControllerConfig{heartbeat_interval, miss_threshold} (controller.hpp:31-34) */
int ffx_heartbeats_create(uint32_t pods, int64_t interval_ns, uint32_t miss_threshold, ffx_heartbeats** out);
int ffx_heartbeats_destroy(ffx_heartbeats* h);
/* enroll: registration / substitution re-activates the slot (FFX_ERANGE past
 * the pod count, as slots_.at throws). */
int ffx_heartbeats_enroll(ffx_heartbeats* h, uint32_t node, uint64_t iteration, int64_t now_ns);
/* observe: unknown / already-failed senders and regressed iterations are
 * counted (ffx_heartbeats_counters), never an error. */
int ffx_heartbeats_observe(ffx_heartbeats* h, uint32_t node, uint64_t iteration, int64_t now_ns);
/* sweep: pods silent for more than interval * miss_threshold, newly marked
 * failed, in node order.  Writes min(n, cap) ids; *n_dead = n. */
int ffx_heartbeats_sweep(ffx_heartbeats* h, int64_t now_ns, uint32_t* dead, uint32_t cap, uint32_t* n_dead);
int ffx_heartbeats_mark_failed(ffx_heartbeats* h, uint32_t node);
int ffx_heartbeats_query(ffx_heartbeats* h, uint32_t node, ffx_heartbeat_slot* out);
int ffx_heartbeats_counters(ffx_heartbeats* h, uint64_t* unknown, uint64_t* late, uint64_t* regressed);

/* ctl::IterationLedger (controller.hpp:106-130, controller.cpp:81-121). */
struct ffx_replica;
typedef struct ffx_ledger ffx_ledger;
int ffx_ledger_create(const ffx_cluster_spec* spec, ffx_ledger** out);
int ffx_ledger_destroy(ffx_ledger* g);
/* Monotone per worker; FFX_ERANGE for a role outside the grid (ProtocolError). */
int ffx_ledger_record(ffx_ledger* g, ffx_role role, uint64_t iteration);
/* Minimum over the whole grid; 0 until every worker has recorded. */
uint64_t ffx_ledger_global_consistent(ffx_ledger* g);
/* Minimum over DP group pp * tensor_parallel + tp (absent members = 0). */
uint64_t ffx_ledger_group_latest(ffx_ledger* g, uint32_t dp_group);
uint64_t ffx_ledger_worker_latest(ffx_ledger* g, ffx_role role);
/* Post-recovery reset: every worker at `iteration`. */
int ffx_ledger_rebase(ffx_ledger* g, uint64_t iteration);
/* The CkptRecord after a completed replica (wire.hpp:85-90): record the
 * origin of the replica `held` at its newest COMMITTED iteration (a slot
 * still being written never counts).  *recorded = that iteration, or 0 when
 * nothing is committed yet (no record made). */
int ffx_ledger_record_replica(ffx_ledger* g, struct ffx_replica* held, uint64_t* recorded);

/* ---- sizing: the state partitioner's rules ------------------------------- */

int ffx_razor(const ffx_cluster_spec* spec, ffx_uniqueness_plan* out); /* ckpt.cpp:13-21 */
uint64_t ffx_weights_bytes(const ffx_cluster_spec* spec);               /* evolution.cpp:11-13 */
uint64_t ffx_optimizer_bytes(const ffx_cluster_spec* spec);             /* evolution.cpp:15-19 */
/* *out = 0 current / 1 previous; FFX_EVERSION outside the window.  ckpt.cpp:27-33 */
int ffx_version_for_target(uint64_t held_iteration, uint64_t target, int* out);

/* ---- SNP1 framing (storage.hpp:12-25) ------------------------------------ */

typedef struct ffx_blob_info { /* store::BlobInfo, storage.hpp:46-52 */
  ffx_role role;
  uint8_t kind; /* 0 weights, 1 optimizer */
  uint8_t pad_[1];
  uint32_t payload_len;
  uint64_t iteration;
  uint64_t checksum;
} ffx_blob_info;

/* Header bytes of store::pack_blob (storage.cpp:45-66); `checksum` is the
 * whole-payload FNV-1a (ffx_checksum64).  FFX_EINVAL when len > 4 GiB-1. */
int ffx_pack_header(ffx_role role, uint64_t iteration, uint8_t kind, uint64_t len,
                    uint64_t checksum, uint8_t out[32]);
/* store::parse_header (storage.cpp:74-90) plus the length check of
 * unpack_blob (:95-96) when framed_len != 0.  FFX_ECORRUPT on failure. */
int ffx_parse_header(const uint8_t* header, uint64_t framed_len, ffx_blob_info* out);

/* ---- device primitives (hash.cpp, evolution.cpp) ------------------------ */

/* checksum64 (hash.cpp:102-110) over a whole device buffer, bit-exact.
 * Byte-serial FNV-1a is parallelised by low-byte-state speculation and an
 * affine combine.  Blocks until *host_out is set. */
int ffx_checksum64(const void* dev, uint64_t len, uint64_t* host_out, void* stream);
/* dev_out[s] = checksum64(dev + s*slice_bytes, min(slice_bytes, len - s*slice_bytes)). */
int ffx_slice_checksums(const void* dev, uint64_t len, uint64_t slice_bytes,
                        uint64_t* dev_out, void* stream);
/* Fused copy + per-slice checksum: dst <- src, dev_out as above. */
int ffx_copy_checksums(void* dst, const void* src, uint64_t len, uint64_t slice_bytes,
                       uint64_t* dev_out, void* stream);
/* Fused copy + verify against dev_expected; dev_result[0] <- first bad slice
 * (UINT64_MAX if none), dev_result[1] <- number of bad slices. */
int ffx_copy_verify(void* dst, const void* src, uint64_t len, uint64_t slice_bytes,
                    const uint64_t* dev_expected, uint64_t* dev_result, void* stream);
/* Copy only (no checksum): the split policy's TMA copy kernel, `ctas` CTAs of
 * one warp each (0 = 16).  dst may be a peer-mapped pointer. */
int ffx_copy(void* dst, const void* src, uint64_t len, uint32_t ctas, void* stream);
/* evo::expand / evo::materialize (evolution.cpp:71-97) into device memory.
 * materialize: FFX_EINVAL when bytes < 32. */
int ffx_expand(void* dst, const uint8_t digest[32], uint64_t bytes, void* stream);
int ffx_materialize(void* dst, const uint8_t digest[32], uint64_t bytes, void* stream);
/* evo::blob_is_sound (evolution.cpp:106-110).  Blocks; *host_first_bad is the
 * first byte that differs from materialize(prefix), UINT64_MAX if sound. */
int ffx_blob_check(const void* dev, uint64_t bytes, uint64_t* host_first_bad, void* stream);

/* ---- buffer plumbing (for hosts without their own CUDA runtime, e.g. the
 * C++ facade over the reference API) ---------------------------------------- */

int ffx_device_alloc(int device, uint64_t bytes, void** dev);
/* Enable peer access from `device` to every peer it can reach over NVLink
 * (a warm spare does this before any failure, so mapping a holder's replica
 * later skips the lazy enable).  *enabled = peers now accessible. */
int ffx_prepare_peers(int device, uint32_t* enabled);
int ffx_device_free(int device, void* dev);
/* cudaMemcpyAsync(kind = default) on `stream`; blocks when sync != 0. */
int ffx_memcpy(void* dst, const void* src, uint64_t bytes, void* stream, int sync);
/* *is_device = 1 when p is device (or managed) memory visible to CUDA. */
int ffx_pointer_is_device(const void* p, int* is_device);
int ffx_stream_sync(void* stream);

/* ---- contexts and the state registry -------------------------------------- */

typedef struct ffx_ctx ffx_ctx;
typedef struct ffx_replica ffx_replica;

enum ffx_region_kind {
  FFX_REGION_MASTER = 0, /* fp32 master params shard */
  FFX_REGION_ADAM_M = 1,
  FFX_REGION_ADAM_V = 2,
  FFX_REGION_PARAMS = 3, /* bf16 params (unique under ZeRO-3, else redundant) */
  FFX_REGION_CURSOR = 4, /* data-loader cursor */
  FFX_REGION_RNG = 5,    /* RNG state */
  FFX_REGION_BLOB = 6    /* an opaque unique-state blob (the reference's model) */
};

/* slice_bytes: integrity/scheduling unit, a multiple of 256 (0 = default 4096). */
int ffx_open(int device, const ffx_cluster_spec* spec, ffx_role self, uint64_t slice_bytes,
             ffx_ctx** out);
int ffx_close(ffx_ctx* ctx);

/* Register a device region.  unique != 0: carried by every snapshot (the
 * razor's per-iteration payload); unique == 0: redundant across the DP ring,
 * re-read from a live peer on recovery.  Order of registration is the payload
 * order.  FFX_ECONFIG when the registry is full, FFX_EINVAL on misalignment. */
int ffx_register_region(ffx_ctx* ctx, int kind, void* dev, uint64_t bytes, int unique);
int ffx_clear_regions(ffx_ctx* ctx);

typedef struct ffx_plan_info {
  ffx_uniqueness_plan razor;           /* the reference rule for ctx's spec */
  uint64_t registered_unique_bytes;    /* what one snapshot moves */
  uint64_t registered_redundant_bytes; /* what a recovery re-reads from a live peer */
  uint64_t slice_bytes;
  uint64_t num_slices; /* unique slices (checksum table entries) */
  uint32_t num_regions;
  uint32_t num_unique_regions;
} ffx_plan_info;
int ffx_plan(ffx_ctx* ctx, ffx_plan_info* out);

/* How a snapshot's payload is cut into checksum slices (the checksum table
 * order).  Every region is one run of slice_bytes slices, except that the
 * first region of a payload of fewer than FFX_MAX_REGIONS regions, when it
 * holds at least 4 x 48 MiB and slice_bytes is a multiple of 1 KiB, opens
 * with a 48 MiB head of slice_bytes/4 slices: the tasks claimed last by the
 * persistent snapshot kernel are then short, which trims its tail.  Writes
 * up to `cap` runs and their count (<= n + 1). */
typedef struct ffx_slice_run {
  uint32_t region;      /* index into region_bytes */
  uint32_t slice_bytes; /* slice size of this run */
  uint64_t offset;      /* byte offset of the run inside its region */
  uint64_t bytes;
  uint64_t first_slice; /* checksum-table index of the run's first slice */
} ffx_slice_run;
int ffx_slice_runs(const uint64_t* region_bytes, uint32_t n, uint64_t slice_bytes, ffx_slice_run* out,
                   uint32_t cap, uint32_t* count);

/* ---- neighbour replica manager (NeighborBuffer, ckpt.hpp:105-120) --------- */

/* Holder side: device slots for `origin`'s snapshots, `versions` of them
 * (the reference keeps 2: ckpt.cpp:92), each with `capacity` payload bytes.
 * capacity mirrors HostSnapshots(role, capacity) (ckpt.hpp:82-86). */
int ffx_replica_create(ffx_ctx* ctx, ffx_role origin, uint64_t capacity, uint32_t versions,
                       ffx_replica** out);
/* Opaque FFX_HANDLE_BYTES blob (CUDA IPC handle + layout) for another rank. */
int ffx_replica_export(const ffx_replica* r, uint8_t handle[FFX_HANDLE_BYTES]);
/* Map a replica exported by another rank (or this process) into ctx. */
int ffx_replica_open(ffx_ctx* ctx, const uint8_t handle[FFX_HANDLE_BYTES], ffx_replica** out);
int ffx_replica_destroy(ffx_replica* r);

typedef struct ffx_slot_info {
  uint32_t state; /* 0 empty, 1 writing (torn if seen at rest), 2 committed */
  uint32_t num_regions;
  ffx_role role;
  uint8_t kind;
  uint8_t whole_checksum_valid;
  uint64_t iteration;
  uint64_t payload_len;
  uint64_t slice_bytes;
  uint64_t num_slices;
  uint64_t whole_checksum;
  uint64_t seq; /* write sequence number: larger is newer */
} ffx_slot_info;
int ffx_replica_slots(const ffx_replica* r, uint32_t* versions);
int ffx_replica_slot_info(ffx_replica* r, uint32_t slot, ffx_slot_info* out);
/* The state registry a committed slot was taken from: *n regions (at most
 * FFX_MAX_REGIONS) with their ffx_region_kind and byte sizes, in payload
 * order -- what a replacement process allocates and registers before
 * ffx_recover (the reference's StateBundle shape, domain.hpp:105-110).
 * kinds / bytes may be NULL.  FFX_ERESTORE if the slot is not committed. */
#define FFX_MAX_REGIONS 16
int ffx_replica_slot_regions(ffx_replica* r, uint32_t slot, uint32_t* n, int32_t* kinds, uint64_t* bytes);
/* NeighborBuffer::newest() (ckpt.cpp:102-105): FFX_ERESTORE if nothing committed. */
int ffx_replica_newest(ffx_replica* r, uint64_t* iteration);
/* Device pointers into slot `slot` (payload, checksum table). */
int ffx_replica_slot_ptrs(ffx_replica* r, uint32_t slot, void** payload, uint64_t** sums);
/* NeighborBuffer::clear() (ckpt.hpp:117). */
int ffx_replica_clear(ffx_replica* r);
/* Rollback to the global consistent iteration (the new epoch after
 * orchestrate_recovery, controller.cpp:315-318): slots holding an iteration
 * newer than `iteration` were committed before the failure and are dropped
 * (marked empty), so a CkptRecord read from this replica
 * (ffx_ledger_record_replica) cannot re-raise the rebased ledger before the
 * replay re-commits them -- the reference ignores stale-epoch CkptRecords
 * (Controller::on_ckpt_record).  *dropped = slots emptied (may be NULL).
 * Writers into this replica re-arm it afterwards (ffx_snapshot_target re-reads
 * the slot table), as every rank does when the new epoch starts. */
int ffx_replica_rollback(ffx_replica* r, uint64_t iteration, uint32_t* dropped);
/* SNP1 frame export (framed_at(), ckpt.cpp:95-100 + pack_blob layout): copies
 * header + payload (regions concatenated) to host memory; computes the
 * whole-payload FNV on the device if not yet known.  *framed_len = 32 + len.
 * FFX_ERESTORE when the iteration is not held, FFX_ECONFIG when cap is short,
 * FFX_EINVAL when the payload exceeds the 4 GiB SNP1 limit (storage.cpp:48). */
int ffx_replica_export_frame(ffx_replica* r, uint64_t iteration, void* host_dst, uint64_t cap,
                             uint64_t* framed_len, void* stream);
/* The same for payloads of any size: part `part` of *parts SNP1 frames, each
 * carrying FFX_FRAME_PART_BYTES (the last one the rest) of the concatenated
 * regions with its own length and whole-payload FNV -- the split a caller of
 * pack_blob must make above its 4 GiB limit (storage.cpp:48-49).  host_dst
 * NULL = size query (*framed_len, *parts).  FFX_ERANGE past the last part. */
#define FFX_FRAME_PART_BYTES 0xFFFFF000ull /* 4 GiB - 4 KiB: the largest slice-aligned SNP1 payload */
int ffx_replica_export_frame_part(ffx_replica* r, uint64_t iteration, uint32_t part, void* host_dst,
                                  uint64_t cap, uint64_t* framed_len, uint32_t* parts, void* stream);

/* ---- snapshot (HostSnapshots::take + ring stream, ckpt.cpp:38-53) --------- */

/* Where this rank's snapshots land: normally the replica its ring successor
 * created for it and exported (opened with ffx_replica_open). */
int ffx_snapshot_target(ffx_ctx* ctx, ffx_replica* target);
/* Double-neighbour replication: a second holder (dp+2) that
 * receives the same tiles from the same kernel -- one HBM read, two stores,
 * one checksum pass.  NULL removes it. */
int ffx_snapshot_target2(ffx_ctx* ctx, ffx_replica* target);

/* ---- double neighbour over NVSwitch multicast ---------------
 * The same dp+1 / dp+2 replication as ffx_snapshot_target2, but every tile
 * leaves the origin ONCE: the snapshot kernel stores into a multicast range
 * the switch fans out to both holders' slots (egress N instead of 2N).  The
 * reference has no double neighbour; this extends NeighborBuffer
 * (ckpt.cpp:77-105) and the adjacent-pair fallback (controller.cpp:162-167).
 * Measured: a lone writer delivers both replicas at
 * ~560 GB/s vs ~350 per copy for two unicast stores, but with every rank
 * snapshotting at once the writer's own team copy loads its NVLink ingress
 * (3N per GPU vs 2N), so ffx_snapshot_target2 is the faster ring default.
 * Sequence (one process per GPU; handles travel like replica handles, the
 * fds behind them are fetched from the exporting process by libffx):
 *   holders : ffx_replica_create_shared(origin)  -> export handle
 *   origin  : ffx_mcast_create(members = 3)      -> export handle
 *   holders : ffx_mcast_open(handle)
 *   all     : ffx_mcast_join  (every member; before any bind)
 *   holders : ffx_mcast_bind(mc, held replica)
 *   origin  : ffx_replica_open(holder 1 handle) -> view;
 *             ffx_snapshot_target_mcast(ctx, mc, view)
 * Recovery reads either holder's replica as usual (ffx_recover*). */
#define FFX_MCAST_HANDLE_BYTES 64
typedef struct ffx_mcast ffx_mcast;
/* 1 if `device` supports multicast objects (NVSwitch, fabric manager up). */
int ffx_mcast_supported(int device, int* supported);
/* A replica whose memory can be bound to a multicast range (a shareable VMM
 * allocation instead of cudaMalloc); otherwise identical to
 * ffx_replica_create, exported/opened with the same calls. */
/* Tiered replica (SURVEY 7.2 hard part 3: a Llama-3 70B replica does not fit
 * next to its holder's own state in 180 GB): one slot range whose first
 * hbm_bytes are device memory and the rest pinned host memory on the
 * holder's NUMA node -- the reference keeps its replicas in host memory
 * (ckpt.cpp:52, :92).  Exported / opened / snapshotted / recovered like any
 * replica; the host tier moves over PCIe.  ffx_replica_tiers reports the split. */
int ffx_replica_create_tiered(ffx_ctx* ctx, ffx_role origin, uint64_t capacity, uint32_t versions,
                              uint64_t hbm_bytes, ffx_replica** out);
int ffx_replica_tiers(const ffx_replica* r, uint64_t* hbm_bytes, uint64_t* host_bytes);
int ffx_replica_create_shared(ffx_ctx* ctx, ffx_role origin, uint64_t capacity, uint32_t versions,
                              ffx_replica** out);
/* Origin: a multicast object sized for replicas of (capacity, versions,
 * ctx slice bytes) with `members` devices (the origin + its holders). */
int ffx_mcast_create(ffx_ctx* ctx, uint64_t capacity, uint32_t versions, uint32_t members, ffx_mcast** out);
int ffx_mcast_export(const ffx_mcast* m, uint8_t handle[FFX_MCAST_HANDLE_BYTES]);
int ffx_mcast_open(ffx_ctx* ctx, const uint8_t handle[FFX_MCAST_HANDLE_BYTES], ffx_mcast** out);
/* Add this process's device to the team (blocks nothing; binds and the
 * origin's mapping wait until every member joined). */
int ffx_mcast_join(ffx_mcast* m);
/* Holder: bind its shared replica for this origin into the range. */
int ffx_mcast_bind(ffx_mcast* m, ffx_replica* held);
/* Origin: map the range and make it this context's snapshot target; `view`
 * is one holder's replica opened here (slot metadata is read through it).
 * Clears any ffx_snapshot_target2. */
int ffx_snapshot_target_mcast(ffx_ctx* ctx, ffx_mcast* m, ffx_replica* view);
int ffx_mcast_destroy(ffx_mcast* m);

typedef struct ffx_snapshot_opts {
  uint32_t max_ctas;       /* SM budget for the snapshot kernel (0 = whole GPU) */
  uint32_t batches;        /* slice batches the scheduler splits one snapshot into (0/1 = one) */
  void* gate_events;       /* cudaEvent_t[batches] each batch waits on (NULL = none) */
  uint32_t verify_on_store;/* holder-side re-verify after landing (ckpt.cpp:78 semantics) */
  uint32_t weights_kind;   /* nonzero: frame as BlobKind::Weights (0), else Optimizer (1) */
  /* Split policy: copy and checksum are scheduled separately -- copy batches
   * (TMA copy-only kernel, max_ctas CTAs, or the copy engines) for the gaps
   * where NVLink is idle, hash batches (local state -> the slot's checksum
   * table) for the gaps where SMs are idle.  The slot commits once both
   * queues drain.  0 = fused copy+checksum batches. */
  uint32_t split;
  uint32_t hash_batches;   /* split: hash batches (0 = batches) */
  uint32_t hash_ctas;      /* split: SM budget of hash batches (0 = whole GPU) */
  uint32_t copy_engine;    /* split: copy batches by cudaMemcpyAsync (no SMs) */
  /* split + copy_engine: the first fused_permille/1000 of the warp tasks go
   * through the fused kernel (TMA stores to the target, checksummed on the
   * way, issued with the first hash batch); the copy engines move only the
   * rest.  Two NVLink write paths at once beat either alone
   * (DESIGN.md section 6).  0 = copy engines move everything. */
  uint32_t fused_permille;
  /* Measured gaps: relative sizes of the copy batches (`batches` entries,
   * e.g. the durations of the step's idle-link windows measured with events
   * in a calibration step).  NULL = equal batches.  Hash batches of the
   * split policy stay equal. */
  const double* batch_weights;
  /* Nonzero: fused batches launch one CTA per task group and no persistent
   * claim loop, so under stream priorities the block scheduler hands SMs to
   * pending TRAIN CTAs at every task boundary (one 32-slice task, ~0.1 ms) and
   * STATE CTAs only fill what TRAIN leaves idle (wave tails, kernel
   * boundaries) -- the reference's chunk-boundary preemption
   * (sim_net.cpp:401-454) at task granularity; max_ctas is then ignored. */
  uint32_t task_ctas;
  uint32_t pad_;
} ffx_snapshot_opts;

enum ffx_batch_kind { FFX_BATCH_COPY = 0, FFX_BATCH_HASH = 1 };

/* Snapshot all unique regions into the target replica at `iteration`, async
 * on `stream`.  Slot choice follows the two-version rule: replace the slot
 * already holding `iteration`, else overwrite the older of the two
 * (ckpt.cpp:46-52, :86-92).  FFX_ECONFIG when the registered unique bytes
 * exceed the target capacity (ckpt.cpp:40-43). */
int ffx_snapshot(ffx_ctx* ctx, uint64_t iteration, void* stream, const ffx_snapshot_opts* opts);

/* The slice scheduler, step by step: begin() fixes the slot, layout and the
 * split into opts->batches batches (no GPU work); each next() launches one
 * batch on `stream` after `gate_event` (a cudaEvent_t the training step
 * records when a gap opens -- e.g. right after an all-gather completes; NULL
 * = no gate).  The last batch commits the slot.  ffx_snapshot() is
 * begin + next for every batch with opts->gate_events[b]. */
int ffx_snapshot_begin(ffx_ctx* ctx, uint64_t iteration, const ffx_snapshot_opts* opts,
                       uint32_t* batches);
int ffx_snapshot_next(ffx_ctx* ctx, void* stream, void* gate_event, uint32_t* remaining);
/* Issue the next batch of one kind (split policy: FFX_BATCH_COPY or
 * FFX_BATCH_HASH; fused snapshots only have copy batches). */
int ffx_snapshot_next_kind(ffx_ctx* ctx, int kind, void* stream, void* gate_event, uint32_t* remaining);

/* ---- the slice scheduler as a native object ---------------------------------
 * TRAIN > STATE (sim_net.cpp:401-454): the training step reports its gaps and
 * the scheduler issues one snapshot batch per gap on its own low-priority
 * streams, gated on an event recorded on the step's stream, so STATE work
 * only starts where TRAIN leaves the resource idle and can delay TRAIN by
 * at most one batch (its CTA cap).
 *   FFX_GAP_LINK_IDLE   a collective just finished (NVLink idle while the
 *                       step computes): copy batches go here
 *   FFX_GAP_SM_IDLE     a collective is about to start (SMs idle behind
 *                       NCCL): split-policy checksum batches go here
 * ffx_sched_finish() issues whatever is left and makes the step's stream
 * wait for the slot commit -- call it before the optimizer mutates the
 * registered state. */
enum ffx_sched_policy {
  FFX_SCHED_FUSED = 0,     /* copy + checksum batches in the link-idle gaps */
  FFX_SCHED_SPLIT = 1,     /* TMA copy batches (link-idle) + checksum batches (SM-idle) */
  FFX_SCHED_SPLIT_CE = 2   /* copy-engine batches (link-idle) + checksum batches (SM-idle) */
};
enum ffx_gap_kind { FFX_GAP_LINK_IDLE = 0, FFX_GAP_SM_IDLE = 1 };
typedef struct ffx_sched_opts {
  uint32_t policy;         /* ffx_sched_policy */
  uint32_t link_gaps;      /* FFX_GAP_LINK_IDLE reports per step (copy batches) */
  uint32_t sm_gaps;        /* FFX_GAP_SM_IDLE reports per step (checksum batches; split) */
  uint32_t copy_ctas;      /* CTA cap of fused / TMA copy batches (0 = 32 / 8) */
  uint32_t hash_ctas;      /* CTA cap of checksum batches (0 = 96) */
  uint32_t task_ctas;      /* fused policy: task-granular batches (ffx_snapshot_opts.task_ctas) */
  const double* gap_ms;    /* measured link-idle gap durations, link_gaps entries (NULL = equal) */
} ffx_sched_opts;
typedef struct ffx_sched ffx_sched;
int ffx_sched_create(ffx_ctx* ctx, const ffx_sched_opts* opts, ffx_sched** out);
int ffx_sched_begin(ffx_sched* s, uint64_t iteration);
int ffx_sched_gap(ffx_sched* s, int gap_kind, void* train_stream);
int ffx_sched_finish(ffx_sched* s, void* train_stream);
int ffx_sched_destroy(ffx_sched* s);

/* ---- the data loader's preload buffer -------------------
 * data::PreloadBuffer (dataloader.hpp:45-73, dataloader.cpp:59-82) in HBM:
 * byte-capped, ordered by iteration (this rank's TIDs), consumption evicts.
 * Entries are stream-ordered allocations from the device memory pool. */
typedef struct ffx_preload ffx_preload;
typedef struct ffx_preload_state {
  uint64_t capacity, bytes; /* PreloadBuffer::capacity() / bytes() */
  uint64_t entries;         /* size() */
  uint64_t oldest;          /* oldest() iteration, UINT64_MAX when empty */
  uint64_t fetched, taken;
} ffx_preload_state;
int ffx_preload_create(ffx_ctx* ctx, uint64_t capacity_bytes, ffx_preload** out);
int ffx_preload_destroy(ffx_preload* p);
int ffx_preload_fits(ffx_preload* p, uint64_t bytes, int* fits);
/* insert() with the bytes streamed in on `stream` after `gate_event` (either
 * may be NULL): FFX_ECONFIG past the capacity, FFX_ESTATE for an iteration
 * already held (the reference's std::logic_error cases).
 *  _host:      `bytes` from host memory (H2D on the copy engines; pinned
 *              memory must stay valid until the copy completes).
 *  _synthetic: DataServerStub::fetch in synthetic mode, generated on the
 *              device: `count` samples of `sample_bytes`, sample i =
 *              expand(item_digests[i]) -- item_digests[i] =
 *              data_item_digest(seed, window.first + i) (evolution.cpp:112-120),
 *              32 bytes each, computed by the caller's SHA-256. */
int ffx_preload_fetch_host(ffx_preload* p, uint64_t iteration, const void* host_src, uint64_t bytes, void* stream,
                           void* gate_event);
int ffx_preload_fetch_synthetic(ffx_preload* p, uint64_t iteration, const uint8_t* item_digests, uint32_t count,
                                uint32_t sample_bytes, void* stream, void* gate_event);
/* take(): the entry leaves the buffer; `consumer_stream` waits for its fetch
 * and owns the device memory until ffx_preload_free (stream-ordered).
 * FFX_ESTATE when the iteration is not held (take() -> nullopt). */
int ffx_preload_take(ffx_preload* p, uint64_t iteration, void* consumer_stream, void** dev, uint64_t* bytes);
int ffx_preload_free(ffx_preload* p, void* dev, void* consumer_stream);
int ffx_preload_info(ffx_preload* p, ffx_preload_state* out);
/* data::fold_of_blob (dataloader.cpp:150-164) on the device: FFX_EINVAL
 * unless bytes is a whole number of samples. */
int ffx_fold_of_blob(const void* dev, uint64_t bytes, uint32_t bytes_per_sample, uint64_t* host_out, void* stream);
/* Preload through the slice scheduler (SPEC preload_loop: fetch only when
 * the link is idle and the buffer has room): the fetch is queued and issued
 * at the next FFX_GAP_LINK_IDLE report -- with or without a snapshot in
 * flight -- on the scheduler's low-priority copy stream, gated on that gap;
 * a fetch that does not fit stays queued (buffer full: no fetch issued).
 * Host bytes must be pinned and stay valid until taken. */
int ffx_sched_preload_host(ffx_sched* s, ffx_preload* p, uint64_t iteration, const void* host_src, uint64_t bytes);
int ffx_sched_preload_synthetic(ffx_sched* s, ffx_preload* p, uint64_t iteration, const uint8_t* item_digests,
                                uint32_t count, uint32_t sample_bytes);
/* fetches still queued in the scheduler */
int ffx_sched_preload_pending(ffx_sched* s, uint32_t* pending);

/* The logical payload bytes [*lo, *hi) (the registered unique regions
 * concatenated) that fused batch `batch` of the pending snapshot reads:
 * what must have landed before that batch's ffx_snapshot_next.  Batches cover
 * consecutive, increasing spans.  FFX_ESTATE without a pending fused
 * snapshot, FFX_ERANGE past the last batch. */
int ffx_snapshot_batch_span(ffx_ctx* ctx, uint32_t batch, uint64_t* lo, uint64_t* hi);
/* HostSnapshots::take(it, host_ptr, len) (ckpt.hpp:88) for device-resident
 * state: copies `len` host bytes (the registered unique regions
 * concatenated; len must equal their total) into those regions and snapshots
 * them as `iteration`, pipelined -- the H2D copy of batch b+1's span runs on
 * an internal stream while batch b's kernel runs on `stream`.  batches = 0:
 * 8 for payloads >= 64 MiB, else 1.  Stream-ordered like ffx_snapshot; pinned
 * host memory for the overlap (pageable memory is correct, just serial). */
int ffx_snapshot_from_host(ffx_ctx* ctx, uint64_t iteration, const void* host, uint64_t len, uint32_t batches,
                           void* stream);

/* Copy the checksum table written by this ctx's most recent snapshot into
 * host memory (async on `stream`; pinned memory for true overlap).
 * *n_out = entries copied (min(table, max_entries)). */
int ffx_snapshot_read_sums(ffx_ctx* ctx, uint64_t* host_dst, uint64_t max_entries, uint64_t* n_out,
                           void* stream);

/* ---- pull mode: the holder drives the ring stream -------------------------
 * NeighborBuffer::store is the holder's action in the reference
 * (ckpt.cpp:77-93).  In pull mode the holder's kernel reads the origin's
 * registered regions over NVLink (peer loads run at the link's full read
 * rate), hashes them and commits its own slot; the commit also sets the
 * origin's ack word, which the origin's stream waits on before its next
 * optimizer update (ffx_snapshot_wait_pulled). */
#define FFX_REGIONS_HANDLE_BYTES 2048
typedef struct ffx_remote ffx_remote;
/* Origin: describe this ctx's unique regions (CUDA IPC) for its holder. */
int ffx_regions_export(ffx_ctx* ctx, uint8_t handle[FFX_REGIONS_HANDLE_BYTES]);
/* Holder: map an origin's regions. */
int ffx_remote_open(ffx_ctx* ctx, const uint8_t handle[FFX_REGIONS_HANDLE_BYTES], ffx_remote** out);
int ffx_remote_close(ffx_remote* r);
/* Holder: snapshot `origin` at `iteration` into the replica it holds for it. */
int ffx_snapshot_pull(ffx_ctx* ctx, ffx_remote* origin, ffx_replica* held, uint64_t iteration, void* stream,
                      const ffx_snapshot_opts* opts);
int ffx_snapshot_begin_pull(ffx_ctx* ctx, ffx_remote* origin, ffx_replica* held, uint64_t iteration,
                            const ffx_snapshot_opts* opts, uint32_t* batches);
/* Origin: make `stream` wait until the holder has committed `iteration`
 * (cuStreamWaitValue64 on the ack word; no kernel, no host round trip).
 * The ack is a one-shot token: the wait matches the committed iteration
 * exactly and then consumes it, so call it once per pulled iteration. */
int ffx_snapshot_wait_pulled(ffx_ctx* ctx, uint64_t iteration, void* stream);
/* Origin: drop any un-consumed ack (stream-ordered).  Call on a rollback to
 * the global consistent iteration (controller.cpp:315-318, ledger rebase):
 * a replayed iteration must wait for its own re-pull.  ffx_recover* reset it
 * implicitly. */
int ffx_snapshot_ack_reset(ffx_ctx* ctx, void* stream);

/* ---- recovery (assemble_restore, ckpt.cpp:111-167) ------------------------ */

typedef struct ffx_recover_report {
  uint64_t bytes;          /* payload bytes pulled and verified */
  uint64_t first_bad_slice;/* UINT64_MAX when every slice verified */
  uint64_t bad_slices;
  uint32_t slot;           /* replica slot used */
  uint32_t pad_;
  double seconds;          /* device time of the gather/verify */
} ffx_recover_report;

/* Holder: verify a committed slot as landed -- re-hash its payload from the
 * holder's own HBM against the slot's checksum table (NeighborBuffer::store
 * validates before accepting, ckpt.cpp:78; storage.cpp:98-99).  For the split
 * / copy-engine policies, whose table is computed from the origin's source,
 * this is the check on the bytes that crossed NVLink.  FFX_ECORRUPT with the
 * first bad slice in rep (the slot is then marked torn and never restored
 * from; the writer re-arms with ffx_snapshot_target to reuse it first);
 * max_ctas caps the launch (0 = whole GPU).  Blocks on stream. */
int ffx_replica_verify(ffx_ctx* ctx, ffx_replica* held, uint64_t iteration, uint32_t max_ctas, void* stream,
                       ffx_recover_report* rep);


/* Rebuild ctx's unique regions at `target` from a replica (the holder's
 * NeighborBuffer for this role), pulling over NVLink/P2P with fused slice
 * verification.  FFX_ERESTORE: slot missing / stale / torn / wrong role or
 * kind / region layout mismatch / checksum mismatch (report says which slice).
 * Blocks until verified. */
int ffx_recover(ffx_ctx* ctx, ffx_replica* src, uint64_t target, void* stream,
                ffx_recover_report* report);

/* Parallel peer gathers: the same snapshot held by several replicas (e.g. the
 * dp+1 and dp+2 holders of double-neighbour replication); each region's
 * slices are split into nsrc parts pulled concurrently from the nsrc sources
 * by one kernel, all verified against the first source's checksum table.
 * Every source must hold a committed, matching slot (same checks as
 * ffx_recover).  nsrc in 1..4. */
int ffx_recover_from(ffx_ctx* ctx, ffx_replica* const* srcs, uint32_t nsrc, uint64_t target, void* stream,
                     ffx_recover_report* report);

/* A redundant region's live copy on a DP peer (weights, ckpt.cpp:150-152):
 * peer-mapped pointer + the peer's slice table (ffx_slice_checksums).  The
 * table holds ceil(bytes / slice_bytes) entries; it must have been computed
 * with this ctx's slice size (FFX_ECONFIG otherwise -- a table cut at another
 * size would be read past its end). */
typedef struct ffx_peer_region {
  uint32_t region_index; /* index in this ctx's registration order */
  uint32_t slice_bytes;  /* slice size of `sums` (0: this ctx's, as before) */
  const void* src;
  const uint64_t* sums;
} ffx_peer_region;

/* Full-state restore in one kernel (assemble_restore, ckpt.cpp:140-167): the
 * unique regions from the replica holders (split across nsrc sources) and
 * every redundant region from its live peer, all gathered concurrently and
 * each part verified against its own source's checksum table. */
int ffx_recover_full(ffx_ctx* ctx, ffx_replica* const* srcs, uint32_t nsrc, uint64_t target,
                     const ffx_peer_region* redundant, uint32_t nred, void* stream, ffx_recover_report* report);

/* Pull one redundant region (weights from a live DP peer, ckpt.cpp:150-152)
 * from a peer device pointer, verifying against the peer's slice table
 * (computed by the peer with ffx_slice_checksums; same slice-size rule as
 * ffx_recover_full). */
int ffx_recover_region(ffx_ctx* ctx, const ffx_peer_region* peer, void* stream, ffx_recover_report* report);

/* Map / unmap a raw device allocation exported by another process (for the
 * redundant-region pull).  handle = cudaIpcMemHandle_t bytes (64). */
int ffx_ipc_export(void* dev_base, uint8_t handle[64]);
int ffx_ipc_open(const uint8_t handle[64], void** dev_base);
int ffx_ipc_close(void* dev_base);

/* ---- failure injection ---------------------------------- */

enum ffx_fault {
  FFX_FAULT_POISON_STATE = 0,   /* fill ctx's unique regions with a poison pattern */
  FFX_FAULT_CORRUPT_REPLICA = 1,/* flip one payload byte (arg = slot<<48 | offset) */
  FFX_FAULT_TEAR_SLOT = 2,      /* leave slot (arg) in the "writing" state */
  FFX_FAULT_CORRUPT_SUMS = 3    /* flip one checksum-table entry (arg = slot<<48 | index) */
};
int ffx_inject(ffx_ctx* ctx, int fault, ffx_replica* r, uint64_t arg);

typedef struct ffx_stats {
  uint64_t snapshots;
  uint64_t snapshot_bytes; /* backup_bytes in the reference's metrics (metrics.hpp:32-83) */
  uint64_t recoveries;
  uint64_t recovered_bytes;
  uint64_t verify_failures;
  uint64_t kernel_launches;
} ffx_stats;
int ffx_get_stats(ffx_ctx* ctx, ffx_stats* out);

#ifdef __cplusplus
}
#endif

#endif /* FFX_H_ */
