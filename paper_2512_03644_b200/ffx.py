"""ctypes binding of libffx.so (include/ffx.h) -- plumbing for tests and bench.

The product is the C ABI and the C++ facade over it; this module only lets
Python (pytest, bench.py, torch.distributed for handle exchange) drive it.
Device memory comes from torch tensors; every byte of payload work runs in the
sm_100a kernels.  Status codes map 1:1 onto the reference's exception types
(ckpt.hpp:58-68, storage.hpp:55-57), mirrored here as Python exceptions with
the reference's names.

There is deliberately no CPU fallback: importing this module without the
built library raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libffx.so")
ABI_VERSION = 2
HANDLE_BYTES = 256
REGIONS_HANDLE_BYTES = 2048
MCAST_HANDLE_BYTES = 64
MAX_REGIONS = 16

# status codes (ffx.h)
OK, ECONFIG, EVERSION, ERESTORE, ECORRUPT, EINVAL, ERANGE, ECUDA, ENOMEM, ESTATE = range(10)

# region kinds
REGION_MASTER, REGION_ADAM_M, REGION_ADAM_V, REGION_PARAMS, REGION_CURSOR, REGION_RNG, REGION_BLOB = range(7)
# faults
FAULT_POISON_STATE, FAULT_CORRUPT_REPLICA, FAULT_TEAR_SLOT, FAULT_CORRUPT_SUMS = range(4)
SLOT_EMPTY, SLOT_WRITING, SLOT_COMMITTED = 0, 1, 2
BATCH_COPY, BATCH_HASH = 0, 1
U64_MAX = (1 << 64) - 1


class FfxError(RuntimeError):
    status = -1


class ConfigError(FfxError):       # ckpt::ConfigError (ckpt.hpp:58-60)
    status = ECONFIG


class VersionError(FfxError):      # ckpt::VersionError (ckpt.hpp:62-64)
    status = EVERSION


class RestoreError(FfxError):      # ckpt::RestoreError (ckpt.hpp:66-68)
    status = ERESTORE


class CorruptSnapshot(FfxError):   # store::CorruptSnapshot (storage.hpp:55-57)
    status = ECORRUPT


class InvalidArgument(FfxError, ValueError):  # std::invalid_argument
    status = EINVAL


class OutOfRange(FfxError, IndexError):       # std::out_of_range
    status = ERANGE


class CudaError(FfxError):
    status = ECUDA


class OutOfMemory(FfxError, MemoryError):
    status = ENOMEM


class StateError(FfxError):
    status = ESTATE


_EXC = {c.status: c for c in (ConfigError, VersionError, RestoreError, CorruptSnapshot,
                              InvalidArgument, OutOfRange, CudaError, OutOfMemory, StateError)}


class Role(ctypes.Structure):
    _fields_ = [("dp", ctypes.c_uint16), ("pp", ctypes.c_uint16), ("tp", ctypes.c_uint16)]

    def __repr__(self):
        return "d%dp%dt%d" % (self.dp, self.pp, self.tp)

    def __eq__(self, o):
        return isinstance(o, Role) and (self.dp, self.pp, self.tp) == (o.dp, o.pp, o.tp)

    def __hash__(self):
        return hash((self.dp, self.pp, self.tp))

    def tuple(self):
        return (self.dp, self.pp, self.tp)


class ClusterSpec(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_uint32), ("gpus_per_node", ctypes.c_uint32),
                ("data_parallel", ctypes.c_uint32), ("pipeline_parallel", ctypes.c_uint32),
                ("tensor_parallel", ctypes.c_uint32), ("distributed_optimizer", ctypes.c_uint32),
                ("params_per_device", ctypes.c_uint64)]


def make_spec(d=1, p=1, t=1, phi=1_000_000_000, distributed=False, num_nodes=None, gpus_per_node=None):
    world = d * p * t
    if gpus_per_node is None:
        gpus_per_node = world if num_nodes is None else world // num_nodes
    if num_nodes is None:
        num_nodes = max(1, world // gpus_per_node)
    return ClusterSpec(num_nodes, gpus_per_node, d, p, t, int(bool(distributed)), phi)


class UniquenessPlan(ctypes.Structure):
    _fields_ = [("weights_redundant", ctypes.c_uint32), ("optimizer_redundant", ctypes.c_uint32),
                ("unique_bytes_per_device", ctypes.c_uint64)]


class BlobInfo(ctypes.Structure):
    _fields_ = [("role", Role), ("kind", ctypes.c_uint8), ("pad_", ctypes.c_uint8 * 1),
                ("payload_len", ctypes.c_uint32), ("iteration", ctypes.c_uint64),
                ("checksum", ctypes.c_uint64)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("razor", UniquenessPlan), ("registered_unique_bytes", ctypes.c_uint64),
                ("registered_redundant_bytes", ctypes.c_uint64), ("slice_bytes", ctypes.c_uint64),
                ("num_slices", ctypes.c_uint64), ("num_regions", ctypes.c_uint32),
                ("num_unique_regions", ctypes.c_uint32)]


class SliceRun(ctypes.Structure):
    _fields_ = [("region", ctypes.c_uint32), ("slice_bytes", ctypes.c_uint32), ("offset", ctypes.c_uint64),
                ("bytes", ctypes.c_uint64), ("first_slice", ctypes.c_uint64)]


class SlotInfo(ctypes.Structure):
    _fields_ = [("state", ctypes.c_uint32), ("num_regions", ctypes.c_uint32), ("role", Role),
                ("kind", ctypes.c_uint8), ("whole_checksum_valid", ctypes.c_uint8),
                ("iteration", ctypes.c_uint64), ("payload_len", ctypes.c_uint64),
                ("slice_bytes", ctypes.c_uint64), ("num_slices", ctypes.c_uint64),
                ("whole_checksum", ctypes.c_uint64), ("seq", ctypes.c_uint64)]


class SnapshotOpts(ctypes.Structure):
    _fields_ = [("max_ctas", ctypes.c_uint32), ("batches", ctypes.c_uint32),
                ("gate_events", ctypes.c_void_p), ("verify_on_store", ctypes.c_uint32),
                ("weights_kind", ctypes.c_uint32), ("split", ctypes.c_uint32),
                ("hash_batches", ctypes.c_uint32), ("hash_ctas", ctypes.c_uint32),
                ("copy_engine", ctypes.c_uint32), ("fused_permille", ctypes.c_uint32),
                ("batch_weights", ctypes.POINTER(ctypes.c_double)),
                ("task_ctas", ctypes.c_uint32), ("pad_", ctypes.c_uint32)]


class SchedOpts(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_uint32), ("link_gaps", ctypes.c_uint32), ("sm_gaps", ctypes.c_uint32),
                ("copy_ctas", ctypes.c_uint32), ("hash_ctas", ctypes.c_uint32), ("task_ctas", ctypes.c_uint32),
                ("gap_ms", ctypes.POINTER(ctypes.c_double))]


SCHED_FUSED, SCHED_SPLIT, SCHED_SPLIT_CE = 0, 1, 2
GAP_LINK_IDLE, GAP_SM_IDLE = 0, 1


class RecoverReport(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_uint64), ("first_bad_slice", ctypes.c_uint64),
                ("bad_slices", ctypes.c_uint64), ("slot", ctypes.c_uint32), ("pad_", ctypes.c_uint32),
                ("seconds", ctypes.c_double)]


class PeerRegion(ctypes.Structure):
    _fields_ = [("region_index", ctypes.c_uint32), ("slice_bytes", ctypes.c_uint32),
                ("src", ctypes.c_void_p), ("sums", ctypes.c_void_p)]


class Stats(ctypes.Structure):
    _fields_ = [("snapshots", ctypes.c_uint64), ("snapshot_bytes", ctypes.c_uint64),
                ("recoveries", ctypes.c_uint64), ("recovered_bytes", ctypes.c_uint64),
                ("verify_failures", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64)]


class Forward(ctypes.Structure):
    _fields_ = [("origin", Role), ("pad_", ctypes.c_uint16), ("holder_node", ctypes.c_uint32),
                ("dest_node", ctypes.c_uint32), ("holder_dp", ctypes.c_uint32)]


class RedundantSource(ctypes.Structure):
    _fields_ = [("target", Role), ("source", Role)]


class HeartbeatSlot(ctypes.Structure):  # ffx_heartbeat_slot
    _fields_ = [("enrolled", ctypes.c_uint32), ("failed", ctypes.c_uint32), ("last_seen_ns", ctypes.c_int64),
                ("last_iteration", ctypes.c_uint64)]


class PreloadState(ctypes.Structure):  # ffx_preload_state
    _fields_ = [("capacity", ctypes.c_uint64), ("bytes", ctypes.c_uint64), ("entries", ctypes.c_uint64),
                ("oldest", ctypes.c_uint64), ("fetched", ctypes.c_uint64), ("taken", ctypes.c_uint64)]


class RecoveryPlanC(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_uint32), ("capacity", ctypes.c_uint32),
                ("resume_iteration", ctypes.c_uint64),
                ("failed_pods", ctypes.POINTER(ctypes.c_uint32)),
                ("failed_roles", ctypes.POINTER(Role)),
                ("lazy_backup_targets", ctypes.POINTER(Role)),
                ("forwards", ctypes.POINTER(Forward)),
                ("redundant_from", ctypes.POINTER(RedundantSource)),
                ("n_failed_pods", ctypes.c_uint32), ("n_failed_roles", ctypes.c_uint32),
                ("n_lazy", ctypes.c_uint32), ("n_forwards", ctypes.c_uint32),
                ("n_redundant", ctypes.c_uint32)]


_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_U32 = ctypes.c_uint32
_I = ctypes.c_int
_U8P = ctypes.c_char_p

# name -> (restype, argtypes)
SIGNATURES = {
    "ffx_status_str": (ctypes.c_char_p, [_I]),
    "ffx_last_error": (ctypes.c_char_p, []),
    "ffx_abi_version": (_I, []),
    "ffx_role_of": (_I, [ctypes.POINTER(ClusterSpec), _U32, ctypes.POINTER(Role)]),
    "ffx_index_of": (_I, [ctypes.POINTER(ClusterSpec), Role, ctypes.POINTER(_U32)]),
    "ffx_node_of": (_I, [ctypes.POINTER(ClusterSpec), Role, ctypes.POINTER(_U32)]),
    "ffx_dp_neighbor": (_I, [ctypes.POINTER(ClusterSpec), Role, ctypes.POINTER(Role)]),
    "ffx_dp_predecessor": (_I, [ctypes.POINTER(ClusterSpec), Role, ctypes.POINTER(Role)]),
    "ffx_plan_recovery": (_I, [ctypes.POINTER(ClusterSpec), ctypes.POINTER(_U32), _U32,
                               ctypes.POINTER(Role), _U32, _U64, _U64, _U32,
                               ctypes.POINTER(RecoveryPlanC)]),
    "ffx_razor": (_I, [ctypes.POINTER(ClusterSpec), ctypes.POINTER(UniquenessPlan)]),
    "ffx_weights_bytes": (_U64, [ctypes.POINTER(ClusterSpec)]),
    "ffx_optimizer_bytes": (_U64, [ctypes.POINTER(ClusterSpec)]),
    "ffx_version_for_target": (_I, [_U64, _U64, ctypes.POINTER(_I)]),
    "ffx_pack_header": (_I, [Role, _U64, ctypes.c_uint8, _U64, _U64, _P]),
    "ffx_parse_header": (_I, [_P, _U64, ctypes.POINTER(BlobInfo)]),
    "ffx_checksum64": (_I, [_P, _U64, ctypes.POINTER(_U64), _P]),
    "ffx_slice_checksums": (_I, [_P, _U64, _U64, _P, _P]),
    "ffx_copy_checksums": (_I, [_P, _P, _U64, _U64, _P, _P]),
    "ffx_copy_verify": (_I, [_P, _P, _U64, _U64, _P, _P, _P]),
    "ffx_copy": (_I, [_P, _P, _U64, _U32, _P]),
    "ffx_expand": (_I, [_P, _P, _U64, _P]),
    "ffx_materialize": (_I, [_P, _P, _U64, _P]),
    "ffx_blob_check": (_I, [_P, _U64, ctypes.POINTER(_U64), _P]),
    "ffx_prepare_peers": (_I, [_I, ctypes.POINTER(_U32)]),
    "ffx_device_alloc": (_I, [_I, _U64, ctypes.POINTER(_P)]),
    "ffx_device_free": (_I, [_I, _P]),
    "ffx_memcpy": (_I, [_P, _P, _U64, _P, _I]),
    "ffx_pointer_is_device": (_I, [_P, ctypes.POINTER(_I)]),
    "ffx_stream_sync": (_I, [_P]),
    "ffx_open": (_I, [_I, ctypes.POINTER(ClusterSpec), Role, _U64, ctypes.POINTER(_P)]),
    "ffx_close": (_I, [_P]),
    "ffx_register_region": (_I, [_P, _I, _P, _U64, _I]),
    "ffx_clear_regions": (_I, [_P]),
    "ffx_plan": (_I, [_P, ctypes.POINTER(PlanInfo)]),
    "ffx_slice_runs": (_I, [ctypes.POINTER(_U64), _U32, _U64, ctypes.POINTER(SliceRun), _U32, ctypes.POINTER(_U32)]),
    "ffx_replica_create": (_I, [_P, Role, _U64, _U32, ctypes.POINTER(_P)]),
    "ffx_replica_export": (_I, [_P, _P]),
    "ffx_replica_open": (_I, [_P, _P, ctypes.POINTER(_P)]),
    "ffx_replica_destroy": (_I, [_P]),
    "ffx_replica_slots": (_I, [_P, ctypes.POINTER(_U32)]),
    "ffx_replica_slot_regions": (_I, [_P, _U32, ctypes.POINTER(_U32), ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(_U64)]),
    "ffx_replica_slot_info": (_I, [_P, _U32, ctypes.POINTER(SlotInfo)]),
    "ffx_replica_newest": (_I, [_P, ctypes.POINTER(_U64)]),
    "ffx_replica_slot_ptrs": (_I, [_P, _U32, ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "ffx_replica_rollback": (_I, [_P, _U64, ctypes.POINTER(_U32)]),
    "ffx_replica_clear": (_I, [_P]),
    "ffx_replica_export_frame": (_I, [_P, _U64, _P, _U64, ctypes.POINTER(_U64), _P]),
    "ffx_replica_export_frame_part": (_I, [_P, _U64, _U32, _P, _U64, ctypes.POINTER(_U64),
                                           ctypes.POINTER(_U32), _P]),
    "ffx_snapshot_target": (_I, [_P, _P]),
    "ffx_snapshot": (_I, [_P, _U64, _P, ctypes.POINTER(SnapshotOpts)]),
    "ffx_snapshot_target2": (_I, [_P, _P]),
    "ffx_mcast_supported": (_I, [_I, ctypes.POINTER(_I)]),
    "ffx_sched_create": (_I, [_P, ctypes.POINTER(SchedOpts), ctypes.POINTER(_P)]),
    "ffx_sched_begin": (_I, [_P, _U64]),
    "ffx_sched_gap": (_I, [_P, _I, _P]),
    "ffx_sched_finish": (_I, [_P, _P]),
    "ffx_sched_destroy": (_I, [_P]),
    "ffx_replica_create_tiered": (_I, [_P, Role, _U64, _U32, _U64, ctypes.POINTER(_P)]),
    "ffx_replica_tiers": (_I, [_P, ctypes.POINTER(_U64), ctypes.POINTER(_U64)]),
    "ffx_replica_create_shared": (_I, [_P, Role, _U64, _U32, ctypes.POINTER(_P)]),
    "ffx_mcast_create": (_I, [_P, _U64, _U32, _U32, ctypes.POINTER(_P)]),
    "ffx_mcast_export": (_I, [_P, _P]),
    "ffx_mcast_open": (_I, [_P, _P, ctypes.POINTER(_P)]),
    "ffx_mcast_join": (_I, [_P]),
    "ffx_mcast_bind": (_I, [_P, _P]),
    "ffx_snapshot_target_mcast": (_I, [_P, _P, _P]),
    "ffx_mcast_destroy": (_I, [_P]),
    "ffx_regions_export": (_I, [_P, _P]),
    "ffx_remote_open": (_I, [_P, _P, ctypes.POINTER(_P)]),
    "ffx_remote_close": (_I, [_P]),
    "ffx_snapshot_pull": (_I, [_P, _P, _P, _U64, _P, ctypes.POINTER(SnapshotOpts)]),
    "ffx_snapshot_begin_pull": (_I, [_P, _P, _P, _U64, ctypes.POINTER(SnapshotOpts), ctypes.POINTER(_U32)]),
    "ffx_snapshot_wait_pulled": (_I, [_P, _U64, _P]),
    "ffx_snapshot_ack_reset": (_I, [_P, _P]),
    "ffx_snapshot_begin": (_I, [_P, _U64, ctypes.POINTER(SnapshotOpts), ctypes.POINTER(_U32)]),
    "ffx_snapshot_next": (_I, [_P, _P, _P, ctypes.POINTER(_U32)]),
    "ffx_snapshot_next_kind": (_I, [_P, _I, _P, _P, ctypes.POINTER(_U32)]),
    "ffx_snapshot_read_sums": (_I, [_P, _P, _U64, ctypes.POINTER(_U64), _P]),
    "ffx_snapshot_batch_span": (_I, [_P, _U32, ctypes.POINTER(_U64), ctypes.POINTER(_U64)]),
    "ffx_snapshot_from_host": (_I, [_P, _U64, _P, _U64, _U32, _P]),
    "ffx_replica_verify": (_I, [_P, _P, _U64, _U32, _P, ctypes.POINTER(RecoverReport)]),
    "ffx_recover": (_I, [_P, _P, _U64, _P, ctypes.POINTER(RecoverReport)]),
    "ffx_recover_full": (_I, [_P, ctypes.POINTER(_P), _U32, _U64, ctypes.POINTER(PeerRegion), _U32, _P,
                              ctypes.POINTER(RecoverReport)]),
    "ffx_recover_from": (_I, [_P, ctypes.POINTER(_P), _U32, _U64, _P, ctypes.POINTER(RecoverReport)]),
    "ffx_recover_region": (_I, [_P, ctypes.POINTER(PeerRegion), _P, ctypes.POINTER(RecoverReport)]),
    "ffx_ipc_export": (_I, [_P, _P]),
    "ffx_ipc_open": (_I, [_P, ctypes.POINTER(_P)]),
    "ffx_ipc_close": (_I, [_P]),
    "ffx_inject": (_I, [_P, _I, _P, _U64]),
    "ffx_get_stats": (_I, [_P, ctypes.POINTER(Stats)]),
    "ffx_now_ns": (ctypes.c_int64, []),
    "ffx_preload_create": (_I, [_P, _U64, ctypes.POINTER(_P)]),
    "ffx_preload_destroy": (_I, [_P]),
    "ffx_preload_fits": (_I, [_P, _U64, ctypes.POINTER(_I)]),
    "ffx_preload_fetch_host": (_I, [_P, _U64, _P, _U64, _P, _P]),
    "ffx_preload_fetch_synthetic": (_I, [_P, _U64, _P, _U32, _U32, _P, _P]),
    "ffx_preload_take": (_I, [_P, _U64, _P, ctypes.POINTER(_P), ctypes.POINTER(_U64)]),
    "ffx_preload_free": (_I, [_P, _P, _P]),
    "ffx_preload_info": (_I, [_P, ctypes.POINTER(PreloadState)]),
    "ffx_fold_of_blob": (_I, [_P, _U64, _U32, ctypes.POINTER(_U64), _P]),
    "ffx_sched_preload_host": (_I, [_P, _P, _U64, _P, _U64]),
    "ffx_sched_preload_synthetic": (_I, [_P, _P, _U64, _P, _U32, _U32]),
    "ffx_sched_preload_pending": (_I, [_P, ctypes.POINTER(_U32)]),
    "ffx_heartbeats_create": (_I, [_U32, ctypes.c_int64, _U32, ctypes.POINTER(_P)]),
    "ffx_heartbeats_destroy": (_I, [_P]),
    "ffx_heartbeats_enroll": (_I, [_P, _U32, _U64, ctypes.c_int64]),
    "ffx_heartbeats_observe": (_I, [_P, _U32, _U64, ctypes.c_int64]),
    "ffx_heartbeats_sweep": (_I, [_P, ctypes.c_int64, ctypes.POINTER(_U32), _U32, ctypes.POINTER(_U32)]),
    "ffx_heartbeats_mark_failed": (_I, [_P, _U32]),
    "ffx_heartbeats_query": (_I, [_P, _U32, ctypes.POINTER(HeartbeatSlot)]),
    "ffx_heartbeats_counters": (_I, [_P, ctypes.POINTER(_U64), ctypes.POINTER(_U64), ctypes.POINTER(_U64)]),
    "ffx_ledger_create": (_I, [ctypes.POINTER(ClusterSpec), ctypes.POINTER(_P)]),
    "ffx_ledger_destroy": (_I, [_P]),
    "ffx_ledger_record": (_I, [_P, Role, _U64]),
    "ffx_ledger_global_consistent": (_U64, [_P]),
    "ffx_ledger_group_latest": (_U64, [_P, _U32]),
    "ffx_ledger_worker_latest": (_U64, [_P, Role]),
    "ffx_ledger_rebase": (_I, [_P, _U64]),
    "ffx_ledger_record_replica": (_I, [_P, _P, ctypes.POINTER(_U64)]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError("libffx.so not built at %s: run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (no CPU fallback exists)" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ffx_abi_version() != ABI_VERSION:
        raise ImportError("libffx ABI %d != %d" % (lib.ffx_abi_version(), ABI_VERSION))
    return lib


lib = _load()


def check(status: int, what: str = ""):
    if status != OK:
        msg = lib.ffx_last_error().decode(errors="replace")
        raise _EXC.get(status, FfxError)("%s: %s" % (what or lib.ffx_status_str(status).decode(), msg))


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


def _ptr(t) -> int:
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    return t.data_ptr()


# ---- host-side functions (no GPU needed) -----------------------------------

def razor(spec: ClusterSpec) -> UniquenessPlan:
    p = UniquenessPlan()
    check(lib.ffx_razor(ctypes.byref(spec), ctypes.byref(p)), "razor")
    return p


def weights_bytes(spec: ClusterSpec) -> int:
    return lib.ffx_weights_bytes(ctypes.byref(spec))


def optimizer_bytes(spec: ClusterSpec) -> int:
    return lib.ffx_optimizer_bytes(ctypes.byref(spec))


def version_for_target(held: int, target: int) -> int:
    out = ctypes.c_int()
    check(lib.ffx_version_for_target(held, target, ctypes.byref(out)), "version_for_target")
    return out.value


def role_of(spec, idx) -> Role:
    r = Role()
    check(lib.ffx_role_of(ctypes.byref(spec), idx, ctypes.byref(r)), "role_of")
    return r


def index_of(spec, role) -> int:
    o = ctypes.c_uint32()
    check(lib.ffx_index_of(ctypes.byref(spec), role, ctypes.byref(o)), "index_of")
    return o.value


def node_of(spec, role) -> int:
    o = ctypes.c_uint32()
    check(lib.ffx_node_of(ctypes.byref(spec), role, ctypes.byref(o)), "node_of")
    return o.value


def dp_neighbor(spec, role) -> Role:
    r = Role()
    check(lib.ffx_dp_neighbor(ctypes.byref(spec), role, ctypes.byref(r)), "dp_neighbor")
    return r


def dp_predecessor(spec, role) -> Role:
    r = Role()
    check(lib.ffx_dp_predecessor(ctypes.byref(spec), role, ctypes.byref(r)), "dp_predecessor")
    return r


def pack_header(role: Role, iteration: int, kind: int, length: int, checksum: int) -> bytes:
    out = ctypes.create_string_buffer(32)
    check(lib.ffx_pack_header(role, iteration, kind, length, checksum, out), "pack_header")
    return out.raw


def parse_header(header: bytes, framed_len: int = 0) -> BlobInfo:
    info = BlobInfo()
    buf = ctypes.create_string_buffer(bytes(header[:32]).ljust(32, b"\0"), 32)
    check(lib.ffx_parse_header(buf, framed_len, ctypes.byref(info)), "parse_header")
    return info


@dataclass
class RecoveryPlan:
    kind: str
    resume_iteration: int
    failed_pods: list
    failed_roles: list
    lazy_backup_targets: list
    forwards: list       # (origin Role, holder_node, dest_node, holder_dp)
    redundant_from: list  # (target Role, source Role)


def plan_recovery(spec, failed_pods: Sequence[int], failed_roles: Sequence, global_consistent: int,
                  latest_fallback_round: int, replicas: int = 1) -> RecoveryPlan:
    cap = max(spec.num_nodes * spec.gpus_per_node, len(failed_roles) + 1, 1) + len(failed_pods) * spec.gpus_per_node
    pods = (ctypes.c_uint32 * cap)()
    roles_out = (Role * cap)()
    lazy = (Role * cap)()
    fwd = (Forward * cap)()
    red = (RedundantSource * cap)()
    p = RecoveryPlanC()
    p.capacity = cap
    p.failed_pods = pods
    p.failed_roles = roles_out
    p.lazy_backup_targets = lazy
    p.forwards = fwd
    p.redundant_from = red
    in_pods = (ctypes.c_uint32 * max(1, len(failed_pods)))(*failed_pods)
    rl = [r if isinstance(r, Role) else Role(*r) for r in failed_roles]
    in_roles = (Role * max(1, len(rl)))(*rl)
    check(lib.ffx_plan_recovery(ctypes.byref(spec), in_pods, len(failed_pods), in_roles, len(rl),
                                global_consistent, latest_fallback_round, replicas, ctypes.byref(p)),
          "plan_recovery")
    cp = lambda r: Role(r.dp, r.pp, r.tp)
    return RecoveryPlan(
        kind="neighbor" if p.kind == 0 else "fallback",
        resume_iteration=p.resume_iteration,
        failed_pods=[pods[i] for i in range(p.n_failed_pods)],
        failed_roles=[cp(roles_out[i]) for i in range(p.n_failed_roles)],
        lazy_backup_targets=[cp(lazy[i]) for i in range(p.n_lazy)],
        forwards=[(cp(fwd[i].origin), fwd[i].holder_node, fwd[i].dest_node, fwd[i].holder_dp)
                  for i in range(p.n_forwards)],
        redundant_from=[(cp(red[i].target), cp(red[i].source)) for i in range(p.n_redundant)],
    )


# ---- controller state (controller.cpp:16-121; host-only, no GPU) -----------

SECOND_NS = 1_000_000_000  # rt::kSecond


def now_ns() -> int:
    return lib.ffx_now_ns()


class Heartbeats:
    """ctl::HeartbeatTable (controller.hpp:56-101) over ffx_heartbeats_*.
    Defaults = ControllerConfig (1 s interval, 3 misses)."""

    def __init__(self, pods: int, interval_ns: int = SECOND_NS, miss_threshold: int = 3):
        self.pods = pods
        self._h = ctypes.c_void_p()
        check(lib.ffx_heartbeats_create(pods, interval_ns, miss_threshold, ctypes.byref(self._h)),
              "heartbeats_create")

    def enroll(self, node: int, iteration: int, now: int):
        check(lib.ffx_heartbeats_enroll(self._h, node, iteration, now), "heartbeats_enroll")

    def observe(self, node: int, iteration: int, now: int):
        check(lib.ffx_heartbeats_observe(self._h, node & 0xFFFFFFFF, iteration, now), "heartbeats_observe")

    def sweep(self, now: int) -> list:
        out = (_U32 * max(1, self.pods))()
        n = _U32()
        check(lib.ffx_heartbeats_sweep(self._h, now, out, self.pods, ctypes.byref(n)), "heartbeats_sweep")
        return [out[i] for i in range(n.value)]

    def mark_failed(self, node: int):
        check(lib.ffx_heartbeats_mark_failed(self._h, node), "heartbeats_mark_failed")

    def _slot(self, node):
        s = HeartbeatSlot()
        check(lib.ffx_heartbeats_query(self._h, node, ctypes.byref(s)), "heartbeats_query")
        return s

    def enrolled(self, node: int) -> bool:
        return 0 <= node < self.pods and bool(self._slot(node).enrolled)

    def failed(self, node: int) -> bool:
        return 0 <= node < self.pods and bool(self._slot(node).failed)

    def last_iteration(self, node: int) -> int:
        return self._slot(node).last_iteration

    def last_seen(self, node: int) -> int:
        return self._slot(node).last_seen_ns

    def counters(self):
        u, l, r = _U64(), _U64(), _U64()
        check(lib.ffx_heartbeats_counters(self._h, ctypes.byref(u), ctypes.byref(l), ctypes.byref(r)),
              "heartbeats_counters")
        return u.value, l.value, r.value

    def unknown_reports(self) -> int:
        return self.counters()[0]

    def late_reports(self) -> int:
        return self.counters()[1]

    def regressions(self) -> int:
        return self.counters()[2]

    def destroy(self):
        if self._h:
            lib.ffx_heartbeats_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    __del__ = destroy


class Ledger:
    """ctl::IterationLedger (controller.hpp:106-130) over ffx_ledger_*."""

    def __init__(self, spec: ClusterSpec):
        self._h = ctypes.c_void_p()
        check(lib.ffx_ledger_create(ctypes.byref(spec), ctypes.byref(self._h)), "ledger_create")

    def record(self, role, iteration: int):
        r = role if isinstance(role, Role) else Role(*role)
        check(lib.ffx_ledger_record(self._h, r, iteration), "ledger_record")

    def record_replica(self, held: "Replica") -> int:
        """CkptRecord after a completed replica (wire.hpp:85-90); returns the
        iteration recorded (0: nothing committed yet)."""
        it = _U64()
        check(lib.ffx_ledger_record_replica(self._h, held.ptr, ctypes.byref(it)), "ledger_record_replica")
        return it.value

    def global_consistent(self) -> int:
        return lib.ffx_ledger_global_consistent(self._h)

    def group_latest(self, dp_group: int) -> int:
        return lib.ffx_ledger_group_latest(self._h, dp_group)

    def worker_latest(self, role) -> int:
        r = role if isinstance(role, Role) else Role(*role)
        return lib.ffx_ledger_worker_latest(self._h, r)

    def rebase(self, iteration: int):
        check(lib.ffx_ledger_rebase(self._h, iteration), "ledger_rebase")

    def destroy(self):
        if self._h:
            lib.ffx_ledger_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    __del__ = destroy


# ---- device primitives ------------------------------------------------------

def checksum64(dev_tensor, nbytes: Optional[int] = None, stream=None) -> int:
    n = dev_tensor.numel() * dev_tensor.element_size() if nbytes is None else nbytes
    out = ctypes.c_uint64()
    check(lib.ffx_checksum64(_ptr(dev_tensor), n, ctypes.byref(out), _stream_ptr(stream)), "checksum64")
    return out.value


def slice_runs(region_bytes: Sequence[int], slice_bytes: int) -> list:
    """The payload's checksum-slice runs, in table order (ffx_slice_runs):
    [(region, offset, bytes, slice_bytes, first_slice), ...]."""
    n = len(region_bytes)
    arr = (_U64 * max(1, n))(*region_bytes)
    out = (SliceRun * (n + 1))()
    cnt = _U32()
    check(lib.ffx_slice_runs(arr, n, slice_bytes, out, n + 1, ctypes.byref(cnt)), "slice_runs")
    return [(r.region, r.offset, r.bytes, r.slice_bytes, r.first_slice) for r in out[:cnt.value]]


def slice_index(runs: list, region: int, offset: int) -> int:
    """Checksum-table index of the slice holding byte `offset` of `region`."""
    for reg, off, nb, sl, first in runs:
        if reg == region and off <= offset < off + max(nb, 1):
            return first + (offset - off) // sl
    raise ValueError(f"offset {offset} outside region {region}")


def slice_checksums(dev_tensor, slice_bytes: int, out_tensor, nbytes=None, stream=None):
    n = dev_tensor.numel() * dev_tensor.element_size() if nbytes is None else nbytes
    check(lib.ffx_slice_checksums(_ptr(dev_tensor), n, slice_bytes, _ptr(out_tensor),
                                  _stream_ptr(stream)), "slice_checksums")


def copy_checksums(dst, src, slice_bytes: int, out_tensor, nbytes=None, stream=None):
    n = src.numel() * src.element_size() if nbytes is None else nbytes
    check(lib.ffx_copy_checksums(_ptr(dst), _ptr(src), n, slice_bytes, _ptr(out_tensor),
                                 _stream_ptr(stream)), "copy_checksums")


def copy_verify(dst, src, slice_bytes: int, expected, result, nbytes=None, stream=None):
    n = src.numel() * src.element_size() if nbytes is None else nbytes
    check(lib.ffx_copy_verify(_ptr(dst), _ptr(src), n, slice_bytes, _ptr(expected), _ptr(result),
                              _stream_ptr(stream)), "copy_verify")


def materialize(dst, digest: bytes, nbytes: Optional[int] = None, stream=None):
    n = dst.numel() * dst.element_size() if nbytes is None else nbytes
    check(lib.ffx_materialize(_ptr(dst), bytes(digest), n, _stream_ptr(stream)), "materialize")


def expand(dst, digest: bytes, nbytes: Optional[int] = None, stream=None):
    n = dst.numel() * dst.element_size() if nbytes is None else nbytes
    check(lib.ffx_expand(_ptr(dst), bytes(digest), n, _stream_ptr(stream)), "expand")


def blob_first_bad(dev, nbytes: Optional[int] = None, stream=None) -> int:
    n = dev.numel() * dev.element_size() if nbytes is None else nbytes
    out = ctypes.c_uint64()
    check(lib.ffx_blob_check(_ptr(dev), n, ctypes.byref(out), _stream_ptr(stream)), "blob_check")
    return out.value


def blob_is_sound(dev, nbytes=None, stream=None) -> bool:
    n = dev.numel() * dev.element_size() if nbytes is None else nbytes
    return n >= 32 and blob_first_bad(dev, n, stream) == U64_MAX


def ipc_export(ptr: int) -> bytes:
    h = ctypes.create_string_buffer(64)
    check(lib.ffx_ipc_export(ptr, h), "ipc_export")
    return h.raw


def ipc_open(handle: bytes) -> int:
    p = ctypes.c_void_p()
    check(lib.ffx_ipc_open(ctypes.create_string_buffer(bytes(handle), 64), ctypes.byref(p)), "ipc_open")
    return p.value


def ipc_close(ptr: int):
    check(lib.ffx_ipc_close(ptr), "ipc_close")


# ---- context / replica objects -------------------------------------------------

class Replica:
    """A neighbour replica (holder-side NeighborBuffer, ckpt.hpp:105-120)."""

    def __init__(self, handle_ptr: int, owner: "Context"):
        self._h = ctypes.c_void_p(handle_ptr)
        self._owner = owner

    @property
    def ptr(self):
        return self._h

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(HANDLE_BYTES)
        check(lib.ffx_replica_export(self._h, buf), "replica_export")
        return buf.raw

    def versions(self) -> int:
        v = ctypes.c_uint32()
        check(lib.ffx_replica_slots(self._h, ctypes.byref(v)), "replica_slots")
        return v.value

    def slot_info(self, slot: int) -> SlotInfo:
        s = SlotInfo()
        check(lib.ffx_replica_slot_info(self._h, slot, ctypes.byref(s)), "slot_info")
        return s

    def slot_regions(self, slot: int):
        """[(region kind, bytes)] of the committed snapshot in `slot`."""
        n = _U32()
        kinds = (ctypes.c_int32 * 16)()
        sizes = (_U64 * 16)()
        check(lib.ffx_replica_slot_regions(self._h, slot, ctypes.byref(n), kinds, sizes), "slot_regions")
        return [(int(kinds[i]), int(sizes[i])) for i in range(n.value)]

    def newest(self) -> Optional[int]:
        it = ctypes.c_uint64()
        st = lib.ffx_replica_newest(self._h, ctypes.byref(it))
        if st == ERESTORE:
            return None
        check(st, "replica_newest")
        return it.value

    def held(self) -> dict:
        """{iteration: slot} for committed slots."""
        out = {}
        for v in range(self.versions()):
            s = self.slot_info(v)
            if s.state == SLOT_COMMITTED:
                out[s.iteration] = v
        return out

    def slot_ptrs(self, slot: int):
        pay, sums = ctypes.c_void_p(), ctypes.c_void_p()
        check(lib.ffx_replica_slot_ptrs(self._h, slot, ctypes.byref(pay), ctypes.byref(sums)), "slot_ptrs")
        return pay.value, sums.value

    def clear(self):
        check(lib.ffx_replica_clear(self._h), "replica_clear")

    def tiers(self):
        """(bytes in HBM, bytes in host memory) of this replica's range."""
        a, b = _U64(), _U64()
        check(lib.ffx_replica_tiers(self._h, ctypes.byref(a), ctypes.byref(b)), "replica_tiers")
        return a.value, b.value

    def rollback(self, iteration: int) -> int:
        """Drop slots newer than `iteration` (ffx_replica_rollback); returns
        how many.  Writers re-arm their target afterwards (set_target)."""
        n = _U32()
        check(lib.ffx_replica_rollback(self._h, iteration, ctypes.byref(n)), "replica_rollback")
        return n.value

    def export_frame(self, iteration: int, stream=None) -> bytes:
        n = ctypes.c_uint64()
        check(lib.ffx_replica_export_frame(self._h, iteration, None, 0, ctypes.byref(n),
                                           _stream_ptr(stream)), "export_frame")
        buf = ctypes.create_string_buffer(n.value)
        check(lib.ffx_replica_export_frame(self._h, iteration, buf, n.value, ctypes.byref(n),
                                           _stream_ptr(stream)), "export_frame")
        return buf.raw

    def export_frame_parts(self, iteration: int, stream=None):
        """Every SNP1 frame of the snapshot at `iteration` (several above the
        4 GiB SNP1 limit), as bytes objects."""
        n, parts = ctypes.c_uint64(), ctypes.c_uint32()
        check(lib.ffx_replica_export_frame_part(self._h, iteration, 0, None, 0, ctypes.byref(n),
                                                ctypes.byref(parts), _stream_ptr(stream)), "export_frame_part")
        out = []
        for i in range(parts.value):
            check(lib.ffx_replica_export_frame_part(self._h, iteration, i, None, 0, ctypes.byref(n), None,
                                                    _stream_ptr(stream)), "export_frame_part")
            buf = ctypes.create_string_buffer(n.value)
            check(lib.ffx_replica_export_frame_part(self._h, iteration, i, buf, n.value, ctypes.byref(n), None,
                                                    _stream_ptr(stream)), "export_frame_part")
            out.append(buf.raw)
        return out

    def destroy(self):
        if self._h:
            check(lib.ffx_replica_destroy(self._h), "replica_destroy")
            self._h = ctypes.c_void_p(0)


class Mcast:
    """An NVSwitch multicast range over one origin's replica slots on its
    dp+1 and dp+2 holders (double neighbour with one egress per tile)."""

    def __init__(self, handle_ptr: int):
        self._h = ctypes.c_void_p(handle_ptr)

    @property
    def ptr(self):
        return self._h

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(MCAST_HANDLE_BYTES)
        check(lib.ffx_mcast_export(self._h, buf), "mcast_export")
        return buf.raw

    def join(self):
        check(lib.ffx_mcast_join(self._h), "mcast_join")

    def bind(self, held: "Replica"):
        check(lib.ffx_mcast_bind(self._h, held.ptr), "mcast_bind")

    def destroy(self):
        if self._h:
            check(lib.ffx_mcast_destroy(self._h), "mcast_destroy")
            self._h = ctypes.c_void_p(0)


def mcast_supported(device: int = 0) -> bool:
    v = _I()
    check(lib.ffx_mcast_supported(device, ctypes.byref(v)), "mcast_supported")
    return bool(v.value)


class Sched:
    """The native slice scheduler (ffx_sched_*): one snapshot batch per gap
    the training step reports."""

    def __init__(self, ctx: "Context", policy: int, link_gaps: int, sm_gaps: int = 0, copy_ctas: int = 0,
                 hash_ctas: int = 0, gap_ms=None, task_ctas: bool = False):
        o = SchedOpts()
        o.policy, o.link_gaps, o.sm_gaps = policy, link_gaps, sm_gaps
        o.copy_ctas, o.hash_ctas = copy_ctas, hash_ctas
        o.task_ctas = int(task_ctas)
        if gap_ms is not None:
            self._gaps = (ctypes.c_double * len(gap_ms))(*gap_ms)
            o.gap_ms = self._gaps
        self._h = ctypes.c_void_p()
        self._ctx = ctx
        check(lib.ffx_sched_create(ctx.ptr, ctypes.byref(o), ctypes.byref(self._h)), "sched_create")

    def begin(self, iteration: int):
        check(lib.ffx_sched_begin(self._h, iteration), "sched_begin")

    def gap(self, kind: int, train_stream=None):
        check(lib.ffx_sched_gap(self._h, kind, _stream_ptr(train_stream)), "sched_gap")

    def finish(self, train_stream=None):
        check(lib.ffx_sched_finish(self._h, _stream_ptr(train_stream)), "sched_finish")

    def preload_host(self, preload: "Preload", iteration: int, host_tensor):
        """Queue a fetch of pinned host bytes for the next link-idle gap."""
        preload._keep[iteration] = host_tensor  # must outlive the copy
        check(lib.ffx_sched_preload_host(self._h, preload._h, iteration, host_tensor.data_ptr(),
                                         host_tensor.numel() * host_tensor.element_size()), "sched_preload_host")

    def preload_synthetic(self, preload: "Preload", iteration: int, item_digests: bytes, sample_bytes: int):
        check(lib.ffx_sched_preload_synthetic(self._h, preload._h, iteration, item_digests, len(item_digests) // 32,
                                              sample_bytes), "sched_preload_synthetic")

    def preload_pending(self) -> int:
        n = _U32()
        check(lib.ffx_sched_preload_pending(self._h, ctypes.byref(n)), "sched_preload_pending")
        return n.value

    def destroy(self):
        if self._h:
            check(lib.ffx_sched_destroy(self._h), "sched_destroy")
            self._h = ctypes.c_void_p(0)


def data_item_digests(seed: int, first: int, count: int) -> bytes:
    """data_item_digest(seed, first + i) for a window (evolution.cpp:112-114):
    SHA-256 of HashIn{}.str("D").u64(seed).u64(index) -- 32-byte keys on the
    host, as the reference computes them (OpenSSL); the sample bytes are then
    generated on the device (Preload.fetch_synthetic)."""
    import hashlib
    import struct
    head = struct.pack("<Q", 1) + b"D" + struct.pack("<Q", seed)
    return b"".join(hashlib.sha256(head + struct.pack("<Q", first + i)).digest() for i in range(count))


def fold_of_blob(dev, bytes_per_sample: int, nbytes=None, stream=None) -> int:
    """data::fold_of_blob (dataloader.cpp:150-164) on the device."""
    out = _U64()
    n = nbytes if nbytes is not None else dev.numel() * dev.element_size()
    check(lib.ffx_fold_of_blob(_ptr(dev), n, bytes_per_sample, ctypes.byref(out), _stream_ptr(stream)),
          "fold_of_blob")
    return out.value


class Preload:
    """data::PreloadBuffer in HBM (dataloader.hpp:45-73) over ffx_preload_*."""

    def __init__(self, ctx: "Context", capacity_bytes: int):
        self._h = ctypes.c_void_p()
        self._keep = {}
        check(lib.ffx_preload_create(ctx.ptr, capacity_bytes, ctypes.byref(self._h)), "preload_create")

    def fits(self, nbytes: int) -> bool:
        v = _I()
        check(lib.ffx_preload_fits(self._h, nbytes, ctypes.byref(v)), "preload_fits")
        return bool(v.value)

    def fetch_host(self, iteration: int, host_tensor, stream=None, gate_event=None):
        self._keep[iteration] = host_tensor
        check(lib.ffx_preload_fetch_host(self._h, iteration, host_tensor.data_ptr(),
                                         host_tensor.numel() * host_tensor.element_size(), _stream_ptr(stream),
                                         gate_event.cuda_event if gate_event is not None else None),
              "preload_fetch_host")

    def fetch_synthetic(self, iteration: int, item_digests: bytes, sample_bytes: int, stream=None, gate_event=None):
        check(lib.ffx_preload_fetch_synthetic(self._h, iteration, item_digests, len(item_digests) // 32,
                                              sample_bytes, _stream_ptr(stream),
                                              gate_event.cuda_event if gate_event is not None else None),
              "preload_fetch_synthetic")

    def take(self, iteration: int, consumer_stream=None):
        """-> (device pointer, bytes); the caller frees it with free()."""
        p, n = ctypes.c_void_p(), _U64()
        check(lib.ffx_preload_take(self._h, iteration, _stream_ptr(consumer_stream), ctypes.byref(p),
                                   ctypes.byref(n)), "preload_take")
        self._keep.pop(iteration, None)
        return p.value, n.value

    def free(self, dev_ptr: int, consumer_stream=None):
        check(lib.ffx_preload_free(self._h, dev_ptr, _stream_ptr(consumer_stream)), "preload_free")

    def info(self) -> PreloadState:
        st = PreloadState()
        check(lib.ffx_preload_info(self._h, ctypes.byref(st)), "preload_info")
        return st

    def destroy(self):
        if self._h:
            check(lib.ffx_preload_destroy(self._h), "preload_destroy")
            self._h = ctypes.c_void_p(0)


class Remote:
    """An origin rank's regions mapped into a holder (pull mode)."""

    def __init__(self, handle_ptr: int):
        self._h = ctypes.c_void_p(handle_ptr)

    @property
    def ptr(self):
        return self._h

    def close(self):
        if self._h:
            check(lib.ffx_remote_close(self._h), "remote_close")
            self._h = ctypes.c_void_p(0)


class Context:
    """One rank's ffx context: state registry, snapshot issue, recovery."""

    def __init__(self, device: int, spec: ClusterSpec, role, slice_bytes: int = 4096):
        self.spec = spec
        self.role = role if isinstance(role, Role) else Role(*role)
        self.device = device
        self._c = ctypes.c_void_p()
        self._keep = []  # tensors whose memory is registered
        check(lib.ffx_open(device, ctypes.byref(spec), self.role, slice_bytes, ctypes.byref(self._c)), "open")

    @property
    def ptr(self):
        return self._c

    def close(self):
        if self._c:
            check(lib.ffx_close(self._c), "close")
            self._c = ctypes.c_void_p(0)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def register(self, kind: int, tensor, unique: bool = True, nbytes: Optional[int] = None):
        n = tensor.numel() * tensor.element_size() if nbytes is None else nbytes
        check(lib.ffx_register_region(self._c, kind, _ptr(tensor), n, int(unique)), "register_region")
        self._keep.append(tensor)

    def clear_regions(self):
        check(lib.ffx_clear_regions(self._c), "clear_regions")
        self._keep.clear()

    def plan(self) -> PlanInfo:
        p = PlanInfo()
        check(lib.ffx_plan(self._c, ctypes.byref(p)), "plan")
        return p

    def create_replica(self, origin, capacity: int, versions: int = 2) -> Replica:
        origin = origin if isinstance(origin, Role) else Role(*origin)
        h = ctypes.c_void_p()
        check(lib.ffx_replica_create(self._c, origin, capacity, versions, ctypes.byref(h)), "replica_create")
        return Replica(h.value, self)

    def create_shared_replica(self, origin, capacity: int, versions: int = 2) -> Replica:
        """A replica that can be bound to an NVSwitch multicast range."""
        origin = origin if isinstance(origin, Role) else Role(*origin)
        h = ctypes.c_void_p()
        check(lib.ffx_replica_create_shared(self._c, origin, capacity, versions, ctypes.byref(h)),
              "replica_create_shared")
        return Replica(h.value, self)

    def create_tiered_replica(self, origin, capacity: int, versions: int, hbm_bytes: int) -> Replica:
        """A replica whose first hbm_bytes live in HBM and the rest in pinned
        host memory (ffx_replica_create_tiered)."""
        origin = origin if isinstance(origin, Role) else Role(*origin)
        h = ctypes.c_void_p()
        check(lib.ffx_replica_create_tiered(self._c, origin, capacity, versions, hbm_bytes, ctypes.byref(h)),
              "replica_create_tiered")
        return Replica(h.value, self)

    def create_mcast(self, capacity: int, versions: int = 2, members: int = 3) -> Mcast:
        h = ctypes.c_void_p()
        check(lib.ffx_mcast_create(self._c, capacity, versions, members, ctypes.byref(h)), "mcast_create")
        return Mcast(h.value)

    def open_mcast(self, handle: bytes) -> Mcast:
        h = ctypes.c_void_p()
        check(lib.ffx_mcast_open(self._c, ctypes.create_string_buffer(bytes(handle), MCAST_HANDLE_BYTES),
                                 ctypes.byref(h)), "mcast_open")
        return Mcast(h.value)

    def set_target_mcast(self, mc: Mcast, view: Replica):
        check(lib.ffx_snapshot_target_mcast(self._c, mc.ptr, view.ptr), "snapshot_target_mcast")

    def open_replica(self, handle: bytes) -> Replica:
        h = ctypes.c_void_p()
        check(lib.ffx_replica_open(self._c, ctypes.create_string_buffer(bytes(handle), HANDLE_BYTES),
                                   ctypes.byref(h)), "replica_open")
        return Replica(h.value, self)

    def set_target(self, replica: Optional[Replica]):
        check(lib.ffx_snapshot_target(self._c, replica.ptr if replica else None), "snapshot_target")

    # ---- pull mode -------------------------------------------------------------
    def export_regions(self) -> bytes:
        buf = ctypes.create_string_buffer(REGIONS_HANDLE_BYTES)
        check(lib.ffx_regions_export(self._c, buf), "regions_export")
        return buf.raw

    def open_remote(self, handle: bytes) -> "Remote":
        h = ctypes.c_void_p()
        check(lib.ffx_remote_open(self._c, ctypes.create_string_buffer(bytes(handle), REGIONS_HANDLE_BYTES),
                                  ctypes.byref(h)), "remote_open")
        return Remote(h.value)

    def snapshot_pull(self, origin: "Remote", held: Replica, iteration: int, stream=None, max_ctas: int = 0,
                      batches: int = 1):
        o = SnapshotOpts()
        o.max_ctas = max_ctas
        o.batches = batches
        check(lib.ffx_snapshot_pull(self._c, origin.ptr, held.ptr, iteration, _stream_ptr(stream),
                                    ctypes.byref(o)), "snapshot_pull")

    def wait_pulled(self, iteration: int, stream=None):
        check(lib.ffx_snapshot_wait_pulled(self._c, iteration, _stream_ptr(stream)), "snapshot_wait_pulled")

    def ack_reset(self, stream=None):
        """Drop an un-consumed pull ack (rollback): see ffx_snapshot_ack_reset."""
        check(lib.ffx_snapshot_ack_reset(self._c, _stream_ptr(stream)), "snapshot_ack_reset")

    def set_target2(self, replica: Optional[Replica]):
        check(lib.ffx_snapshot_target2(self._c, replica.ptr if replica else None), "snapshot_target2")

    def snapshot(self, iteration: int, stream=None, max_ctas: int = 0, batches: int = 1,
                 gate_events=None, verify_on_store: bool = False, weights_kind: bool = False,
                 split: bool = False, hash_batches: int = 0, hash_ctas: int = 0, copy_engine: bool = False,
                 fused_permille: int = 0, task_ctas: bool = False):
        o = SnapshotOpts()
        o.task_ctas = int(task_ctas)
        o.split = int(split)
        o.fused_permille = fused_permille
        o.hash_batches = hash_batches
        o.hash_ctas = hash_ctas
        o.copy_engine = int(copy_engine)
        o.max_ctas = max_ctas
        o.batches = batches
        o.verify_on_store = int(verify_on_store)
        o.weights_kind = int(weights_kind)
        arr = None
        if gate_events:
            arr = (ctypes.c_void_p * len(gate_events))(*[e.cuda_event if hasattr(e, "cuda_event") else e
                                                          for e in gate_events])
            o.gate_events = ctypes.cast(arr, ctypes.c_void_p)
        check(lib.ffx_snapshot(self._c, iteration, _stream_ptr(stream), ctypes.byref(o)), "snapshot")

    def snapshot_begin(self, iteration: int, batches: int = 1, max_ctas: int = 0,
                       verify_on_store: bool = False, split: bool = False, hash_batches: int = 0,
                       hash_ctas: int = 0, copy_engine: bool = False, batch_weights=None,
                       fused_permille: int = 0, task_ctas: bool = False) -> int:
        o = SnapshotOpts()
        o.task_ctas = int(task_ctas)
        o.fused_permille = fused_permille
        if batch_weights is not None:
            self._weights = (ctypes.c_double * len(batch_weights))(*batch_weights)  # kept alive
            o.batch_weights = self._weights
        o.max_ctas = max_ctas
        o.batches = batches
        o.verify_on_store = int(verify_on_store)
        o.split = int(split)
        o.hash_batches = hash_batches
        o.hash_ctas = hash_ctas
        o.copy_engine = int(copy_engine)
        n = ctypes.c_uint32()
        check(lib.ffx_snapshot_begin(self._c, iteration, ctypes.byref(o), ctypes.byref(n)), "snapshot_begin")
        return n.value

    def snapshot_next(self, stream=None, gate_event=None, kind: Optional[int] = None) -> int:
        """Issue the next batch (of `kind` under the split policy); returns how
        many batches of that kind (or in total, kind=None) remain."""
        left = ctypes.c_uint32()
        ev = None
        if gate_event is not None:
            ev = gate_event.cuda_event if hasattr(gate_event, "cuda_event") else gate_event
        if kind is None:
            check(lib.ffx_snapshot_next(self._c, _stream_ptr(stream), ev, ctypes.byref(left)), "snapshot_next")
        else:
            check(lib.ffx_snapshot_next_kind(self._c, kind, _stream_ptr(stream), ev, ctypes.byref(left)),
                  "snapshot_next_kind")
        return left.value

    def batch_span(self, batch: int):
        """Logical payload bytes [lo, hi) fused batch `batch` of the pending snapshot reads."""
        lo, hi = _U64(), _U64()
        check(lib.ffx_snapshot_batch_span(self._c, batch, ctypes.byref(lo), ctypes.byref(hi)), "batch_span")
        return lo.value, hi.value

    def snapshot_from_host(self, iteration: int, host_tensor, nbytes: Optional[int] = None, batches: int = 0,
                           stream=None):
        """HostSnapshots::take from host memory: H2D into the registered regions,
        pipelined under the snapshot batches (ffx_snapshot_from_host)."""
        n = host_tensor.numel() * host_tensor.element_size() if nbytes is None else nbytes
        check(lib.ffx_snapshot_from_host(self._c, iteration, _ptr(host_tensor), n, batches, _stream_ptr(stream)),
              "snapshot_from_host")

    def read_sums(self, host_tensor, stream=None) -> int:
        """D2H of the last snapshot's checksum table into a (pinned) int64 tensor."""
        n = ctypes.c_uint64()
        check(lib.ffx_snapshot_read_sums(self._c, _ptr(host_tensor), host_tensor.numel(), ctypes.byref(n),
                                         _stream_ptr(stream)), "snapshot_read_sums")
        return n.value

    def verify_held(self, held: Replica, iteration: int, max_ctas: int = 0, stream=None) -> RecoverReport:
        """Holder-side checksum-as-landed of a committed slot (ffx_replica_verify)."""
        rep = RecoverReport()
        check(lib.ffx_replica_verify(self._c, held.ptr, iteration, max_ctas, _stream_ptr(stream),
                                     ctypes.byref(rep)), "replica_verify")
        return rep

    def recover(self, replica: Replica, target: int, stream=None) -> RecoverReport:
        rep = RecoverReport()
        check(lib.ffx_recover(self._c, replica.ptr, target, _stream_ptr(stream), ctypes.byref(rep)), "recover")
        return rep

    def recover_full(self, replicas, target: int, redundant=(), stream=None) -> RecoverReport:
        """Full-state restore: unique regions from the replica holders, redundant
        regions [(region_index, peer_ptr, peer_sums_ptr[, table_slice_bytes])]
        from live peers, one kernel."""
        rep = RecoverReport()
        arr = (ctypes.c_void_p * max(1, len(replicas)))(*[r.ptr.value for r in replicas])
        red = (PeerRegion * max(1, len(redundant)))(*[PeerRegion(e[0], e[3] if len(e) > 3 else 0, e[1], e[2])
                                                      for e in redundant])
        check(lib.ffx_recover_full(self._c, arr, len(replicas), target, red, len(redundant),
                                   _stream_ptr(stream), ctypes.byref(rep)), "recover_full")
        return rep

    def recover_from(self, replicas, target: int, stream=None) -> RecoverReport:
        """Parallel gather of one snapshot from several holders."""
        rep = RecoverReport()
        arr = (ctypes.c_void_p * len(replicas))(*[r.ptr.value for r in replicas])
        check(lib.ffx_recover_from(self._c, arr, len(replicas), target, _stream_ptr(stream), ctypes.byref(rep)),
              "recover_from")
        return rep

    def recover_region(self, index: int, peer_src: int, peer_sums: int, stream=None,
                       slice_bytes: int = 0) -> RecoverReport:
        rep = RecoverReport()
        pr = PeerRegion(index, slice_bytes, peer_src, peer_sums)
        check(lib.ffx_recover_region(self._c, ctypes.byref(pr), _stream_ptr(stream), ctypes.byref(rep)),
              "recover_region")
        return rep

    def inject(self, fault: int, replica: Optional[Replica] = None, arg: int = 0):
        check(lib.ffx_inject(self._c, fault, replica.ptr if replica else None, arg), "inject")

    def stats(self) -> Stats:
        s = Stats()
        check(lib.ffx_get_stats(self._c, ctypes.byref(s)), "stats")
        return s
