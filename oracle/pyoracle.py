"""Python handle on the CPU oracle (TEST INFRASTRUCTURE ONLY).

Loads oracle/liboracle.so (the C restatement, ffx_oracle.c) and, when built,
oracle/_ref/libftsim_ref.so (the reference itself).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may
import this module; the product path never does.

plan_recovery below is a small pure-Python restatement of
proj/src/controller.cpp:144-209 used as the oracle for ffx_plan_recovery.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libftsim_ref.so")

_u64 = ctypes.c_uint64
_P = ctypes.c_void_p


def _load_oracle():
    lib = ctypes.CDLL(ORACLE_SO)
    sig = {
        "orc_fnv1a64": (_u64, [_P, _u64]),
        "orc_fnv1a64_from": (_u64, [_u64, _P, _u64]),
        "orc_slice_fnv": (_u64, [_P, _u64, _u64, _P]),
        "orc_fold64": (_u64, [_P]),
        "orc_mix64": (_u64, [_u64]),
        "orc_expand": (None, [_P, _u64, _P]),
        "orc_materialize": (ctypes.c_int, [_P, _u64, _P]),
        "orc_blob_is_sound": (ctypes.c_int, [_P, _u64]),
        "orc_weights_bytes": (_u64, [_u64]),
        "orc_optimizer_bytes": (_u64, [_u64, ctypes.c_uint32, ctypes.c_int]),
        "orc_razor": (_u64, [_u64, ctypes.c_uint32, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
        "orc_version_for_target": (ctypes.c_int, [_u64, _u64]),
        "orc_pack_header": (ctypes.c_int, [ctypes.c_uint16] * 3 + [_u64, ctypes.c_uint8, _u64, _u64, _P]),
        "orc_pack_blob": (ctypes.c_int, [ctypes.c_uint16] * 3 + [_u64, ctypes.c_uint8, _P, _u64, _P]),
        "orc_unpack": (ctypes.c_int, [_P, _u64, ctypes.POINTER(_u64)]),
        "orc_sha256": (ctypes.c_int, [_P, _u64, _P]),
        "orc_weights_init": (None, [_u64, ctypes.c_uint16, ctypes.c_uint16, _P]),
        "orc_optimizer_init": (None, [_u64] + [ctypes.c_uint16] * 3 + [ctypes.c_int, _P]),
        "orc_state_next": (None, [ctypes.c_char_p, _P, _P, _P]),
        "orc_materialize_range": (ctypes.c_int, [_P, _u64, _u64, _u64, _P]),
        "orc_item_fold": (_u64, [_u64, _u64]),
        "orc_window_fold": (_u64, [_u64, _u64, ctypes.c_uint32]),
        "orc_optimizer_at": (ctypes.c_int, [_u64] + [ctypes.c_uint16] * 3 + [ctypes.c_uint32] * 4
                             + [_u64, ctypes.c_int, _P]),
    }
    for n, (r, a) in sig.items():
        f = getattr(lib, n)
        f.restype = r
        f.argtypes = a
    return lib


lib = _load_oracle()


def _buf(n):
    return ctypes.create_string_buffer(max(n, 1))


def fnv1a64(data: bytes) -> int:
    return lib.orc_fnv1a64(data, len(data))


def slice_fnv(data: bytes, slice_bytes: int):
    n = (len(data) + slice_bytes - 1) // slice_bytes
    out = (ctypes.c_uint64 * max(n, 1))()
    lib.orc_slice_fnv(data, len(data), slice_bytes, out)
    return [out[i] for i in range(n)]


def expand(digest: bytes, n: int) -> bytes:
    b = _buf(n)
    lib.orc_expand(digest, n, b)
    return b.raw[:n]


def materialize(digest: bytes, n: int) -> bytes:
    b = _buf(n)
    if lib.orc_materialize(digest, n, b) != 0:
        raise ValueError("state blob smaller than its digest prefix")
    return b.raw[:n]


def materialize_range(digest: bytes, total: int, lo: int, n: int) -> bytes:
    b = _buf(n)
    if lib.orc_materialize_range(digest, total, lo, n, b) != 0:
        raise ValueError("range outside blob")
    return b.raw[:n]


def blob_is_sound(blob: bytes) -> bool:
    return bool(lib.orc_blob_is_sound(blob, len(blob)))


def optimizer_init(seed, dp, pp, tp, distributed=True) -> bytes:
    b = _buf(32)
    lib.orc_optimizer_init(seed, dp, pp, tp, int(distributed), b)
    return b.raw[:32]


def optimizer_at(seed, dp, pp, tp, n, d, p=1, t=1, batch=256, distributed=True) -> bytes:
    """Optimizer digest of rank (dp,pp,tp) after n iterations:
    optimizer_next over the grad digest of the rank's data window."""
    b = _buf(32)
    if lib.orc_optimizer_at(seed, dp, pp, tp, d, p, t, batch, n, int(distributed), b) != 0:
        raise ValueError("batch size must divide evenly over the workers")
    return b.raw[:32]


def weights_init(seed, pp, tp) -> bytes:
    b = _buf(32)
    lib.orc_weights_init(seed, pp, tp, b)
    return b.raw[:32]


def optimizer_bytes(phi, d, distributed) -> int:
    return lib.orc_optimizer_bytes(phi, d, int(distributed))


def razor(phi, d, distributed):
    fl = (ctypes.c_int * 2)()
    u = lib.orc_razor(phi, d, int(distributed), fl)
    return bool(fl[0]), bool(fl[1]), u


def version_for_target(held, target):
    return lib.orc_version_for_target(held, target)


def pack_header(role, iteration, kind, length, checksum) -> bytes:
    b = _buf(32)
    if lib.orc_pack_header(role[0], role[1], role[2], iteration, kind, length, checksum, b) != 0:
        raise ValueError("snapshot payload exceeds 4 GiB framing limit")
    return b.raw[:32]


def pack_blob(role, iteration, kind, payload: bytes) -> bytes:
    b = _buf(32 + len(payload))
    if lib.orc_pack_blob(role[0], role[1], role[2], iteration, kind, payload, len(payload), b) != 0:
        raise ValueError("snapshot payload exceeds 4 GiB framing limit")
    return b.raw[:32 + len(payload)]


def unpack(frame: bytes):
    f = (ctypes.c_uint64 * 7)()
    rc = lib.orc_unpack(frame, len(frame), f)
    return rc, tuple(f[i] for i in range(7))


def sha256(data: bytes) -> bytes:
    b = _buf(32)
    lib.orc_sha256(data, len(data), b)
    return b.raw[:32]


# ---- the data loader's synthetic samples (evolution.cpp:112-128, dataloader.cpp:104-164)

def data_item_digest(seed: int, index: int) -> bytes:
    """HashIn{}.str("D").u64(seed).u64(index).digest(): str = u64 length + bytes."""
    import struct
    return sha256(struct.pack("<Q", 1) + b"D" + struct.pack("<QQ", seed, index))


def data_item(seed: int, index: int, nbytes: int) -> bytes:
    return expand(data_item_digest(seed, index), nbytes)


def fetch(seed: int, first: int, count: int, sample_bytes: int) -> bytes:
    """DataServerStub::fetch in synthetic mode (dataloader.cpp:119-127)."""
    return b"".join(data_item(seed, first + i, sample_bytes) for i in range(count))


def fold_of_blob(blob: bytes, bytes_per_sample: int) -> int:
    """dataloader.cpp:150-164."""
    if bytes_per_sample == 0 or len(blob) % bytes_per_sample:
        raise ValueError("blob is not a whole number of samples")
    n = min(8, bytes_per_sample)
    acc = 0
    for off in range(0, len(blob), bytes_per_sample):
        acc = (acc + int.from_bytes(blob[off:off + n], "little")) & (2**64 - 1)
    return acc


def ref_lib():
    """The reference library itself, or None when not built (GPU box w/o build)."""
    if not os.path.exists(REF_SO):
        return None
    r = ctypes.CDLL(REF_SO)
    r.ref_checksum64.restype = _u64
    r.ref_checksum64.argtypes = [_P, _u64]
    r.ref_materialize.restype = ctypes.c_int
    r.ref_materialize.argtypes = [_P, _u64, _P]
    r.ref_ring_setup.restype = _P
    r.ref_ring_setup.argtypes = [ctypes.c_int, _u64]
    r.ref_ring_run.restype = ctypes.c_int
    r.ref_ring_run.argtypes = [_P, _u64, ctypes.POINTER(ctypes.c_double)]
    r.ref_ring_free.argtypes = [_P]
    r.ref_optimizer_init.argtypes = [_u64, ctypes.c_uint16, ctypes.c_uint16, ctypes.c_uint16, ctypes.c_int, _P]
    r.ref_optimizer_at.restype = ctypes.c_int
    r.ref_optimizer_at.argtypes = [_u64] + [ctypes.c_uint16] * 3 + [ctypes.c_uint32] * 4 + [_u64, ctypes.c_int, _P]
    if hasattr(r, "ref_hs_create"):  # ckpt::HostSnapshots / NeighborBuffer (ckpt.cpp:35-105)
        u16 = ctypes.c_uint16
        r.ref_hs_create.restype = _P
        r.ref_hs_create.argtypes = [u16, u16, u16, _u64]
        r.ref_hs_free.argtypes = [_P]
        r.ref_hs_take.argtypes = [_P, _u64, _P, _u64]
        r.ref_hs_newest.argtypes = [_P, ctypes.POINTER(_u64)]
        r.ref_hs_previous.argtypes = [_P, ctypes.POINTER(_u64)]
        r.ref_hs_framed.restype = _u64
        r.ref_hs_framed.argtypes = [_P, _u64, _P, _u64]
        r.ref_nb_create.restype = _P
        r.ref_nb_create.argtypes = [u16, u16, u16]
        r.ref_nb_free.argtypes = [_P]
        r.ref_nb_store.argtypes = [_P, _P, _u64]
        r.ref_nb_newest.argtypes = [_P, ctypes.POINTER(_u64)]
        r.ref_nb_framed_at.restype = _u64
        r.ref_nb_framed_at.argtypes = [_P, _u64, _P, _u64]
    if hasattr(r, "ref_hb_create"):  # controller state machines (controller.cpp:16-121, :144-209)
        i64, u32, u16 = ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint16
        r.ref_hb_create.restype = _P
        r.ref_hb_create.argtypes = [u32, i64, u32]
        r.ref_hb_free.argtypes = [_P]
        r.ref_hb_enroll.argtypes = [_P, u32, _u64, i64]
        r.ref_hb_observe.argtypes = [_P, u32, _u64, i64]
        r.ref_hb_sweep.restype = u32
        r.ref_hb_sweep.argtypes = [_P, i64, ctypes.POINTER(u32), u32]
        r.ref_hb_mark_failed.argtypes = [_P, u32]
        r.ref_hb_query.argtypes = [_P, u32, ctypes.POINTER(i64)]
        r.ref_hb_counters.argtypes = [_P, ctypes.POINTER(_u64)]
        r.ref_ledger_create.restype = _P
        r.ref_ledger_create.argtypes = [u32] * 5
        r.ref_ledger_free.argtypes = [_P]
        r.ref_ledger_record.argtypes = [_P, u16, u16, u16, _u64]
        r.ref_ledger_global.restype = _u64
        r.ref_ledger_global.argtypes = [_P]
        r.ref_ledger_group.restype = _u64
        r.ref_ledger_group.argtypes = [_P, u32]
        r.ref_ledger_worker.restype = _u64
        r.ref_ledger_worker.argtypes = [_P, u16, u16, u16]
        r.ref_ledger_rebase.argtypes = [_P, _u64]
        r.ref_fetch.argtypes = [_u64, _u64, u32, u32, _P]
        r.ref_fold_of_blob.argtypes = [_P, _u64, u32, ctypes.POINTER(_u64)]
        r.ref_plan_recovery.restype = ctypes.c_long
        r.ref_plan_recovery.argtypes = [u32] * 5 + [ctypes.c_int, _u64, ctypes.POINTER(u32), u32,
                                                    ctypes.POINTER(u16), u32, _u64, _u64,
                                                    ctypes.POINTER(i64), ctypes.c_long]
    return r


def ref_plan_recovery(r, nodes, gpn, d, p, t, distributed, phi, failed_pods, failed_roles,
                      global_consistent, latest_fallback):
    """The reference's own ctl::plan_recovery through ref_shim, decoded into
    the dict layout of plan_recovery() below."""
    pods = (ctypes.c_uint32 * max(1, len(failed_pods)))(*failed_pods)
    flat = [x for role in failed_roles for x in role]
    roles = (ctypes.c_uint16 * max(1, len(flat)))(*flat)
    cap = 64 + 16 * (nodes * gpn + len(failed_roles) + len(failed_pods) * gpn)
    out = (ctypes.c_int64 * cap)()
    n = r.ref_plan_recovery(nodes, gpn, d, p, t, int(distributed), phi, pods, len(failed_pods), roles,
                            len(failed_roles), global_consistent, latest_fallback, out, cap)
    if n < 0:
        raise RuntimeError("reference plan_recovery threw")
    w = list(out[:n])
    pos = 2

    def take(k):
        nonlocal pos
        cnt = w[pos]
        pos += 1
        items = [tuple(w[pos + i * k:pos + (i + 1) * k]) for i in range(cnt)]
        pos += cnt * k
        return items

    plan = {"kind": "fallback" if w[0] else "neighbor", "resume": w[1]}
    plan["failed_pods"] = [x[0] for x in take(1)]
    plan["failed_roles"] = take(3)
    plan["lazy"] = take(3)
    plan["forwards"] = [((f[0], f[1], f[2]), f[3], f[4]) for f in take(5)]
    plan["redundant_from"] = [((x[0], x[1], x[2]), (x[3], x[4], x[5])) for x in take(6)]
    return plan


# ---- controller.cpp:16-121, restated (HeartbeatTable, IterationLedger) ------

class HeartbeatTable:
    """controller.cpp:16-77: one slot per pod; sweep declares pods silent for
    more than interval * miss_threshold."""

    def __init__(self, pods, interval=1_000_000_000, miss_threshold=3):
        self.slots = [dict(enrolled=False, failed=False, last_seen=0, last_iteration=0) for _ in range(pods)]
        self.limit = interval * miss_threshold
        self.unknown = self.late = self.regressed = 0

    def enroll(self, node, it, now):  # :21-28 (slots_.at)
        s = self.slots[node]
        s.update(enrolled=True, failed=False, last_seen=now, last_iteration=it)

    def observe(self, node, it, now):  # :30-44
        if node >= len(self.slots) or not self.slots[node]["enrolled"]:
            self.unknown += 1
            return
        s = self.slots[node]
        if s["failed"]:
            self.late += 1
            return
        if it < s["last_iteration"]:
            self.regressed += 1
        s.update(last_iteration=it, last_seen=now)

    def sweep(self, now):  # :46-58
        dead = []
        for i, s in enumerate(self.slots):
            if not s["enrolled"] or s["failed"]:
                continue
            if now - s["last_seen"] > self.limit:
                s["failed"] = True
                dead.append(i)
        return dead

    def mark_failed(self, node):  # :60-62
        self.slots[node]["failed"] = True


class IterationLedger:
    """controller.cpp:81-121: per-worker latest recoverable iteration; the
    global consistent one is the minimum over world_size() workers."""

    def __init__(self, nodes, gpn, d, p, t):
        self.world, self.d, self.p, self.t = nodes * gpn, d, p, t
        self.latest = {}

    def record(self, role, it):  # :83-90 (ProtocolError -> ValueError)
        dp, pp, tp = role
        if dp >= self.d or pp >= self.p or tp >= self.t:
            raise ValueError("role outside the grid")
        self.latest[role] = max(self.latest.get(role, 0), it)

    def global_consistent(self):  # :92-97
        if len(self.latest) < self.world:
            return 0
        return min(self.latest.values())

    def group_latest(self, g):  # :99-110
        pp, tp = (g // self.t) & 0xFFFF, (g % self.t) & 0xFFFF
        vals = [self.latest.get((dp, pp, tp), 0) for dp in range(self.d)]
        return min(vals) if vals else 0

    def worker_latest(self, role):  # :112-115
        return self.latest.get(tuple(role), 0)

    def rebase(self, it):  # :117-121
        for dp in range(self.d):
            for pp in range(self.p):
                for tp in range(self.t):
                    self.latest[(dp, pp, tp)] = it


# ---- controller.cpp:144-209, restated (small cases only) ---------------------

def role_of(idx, d, p, t):
    return (idx // (t * p), (idx // t) % p, idx % t)


def index_of(role, p, t):
    return (role[0] * p + role[1]) * t + role[2]


def plan_recovery(d, p, t, gpus_per_node, distributed, failed_pods, failed_roles,
                  global_consistent, latest_fallback, phi=1):
    pods = sorted(set(failed_pods))
    lost = set(tuple(r) for r in failed_roles)
    for pod in pods:
        for lr in range(gpus_per_node):
            lost.add(role_of(pod * gpus_per_node + lr, d, p, t))
    lost = sorted(lost)
    nb = lambda r: ((r[0] + 1) % d, r[1], r[2])
    neighbor_ok = d > 1 and not any(nb(f) in lost for f in lost)
    wr, orr, unique = razor(phi, d, distributed)
    plan = {"kind": "neighbor" if neighbor_ok else "fallback", "failed_pods": pods,
            "failed_roles": lost, "forwards": [], "redundant_from": [], "lazy": []}
    if not neighbor_ok:
        plan["resume"] = latest_fallback
        return plan
    plan["resume"] = global_consistent
    if global_consistent == 0:
        return plan
    node = lambda r: index_of(r, p, t) // gpus_per_node
    for f in lost:
        if unique > 0:
            plan["forwards"].append((f, node(nb(f)), node(f)))
        if wr or orr:
            for dp in range(d):
                c = (dp, f[1], f[2])
                if c not in lost:
                    plan["redundant_from"].append((f, c))
                    break
    if wr or orr:
        for pp in range(p):
            for tp in range(t):
                for dp in range(d):
                    c = (dp, pp, tp)
                    if c not in lost:
                        plan["lazy"].append(c)
                        break
    return plan
