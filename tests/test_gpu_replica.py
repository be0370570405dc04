"""GPU parity of the replica manager, snapshot and recovery (single process).

Restates the hot-path cases of proj/tests/test_ckpt.cpp against the B200
path: two-version retention and replace-in-place (:198-263), capacity
ConfigError (:220-221), header-only frames (:222-226), SNP1 frame bytes
(:50-72), and ring restore with its failure modes (:278-330) -- missing,
stale, wrong origin, flipped byte -- plus the B200-specific faults (torn slot,
corrupted checksum table).  Frames are compared byte for byte with the
oracle's pack_blob; restored state with the oracle's materialize.
"""
import os

import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def host(t):
    return bytes(t.cpu().numpy().tobytes())


def spec2(ffx, phi=64, d=2):
    return ffx.make_spec(d=d, phi=phi, distributed=True)


def blob_for(ffx, dp, nbytes, seed=42):
    d = orc.optimizer_init(seed, dp, 0, 0, True)
    t = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    ffx.materialize(t, d)
    return t, orc.materialize(d, nbytes)


def ring_pair(ffx, nbytes, slice_bytes=4096, versions=2):
    """origin d1 snapshots into a replica held by d0's context (one GPU)."""
    spec = spec2(ffx)
    holder = ffx.Context(0, spec, (0, 0, 0), slice_bytes)
    origin = ffx.Context(0, spec, (1, 0, 0), slice_bytes)
    rep = holder.create_replica((1, 0, 0), max(nbytes, 1), versions)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    return spec, holder, origin, rep, view


def test_snapshot_roundtrip_frame_is_reference_bytes(ffx):
    n = 100_003
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    origin.snapshot(9)
    torch.cuda.synchronize()
    s = rep.slot_info(0)
    assert s.state == ffx.SLOT_COMMITTED and s.iteration == 9 and s.payload_len == n
    assert s.role.tuple() == (1, 0, 0) and s.kind == 1
    pay, sums = rep.slot_ptrs(0)
    # payload bytes and slice table
    frame = rep.export_frame(9)
    assert frame == orc.pack_blob((1, 0, 0), 9, 1, want)
    assert rep.slot_info(0).whole_checksum == orc.fnv1a64(want)
    # second export is served from the cached checksum
    assert rep.export_frame(9) == frame


def test_two_version_rule_and_replace_in_place(ffx):
    # proj/tests/test_ckpt.cpp:198-216, :229-263
    n = 8192
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    state = torch.zeros(n, dtype=torch.uint8, device="cuda")
    origin.register(ffx.REGION_BLOB, state)
    payloads = {}
    for it in (1, 2, 3, 4, 5):
        state.fill_(it)
        payloads[it] = bytes([it]) * n
        origin.snapshot(it)
    torch.cuda.synchronize()
    assert rep.newest() == 5
    assert sorted(rep.held()) == [4, 5]
    assert rep.export_frame(4)[32:] == payloads[4]
    with pytest.raises(ffx.RestoreError):
        rep.export_frame(3)
    slot5 = rep.held()[5]
    state.fill_(55)
    origin.snapshot(5)  # replace-in-place keeps iteration 4
    torch.cuda.synchronize()
    assert rep.held() == {4: 1 - slot5, 5: slot5}
    assert rep.export_frame(5)[32:] == bytes([55]) * n
    assert rep.export_frame(4)[32:] == payloads[4]


@pytest.mark.parametrize("dual", [False, True])
def test_replace_older_iteration_keeps_insertion_order(ffx, dual):
    # ckpt.cpp:46-52 / :86-92: re-taking the OLDER held iteration swaps its
    # bytes but leaves it first in the deque, so take(1) take(2) take(1)
    # take(3) keeps {2, 3} and newest() stays 2 after the re-take.
    n = 8192
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    rep2 = view2 = None
    if dual:
        rep2 = holder.create_replica((1, 0, 0), n, 2)
        view2 = origin.open_replica(rep2.export())
        origin.set_target2(view2)
    state = torch.zeros(n, dtype=torch.uint8, device="cuda")
    origin.register(ffx.REGION_BLOB, state)
    for it, fill in ((1, 1), (2, 2), (1, 11)):
        state.fill_(fill)
        origin.snapshot(it)
    torch.cuda.synchronize()
    for r in [rep] + ([rep2] if dual else []):
        assert r.newest() == 2
        assert sorted(r.held()) == [1, 2]
        assert r.export_frame(1)[32:] == bytes([11]) * n
    state.fill_(3)
    origin.snapshot(3)
    torch.cuda.synchronize()
    for r in [rep] + ([rep2] if dual else []):
        assert sorted(r.held()) == [2, 3]
        assert r.newest() == 3
        assert r.export_frame(2)[32:] == bytes([2]) * n


def test_capacity_config_error(ffx):
    # proj/tests/test_ckpt.cpp:220-221
    spec, holder, origin, rep, view = ring_pair(ffx, 16)
    big = torch.zeros(17, dtype=torch.uint8, device="cuda")
    origin.register(ffx.REGION_BLOB, big)
    with pytest.raises(ffx.ConfigError):
        origin.snapshot(7)


def test_header_only_snapshot(ffx):
    # proj/tests/test_ckpt.cpp:222-226: a zero-byte plan produces header-only frames
    spec = ffx.make_spec(d=2, phi=64, distributed=False)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    rep = holder.create_replica((1, 0, 0), 0, 2)
    origin.set_target(origin.open_replica(rep.export()))
    origin.snapshot(1)
    torch.cuda.synchronize()
    fr = rep.export_frame(1)
    assert fr == orc.pack_blob((1, 0, 0), 1, 1, b"")
    assert len(fr) == 32


def test_multi_region_state_roundtrip(ffx):
    # fp32 master + Adam m/v shards + cursor + RNG state, ragged sizes
    spec, holder, origin, rep, view = ring_pair(ffx, 1 << 20)
    g = torch.Generator(device="cuda").manual_seed(1)
    master = torch.randn(40_001, device="cuda", generator=g)
    m = torch.randn(40_001, device="cuda", generator=g)
    v = torch.rand(40_001, device="cuda", generator=g)
    cursor = torch.tensor([1234, 5678], dtype=torch.int64, device="cuda")
    rng = torch.randint(0, 2**31, (4,), dtype=torch.int32, device="cuda", generator=g)
    regions = [(ffx.REGION_MASTER, master), (ffx.REGION_ADAM_M, m), (ffx.REGION_ADAM_V, v),
               (ffx.REGION_CURSOR, cursor), (ffx.REGION_RNG, rng)]
    for k, t in regions:
        origin.register(k, t)
    weights = torch.randn(1000, device="cuda", generator=g).to(torch.bfloat16)
    origin.register(ffx.REGION_PARAMS, weights, unique=False)
    plan = origin.plan()
    concat = b"".join(host(t) for _, t in regions)
    assert plan.registered_unique_bytes == len(concat)
    assert plan.registered_redundant_bytes == 2000
    assert plan.num_unique_regions == 5 and plan.num_regions == 6
    origin.snapshot(3)
    torch.cuda.synchronize()
    assert rep.export_frame(3) == orc.pack_blob((1, 0, 0), 3, 1, concat)
    saved = [t.clone() for _, t in regions]
    origin.inject(ffx.FAULT_POISON_STATE)
    assert not torch.equal(master, saved[0])
    rpt = origin.recover(view, 3)
    assert rpt.bad_slices == 0 and rpt.bytes == len(concat)
    for (_, t), s in zip(regions, saved):
        assert torch.equal(t, s)


def test_recover_bit_exact_and_failure_modes(ffx):
    # proj/tests/test_ckpt.cpp:278-330
    n = 3 * (1 << 20) + 1001
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    origin.snapshot(8)
    origin.snapshot(9)
    torch.cuda.synchronize()
    origin.inject(ffx.FAULT_POISON_STATE)
    assert not ffx.blob_is_sound(state)
    rpt = origin.recover(view, 9)
    assert host(state) == want and ffx.blob_is_sound(state)
    assert rpt.bytes == n and rpt.bad_slices == 0 and rpt.seconds > 0

    # missing iteration
    with pytest.raises(ffx.RestoreError, match="missing"):
        origin.recover(view, 7)
    # wrong worker: a context for d0 must not accept d1's snapshot
    other = ffx.Context(0, spec, (0, 0, 0))
    t0 = torch.empty(n, dtype=torch.uint8, device="cuda")
    other.register(ffx.REGION_BLOB, t0)
    with pytest.raises(ffx.RestoreError, match="d1p0t0"):
        other.recover(view, 9)
    # layout mismatch
    other2 = ffx.Context(0, spec, (1, 0, 0))
    t1 = torch.empty(n - 1, dtype=torch.uint8, device="cuda")
    other2.register(ffx.REGION_BLOB, t1)
    with pytest.raises(ffx.RestoreError):
        other2.recover(view, 9)
    # flipped payload byte -> the slice that holds it is named
    slot9 = rep.held()[9]
    off = 4096 * 300 + 17
    origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (slot9 << 48) | off)
    with pytest.raises(ffx.RestoreError, match="checksum mismatch"):
        origin.recover(view, 9)
    origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (slot9 << 48) | off)  # flip back
    origin.recover(view, 9)
    # corrupted checksum table entry
    origin.inject(ffx.FAULT_CORRUPT_SUMS, view, (slot9 << 48) | 5)
    with pytest.raises(ffx.RestoreError):
        origin.recover(view, 9)
    origin.inject(ffx.FAULT_CORRUPT_SUMS, view, (slot9 << 48) | 5)
    # torn slot (origin died mid-snapshot): iteration 8 still recoverable
    slot8 = rep.held()[8]
    origin.inject(ffx.FAULT_TEAR_SLOT, view, slot9)
    with pytest.raises(ffx.RestoreError, match="torn"):
        origin.recover(view, 9)
    assert rep.newest() == 8
    origin.recover(view, 8)
    assert ffx.blob_is_sound(state)


def test_recover_reports_first_bad_slice(ffx):
    n = 1 << 20
    spec, holder, origin, rep, view = ring_pair(ffx, n, slice_bytes=4096)
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    origin.snapshot(1)
    torch.cuda.synchronize()
    origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (0 << 48) | (4096 * 100 + 1))
    origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (0 << 48) | (4096 * 40))
    rep_c = ffx.RecoverReport()
    st = ffx.lib.ffx_recover(origin.ptr, view.ptr, 1, None, ffx.ctypes.byref(rep_c))
    assert st == ffx.ERESTORE
    assert rep_c.first_bad_slice == 40 and rep_c.bad_slices == 2


def test_batched_gated_snapshot_equals_single(ffx):
    n = (1 << 22) + 77
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    side = torch.cuda.Stream(priority=0)
    low = torch.cuda.Stream(priority=0)
    events = [torch.cuda.Event() for _ in range(4)]
    for e in events:
        e.record(side)
    origin.snapshot(21, stream=low, batches=4, gate_events=events, max_ctas=16)
    low.synchronize()
    assert rep.export_frame(21) == orc.pack_blob((1, 0, 0), 21, 1, want)


def test_verify_on_store(ffx):
    n = 500_000
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    origin.snapshot(2, verify_on_store=True)
    assert origin.stats().verify_failures == 0


def test_recover_redundant_region_from_peer(ffx):
    # ckpt.cpp:150-152: weights come from a live DP peer, checksum-verified.
    n = 2 * 50_000
    spec = spec2(ffx)
    peer_w = torch.randn(50_000, device="cuda").to(torch.bfloat16)
    sums = torch.zeros((n + 4095) // 4096, dtype=torch.int64, device="cuda")
    ffx.slice_checksums(peer_w, 4096, sums)
    me = ffx.Context(0, spec, (1, 0, 0))
    mine = torch.zeros_like(peer_w)
    me.register(ffx.REGION_PARAMS, mine, unique=False)
    r = me.recover_region(0, peer_w.data_ptr(), sums.data_ptr())
    assert torch.equal(mine, peer_w) and r.bytes == n
    peer_w.view(torch.uint8)[12345] ^= 1
    with pytest.raises(ffx.RestoreError):
        me.recover_region(0, peer_w.data_ptr(), sums.data_ptr())


def test_stats_count_backup_bytes(ffx):
    n = 65536
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    state, _ = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    for it in range(5):
        origin.snapshot(it)
    torch.cuda.synchronize()
    s = origin.stats()
    assert s.snapshots == 5 and s.snapshot_bytes == 5 * n


@pytest.mark.skipif(os.environ.get("FFX_FULL_SIZE", "1") == "0", reason="full-size disabled")
def test_full_size_gpt2xl_shard_roundtrip(ffx):
    # BASELINE configs[1]: GPT-2 XL ZeRO-1 d=8 shard, N = ceil(12*1,557,611,200/8).
    spec = ffx.make_spec(d=8, phi=1_557_611_200, distributed=True)
    n = ffx.razor(spec).unique_bytes_per_device
    assert n == 2_336_416_800
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (7, 0, 0))
    rep = holder.create_replica((7, 0, 0), n, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    d = orc.optimizer_init(42, 7, 0, 0, True)
    state = torch.empty(n, dtype=torch.uint8, device="cuda")
    ffx.materialize(state, d)
    origin.register(ffx.REGION_BLOB, state)
    origin.snapshot(10)
    origin.snapshot(11)
    torch.cuda.synchronize()
    # size-independent properties: the restored blob is sound, and sampled
    # slices (bytes and table entries) equal the oracle's.
    pay, sums = rep.slot_ptrs(rep.held()[11])
    runs = ffx.slice_runs([n], 4096)  # a 48 MiB head of 1 KiB slices, then 4 KiB slices
    assert [(r[1], r[3]) for r in runs] == [(0, 1024), (48 << 20, 4096)]
    nsl = runs[-1][4] + (runs[-1][2] + 4095) // 4096
    assert rep.slot_info(rep.held()[11]).num_slices == nsl
    table = torch.empty(nsl, dtype=torch.int64, device="cuda")
    scratch = torch.empty((nsl * 8 + 4095) // 4096, dtype=torch.int64, device="cuda")
    ffx.copy_checksums(table, sums, 4096, scratch, nbytes=nsl * 8)  # device copy of the table
    tab = [v & ffx.U64_MAX for v in table.cpu().tolist()]
    origin.inject(ffx.FAULT_POISON_STATE)
    rpt = origin.recover(view, 11)
    assert rpt.bad_slices == 0 and rpt.bytes == n
    assert ffx.blob_is_sound(state)
    for _, off, nb, sl, first in runs:
        ns = (nb + sl - 1) // sl
        for s in (0, 1, 12345, ns // 2, ns - 2, ns - 1):
            lo = off + s * sl
            ln = min(sl, off + nb - lo)
            want = orc.materialize_range(d, n, lo, ln)
            assert host(state[lo:lo + ln]) == want
            assert tab[first + s] == orc.fnv1a64(want)


def test_scheduler_begin_next_gated(ffx):
    # The slice scheduler driven step by step from a training loop: each batch
    # waits on an event the "train" stream records when a gap opens.
    n = (1 << 23) + 4097
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    train = torch.cuda.Stream()
    low = torch.cuda.Stream(priority=0)
    nb = origin.snapshot_begin(30, batches=5, max_ctas=8)
    assert nb == 5
    x = torch.randn(1024, 1024, device="cuda")
    left = nb
    while left:
        with torch.cuda.stream(train):
            x = x @ x.T / 1024.0  # a "compute phase"
            ev = torch.cuda.Event()
            ev.record(train)
        left = origin.snapshot_next(stream=low, gate_event=ev)
    low.synchronize()
    assert rep.newest() == 30
    assert rep.export_frame(30) == orc.pack_blob((1, 0, 0), 30, 1, want)
    with pytest.raises(ffx.StateError):
        origin.snapshot_next(stream=low)


@pytest.mark.parametrize("copy_engine", [False, True])
def test_split_policy_copy_and_hash_batches(ffx, copy_engine):
    # Split scheduling: copy batches (TMA copy-only / copy engines) and hash
    # batches (local state -> slot table) on different streams; the slot
    # commits after both drain and is byte-identical to the fused result.
    n = (1 << 22) + 12345
    spec, holder, origin, rep, view = ring_pair(ffx, n + 4000)
    state, want = blob_for(ffx, 1, n)
    extra = torch.arange(1000, dtype=torch.int32, device="cuda")
    origin.register(ffx.REGION_BLOB, state)
    origin.register(ffx.REGION_RNG, extra)
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    origin.snapshot_begin(40, batches=3, max_ctas=4, split=True, hash_batches=5, hash_ctas=16,
                          copy_engine=copy_engine)
    left_h = left_c = 1
    while left_h or left_c:
        if left_h:
            left_h = origin.snapshot_next(stream=b, kind=ffx.BATCH_HASH)
        if left_c:
            left_c = origin.snapshot_next(stream=a, kind=ffx.BATCH_COPY)
    torch.cuda.synchronize()
    concat = want + bytes(extra.cpu().numpy().tobytes())
    assert rep.newest() == 40
    assert rep.export_frame(40) == orc.pack_blob((1, 0, 0), 40, 1, concat)
    origin.inject(ffx.FAULT_POISON_STATE)
    origin.recover(view, 40)
    assert host(state) == want
    # the blocking form interleaves copy then hash batches on one stream
    origin.snapshot(41, split=True, batches=2, hash_batches=2, max_ctas=2, copy_engine=copy_engine,
                    verify_on_store=True)
    torch.cuda.synchronize()
    assert rep.export_frame(41) == orc.pack_blob((1, 0, 0), 41, 1, concat)


@pytest.mark.parametrize("permille", [1, 300, 500, 999, 1000])
def test_hybrid_fused_share_plus_copy_engines(ffx, permille):
    # Hybrid split (opts.fused_permille): the first share of the warp tasks is
    # copied + hashed by the fused kernel, the copy engines move the rest and
    # the hash kernel checksums it; the cut falls inside and between regions.
    n = (1 << 22) + 12345
    spec, holder, origin, rep, view = ring_pair(ffx, 2 * n + 8000)
    state, want = blob_for(ffx, 1, n)
    state2, want2 = blob_for(ffx, 1, n, seed=7)
    extra = torch.arange(1000, dtype=torch.int32, device="cuda")
    origin.register(ffx.REGION_BLOB, state)
    origin.register(ffx.REGION_PARAMS, state2)
    origin.register(ffx.REGION_RNG, extra)
    a, b = torch.cuda.Stream(), torch.cuda.Stream()
    origin.snapshot_begin(50, batches=2, split=True, hash_batches=2, copy_engine=True, fused_permille=permille)
    origin.snapshot_next(stream=a, kind=ffx.BATCH_COPY)
    origin.snapshot_next(stream=b, kind=ffx.BATCH_HASH)
    origin.snapshot_next(stream=a, kind=ffx.BATCH_COPY)
    origin.snapshot_next(stream=b, kind=ffx.BATCH_HASH)
    torch.cuda.synchronize()
    concat = want + want2 + bytes(extra.cpu().numpy().tobytes())
    assert rep.newest() == 50
    assert rep.export_frame(50) == orc.pack_blob((1, 0, 0), 50, 1, concat)
    origin.inject(ffx.FAULT_POISON_STATE)
    assert origin.recover(view, 50).bad_slices == 0
    assert host(state) == want and host(state2) == want2
    # blocking form with the holder-side re-verify
    origin.snapshot(51, split=True, copy_engine=True, fused_permille=permille, verify_on_store=True)
    torch.cuda.synchronize()
    assert rep.export_frame(51) == orc.pack_blob((1, 0, 0), 51, 1, concat)
    with pytest.raises(ffx.InvalidArgument):
        origin.snapshot(52, split=True, copy_engine=False, fused_permille=permille)


@pytest.mark.parametrize("split", [False, True])
def test_double_neighbour_dual_store(ffx, split):
    # Replicas at dp+1 and dp+2: one kernel, two stores per tile.
    n = (1 << 22) + 999
    spec = ffx.make_spec(d=4, phi=64, distributed=True)
    h1 = ffx.Context(0, spec, (2, 0, 0))
    h2 = ffx.Context(0, spec, (3, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    r1 = h1.create_replica((1, 0, 0), n, 2)
    r2 = h2.create_replica((1, 0, 0), n, 2)
    v1 = origin.open_replica(r1.export())
    v2 = origin.open_replica(r2.export())
    origin.set_target(v1)
    origin.set_target2(v2)
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    for it in (5, 6, 7):
        origin.snapshot(it, split=split, batches=2, hash_batches=3)
    torch.cuda.synchronize()
    frame = orc.pack_blob((1, 0, 0), 7, 1, want)
    assert r1.export_frame(7) == frame and r2.export_frame(7) == frame
    assert sorted(r1.held()) == [6, 7] and sorted(r2.held()) == [6, 7]
    # the first holder is lost with its neighbour: recover from dp+2
    origin.inject(ffx.FAULT_POISON_STATE)
    origin.recover(v2, 7)
    assert host(state) == want


def test_ledger_records_committed_replicas_only(ffx):
    """CkptRecord after a completed replica (wire.hpp:85-90) read from the
    replica's slot headers: the holder records its origin at the newest
    COMMITTED iteration; a torn slot (origin died mid-snapshot) never counts,
    and the ledger's global consistent iteration drives the recovery target
    (controller.cpp:92-97, :144-209)."""
    n = 3 * 4096 + 11
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    spec.num_nodes, spec.gpus_per_node = 2, 1
    led = ffx.Ledger(spec)
    assert led.record_replica(rep) == 0  # nothing committed yet: no record
    assert led.worker_latest((1, 0, 0)) == 0
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    for it in (4, 5, 6):
        origin.snapshot(it)
        torch.cuda.synchronize()
        assert led.record_replica(rep) == it
    assert led.worker_latest((1, 0, 0)) == 6
    led.record((0, 0, 0), 6)
    assert led.global_consistent() == 6
    slot6 = rep.held()[6]
    origin.inject(ffx.FAULT_TEAR_SLOT, view, slot6)  # dies while writing 6 again
    assert led.record_replica(rep) == 5  # the older record is a no-op: still 6
    assert led.worker_latest((1, 0, 0)) == 6
    # the controller rewinds to what every worker can reproduce
    led2 = ffx.Ledger(spec)
    led2.record((0, 0, 0), 6)
    assert led2.record_replica(rep) == 5
    target = led2.global_consistent()
    assert target == 5
    plan = ffx.plan_recovery(spec, [1], [], target, 0)
    assert plan.kind == "neighbor" and plan.forwards[0][1] == 0  # held by node 0
    ffx.materialize(state, b"\xee" * 32)
    origin.recover(view, target)
    assert host(state) == want
    led2.rebase(target)
    assert led2.global_consistent() == 5


def test_damaged_handle_is_refused(ffx):
    """A replica handle travels between processes as 256 opaque bytes; one
    whose geometry does not add up is refused before any slot is addressed."""
    import struct
    spec, holder, origin, rep, view = ring_pair(ffx, 10_000)
    good = bytearray(rep.export())
    for off, fmt, val in ((40, "<I", 0), (40, "<I", 9), (32, "<Q", 100), (24, "<Q", 1 << 40), (0, "<I", 0)):
        bad = bytearray(good)
        struct.pack_into(fmt, bad, off, val)
        with pytest.raises(ffx.InvalidArgument):
            origin.open_replica(bytes(bad))
    origin.open_replica(bytes(good)).destroy()


def test_rollback_drops_pre_failure_slots_from_the_ledger(ffx):
    """after ffx_ledger_rebase(N) a holder still has slots newer
    than N committed before the failure; read back as a CkptRecord they would
    re-raise the rebased ledger before the replay re-commits them (the
    reference drops stale-epoch CkptRecords, Controller::on_ckpt_record).
    ffx_replica_rollback(N) empties them; the replay then refills the slot."""
    n = 2 * 4096 + 5
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    spec.num_nodes, spec.gpus_per_node = 2, 1
    led = ffx.Ledger(spec)
    state = torch.zeros(n, dtype=torch.uint8, device="cuda")
    origin.register(ffx.REGION_BLOB, state)
    for it in (1, 2, 3):
        state.fill_(it)
        origin.snapshot(it)
    torch.cuda.synchronize()
    assert sorted(rep.held()) == [2, 3]
    led.rebase(2)  # the new epoch resumes from global consistent iteration 2
    assert rep.rollback(2) == 1
    assert sorted(rep.held()) == [2]
    assert led.record_replica(rep) == 2 and led.worker_latest((1, 0, 0)) == 2
    origin.set_target(view)  # the writer re-arms its target in the new epoch
    state.fill_(33)  # the replayed iteration 3 differs from the lost one
    origin.snapshot(3)
    torch.cuda.synchronize()
    assert sorted(rep.held()) == [2, 3]
    assert rep.export_frame(3)[32:] == bytes([33]) * n
    assert rep.export_frame(2)[32:] == bytes([2]) * n
    assert led.record_replica(rep) == 3


def test_snapshots_on_two_streams_do_not_overlap(ffx):
    """two snapshots of one ctx share its task / commit counters;
    issued back to back on different streams, the second must wait for the
    first (snap_done event) instead of racing it -- both frames stay exact."""
    n = 64 * (1 << 20) + 3
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d1 = orc.optimizer_init(5, 1, 0, 0, True)
    d2 = orc.optimizer_init(6, 1, 0, 0, True)
    ffx.materialize(a, d1)
    origin.register(ffx.REGION_BLOB, a)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    origin.snapshot(1, stream=s1)
    ev = torch.cuda.Event()
    ev.record(s1)
    origin.snapshot(2, stream=s2)  # same bytes, different stream, no caller-side ordering
    torch.cuda.synchronize()
    want = orc.materialize(d1, n)
    assert rep.export_frame(1) == orc.pack_blob((1, 0, 0), 1, 1, want)
    assert rep.export_frame(2) == orc.pack_blob((1, 0, 0), 2, 1, want)
    del d2


@pytest.mark.parametrize("copy_engine", [False, True])
def test_holder_verifies_landed_bytes(ffx, copy_engine):
    """Checksum-as-landed on the holder (ffx_replica_verify; NeighborBuffer::
    store validates before accepting, ckpt.cpp:78): the split / copy-engine
    policies hash the origin's SOURCE, so a byte damaged after the table was
    computed is caught only by re-hashing what landed.  The holder re-hashes
    its committed slot from its own HBM; a flipped byte drops the slot (torn)
    and recovery then refuses it."""
    n = 5 * (1 << 20) + 333
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    origin.snapshot(4, split=True, copy_engine=copy_engine, hash_ctas=32)
    torch.cuda.synchronize()
    r = holder.verify_held(rep, 4, max_ctas=16)
    assert r.bad_slices == 0 and r.bytes == n
    slot = rep.held()[4]
    origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (slot << 48) | 777_777)
    with pytest.raises(ffx.CorruptSnapshot) as ei:
        holder.verify_held(rep, 4)
    assert "first 189" in str(ei.value)  # 777777 // 4096
    assert 4 not in rep.held()          # dropped: torn
    with pytest.raises(ffx.RestoreError):
        origin.recover(view, 4)
    with pytest.raises(ffx.InvalidArgument):
        origin.verify_held(view, 4)      # only the holder (its local HBM) verifies
    # the writer re-arms and re-sends: the dropped slot is reused first, so
    # the other version (3) is never evicted for it
    origin.snapshot(3, split=True, copy_engine=copy_engine, hash_ctas=32)
    torch.cuda.synchronize()
    origin.set_target(view)
    origin.snapshot(5, split=True, copy_engine=copy_engine, hash_ctas=32)
    torch.cuda.synchronize()
    assert sorted(rep.held()) == [3, 5]
    assert holder.verify_held(rep, 5).bad_slices == 0


def test_corrupt_slot_metadata_is_refused_not_followed(ffx):
    """A slot whose metadata lies about its slicing (slice size, table
    length) is refused with CorruptSnapshot by recovery and by the holder's
    verify -- the job is never built from it (ffx_recover.cu check_table)."""
    import ctypes
    n = 3 * (1 << 20) + 77
    spec, holder, origin, rep, view = ring_pair(ffx, n)
    state, want = blob_for(ffx, 1, n)
    origin.register(ffx.REGION_BLOB, state)
    origin.snapshot(6)
    torch.cuda.synchronize()
    slot = rep.held()[6]
    pay, sums = rep.slot_ptrs(slot)
    meta = sums - 256  # SlotMeta sits right before the table

    def poke(off, value):
        v = ctypes.c_uint64(value)
        ffx.check(ffx.lib.ffx_memcpy(ctypes.c_void_p(meta + off), ctypes.c_void_p(ctypes.addressof(v)), 8, None, 1), "poke")

    nsl = rep.slot_info(slot).num_slices
    try:
        # slice size, table length, payload length, a region's size
        for off, bad, good in ((32, 0, 4096), (32, 100, 4096), (40, nsl + 1, nsl), (40, 1 << 40, nsl),
                               (24, n + 1, n), (72, 1 << 50, n)):
            poke(off, bad)
            with pytest.raises(ffx.CorruptSnapshot, match="slot metadata"):
                origin.recover(view, 6)
            with pytest.raises(ffx.CorruptSnapshot, match="slot metadata"):
                holder.verify_held(rep, 6)
            with pytest.raises(ffx.CorruptSnapshot, match="slot metadata"):
                rep.export_frame(6)
            with pytest.raises(ffx.CorruptSnapshot, match="slot metadata"):
                rep.slot_regions(slot)
            poke(off, good)
        assert rep.export_frame(6) == orc.pack_blob((1, 0, 0), 6, 1, want)
        origin.inject(ffx.FAULT_POISON_STATE)
        assert origin.recover(view, 6).bad_slices == 0
        assert host(state) == want
    finally:
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()
