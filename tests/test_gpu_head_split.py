"""Head-split slicing: the first region of a payload of >= 192 MiB opens with
a 48 MiB run of quarter-size slices (ffx_layout.h region_runs, exported as
ffx_slice_runs), so the persistent snapshot kernel's last-claimed tasks are
short.  The checksum table is then per run; these tests pin it, in full,
against the oracle's FNV-1a over the same runs, on every path that writes or
reads such a table: fused push, split push (SM copy and copy engines), the
second replica target, pull, holder verify, single- and two-source recover.
"""
import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
MiB = 1 << 20
SIZES = [192 * MiB + 4099, 5 * MiB + 3, 16]


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def host(t):
    return bytes(t.cpu().numpy().tobytes())


def fill(ts, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    for t in ts:
        t.copy_(torch.randint(0, 256, t.shape, dtype=torch.uint8, device="cuda", generator=g))


def want_table(ffx, regions, slice_bytes=4096):
    runs = ffx.slice_runs([len(r) for r in regions], slice_bytes)
    out = []
    for reg, off, nb, sl, first in runs:
        assert first == len(out)
        out += orc.slice_fnv(regions[reg][off:off + nb], sl)
    return runs, out


def slot_table(ffx, rep, slot, nsl):
    pay, sums = rep.slot_ptrs(slot)
    table = torch.empty(nsl, dtype=torch.int64, device="cuda")
    scratch = torch.empty((nsl * 8 + 4095) // 4096, dtype=torch.int64, device="cuda")
    ffx.copy_checksums(table, sums, 4096, scratch, nbytes=nsl * 8)
    return [v & ffx.U64_MAX for v in table.cpu().tolist()]


def test_slice_runs_threshold(ffx):
    assert len(ffx.slice_runs([192 * MiB - 1], 4096)) == 1
    assert ffx.slice_runs([192 * MiB], 4096)[:2] == [(0, 0, 48 * MiB, 1024, 0), (0, 48 * MiB, 144 * MiB, 4096, 49152)]
    assert len(ffx.slice_runs([192 * MiB], 512)) == 1     # not a multiple of 1 KiB: no head
    assert ffx.slice_runs([192 * MiB], 2048)[0][3] == 512
    assert len(ffx.slice_runs([192 * MiB] * 16, 4096)) == 16  # a full region table: no room for the head
    assert len(ffx.slice_runs([1, 192 * MiB], 4096)) == 2     # only the first region is split


@pytest.mark.parametrize("mode", ["fused", "split", "split_ce", "two_targets"])
def test_head_split_table_and_restore(ffx, mode):
    spec = ffx.make_spec(d=4, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    holder2 = ffx.Context(0, spec, (2, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    cap = sum(SIZES) + 3 * 4096
    rep = holder.create_replica((1, 0, 0), cap, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    rep2 = view2 = None
    if mode == "two_targets":
        rep2 = holder2.create_replica((1, 0, 0), cap, 2)
        view2 = origin.open_replica(rep2.export())
        origin.set_target2(view2)
    ts = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in SIZES]
    try:
        fill(ts, 7)
        for t in ts:
            origin.register(ffx.REGION_MASTER, t)
        kw = {"split": True, "hash_ctas": 32} if mode.startswith("split") else {}
        origin.snapshot(5, copy_engine=(mode == "split_ce"), **kw)
        torch.cuda.synchronize()
        regions = [host(t) for t in ts]
        runs, want = want_table(ffx, regions)
        assert len(runs) == 4 and runs[0][3] == 1024
        for r in [rep] + ([rep2] if rep2 is not None else []):
            slot = r.held()[5]
            info = r.slot_info(slot)
            assert info.num_slices == len(want) == origin.plan().num_slices
            assert info.num_regions == 3
            assert slot_table(ffx, r, slot, len(want)) == want
            assert r.export_frame(5) == orc.pack_blob((1, 0, 0), 5, 1, b"".join(regions))
        assert holder.verify_held(rep, 5).bad_slices == 0
        origin.inject(ffx.FAULT_POISON_STATE)
        rpt = origin.recover(view, 5)
        assert rpt.bad_slices == 0 and [host(t) for t in ts] == regions
        if view2 is not None:
            origin.inject(ffx.FAULT_POISON_STATE)
            assert origin.recover_from([view, view2], 5).bad_slices == 0
            assert [host(t) for t in ts] == regions
        # a flipped byte at the last byte of the head / first of the body is
        # located at its own slice, by the restore and by the holder's verify
        slot = rep.held()[5]
        for off, first in ((48 * MiB - 1, 49151), (48 * MiB, 49152)):
            origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (slot << 48) | off)
            with pytest.raises(ffx.RestoreError, match="first slice %d\\b" % first):
                origin.recover(view, 5)
            origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (slot << 48) | off)  # flip it back
        origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (slot << 48) | (3 * MiB))
        with pytest.raises(ffx.CorruptSnapshot, match="first 3072\\b"):
            holder.verify_held(rep, 5)
        assert 5 not in rep.held()
    finally:
        torch.cuda.synchronize()
        for v in (view, view2):
            if v is not None:
                v.destroy()
        for r in (rep, rep2):
            if r is not None:
                r.destroy()
        origin.close()
        holder2.close()
        holder.close()


def test_head_split_two_source_gather_locates_the_part(ffx):
    """recover_from cuts every run across the sources: the head's second half
    comes from source 2, and a flipped byte there is caught at its slice."""
    spec = ffx.make_spec(d=4, phi=64, distributed=True)
    h1, h2 = ffx.Context(0, spec, (2, 0, 0)), ffx.Context(0, spec, (3, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    n = SIZES[0]
    r1, r2 = h1.create_replica((1, 0, 0), n + 4096, 2), h2.create_replica((1, 0, 0), n + 4096, 2)
    v1, v2 = origin.open_replica(r1.export()), origin.open_replica(r2.export())
    state = torch.empty(n, dtype=torch.uint8, device="cuda")
    try:
        origin.set_target(v1)
        origin.set_target2(v2)
        fill([state], 11)
        origin.register(ffx.REGION_BLOB, state)
        origin.snapshot(3)
        torch.cuda.synchronize()
        want = host(state)
        origin.inject(ffx.FAULT_POISON_STATE)
        assert origin.recover_from([v1, v2], 3).bad_slices == 0 and host(state) == want
        off = 30_000 * 1024 + 5  # head slice 30000: in source 2's half of the head (24576..49151)
        slot = r2.held()[3]
        origin.inject(ffx.FAULT_CORRUPT_REPLICA, v2, (slot << 48) | off)
        with pytest.raises(ffx.RestoreError, match="first slice 30000\\b"):
            origin.recover_from([v1, v2], 3)
        origin.recover_from([v1], 3)  # the intact holder alone
        assert host(state) == want
    finally:
        torch.cuda.synchronize()
        v1.destroy(), v2.destroy(), r1.destroy(), r2.destroy()
        origin.close(), h1.close(), h2.close()


def test_head_split_pull(ffx):
    """Pull mode (the holder drives the kernel over the origin's mapped
    regions) writes the same per-run table."""
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    ts = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in SIZES]
    rep = holder.create_replica((1, 0, 0), sum(SIZES) + 3 * 4096, 2)
    remote = None
    try:
        fill(ts, 5)
        for t in ts:
            origin.register(ffx.REGION_MASTER, t)
        remote = holder.open_remote(origin.export_regions())
        holder.snapshot_pull(remote, rep, 9)
        torch.cuda.synchronize()
        regions = [host(t) for t in ts]
        runs, want = want_table(ffx, regions)
        slot = rep.held()[9]
        assert rep.slot_info(slot).num_slices == len(want)
        assert slot_table(ffx, rep, slot, len(want)) == want
    finally:
        torch.cuda.synchronize()
        if remote is not None:
            remote.close()
        rep.destroy()
        origin.close()
        holder.close()


@pytest.mark.parametrize("policy,copy_ctas,task_ctas", [(0, 16, False), (0, 16, True), (1, 8, False),
                                                        (2, 8, False), (0, 0, False)])
def test_head_split_scheduled_batches(ffx, policy, copy_ctas, task_ctas):
    """The slice scheduler cuts a snapshot into gap-sized batches by task
    range; with the head the task ranges span runs of two slice sizes (and,
    CTA-capped, the 64-slice task configuration)."""
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    ts = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in SIZES]
    rep = holder.create_replica((1, 0, 0), sum(SIZES) + 3 * 4096, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    gaps = 7
    train = torch.cuda.Stream(priority=-1)
    sched = None
    try:
        fill(ts, 3)
        for t in ts:
            origin.register(ffx.REGION_MASTER, t)
        # the batches run on the scheduler's own stream, gated only on events
        # of `train`: the state must be complete before the step starts
        torch.cuda.synchronize()
        sched = ffx.Sched(origin, policy, link_gaps=gaps, sm_gaps=0 if policy == ffx.SCHED_FUSED else gaps,
                          copy_ctas=copy_ctas or (1 << 20), hash_ctas=32,
                          gap_ms=[1.0, 3.0, 0.5, 2.0, 2.0, 1.5, 0.7], task_ctas=task_ctas)
        sched.begin(4)
        for _ in range(gaps):
            sched.gap(ffx.GAP_SM_IDLE, train)
            sched.gap(ffx.GAP_LINK_IDLE, train)
        sched.finish(train)
        train.synchronize()
        torch.cuda.synchronize()
        regions = [host(t) for t in ts]
        runs, want = want_table(ffx, regions)
        slot = rep.held()[4]
        assert slot_table(ffx, rep, slot, len(want)) == want
        assert rep.export_frame(4) == orc.pack_blob((1, 0, 0), 4, 1, b"".join(regions))
        origin.inject(ffx.FAULT_POISON_STATE)
        assert origin.recover(view, 4).bad_slices == 0 and [host(t) for t in ts] == regions
    finally:
        if sched is not None:
            sched.destroy()
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()


@pytest.mark.parametrize("slice_bytes", [1024, 2048])
def test_head_split_other_slice_sizes(ffx, slice_bytes):
    """Head slices of 256 B (one 2-plane TMA box per slice) and 512 B."""
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0), slice_bytes)
    origin = ffx.Context(0, spec, (1, 0, 0), slice_bytes)
    ts = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in SIZES]
    rep = holder.create_replica((1, 0, 0), sum(SIZES) + 3 * 4096, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    try:
        fill(ts, 9)
        for t in ts:
            origin.register(ffx.REGION_MASTER, t)
        origin.snapshot(2)
        torch.cuda.synchronize()
        regions = [host(t) for t in ts]
        runs, want = want_table(ffx, regions, slice_bytes)
        assert runs[0][3] == slice_bytes // 4
        slot = rep.held()[2]
        assert rep.slot_info(slot).num_slices == len(want)
        assert slot_table(ffx, rep, slot, len(want)) == want
        assert holder.verify_held(rep, 2).bad_slices == 0
        origin.inject(ffx.FAULT_POISON_STATE)
        assert origin.recover(view, 2).bad_slices == 0 and [host(t) for t in ts] == regions
    finally:
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()


def test_every_large_run_is_on_the_tma_path(ffx):
    """Guard against a large job region falling to the register path (no
    tensor map): six regions like a ZeRO-3 shard -- five large job runs with
    the head -- must snapshot at HBM speed.  The register path alone runs
    at well under half of it (1286 vs 3229 GB/s on the 14 GB shard)."""
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    sizes = [768 * MiB, 512 * MiB, 512 * MiB, 256 * MiB + 4096, 8, 4]
    ts = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in sizes]
    rep = holder.create_replica((1, 0, 0), sum(sizes) + 8 * 4096, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    try:
        fill(ts, 1)
        for t in ts:
            origin.register(ffx.REGION_MASTER, t)
        assert len(ffx.slice_runs(sizes, 4096)) == 7
        for it in range(3):  # warm-up
            origin.snapshot(it + 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for it in range(5):
            origin.snapshot(it + 10)
        e1.record()
        torch.cuda.synchronize()
        gbs = 5 * sum(sizes) / (e0.elapsed_time(e1) * 1e-3) / 1e9
        assert gbs > 2400, gbs
        origin.inject(ffx.FAULT_POISON_STATE)
        assert origin.recover(view, 14).bad_slices == 0
    finally:
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()
