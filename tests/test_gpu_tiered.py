"""Tiered replicas (configs[4]: a Llama-3 70B ZeRO-3 replica does not fit in
HBM beside its holder's own 123.5 GB of state; SURVEY 7.2 hard part 3).  The
replica's slot range is device memory up to hbm_bytes and pinned host memory
after it, one VA range, so the same kernels snapshot into it and recover from
it; every byte, the checksum table and the SNP1 frame must be exactly what an
all-HBM replica holds -- with the tier boundary inside a region's payload,
and with no HBM at all (slot metadata and checksum table in host memory)."""
import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MiB = 1 << 20


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def host(t):
    return bytes(t.cpu().numpy().tobytes())


@pytest.mark.parametrize("versions,hbm", [(2, 16 * MiB), (1, 2 * MiB), (2, 0)])
def test_tiered_replica_roundtrip(ffx, versions, hbm):
    spec = ffx.make_spec(d=2, phi=1 << 20, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    sizes = [40 * MiB + 4099, 16, 3 * MiB + 5]
    cap = sum(sizes) + 4096
    rep = holder.create_tiered_replica((1, 0, 0), cap, versions, hbm)
    dev, hostb = rep.tiers()
    assert dev == hbm and hostb > 0
    ref = holder.create_replica((1, 0, 0), cap, versions)  # an all-HBM replica for comparison
    view = origin.open_replica(rep.export())
    try:
        ts = []
        for i, n in enumerate(sizes):
            t = torch.empty(n, dtype=torch.uint8, device="cuda")
            if n >= 32:
                ffx.materialize(t, orc.optimizer_init(30 + i, 1, 0, 0, True))
            else:
                t.copy_(torch.arange(n, dtype=torch.uint8, device="cuda"))
            origin.register(ffx.REGION_MASTER, t)
            ts.append(t)
        want = b"".join(host(t) for t in ts)
        for target in (view, origin.open_replica(ref.export())):
            origin.set_target(target)
            origin.snapshot(7)
            origin.snapshot(8, verify_on_store=True)
        torch.cuda.synchronize()
        assert rep.export_frame(8) == ref.export_frame(8) == orc.pack_blob((1, 0, 0), 8, 1, want)
        for t in ts:
            t.fill_(0)
        rpt = origin.recover(view, 8)
        assert rpt.bad_slices == 0 and b"".join(host(t) for t in ts) == want
        # a flipped byte in the host tier is caught at its slice
        off = sizes[0] - 4096 * 3 + 17
        slot = rep.held()[8]
        origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (slot << 48) | off)
        with pytest.raises(ffx.RestoreError, match="first slice %d" % (off // 4096)):
            origin.recover(view, 8)
    finally:
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        ref.destroy()
        origin.close()
        holder.close()


@pytest.mark.skipif(__import__("os").environ.get("FFX_FULL_SIZE", "1") == "0", reason="full-size disabled")
def test_llama3_70b_zero3_full_replica_on_a_tiered_slot(ffx):
    """configs[4] at full size on one B200: a Llama-3 70B ZeRO-3 d=8 rank's
    six regions (123,468,986,400 B) and one complete replica of them, which
    cannot fit in HBM beside the state, on a tiered slot.  Snapshot, poison,
    recover: every region blob_is_sound, sampled slices equal to the oracle's
    materialize_range (both tiers: the samples straddle the HBM/host split)."""
    import os
    from paper_2512_03644_b200 import state
    regs = state.zero3_shard(state.PHI_LLAMA3_70B, 8, 1)
    n = state.shard_bytes(regs)
    assert n == 123_468_986_400
    free, _ = torch.cuda.mem_get_info()
    host_free = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    if free < n + (24 << 30) or host_free < n - (free - n) + (32 << 30):
        pytest.skip("needs ~150 GB HBM + ~100 GB host memory free")
    spec = ffx.make_spec(d=8, phi=state.PHI_LLAMA3_70B, distributed=True)
    holder = ffx.Context(0, spec, (2, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    ts, rep, view = [], None, None
    try:
        ts = state.allocate(ffx, torch, origin, regs)
        torch.cuda.synchronize()
        free, _ = torch.cuda.mem_get_info()
        rep = holder.create_tiered_replica((1, 0, 0), n, 1, max(0, free - (12 << 30)))
        dev, hostb = rep.tiers()
        assert hostb > 0
        view = origin.open_replica(rep.export())
        origin.set_target(view)
        origin.snapshot(1)
        torch.cuda.synchronize()
        assert rep.slot_regions(rep.held()[1]) == [(r.kind, r.nbytes) for r in regs]
        origin.inject(ffx.FAULT_POISON_STATE)
        rpt = origin.recover(view, 1)
        assert rpt.bad_slices == 0 and rpt.bytes == n
        off = 0
        for t, r in zip(ts, regs):
            if r.literal is not None:
                assert host(t) == r.literal
            else:
                assert ffx.blob_is_sound(t)
                ns = (r.nbytes + 4095) // 4096
                for sl in (0, ns // 2, ns - 1):
                    lo = sl * 4096
                    ln = min(4096, r.nbytes - lo)
                    assert host(t[lo:lo + ln]) == orc.materialize_range(r.digest, r.nbytes, lo, ln)
            off += r.nbytes
    finally:
        torch.cuda.synchronize()
        if view is not None:
            view.destroy()
        if rep is not None:
            rep.destroy()
        del ts
        origin.close()
        holder.close()
        torch.cuda.empty_cache()
