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
