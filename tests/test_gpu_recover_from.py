"""Parallel peer gathers (ffx_recover_from) and measured-gap batch weights."""
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


def dual_setup(ffx, n, regions_extra=True):
    spec = ffx.make_spec(d=4, phi=64, distributed=True)
    h1, h2 = ffx.Context(0, spec, (2, 0, 0)), ffx.Context(0, spec, (3, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    r1, r2 = h1.create_replica((1, 0, 0), n + 4096, 2), h2.create_replica((1, 0, 0), n + 4096, 2)
    v1, v2 = origin.open_replica(r1.export()), origin.open_replica(r2.export())
    origin.set_target(v1)
    origin.set_target2(v2)
    d = orc.optimizer_init(42, 1, 0, 0, True)
    state = torch.empty(n, dtype=torch.uint8, device="cuda")
    ffx.materialize(state, d)
    origin.register(ffx.REGION_BLOB, state)
    extra = torch.arange(333, dtype=torch.int32, device="cuda")
    if regions_extra:
        origin.register(ffx.REGION_RNG, extra)
    return origin, (h1, h2), (r1, r2), (v1, v2), state, extra, orc.materialize(d, n)


@pytest.mark.parametrize("n", [(1 << 22) + 5, 3 * 4096 + 17])
def test_recover_from_two_holders(ffx, n):
    origin, hs, reps, views, state, extra, want = dual_setup(ffx, n)
    origin.snapshot(4)
    torch.cuda.synchronize()
    saved_extra = host(extra)
    origin.inject(ffx.FAULT_POISON_STATE)
    rpt = origin.recover_from(list(views), 4)
    assert rpt.bad_slices == 0 and rpt.bytes == n + 333 * 4
    assert host(state) == want and host(extra) == saved_extra
    # a corrupted byte in the second holder's half is caught and located
    nsl = (n + 4095) // 4096
    off = min(n - 1, (nsl - 1) * 4096 + 3)  # last slice: pulled from source 2
    slot = reps[1].held()[4]
    origin.inject(ffx.FAULT_CORRUPT_REPLICA, views[1], (slot << 48) | off)
    with pytest.raises(ffx.RestoreError, match="checksum mismatch"):
        origin.recover_from(list(views), 4)
    # the intact holder alone still restores it
    origin.recover_from([views[0]], 4)
    assert host(state) == want


def test_recover_from_rejects_mismatched_sources(ffx):
    origin, hs, reps, views, state, extra, want = dual_setup(ffx, 1 << 20)
    origin.snapshot(4)
    origin.set_target2(None)
    origin.snapshot(5)  # only the first holder has iteration 5
    torch.cuda.synchronize()
    with pytest.raises(ffx.RestoreError, match="missing"):
        origin.recover_from(list(views), 5)
    origin.recover_from([views[0]], 5)


def test_batch_weights_shape_batches(ffx):
    # measured-gap weights change where batches cut the task range, never the bytes
    origin, hs, reps, views, state, extra, want = dual_setup(ffx, (1 << 22) + 99, regions_extra=False)
    origin.set_target2(None)
    s = torch.cuda.Stream()
    nb = origin.snapshot_begin(7, batches=4, max_ctas=8, batch_weights=[5.0, 0.0, 1.0, 2.0])
    left = nb
    while left:
        left = origin.snapshot_next(stream=s)
    s.synchronize()
    assert reps[0].export_frame(7) == orc.pack_blob((1, 0, 0), 7, 1, want)
