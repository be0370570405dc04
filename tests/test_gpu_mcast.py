"""Double neighbour over NVSwitch multicast: the snapshot
kernel stores each tile once into a multicast range bound to the replica
slots of every holder; each holder's slot must then restore bit-exactly
through the ordinary recovery path (ckpt.cpp:140-167 semantics).

Needs >= 2 GPUs with multicast support (NVSwitch); one process drives every
GPU, the multi-process path is exercised by bench.py's 70B leg."""
import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    if torch.cuda.device_count() < 2:
        pytest.skip("multicast needs >= 2 GPUs")
    if not all(m.mcast_supported(d) for d in range(torch.cuda.device_count())):
        pytest.skip("no multicast support on this node")
    return m


def host(t):
    return bytes(t.cpu().numpy().tobytes())


def build_team(ffx, n_holders, nbytes, versions=2):
    spec = ffx.make_spec(d=n_holders + 1, phi=(1 << 20), distributed=True)
    origin = ffx.Context(0, spec, (0, 0, 0))
    holders = [ffx.Context(1 + i, spec, (1 + i, 0, 0)) for i in range(n_holders)]
    held = [h.create_shared_replica((0, 0, 0), nbytes, versions) for h in holders]
    mc = origin.create_mcast(nbytes, versions, members=n_holders + 1)
    handle = mc.export()
    mcs = [h.open_mcast(handle) for h in holders]
    for m in [mc] + mcs:  # every member joins before any bind / map
        m.join()
    for m, r in zip(mcs, held):
        m.bind(r)
    views = [origin.open_replica(r.export()) for r in held]
    origin.set_target_mcast(mc, views[0])
    return origin, holders, held, mc, mcs, views


def teardown(origin, holders, held, mc, mcs, views):
    torch.cuda.synchronize()
    for v in views:
        v.destroy()
    mc.destroy()
    for m in mcs:
        m.destroy()
    for r in held:
        r.destroy()
    for c in [origin] + holders:
        c.close()


@pytest.mark.parametrize("n_holders", [1, 2])
def test_multicast_snapshot_lands_in_every_holder(ffx, n_holders):
    if torch.cuda.device_count() < n_holders + 1:
        pytest.skip("needs %d GPUs" % (n_holders + 1))
    n = 3 * (1 << 20) + 12345  # ragged tail
    team = build_team(ffx, n_holders, n)
    origin, holders, held, mc, mcs, views = team
    try:
        torch.cuda.set_device(0)
        d0 = orc.optimizer_init(42, 0, 0, 0, True)
        state = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        ffx.materialize(state, d0)
        origin.register(ffx.REGION_BLOB, state)
        origin.snapshot(5)
        torch.cuda.synchronize()
        want = orc.materialize(d0, n)
        for v in views:
            assert v.newest() == 5
            state.fill_(0)
            r = origin.recover(v, 5)
            assert r.bad_slices == 0 and r.bytes == n
            assert host(state) == want
        # second version, then the first one is still restorable from every holder
        d1 = orc.optimizer_init(43, 0, 0, 0, True)
        ffx.materialize(state, d1)
        origin.snapshot(6)
        torch.cuda.synchronize()
        for v in views:
            state.fill_(0)
            assert origin.recover(v, 5).bad_slices == 0
            assert host(state) == want
            state.fill_(0)
            assert origin.recover(v, 6).bad_slices == 0
            assert host(state) == orc.materialize(d1, n)
    finally:
        teardown(*team)


@pytest.mark.parametrize("n_holders", [1, 2])
def test_multicast_with_the_small_slice_head(ffx, n_holders):
    """A payload large enough for the head run (ffx_slice_runs): the tiles of
    both slice sizes go through the multicast range, verify-on-store re-hashes
    what landed, every holder verifies its own slot and restores bit-exactly."""
    if torch.cuda.device_count() < n_holders + 1:
        pytest.skip("needs %d GPUs" % (n_holders + 1))
    n = (200 << 20) + 4099
    assert ffx.slice_runs([n], 4096)[0][3] == 1024
    team = build_team(ffx, n_holders, n)
    origin, holders, held, mc, mcs, views = team
    try:
        torch.cuda.set_device(0)
        d0 = orc.optimizer_init(44, 0, 0, 0, True)
        state = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        ffx.materialize(state, d0)
        origin.register(ffx.REGION_BLOB, state)
        origin.snapshot(3, verify_on_store=True)
        torch.cuda.synchronize()
        want = orc.materialize(d0, n)
        for h, r in zip(holders, held):
            assert h.verify_held(r, 3).bad_slices == 0
        for v in views:
            state.fill_(0)
            assert origin.recover(v, 3).bad_slices == 0
            assert host(state) == want
        # a flipped byte in the head is located at its 1 KiB slice
        origin.inject(ffx.FAULT_CORRUPT_REPLICA, views[0], (held[0].held()[3] << 48) | (5 * 1024 + 7))
        with pytest.raises(ffx.RestoreError, match="first slice 5\\b"):
            origin.recover(views[0], 3)
    finally:
        teardown(*team)


def test_multicast_verify_on_store_and_corruption(ffx):
    n = 1 << 20
    team = build_team(ffx, 1, n)
    origin, holders, held, mc, mcs, views = team
    try:
        torch.cuda.set_device(0)
        d0 = orc.optimizer_init(7, 0, 0, 0, True)
        state = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        ffx.materialize(state, d0)
        origin.register(ffx.REGION_BLOB, state)
        origin.snapshot(1, verify_on_store=True)  # re-hash what landed, read back over the holder's mapping
        torch.cuda.synchronize()
        origin.inject(ffx.FAULT_CORRUPT_REPLICA, views[0], (0 << 48) | 4097)
        with pytest.raises(ffx.RestoreError, match="checksum mismatch"):
            origin.recover(views[0], 1)
    finally:
        teardown(*team)


def test_multicast_layout_mismatch_is_refused(ffx):
    spec = ffx.make_spec(d=2, phi=(1 << 20), distributed=True)
    origin = ffx.Context(0, spec, (0, 0, 0))
    holder = ffx.Context(1, spec, (1, 0, 0))
    held = holder.create_shared_replica((0, 0, 0), 1 << 20, 2)
    plain = holder.create_replica((0, 0, 0), 1 << 20, 2)
    mc = origin.create_mcast(2 << 20, 2, members=2)
    hm = holder.open_mcast(mc.export())
    try:
        with pytest.raises(ffx.StateError):
            hm.bind(held)  # not joined yet
        mc.join()
        hm.join()
        with pytest.raises(ffx.FfxError):
            hm.bind(plain)  # a cudaMalloc replica cannot back a multicast range
        with pytest.raises(ffx.ConfigError):
            hm.bind(held)  # capacity differs from the range
    finally:
        hm.destroy()
        mc.destroy()
        plain.destroy()
        held.destroy()
        origin.close()
        holder.close()


@pytest.fixture(scope="module")
def ffx1():
    """Any GPU with multicast support: the one-device team below."""
    from paper_2512_03644_b200 import ffx as m
    if not m.mcast_supported(0):
        pytest.skip("no multicast support on device 0")
    return m


def test_one_gpu_team_multicast_target_commits_and_restores(ffx1):
    """The multicast write path on a single GPU (runs on the driver's 1-GPU
    box): a one-member team whose range the holder's shareable replica backs
    on the writer's own device.  The fused kernel's tiles, the slot metadata
    (multimem.st) and the COMMITTED flag all go through the multicast VA; the
    slot must then read back (unicast) as the reference frame and restore
    bit-exactly, verify-on-store included; a flipped byte is still caught."""
    ffx = ffx1
    spec = ffx.make_spec(d=2, phi=(1 << 20), distributed=True)
    origin = ffx.Context(0, spec, (1, 0, 0))
    holder = ffx.Context(0, spec, (0, 0, 0))
    n = 3 * (1 << 20) + 12345
    held = holder.create_shared_replica((1, 0, 0), n, 2)
    try:
        mc = origin.create_mcast(n, 2, members=1)
    except ffx.CudaError as ex:
        # measured on the pool's B200 (driver 580): cuMulticastCreate refuses
        # numDevices = 1 with CUDA_ERROR_INVALID_VALUE -- a multicast team
        # needs two GPUs (profiles/r2_multicast_one_gpu.txt)
        held.destroy()
        origin.close()
        holder.close()
        pytest.skip("driver refuses a one-device multicast team: %s" % ex)
    view = None
    try:
        mc.join()
        mc.bind(held)  # the holder's memory backs the range on this device
        view = origin.open_replica(held.export())
        origin.set_target_mcast(mc, view)
        d0 = orc.optimizer_init(42, 1, 0, 0, True)
        state = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        ffx.materialize(state, d0)
        origin.register(ffx.REGION_BLOB, state)
        origin.snapshot(5)
        d1 = orc.optimizer_init(43, 1, 0, 0, True)
        ffx.materialize(state, d1)
        origin.snapshot(6, verify_on_store=True)
        torch.cuda.synchronize()
        assert sorted(held.held()) == [5, 6]
        assert held.export_frame(5) == orc.pack_blob((1, 0, 0), 5, 1, orc.materialize(d0, n))
        assert held.export_frame(6) == orc.pack_blob((1, 0, 0), 6, 1, orc.materialize(d1, n))
        state.fill_(0)
        assert origin.recover(view, 5).bad_slices == 0
        assert host(state) == orc.materialize(d0, n)
        origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (held.held()[6] << 48) | 4097)
        with pytest.raises(ffx.RestoreError, match="checksum mismatch"):
            origin.recover(view, 6)
    finally:
        torch.cuda.synchronize()
        if view is not None:
            view.destroy()
        mc.destroy()
        held.destroy()
        origin.close()
        holder.close()
