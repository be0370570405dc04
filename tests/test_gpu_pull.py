"""Pull-mode ring stream: the holder's kernel reads the origin's registered
regions (peer-mapped), hashes them and commits its own slot, then releases the
origin's optimizer through the ack word (ffx_snapshot_wait_pulled).  Frames
must be byte-identical to the push path and to the oracle's pack_blob."""
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


def test_pull_snapshot_frames_ack_and_recovery(ffx):
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    origin = ffx.Context(0, spec, (1, 0, 0))
    holder = ffx.Context(0, spec, (0, 0, 0))
    n = (1 << 22) + 321
    d = orc.optimizer_init(42, 1, 0, 0, True)
    state = torch.empty(n, dtype=torch.uint8, device="cuda")
    ffx.materialize(state, d)
    cursor = torch.tensor([7, 8, 9], dtype=torch.int64, device="cuda")
    origin.register(ffx.REGION_BLOB, state)
    origin.register(ffx.REGION_CURSOR, cursor)
    held = holder.create_replica((1, 0, 0), n + 64, 2)
    remote = holder.open_remote(origin.export_regions())
    s = torch.cuda.Stream()
    for it in (1, 2, 3):
        holder.snapshot_pull(remote, held, it, stream=s)
    # the origin's stream is released once iteration 3 is committed
    o = torch.cuda.Stream()
    origin.wait_pulled(3, stream=o)
    ev = torch.cuda.Event()
    ev.record(o)
    ev.synchronize()
    torch.cuda.synchronize()
    concat = orc.materialize(d, n) + host(cursor)
    assert sorted(held.held()) == [2, 3]
    assert held.export_frame(3) == orc.pack_blob((1, 0, 0), 3, 1, concat)
    assert held.slot_info(held.held()[3]).role.tuple() == (1, 0, 0)
    # failure: the origin restores from the replica the holder filled
    view = origin.open_replica(held.export())
    origin.inject(ffx.FAULT_POISON_STATE)
    origin.recover(view, 3)
    assert host(state) == orc.materialize(d, n) and host(cursor) == concat[n:]
    remote.close()


def test_pull_rejects_mismatched_replica(ffx):
    spec = ffx.make_spec(d=4, phi=64, distributed=True)
    origin = ffx.Context(0, spec, (1, 0, 0))
    holder = ffx.Context(0, spec, (2, 0, 0))
    t = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    origin.register(ffx.REGION_BLOB, t)
    wrong = holder.create_replica((3, 0, 0), 4096, 2)
    remote = holder.open_remote(origin.export_regions())
    with pytest.raises(ffx.ConfigError):
        holder.snapshot_pull(remote, wrong, 1)
    small = holder.create_replica((1, 0, 0), 100, 2)
    with pytest.raises(ffx.ConfigError):
        holder.snapshot_pull(remote, small, 1)
    remote.close()


def test_pull_matches_push_bytes(ffx):
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    origin = ffx.Context(0, spec, (1, 0, 0))
    holder = ffx.Context(0, spec, (0, 0, 0))
    n = 3 * (1 << 20) + 17
    state = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    origin.register(ffx.REGION_BLOB, state)
    pushed = holder.create_replica((1, 0, 0), n, 2)
    pulled = holder.create_replica((1, 0, 0), n, 2)
    origin.set_target(origin.open_replica(pushed.export()))
    origin.snapshot(5)
    remote = holder.open_remote(origin.export_regions())
    holder.snapshot_pull(remote, pulled, 5)
    torch.cuda.synchronize()
    assert pushed.export_frame(5) == pulled.export_frame(5)
    remote.close()


def _released(ev, wait_s=0.05):
    import time
    time.sleep(wait_s)
    return ev.query()


def test_pull_ack_is_a_one_shot_token(ffx):
    """The origin's wait matches the pulled iteration exactly and consumes
    it: a fresh ctx does not release wait(0), a consumed ack does not
    release the same iteration twice, and after a rollback (ack_reset, or a
    recovery) a replayed iteration waits for its own re-pull instead of
    passing on the pre-failure ack (GEQ on a monotone word)."""
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    origin = ffx.Context(0, spec, (1, 0, 0))
    holder = ffx.Context(0, spec, (0, 0, 0))
    n = 1 << 20
    state = torch.zeros(n, dtype=torch.uint8, device="cuda")
    origin.register(ffx.REGION_BLOB, state)
    held = holder.create_replica((1, 0, 0), n, 2)
    remote = holder.open_remote(origin.export_regions())
    s, o = torch.cuda.Stream(), torch.cuda.Stream()
    pending = []  # iterations an origin wait is still blocked on (released in finally)
    try:
        # fresh ctx: nothing pulled yet, wait(0) must block
        origin.wait_pulled(0, stream=o)
        pending.append(0)
        ev = torch.cuda.Event()
        ev.record(o)
        assert not _released(ev)
        holder.snapshot_pull(remote, held, 0, stream=s)
        ev.synchronize()
        pending.pop()
        # pulled 1, consumed once; a second wait on 1 blocks until a re-pull
        holder.snapshot_pull(remote, held, 1, stream=s)
        origin.wait_pulled(1, stream=o)
        ev1 = torch.cuda.Event()
        ev1.record(o)
        ev1.synchronize()
        origin.wait_pulled(1, stream=o)
        pending.append(1)
        ev2 = torch.cuda.Event()
        ev2.record(o)
        assert not _released(ev2)
        holder.snapshot_pull(remote, held, 1, stream=s)
        ev2.synchronize()
        pending.pop()
        # pulled 2, never waited on (the origin failed); rollback to 1 and
        # replay 2: the stale ack must not release the replay
        holder.snapshot_pull(remote, held, 2, stream=s)
        s.synchronize()
        origin.ack_reset(stream=o)
        origin.wait_pulled(2, stream=o)
        pending.append(2)
        ev3 = torch.cuda.Event()
        ev3.record(o)
        assert not _released(ev3)
        holder.snapshot_pull(remote, held, 2, stream=s)
        ev3.synchronize()
        pending.pop()
        # recovery resets it too
        holder.snapshot_pull(remote, held, 3, stream=s)
        s.synchronize()
        view = origin.open_replica(held.export())
        origin.recover(view, 3)
        origin.wait_pulled(3, stream=o)
        pending.append(3)
        ev4 = torch.cuda.Event()
        ev4.record(o)
        assert not _released(ev4)
        holder.snapshot_pull(remote, held, 3, stream=s)
        ev4.synchronize()
        pending.pop()
    finally:
        for it in pending:  # never leave a stream blocked on the device
            holder.snapshot_pull(remote, held, it, stream=s)
        torch.cuda.synchronize()
        remote.close()
