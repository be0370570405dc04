"""The native slice scheduler (ffx_sched_*): a fake training step reports
its gaps, every policy commits a slot byte-identical to the reference frame,
the optimizer stream only proceeds after the commit, and the scheduler
refuses to start a step while the previous one is unfinished."""
import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def busy(stream, n=1 << 22):
    """A little TRAIN work on the step's stream between gap reports."""
    with torch.cuda.stream(stream):
        a = torch.empty(n, device="cuda")
        a.fill_(1.0)
        a.mul_(2.0)


@pytest.mark.parametrize("policy", [0, 1, 2])
@pytest.mark.parametrize("weights", [False, True])
def test_sched_policies_commit_the_reference_frame(ffx, policy, weights):
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    n = (1 << 23) + 777
    rep = holder.create_replica((1, 0, 0), n, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    d = orc.optimizer_init(42, 1, 0, 0, True)
    state = torch.empty(n, dtype=torch.uint8, device="cuda")
    ffx.materialize(state, d)
    origin.register(ffx.REGION_BLOB, state)
    gaps = 6
    train = torch.cuda.Stream(priority=-1)
    sched = ffx.Sched(origin, policy, link_gaps=gaps, sm_gaps=0 if policy == ffx.SCHED_FUSED else gaps,
                      gap_ms=[1.0, 3.0, 0.5, 2.0, 2.0, 1.5] if weights else None)
    try:
        for it in (7, 8):
            sched.begin(it)
            with pytest.raises(ffx.StateError):
                sched.begin(it + 100)  # the previous step is unfinished
            for g in range(gaps):
                sched.gap(ffx.GAP_SM_IDLE, train)
                busy(train)
                sched.gap(ffx.GAP_LINK_IDLE, train)
                busy(train)
            sched.finish(train)
            marker = torch.zeros(1, device="cuda")
            with torch.cuda.stream(train):
                marker.fill_(1.0)  # "the optimizer": ordered after the commit
            train.synchronize()
            assert rep.newest() == it
        assert rep.export_frame(8) == orc.pack_blob((1, 0, 0), 8, 1, orc.materialize(d, n))
        origin.inject(ffx.FAULT_POISON_STATE)
        assert origin.recover(view, 8).bad_slices == 0
        # fewer reports than batches: finish() flushes the rest
        sched.begin(9)
        sched.gap(ffx.GAP_LINK_IDLE, train)
        sched.finish(train)
        train.synchronize()
        assert rep.newest() == 9
    finally:
        sched.destroy()
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()


def test_sched_zero_weight_gaps_and_idle_calls(ffx):
    # measured gaps that are all but one empty: every byte goes through the one
    # non-empty batch; finish() / gap() outside a step are no-ops
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    n = (1 << 20) + 5
    rep = holder.create_replica((1, 0, 0), n, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    d = orc.optimizer_init(5, 1, 0, 0, True)
    state = torch.empty(n, dtype=torch.uint8, device="cuda")
    ffx.materialize(state, d)
    origin.register(ffx.REGION_BLOB, state)
    train = torch.cuda.Stream()
    sched = ffx.Sched(origin, ffx.SCHED_SPLIT_CE, link_gaps=4, sm_gaps=4, gap_ms=[0.0, 0.0, 2.0, 0.0])
    try:
        sched.finish(train)                      # nothing in flight: no-op
        sched.gap(ffx.GAP_LINK_IDLE, train)      # no step: no-op
        sched.begin(3)
        for _ in range(4):
            sched.gap(ffx.GAP_SM_IDLE, train)
            sched.gap(ffx.GAP_LINK_IDLE, train)
        sched.finish(train)
        train.synchronize()
        assert rep.export_frame(3) == orc.pack_blob((1, 0, 0), 3, 1, orc.materialize(d, n))
        with pytest.raises(ffx.InvalidArgument):
            ffx.Sched(origin, 7, link_gaps=4)
        with pytest.raises(ffx.InvalidArgument):
            ffx.Sched(origin, ffx.SCHED_SPLIT, link_gaps=4, sm_gaps=0)
    finally:
        sched.destroy()
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()
