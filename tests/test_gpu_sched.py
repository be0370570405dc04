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
    torch.cuda.synchronize()  # the scheduler's streams do not wait on the default stream
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
    torch.cuda.synchronize()  # the scheduler's streams do not wait on the default stream
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


def _train_ms(train, a, b, reps=1):
    """Device time of a full-GPU TRAIN kernel (bf16 GEMM) on the train stream."""
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(train):
        e0.record(train)
        for _ in range(reps):
            torch.matmul(a, b)
        e1.record(train)
    return e0, e1


@pytest.mark.parametrize("cap,tasks", [(32, False), (0, False), (0, True)])
def test_train_waits_at_most_one_state_batch(ffx, cap, tasks):
    """TRAIN > STATE with bounded inversion (sim_net.cpp:401-454; the pin is
    test_transport.cpp:173-197: a TRAIN chunk queued while a STATE chunk is
    on the wire starts at the next chunk boundary).  Here a STATE batch (one
    fused snapshot batch, low-priority stream, optionally CTA-capped) is
    resident when one full-GPU TRAIN GEMM arrives on the high-priority
    stream: the GEMM's extra time is at most one batch's duration (the batch
    is never cut; nothing of STATE starts ahead of the queued TRAIN kernel).
    With task-granular batches (task_ctas) the unit of inversion shrinks to
    one task: TRAIN's CTAs take every SM a finished task frees."""
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    n = 1 << 30
    rep = holder.create_replica((1, 0, 0), n, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    state = torch.empty(n, dtype=torch.uint8, device="cuda")
    ffx.materialize(state, orc.optimizer_init(3, 1, 0, 0, True))
    torch.cuda.synchronize()  # the scheduler's streams do not wait on the default stream
    origin.register(ffx.REGION_BLOB, state)
    train = torch.cuda.Stream(priority=-1)
    low = torch.cuda.Stream(priority=0)
    a = torch.randn(16384, 8192, dtype=torch.bfloat16, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
    try:
        batches = 4
        # one STATE batch alone
        origin.snapshot_begin(1, batches=batches, max_ctas=cap, task_ctas=tasks)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(low)
        origin.snapshot_next(stream=low)
        f1.record(low)
        while origin.snapshot_next(stream=low):
            pass
        torch.cuda.synchronize()
        batch_ms = f0.elapsed_time(f1)
        # TRAIN alone
        for _ in range(3):
            e0, e1 = _train_ms(train, a, b)
            torch.cuda.synchronize()
        alone = e0.elapsed_time(e1)
        # TRAIN arriving while the first STATE batch is resident; the other
        # batches are issued only after TRAIN finished
        worst = 0.0
        for it in (2, 3, 4):
            origin.snapshot_begin(it, batches=batches, max_ctas=cap, task_ctas=tasks)
            origin.snapshot_next(stream=low)
            e0, e1 = _train_ms(train, a, b)
            train.synchronize()
            worst = max(worst, e0.elapsed_time(e1) - alone)
            while origin.snapshot_next(stream=low):
                pass
            torch.cuda.synchronize()
        assert rep.newest() == 4
        print("inversion cap=%d tasks=%d: batch %.3f ms, train alone %.3f ms, worst extra %.3f ms"
              % (cap, tasks, batch_ms, alone, worst))
        assert worst <= batch_ms * 1.1 + 0.05, (worst, batch_ms, alone)
    finally:
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()
