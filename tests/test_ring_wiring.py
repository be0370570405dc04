"""Multi-process host logic of the DP ring on CPU (gloo, world_size 2, 4 and 8 — the driver's 8-GPU scaling run).

The replica handles are stand-in byte strings; what is checked is that every
rank writes into exactly the replica its ring successor holds for it, and
that recovery sources derived from plan_recovery point at the right holder
(reference controller.cpp:177-189, domain.cpp:51-62).
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_03644_b200 import ring


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, replicas, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        created = []

        def create_for(origin):
            created.append(origin)
            return origin

        def export(origin):
            return b"H%02d<%02d" % (rank, origin)  # "held by rank, for origin"

        opened = []

        def open_handle(h):
            opened.append(h)
            return h

        def all_gather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        held, targets, handles = ring.wire_ring(rank, world, create_for, export, open_handle, all_gather,
                                                replicas=replicas)
        q.put((rank, created, [bytes(t) for t in targets], [[bytes(x) for x in h] for h in handles]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,replicas", [(2, 1), (4, 1), (4, 2), (8, 1), (8, 2)])
def test_ring_wiring_gloo(world, replicas):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, replicas, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, created, targets, handles = q.get(timeout=120)
        res[rank] = (created, targets, handles)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        created, targets, handles = res[r]
        assert created == [(r - k) % world for k in range(1, replicas + 1)]
        for k in range(replicas):
            holder = (r + k + 1) % world
            assert targets[k] == b"H%02d<%02d" % (holder, r)  # my snapshots land at my k-th successor
        assert handles == res[0][2]


def test_recovery_sources_follow_plan():
    from paper_2512_03644_b200 import ffx
    spec = ffx.make_spec(d=8, phi=1000, distributed=True, num_nodes=8, gpus_per_node=1)
    plan = ffx.plan_recovery(spec, [3], [], 10, 0)
    assert ring.recovery_sources(plan.forwards, 8) == [(3, 4, 0)]
    plan2 = ffx.plan_recovery(spec, [3, 4], [], 10, 0, replicas=2)
    assert sorted(ring.recovery_sources(plan2.forwards, 8)) == [(3, 5, 1), (4, 6, 1)]


def test_successor_predecessor_with_pp_tp():
    # d=2, p=2, t=2: ring successor keeps (pp, tp) and moves dp.
    w = 8
    for r in range(w):
        s = ring.successor(r, w, 2, 2)
        assert ring.ring_roles(w, 2, 2)[s][1:] == ring.ring_roles(w, 2, 2)[r][1:]
        assert ring.predecessor(s, w, 2, 2) == r


class _FakeMcast:
    """Stand-in multicast team member: records the protocol steps."""

    def __init__(self, origin, log):
        self.origin, self.log = origin, log

    def join(self):
        self.log.append(("join", self.origin))

    def bind(self, held):
        self.log.append(("bind", self.origin, held))


def _mcast_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        log = []

        def all_gather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        held, own, preds, view, handles = ring.wire_mcast_ring(
            rank, world, create_for=lambda origin: origin, export=lambda o: b"H%02d<%02d" % (rank, o),
            open_handle=lambda h: bytes(h), create_mcast=lambda: _FakeMcast(rank, log),
            export_mcast=lambda m: b"M%02d" % m.origin,
            open_mcast=lambda h: _FakeMcast(int(h[1:]), log), all_gather=all_gather,
            barrier=lambda: (log.append(("barrier",)), dist.barrier()))
        q.put((rank, held, [p.origin for p in preds], view, log))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_mcast_ring_wiring_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mcast_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, held, preds, view, log = q.get(timeout=120)
        res[rank] = (held, preds, view, log)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        held, preds, view, log = res[r]
        assert held == [(r - 1) % world, (r - 2) % world]
        assert preds == held  # the teams this rank joins as a holder
        assert view == b"H%02d<%02d" % ((r + 1) % world, r)  # read view: first holder's replica of me
        first_barrier = log.index(("barrier",))
        joins = [e for e in log[:first_barrier] if e[0] == "join"]
        assert sorted(j[1] for j in joins) == sorted([r] + held)  # own team + both predecessors' teams
        binds = [e for e in log if e[0] == "bind"]
        assert all(log.index(b) > first_barrier for b in binds)  # no bind before every team is complete
        assert sorted((b[1], b[2]) for b in binds) == sorted((o, o) for o in held)


def _mcast_fail_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        log = []

        def all_gather(b):
            out = [None] * world
            dist.all_gather_object(out, b)
            return out

        def create_mcast():
            if rank == 1:
                raise RuntimeError("no multicast here")
            return _FakeMcast(rank, log)

        try:
            ring.wire_mcast_ring(rank, world, create_for=lambda o: o, export=lambda o: b"H%02d<%02d" % (rank, o),
                                 open_handle=bytes, create_mcast=create_mcast, export_mcast=lambda m: b"M00",
                                 open_mcast=lambda h: _FakeMcast(0, log), all_gather=all_gather,
                                 barrier=dist.barrier)
            q.put((rank, "no error", log))
        except ring.WiringError as ex:
            dist.barrier()  # every rank got here: nobody is stuck in a collective
            q.put((rank, str(ex), log))
    finally:
        dist.destroy_process_group()


def test_mcast_ring_failure_is_collective():
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mcast_fail_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, msg, log = q.get(timeout=120)
        res[rank] = (msg, log)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        msg, log = res[r]
        assert "failed on ranks [1]" in msg and "no multicast here" in msg
        assert not any(e[0] in ("join", "bind") for e in log)  # nothing joined or bound
