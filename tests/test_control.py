"""The controller state that drives recovery, host-only:
ffx_heartbeats (ctl::HeartbeatTable) and ffx_ledger (ctl::IterationLedger).

- test_controller.cpp:37-164 restated against libffx (same cases, same
  expectations);
- seeded random operation sequences replayed on libffx, on the Python
  restatement (oracle/pyoracle.py) and -- when oracle/_ref was built -- on the
  reference's own classes (controller.cpp compiled unmodified), compared after
  every operation;
- ffx_plan_recovery (replicas=1) against the reference's own plan_recovery on
  random failure sets.
"""
import itertools
import random

import pytest

import pyoracle as orc
from paper_2512_03644_b200 import ffx

S = ffx.SECOND_NS


def shape(d, p, t, gpn):  # test_controller.cpp:21-31
    return ffx.make_spec(d=d, p=p, t=t, num_nodes=d * p * t // gpn, gpus_per_node=gpn)


def _ref():
    r = orc.ref_lib()
    if r is None or not hasattr(r, "ref_hb_create"):
        return None
    return r


# ---- test_controller.cpp:37-81 -------------------------------------------------

@pytest.fixture
def hb():
    h = ffx.Heartbeats(4)
    h.enroll(0, 0, 0)
    h.enroll(1, 0, 0)
    yield h
    h.destroy()


def test_reports_refresh_the_slot(hb):
    hb.observe(0, 5, 2 * S)
    assert hb.last_iteration(0) == 5 and hb.last_seen(0) == 2 * S
    assert hb.unknown_reports() == 0


def test_unregistered_and_out_of_range_senders_are_counted(hb):
    hb.observe(2, 1, S)   # slot exists but never enrolled
    hb.observe(99, 1, S)  # no such slot
    assert hb.unknown_reports() == 2
    assert not hb.enrolled(99)


def test_regressed_iteration_is_stored_but_flagged(hb):
    hb.observe(0, 7, S)
    hb.observe(0, 4, 2 * S)
    assert hb.regressions() == 1
    assert hb.last_iteration(0) == 4 and hb.last_seen(0) == 2 * S


def test_reports_after_the_failure_mark_are_dropped(hb):
    hb.mark_failed(1)
    hb.observe(1, 9, 5 * S)
    assert hb.late_reports() == 1 and hb.last_iteration(1) == 0 and hb.failed(1)


def test_reenrollment_revives_a_failed_slot(hb):
    hb.mark_failed(1)
    hb.enroll(1, 42, 9 * S)
    assert not hb.failed(1)
    hb.observe(1, 43, 10 * S)
    assert hb.last_iteration(1) == 43 and hb.late_reports() == 0


def test_out_of_range_accessors_raise(hb):
    with pytest.raises(ffx.OutOfRange):
        hb.enroll(4, 0, 0)
    with pytest.raises(ffx.OutOfRange):
        hb.mark_failed(4)
    with pytest.raises(ffx.OutOfRange):
        hb.last_iteration(4)


# ---- test_controller.cpp:83-105 ------------------------------------------------

def test_silence_is_declared_within_threshold_plus_one_intervals():
    hb = ffx.Heartbeats(2)  # 1 s interval, 3 misses
    hb.enroll(0, 0, 0)
    hb.enroll(1, 0, 0)
    hb.observe(0, 10, 10 * S)
    for t in range(10, 16):
        hb.observe(1, 10 + t, t * S)
    log = [hb.sweep(t * S) for t in range(11, 16)]
    assert log == [[], [], [], [0], []]  # 13 s is exactly 3 s: quiet; 14 s declares; once
    assert hb.failed(0) and not hb.failed(1)


# ---- test_controller.cpp:107-123 -----------------------------------------------

def test_heartbeat_table_holds_tens_of_thousands_of_senders():
    pods = 32768
    hb = ffx.Heartbeats(pods)
    for n in range(pods):
        hb.enroll(n, 0, 0)
    for batch in range(1, 6):
        for n in range(pods):
            if batch >= 3 and n % 4096 == 7:
                continue
            hb.observe(n, batch, batch * S)
        assert hb.sweep(batch * S) == []
    assert hb.sweep(6 * S) == list(range(7, pods, 4096))


# ---- test_controller.cpp:125-163 -----------------------------------------------

@pytest.fixture
def led():
    g = ffx.Ledger(shape(2, 2, 1, 2))  # 2 nodes, 4 workers
    assert g.global_consistent() == 0
    g.record((0, 0, 0), 3)
    g.record((0, 1, 0), 3)
    g.record((1, 0, 0), 3)
    assert g.global_consistent() == 0  # one worker still absent
    g.record((1, 1, 0), 2)
    assert g.global_consistent() == 2
    yield g
    g.destroy()


def test_groups_one_apart_give_the_lower_value(led):
    led.record((1, 1, 0), 3)
    led.record((0, 0, 0), 4)
    led.record((1, 0, 0), 4)
    assert led.group_latest(0) == 4 and led.group_latest(1) == 3 and led.global_consistent() == 3


def test_records_are_monotone_per_worker(led):
    led.record((1, 1, 0), 1)
    assert led.worker_latest((1, 1, 0)) == 2


def test_rebase_pins_every_worker(led):
    led.rebase(7)
    assert led.global_consistent() == 7 and led.group_latest(0) == 7
    led.record((0, 0, 0), 8)
    assert led.global_consistent() == 7


def test_roles_outside_the_grid_are_rejected(led):
    with pytest.raises(ffx.OutOfRange):
        led.record((5, 0, 0), 1)
    assert led.worker_latest((5, 0, 0)) == 0


# ---- differential: libffx vs restatement vs the reference itself ---------------

def _hb_state(h, pods):
    return [(h.enrolled(n), h.failed(n), h.last_seen(n), h.last_iteration(n)) for n in range(pods)]


@pytest.mark.parametrize("seed", range(6))
def test_heartbeats_random_sequences_match_reference(seed):
    rng = random.Random(seed)
    pods = rng.choice([1, 3, 8, 17])
    interval, miss = rng.choice([(S, 3), (5, 2), (7, 1), (3, 0)])
    nat = ffx.Heartbeats(pods, interval, miss)
    py = orc.HeartbeatTable(pods, interval, miss)
    r = _ref()
    ref = r.ref_hb_create(pods, interval, miss) if r else None
    import ctypes
    now = 0
    for _ in range(400):
        now += rng.choice([0, 1, 2, interval, 2 * interval])
        op = rng.random()
        node = rng.randrange(pods + 2)
        it = rng.randrange(20)
        if op < 0.15 and node < pods:
            nat.enroll(node, it, now)
            py.enroll(node, it, now)
            if ref:
                assert r.ref_hb_enroll(ref, node, it, now) == 0
        elif op < 0.7:
            nat.observe(node, it, now)
            py.observe(node, it, now)
            if ref:
                r.ref_hb_observe(ref, node, it, now)
        elif op < 0.8 and node < pods:
            nat.mark_failed(node)
            py.mark_failed(node)
            if ref:
                assert r.ref_hb_mark_failed(ref, node) == 0
        else:
            got = nat.sweep(now)
            assert got == py.sweep(now)
            if ref:
                buf = (ctypes.c_uint32 * (pods + 1))()
                n = r.ref_hb_sweep(ref, now, buf, pods + 1)
                assert got == list(buf[:n])
        st = _hb_state(nat, pods)
        assert st == [(s["enrolled"], s["failed"], s["last_seen"], s["last_iteration"]) for s in py.slots]
        assert nat.counters() == (py.unknown, py.late, py.regressed)
        if ref:
            q = (ctypes.c_int64 * 4)()
            for n in range(pods):
                assert r.ref_hb_query(ref, n, q) == 0
                assert (bool(q[0]), bool(q[1]), q[2], q[3]) == st[n]
            c = (ctypes.c_uint64 * 3)()
            r.ref_hb_counters(ref, c)
            assert tuple(c) == nat.counters()
    if ref:
        r.ref_hb_free(ref)
    nat.destroy()


@pytest.mark.parametrize("seed", range(6))
def test_ledger_random_sequences_match_reference(seed):
    rng = random.Random(100 + seed)
    d, p, t = rng.choice([(2, 2, 1), (4, 1, 1), (3, 2, 2), (8, 1, 2)])
    world = d * p * t
    gpn = rng.choice([g for g in (1, 2, 4) if world % g == 0])
    nodes = world // gpn
    if seed == 5:
        nodes += 1  # world_size() != d*p*t: global_consistent never leaves 0 until rebase
    spec = ffx.make_spec(d=d, p=p, t=t, num_nodes=nodes, gpus_per_node=gpn)
    nat = ffx.Ledger(spec)
    py = orc.IterationLedger(nodes, gpn, d, p, t)
    r = _ref()
    ref = r.ref_ledger_create(nodes, gpn, d, p, t) if r else None
    for _ in range(300):
        op = rng.random()
        role = (rng.randrange(d + 1), rng.randrange(p + 1), rng.randrange(t + 1))
        it = rng.randrange(50)
        if op < 0.7:
            bad = False
            try:
                py.record(role, it)
            except ValueError:
                bad = True
            if bad:
                with pytest.raises(ffx.OutOfRange):
                    nat.record(role, it)
            else:
                nat.record(role, it)
            if ref:
                assert r.ref_ledger_record(ref, *role, it) == (-1 if bad else 0)
        elif op < 0.75:
            nat.rebase(it)
            py.rebase(it)
            if ref:
                r.ref_ledger_rebase(ref, it)
        g = nat.global_consistent()
        assert g == py.global_consistent()
        groups = [nat.group_latest(x) for x in range(p * t + 2)]
        assert groups == [py.group_latest(x) for x in range(p * t + 2)]
        w = nat.worker_latest(role)
        assert w == py.worker_latest(role)
        if ref:
            assert g == r.ref_ledger_global(ref)
            assert groups == [r.ref_ledger_group(ref, x) for x in range(p * t + 2)]
            assert w == r.ref_ledger_worker(ref, *role)
    if ref:
        r.ref_ledger_free(ref)
    nat.destroy()


@pytest.mark.parametrize("d,p,t,gpn,dist", [(4, 1, 1, 1, 1), (4, 2, 1, 2, 1), (6, 1, 1, 3, 0),
                                            (8, 1, 1, 8, 1), (3, 2, 2, 2, 1), (5, 1, 2, 1, 0), (1, 2, 1, 1, 1)])
def test_plan_recovery_matches_reference_plan_recovery(d, p, t, gpn, dist):
    r = _ref()
    if r is None:
        pytest.skip("oracle/_ref not built (reference checkout absent)")
    world = d * p * t
    nodes = world // gpn
    spec = ffx.make_spec(d=d, p=p, t=t, phi=1000, distributed=bool(dist), num_nodes=nodes, gpus_per_node=gpn)
    rng = random.Random(d * 100 + p * 10 + t)
    cases = [list(c) for k in (0, 1, 2) for c in itertools.combinations(range(nodes), min(k, nodes))]
    for pods in cases:
        for _ in range(3):
            extra = [orc.role_of(rng.randrange(world), d, p, t) for _ in range(rng.randrange(3))]
            gc, fb = rng.choice([(0, 0), (9, 5), (120, 100)])
            want = orc.ref_plan_recovery(r, nodes, gpn, d, p, t, dist, 1000, pods, extra, gc, fb)
            got = ffx.plan_recovery(spec, pods, [ffx.Role(*x) for x in extra], gc, fb)
            assert got.kind == want["kind"] and got.resume_iteration == want["resume"]
            assert got.failed_pods == want["failed_pods"]
            assert [x.tuple() for x in got.failed_roles] == want["failed_roles"]
            assert [x.tuple() for x in got.lazy_backup_targets] == want["lazy"]
            assert [(f[0].tuple(), f[1], f[2]) for f in got.forwards] == want["forwards"]
            assert [(a.tuple(), b.tuple()) for a, b in got.redundant_from] == want["redundant_from"]


def test_detection_to_plan_cycle():
    """Heartbeat silence -> sweep -> plan_recovery at the ledger's global
    consistent iteration -> rebase (the controller.cpp:46-58, :92-97, :144-209,
    :117-121 chain the reference's Controller runs), all on libffx."""
    d, gpn = 4, 1
    spec = ffx.make_spec(d=d, phi=1000, distributed=True, num_nodes=d, gpus_per_node=gpn)
    hb, led = ffx.Heartbeats(d), ffx.Ledger(spec)
    for n in range(d):
        hb.enroll(n, 0, 0)
    for it in range(1, 8):
        for n in range(d):
            if n == 2 and it > 4:
                continue  # pod 2 dies after iteration 4
            hb.observe(n, it, it * S)
            led.record(ffx.role_of(spec, n), it)
    dead = []
    for now in range(8, 11):  # the live pods last reported at 7 s
        dead += hb.sweep(now * S)
    assert dead == [2]
    assert led.global_consistent() == 4
    plan = ffx.plan_recovery(spec, dead, [], led.global_consistent(), 0)
    assert plan.kind == "neighbor" and plan.resume_iteration == 4
    assert [(f[0].tuple(), f[1], f[2]) for f in plan.forwards] == [((2, 0, 0), 3, 2)]
    led.rebase(plan.resume_iteration)
    hb.enroll(2, 4, 12 * S)  # the substitute registers
    assert led.global_consistent() == 4 and not hb.failed(2)


def test_facade_controller_cpp():
    """The C++ facade's ftsim::ctl (HeartbeatTable, IterationLedger,
    plan_recovery over libffx) against test_controller.cpp:37-276's
    expectations, restated in tests/cpp/test_facade_controller.cpp."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    binary = os.path.join(root, "paper_2512_03644_b200", "facade", "build", "test_facade_controller")
    if not os.path.exists(binary):
        pytest.fail("facade not built: run __graft_entry__.build()")
    r = subprocess.run([binary], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_controller_state_is_race_free_under_tsan(tmp_path):
    """ffx_control.cpp built with -fsanitize=thread and driven from 4
    heartbeat reporters + a sweeper + a reader, then 8 ledger recorders + 2
    readers (tests/cpp/test_control_threads.cpp); TSan aborts on any race."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "test_control_threads"
    cc = subprocess.run(["g++", "-std=c++17", "-O1", "-g", "-fsanitize=thread", "-I" + os.path.join(root, "include"),
                         "-o", str(exe), os.path.join(root, "tests", "cpp", "test_control_threads.cpp"),
                         os.path.join(root, "paper_2512_03644_b200", "csrc", "ffx_control.cpp"), "-lpthread"],
                        capture_output=True, text=True)
    if cc.returncode != 0 and "tsan" in cc.stderr.lower():
        pytest.skip("no ThreadSanitizer runtime: " + cc.stderr[-200:])
    assert cc.returncode == 0, cc.stderr
    env = dict(os.environ, TSAN_OPTIONS="halt_on_error=1")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stdout + r.stderr[-2000:]
    assert "control threads ok" in r.stdout
