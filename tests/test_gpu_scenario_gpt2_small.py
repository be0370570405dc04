"""BASELINE configs[0] end to end: GPT-2 small (124M) fp32 Adam state over
2 DP ranks (ZeRO-1: N = ceil(12 phi / 2) = 746,638,848 B per rank).

Ring snapshots for iterations 1..10 with the state evolving per iteration
exactly as SURVEY 8(d) specifies (optimizer_next over the grad digest of each
rank's data window, evolution.cpp:26-69, dataloader.cpp:36-49), rank d1 is
killed after iteration 10, its replacement restores from the holder d0
(plan_recovery, controller.cpp:177-189), and the result is compared with the
reference CPU path: the SNP1 frame the holder exports must be byte-identical
to the reference's own pack_blob of the reference's own materialize
(oracle/_ref, compiled from the reference sources; the C oracle when that is
absent)."""
import ctypes

import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PHI_GPT2_SMALL = 124_439_808
D = 2


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def reference_frame(role, iteration, digest, n):
    """SNP1 frame of materialize(digest, n) by the reference itself."""
    ref = orc.ref_lib()
    if ref is None:
        return orc.pack_blob(role, iteration, 1, orc.materialize(digest, n)), "oracle"
    ref.ref_pack_blob.restype = ctypes.c_int
    ref.ref_pack_blob.argtypes = [ctypes.c_uint16] * 3 + [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                                          ctypes.c_uint64, ctypes.c_void_p]
    payload = ctypes.create_string_buffer(n)
    assert ref.ref_materialize(digest, n, payload) == 0
    frame = ctypes.create_string_buffer(32 + n)
    assert ref.ref_pack_blob(role[0], role[1], role[2], iteration, 1, payload, n, frame) == 0
    return frame.raw, "reference"


def test_gpt2_small_ring_ten_iterations_then_single_rank_failure(ffx):
    spec = ffx.make_spec(d=D, phi=PHI_GPT2_SMALL, distributed=True)
    n = ffx.optimizer_bytes(spec)
    assert n == 746_638_848
    devs = [r % torch.cuda.device_count() for r in range(D)]
    ctx = [ffx.Context(devs[r], spec, (r, 0, 0)) for r in range(D)]
    # rank r holds the replica of its ring predecessor (domain.cpp:51-55)
    held = [ctx[r].create_replica(((r - 1) % D, 0, 0), n, 2) for r in range(D)]
    views = [ctx[r].open_replica(held[(r + 1) % D].export()) for r in range(D)]
    state = []
    for r in range(D):
        ctx[r].set_target(views[r])
        with torch.cuda.device(devs[r]):
            state.append(torch.empty(n, dtype=torch.uint8, device="cuda:%d" % devs[r]))
        ctx[r].register(ffx.REGION_BLOB, state[r])
    try:
        for it in range(1, 11):
            for r in range(D):
                ffx.materialize(state[r], orc.optimizer_at(42, r, 0, 0, it, D))
                ctx[r].snapshot(it)
            for d in set(devs):
                torch.cuda.synchronize(d)
        for r in range(D):  # two-version window (ckpt.cpp:46-52): 9 and 10 held
            assert held[r].newest() == 10
        # rank d1 dies; its shard comes back from the holder plan_recovery names
        plan = ffx.plan_recovery(spec, [], [ffx.Role(1, 0, 0)], 10, 0)
        assert plan.kind == "neighbor"
        (origin, _hn, _dn, holder_dp), = plan.forwards
        assert tuple(origin.tuple()) == (1, 0, 0) and holder_dp == 0
        source = ctx[1].open_replica(held[holder_dp].export())
        want = orc.optimizer_at(42, 1, 0, 0, 10, D)
        ctx[1].inject(ffx.FAULT_POISON_STATE)
        rpt = ctx[1].recover(source, 10)
        assert rpt.bad_slices == 0 and rpt.bytes == n
        assert ffx.blob_is_sound(state[1])
        assert bytes(state[1][:32].cpu().numpy().tobytes()) == want
        for lo in (0, 32, 4096 * 1000 + 17, n - 4099):
            got = bytes(state[1][lo:lo + 4099].cpu().numpy().tobytes())
            assert got == orc.materialize_range(want, n, lo, min(4099, n - lo))
        # the previous version is restorable too; older ones are gone (VersionError window)
        rpt9 = ctx[1].recover(source, 9)
        assert rpt9.bad_slices == 0
        assert bytes(state[1][:32].cpu().numpy().tobytes()) == orc.optimizer_at(42, 1, 0, 0, 9, D)
        with pytest.raises(ffx.RestoreError):
            ctx[1].recover(source, 8)
        source.destroy()
        # the reference CPU path on the same inputs: byte-identical SNP1 frame
        frame = held[0].export_frame(10)
        ref, who = reference_frame((1, 0, 0), 10, want, n)
        assert len(frame) == len(ref) == 32 + n
        assert frame[:32] == ref[:32], who   # header incl. the whole-payload FNV
        assert frame == ref, who
    finally:
        for d in set(devs):
            torch.cuda.synchronize(d)
        for v in views:
            v.destroy()
        for h in held:
            h.destroy()
        for c in ctx:
            c.close()
