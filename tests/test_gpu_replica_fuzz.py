"""Differential fuzz of the two-version semantics against the REFERENCE
ITSELF: seeded random sequences of snapshots (fresh iterations, re-takes of
the newest and of the older held iteration, payloads of random size
including 0 and over capacity) applied at once to
  * the reference's own ckpt::HostSnapshots and ckpt::NeighborBuffer
    (proj/src/ckpt.cpp:35-105, compiled into oracle/_ref by oracle/Makefile),
  * the facade's ckpt::HostSnapshots over the device slots (include/ftsim_capi.h),
  * an ffx replica written by the snapshot kernel (the holder's view),
and compared after every step: newest / previous, and framed(it) /
framed_at(it) for every iteration -- the bytes, or absence -- must agree.
Skipped where the reference library was not built (it needs the reference
checkout at build time)."""
import ctypes
import os
import random

import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CAP = 20_000


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


@pytest.fixture(scope="module")
def ref():
    r = orc.ref_lib()
    if r is None or not hasattr(r, "ref_hs_create"):
        pytest.skip("oracle/_ref not built")
    return r


@pytest.fixture(scope="module")
def fl():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2512_03644_b200", "libftsim_b200.so"))
    P, U64 = ctypes.c_void_p, ctypes.c_uint64
    lib.ftsim_hs_create.argtypes = [ctypes.c_uint16] * 3 + [U64, ctypes.POINTER(P)]
    lib.ftsim_hs_take.argtypes = [P, U64, P, U64]
    lib.ftsim_hs_newest.argtypes = [P, ctypes.POINTER(U64)]
    lib.ftsim_hs_framed.argtypes = [P, U64, P, U64, ctypes.POINTER(U64)]
    lib.ftsim_hs_destroy.argtypes = [P]
    return lib


def ref_framed(ref, fn, h, it):
    buf = ctypes.create_string_buffer(CAP + 64)
    n = fn(h, it, buf, CAP + 64)
    return buf.raw[:n] if n else None


def fac_framed(fl, h, it):
    n = ctypes.c_uint64()
    if fl.ftsim_hs_framed(h, it, None, 0, ctypes.byref(n)) != 0:
        return None
    buf = ctypes.create_string_buffer(n.value)
    assert fl.ftsim_hs_framed(h, it, buf, n.value, ctypes.byref(n)) == 0
    return buf.raw[:n.value]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_two_version_semantics_match_the_reference(ffx, ref, fl, seed):
    rng = random.Random(seed)
    me = (1, 0, 0)
    hs_ref = ref.ref_hs_create(*me, CAP)
    nb_ref = ref.ref_nb_create(*me)
    hs_fac = ctypes.c_void_p()
    assert fl.ftsim_hs_create(*me, CAP, ctypes.byref(hs_fac)) == 0
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, me)
    rep = holder.create_replica(me, CAP, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    try:
        newest = 0
        for step in range(60):
            r = rng.random()
            if r < 0.25 and newest:
                it = newest                      # re-take the newest
            elif r < 0.45 and newest > 1:
                it = rng.randint(max(1, newest - 2), newest - 1)  # an older one (held or evicted)
            else:
                it = newest + rng.randint(1, 2)  # a fresh iteration
            n = rng.choice([0, 1, 31, 4096, 4097, rng.randint(1, CAP), CAP, CAP + 1 + rng.randint(0, 99)])
            payload = bytes(rng.getrandbits(8) for _ in range(n))
            buf = ctypes.create_string_buffer(payload, max(1, n))
            rc_ref = ref.ref_hs_take(hs_ref, it, buf, n)
            rc_fac = fl.ftsim_hs_take(hs_fac, it, buf, n)
            # the ffx replica written by the snapshot kernel (device payload)
            origin.clear_regions()
            dev = torch.frombuffer(bytearray(payload or b"\0"), dtype=torch.uint8).cuda()
            if n:
                origin.register(ffx.REGION_BLOB, dev, nbytes=n)
            try:
                origin.snapshot(it)
                rc_ffx = 0
            except ffx.ConfigError:
                rc_ffx = 1
            torch.cuda.synchronize()
            assert rc_ref == rc_fac == (1 if n > CAP else 0) == rc_ffx, (step, it, n, rc_ref, rc_fac, rc_ffx)
            if rc_ref == 0:
                newest = max(newest, it)
                f = ref_framed(ref, ref.ref_hs_framed, hs_ref, it)
                assert ref.ref_nb_store(nb_ref, f, len(f)) == 0  # the holder accepts it
            # newest / previous
            a, b = ctypes.c_uint64(), ctypes.c_uint64()
            has_n = ref.ref_hs_newest(hs_ref, ctypes.byref(a))
            has_p = ref.ref_hs_previous(hs_ref, ctypes.byref(b))
            fn = ctypes.c_uint64()
            assert (fl.ftsim_hs_newest(hs_fac, ctypes.byref(fn)) == 0) == bool(has_n)
            if has_n:
                assert fn.value == a.value
                assert rep.newest() == a.value
            nbn = ctypes.c_uint64()
            ref.ref_nb_newest(nb_ref, ctypes.byref(nbn))
            held = rep.held()
            want_held = sorted([a.value] + ([b.value] if has_p else [])) if has_n else []
            assert sorted(held) == want_held, (step, held, want_held)
            if has_n:
                assert nbn.value == a.value
            # every iteration's frame: bytes or absence agree everywhere
            for q in range(1, newest + 3):
                fr = ref_framed(ref, ref.ref_hs_framed, hs_ref, q)
                assert fac_framed(fl, hs_fac, q) == fr, (step, q)
                assert ref_framed(ref, ref.ref_nb_framed_at, nb_ref, q) == fr, (step, q)
                if fr is None:
                    assert q not in held
                else:
                    assert rep.export_frame(q) == fr, (step, q)
    finally:
        torch.cuda.synchronize()
        ref.ref_hs_free(hs_ref)
        ref.ref_nb_free(nb_ref)
        fl.ftsim_hs_destroy(hs_fac)
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()
