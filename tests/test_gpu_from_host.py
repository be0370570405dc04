"""Snapshots from host memory (HostSnapshots::take(it, host_ptr, len),
ckpt.hpp:88): ffx_snapshot_from_host copies the host bytes into the
registered regions under the snapshot's own batches (ffx_snapshot_batch_span
says which bytes each batch reads).  The result must be exactly what a copy
followed by ffx_snapshot gives: the regions hold the host bytes, the slot's
table is the oracle's FNV over the slice runs, the frame is the reference's.
"""
import ctypes
import os

import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
MiB = 1 << 20
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def host(t):
    return bytes(t.cpu().numpy().tobytes())


def setup(ffx, sizes):
    spec = ffx.make_spec(d=2, phi=64, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0))
    origin = ffx.Context(0, spec, (1, 0, 0))
    rep = holder.create_replica((1, 0, 0), sum(sizes) + 4096 * len(sizes), 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    ts = [torch.zeros(n, dtype=torch.uint8, device="cuda") for n in sizes]
    for t in ts:
        origin.register(ffx.REGION_MASTER, t)
    return holder, origin, rep, view, ts


def teardown(holder, origin, rep, view, ts):
    torch.cuda.synchronize()
    view.destroy()
    rep.destroy()
    origin.close()
    holder.close()


def table(ffx, rep, slot, nsl):
    pay, sums = rep.slot_ptrs(slot)
    t = torch.empty(nsl, dtype=torch.int64, device="cuda")
    scratch = torch.empty((nsl * 8 + 4095) // 4096, dtype=torch.int64, device="cuda")
    ffx.copy_checksums(t, sums, 4096, scratch, nbytes=nsl * 8)
    return [v & ffx.U64_MAX for v in t.cpu().tolist()]


@pytest.mark.parametrize("batches,pinned", [(0, True), (1, True), (3, True), (8, False)])
def test_from_host_equals_copy_then_snapshot(ffx, batches, pinned):
    sizes = [(200 * MiB) + 4099, 5 * MiB + 3, 16]
    holder, origin, rep, view, ts = setup(ffx, sizes)
    try:
        n = sum(sizes)
        g = torch.Generator().manual_seed(batches)
        src = torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g)
        if pinned:
            src = src.pin_memory()
        payload = bytes(src.numpy().tobytes())
        origin.snapshot_from_host(4, src, batches=batches)
        torch.cuda.synchronize()
        # the regions hold the host bytes
        off = 0
        for t, nb in zip(ts, sizes):
            assert host(t) == payload[off:off + nb]
            off += nb
        # the slot: the oracle's table over the slice runs, the reference frame
        runs = ffx.slice_runs(sizes, 4096)
        want, starts = [], [0]
        for nb in sizes:
            starts.append(starts[-1] + nb)
        for reg, roff, nb, sl, first in runs:
            assert first == len(want)
            want += orc.slice_fnv(payload[starts[reg] + roff:starts[reg] + roff + nb], sl)
        slot = rep.held()[4]
        assert rep.slot_info(slot).num_slices == len(want)
        assert table(ffx, rep, slot, len(want)) == want
        assert rep.export_frame(4) == orc.pack_blob((1, 0, 0), 4, 1, payload)
        assert holder.verify_held(rep, 4).bad_slices == 0
        origin.inject(ffx.FAULT_POISON_STATE)
        assert origin.recover(view, 4).bad_slices == 0
        assert b"".join(host(t) for t in ts) == payload
    finally:
        teardown(holder, origin, rep, view, ts)


def test_batch_spans_tile_the_payload(ffx):
    sizes = [(200 * MiB) + 4099, 0, 5 * MiB + 3, 16]
    holder, origin, rep, view, ts = setup(ffx, sizes)
    try:
        for nb in (1, 2, 5, 8, 13):
            got = origin.snapshot_begin(7 + nb, batches=nb)
            assert got == nb
            spans = []
            for b in range(nb):
                spans.append(origin.batch_span(b))
                origin.snapshot_next()
            torch.cuda.synchronize()
            assert spans[0][0] == 0 and spans[-1][1] == sum(sizes)
            for (lo, hi), (lo2, hi2) in zip(spans, spans[1:]):
                assert lo <= hi == lo2 <= hi2  # consecutive, increasing
        with pytest.raises(ffx.StateError):
            origin.batch_span(0)  # nothing pending
    finally:
        teardown(holder, origin, rep, view, ts)


def test_from_host_refuses_a_wrong_length(ffx):
    sizes = [1 * MiB, 77]
    holder, origin, rep, view, ts = setup(ffx, sizes)
    try:
        src = torch.zeros(sum(sizes) + 1, dtype=torch.uint8)
        with pytest.raises(ffx.ConfigError):
            origin.snapshot_from_host(1, src)
        origin.snapshot_from_host(1, src, nbytes=sum(sizes))  # the right length is taken
        torch.cuda.synchronize()
        assert rep.newest() == 1
    finally:
        teardown(holder, origin, rep, view, ts)


def test_facade_take_from_host_is_the_reference_frame(ffx):
    """ckpt::HostSnapshots::take(it, host_ptr, len) through the facade's C
    entry points (include/ftsim_capi.h) with a payload large enough to be
    pipelined in batches (and the head run), pinned and pageable."""
    fl = ctypes.CDLL(os.path.join(ROOT, "paper_2512_03644_b200", "libftsim_b200.so"))
    P, U64 = ctypes.c_void_p, ctypes.c_uint64
    fl.ftsim_hs_create.argtypes = [ctypes.c_uint16] * 3 + [U64, ctypes.POINTER(P)]
    fl.ftsim_hs_take.argtypes = [P, U64, P, U64]
    fl.ftsim_hs_framed.argtypes = [P, U64, P, U64, ctypes.POINTER(U64)]
    fl.ftsim_hs_destroy.argtypes = [P]
    n = 300 * MiB + 12345
    hs = P()
    assert fl.ftsim_hs_create(2, 0, 0, n, ctypes.byref(hs)) == 0
    try:
        for it, pinned in ((1, True), (2, False)):
            src = torch.randint(0, 256, (n,), dtype=torch.uint8, generator=torch.Generator().manual_seed(it))
            if pinned:
                src = src.pin_memory()
            assert fl.ftsim_hs_take(hs, it, src.data_ptr(), n) == 0
            ln = U64()
            assert fl.ftsim_hs_framed(hs, it, None, 0, ctypes.byref(ln)) == 0
            buf = torch.empty(ln.value, dtype=torch.uint8)
            assert fl.ftsim_hs_framed(hs, it, buf.data_ptr(), ln.value, ctypes.byref(ln)) == 0
            frame = bytes(buf.numpy().tobytes())
            payload = bytes(src.numpy().tobytes())
            assert frame[:32] == orc.pack_header((2, 0, 0), it, 1, n, orc.fnv1a64(payload))
            assert frame[32:] == payload
    finally:
        fl.ftsim_hs_destroy(hs)
