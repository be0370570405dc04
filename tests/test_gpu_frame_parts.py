"""SNP1 export of snapshots above the 4 GiB frame limit (storage.cpp:48-49
throws invalid_argument there; SURVEY 8 sizes: a Llama-3 8B d=8 shard is 3
frames, d=2 is 12).  ffx_replica_export_frame_part cuts the concatenated
regions into FFX_FRAME_PART_BYTES pieces, each a complete SNP1 frame whose
header the reference parser accepts and whose FNV is the oracle's."""
import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

PART = 0xFFFFF000


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def test_frames_above_4gib_split_into_parts(ffx):
    spec = ffx.make_spec(d=2, phi=1 << 30, distributed=True)
    a_bytes, b_bytes = 3 * (1 << 30) + 17, (1 << 30) + 300 * (1 << 20)  # ragged, crosses the part boundary
    total = a_bytes + b_bytes
    assert total > PART
    holder = ffx.Context(0, spec, (1, 0, 0))
    me = ffx.Context(0, spec, (0, 0, 0))
    rep = holder.create_replica((0, 0, 0), total, 1)
    view = me.open_replica(rep.export())
    me.set_target(view)
    a = torch.empty(a_bytes, dtype=torch.uint8, device="cuda")
    b = torch.empty(b_bytes + 15, dtype=torch.uint8, device="cuda")[:b_bytes]
    ffx.materialize(a, orc.optimizer_init(1, 0, 0, 0, True))
    ffx.materialize(b, orc.optimizer_init(2, 0, 0, 0, True))
    me.register(ffx.REGION_BLOB, a)
    me.register(ffx.REGION_PARAMS, b)
    try:
        me.snapshot(7)
        torch.cuda.synchronize()
        with pytest.raises(ffx.InvalidArgument):
            rep.export_frame(7)  # one frame cannot hold it (storage.cpp:48-49)
        frames = rep.export_frame_parts(7)
        assert len(frames) == 2
        payload = memoryview(bytes(a.cpu().numpy().tobytes()) + bytes(b.cpu().numpy().tobytes()))
        off = 0
        for f in frames:
            n = min(PART, total - off)
            assert len(f) == 32 + n
            rc, fields = orc.unpack(f)  # the reference framing rules: header, length, FNV
            assert rc == 0
            assert memoryview(f)[32:] == payload[off:off + n]
            assert f[:32] == orc.pack_header((0, 0, 0), 7, 1, n, orc.fnv1a64(f[32:]))
            off += n
        assert off == total
        n_out = ffx.ctypes.c_uint64()
        assert ffx.lib.ffx_replica_export_frame_part(rep.ptr, 7, 2, None, 0, ffx.ctypes.byref(n_out),
                                                     None, None) == ffx.ERANGE  # past the last part
    finally:
        view.destroy()
        rep.destroy()
        me.close()
        holder.close()


def test_small_snapshot_is_one_part_equal_to_the_single_frame(ffx):
    spec = ffx.make_spec(d=2, phi=1 << 20, distributed=True)
    holder = ffx.Context(0, spec, (1, 0, 0))
    me = ffx.Context(0, spec, (0, 0, 0))
    rep = holder.create_replica((0, 0, 0), 1 << 20, 2)
    view = me.open_replica(rep.export())
    me.set_target(view)
    s = torch.empty(1000003, dtype=torch.uint8, device="cuda")
    ffx.materialize(s, orc.optimizer_init(3, 0, 0, 0, True))
    me.register(ffx.REGION_BLOB, s)
    try:
        me.snapshot(4)
        torch.cuda.synchronize()
        parts = rep.export_frame_parts(4)
        assert parts == [rep.export_frame(4)]
    finally:
        view.destroy()
        rep.destroy()
        me.close()
        holder.close()


def test_frame_part_boundary_exactly_one_part(ffx):
    # a payload of exactly FFX_FRAME_PART_BYTES is one frame; one byte more is two
    spec = ffx.make_spec(d=2, phi=1 << 30, distributed=True)
    holder = ffx.Context(0, spec, (1, 0, 0))
    me = ffx.Context(0, spec, (0, 0, 0))
    rep = holder.create_replica((0, 0, 0), PART + 1, 1)
    view = me.open_replica(rep.export())
    me.set_target(view)
    t = torch.empty(PART + 1, dtype=torch.uint8, device="cuda")
    ffx.materialize(t, orc.optimizer_init(9, 0, 0, 0, True))
    try:
        for n, parts in ((PART, 1), (PART + 1, 2)):
            me.clear_regions()
            me.register(ffx.REGION_BLOB, t, nbytes=n)
            me.snapshot(n)
            torch.cuda.synchronize()
            n_out, p_out = ffx.ctypes.c_uint64(), ffx.ctypes.c_uint32()
            ffx.check(ffx.lib.ffx_replica_export_frame_part(rep.ptr, n, 0, None, 0, ffx.ctypes.byref(n_out),
                                                            ffx.ctypes.byref(p_out), None), "size query")
            assert p_out.value == parts and n_out.value == 32 + min(n, PART)
    finally:
        view.destroy()
        rep.destroy()
        me.close()
        holder.close()
