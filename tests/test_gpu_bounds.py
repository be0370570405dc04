"""Out-of-bounds write checks for every kernel path (compute-sanitizer is
closed on this GPU pool -- profiles/r2_sanitizer_refused.txt -- so the
kernels are fenced with canaries instead): every buffer a kernel may touch
sits inside a larger allocation filled with a canary pattern, and after the
launch every byte outside the bytes the kernel is allowed to write must still
be the canary -- source regions (read-only), the replica's unused table
entries, region-alignment gaps, slot padding and the other slot, recovery
destinations and checksum outputs.  Ragged sizes and 16-byte misalignment put
every warp-task kind (tensor TMA, register path, tiny regions) in play."""
import ctypes

import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CANARY = 0xA5
SLICE = 4096
GAP = 64 * 1024


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def align_up(x, a):
    return (x + a - 1) // a * a


def layout(capacity, slice_bytes=SLICE):
    """ffx_layout.h make_layout (the slot geometry)."""
    payload_cap = align_up(capacity, 256) + 16 * 256
    table_cap = (capacity + slice_bytes - 1) // slice_bytes + 16
    payload_off = align_up(256 + 8 * table_cap + 32, 4096)
    stride = align_up(payload_off + payload_cap, 1 << 21)
    return payload_off, table_cap, stride


class Fenced:
    """Views of `sizes` bytes (at offsets `misalign` past 16-byte alignment)
    inside one canary-filled buffer, GAP bytes apart."""

    def __init__(self, sizes, misalign=0):
        self.offs = []
        o = GAP
        for n in sizes:
            o = align_up(o, 256) + misalign
            self.offs.append(o)
            o += n + GAP
        self.buf = torch.full((o + GAP,), CANARY, dtype=torch.uint8, device="cuda")
        self.views = [self.buf[a:a + n] for a, n in zip(self.offs, sizes)]
        self.sizes = list(sizes)

    def outside_intact(self):
        host = self.buf.cpu()
        mask = torch.ones_like(host, dtype=torch.bool)
        for a, n in zip(self.offs, self.sizes):
            mask[a:a + n] = False
        return bool((host[mask] == CANARY).all())


def read_dev(ffx, ptr, n):
    out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    ffx.check(ffx.lib.ffx_memcpy(ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ptr), n, None, 1), "D2H")
    return out


def fill_dev(ffx, ptr, n):
    src = torch.full((n,), CANARY, dtype=torch.uint8, pin_memory=True)
    ffx.check(ffx.lib.ffx_memcpy(ctypes.c_void_p(ptr), ctypes.c_void_p(src.data_ptr()), n, None, 1), "H2D")


def replica_allowed(sizes, nslices, payload_off):
    """Byte ranges of a slot a snapshot may write: meta, the used table
    entries, the SNP1 header, each region's payload bytes."""
    rng = [(0, 256 + 8 * nslices), (payload_off - 32, payload_off)]
    o = 0
    for n in sizes:
        rng.append((payload_off + o, payload_off + o + n))
        o = align_up(o + n, 256)
    return rng


def check_slot(ffx, rep, slot, stride, allowed):
    pay, sums = rep.slot_ptrs(slot)
    base = sums - 256
    host = read_dev(ffx, base, stride)
    mask = torch.ones(stride, dtype=torch.bool)
    for a, b in allowed:
        mask[a:b] = False
    return bool((host[mask] == CANARY).all())


@pytest.mark.parametrize("mode", ["fused", "batched", "tasks", "split", "split_ce", "verify", "hybrid"])
@pytest.mark.parametrize("misalign", [0, 16])
def test_snapshot_and_recover_write_only_their_bytes(ffx, mode, misalign):
    sizes = [3 * (1 << 20) + 4099, 16, 200_000 + 3]
    cap = sum(sizes) + 4096
    spec = ffx.make_spec(d=2, phi=1 << 20, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0), SLICE)
    origin = ffx.Context(0, spec, (1, 0, 0), SLICE)
    rep = holder.create_replica((1, 0, 0), cap, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    payload_off, table_cap, stride = layout(cap)
    try:
        pay0, sums0 = rep.slot_ptrs(0)
        fill_dev(ffx, sums0 - 256, 2 * stride)  # both slots: canary everywhere
        src = Fenced(sizes, misalign)
        digests = [orc.optimizer_init(20 + i, 1, 0, 0, True) for i in range(len(sizes))]
        for v, n, d in zip(src.views, sizes, digests):
            if n >= 32:
                ffx.materialize(v, d)
            else:
                v.copy_(torch.arange(n, dtype=torch.uint8, device="cuda"))
            origin.register(ffx.REGION_MASTER, v)
        before = src.buf.clone()
        kw = {"fused": {}, "batched": {"batches": 3, "max_ctas": 8}, "tasks": {"batches": 3, "task_ctas": True},
              "split": {"split": True, "batches": 2, "hash_batches": 2},
              "split_ce": {"split": True, "copy_engine": True, "hash_ctas": 16},
              "verify": {"verify_on_store": True},
              "hybrid": {"split": True, "copy_engine": True, "fused_permille": 400}}[mode]
        origin.snapshot(1, **kw)
        torch.cuda.synchronize()
        assert torch.equal(src.buf, before), "a snapshot wrote into its source regions"
        nsl = sum((n + SLICE - 1) // SLICE for n in sizes)
        slot = rep.held()[1]
        assert check_slot(ffx, rep, slot, stride, replica_allowed(sizes, nsl, payload_off)), "slot overrun"
        assert check_slot(ffx, rep, 1 - slot, stride, []), "the other slot was touched"
        want = b"".join(bytes(v.cpu().numpy().tobytes()) for v in src.views)
        assert rep.export_frame(1) == orc.pack_blob((1, 0, 0), 1, 1, want)
        # recovery into fenced destinations (the state is lost: re-register fresh buffers)
        dst = Fenced(sizes, misalign)
        origin.clear_regions()
        for v in dst.views:
            origin.register(ffx.REGION_MASTER, v)
        rpt = origin.recover(view, 1)
        assert rpt.bad_slices == 0
        assert dst.outside_intact(), "recovery wrote outside its destinations"
        assert b"".join(bytes(v.cpu().numpy().tobytes()) for v in dst.views) == want
    finally:
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()


@pytest.mark.parametrize("n", [1, 4095, 4097, 3 * (1 << 20) + 77])
def test_checksum_outputs_stay_in_bounds(ffx, n):
    src = Fenced([n], 3)
    ffx.materialize(src.views[0], orc.optimizer_init(1, 0, 0, 0, True)) if n >= 32 else src.views[0].fill_(7)
    nsl = (n + SLICE - 1) // SLICE
    out = Fenced([nsl * 8])
    before = src.buf.clone()
    ffx.slice_checksums(src.views[0], SLICE, out.views[0])
    torch.cuda.synchronize()
    assert torch.equal(src.buf, before)
    assert out.outside_intact()
    data = bytes(src.views[0].cpu().numpy().tobytes())
    got = out.views[0].cpu().view(torch.int64).tolist()
    assert [g & ffx.U64_MAX for g in got] == [orc.fnv1a64(data[i:i + SLICE]) for i in range(0, n, SLICE)]
    assert ffx.checksum64(src.views[0]) == orc.fnv1a64(data)
    # fused copy + checksums into a fenced destination
    dst = Fenced([n], 9)
    out2 = Fenced([nsl * 8])
    ffx.copy_checksums(dst.views[0], src.views[0], SLICE, out2.views[0])
    torch.cuda.synchronize()
    assert dst.outside_intact() and out2.outside_intact()
    assert bytes(dst.views[0].cpu().numpy().tobytes()) == data
