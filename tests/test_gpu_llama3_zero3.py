"""BASELINE configs[2]/[3] at full size on one B200: the Llama-3 8B ZeRO-3
d=8 shard a DP rank owns -- six regions (fp32 master, Adam m, Adam v, bf16
params, data-loader cursor, RNG; paper_2512_03644_b200/state.py), 14.05 GB --
snapshotted twice into its ring neighbour's two-version replica, lost, and
restored bit-exactly.

Size-independent properties at the full size (the oracle is far too slow to
materialize 14 GB): every restored region is blob_is_sound, sampled slices
of every region equal the oracle's materialize_range, the slot's checksum
table entries at those slices equal the oracle's FNV, the older version
restores too, and the SNP1 export splits into ceil(N / FFX_FRAME_PART_BYTES)
frames that the oracle's unpack (the reference framing rules: header,
length, whole-payload FNV-1a-64, storage.cpp:74-101) accepts.
Sizes: evolution.cpp:15-19, ckpt.cpp:13-21; the 4 GiB frame limit
storage.cpp:48-49.
"""
import os

import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("FFX_FULL_SIZE", "1") == "0", reason="full-size disabled")]

PART = 0xFFFFF000
SLICE = 4096


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def host(t):
    return bytes(t.cpu().numpy().tobytes())


def sample_slices(nbytes):
    ns = (nbytes + SLICE - 1) // SLICE
    return sorted({0, 1, 7919 % ns, ns // 3, ns // 2, ns - 2, ns - 1} & set(range(ns)))


def check_region(ffx, t, r, label):
    if r.literal is not None:
        assert host(t) == r.literal, label
        return
    assert ffx.blob_is_sound(t), label
    for s in sample_slices(r.nbytes):
        lo = s * SLICE
        ln = min(SLICE, r.nbytes - lo)
        assert host(t[lo:lo + ln]) == orc.materialize_range(r.digest, r.nbytes, lo, ln), (label, s)


def test_llama3_8b_zero3_d8_shard_snapshot_recover_export(ffx):
    from paper_2512_03644_b200 import state
    free, _ = torch.cuda.mem_get_info()
    d, dp = 8, 1
    regs1 = state.zero3_shard(state.PHI_LLAMA3_8B, d, dp, iteration=1)
    regs2 = state.zero3_shard(state.PHI_LLAMA3_8B, d, dp, iteration=2)
    n = state.shard_bytes(regs1)
    assert n == 14_052_957_216
    if free < 3.3 * n:
        pytest.skip("needs ~47 GB of free HBM")
    spec = ffx.make_spec(d=d, phi=state.PHI_LLAMA3_8B, distributed=True)
    assert sum(r.nbytes for r in regs1[:3]) == ffx.razor(spec).unique_bytes_per_device
    holder = ffx.Context(0, spec, (2, 0, 0), SLICE)
    origin = ffx.Context(0, spec, (dp, 0, 0), SLICE)
    rep = holder.create_replica((dp, 0, 0), n, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    try:
        ts = state.allocate(ffx, torch, origin, regs1)
        plan = origin.plan()
        assert plan.registered_unique_bytes == n and plan.num_unique_regions == 6
        origin.snapshot(1)
        for t, r in zip(ts, regs2):  # the optimizer step rewrites the state in place
            state.fill(ffx, torch, t, r)
        origin.snapshot(2)
        torch.cuda.synchronize()
        assert sorted(rep.held()) == [1, 2]
        slot2 = rep.held()[2]
        info = rep.slot_info(slot2)
        assert info.payload_len == n and info.num_regions == 6
        runs = ffx.slice_runs([r.nbytes for r in regs2], SLICE)  # the table's slicing (head split included)
        assert runs[0][3] == SLICE // 4 and len(runs) == 7  # the first region (> 192 MiB) opens with a small-slice head
        assert info.num_slices == plan.num_slices == runs[-1][4] + (runs[-1][2] + SLICE - 1) // SLICE
        assert rep.slot_regions(slot2) == [(r.kind, r.nbytes) for r in regs2]

        # the slot's checksum table at the sampled slices = the oracle's FNV
        pay, sums = rep.slot_ptrs(slot2)
        table = torch.empty(info.num_slices, dtype=torch.int64, device="cuda")
        scratch = torch.empty((info.num_slices * 8 + SLICE - 1) // SLICE, dtype=torch.int64, device="cuda")
        ffx.copy_checksums(table, sums, SLICE, scratch, nbytes=info.num_slices * 8)
        tab = table.cpu()
        for reg, off, nb, sl, first in runs:
            r = regs2[reg]
            if r.digest is not None:
                ns = (nb + sl - 1) // sl
                for s in sorted({0, 1, ns // 2, ns - 1} & set(range(ns))):
                    lo = off + s * sl
                    ln = min(sl, off + nb - lo)
                    want = orc.materialize_range(r.digest, r.nbytes, lo, ln)
                    assert int(tab[first + s]) & ffx.U64_MAX == orc.fnv1a64(want), (reg, off, s)
        del table, scratch, tab

        # failure of the origin rank: every region poisoned, restored from the replica
        origin.inject(ffx.FAULT_POISON_STATE)
        rpt = origin.recover(view, 2)
        assert rpt.bad_slices == 0 and rpt.bytes == n
        for t, r in zip(ts, regs2):
            check_region(ffx, t, r, ("it2", r.kind))
        # the previous version is intact and restorable (two-version rule, ckpt.cpp:92)
        origin.inject(ffx.FAULT_POISON_STATE)
        rpt = origin.recover(view, 1)
        assert rpt.bad_slices == 0
        for t, r in zip(ts, regs1):
            check_region(ffx, t, r, ("it1", r.kind))

        # a flipped byte deep inside Adam v is caught at the right slice
        v_off = regs2[0].nbytes + regs2[1].nbytes  # logical payload offset of ADAM_V
        off = v_off + 123_456_789
        origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (slot2 << 48) | off)
        with pytest.raises(ffx.RestoreError) as ei:
            origin.recover(view, 2)
        want_slice = ffx.slice_index(runs, 2, 123_456_789)  # per-region slicing
        assert "first slice %d" % want_slice in str(ei.value)

        # SNP1 export above 4 GiB: the parts the reference's parser accepts
        origin.inject(ffx.FAULT_CORRUPT_REPLICA, view, (slot2 << 48) | off)  # flip it back
        parts = rep.export_frame_parts(2)
        assert len(parts) == (n + PART - 1) // PART == 4
        off = 0
        for i, f in enumerate(parts):
            ln = min(PART, n - off)
            assert len(f) == 32 + ln
            rc, fields = orc.unpack(f)
            assert rc == 0, ("part", i)
            off += ln
        assert off == n
        del parts
    finally:
        view.destroy()
        rep.destroy()
        origin.close()
        holder.close()
        torch.cuda.empty_cache()
