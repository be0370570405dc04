"""GPU parity of the device primitives against the CPU oracle (bit-exact).

Every kernel result is compared with oracle/ffx_oracle.c (itself pinned to
the reference by tests/test_oracle.py) and with the reference-produced golden
vectors in tests/golden/.  Sizes cover empty, ragged, sub-vector, unaligned
and multi-slice cases; full-size behaviour is covered by properties in
test_gpu_replica.py.
"""
import hashlib
import json
import os
import random

import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def dev_bytes(data: bytes, offset: int = 0):
    """Device copy of `data` starting `offset` bytes into a fresh allocation."""
    buf = torch.zeros(len(data) + offset + 16, dtype=torch.uint8, device="cuda")
    if data:
        buf[offset:offset + len(data)] = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    return buf, buf.data_ptr() + offset


def host(t, n=None):
    return bytes(t[:n].cpu().numpy().tobytes()) if n is not None else bytes(t.cpu().numpy().tobytes())


def rand_bytes(n, seed):
    g = torch.Generator().manual_seed(seed)
    return bytes(torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g).numpy().tobytes())


SIZES = [1, 15, 16, 17, 255, 256, 4095, 4096, 4097, 100_000, (1 << 20) + 13, 3 * (1 << 20) + 1001]


@pytest.mark.parametrize("slice_bytes", [256, 4096, 65536])
@pytest.mark.parametrize("n", SIZES)
def test_slice_checksums_vs_oracle(ffx, n, slice_bytes):
    data = rand_bytes(n, n ^ slice_bytes)
    src, p = dev_bytes(data)
    ns = (n + slice_bytes - 1) // slice_bytes
    sums = torch.zeros(ns, dtype=torch.int64, device="cuda")
    ffx.slice_checksums(p, slice_bytes, sums, nbytes=n)
    got = [v & ffx.U64_MAX for v in sums.cpu().tolist()]
    assert got == orc.slice_fnv(data, slice_bytes)


@pytest.mark.parametrize("offset", [1, 3, 8])
def test_slice_checksums_unaligned(ffx, offset):
    n = 70_001
    data = rand_bytes(n, offset)
    src, p = dev_bytes(data, offset)
    sums = torch.zeros((n + 4095) // 4096, dtype=torch.int64, device="cuda")
    ffx.slice_checksums(p, 4096, sums, nbytes=n)
    assert [v & ffx.U64_MAX for v in sums.cpu().tolist()] == orc.slice_fnv(data, 4096)


def test_slice_checksums_golden(ffx):
    for e in GOLDEN["blobs"]:
        if "slices" not in e:
            continue
        d = bytes.fromhex(GOLDEN["digests"]["opt_42_%sp0t0_dist" % e["digest"]])
        blob = torch.empty(e["bytes"], dtype=torch.uint8, device="cuda")
        ffx.materialize(blob, d)
        for s, table in e["slices"].items():
            sums = torch.zeros(len(table), dtype=torch.int64, device="cuda")
            ffx.slice_checksums(blob, int(s), sums)
            assert ["%016x" % (v & ffx.U64_MAX) for v in sums.cpu().tolist()] == table


@pytest.mark.parametrize("n", [0, 1, 17, 4096, 100_003, (1 << 22) + 5])
def test_copy_checksums(ffx, n):
    data = rand_bytes(n, 11 + n)
    src, p = dev_bytes(data)
    dst = torch.zeros(n + 16, dtype=torch.uint8, device="cuda")
    sums = torch.zeros(max(1, (n + 4095) // 4096), dtype=torch.int64, device="cuda")
    ffx.copy_checksums(dst, p, 4096, sums, nbytes=n)
    assert host(dst, n) == data
    assert host(dst)[n:] == bytes(16)  # no overrun
    if n:
        assert [v & ffx.U64_MAX for v in sums.cpu().tolist()] == orc.slice_fnv(data, 4096)


def test_copy_verify_detects_each_bad_slice(ffx):
    n = 1 << 20
    data = rand_bytes(n, 5)
    src, p = dev_bytes(data)
    sums = torch.tensor([v - (1 << 64) if v >= 1 << 63 else v for v in orc.slice_fnv(data, 4096)],
                        dtype=torch.int64, device="cuda")
    dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
    res = torch.zeros(2, dtype=torch.int64, device="cuda")
    ffx.copy_verify(dst, p, 4096, sums, res, nbytes=n)
    r = res.cpu().tolist()
    assert (r[0] & ffx.U64_MAX) == ffx.U64_MAX and r[1] == 0
    assert host(dst) == data
    src[4096 * 77 + 5] ^= 0x40
    src[4096 * 200] ^= 0x01
    ffx.copy_verify(dst, p, 4096, sums, res, nbytes=n)
    r = res.cpu().tolist()
    assert r[0] == 77 and r[1] == 2


@pytest.mark.parametrize("entry", GOLDEN["blobs"], ids=lambda e: "%s-%d" % (e["digest"], e["bytes"]))
def test_materialize_golden(ffx, entry):
    d = bytes.fromhex(GOLDEN["digests"]["opt_42_%sp0t0_dist" % entry["digest"]])
    blob = torch.empty(entry["bytes"], dtype=torch.uint8, device="cuda")
    ffx.materialize(blob, d)
    b = host(blob)
    assert hashlib.sha256(b).hexdigest() == entry["sha256"]
    assert ffx.blob_is_sound(blob) == bool(entry["sound"])
    assert ffx.checksum64(blob) == int(entry["fnv"], 16)


def test_expand_golden_and_unaligned(ffx):
    d0 = bytes.fromhex(GOLDEN["digests"]["opt_42_d0p0t0_dist"])
    for e in GOLDEN["expand"]:
        n = e["bytes"]
        for off in (0, 5):
            buf = torch.zeros(n + off + 16, dtype=torch.uint8, device="cuda")
            ffx.expand(buf.data_ptr() + off, d0, n)
            h = host(buf)
            assert h[off:off + n].hex() == e["hex"]
            assert h[:off] == bytes(off) and h[off + n:] == bytes(16)


def test_materialize_below_digest_raises(ffx):
    buf = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(ffx.InvalidArgument):
        ffx.materialize(buf, bytes(32), 16)


@pytest.mark.parametrize("n", [32, 33, 45, 4096, 1_000_003])
def test_blob_check_first_bad(ffx, n):
    d = orc.sha256(b"state-%d" % n)
    blob = torch.empty(n, dtype=torch.uint8, device="cuda")
    ffx.materialize(blob, d)
    assert host(blob) == orc.materialize(d, n)
    assert ffx.blob_first_bad(blob) == ffx.U64_MAX
    if n > 40:
        k = n - 1 if n < 100 else n // 3
        blob[k] ^= 1
        assert ffx.blob_first_bad(blob) == k
        blob[40] ^= 0x80
        assert ffx.blob_first_bad(blob) == 40
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    assert not ffx.blob_is_sound(small)


WHOLE_SIZES = [0, 1, 2, 45, 255, 4095, 4096, 4097, 65536 + 13, 70_000, (1 << 20), (1 << 20) + 7,
               3 * (1 << 20) + 1001, 9_999_991]


@pytest.mark.parametrize("n", WHOLE_SIZES)
def test_whole_checksum64_vs_oracle(ffx, n):
    data = rand_bytes(n, 1000 + n)
    src, p = dev_bytes(data)
    assert ffx.checksum64(p, nbytes=n) == orc.fnv1a64(data)


@pytest.mark.parametrize("offset", [1, 7])
def test_whole_checksum64_unaligned(ffx, offset):
    n = 1_234_567
    data = rand_bytes(n, offset)
    src, p = dev_bytes(data, offset)
    assert ffx.checksum64(p, nbytes=n) == orc.fnv1a64(data)


def test_whole_checksum64_kat(ffx):
    for k, v in GOLDEN["fnv_kat"].items():
        src, p = dev_bytes(k.encode())
        assert ffx.checksum64(p, nbytes=len(k)) == int(v, 16)


def test_whole_checksum64_large_random(ffx):
    rng = random.Random(3)
    for _ in range(3):
        n = rng.randrange(16 << 20, 64 << 20)
        data = rand_bytes(n, n)
        src, p = dev_bytes(data)
        assert ffx.checksum64(p, nbytes=n) == orc.fnv1a64(data)
