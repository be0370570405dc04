"""Pin the CPU oracle (oracle/ffx_oracle.c) before trusting it.

1. Known-answer tests held by the reference's own suite
   (proj/tests/test_evolution.cpp:37-50, proj/tests/test_ckpt.cpp:50-72).
2. Golden vectors produced by the reference itself (tests/golden/
   reference_vectors.json, written by oracle/gen_golden.py from
   oracle/_ref/libftsim_ref.so).
3. When oracle/_ref is built here, a direct randomized cross-check.
"""
import hashlib
import json
import os
import random

import pytest

import pyoracle as orc

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.json")))


def test_fnv_kat_reference_suite():
    # proj/tests/test_evolution.cpp:44-50
    assert orc.fnv1a64(b"") == 0xcbf29ce484222325
    assert orc.fnv1a64(b"a") == 0xaf63dc4c8601ec8c
    assert orc.fnv1a64(b"foobar") == 0x85944171f73967e8


def test_sha256_kat_reference_suite():
    # proj/tests/test_evolution.cpp:37-42 (OpenSSL, the reference's own dependency)
    assert orc.sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    assert orc.sha256(b"").hex() == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"


def test_fnv_golden():
    for k, v in GOLDEN["fnv_kat"].items():
        assert orc.fnv1a64(k.encode()) == int(v, 16)


def test_digests_golden():
    g = GOLDEN["digests"]
    for dp in range(4):
        assert orc.optimizer_init(42, dp, 0, 0, True).hex() == g["opt_42_d%dp0t0_dist" % dp]
    assert orc.optimizer_init(42, 0, 0, 0, False).hex() == g["opt_42_d0p0t0_shared"]
    assert orc.optimizer_init(99, 2, 1, 3, True).hex() == g["opt_99_d2p1t3_dist"]
    assert orc.weights_init(42, 0, 0).hex() == g["w_42_p0t0"]
    assert orc.weights_init(1, 1, 0).hex() == g["w_1_p1t0"]


def _digest(name):
    return bytes.fromhex(GOLDEN["digests"]["opt_42_%sp0t0_dist" % name])


@pytest.mark.parametrize("entry", GOLDEN["blobs"], ids=lambda e: "%s-%d" % (e["digest"], e["bytes"]))
def test_materialize_golden(entry):
    b = orc.materialize(_digest(entry["digest"]), entry["bytes"])
    assert len(b) == entry["bytes"]
    assert hashlib.sha256(b).hexdigest() == entry["sha256"]
    assert b[:48].hex() == entry["head"] and b[-16:].hex() == entry["tail"]
    assert orc.fnv1a64(b) == int(entry["fnv"], 16)
    assert orc.blob_is_sound(b) == bool(entry["sound"])
    for s, table in entry.get("slices", {}).items():
        assert ["%016x" % v for v in orc.slice_fnv(b, int(s))] == table


def test_expand_golden():
    d0 = _digest("d0")
    for e in GOLDEN["expand"]:
        assert orc.expand(d0, e["bytes"]).hex() == e["hex"]


def test_materialize_below_digest_throws():
    assert GOLDEN["materialize_16_throws"]
    with pytest.raises(ValueError):
        orc.materialize(_digest("d0"), 16)


def test_blob_is_sound_detects_flip():
    # proj/tests/test_ckpt.cpp:265-276
    b = bytearray(orc.materialize(orc.sha256(b"state"), 4096))
    assert orc.blob_is_sound(bytes(b))
    b[4000] ^= 1
    assert not orc.blob_is_sound(bytes(b))


def test_frames_golden():
    d0 = _digest("d0")
    for f in GOLDEN["frames"]:
        if "frame" in f:
            got = orc.pack_blob(tuple(f["role"]), f["iteration"], f["kind"], bytes.fromhex(f["payload"]))
            assert got.hex() == f["frame"]
        else:
            payload = orc.materialize(d0, f["materialize"][1])
            got = orc.pack_blob(tuple(f["role"]), f["iteration"], f["kind"], payload)
            assert got[:32].hex() == f["header"]


def test_header_layout_reference_suite():
    # proj/tests/test_ckpt.cpp:50-72
    fr = orc.pack_blob((3, 2, 1), 0x0102030405060708, 1, b"xy")
    assert len(fr) == 34
    assert fr[0:4] == b"SNP1" and fr[4] == 1 and fr[5] == 1
    assert fr[6] == 3 and fr[8] == 2 and fr[10] == 1
    assert fr[12] == 0x08 and fr[19] == 0x01 and fr[20] == 2
    rc, fields = orc.unpack(fr)
    assert rc == 0 and fields[:6] == (3, 2, 1, 0x0102030405060708, 1, 2)
    assert fields[6] == orc.fnv1a64(b"xy")


def test_unpack_golden():
    for name, e in GOLDEN["unpack"].items():
        rc, _ = orc.unpack(bytes.fromhex(e["frame"]))
        assert (rc != 0) == bool(e["corrupt"]), name


def test_razor_golden():
    for e in GOLDEN["razor"]:
        wr, orr, u = orc.razor(e["phi"], e["d"], e["distributed"])
        assert (wr, orr, u) == (bool(e["weights_redundant"]), bool(e["optimizer_redundant"]), e["unique"])
        assert orc.optimizer_bytes(e["phi"], e["d"], e["distributed"]) == e["optimizer_bytes"]


def test_version_window_golden():
    for e in GOLDEN["version_for_target"]:
        assert orc.version_for_target(e["held"], e["target"]) == e["out"]


@pytest.mark.skipif(orc.ref_lib() is None, reason="oracle/_ref not built")
def test_oracle_vs_reference_randomized():
    ref = orc.ref_lib()
    rng = random.Random(7)
    for _ in range(60):
        n = rng.choice([0, 1, 2, 7, 31, 32, 33, rng.randrange(0, 70000)])
        data = bytes(rng.getrandbits(8) for _ in range(n))
        assert orc.fnv1a64(data) == ref.ref_checksum64(data, n)
    import ctypes
    for _ in range(20):
        seed, dp = rng.randrange(0, 1 << 30), rng.randrange(0, 16)
        dig = ctypes_digest(ref, seed, dp)
        assert dig == orc.optimizer_init(seed, dp, 0, 0, True)
        n = rng.randrange(32, 50000)
        buf = ctypes.create_string_buffer(n)
        assert ref.ref_materialize(dig, n, buf) == 0
        assert buf.raw[:n] == orc.materialize(dig, n)


def ctypes_digest(ref, seed, dp):
    import ctypes
    b = ctypes.create_string_buffer(32)
    ref.ref_optimizer_init(seed, dp, 0, 0, 1, b)
    return b.raw[:32]


@pytest.mark.parametrize("e", GOLDEN["evolution"],
                         ids=lambda e: "r%s-g%s-it%d" % ("".join(map(str, e["role"])), "".join(map(str, e["grid"])),
                                                         e["iteration"]))
def test_evolution_golden(e):
    # optimizer_init -> optimizer_next(grad_digest(grad_contribution(window_fold)))
    # per iteration, pinned to the reference's own functions (gen_golden.py)
    dp, pp, tp = e["role"]
    d, p, t = e["grid"]
    assert orc.optimizer_at(e["seed"], dp, pp, tp, e["iteration"], d, p, t, e["batch"],
                            bool(e["distributed"])).hex() == e["digest"]


def test_evolution_uneven_batch_is_refused():
    with pytest.raises(ValueError):
        orc.optimizer_at(42, 0, 0, 0, 1, 3, batch=256)  # controller.cpp:131-132
