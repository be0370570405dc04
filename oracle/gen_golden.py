#!/usr/bin/env python3
"""Generate tests/golden/*.json from the reference itself (TEST INFRASTRUCTURE).

Runs the UNMODIFIED reference C++ (oracle/_ref/libftsim_ref.so, built by
oracle/Makefile from /root/reference/proj/src) and records its outputs for the
hot-path functions, so the GPU box -- where /root/reference does not exist --
can pin both the C restatement (oracle/ffx_oracle.c) and the CUDA path against
reference-produced vectors.

    make -C oracle && python oracle/gen_golden.py

Reference functions exercised (proj/ paths):
  checksum64            src/hash.cpp:102-110
  optimizer_init/weights_init   src/evolution.cpp:21-31
  materialize / expand  src/evolution.cpp:71-97
  blob_is_sound         src/evolution.cpp:106-110
  pack_blob / unpack    src/storage.cpp:45-101
  razor / optimizer_bytes  src/ckpt.cpp:13-21, src/evolution.cpp:15-19
  version_for_target    src/ckpt.cpp:27-33
  per-iteration evolution  src/evolution.cpp:26-69, src/dataloader.cpp:36-49, :166-171
"""
import ctypes
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden", "reference_vectors.json")

# params_per_device of the BASELINE.json configs.
MODELS = {
    "gpt2_small": 124_439_808,
    "gpt2_xl": 1_557_611_200,
    "llama3_8b": 8_030_261_248,
    "llama3_70b": 70_553_706_496,
}


def load():
    lib = ctypes.CDLL(os.path.join(HERE, "_ref", "libftsim_ref.so"))
    u8p = ctypes.POINTER(ctypes.c_uint8)
    lib.ref_checksum64.restype = ctypes.c_uint64
    lib.ref_checksum64.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    lib.ref_optimizer_init.argtypes = [ctypes.c_uint64, ctypes.c_uint16, ctypes.c_uint16,
                                       ctypes.c_uint16, ctypes.c_int, ctypes.c_void_p]
    lib.ref_weights_init.argtypes = [ctypes.c_uint64, ctypes.c_uint16, ctypes.c_uint16,
                                     ctypes.c_void_p]
    lib.ref_materialize.restype = ctypes.c_int
    lib.ref_materialize.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    lib.ref_expand.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    lib.ref_blob_is_sound.restype = ctypes.c_int
    lib.ref_blob_is_sound.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    lib.ref_optimizer_bytes.restype = ctypes.c_uint64
    lib.ref_optimizer_bytes.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int]
    lib.ref_razor.restype = ctypes.c_uint64
    lib.ref_razor.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_int)]
    lib.ref_version_for_target.restype = ctypes.c_int
    lib.ref_version_for_target.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    lib.ref_pack_blob.restype = ctypes.c_int
    lib.ref_pack_blob.argtypes = [ctypes.c_uint16, ctypes.c_uint16, ctypes.c_uint16,
                                  ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p,
                                  ctypes.c_uint64, ctypes.c_void_p]
    lib.ref_optimizer_at.restype = ctypes.c_int
    lib.ref_optimizer_at.argtypes = [ctypes.c_uint64] + [ctypes.c_uint16] * 3 + [ctypes.c_uint32] * 4 + \
        [ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p]
    lib.ref_unpack_ok.restype = ctypes.c_int
    lib.ref_unpack_ok.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    del u8p
    return lib


def buf(n):
    return (ctypes.c_uint8 * max(n, 1))()


def fnv(lib, data: bytes) -> int:
    return lib.ref_checksum64(data, len(data))


def opt_init(lib, seed, dp, pp, tp, dist=True) -> bytes:
    b = buf(32)
    lib.ref_optimizer_init(seed, dp, pp, tp, int(dist), b)
    return bytes(b)


def w_init(lib, seed, pp, tp) -> bytes:
    b = buf(32)
    lib.ref_weights_init(seed, pp, tp, b)
    return bytes(b)


def materialize(lib, digest: bytes, n: int) -> bytes:
    b = buf(n)
    rc = lib.ref_materialize(digest, n, b)
    if rc != 0:
        raise ValueError("reference threw invalid_argument")
    return bytes(b)[:n]


def pack(lib, role, it, kind, payload: bytes) -> bytes:
    b = buf(32 + len(payload))
    rc = lib.ref_pack_blob(role[0], role[1], role[2], it, kind, payload, len(payload), b)
    assert rc == 0
    return bytes(b)[: 32 + len(payload)]


def slices(lib, data: bytes, s: int):
    return ["%016x" % fnv(lib, data[o:o + s]) for o in range(0, len(data), s)]


def main():
    lib = load()
    g = {"generator": "oracle/gen_golden.py over oracle/_ref/libftsim_ref.so (reference proj/src)"}

    g["fnv_kat"] = {k: "%016x" % fnv(lib, k.encode()) for k in ["", "a", "foobar", "xy", "payload"]}

    digests = {}
    for dp in range(4):
        digests["opt_42_d%dp0t0_dist" % dp] = opt_init(lib, 42, dp, 0, 0, True).hex()
    digests["opt_42_d0p0t0_shared"] = opt_init(lib, 42, 0, 0, 0, False).hex()
    digests["opt_99_d2p1t3_dist"] = opt_init(lib, 99, 2, 1, 3, True).hex()
    digests["w_42_p0t0"] = w_init(lib, 42, 0, 0).hex()
    digests["w_1_p1t0"] = w_init(lib, 1, 1, 0).hex()
    g["digests"] = digests

    # Per-iteration optimizer digests: GPT-2 small d=2 ranks over
    # iterations 0..10 (configs[0]), a d=8 rank, a p x t grid, a shared optimizer.
    evolution = []
    for (dp, pp, tp, d, p, t, batch, n, dist) in (
            [(r, 0, 0, 2, 1, 1, 256, n, 1) for r in (0, 1) for n in range(11)] +
            [(5, 0, 0, 8, 1, 1, 256, 4, 1), (1, 1, 1, 2, 2, 2, 256, 3, 1), (0, 0, 0, 2, 1, 1, 256, 2, 0)]):
        b = buf(32)
        assert lib.ref_optimizer_at(42, dp, pp, tp, d, p, t, batch, n, dist, b) == 0
        evolution.append({"seed": 42, "role": [dp, pp, tp], "grid": [d, p, t], "batch": batch, "iteration": n,
                          "distributed": dist, "digest": bytes(b).hex()})
    g["evolution"] = evolution

    # Blobs: whole-payload FNV, slice tables at several slice sizes, SHA-256 of
    # the bytes (compact full-content pin), and the first/last bytes.
    blobs = []
    d0 = bytes.fromhex(digests["opt_42_d0p0t0_dist"])
    d1 = bytes.fromhex(digests["opt_42_d1p0t0_dist"])
    sizes = [32, 33, 39, 40, 41, 45, 47, 48, 64, 100, 255, 256, 257, 4095, 4096, 4097,
             65536 + 13, 1 << 20, (1 << 20) + 7, 3 * (1 << 20) + 1001]
    for name, d in [("d0", d0), ("d1", d1)]:
        for n in sizes:
            b = materialize(lib, d, n)
            e = {"digest": name, "bytes": n, "fnv": "%016x" % fnv(lib, b),
                 "sha256": hashlib.sha256(b).hexdigest(),
                 "head": b[:48].hex(), "tail": b[-16:].hex(),
                 "sound": lib.ref_blob_is_sound(b, n)}
            if n >= 4096:
                e["slices"] = {str(s): slices(lib, b, s) for s in (256, 4096, 65536) if n // s <= 4096}
            blobs.append(e)
    g["blobs"] = blobs

    # expand() on its own (no prefix) including 0..13 byte edge cases.
    g["expand"] = [{"bytes": n, "hex": (lambda b: (lib.ref_expand(d0, n, b), bytes(b)[:n])[1])(buf(n)).hex()}
                   for n in [0, 1, 7, 8, 13, 16, 24, 77]]

    # materialize below the digest size throws.
    try:
        materialize(lib, d0, 16)
        g["materialize_16_throws"] = False
    except ValueError:
        g["materialize_16_throws"] = True

    # SNP1 frames (storage.hpp:12-25): header golden bytes for the test_ckpt.cpp case
    # and for synthetic blobs at iteration 9.
    frames = []
    frames.append({"role": [3, 2, 1], "iteration": 0x0102030405060708, "kind": 1,
                   "payload": b"xy".hex(), "frame": pack(lib, (3, 2, 1), 0x0102030405060708, 1, b"xy").hex()})
    frames.append({"role": [1, 0, 0], "iteration": 3, "kind": 1, "payload": "",
                   "frame": pack(lib, (1, 0, 0), 3, 1, b"").hex()})
    frames.append({"role": [0, 0, 0], "iteration": 7, "kind": 0, "payload": b"payload".hex(),
                   "frame": pack(lib, (0, 0, 0), 7, 0, b"payload").hex()})
    for n in [45, 4096, 1 << 20]:
        b = materialize(lib, d0, n)
        f = pack(lib, (0, 0, 0), 9, 1, b)
        frames.append({"role": [0, 0, 0], "iteration": 9, "kind": 1, "materialize": ["d0", n],
                       "header": f[:32].hex()})
    g["frames"] = frames

    # Validation outcomes of unpack_blob (storage.cpp:74-101) on damaged frames.
    base = pack(lib, (0, 0, 0), 7, 0, b"payload")
    def damaged(mut):
        f = bytearray(base)
        mut(f)
        return bytes(f)
    cases = {
        "ok": base,
        "flip_payload": damaged(lambda f: f.__setitem__(32 + 3, f[32 + 3] ^ 1)),
        "bad_magic": damaged(lambda f: f.__setitem__(0, ord("X"))),
        "bad_version": damaged(lambda f: f.__setitem__(4, 9)),
        "bad_kind": damaged(lambda f: f.__setitem__(5, 7)),
        "short": base[:16],
        "long": base + b"\0",
    }
    g["unpack"] = {k: {"frame": v.hex(), "corrupt": lib.ref_unpack_ok(v, len(v))} for k, v in cases.items()}

    # Sizing (razor) at the BASELINE configs and the test_ckpt.cpp shapes.
    razor = []
    for model, phi in MODELS.items():
        for d in (1, 2, 4, 8):
            for dist in (0, 1):
                fl = (ctypes.c_int * 2)()
                u = lib.ref_razor(phi, d, dist, fl)
                razor.append({"model": model, "phi": phi, "d": d, "distributed": dist,
                              "unique": u, "weights_redundant": fl[0], "optimizer_redundant": fl[1],
                              "optimizer_bytes": lib.ref_optimizer_bytes(phi, d, dist)})
    for phi, d, dist in [(10, 7, 1), (1_000_000_000, 4, 1), (1_000_000, 4, 0), (1_000_000_000, 1, 0),
                         (1_000_000_000, 1, 1), (64, 2, 1), (64, 2, 0)]:
        fl = (ctypes.c_int * 2)()
        u = lib.ref_razor(phi, d, dist, fl)
        razor.append({"phi": phi, "d": d, "distributed": dist, "unique": u,
                      "weights_redundant": fl[0], "optimizer_redundant": fl[1],
                      "optimizer_bytes": lib.ref_optimizer_bytes(phi, d, dist)})
    g["razor"] = razor

    g["version_for_target"] = [{"held": h, "target": t, "out": lib.ref_version_for_target(h, t)}
                               for h, t in [(7, 7), (8, 7), (9, 7), (6, 7), (0, 0), (1, 0), (2**64 - 1, 2**64 - 2)]]

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    sys.exit(main())
