"""CPU-side checks of the C ABI (no GPU compute calls).

- libffx.so loads and exports every symbol include/ffx.h declares.
- The host-only entry points (sizing, version window, SNP1 header, domain
  layout, recovery planning) agree with the oracle and the reference's golden
  vectors / unit-test expectations.
"""
import ctypes
import itertools
import json
import os
import re

import pytest

import pyoracle as orc
from paper_2512_03644_b200 import ffx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_vectors.json")))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ffx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(ffx_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 40
    lib = ctypes.CDLL(ffx.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the binding covers the whole ABI
    assert sorted(ffx.SIGNATURES) == syms


def test_abi_version():
    assert ffx.lib.ffx_abi_version() == ffx.ABI_VERSION


def test_razor_matches_reference():
    for e in GOLDEN["razor"]:
        spec = ffx.make_spec(d=e["d"], phi=e["phi"], distributed=e["distributed"])
        p = ffx.razor(spec)
        assert (p.weights_redundant, p.optimizer_redundant, p.unique_bytes_per_device) == \
            (e["weights_redundant"], e["optimizer_redundant"], e["unique"])
        assert ffx.optimizer_bytes(spec) == e["optimizer_bytes"]
        assert ffx.weights_bytes(spec) == 2 * e["phi"]


def test_razor_reference_suite_shapes():
    # proj/tests/test_ckpt.cpp:153-181 and test_evolution.cpp:193-207
    p = ffx.razor(ffx.make_spec(d=4, phi=1_000_000_000, distributed=True))
    assert p.weights_redundant and not p.optimizer_redundant and p.unique_bytes_per_device == 3_000_000_000
    p = ffx.razor(ffx.make_spec(d=4, phi=1_000_000, distributed=False))
    assert p.weights_redundant and p.optimizer_redundant and p.unique_bytes_per_device == 0
    p = ffx.razor(ffx.make_spec(d=1, phi=1_000_000_000, distributed=True))
    assert not p.weights_redundant and p.unique_bytes_per_device == 12_000_000_000
    assert ffx.optimizer_bytes(ffx.make_spec(d=7, phi=10, distributed=True)) == 18


def test_version_window():
    for e in GOLDEN["version_for_target"]:
        if e["out"] < 0:
            with pytest.raises(ffx.VersionError):
                ffx.version_for_target(e["held"], e["target"])
        else:
            assert ffx.version_for_target(e["held"], e["target"]) == e["out"]


def test_pack_header_matches_reference_frames():
    d0 = bytes.fromhex(GOLDEN["digests"]["opt_42_d0p0t0_dist"])
    for f in GOLDEN["frames"]:
        if "frame" in f:
            payload = bytes.fromhex(f["payload"])
            want = bytes.fromhex(f["frame"])[:32]
        else:
            payload = orc.materialize(d0, f["materialize"][1])
            want = bytes.fromhex(f["header"])
        got = ffx.pack_header(ffx.Role(*f["role"]), f["iteration"], f["kind"], len(payload),
                              orc.fnv1a64(payload))
        assert got == want


def test_pack_header_4gib_limit():
    # storage.cpp:48-49
    with pytest.raises(ffx.InvalidArgument):
        ffx.pack_header(ffx.Role(0, 0, 0), 1, 1, 1 << 32, 0)
    ffx.pack_header(ffx.Role(0, 0, 0), 1, 1, (1 << 32) - 1, 0)


def test_parse_header_validation_matches_reference():
    for name, e in GOLDEN["unpack"].items():
        fr = bytes.fromhex(e["frame"])
        if name == "flip_payload":
            continue  # payload checksum is checked on the device path
        if e["corrupt"]:
            with pytest.raises(ffx.CorruptSnapshot):
                ffx.parse_header(fr, len(fr))
        else:
            info = ffx.parse_header(fr, len(fr))
            assert info.iteration == 7 and info.kind == 0 and info.payload_len == 7
            assert info.checksum == orc.fnv1a64(b"payload")


def test_domain_layout():
    # domain.cpp:18-62: tp fastest, then pp, then dp; ring successor/predecessor
    spec = ffx.make_spec(d=4, p=2, t=2, num_nodes=4)
    for idx in range(16):
        r = ffx.role_of(spec, idx)
        assert r.tuple() == orc.role_of(idx, 4, 2, 2)
        assert ffx.index_of(spec, r) == idx
        assert ffx.node_of(spec, r) == idx // 4
        assert ffx.dp_neighbor(spec, r).tuple() == ((r.dp + 1) % 4, r.pp, r.tp)
        assert ffx.dp_predecessor(spec, r).tuple() == ((r.dp + 3) % 4, r.pp, r.tp)
    with pytest.raises(ffx.OutOfRange):
        ffx.role_of(spec, 16)
    with pytest.raises(ffx.OutOfRange):
        ffx.index_of(spec, ffx.Role(4, 0, 0))


def _shape(nodes, gpn, d, p, t=1):
    return ffx.make_spec(d=d, p=p, t=t, num_nodes=nodes, gpus_per_node=gpn)


def test_plan_recovery_ring_adjacency_enumeration():
    # proj/tests/test_controller.cpp:191-216
    spec = _shape(6, 1, 6, 1)
    spec.distributed_optimizer = 1
    for mask in range(1, 1 << 6):
        pods = [i for i in range(6) if mask & (1 << i)]
        adjacent = any(mask & (1 << i) and mask & (1 << ((i + 1) % 6)) for i in range(6))
        plan = ffx.plan_recovery(spec, pods, [], 40, 35)
        if adjacent:
            assert plan.kind == "fallback" and plan.resume_iteration == 35
            assert not plan.forwards and not plan.redundant_from
        else:
            assert plan.kind == "neighbor" and plan.resume_iteration == 40
            assert len(plan.forwards) == len(pods)


def test_plan_recovery_names_holders_sources_targets():
    # proj/tests/test_controller.cpp:218-276
    spec = _shape(4, 2, 4, 2)
    spec.distributed_optimizer = 1
    plan = ffx.plan_recovery(spec, [1], [], 17, 10)
    assert plan.kind == "neighbor" and plan.resume_iteration == 17
    assert plan.failed_pods == [1]
    assert [r.tuple() for r in plan.failed_roles] == [(1, 0, 0), (1, 1, 0)]
    assert len(plan.forwards) == 2 and all(f[1] == 2 and f[2] == 1 for f in plan.forwards)
    assert len(plan.redundant_from) == 2 and all(s.dp == 0 for _, s in plan.redundant_from)
    assert len(plan.lazy_backup_targets) == 2 and all(t.dp == 0 for t in plan.lazy_backup_targets)
    spec.distributed_optimizer = 0
    p2 = ffx.plan_recovery(spec, [1], [], 17, 10)
    assert p2.kind == "neighbor" and not p2.forwards and len(p2.redundant_from) == 2
    assert ffx.plan_recovery(_shape(2, 2, 2, 2), [0, 1], [], 17, 10).kind == "fallback"
    assert ffx.plan_recovery(_shape(1, 4, 1, 2, 2), [0], [], 17, 10).kind == "fallback"
    spec.distributed_optimizer = 1
    p3 = ffx.plan_recovery(spec, [1], [], 0, 0)
    assert p3.kind == "neighbor" and p3.resume_iteration == 0
    assert not p3.forwards and not p3.redundant_from and not p3.lazy_backup_targets
    assert len(p3.failed_roles) == 2


@pytest.mark.parametrize("d,p,gpn,dist", [(4, 1, 1, 1), (4, 2, 2, 1), (6, 1, 3, 0), (8, 1, 8, 1), (3, 2, 2, 1)])
def test_plan_recovery_vs_oracle(d, p, gpn, dist):
    world = d * p
    nodes = world // gpn
    spec = _shape(nodes, gpn, d, p)
    spec.distributed_optimizer = dist
    roles = [orc.role_of(i, d, p, 1) for i in range(world)]
    for k in (1, 2):
        for pods in itertools.combinations(range(nodes), min(k, nodes)):
            for extra in ([], [roles[(pods[0] * gpn + 1) % world]]):
                got = ffx.plan_recovery(spec, list(pods), [ffx.Role(*r) for r in extra], 9, 5)
                want = orc.plan_recovery(d, p, 1, gpn, dist, pods, extra, 9, 5)
                assert got.kind == want["kind"] and got.resume_iteration == want["resume"]
                assert [r.tuple() for r in got.failed_roles] == want["failed_roles"]
                assert [(f[0].tuple(), f[1], f[2]) for f in got.forwards] == want["forwards"]
                assert [(a.tuple(), b.tuple()) for a, b in got.redundant_from] == want["redundant_from"]
                assert [r.tuple() for r in got.lazy_backup_targets] == want["lazy"]


def test_plan_recovery_double_neighbour_extension():
    # Adjacent pair on an 8-ring: the reference falls back (controller.cpp:162-167);
    # with replicas at dp+1 and dp+2 the lost dp=2 is served by dp=4 (its only
    # surviving holder) and dp=3 by dp=5, so the two gathers use two holders.
    spec = _shape(8, 1, 8, 1)
    spec.distributed_optimizer = 1
    assert ffx.plan_recovery(spec, [2, 3], [], 11, 5, replicas=1).kind == "fallback"
    p = ffx.plan_recovery(spec, [2, 3], [], 11, 5, replicas=2)
    assert p.kind == "neighbor"
    holders = {f[0].dp: f[3] for f in p.forwards}
    assert holders == {2: 4, 3: 5}
    # a single loss keeps the reference's ring successor
    assert {f[0].dp: f[3] for f in ffx.plan_recovery(spec, [6], [], 11, 5, replicas=2).forwards} == {6: 7}
    assert ffx.plan_recovery(spec, [2, 3, 4], [], 11, 5, replicas=2).kind == "fallback"


def test_plain_c_host_compiles_against_the_abi(tmp_path):
    # include/ffx.h is a C header: examples/c_snapshot.c (the whole backup /
    # failure / recovery path from C99) builds and links against libffx.so
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "c_snapshot"
    r = subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Werror", "-I" + os.path.join(root, "include"),
                        os.path.join(root, "examples", "c_snapshot.c"),
                        "-L" + os.path.join(root, "paper_2512_03644_b200"), "-lffx",
                        "-Wl,-rpath," + os.path.join(root, "paper_2512_03644_b200"), "-o", str(out)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_facade_c_entry_points_exported():
    """include/ftsim_capi.h: every declared ftsim_* symbol is exported by the
    facade library (the C route to HostSnapshots for ctypes / cgo / JNI)."""
    src = open(os.path.join(ROOT, "include", "ftsim_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    syms = sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(ftsim_\w+)\s*\(", src, flags=re.M)))
    assert len(syms) == 7
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2512_03644_b200", "libftsim_b200.so"))
    assert [s for s in syms if not hasattr(lib, s)] == []


def _runs_spec(sizes, S):
    """The slice-run rule restated (ffx_layout.h region_runs / DESIGN §4.1):
    the first of fewer than 16 regions, when it holds >= 4 x 48 MiB and S is
    a multiple of 1 KiB, opens with a 48 MiB run of S/4 slices."""
    head = 48 << 20
    out, first = [], 0
    for i, nb in enumerate(sizes):
        runs = [(0, nb, S)]
        if i == 0 and len(sizes) < 16 and S % 1024 == 0 and nb >= 4 * head:
            runs = [(0, head, S // 4), (head, nb - head, S)]
        for off, b, sl in runs:
            out.append((i, off, b, sl, first))
            first += (b + sl - 1) // sl
    return out


@pytest.mark.parametrize("sizes,S", [
    ([], 4096), ([0], 4096), ([1], 256), ([192 << 20], 4096), ([(192 << 20) - 1], 4096),
    ([(192 << 20) + 4099, 5 << 20, 16], 4096), ([400 << 20, 400 << 20], 2048), ([300 << 20], 1280),
    ([300 << 20], 1536), ([1 << 30] * 15, 4096), ([1 << 30] * 16, 4096), ([14_052_957_216 // 2, 7], 1024)])
def test_slice_runs_match_the_rule(sizes, S):
    assert ffx.slice_runs(sizes, S) == _runs_spec(sizes, S)


def test_slice_runs_rejects_bad_arguments():
    with pytest.raises(ffx.FfxError):
        ffx.slice_runs([1 << 20], 100)  # not a multiple of 256
