"""examples/c_snapshot.c on the B200: the backup / failure / recovery path
driven from plain C through include/ffx.h (no Python, no torch)."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_host_snapshot_and_recover(tmp_path):
    exe = tmp_path / "c_snapshot"
    subprocess.run(["gcc", "-std=c99", "-O2", "-I" + os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "c_snapshot.c"),
                    "-L" + os.path.join(ROOT, "paper_2512_03644_b200"), "-lffx",
                    "-Wl,-rpath," + os.path.join(ROOT, "paper_2512_03644_b200"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["ok"] is True and out["newest"] == 3 and out["bad_slices"] == 0
