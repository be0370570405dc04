"""examples/ring_train.py under torchrun (needs >= 2 GPUs): ZeRO-1 training
with per-iteration neighbour backup survives a rank failure with a
bit-identical trajectory."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("overlap", [False, True])
def test_ring_train_example_two_ranks(overlap):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "examples", "ring_train.py"), "--iters", "10", "--fail-at", "5"]
    if overlap:  # snapshot of iteration n during iteration n+1; only the optimizer update waits
        cmd.append("--overlap")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    out = json.loads(line)
    assert out["bit_identical_to_uninterrupted_run"] is True
    assert out["recovery"]["bad_slices"] == 0 and out["recovery"]["holder"] == 0
