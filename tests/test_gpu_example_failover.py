"""examples/failover_train.py on two B200s: a ZeRO-1 training job loses a
worker PROCESS (SIGKILL), a warm spare restores its optimizer shard from the
survivor's HBM replica and joins a new process-group generation, and the run
is bit-identical to an uninterrupted one."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_real_process_failover_is_bit_identical():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "examples", "failover_train.py"),
                        "--iters", "8", "--fail-at", "4"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["bit_identical_to_uninterrupted_run"] is True
    sp = out["spare"]
    assert sp["restored_iteration"] == 4 and sp["bad_slices"] == 0
    assert sp["notice_to_verified_s"] < 1.0
    assert len(out["losses"]) == 8
