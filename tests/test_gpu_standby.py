"""Time-to-restore of a REPLACED rank (north star: bit-exact single-rank
recovery of a Llama-3-8B ZeRO state in under 1 s), measured the way the
reference's flow defines it: Controller::orchestrate_recovery ->
plan_recovery (controller.cpp:144-209, :307-322) -> the holder's
framed_at -> assemble_restore (ckpt.cpp:140-167) in a new process.

Three processes on one GPU (CUDA IPC works between processes on one device),
all the native tool paper_2512_03644_b200/bin/ffx_standby over libffx's C ABI:
  holder  -- owns the two-version replica for its ring predecessor;
  origin  -- registers its six-region ZeRO-3 state, snapshots iterations 1, 2
             into the holder's replica, and is then killed with SIGKILL;
  standby -- the replacement: (warm) a spare with its CUDA context already up,
             or (cold) a process started after the failure; it plans, maps the
             holder's replica, allocates fresh regions from the slot's
             registry, gathers + verifies, and reports the time from the
             failure notice (CLOCK_MONOTONIC, after waitpid) to verified state.
The restored bytes are then checked against the oracle (head / tail of every
region) and with blob_is_sound on the device.
"""
import json
import os
import signal
import subprocess
import time

import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2512_03644_b200", "bin", "ffx_standby")


def _readline(p, want, timeout=600):
    t_end = time.time() + timeout
    while time.time() < t_end:
        line = p.stdout.readline()
        if not line:
            raise RuntimeError("%s exited (rc=%s) before '%s': %s" % (p.args[1], p.poll(), want,
                                                                       p.stderr.read() if p.stderr else ""))
        if line.startswith(want):
            return line.strip()
    raise TimeoutError(want)


def failover(tmp_path, regs1, regs2, d, phi, role=1, warm=True, device=0):
    """Run holder + origin, SIGKILL the origin, restore in a standby; returns
    (report dict, samples bytes)."""
    from paper_2512_03644_b200 import state
    if not os.path.exists(BIN):
        pytest.fail("ffx_standby not built (run __graft_entry__.build())")
    store = str(tmp_path)
    n = state.shard_bytes(regs1)
    common = ["--device", str(device), "--d", str(d), "--phi", str(phi), "--store", store]
    procs = []

    def spawn(args):
        p = subprocess.Popen([BIN] + args + common, stdin=subprocess.PIPE, stdout=subprocess.PIPE,
                             stderr=subprocess.PIPE, text=True)
        procs.append(p)
        return p

    try:
        holder = spawn(["holder", "--origin", str(role), "--capacity", str(n), "--versions", "2"])
        hdp = int(_readline(holder, "READY").split()[1])
        assert hdp == (role + 1) % d
        origin = spawn(["origin", "--role", str(role), "--holder", str(hdp),
                        "--regions", ",".join(r.spec() for r in regs1),
                        "--regions2", ",".join(r.spec() for r in regs2)])
        assert _readline(origin, "SNAPSHOTTED") == "SNAPSHOTTED 2"
        samples = os.path.join(store, "samples.bin")
        # --target: the ledger's global consistent iteration after the failure
        sb = ["standby", "--role", str(role), "--check", "--samples", samples, "--target", "2"]
        standby = None
        if warm:
            standby = spawn(sb + ["--warm"])
            _readline(standby, "ARMED")
        os.kill(origin.pid, signal.SIGKILL)  # the rank dies: its HBM state is gone
        origin.wait()
        t0 = time.monotonic_ns()             # failure notice
        if warm:
            standby.stdin.write("FAIL %d\n" % t0)
            standby.stdin.flush()
        else:
            standby = spawn(sb + ["--t0", str(t0)])
        out, err = standby.communicate(timeout=600)
        assert standby.returncode == 0, err
        rep = json.loads(out.strip().splitlines()[-1])
        with open(samples, "rb") as f:
            blob = f.read()
        return rep, blob
    finally:
        for p in procs:
            if p.poll() is None:
                try:
                    p.stdin.close()
                except Exception:
                    pass
        for p in procs:
            try:
                p.wait(timeout=60)
            except subprocess.TimeoutExpired:
                p.kill()
                p.wait()


def check_samples(regs, blob):
    off = 0
    for r in regs:
        if r.nbytes < 8192:
            want = r.literal if r.literal is not None else orc.materialize(r.digest, r.nbytes)
            got = blob[off:off + r.nbytes]
            off += r.nbytes
            assert got == want, r.kind
            continue
        head = orc.materialize_range(r.digest, r.nbytes, 0, 4096)
        tail = orc.materialize_range(r.digest, r.nbytes, r.nbytes - 4096, 4096)
        assert blob[off:off + 4096] == head, r.kind
        assert blob[off + 4096:off + 8192] == tail, r.kind
        off += 8192
    assert off == len(blob)


@pytest.mark.parametrize("warm", [True, False])
def test_replacement_process_restores_killed_rank(tmp_path, warm):
    from paper_2512_03644_b200 import state
    phi, d = 1 << 26, 8
    regs1 = state.zero3_shard(phi, d, 1, iteration=1)
    regs2 = state.zero3_shard(phi, d, 1, iteration=2)
    rep, blob = failover(tmp_path, regs1, regs2, d, phi, warm=warm)
    assert rep["verified"] and rep["bad_slices"] == 0 and rep["blob_is_sound"] == 1
    assert rep["target_iteration"] == 2 and rep["bytes"] == state.shard_bytes(regs2)
    assert rep["regions"] == 6 and rep["holder_dp"] == 2
    check_samples(regs2, blob)


@pytest.mark.skipif(os.environ.get("FFX_FULL_SIZE", "1") == "0", reason="full-size disabled")
def test_llama3_8b_shard_time_to_restore_under_1s(tmp_path):
    """configs[3]: the 14.05 GB Llama-3 8B ZeRO-3 d=8 shard; a warm spare
    must restore and verify it in under a second from the failure notice."""
    from paper_2512_03644_b200 import state
    free, _ = torch.cuda.mem_get_info()
    regs1 = state.zero3_shard(state.PHI_LLAMA3_8B, 8, 1, iteration=1)
    regs2 = state.zero3_shard(state.PHI_LLAMA3_8B, 8, 1, iteration=2)
    if free < 4.2 * state.shard_bytes(regs1):
        pytest.skip("needs ~60 GB of free HBM")
    rep, blob = failover(tmp_path, regs1, regs2, 8, state.PHI_LLAMA3_8B, warm=True)
    print(json.dumps(rep))
    assert rep["verified"] and rep["blob_is_sound"] == 1
    check_samples(regs2, blob)
    assert rep["time_to_restore_s"] < 1.0, rep
