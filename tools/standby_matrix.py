#!/usr/bin/env python3
"""Time-to-restore matrix of the replacement process (bin/ffx_standby) for the
Llama-3 8B ZeRO-3 d=8 shard: warm / cold x cudaMalloc+IPC / VMM (shared)
replica x preallocated arena or not.  One JSON line per run.

  python tools/standby_matrix.py [holder_device]
"""
import json
import os
import signal
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_03644_b200 import state  # noqa: E402

EXE = os.path.join(ROOT, "paper_2512_03644_b200", "bin", "ffx_standby")


def run(warm, shared, prealloc, hdev=0, phi=state.PHI_LLAMA3_8B, d=8, role=1):
    regs1 = state.zero3_shard(phi, d, role, iteration=1)
    regs2 = state.zero3_shard(phi, d, role, iteration=2)
    nbytes = state.shard_bytes(regs1)
    with tempfile.TemporaryDirectory() as store:
        common = ["--d", str(d), "--phi", str(phi), "--store", store]
        procs = []

        def spawn(a, dev, env=None):
            p = subprocess.Popen([EXE] + a + common + ["--device", str(dev)], stdin=subprocess.PIPE,
                                 stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, env=env)
            procs.append(p)
            return p

        def line(p, want):
            while True:
                ln = p.stdout.readline()
                if not ln:
                    raise RuntimeError(p.stderr.read()[-400:])
                if ln.startswith(want):
                    return ln.strip()

        try:
            h = spawn(["holder", "--origin", str(role), "--capacity", str(nbytes)] + (["--shared"] if shared else []),
                      hdev)
            hdp = int(line(h, "READY").split()[1])
            o = spawn(["origin", "--role", str(role), "--holder", str(hdp),
                       "--regions", ",".join(r.spec() for r in regs1),
                       "--regions2", ",".join(r.spec() for r in regs2)], 0)
            line(o, "SNAPSHOTTED")
            sb = ["standby", "--role", str(role), "--check", "--target", "2"]
            s = None
            senv = None
            if os.environ.get("STANDBY_VISIBLE"):  # e.g. "0": the replacement sees only its own GPU
                senv = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ["STANDBY_VISIBLE"])
            sb += ["--repeat", "2"] + (["--touch"] if os.environ.get("STANDBY_TOUCH") else [])
            if warm:
                s = spawn(sb + ["--warm"] + (["--prealloc", str(nbytes + 4096)] if prealloc else []), 0, senv)
                line(s, "ARMED")
            os.kill(o.pid, signal.SIGKILL)
            o.wait()
            t0 = time.monotonic_ns()
            if warm:
                s.stdin.write("FAIL %d\n" % t0)
                s.stdin.flush()
            else:
                s = spawn(sb + ["--t0", str(t0)], 0, senv)
            out, err = s.communicate(timeout=600)
            if s.returncode:
                return {"error": err[-400:]}
            r = json.loads(out.strip().splitlines()[-1])
            r.update(shared=shared, prealloc=prealloc, holder_device=hdev,
                     standby_visible=os.environ.get("STANDBY_VISIBLE", "all"))
            return r
        finally:
            for p in procs:
                if p.poll() is None:
                    try:
                        p.stdin.close()
                    except Exception:
                        pass
            for p in procs:
                try:
                    p.wait(timeout=120)
                except subprocess.TimeoutExpired:
                    p.kill()


if __name__ == "__main__":
    hdev = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    for warm, shared, prealloc in ((True, False, False), (True, False, True), (True, True, False),
                                   (True, True, True), (False, False, False), (False, True, False),
                                   (True, False, False)):
        print(json.dumps(run(warm, shared, prealloc, hdev)), flush=True)
