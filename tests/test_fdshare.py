"""The per-process fd server that carries shareable-replica and multicast
handles between ranks (csrc/ffx_share.cpp): two processes, no GPU."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2512_03644_b200", "csrc", "build", "test_fdshare")


def test_fd_server_across_processes():
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.dirname(os.path.dirname(BIN)), "build/test_fdshare"], check=True)
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    assert "fdshare ok" in r.stdout
