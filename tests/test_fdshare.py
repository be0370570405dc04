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


def test_fd_server_under_sanitizers(tmp_path):
    """The same two-process exchange with the fd server built under
    AddressSanitizer + UBSan, then ThreadSanitizer (its accept thread runs
    beside the caller's)."""
    src = [os.path.join(ROOT, "tests", "cpp", "test_fdshare.cpp"),
           os.path.join(ROOT, "paper_2512_03644_b200", "csrc", "ffx_share.cpp")]
    inc = "-I" + os.path.join(ROOT, "paper_2512_03644_b200", "csrc")
    for name, flags, env in (("asan", ["-fsanitize=address,undefined", "-fno-sanitize-recover=all"],
                              {"ASAN_OPTIONS": "detect_leaks=1"}),
                             ("tsan", ["-fsanitize=thread"], {"TSAN_OPTIONS": "halt_on_error=1"})):
        exe = str(tmp_path / ("fdshare_" + name))
        subprocess.run(["g++", "-std=c++17", "-O1", "-g", inc, *flags, "-o", exe, *src, "-lpthread"], check=True)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=120, env=dict(os.environ, **env))
        assert r.returncode == 0, name + ": " + r.stderr[-2000:]
        assert "fdshare ok" in r.stdout
