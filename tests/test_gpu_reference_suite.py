"""The reference's own unit tests, compiled unmodified, as parity checks.

oracle/Makefile compiles proj/tests/test_{ckpt,evolution,domain}.cpp twice
with a doctest-compatible shim (the reference vendors doctest under a
gitignored directory that is absent from the checkout):
  *_ref  against the reference library itself  -> pins the shim;
  *_ffx  against the B200 facade (ftsim API over libffx.so) -> the parity run.
The binaries live in oracle/_ref (built by __graft_entry__.build() where the
reference checkout exists, shipped to the GPU box with the snapshot).
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref")


def _run(name):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip("%s not built (needs the reference checkout at build time)" % name)
    p = subprocess.run([path], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("suite", ["ckpt", "evolution", "domain"])
def test_reference_suite_pins_shim(suite):
    rc, out = _run("test_%s_ref" % suite)
    assert rc == 0, out
    assert "0 failed" in out


def test_reference_domain_suite_on_facade_host_only():
    # domain is pure host arithmetic (ffx_role_of / ffx_index_of ...): no GPU.
    rc, out = _run("test_domain_ffx")
    assert rc == 0, out


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["ckpt", "evolution"])
def test_reference_suite_on_b200_facade(suite):
    rc, out = _run("test_%s_ffx" % suite)
    assert rc == 0, out
    assert "| 0 failed" in out
