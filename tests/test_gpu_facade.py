"""The C++ facade driven with device state (tests/cpp/test_facade_device.cpp):
HostSnapshots::take on a device pointer, NeighborBuffer::store, and
assemble_restore through the reference's own API, on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2512_03644_b200", "facade", "build", "test_facade_device")


@pytest.mark.gpu
def test_facade_device_path():
    if not os.path.exists(BIN):
        pytest.fail("facade test program not built (run __graft_entry__.build())")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "[facade-device] ok" in p.stdout
