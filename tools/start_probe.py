"""Start-of-launch behaviour of the three TMA kernels on one 2.34 GB buffer
(run under ncu --set full; read with tools/pm_timeline.py):
  copy_kernel (TMA copy only, split policy), slice_kernel<Hash> (checksum
  only), slice_kernel<Copy> (fused copy + checksum, uniform 4 KiB slices).
Each runs 3x untimed, then once more; capture the last three launches."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2512_03644_b200 import ffx  # noqa: E402

n = 2_336_416_800
src = torch.empty(n, dtype=torch.uint8, device="cuda")
src.random_(0, 256)
dst = torch.empty_like(src)
sums = torch.empty((n + 4095) // 4096, dtype=torch.int64, device="cuda")


def run_copy():
    ffx.check(ffx.lib.ffx_copy(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()), n, 0, None), "copy")


def run_hash():
    ffx.slice_checksums(src, 4096, sums)


def run_fused():
    ffx.copy_checksums(dst, src, 4096, sums)


for f in (run_copy, run_hash, run_fused):
    for _ in range(3):
        f()
torch.cuda.synchronize()
for f in (run_copy, run_hash, run_fused):
    f()
torch.cuda.synchronize()
print("ok")
