"""Host-side timing of the synchronous ABI calls (measurement tooling, not
product code): wall time per call next to the device time of the same call,
to separate kernel time from host/allocator overhead."""
import json
import time

import torch

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_03644_b200 import ffx  # noqa: E402


def main(n=2_336_416_800):
    torch.cuda.set_device(0)
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    ffx.materialize(src, bytes(range(32)))
    torch.cuda.synchronize()
    out = {"bytes": n}
    for name, fn in (("checksum64", lambda: ffx.checksum64(src)),
                     ("blob_first_bad", lambda: ffx.blob_first_bad(src))):
        walls = []
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            walls.append(time.perf_counter() - t0)
        out[name + "_wall_ms"] = [round(w * 1e3, 3) for w in walls]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
