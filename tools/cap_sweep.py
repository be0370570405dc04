#!/usr/bin/env python3
"""SM cost of the snapshot kernel when it is CTA-capped (the slice
scheduler's regime inside a training step): GB/s of a local-replica
snapshot at several CTA caps, for the kernel configuration selected by
FFX_SLICE_VARIANT (needs the development build: make -C
paper_2512_03644_b200/csrc DEV=1).  One JSON line per cap.

  FFX_SLICE_VARIANT=2 python tools/cap_sweep.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_03644_b200 import ffx, state  # noqa: E402


def main():
    n = int(os.environ.get("CAP_BYTES", str(2_336_416_800)))
    slice_bytes = int(os.environ.get("CAP_SLICE", "4096"))
    spec = ffx.make_spec(d=8, phi=1_557_611_200, distributed=True)
    holder = ffx.Context(0, spec, (0, 0, 0), slice_bytes)
    origin = ffx.Context(0, spec, (1, 0, 0), slice_bytes)
    rep = holder.create_replica((1, 0, 0), n, 2)
    view = origin.open_replica(rep.export())
    origin.set_target(view)
    t = torch.empty(n, dtype=torch.uint8, device="cuda")
    ffx.materialize(t, state.optimizer_init(42, 1, 0, 0))
    origin.register(ffx.REGION_BLOB, t)
    s = torch.cuda.Stream()
    it = 0
    for cap in [int(x) for x in os.environ.get("CAP_CTAS", "8,16,32,48,64,0").split(",")]:
        for _ in range(2):
            it += 1
            origin.snapshot(it, stream=s, max_ctas=cap)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k = 5
        e0.record(s)
        for _ in range(k):
            it += 1
            origin.snapshot(it, stream=s, max_ctas=cap)
        e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1) / k
        print(json.dumps({"variant": int(os.environ.get("FFX_SLICE_VARIANT", "0")), "slice": slice_bytes,
                          "max_ctas": cap, "ms": round(ms, 4), "gbs": round(n / ms / 1e6, 1)}), flush=True)
    torch.cuda.synchronize()
    origin.inject(ffx.FAULT_POISON_STATE)
    assert origin.recover(view, it).bad_slices == 0 and ffx.blob_is_sound(t)


if __name__ == "__main__":
    main()
