"""Copy-engine ring-shift probe (measurement tooling, not product code).

    python tools/probe_ce.py

Two GPUs, both directions at once (a 2-rank ring shift by the DMA engines
alone): GB/s per GPU of a peer cudaMemcpyAsync of ~2.3 GB as a function of
the source / destination offsets inside their allocations, and of whether a
kernel runs on the SMs at the same time.  Explains the copy-engine legs of
the hybrid snapshot.
"""
import json

import torch

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_03644_b200 import ffx  # noqa: E402


def main(n=2_336_416_800 // 4096 * 4096):
    if torch.cuda.device_count() < 2:
        print(json.dumps({"skipped": "needs 2 GPUs"}))
        return
    pad = 16 << 20
    src, dst, st = [], [], []
    for d in (0, 1):
        with torch.cuda.device(d):
            src.append(torch.empty(n + pad, dtype=torch.uint8, device=d))
            dst.append(torch.empty(n + pad, dtype=torch.uint8, device=d))
            st.append(torch.cuda.Stream(device=d))
    for d in (0, 1):
        dst[1 - d][:1 << 20].copy_(src[d][:1 << 20])
    sums = [torch.empty(n // 4096 + 1, dtype=torch.int64, device=d) for d in (0, 1)]

    def timed(so, do, hash_too=False, reps=4):
        def once():
            for d in (0, 1):
                with torch.cuda.device(d), torch.cuda.stream(st[d]):
                    dst[1 - d][do:do + n].copy_(src[d][so:so + n], non_blocking=True)
                if hash_too:
                    with torch.cuda.device(d):
                        ffx.slice_checksums(src[d][:n], 4096, sums[d], stream=torch.cuda.current_stream(d))
        once()
        for d in (0, 1):
            torch.cuda.synchronize(d)
        ev = []
        for d in (0, 1):
            with torch.cuda.device(d):
                e = torch.cuda.Event(enable_timing=True)
                e.record(st[d])
                ev.append([e])
        for _ in range(reps):
            once()
        for d in (0, 1):
            with torch.cuda.device(d):
                e = torch.cuda.Event(enable_timing=True)
                e.record(st[d])
                ev[d].append(e)
        for d in (0, 1):
            torch.cuda.synchronize(d)
        ms = max(ev[d][0].elapsed_time(ev[d][1]) for d in (0, 1))
        return round(n * reps / (ms * 1e-3) / 1e9, 1)

    out = {"bytes": n}
    for so, do in [(0, 0), (4096, 4096), (0, 4096), (65536, 65536), (2 << 20, 2 << 20),
                   (2228224, 2228224), (0, 2228224), (2228224, 0)]:
        out["src%d_dst%d" % (so, do)] = timed(so, do)
    # the snapshot's layout: source = a region at its allocation start, destination
    # = a replica slot payload (P = 4,567,040 for the GPT-2 XL shard), both moved
    # by the same shift (the hybrid mode's fused share)
    P = 4_567_040
    for k in (0, 1, 16, 17, 32, 256, 512, 544, 1024):
        out["slot_shift%d" % (k * 4096)] = timed(k * 4096, P + k * 4096)
    out["src0_dst0_with_hash_kernel"] = timed(0, 0, hash_too=True)
    out["src2228224_dst2228224_with_hash_kernel"] = timed(2228224, 2228224, hash_too=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
