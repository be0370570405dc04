"""Ring-shift mechanism probe (measurement tooling, not product code).

    python tools/probe_mix.py [--bytes N]

Two GPUs driven from one process, both directions at once (the ring shift
of a 2-rank ring).  Times moving N bytes per GPU to the other GPU (with the
per-slice checksum) when the bytes are split between mechanisms:
  fused         the snapshot kernel pushes everything (TMA stores to the peer)
  fused+ce f    the kernel pushes a fraction f, the copy engines move the
                rest while a hash kernel checksums it locally
  push+pull f   the kernel pushes a fraction f; the peer's kernel pulls the
                rest (TMA loads from the peer)
Prints one JSON line of per-GPU GB/s per variant.
"""
import argparse
import json

import torch

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_03644_b200 import ffx  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=2_336_416_800)
    ap.add_argument("--slice", type=int, default=4096)
    args = ap.parse_args()
    if torch.cuda.device_count() < 2:
        print(json.dumps({"skipped": "needs 2 GPUs"}))
        return
    n = args.bytes // args.slice * args.slice
    S = args.slice
    src, land, sums, streams = [], [], [], []
    for d in (0, 1):
        with torch.cuda.device(d):
            src.append(torch.empty(n, dtype=torch.uint8, device=d))
            ffx.materialize(src[d], bytes([d]) * 32)
            land.append(torch.empty(n, dtype=torch.uint8, device=d))  # what the OTHER gpu sends here
            sums.append(torch.empty(n // S, dtype=torch.int64, device=d))
            streams.append([torch.cuda.Stream(device=d) for _ in range(3)])
    for d in (0, 1):  # enable peer access both ways (torch does on the first cross-device copy)
        land[1 - d][:1 << 20].copy_(src[d][:1 << 20])
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)

    def run(variant, f):
        k = int(n * f) // S * S
        for d in (0, 1):
            p = 1 - d
            with torch.cuda.device(d):
                s0, s1, s2 = streams[d]
                if variant == "fused":
                    ffx.copy_checksums(land[p], src[d], S, sums[d], stream=s0)
                elif variant == "fused+ce":
                    if k:
                        ffx.copy_checksums(land[p][:k], src[d][:k], S, sums[d][:k // S], stream=s0)
                    with torch.cuda.stream(s1):
                        land[p][k:].copy_(src[d][k:], non_blocking=True)
                    ffx.slice_checksums(src[d][k:], S, sums[d][k // S:], stream=s2)
                elif variant == "push+pull":
                    if k:
                        ffx.copy_checksums(land[p][:k], src[d][:k], S, sums[d][:k // S], stream=s0)
                    # pull the peer's remaining bytes into this GPU (loads over NVLink)
                    ffx.copy_checksums(land[d][k:], src[p][k:], S, sums[d][k // S:], stream=s1)

    def timed(variant, f, reps=5):
        for _ in range(2):
            run(variant, f)
        for d in (0, 1):
            torch.cuda.synchronize(d)
        ev = []
        for d in (0, 1):
            with torch.cuda.device(d):
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(streams[d][0])
                for s in streams[d][1:]:
                    s.wait_event(e0)
                ev.append([e0])
        for _ in range(reps):
            run(variant, f)
        for d in (0, 1):
            with torch.cuda.device(d):
                e1 = torch.cuda.Event(enable_timing=True)
                for s in streams[d][1:]:
                    streams[d][0].wait_stream(s)
                e1.record(streams[d][0])
                ev[d].append(e1)
        for d in (0, 1):
            torch.cuda.synchronize(d)
        ms = max(ev[d][0].elapsed_time(ev[d][1]) for d in (0, 1))
        return round(n * reps / (ms * 1e-3) / 1e9, 1)

    out = {"bytes": n, "fused": timed("fused", 1.0)}
    for f in (0.9, 0.8, 0.7, 0.5):
        out["fused+ce_%.1f" % f] = timed("fused+ce", f)
    for f in (0.8, 0.6, 0.5, 0.3):
        out["push+pull_%.1f" % f] = timed("push+pull", f)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
