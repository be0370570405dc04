"""Kernel decomposition probe (measurement tooling, not product code).

    python tools/probe.py [--bytes N] [--peer]

Times, on the same buffers and with CUDA events, the pieces the snapshot
kernel fuses so its roofline fraction can be explained:
  copy_ce      torch copy_ (copy engines / cudaMemcpy D2D)       2N HBM bytes
  copy_tma     ffx_copy (TMA copy-only kernel)                     2N
  hash         ffx_slice_checksums (read + per-slice FNV)           N
  fused        ffx_copy_checksums (copy + per-slice FNV)           2N
With --peer (>= 2 visible GPUs) the same copies target a buffer on GPU 1
through peer access: the NVLink per-direction figures.
"""
import argparse
import json

import torch

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_03644_b200 import ffx  # noqa: E402


def timed(fn, reps=10, warm=3, stream=None):
    s = stream or torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=2_336_416_800)
    ap.add_argument("--slice", type=int, default=4096)
    ap.add_argument("--peer", action="store_true")
    args = ap.parse_args()
    n = args.bytes
    torch.cuda.set_device(0)
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    ffx.materialize(src, bytes(range(32)))
    out = {"bytes": n, "slice": args.slice}
    sums = torch.empty((n + args.slice - 1) // args.slice, dtype=torch.int64, device="cuda:0")
    targets = [("local", torch.empty(n, dtype=torch.uint8, device="cuda:0"))]
    if args.peer and torch.cuda.device_count() > 1:
        try:
            torch.cuda.set_device(1)
            peer = torch.empty(n, dtype=torch.uint8, device="cuda:1")
            torch.cuda.set_device(0)
            targets.append(("peer", peer))
        except Exception as ex:
            out["peer_error"] = repr(ex)
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    for name, dst in targets:
        scale = 2 if name == "local" else 1  # HBM counts read+write; NVLink counts egress
        t = timed(lambda: dst.copy_(src))
        out["%s_copy_ce_gbs" % name] = round(scale * n / t / 1e9, 1)
        for ctas in (16, 32, 64, sm):
            t = timed(lambda: ffx.lib.ffx_copy(dst.data_ptr(), src.data_ptr(), n, ctas, None))
            out["%s_copy_tma_%dctas_gbs" % (name, ctas)] = round(scale * n / t / 1e9, 1)
        t = timed(lambda: ffx.copy_checksums(dst, src, args.slice, sums))
        out["%s_fused_gbs" % name] = round(scale * n / t / 1e9, 1)
    t = timed(lambda: ffx.slice_checksums(src, args.slice, sums))
    out["hash_read_gbs"] = round(n / t / 1e9, 1)
    # whole-payload checksum64 (SNP1 export path): speculative low byte + affine combine
    t = timed(lambda: ffx.checksum64(src), reps=3, warm=1)
    out["whole_checksum64_gbs"] = round(n / t / 1e9, 1)
    # synthetic state generation (evo::materialize) and soundness check
    t = timed(lambda: ffx.materialize(src, bytes(range(32))))
    out["materialize_gbs"] = round(n / t / 1e9, 1)
    t = timed(lambda: ffx.blob_first_bad(src), reps=3, warm=1)
    out["blob_check_gbs"] = round(n / t / 1e9, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
