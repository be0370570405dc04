#!/usr/bin/env python3
"""Ring-stream sweep at N GPUs (torchrun): per-GPU GB/s of the snapshot ring
for push (origin's fused kernel stores into the successor's replica) and pull
(the holder's fused kernel loads its predecessor's regions) over a range of
CTA caps, plus a single-puller control.  One JSON line per point on rank 0.

  torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/ring_sweep.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2512_03644_b200 import ffx  # noqa: E402


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = int(os.environ.get("SWEEP_BYTES", str((12 * bench.PHI_GPT2_XL + 7) // 8)))
    spec = ffx.make_spec(d=max(world, 2), phi=bench.PHI_GPT2_XL, distributed=True)
    R = bench.Ring(ffx, torch, dist, world, rank, local, n, spec, 4096, bench.gpt2xl_regions(n))
    s = torch.cuda.Stream()
    it = [0]
    modes = os.environ.get("SWEEP_MODES", "push,pull").split(",")
    ctas = [int(x) for x in os.environ.get("SWEEP_CTAS", "0,16,24,32,48,64,96,128,160,200").split(",")]
    k = int(os.environ.get("SWEEP_STEPS", "8"))

    def timed(fn, reps):
        for _ in range(2):
            fn()
        s.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            fn()
        e1.record(s)
        s.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) / reps

    for mode in modes:
        for c in ctas:
            def fn():
                it[0] += 1
                R.snapshot(it[0], s, mode, c)
            ms = timed(fn, k)
            if rank == 0:
                print(json.dumps({"mode": mode, "max_ctas": c, "world": world, "ms": round(ms, 4),
                                  "gbs_per_gpu": round(n / ms / 1e6, 1)}), flush=True)
    # control: a single puller (rank 1 pulls from rank 0, nobody else moves)
    if world > 1 and R.remote is not None:
        for c in [0, 32, 64, 148]:
            def fn1():
                it[0] += 1
                if rank == 1:
                    R.ctx.snapshot_pull(R.remote, R.held, it[0], stream=s, max_ctas=c)
            ms = timed(fn1, k)
            if rank == 0:
                print(json.dumps({"mode": "single-puller", "max_ctas": c, "ms": round(ms, 4),
                                  "gbs": round(n / ms / 1e6, 1)}), flush=True)
        for c in [0, 32, 64]:
            def fn2():
                it[0] += 1
                if rank == 0:
                    R.ctx.snapshot(it[0], stream=s, max_ctas=c)
            ms = timed(fn2, k)
            if rank == 0:
                print(json.dumps({"mode": "single-pusher", "max_ctas": c, "ms": round(ms, 4),
                                  "gbs": round(n / ms / 1e6, 1)}), flush=True)
    R.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
