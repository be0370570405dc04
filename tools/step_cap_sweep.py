#!/usr/bin/env python3
"""Step-time overhead of the fused snapshot policy inside the synthetic
ZeRO-3 step, per kernel configuration (FFX_SLICE_VARIANT, DEV build) and CTA
cap.  One-rank NCCL group at N=1, torchrun for N>1.  JSON lines on rank 0.

  FFX_SLICE_VARIANT=13 python tools/step_cap_sweep.py
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
from paper_2512_03644_b200.step import SliceScheduler, SyntheticStep, measure_overhead  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world == 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(bench.free_port()))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    regions, nbytes = bench.llama_regions(8)
    spec = ffx.make_spec(d=max(world, 2), phi=bench.PHI_LLAMA3_8B, distributed=True)
    R = bench.Ring(ffx, torch, dist, world, rank, local, nbytes, spec, 4096, regions)
    step = SyntheticStep(world)
    steps = int(os.environ.get("STEPS", "20"))
    policy = os.environ.get("POLICY", "fused")
    for cap in [int(x) for x in os.environ.get("CAPS", "16,32,64").split(",")]:
        kw = {"copy_ctas": cap} if policy == "fused" else {"copy_ctas": 8, "hash_ctas": cap, "copy_engine": True}
        if policy == "fused" and cap == 0:
            kw = {"copy_ctas": 32, "task_ctas": True}  # cap 0: task-granular batches
        sched = SliceScheduler(R.ctx, step, policy=policy, **kw)
        r = measure_overhead(step, sched, steps=steps, warmup=2, it0=10 + 1000 * cap)
        sched.close()
        if rank == 0:
            print(json.dumps({"variant": int(os.environ.get("FFX_SLICE_VARIANT", "-1")), "world": world,
                              "policy": policy, "cap": cap, "overhead_pct": r["overhead_pct"],
                              "step_ms_without": r["step_ms_without"], "step_ms_with": r["step_ms_with"]}),
                  flush=True)
    R.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
