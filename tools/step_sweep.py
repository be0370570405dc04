"""Step-overhead sweep of the slice scheduler's knobs (measurement tooling).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tools/step_sweep.py [--steps 30]

The Llama-3 8B ZeRO-3 d=8 shard (14.05 GB per rank, BASELINE configs[2])
snapshotted inside the synthetic ZeRO-3 step (paper_2512_03644_b200/step.py)
under each policy / CTA budget; prints one JSON line with the median
overhead of every variant (interleaved A/B steps, max over ranks).
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=30)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    opts = None
    if os.environ.get("FFX_NCCL_HIGH_PRIORITY"):
        # TRAIN > STATE for the collectives too: NCCL's kernels on a
        # high-priority stream outrank the snapshot's low-priority batches
        opts = dist.ProcessGroupNCCL.Options(is_high_priority_stream=True)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local), pg_options=opts)
    from paper_2512_03644_b200 import ffx, ring
    from paper_2512_03644_b200.step import SliceScheduler, SyntheticStep, measure_overhead
    phi, d_ref = 8_030_261_248, 8
    adam, params = (12 * phi + d_ref - 1) // d_ref, (2 * phi + d_ref - 1) // d_ref
    spec = ffx.make_spec(d=world, phi=phi, distributed=True)
    ctx = ffx.Context(local, spec, ffx.Role(rank, 0, 0))
    state = [torch.empty(adam, dtype=torch.uint8, device="cuda"), torch.empty(params, dtype=torch.uint8, device="cuda")]
    for t, k in zip(state, (ffx.REGION_BLOB, ffx.REGION_PARAMS)):
        ffx.materialize(t, bytes([rank, k]) * 16)
        ctx.register(k, t)

    def all_gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    held, targets, _ = ring.wire_ring(rank, world, lambda o: ctx.create_replica(ffx.Role(o, 0, 0), adam + params, 2),
                                      lambda r: r.export(), ctx.open_replica, all_gather)
    ctx.set_target(targets[0])
    step = SyntheticStep(world)
    variants = [("fused", dict(copy_ctas=32)),
                ("split", dict(copy_ctas=8, hash_ctas=96, copy_engine=True)),
                ("split", dict(copy_ctas=8, hash_ctas=64, copy_engine=True)),
                ("split", dict(copy_ctas=8, hash_ctas=96, copy_engine=True))]

    class GemmHash(SliceScheduler):
        """Checksum batches alongside the GEMMs (link-idle gaps) on few SMs,
        instead of in the SM-idle windows before the collectives."""

        def hook(self, kind, layer):
            if kind in ("fwd", "bwd"):
                self.native.gap(self.ffx.GAP_SM_IDLE, self.step.train)
                self.native.gap(self.ffx.GAP_LINK_IDLE, self.step.train)
            elif kind == "opt":
                self.native.finish(self.step.train)
    if os.environ.get("FFX_SWEEP_ALL"):
        variants = [("fused", dict(copy_ctas=c)) for c in (16, 32, 64)] + \
                   [("split", dict(copy_ctas=8, hash_ctas=h, copy_engine=True)) for h in (32, 48, 64, 96, 148)]
    out = []
    # component isolation: the copy alone (copy engines, gated on the same
    # idle-link gaps, sized by the measured gaps) and the checksum alone
    # (gated before each all-gather), with no slot / commit protocol
    import statistics
    from paper_2512_03644_b200.step import time_steps
    payload, _ = targets[0].slot_ptrs(0)
    cal = SliceScheduler(ctx, step, policy="split", copy_engine=True)
    time_steps(step, 2)
    gaps = cal.calibrate()
    sums = torch.empty((adam + params) // 4096 + 2, dtype=torch.int64, device="cuda")

    class Raw:
        def __init__(self, what):
            self.what = what
            self.low = torch.cuda.Stream(priority=0)
            self.done = torch.cuda.Event()

        def begin(self, it):
            self.g = 0
            self.h = 0

        def hook(self, kind, layer):
            G = len(gaps)
            if self.what == "hash" and kind == "pre_ag" and self.h < G:
                ev = torch.cuda.Event()
                ev.record(step.train)
                self.low.wait_event(ev)
                t = state[0] if self.h < G // 2 else state[1]
                n = t.numel()
                half = self.h if self.h < G // 2 else self.h - G // 2
                lo = (n * half // (G // 2)) // 4096 * 4096
                hi = (n * (half + 1) // (G // 2)) // 4096 * 4096 if half + 1 < G // 2 else n
                if hi > lo:
                    ffx.slice_checksums(t[lo:hi], 4096, sums[lo // 4096:], stream=self.low)
                self.h += 1
            elif self.what == "copy" and kind in ("fwd", "bwd") and self.g < G:
                ev = torch.cuda.Event()
                ev.record(step.train)
                self.low.wait_event(ev)
                tot = sum(gaps)
                a = int(adam * sum(gaps[:self.g]) / tot) // 16 * 16
                b = int(adam * sum(gaps[:self.g + 1]) / tot) // 16 * 16 if self.g + 1 < G else adam
                if b > a:
                    ffx.check(ffx.lib.ffx_memcpy(payload + a, state[0].data_ptr() + a, b - a,
                                                 self.low.cuda_stream, 0), "memcpy")
                self.g += 1
            elif kind == "opt":
                self.done.record(self.low)
                step.train.wait_event(self.done)

    for what in ("copy", "hash"):
        raw = Raw(what)
        time_steps(step, 2, raw, it0=0)
        base, w = [], []
        for _ in range(args.steps):
            base += time_steps(step, 1)
            w += time_steps(step, 1, raw, it0=0)
        b, m = statistics.median(base), statistics.median(w)
        out.append({"policy": what + " only (raw)", "overhead_pct": round(100 * (m - b) / b, 3),
                    "step_ms_without": round(b, 3)})
    for i, (policy, kw) in enumerate(variants):
        kw = dict(kw)
        cls = GemmHash if kw.pop("hash_in_gemm", False) else SliceScheduler
        sched = cls(ctx, step, policy=policy, **kw)
        r = measure_overhead(step, sched, steps=args.steps, warmup=2, it0=10 + 1000 * i)
        sched.close()
        out.append({"policy": r["policy"], "copy_ctas": kw.get("copy_ctas"), "hash_ctas": kw.get("hash_ctas"),
                    "front": kw.get("front", 1.0), "rs_gaps": kw.get("rs_gaps", False),
                    "hash_in_gemm": cls is GemmHash,
                    "overhead_pct": r["overhead_pct"], "step_ms_without": r["step_ms_without"]})
    if rank == 0:
        print(json.dumps({"world": world, "steps_each": args.steps, "variants": out}))
    torch.cuda.synchronize()
    for r in targets + held:
        r.destroy()
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
