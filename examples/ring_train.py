"""ZeRO-1 data-parallel training with per-iteration neighbour backup and a
rank failure in the middle -- the FFTrainer path end to end on real state.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        examples/ring_train.py [--iters 12] [--fail-at 6] [--fail-rank 1] [--overlap]

Every rank holds the full (bf16-free, fp32) MLP parameters, computes
gradients on its own data -- windows of the synthetic data server
(DataServerStub, one IN-byte sample per row) preloaded into an HBM
PreloadBuffer a few iterations ahead, the fetches issued in the step's
link-idle gap through the slice scheduler -- and owns one shard of the optimizer state
(ZeRO-1): the fp32 master shard, Adam m / v for that shard, and the data
cursor.  Those four regions are registered with ffx and snapshotted into the
ring successor's replica after every optimizer update (NVLink, one kernel).
At --fail-at the failing rank loses all four regions (poisoned), the plan
names its holder, it pulls and verifies the replica, the ring re-gathers
the parameters from the shards, and training continues.  The script then
replays the run without the failure and prints one JSON line comparing the
two: losses and final parameters must be bit-identical.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_03644_b200 import ffx, ring  # noqa: E402

IN, HID, OUT, BATCH = 512, 1024, 16, 256
DATA_SEED = 11
SHAPES = [(IN, HID), (HID,), (HID, OUT), (OUT,)]
NPARAM = sum(torch.Size(s).numel() for s in SHAPES)


class Rank:
    def __init__(self, rank, world, seed=3):
        self.rank, self.world = rank, world
        self.shard = (NPARAM + world - 1) // world
        total = self.shard * world
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.params = torch.zeros(total, device="cuda")
        self.params[:NPARAM] = torch.randn(NPARAM, device="cuda", generator=g) * 0.05
        lo = rank * self.shard
        self.master = self.params[lo:lo + self.shard].clone()  # this rank's fp32 master shard
        self.m = torch.zeros(self.shard, device="cuda")
        self.v = torch.zeros(self.shard, device="cuda")
        self.cursor = torch.zeros(2, dtype=torch.int64, device="cuda")  # [step, data position]

    def regions(self):
        return [(ffx.REGION_MASTER, self.master), (ffx.REGION_ADAM_M, self.m), (ffx.REGION_ADAM_V, self.v),
                (ffx.REGION_CURSOR, self.cursor)]

    def views(self):
        out, o = [], 0
        for s in SHAPES:
            n = torch.Size(s).numel()
            out.append(self.params[o:o + n].view(s))
            o += n
        return out

    # ---- the data loader: an HBM PreloadBuffer fed through the scheduler ----
    DEPTH = 3  # iterations of data kept ahead (ClusterSpec.preload_depth)

    def attach_loader(self, ctx):
        self.preload = ffx.Preload(ctx, self.DEPTH * BATCH * IN)
        self.loader_sched = ffx.Sched(ctx, ffx.SCHED_FUSED, link_gaps=1)
        self.queued = set()

    def lose_loader(self, ctx):
        """The failed rank's buffered windows are gone with it; the
        replacement refetches from its restored cursor."""
        self.close_loader()
        self.attach_loader(ctx)

    def close_loader(self):
        torch.cuda.synchronize()
        self.loader_sched.destroy()
        self.preload.destroy()

    def window(self, pos):
        # disjoint per (position, rank): the data_assignment geometry
        first = (pos * self.world + self.rank) * BATCH
        return ffx.data_item_digests(DATA_SEED, first, BATCH)

    def batch(self, pos):
        cur = torch.cuda.current_stream()
        if pos not in self.queued:  # first step, or after a failure: fetch now
            self.preload.fetch_synthetic(pos, self.window(pos), IN, stream=cur)
            self.queued.add(pos)
        for ahead in range(pos + 1, pos + self.DEPTH):
            if ahead not in self.queued:
                self.loader_sched.preload_synthetic(self.preload, ahead, self.window(ahead), IN)
                self.queued.add(ahead)
        dev, n = self.preload.take(pos, cur)  # the step's stream waits for the fetch
        self.queued.discard(pos)
        raw = torch.empty(BATCH, IN, dtype=torch.uint8, device="cuda")
        ffx.check(ffx.lib.ffx_memcpy(raw.data_ptr(), dev, n, cur.cuda_stream, 0), "memcpy")
        self.preload.free(dev, cur)
        x = (raw.float() - 127.5) / 64.0
        y = raw[:, 0].long() % OUT
        return x, y

    def step(self, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, before_update=None):
        pos = int(self.cursor[1].item())
        x, y = self.batch(pos)
        p = self.params.detach().requires_grad_(True)
        self.params = p
        w1, c1, w2, c2 = self.views()
        loss = torch.nn.functional.cross_entropy(torch.relu(x @ w1 + c1) @ w2 + c2, y)
        # the link is idle while forward / backward compute: the preloads go now
        self.loader_sched.gap(ffx.GAP_LINK_IDLE, torch.cuda.current_stream())
        loss.backward()
        with torch.no_grad():
            grad = p.grad
            gshard = torch.empty(self.shard, device="cuda")
            dist.reduce_scatter_tensor(gshard, grad, op=dist.ReduceOp.SUM)  # ZeRO-1: my shard's grads
            gshard /= self.world
            if before_update is not None:
                before_update()  # overlap: the previous snapshot must have read master / m / v
            t = int(self.cursor[0].item()) + 1
            self.m.mul_(b1).add_(gshard, alpha=1 - b1)
            self.v.mul_(b2).addcmul_(gshard, gshard, value=1 - b2)
            self.master.sub_(lr * (self.m / (1 - b1 ** t)) / ((self.v / (1 - b2 ** t)).sqrt() + eps))
            self.cursor += 1
            self.regather()
        lsum = loss.detach().clone()
        dist.all_reduce(lsum)
        return float(lsum.item()) / self.world

    def regather(self):
        params = torch.empty(self.shard * self.world, device="cuda")
        dist.all_gather_into_tensor(params, self.master)
        self.params = params


def run(args, rank, world, local, fail):
    me = Rank(rank, world)
    spec = ffx.make_spec(d=world, phi=NPARAM, distributed=True)
    ctx = ffx.Context(local, spec, ffx.Role(rank, 0, 0))
    for kind, t in me.regions():
        ctx.register(kind, t)
    me.attach_loader(ctx)
    nbytes = sum(t.numel() * t.element_size() for _, t in me.regions())

    def all_gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    held, targets, handles = ring.wire_ring(rank, world,
                                            lambda origin: ctx.create_replica(ffx.Role(origin, 0, 0),
                                                                              nbytes + 4096, 2),
                                            lambda r: r.export(), ctx.open_replica, all_gather)
    ctx.set_target(targets[0])
    losses, recovered = [], None
    snap_stream = torch.cuda.Stream()
    snap_done = None
    try:
        for it in range(1, args.iters + 1):
            if args.overlap:
                # the snapshot of iteration it-1 streams from the live buffers while
                # this iteration's forward / backward runs; only the optimizer
                # update waits for it (no staging copy)
                wait = (lambda ev=snap_done: torch.cuda.current_stream().wait_event(ev)) if snap_done else None
                losses.append(me.step(before_update=wait))
                ready = torch.cuda.Event()
                ready.record()  # the update of iteration `it` is done
                snap_stream.wait_event(ready)
                ctx.snapshot(it, stream=snap_stream)
                snap_done = torch.cuda.Event()
                snap_done.record(snap_stream)
            else:
                losses.append(me.step())
                ctx.snapshot(it)  # after the optimizer update: master / m / v / cursor of iteration `it`
            if fail and it == args.fail_at:
                torch.cuda.synchronize()  # the snapshot of `it` has committed everywhere
                dist.barrier()
                # the controller state (controller.cpp:81-121): every holder reports
                # the newest COMMITTED iteration of the replica it holds (the
                # CkptRecord, wire.hpp:85-90); the restore target is the ledger's
                # global consistent iteration
                probe = ffx.Ledger(spec)
                mine = (held[0].slot_info(held[0].held()[held[0].newest()]).role.tuple(),
                        probe.record_replica(held[0]))
                ledger = ffx.Ledger(spec)
                for role, rec_it in all_gather(mine):
                    ledger.record(role, rec_it)
                target = ledger.global_consistent()
                assert target == it, (target, it)
                plan = ffx.plan_recovery(spec, [], [ffx.Role(args.fail_rank, 0, 0)], target, 0)
                if rank == args.fail_rank:
                    _, holder, k = ring.recovery_sources(plan.forwards, world)[0]
                    ctx.inject(ffx.FAULT_POISON_STATE)  # the rank's optimizer shard is gone
                    me.lose_loader(ctx)                    # and its preloaded data
                    src = ctx.open_replica(handles[holder][k])
                    rpt = ctx.recover(src, target)
                    recovered = {"iteration": it, "holder": holder, "bytes": rpt.bytes,
                                 "seconds": rpt.seconds, "bad_slices": rpt.bad_slices}
                    src.destroy()
                dist.barrier()
                with torch.no_grad():
                    me.regather()  # the replacement's parameters come back from the shards
        final = me.params.detach().clone()
    finally:
        torch.cuda.synchronize()
        me.close_loader()
        for r in targets + held:
            r.destroy()
        ctx.close()
    return losses, final, recovered


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=12)
    ap.add_argument("--fail-at", type=int, default=6)
    ap.add_argument("--fail-rank", type=int, default=1)
    ap.add_argument("--overlap", action="store_true",
                    help="snapshot iteration n while iteration n+1 computes; the optimizer update waits")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    torch.backends.cuda.matmul.allow_tf32 = False
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    args.fail_rank %= world
    l_fail, p_fail, rec = run(args, rank, world, local, fail=True)
    l_ref, p_ref, _ = run(args, rank, world, local, fail=False)
    same = torch.tensor([int(torch.equal(p_fail, p_ref) and l_fail == l_ref)], device="cuda")
    dist.all_reduce(same, op=dist.ReduceOp.MIN)
    recs = [None] * world
    dist.all_gather_object(recs, rec)
    if rank == 0:
        print(json.dumps({"world": world, "iters": args.iters, "fail_at": args.fail_at, "overlap": args.overlap,
                          "fail_rank": args.fail_rank, "recovery": recs[args.fail_rank],
                          "losses": [round(x, 6) for x in l_fail],
                          "bit_identical_to_uninterrupted_run": bool(same.item())}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
