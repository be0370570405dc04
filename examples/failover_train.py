"""A real process failure in a ZeRO-1 training job, and a warm spare taking
over from the ring replica -- FFTrainer's failover end to end on two GPUs.

    python examples/failover_train.py [--iters 10] [--fail-at 5]

Three processes (no torchrun; a launcher starts them):
  worker 0 (GPU 0) and worker 1 (GPU 1) train a small MLP with ZeRO-1 data
    parallelism: every rank owns one shard of the optimizer state (fp32
    master, Adam m / v) and the data cursor, registered with ffx and
    snapshotted after every optimizer update into its ring successor's HBM
    replica over NVLink (CUDA IPC handles exchanged through a store
    directory);
  the spare (GPU 1) is up before anything fails: CUDA context, ffx context,
    NVLink peer access.
After worker 1 commits iteration --fail-at, the launcher SIGKILLs it.  Worker
0's next collective fails (the peer's sockets closed); the launcher's notice
reaches the spare, which plans the recovery (plan_recovery, controller.cpp:
144-209), maps worker 0's replica of rank 1, allocates the four regions the
committed slot records, pulls + verifies them (assemble_restore, ckpt.cpp:
140-167), creates the replica it will hold for worker 0, and joins a new
process-group generation as rank 1.  Worker 0 re-targets its snapshots and
both continue.  The launcher then runs the same job without the failure and
prints one JSON line: losses and final parameters must be bit-identical.
Collectives are gloo on host copies (small model); gloo notices a dead peer
only at its 10 s collective timeout -- failure detection is the controller's
job (heartbeats, controller.cpp:46-58) and is not what this times: the spare's
clock starts at the launcher's notice.  The state path is ffx on the GPUs.
"""
import argparse
import datetime
import json
import os
import signal
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

IN, HID, OUT, BATCH = 256, 512, 16, 128
SHAPES = [(IN, HID), (HID,), (HID, OUT), (OUT,)]


def nparams():
    n = 0
    for s in SHAPES:
        k = 1
        for d in s:
            k *= d
        n += k
    return n


# ---------------------------------------------------------------------------
# store directory: handles, progress and notices as small files (write + rename)

def put(store, name, data):
    tmp = os.path.join(store, name + ".tmp")
    with open(tmp, "wb") as f:
        f.write(data)
        f.flush()
        os.fsync(f.fileno())
    os.rename(tmp, os.path.join(store, name))


def get(store, name, timeout=120.0):
    p = os.path.join(store, name)
    t_end = time.time() + timeout
    while not os.path.exists(p):
        if time.time() > t_end:
            raise TimeoutError(name)
        time.sleep(0.002)
    with open(p, "rb") as f:
        return f.read()


# ---------------------------------------------------------------------------
# the training rank (worker, or the spare once it has taken over)

class Trainer:
    def __init__(self, torch, ffx, rank, world, device):
        self.torch, self.ffx, self.rank, self.world = torch, ffx, rank, world
        n = nparams()
        self.shard = (n + world - 1) // world
        g = torch.Generator(device="cpu").manual_seed(3)
        init = torch.zeros(self.shard * world)
        init[:n] = torch.randn(n, generator=g) * 0.05
        self.params = init.to(device)
        lo = rank * self.shard
        self.master = self.params[lo:lo + self.shard].clone()
        self.m = torch.zeros(self.shard, device=device)
        self.v = torch.zeros(self.shard, device=device)
        self.cursor = torch.zeros(2, dtype=torch.int64, device=device)  # [step, data position]
        self.device = device

    def regions(self):
        f = self.ffx
        return [(f.REGION_MASTER, self.master), (f.REGION_ADAM_M, self.m), (f.REGION_ADAM_V, self.v),
                (f.REGION_CURSOR, self.cursor)]

    def views(self, p):
        out, o = [], 0
        for s in SHAPES:
            k = 1
            for d in s:
                k *= d
            out.append(p[o:o + k].view(s))
            o += k
        return out

    def batch(self, pos):
        torch = self.torch
        g = torch.Generator(device="cpu").manual_seed(1000 * pos + self.rank)
        x = torch.randn(BATCH, IN, generator=g)
        y = torch.randint(0, OUT, (BATCH,), generator=g)
        return x.to(self.device), y.to(self.device)

    def step(self, dist, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        torch = self.torch
        pos = int(self.cursor[1].item())
        x, y = self.batch(pos)
        p = self.params.detach().requires_grad_(True)
        w1, c1, w2, c2 = self.views(p)
        loss = torch.nn.functional.cross_entropy(torch.relu(x @ w1 + c1) @ w2 + c2, y)
        loss.backward()
        with torch.no_grad():
            grad = p.grad.cpu()
            gshard = torch.empty(self.shard)
            dist.reduce_scatter_tensor(gshard, grad, op=dist.ReduceOp.SUM)  # ZeRO-1: my shard's gradients
            gshard = (gshard / self.world).to(self.device)
            t = int(self.cursor[0].item()) + 1
            self.m.mul_(b1).add_(gshard, alpha=1 - b1)
            self.v.mul_(b2).addcmul_(gshard, gshard, value=1 - b2)
            self.master.sub_(lr * (self.m / (1 - b1 ** t)) / ((self.v / (1 - b2 ** t)).sqrt() + eps))
            self.cursor += 1
        self.regather(dist)
        lsum = loss.detach().cpu().reshape(1)
        dist.all_reduce(lsum)
        return float(lsum.item()) / self.world

    def regather(self, dist):
        torch = self.torch
        out = torch.empty(self.shard * self.world)
        dist.all_gather_into_tensor(out, self.master.cpu())
        self.params = out.to(self.device)


def join_group(dist, store, gen, rank, world):
    dist.init_process_group("gloo", init_method="file://" + os.path.join(store, "pg%d" % gen), rank=rank,
                            world_size=world, timeout=datetime.timedelta(seconds=10))


# ---------------------------------------------------------------------------
# process bodies

def worker(args):
    import torch
    import torch.distributed as dist
    from paper_2512_03644_b200 import ffx
    torch.cuda.set_device(args.device)
    torch.backends.cuda.matmul.allow_tf32 = False
    rank, world, store = args.rank, 2, args.store
    me = Trainer(torch, ffx, rank, world, torch.device("cuda", args.device))
    spec = ffx.make_spec(d=world, phi=nparams(), distributed=True)
    ctx = ffx.Context(args.device, spec, ffx.Role(rank, 0, 0))
    for kind, t in me.regions():
        ctx.register(kind, t)
    nbytes = ctx.plan().registered_unique_bytes
    pred = (rank - 1) % world
    held = ctx.create_replica(ffx.Role(pred, 0, 0), nbytes + 4096, 2)  # I hold my predecessor's replica
    put(store, "replica_of_%d_gen0" % pred, held.export())
    target = ctx.open_replica(get(store, "replica_of_%d_gen0" % rank))
    ctx.set_target(target)
    join_group(dist, store, 0, rank, world)
    losses, gen, it = [], 0, 0
    while it < args.iters:
        try:
            loss = me.step(dist)
        except RuntimeError:
            # the peer is gone: this rank's update of `it + 1` never happened
            # (the reduce-scatter failed before it), so its state is still at `it`
            put(store, "worker%d_detected" % rank, str(it).encode())
            dist.destroy_process_group()
            note = json.loads(get(store, "new_generation", timeout=300))
            gen = note["gen"]
            assert note["resume"] == it
            target.destroy()
            target = ctx.open_replica(get(store, "replica_of_%d_gen%d" % (rank, gen)))
            ctx.set_target(target)
            join_group(dist, store, gen, rank, world)
            me.regather(dist)  # parameters from the shards (the replacement's restored master)
            continue
        it += 1
        losses.append(loss)
        ctx.snapshot(it)  # after the optimizer update: master / m / v / cursor of iteration `it`
        torch.cuda.synchronize()
        put(store, "worker%d_committed_%d" % (rank, it), b"1")
        if args.stop_after == it:
            print("WAITING", flush=True)
            sys.stdin.readline()  # the launcher kills this process here
    final = me.params.detach().cpu()
    put(store, "result_rank%d" % rank, json.dumps({"losses": losses}).encode())
    torch.save(final, os.path.join(store, "params_rank%d.pt" % rank))
    dist.barrier()
    dist.destroy_process_group()
    torch.cuda.synchronize()
    target.destroy()
    held.destroy()
    ctx.close()


def spare(args):
    import torch
    import torch.distributed as dist
    from paper_2512_03644_b200 import ffx
    torch.cuda.set_device(args.device)
    torch.backends.cuda.matmul.allow_tf32 = False
    world, store = 2, args.store
    spec = ffx.make_spec(d=world, phi=nparams(), distributed=True)
    torch.zeros(1, device="cuda")  # CUDA context up
    ffx.lib.ffx_prepare_peers(args.device, None)
    print("ARMED", flush=True)
    note = json.loads(sys.stdin.readline())  # the failure notice: lost rank, global consistent iteration
    lost, g, t0 = note["rank"], note["resume"], note["t0"]
    me = Trainer(torch, ffx, lost, world, torch.device("cuda", args.device))
    ctx = ffx.Context(args.device, spec, ffx.Role(lost, 0, 0))
    plan = ffx.plan_recovery(spec, [], [ffx.Role(lost, 0, 0)], g, 0)
    holder = plan.forwards[0][1]  # node of dp_neighbor(lost)
    src = ctx.open_replica(get(store, "replica_of_%d_gen0" % lost))
    for kind, t in me.regions():
        ctx.register(kind, t)
    slot = src.held()[g]
    assert [k for k, _ in src.slot_regions(slot)] == [k for k, _ in me.regions()]
    rpt = ctx.recover(src, g)  # gather + per-slice verify into this process's fresh regions
    t_restored = time.monotonic_ns()
    src.destroy()
    # the replica this rank now holds for its predecessor, and the new group
    nbytes = ctx.plan().registered_unique_bytes
    pred = (lost - 1) % world
    held = ctx.create_replica(ffx.Role(pred, 0, 0), nbytes + 4096, 2)
    gen = note["gen"]
    put(store, "replica_of_%d_gen%d" % (pred, gen), held.export())
    put(store, "replica_of_%d_gen%d" % (lost, gen), get(store, "replica_of_%d_gen0" % lost))
    target = ctx.open_replica(get(store, "replica_of_%d_gen0" % lost))  # worker 0 still holds mine
    ctx.set_target(target)
    join_group(dist, store, gen, lost, world)
    me.regather(dist)
    t_resumed = time.monotonic_ns()
    put(store, "spare_report", json.dumps({
        "restored_iteration": g, "holder_node": holder, "bytes": rpt.bytes, "bad_slices": rpt.bad_slices,
        "kernel_s": rpt.seconds, "notice_to_verified_s": (t_restored - t0) * 1e-9,
        "notice_to_training_resumed_s": (t_resumed - t0) * 1e-9}).encode())
    losses, it = [], g
    while it < args.iters:
        loss = me.step(dist)
        it += 1
        losses.append(loss)
        ctx.snapshot(it)
        torch.cuda.synchronize()
    final = me.params.detach().cpu()
    put(store, "result_rank%d" % lost, json.dumps({"losses": losses}).encode())
    torch.save(final, os.path.join(store, "params_rank%d.pt" % lost))
    dist.barrier()
    dist.destroy_process_group()
    torch.cuda.synchronize()
    target.destroy()
    held.destroy()
    ctx.close()


def launch(args):
    """Run the job with a real failure, then without; compare."""
    me = os.path.abspath(__file__)

    def spawn(role, store, *extra):
        return subprocess.Popen([sys.executable, me, "--role", role, "--store", store,
                                 "--iters", str(args.iters)] + list(extra),
                                stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)

    def wait_line(p, want, timeout=600):
        t_end = time.time() + timeout
        while time.time() < t_end:
            ln = p.stdout.readline()
            if not ln:
                raise RuntimeError("%s exited: %s" % (want, p.stderr.read()[-2000:]))
            if ln.startswith(want):
                return ln
        raise TimeoutError(want)

    import torch
    out = {}
    for label in ("failover", "uninterrupted"):
        with tempfile.TemporaryDirectory() as store:
            fail = label == "failover"
            w0 = spawn("worker", store, "--rank", "0", "--device", "0")
            w1 = spawn("worker", store, "--rank", "1", "--device", "1",
                       *(["--stop-after", str(args.fail_at)] if fail else []))
            sp = spawn("spare", store, "--device", "1") if fail else None
            procs = [w0, w1] + ([sp] if sp else [])
            try:
                if fail:
                    wait_line(sp, "ARMED")
                    wait_line(w1, "WAITING")
                    get(store, "worker0_committed_%d" % args.fail_at)
                    os.kill(w1.pid, signal.SIGKILL)  # rank 1's process and its GPU state are gone
                    w1.wait()
                    t0 = time.monotonic_ns()         # failure notice
                    # both ranks committed fail_at (the ledger's global consistent iteration)
                    note = {"rank": 1, "resume": args.fail_at, "gen": 1, "t0": t0}
                    sp.stdin.write(json.dumps(note) + "\n")
                    sp.stdin.flush()
                    put(store, "new_generation", json.dumps(note).encode())
                    out["spare"] = json.loads(get(store, "spare_report", timeout=300))
                    out["survivor_detected_after_s"] = round((time.monotonic_ns() - t0) * 1e-9, 2) \
                        if os.path.exists(os.path.join(store, "worker0_detected")) else None
                    out["killed_after_iteration"] = args.fail_at
                for p in procs:
                    if p is not w1 or not fail:
                        p.wait(timeout=600)
                        if p.returncode != 0:
                            raise RuntimeError(p.stderr.read()[-3000:])
                res = [json.loads(get(store, "result_rank%d" % r)) for r in (0, 1)]
                params = [torch.load(os.path.join(store, "params_rank%d.pt" % r)) for r in (0, 1)]
                out[label] = {"losses_rank0": res[0]["losses"], "params": params}
            finally:
                for p in procs:
                    if p.poll() is None:
                        p.kill()
    a, b = out["failover"], out["uninterrupted"]
    same = (a["losses_rank0"] == b["losses_rank0"] and all(torch.equal(x, y) for x, y in zip(a["params"], b["params"]))
            and torch.equal(a["params"][0], a["params"][1]))
    print(json.dumps({"killed_after_iteration": out["killed_after_iteration"], "spare": out["spare"],
                      "losses": [round(x, 6) for x in a["losses_rank0"]],
                      "bit_identical_to_uninterrupted_run": bool(same)}), flush=True)
    return 0 if same else 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--role", default="launch", choices=["launch", "worker", "spare"])
    ap.add_argument("--store", default="")
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--fail-at", type=int, default=5)
    ap.add_argument("--stop-after", type=int, default=0)
    args = ap.parse_args()
    if args.role == "worker":
        return worker(args)
    if args.role == "spare":
        return spare(args)
    return launch(args)


if __name__ == "__main__":
    sys.exit(main() or 0)
