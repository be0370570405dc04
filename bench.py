#!/usr/bin/env python3
"""bench.py -- per-iteration neighbour snapshot (+ recovery) throughput.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ffx|reference]

Workload (BASELINE.json configs[1]): the GPT-2 XL ZeRO-1 shard a DP rank
owns at d=8 -- N = ceil(12 * 1,557,611,200 / 8) = 2,336,416,800 bytes of
unique Adam state (evo::optimizer_bytes, reference evolution.cpp:15-19),
synthesised on the device as evo::materialize(optimizer_init(42, role), N).

One step = one per-iteration snapshot of every rank's N bytes into its
replica slot with fused per-slice FNV-1a-64 (the reference's
HostSnapshots::take + ring stream + NeighborBuffer::store):
  N = 1: into a local replica on the same B200 (HBM-bound: 2N bytes).
  N > 1: into the ring successor's replica over NVLink (weak scaling: every
         rank moves its own N bytes; one process per GPU, torchrun).
Inputs (2.3 GB per rank) exceed the 126 MB L2, so no flush is needed.

Also reported on the same line: recovery (pull + verify of a failed rank's
N bytes from its holder), the end-to-end path through the reference-facing
call with host buffers (e2e), the dominant kernel's roofline, the reference
CPU path timed on this host (cpu_baseline), and clocks under load.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PHI_GPT2_XL = 1_557_611_200
D_REF = 8
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
NVLINK_MEASURED_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction (900 nominal)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ffx", choices=["ffx", "reference"])
    ap.add_argument("--slice-bytes", type=int, default=4096)
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--bytes", type=int, default=0, help="override bytes per rank (debug)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def workload_bytes(args):
    if args.bytes:
        return args.bytes
    full = 12 * PHI_GPT2_XL
    return (full + D_REF - 1) // D_REF


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "MEASURED_PEAKS.json"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref: the reference's own C++ compiled here)

def cpu_ring(threads, bytes_per_thread, iters):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    ref = pyoracle.ref_lib()
    if ref is None:
        return None
    h = ref.ref_ring_setup(threads, bytes_per_thread)
    secs = (ctypes.c_double * 4)()
    out = []
    for i in range(iters):
        rc = ref.ref_ring_run(h, i + 1, secs)
        if rc != 0:
            raise RuntimeError("reference ring iteration failed")
        out.append(tuple(secs[k] for k in range(4)))
    ref.ref_ring_free(h)
    return out


def cpu_baseline_line(threads, bytes_per_thread, iters=2):
    res = cpu_ring(threads, bytes_per_thread, iters)
    if res is None:
        return None
    take = min(r[0] for r in res)
    store = min(r[1] for r in res)
    restore = min(r[2] for r in res)
    agg = threads * bytes_per_thread
    return {
        "value": round(agg / (take + store) / 1e9, 3), "unit": "GB/s",
        "cores": threads, "kind": "reference",
        "sample": "%d threads x %d MiB: HostSnapshots::take + NeighborBuffer::store (snapshot), "
                  "assemble_restore timed separately; reference proj/src compiled -O3 into oracle/_ref"
                  % (threads, bytes_per_thread >> 20),
        "stages_gbs": {"take": round(agg / take / 1e9, 3), "store": round(agg / store / 1e9, 3),
                       "restore": round(agg / restore / 1e9, 3)},
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    per = 256 << 20
    steps, warmup = args.steps, args.warmup
    # bounded sample: each step is one ring iteration over `threads` ranks of `per` bytes
    res = cpu_ring(threads, per, max(1, warmup) + steps)
    res = res[max(1, warmup):]
    agg = threads * per
    snap_s = [r[0] + r[1] for r in res]
    t = sum(snap_s)
    value = agg * len(res) / t / 1e9
    line = {
        "impl": "reference", "metric": "snapshot GB/s (per-iteration neighbour backup, all ranks)",
        "value": round(value, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
        "ms_per_step": round(1e3 * t / len(res), 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (evo::materialize, seed 42)",
        "config": {"workload": "reference CPU path on a bounded sample of the GPT-2 XL ZeRO-1 d=8 shard",
                   "bytes_per_rank_sample": per, "ranks": threads},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "kind": "reference",
                         "sample": "%d threads x 256 MiB per step (HostSnapshots::take + NeighborBuffer::store)" % threads},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "restore_gbs": round(agg * len(res) / sum(r[2] for r in res) / 1e9, 3),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 path

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from paper_2512_03644_b200 import ffx

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    n = workload_bytes(args)
    d = max(world, 2)
    spec = ffx.make_spec(d=d, phi=PHI_GPT2_XL, distributed=True)
    me = ffx.Role(rank, 0, 0)
    pred = (rank - 1) % world if world > 1 else rank
    ctx = ffx.Context(local, spec, me, args.slice_bytes)
    if world == 1:
        holder = ffx.Context(local, spec, ffx.Role(1, 0, 0), args.slice_bytes)
        replica = holder.create_replica(me, n, 2)
        target = ctx.open_replica(replica.export())
        succ_replica = target
    else:
        holder = None
        replica = ctx.create_replica(ffx.Role(pred, 0, 0), n, 2)  # I hold my predecessor's snapshots
        handles = [None] * world
        dist.all_gather_object(handles, replica.export())
        target = ctx.open_replica(handles[(rank + 1) % world])  # my successor holds mine
        succ_replica = target
    ctx.set_target(target)

    import hashlib
    digest = hashlib.sha256(b"O0-%d" % rank).digest()
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import pyoracle
        digest = pyoracle.optimizer_init(42, rank, 0, 0, True)
    except Exception:
        pass
    state = torch.empty(n, dtype=torch.uint8, device="cuda")
    ffx.materialize(state, digest)
    ctx.register(ffx.REGION_BLOB, state)
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    it = 0
    for _ in range(args.warmup):
        it += 1
        ctx.snapshot(it, stream=stream, max_ctas=args.max_ctas)
    stream.synchronize()
    launches0 = ctx.stats().kernel_launches
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        it += 1
        ctx.snapshot(it, stream=stream, max_ctas=args.max_ctas)
    e1.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    ck = clocks.stop()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.stats().kernel_launches - launches0
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    per_step_ms = ms_max / args.steps
    value = world * n * args.steps / (ms_max * 1e-3) / 1e9

    # correctness of the last snapshot: holder-side slot committed at `it`
    ok_commit = target.newest() == it

    # ---- recovery: rank (1 % world) loses its state and pulls it back --------
    fail_rank = 1 % world
    rec = {}
    barrier()
    if rank == fail_rank:
        ctx.inject(ffx.FAULT_POISON_STATE)
        src = target  # holder of my snapshots = my successor (or the local holder)
        rpt = ctx.recover(src, it, stream=stream)
        sound = ffx.blob_is_sound(state)
        rec = {"recovery_s": rpt.seconds, "recovery_gbs": n / rpt.seconds / 1e9,
               "recovery_verified": bool(sound and rpt.bad_slices == 0)}
    barrier()
    recs = [rec]
    if world > 1:
        recs = [None] * world
        dist.all_gather_object(recs, rec)
    rec = recs[fail_rank]

    # ---- e2e: the reference-facing call with host buffers --------------------
    e2e = None
    if not args.no_e2e:
        host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        host.copy_(state, non_blocking=False)
        nsl = (n + args.slice_bytes - 1) // args.slice_bytes
        table_host = torch.empty(nsl, dtype=torch.int64, pin_memory=True)
        k = max(2, min(args.steps, 6))
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for j in range(k + 1):
                if j == 1:
                    f0.record(stream)
                it += 1
                state.copy_(host, non_blocking=True)               # H2D: take(it, host_ptr, len)
                ctx.snapshot(it, stream=stream, max_ctas=args.max_ctas)
                ctx.read_sums(table_host, stream=stream)           # D2H of the step's result
            f1.record(stream)
        stream.synchronize()
        ems = f0.elapsed_time(f1)
        t = torch.tensor([ems], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": round(world * n * k / (float(t.item()) * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": n, "d2h_bytes_per_step": nsl * 8,
               "path": "pinned host state -> H2D -> ffx_snapshot -> D2H checksum table (HostSnapshots::take semantics)"}

    peaks, peak_src = measured_peaks()
    if world == 1:
        roof = {"bound": "hbm", "achieved": round(2 * n / (per_step_ms * 1e-3) / 1e9, 1),
                "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                "traffic": None, "kernel": "slice_kernel<Copy,commit> (copy + per-slice FNV-1a)",
                "algorithmic_bytes_per_launch": 2 * n, "peak_source": peak_src}
    else:
        roof = {"bound": "nvlink", "achieved": round(n / (per_step_ms * 1e-3) / 1e9, 1),
                "peak": NVLINK_MEASURED_GBS, "unit": "GB/s", "traffic": None,
                "kernel": "slice_kernel<Copy,commit> (peer stores + per-slice FNV-1a)",
                "algorithmic_bytes_per_launch": n,
                "peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)"}
    roof["frac"] = round(roof["achieved"] / roof["peak"], 4) if roof["peak"] else None
    prof = os.path.join(ROOT, "profiles", "traffic_w%d.json" % world)
    if os.path.exists(prof):
        try:
            roof["traffic"] = json.load(open(prof)).get("traffic_bytes_per_launch")
        except Exception:
            pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_line(min(8, os.cpu_count() or 1), 128 << 20)
        except Exception as ex:  # reported, never fatal
            cpu = {"error": str(ex)}

    if rank == 0:
        line = {
            "metric": "snapshot GB/s (per-iteration neighbour backup, all ranks)",
            "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(per_step_ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (evo::materialize(optimizer_init(42, role)), device-generated)",
            "config": {"workload": "GPT-2 XL ZeRO-1 d=8 shard (BASELINE configs[1]): %d B/rank unique Adam state, "
                                   "%s" % (n, "1-GPU local replica" if world == 1 else "ring-neighbour replica over NVLink"),
                       "bytes_per_rank": n, "slice_bytes": args.slice_bytes, "replica_versions": 2,
                       "l2": "inputs 2.3 GB/rank > 126 MB L2; no flush needed",
                       "parallelism": "dp%d ring" % world if world > 1 else "single GPU"},
            "per_gpu_gbs": round(value / world, 3),
            "nvlink_frac_per_gpu": round(value / world / NVLINK_MEASURED_GBS, 4) if world > 1 else None,
            "roofline": roof,
            "recovery": rec,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": ck,
            "commit_ok": bool(ok_commit),
        }
        print(json.dumps(line), flush=True)

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
