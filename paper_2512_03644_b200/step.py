"""Synthetic ZeRO-3 training step with the slice scheduler in its gaps.

This is the workload the step-overhead number is measured on (BASELINE.json
configs[2]: Llama-3 8B ZeRO-3 state, snapshot overlapped with the step's own
collectives).  The step is plumbing -- NCCL all-gather / reduce-scatter of bf16
layer shards plus cuBLAS bf16 GEMMs sized to a Llama-3-8B layer's compute --
and stands in for a real training step; the product is the snapshot that
rides in its gaps.

Scheduling (reference semantics: STATE traffic only when no TRAIN chunk is
queued, inversion bounded by one chunk -- sim_net.cpp:401-454,
test_transport.cpp:173-197), carried out by the native scheduler in libffx
(ffx_sched_*; this module only reports the step's gaps to it):
  * the step runs on a high-priority stream, snapshot batches on a
    low-priority one with a capped CTA count, so the block scheduler prefers
    the step and a batch can delay TRAIN by at most its in-flight tasks;
  * policy "fused": one fused copy+checksum batch per all-gather gap
    (forward and backward), gated on an event recorded right after the
    all-gather (NVLink goes quiet while the GEMMs run), sized by the measured
    gap durations (calibrate());
  * policy "split": the copy (TMA copy-only kernel, few SMs -- or the copy
    engines) goes into those same compute gaps, while the checksum work
    (SM-heavy, HBM-only) is gated on events recorded right *before* each
    all-gather, i.e. it runs while the SMs idle behind NCCL;
  * the optimizer update of iteration n+1 waits on the snapshot's commit --
    the fp32 master / Adam state is only mutated there (SURVEY 7.2 hard part
    4), so the snapshot streams from the live buffers with no staging copy.
"""
from __future__ import annotations

import statistics

import torch
import torch.distributed as dist

# Llama-3 8B: 32 layers, hidden 4096, 8,030,261,248 parameters.
LLAMA3_8B_PARAMS = 8_030_261_248
LLAMA3_8B_LAYERS = 32


class SyntheticStep:
    def __init__(self, world: int, params: int = LLAMA3_8B_PARAMS, layers: int = LLAMA3_8B_LAYERS,
                 tokens: int = 8192, hidden: int = 4096, fwd_gemms: int = 6, device=None):
        self.world = world
        self.layers = layers
        self.fwd_gemms = fwd_gemms
        layer_params = params // layers
        self.shard_numel = (layer_params + world - 1) // world
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.shard = torch.randn(self.shard_numel, dtype=torch.bfloat16, device=dev)
        self.full = torch.empty(self.shard_numel * world, dtype=torch.bfloat16, device=dev)
        self.grad_full = torch.randn(self.shard_numel * world, dtype=torch.bfloat16, device=dev)
        self.grad_shard = torch.empty(self.shard_numel, dtype=torch.bfloat16, device=dev)
        self.x = torch.randn(tokens, hidden, dtype=torch.bfloat16, device=dev)
        self.y = torch.empty(tokens, hidden, dtype=torch.bfloat16, device=dev)
        self.w = self.full[: hidden * hidden].view(hidden, hidden)
        self.train = torch.cuda.Stream(priority=-1)  # TRAIN outranks STATE
        # bytes one rank moves over NVLink per step in its own collectives
        self.train_link_bytes = 3 * self.shard_numel * 2 * (world - 1) * layers

    def _gemms(self, n):
        for _ in range(n):
            torch.matmul(self.x, self.w, out=self.y)

    def run(self, hook=None):
        """One step on self.train.  hook(kind, layer) marks the gaps:
        'pre_ag' before an all-gather, 'fwd'/'bwd' once it completed,
        'pre_rs' before a reduce-scatter, 'opt' before the optimizer update."""
        h = hook or (lambda kind, layer: None)
        with torch.cuda.stream(self.train):
            for l in range(self.layers):
                h("pre_ag", l)
                dist.all_gather_into_tensor(self.full, self.shard)
                h("fwd", l)
                self._gemms(self.fwd_gemms)
            for l in reversed(range(self.layers)):
                h("pre_ag", self.layers + l)
                dist.all_gather_into_tensor(self.full, self.shard)
                h("bwd", l)
                self._gemms(2 * self.fwd_gemms)
                h("pre_rs", l)
                dist.reduce_scatter_tensor(self.grad_shard, self.grad_full)
            h("opt", None)
            self.shard.add_(self.grad_shard, alpha=-1e-6)  # the optimizer update


class SliceScheduler:
    """Drives one ffx snapshot per step through the gaps of a SyntheticStep."""

    def __init__(self, ctx, step: SyntheticStep, policy: str = "split", copy_ctas: int = 8,
                 hash_ctas: int = 96, copy_engine: bool = False, front: float = 1.0, rs_gaps: bool = False,
                 task_ctas: bool = False):
        from paper_2512_03644_b200 import ffx
        self.ffx = ffx
        self.ctx = ctx
        self.step = step
        self.policy = policy
        self.copy_ctas = copy_ctas
        self.hash_ctas = hash_ctas
        self.copy_engine = copy_engine
        # Only the first `front` share of the step's gaps carries batches: the
        # idle-link windows hold several times what the copy needs, and a batch
        # that overruns the last gaps delays the optimizer (which waits for
        # the commit).
        self.front = front
        self.rs_gaps = rs_gaps  # checksum batches also before each reduce-scatter
        # fused policy: task-granular batches (one CTA per task group, no
        # persistent loop) -- STATE yields SMs to TRAIN at every task boundary
        self.task_ctas = task_ctas
        self.native = None  # ffx.Sched, built on first use / after calibrate()

    weights = None  # measured idle-link window per copy gap (calibrate())

    def calibrate(self):
        """Measure the step's idle-link windows: from each all-gather's
        completion to the next collective (or the optimizer).  The copy
        batches are then sized in proportion (ffx_snapshot_opts.batch_weights)."""
        marks = []

        def rec(kind, layer):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(self.step.train)
            marks.append((kind, ev))

        self.step.run(rec)
        torch.cuda.synchronize()
        w = []
        for i, (kind, ev) in enumerate(marks):
            if kind in ("fwd", "bwd") and i + 1 < len(marks):
                w.append(max(ev.elapsed_time(marks[i + 1][1]), 1e-3))
        self.weights = w
        self._make()
        return w

    def _make(self):
        """(Re)build the native scheduler (ffx_sched_*) for this policy and
        the measured gaps: one copy batch per link-idle gap (after each
        all-gather, 2L per step) and, split policies, one checksum batch per
        SM-idle gap (before each all-gather)."""
        if self.native is not None:
            self.native.destroy()
        G = 2 * self.step.layers
        ffx = self.ffx
        pol = ffx.SCHED_FUSED if self.policy == "fused" else (ffx.SCHED_SPLIT_CE if self.copy_engine
                                                               else ffx.SCHED_SPLIT)
        gaps = self.weights if self.weights and len(self.weights) == G else None
        k = max(1, min(G, int(round(G * self.front))))
        if k < G:
            gaps = [x if i < k else 0.0 for i, x in enumerate(gaps or [1.0] * G)]
        # SM-idle gaps: before every all-gather and, if enabled, every reduce-scatter
        S = G + (self.step.layers if self.rs_gaps else 0)
        ks = max(1, min(S, int(round(S * self.front))))
        self.native = ffx.Sched(self.ctx, pol, link_gaps=G, sm_gaps=0 if pol == ffx.SCHED_FUSED else ks,
                                copy_ctas=self.copy_ctas or (1 << 20), hash_ctas=self.hash_ctas or (1 << 20),
                                gap_ms=gaps, task_ctas=self.task_ctas)

    def begin(self, iteration: int):
        if self.native is None:
            self._make()
        self.native.begin(iteration)

    def hook(self, kind, layer):
        if kind == "pre_ag" or (kind == "pre_rs" and self.rs_gaps):  # NCCL about to run: SMs idle
            self.native.gap(self.ffx.GAP_SM_IDLE, self.step.train)
        elif kind in ("fwd", "bwd"):  # collective done: NVLink idle while the GEMMs run
            self.native.gap(self.ffx.GAP_LINK_IDLE, self.step.train)
        elif kind == "opt":       # flush, and the optimizer waits for the commit
            self.native.finish(self.step.train)

    def close(self):
        if self.native is not None:
            self.native.destroy()
            self.native = None


def time_steps(step: SyntheticStep, n: int, sched: SliceScheduler | None = None, it0: int = 0):
    """Per-step device time (ms) of n steps, max over ranks for each step."""
    out = []
    for i in range(n):
        if sched is not None:
            sched.begin(it0 + i)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(step.train)
        step.run(sched.hook if sched is not None else None)
        e1.record(step.train)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out.append(float(t.item()))
    return out


def measure_overhead(step: SyntheticStep, sched: SliceScheduler, steps: int = 8, warmup: int = 2,
                     it0: int = 1):
    """Interleaved A/B: steps without and with the concurrent snapshot."""
    time_steps(step, warmup)
    sched.calibrate()
    time_steps(step, warmup, sched, it0=it0 + 100_000)
    base, with_snap = [], []
    it = it0
    for _ in range(steps):
        base += time_steps(step, 1)
        with_snap += time_steps(step, 1, sched, it0=it)
        it += 1
    b = statistics.median(base)
    w = statistics.median(with_snap)
    return {"policy": sched.policy + ("+ce" if sched.copy_engine else "") + ("+tasks" if sched.task_ctas else ""),
            "copy_ctas": sched.copy_ctas,
            "measured_gaps_ms": [round(sum(sched.weights), 3), len(sched.weights)] if sched.weights else None,
            "hash_ctas": sched.hash_ctas, "step_ms_without": round(b, 3), "step_ms_with": round(w, 3),
            "overhead_pct": round(100.0 * (w - b) / b, 3), "steps_each": steps,
            "train_link_bytes_per_step": step.train_link_bytes}
