"""Synthetic ZeRO-3 training step with the slice scheduler in its gaps.

This is the workload the step-overhead number is measured on (BASELINE.json
configs[2]: Llama-3 8B ZeRO-3 state, snapshot overlapped with the step's own
collectives).  The step is plumbing -- NCCL all-gather / reduce-scatter of bf16
layer shards plus cuBLAS bf16 GEMMs sized to a Llama-3-8B layer's compute --
and stands in for a real training step; the product is the snapshot that
rides in its gaps.

Scheduling policy (reference semantics: STATE traffic only when no TRAIN
chunk is queued, inversion bounded by one chunk -- sim_net.cpp:401-454,
test_transport.cpp:173-197):
  * the snapshot of iteration n is split into one batch per forward layer;
  * batch l is gated on an event recorded right after layer l's all-gather
    completes, i.e. when NVLink goes quiet and the GEMMs start;
  * it runs on a lower-priority stream with a capped CTA count, so the block
    scheduler prefers the step's kernels and a batch delays TRAIN by at most
    its in-flight warp tasks;
  * the optimizer update of iteration n+1 waits on the snapshot's completion
    event -- the fp32 master / Adam state is only mutated there (SURVEY 7.2
    hard part 4), so the snapshot streams from the live buffers with no
    staging copy.
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
        """One step on self.train.  hook(kind, layer) is called at each gap."""
        with torch.cuda.stream(self.train):
            for l in range(self.layers):
                dist.all_gather_into_tensor(self.full, self.shard)
                if hook:
                    hook("fwd", l)
                self._gemms(self.fwd_gemms)
            for l in reversed(range(self.layers)):
                dist.all_gather_into_tensor(self.full, self.shard)
                if hook:
                    hook("bwd", l)
                self._gemms(2 * self.fwd_gemms)
                dist.reduce_scatter_tensor(self.grad_shard, self.grad_full)
            if hook:
                hook("opt", None)
            self.shard.add_(self.grad_shard, alpha=-1e-6)  # the optimizer update


class SliceScheduler:
    """Issues one snapshot batch per forward-layer gap of a SyntheticStep."""

    def __init__(self, ctx, step: SyntheticStep, max_ctas: int = 32):
        self.ctx = ctx
        self.step = step
        self.max_ctas = max_ctas
        self.low = torch.cuda.Stream(priority=0)
        self.done = torch.cuda.Event()
        self.iteration = 0
        self.remaining = 0

    def begin(self, iteration: int):
        self.iteration = iteration
        self.remaining = self.ctx.snapshot_begin(iteration, batches=self.step.layers, max_ctas=self.max_ctas)

    def hook(self, kind, layer):
        train = self.step.train
        if kind == "fwd" and self.remaining:
            gap = torch.cuda.Event()
            gap.record(train)
            self.remaining = self.ctx.snapshot_next(stream=self.low, gate_event=gap)
            if self.remaining == 0:
                self.done.record(self.low)
        elif kind == "opt":
            while self.remaining:  # more batches than gaps: flush the rest now
                self.remaining = self.ctx.snapshot_next(stream=self.low)
                if self.remaining == 0:
                    self.done.record(self.low)
            train.wait_event(self.done)  # optimizer mutates the snapshotted state


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


def measure_overhead(step: SyntheticStep, sched: SliceScheduler, steps: int = 8, warmup: int = 2):
    """Interleaved A/B: steps without and with the concurrent snapshot."""
    time_steps(step, warmup)
    time_steps(step, warmup, sched, it0=1_000_000)
    base, with_snap = [], []
    it = 1
    for _ in range(steps):
        base += time_steps(step, 1)
        with_snap += time_steps(step, 1, sched, it0=it)
        it += 1
    b = statistics.median(base)
    w = statistics.median(with_snap)
    return {"step_ms_without": round(b, 3), "step_ms_with": round(w, 3),
            "overhead_pct": round(100.0 * (w - b) / b, 3), "steps_each": steps,
            "train_link_bytes_per_step": step.train_link_bytes}
