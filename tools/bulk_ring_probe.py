#!/usr/bin/env python3
"""Does the NVLink rate of SM-issued traffic depend on the transfer shape?
Ring of N ranks (torchrun): every rank moves N bytes to its successor with
  bulk-push   1-D TMA bulk copies (32 KB ops, ffx_copy) stored into the peer
  bulk-pull   the same kernel run by the successor, loading from the peer
  ce          cudaMemcpyAsync (copy engines)
at several CTA counts.  Per-GPU GB/s, max over ranks.  JSON lines on rank 0."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2512_03644_b200 import ffx, state  # noqa: E402


def main():
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = int(os.environ.get("PROBE_BYTES", str(2 << 30)))
    src, dst = ctypes.c_void_p(), ctypes.c_void_p()
    ffx.check(ffx.lib.ffx_device_alloc(local, n, ctypes.byref(src)), "alloc")
    ffx.check(ffx.lib.ffx_device_alloc(local, n, ctypes.byref(dst)), "alloc")
    ffx.materialize(src.value, state.optimizer_init(1, rank, 0, 0), n)
    torch.cuda.synchronize()
    hs = [None] * world
    dist.all_gather_object(hs, (ffx.ipc_export(src.value), ffx.ipc_export(dst.value)))
    succ, pred = (rank + 1) % world, (rank - 1) % world
    succ_dst = ffx.ipc_open(hs[succ][1])
    pred_src = ffx.ipc_open(hs[pred][0])
    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)

    def run(kind, ctas):
        if kind == "bulk-push":
            ffx.check(ffx.lib.ffx_copy(ctypes.c_void_p(succ_dst), src, n, ctas, sp), "copy")
        elif kind == "bulk-pull":
            ffx.check(ffx.lib.ffx_copy(dst, ctypes.c_void_p(pred_src), n, ctas, sp), "copy")
        else:
            ffx.check(ffx.lib.ffx_memcpy(ctypes.c_void_p(succ_dst), src, n, sp, 0), "memcpy")

    for kind, caps in (("bulk-push", (16, 32, 64, 148)), ("bulk-pull", (16, 32, 64, 148)), ("ce", (0,))):
        for c in caps:
            for _ in range(2):
                run(kind, c)
            s.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            k = 5
            e0.record(s)
            for _ in range(k):
                run(kind, c)
            e1.record(s)
            s.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / k], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rank == 0:
                print(json.dumps({"kind": kind, "ctas": c, "world": world, "ms": round(float(t.item()), 4),
                                  "gbs_per_gpu": round(n / float(t.item()) / 1e6, 1)}), flush=True)
    dist.barrier()
    ffx.ipc_close(succ_dst)
    ffx.ipc_close(pred_src)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
