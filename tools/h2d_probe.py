"""Host->device copy bandwidth per GPU, all ranks at once and rank 0 alone
(torchrun).  Separates the host / PCIe side of the e2e number from ffx."""
import json
import os

import torch
import torch.distributed as dist

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
dist.init_process_group("nccl")
n = 2_336_416_800
host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
host.fill_(1)
dev = torch.empty(n, dtype=torch.uint8, device="cuda")


def run(active):
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if active:
        e0.record()
        for _ in range(4):
            dev.copy_(host, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    return 4 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9 if active else 0.0


run(True)
together = run(True)
alone = run(rank == 0)
t = torch.tensor([together], device="cuda")
g = [torch.zeros_like(t) for _ in range(world)]
dist.all_gather(g, t)
if rank == 0:
    print(json.dumps({"world": world, "h2d_gbs_each_all_at_once": [round(float(x), 1) for x in g],
                      "h2d_gbs_total": round(sum(float(x) for x in g), 1), "h2d_gbs_rank0_alone": round(alone, 1),
                      "numa_nodes": len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")])}))
dist.destroy_process_group()
