"""One process, two GPUs: the fused snapshot kernel on GPU 0 pushing a
2.34 GB GPT-2 XL shard into a replica held on GPU 1 (peer access), for an
ncu capture of the NVLink path (one process, so ncu can replay it)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2512_03644_b200 import ffx, state  # noqa: E402

n = (12 * 1_557_611_200 + 7) // 8
spec = ffx.make_spec(d=8, phi=1_557_611_200, distributed=True)
holder = ffx.Context(1, spec, (2, 0, 0))
origin = ffx.Context(0, spec, (1, 0, 0))
rep = holder.create_replica((1, 0, 0), n, 2)
torch.cuda.set_device(0)
view = origin.open_replica(rep.export())
origin.set_target(view)
t = torch.empty(n, dtype=torch.uint8, device="cuda:0")
ffx.materialize(t, state.optimizer_init(42, 1, 0, 0))
origin.register(ffx.REGION_BLOB, t)
s = torch.cuda.Stream(device=0)
for it in range(1, 6):
    origin.snapshot(it, stream=s)
s.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for it in range(6, 11):
    origin.snapshot(it, stream=s)
e1.record(s)
s.synchronize()
print("push GB/s (one writer):", round(5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1))
origin.inject(ffx.FAULT_POISON_STATE)
assert origin.recover(view, 10).bad_slices == 0 and ffx.blob_is_sound(t)
torch.cuda.synchronize()
view.destroy()
rep.destroy()
