"""Whole-payload FNV-1a-64 over the GPT-2 XL shard (2.34 GB): the export path (measurement tooling)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2512_03644_b200 import ffx
n = 2_336_416_800
t = torch.empty(n, dtype=torch.uint8, device='cuda')
ffx.materialize(t, bytes(range(32)))
for _ in range(2):
    h = ffx.checksum64(t)
torch.cuda.synchronize()
print(hex(h))
