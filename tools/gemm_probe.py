"""One bf16 GEMM of the synthetic step's shape (step.py) for ncu's launch stats."""
import torch
x = torch.randn(8192, 4096, dtype=torch.bfloat16, device="cuda")
w = torch.randn(4096, 4096, dtype=torch.bfloat16, device="cuda")
y = torch.empty(8192, 4096, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    torch.matmul(x, w, out=y)
torch.cuda.synchronize()
