"""cuBLAS DGEMM at the E-step shape (reference point for tools/gemm_bench.py under ncu)."""
import torch

a = torch.rand(1024, 2048, device="cuda", dtype=torch.float64)
b = torch.rand(2048, 80200, device="cuda", dtype=torch.float64)
for _ in range(2):
    torch.mm(a, b)
torch.cuda.synchronize()
