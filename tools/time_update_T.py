"""CUDA-event timing of the per-iteration fixed M-step kernels at config-3 shape (C=2048, F=60, D=400)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1906_08556_b200 import _lib
C, F, D = 2048, 60, 400
P = D * (D + 1) // 2
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
M = torch.randn(64, D, D, device=dev, dtype=torch.float64, generator=g)
A = M @ M.transpose(1, 2) / D + torch.eye(D, device=dev, dtype=torch.float64) * 2
il = torch.tril_indices(D, D, device=dev)
Apk = A[:, il[0], il[1]].repeat(C // 64, 1).contiguous()
B = torch.randn(C, F, D, device=dev, dtype=torch.float64, generator=g)
X = torch.empty_like(B)
status = torch.empty(C, dtype=torch.int32, device=dev)
skip = torch.zeros(C, dtype=torch.int32, device=dev)
ws_bytes = int(_lib.load().tvk_posterior_workspace_bytes(D, C))
ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
f = lambda: _lib.call("tvk_spd_solve_rows", _lib.ptr(Apk), _lib.ptr(B), C, D, F, _lib.ptr(skip), _lib.ptr(X),
                      _lib.ptr(status), _lib.ptr(ws), ws_bytes, _lib.stream())
f(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): f()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
ref = torch.linalg.solve(A[0], B[0].T).T
print(f"spd_solve_rows C={C} D={D} R={F}: {ms:.1f} ms; max rel err vs torch {float((X[0]-ref).abs().max()/ref.abs().max()):.2e}")
