"""tvk_posterior at D = 400 on 2048 matrices: full block sweep (M output) vs the phi-only elimination."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1906_08556_b200 import _lib
from paper_1906_08556_b200._lib import call, ptr, stream
U, D = 2048, 400
dev = _lib.device()
g = torch.Generator(device=dev).manual_seed(0)
G = torch.randn((U, D, 48), device=dev, dtype=torch.float64, generator=g)
Lf = G @ G.transpose(1, 2) * (4.0 / 48)
i, j = np.tril_indices(D)
Lpk0 = Lf[:, torch.from_numpy(i).to(dev), torch.from_numpy(j).to(dev)].contiguous()
b = torch.randn((U, D), device=dev, dtype=torch.float64, generator=g)
phi, ld, bp = _lib.empty((U, D)), _lib.empty((U,)), _lib.empty((U,))
st = _lib.empty((U,), torch.int32)
M = _lib.empty(Lpk0.shape)
for mode in ("full", "phi"):
    ts = []
    for _ in range(4):
        lp = Lpk0.clone()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call("tvk_posterior", ptr(lp), ptr(b), U, D, 1 | (2 if mode == "full" else 0), ptr(phi),
             ptr(M if mode == "full" else None), ptr(ld), ptr(bp), ptr(st), None, 0, stream())
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{mode}: {min(ts[1:]):.2f} ms per {U} matrices (D = {D})", flush=True)
