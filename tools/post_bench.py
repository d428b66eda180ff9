"""Time tvk_posterior at the EM shape (D=400, 1024 utterances): block sweep vs Cholesky kernel.

python tools/post_bench.py [U] [D]   -- prints ms per call, TFLOP/s (D^3 flop/utt) and max diffs.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_08556_b200 import _lib  # noqa: E402
from paper_1906_08556_b200._lib import call, ptr, stream  # noqa: E402

U = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
D = int(sys.argv[2]) if len(sys.argv) > 2 else 400
dev = _lib.device()
g = torch.Generator(device=dev).manual_seed(0)
G = torch.randn((U, D, 48), device=dev, dtype=torch.float64, generator=g)
Lfull = G @ G.transpose(1, 2) * (4.0 / 48)  # + I added by the kernel flag
i, j = np.tril_indices(D)
ii, jj = torch.from_numpy(i).to(dev), torch.from_numpy(j).to(dev)
Lpk0 = Lfull[:, ii, jj].contiguous()
b = torch.randn((U, D), device=dev, dtype=torch.float64, generator=g)
P = Lpk0.shape[1]


def run(mode, reps=5):
    if mode == "chol":
        os.environ["TVK_POSTERIOR_CHOL"] = "1"
    else:
        os.environ.pop("TVK_POSTERIOR_CHOL", None)
    outs = None
    times = []
    for r in range(reps + 1):
        Lpk = Lpk0.clone()
        phi = torch.empty((U, D), device=dev, dtype=torch.float64)
        ld = torch.empty((U,), device=dev, dtype=torch.float64)
        bp = torch.empty((U,), device=dev, dtype=torch.float64)
        st = torch.empty((U,), device=dev, dtype=torch.int32)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call("tvk_posterior", ptr(Lpk), ptr(b), U, D, 3, ptr(phi), ptr(Lpk), ptr(ld), ptr(bp), ptr(st), None, 0,
             stream())
        e1.record()
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1))
        outs = (Lpk, phi, ld, bp, st)
    return float(np.median(times)), outs


ts, so = run("sweep")
tc, co = run("chol")
flop = U * float(D) ** 3
print(f"U={U} D={D}: sweep {ts:.3f} ms ({flop / ts / 1e9:.2f} TF), chol {tc:.3f} ms ({flop / tc / 1e9:.2f} TF)")
for name, a, c in zip(["M", "phi", "logdet", "bphi"], so[:4], co[:4]):
    rel = (a - c).abs().max().item() / max(c.abs().max().item(), 1e-300)
    print(f"  {name}: max rel diff {rel:.2e}")
print("  status ok:", int((so[4] == 0).sum()), int((co[4] == 0).sum()))
# direct check of a few utterances against torch fp64 inverse
for u in (0, U - 1):
    Lu = Lfull[u] + torch.eye(D, device=dev, dtype=torch.float64)
    Phi = torch.linalg.inv(Lu)
    ph = Phi @ b[u]
    M = Phi + torch.outer(ph, ph)
    print(f"  utt {u}: M err {((so[0][u] - M[ii, jj]).abs().max() / M.abs().max()).item():.2e}, "
          f"phi err {((so[1][u] - ph).abs().max() / ph.abs().max()).item():.2e}, "
          f"logdet err {abs(so[2][u].item() - torch.linalg.slogdet(Lu)[1].item()):.2e}")
