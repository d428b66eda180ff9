"""Start-up cost of align_frames on host frames (config 2 model): model uploads, table builds, the
SPD status check, then the piece pipeline -- wall clock per step, synchronized after each.

    python tools/e2e_startup.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1906_08556_b200 as pkg  # noqa: E402
from paper_1906_08556_b200 import _device, gmm  # noqa: E402

n = 10_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
dm = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
fm = pkg.GmmFull(w, mu, cov)
host = torch.empty((n, 60), dtype=torch.float32, pin_memory=True)
host.copy_(x)
for rep in range(4):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    ft = fm.device_table()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    gmm._raise_if_not_spd(ft)
    t.append(time.perf_counter())
    dt = dm.device_table()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    _device.align_host(host, dt, ft, 20, 0.025)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    pkg.align_frames(dm, fm, host, top_k=20, prune=0.025)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"rep {rep}: full table {d[0]:.2f} ms, spd check {d[1]:.2f} ms, diag table {d[2]:.2f} ms, "
          f"align_host {d[3]:.1f} ms | align_frames total {d[4]:.1f} ms")
