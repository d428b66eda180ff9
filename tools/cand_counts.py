"""Distribution of pass-1 candidate counts per frame half (TVK_SELECT_DEBUG=9)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _device
n = 500_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
tab = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))).device_table()
for k1 in [None, "0.000976", "0.000244", "0.000061", "0.0000153"]:
    if k1: os.environ["TVK_SELECT_KAPPA1"] = k1
    os.environ["TVK_SELECT_DEBUG"] = "9"; os.environ["TVK_SELECT"] = "tc_noexact"
    sel, val = _device.select_topk(x, tab, 20, values=True)
    v = val.cpu().numpy()
    n0, n1 = v[:, 0], v[:, 1]
    tot = np.where((n0 < 0) | (n1 < 0), 99, n0 + n1)
    print("kappa1", k1, "n0+n1 mean", tot[tot < 99].mean(), "pct", np.percentile(tot, [5, 50, 95, 99]), "overflow frac", (tot == 99).mean(), "<K frac", (tot < 20).mean(), flush=True)
    os.environ.pop("TVK_SELECT_DEBUG"); os.environ.pop("TVK_SELECT")
    os.environ["TVK_SELECT_DEBUG"] = "0"
    import time
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(3): _device.select_topk(x, tab, 20)
    torch.cuda.synchronize(); print("   time per 1e6 frames (ms):", (time.perf_counter() - t0) / 3 / n * 1e9 / 1e3)
    os.environ.pop("TVK_SELECT_DEBUG")
