"""Candidate counts per frame handed from select_tc_kernel to select_post_kernel (config-2 frames,
diagnostics build, TVK_SELECT_DEBUG=9), per pass-0 slack kappa1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from build_diag import use_diag
use_diag()
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib, _device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
tab = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))).device_table()
os.environ["TVK_SELECT"] = "tc_noexact"
for e in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["12", "13", "14", "15"]):
    os.environ["TVK_SELECT_KAPPA1"] = repr(2.0 ** -float(e))
    os.environ["TVK_SELECT_DEBUG"] = "9"
    _, val = _device.select_topk(x, tab, 20, values=True)
    torch.cuda.synchronize()
    v = val[:, :2].cpu().numpy()
    ok = (v >= 0).all(1)
    tot = v[ok].sum(1)
    os.environ["TVK_SELECT_DEBUG"] = "0"
    q = np.percentile(tot, [10, 50, 90, 99])
    print(f"kappa1=2^-{e}: overflow {100 * (~ok).mean():.3f}%  n0+n1 mean {tot.mean():.1f}  p10/50/90/99 {q}  "
          f"n>32 {100 * (tot > 32).mean():.1f}%  per-half max {v[ok].max()}", flush=True)
