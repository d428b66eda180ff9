"""Preselection cost vs the pass-0 slack kappa1 (config-2 frames, product build: TVK_SELECT_KAPPA1 is
the test hook of select_tc.cu).  kappa1 only moves work between the tensor-core kernels and
select_exact_kernel (the window check proves every collection complete), so every row must be
identical to the FP64 DMMA selection."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
k1s = sys.argv[2].split(",") if len(sys.argv) > 2 else ["12", "13", "14", "15", "16"]
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
tab = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))).device_table()
sel = _lib.empty((n, 20), torch.int32)
f = lambda: _lib.call("tvk_select_topk", _lib.ptr(x), 0, n, 60, _lib.ptr(tab.table), 2048, 20, _lib.ptr(sel), None,
                      _lib.stream())
os.environ["TVK_SELECT"] = "dmma"
f(); torch.cuda.synchronize(); ref = sel.clone()
os.environ["TVK_SELECT"] = "tc"
for e in k1s:
    os.environ["TVK_SELECT_KAPPA1"] = repr(2.0 ** -float(e))
    f(); torch.cuda.synchronize()
    same = bool(torch.equal(sel, ref))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"kappa1=2^-{e}: {ms:.2f} ms / {n} frames ({ms * 1e7 / n:.1f} ms per 1e7), identical to dmma: {same}",
          flush=True)
