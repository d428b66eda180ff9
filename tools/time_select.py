"""Time the top-K preselection alone for several K (K=1 ~ GEMM-only cost) on 2e6 config-2 frames."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
w, mu, cov = bench.make_ubm(0)
dev = torch.device("cuda")
x = bench.sample_frames(w, mu, cov, n, 5, dev)
dm = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
tab = dm.device_table()
for k in (1, 4, 20, 32):
    sel = _lib.empty((n, k), torch.int32)
    f = lambda: _lib.call("tvk_select_topk", _lib.ptr(x), 0, n, 60, _lib.ptr(tab.table), 2048, k, _lib.ptr(sel), None, _lib.stream())
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f(); f(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    print(f"K={k:2d}: {ms:8.2f} ms for {n} frames -> {n/ms/1e3:.2f} M frames/s, {bench.FLOP_DIAG_PER_FRAME*n/ms/1e9:.2f} TFLOP/s")
