"""Time the model-table builds that every align_frames call pays (config 2 UBM)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
w, mu, cov = bench.make_ubm(0)
dm = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
fm = pkg.GmmFull(w, mu, cov)
for name, f in [("diag", dm.device_table), ("full", fm.device_table)]:
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): f()
    torch.cuda.synchronize()
    print(f"{name} device_table: {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms", flush=True)
