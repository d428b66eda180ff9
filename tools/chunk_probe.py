"""align_host (config 2, 1e7 pinned host frames) for several piece / ramp sizes."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _device
n = 10_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
dm = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
fm = pkg.GmmFull(w, mu, cov)
host = torch.empty((n, 60), dtype=torch.float32, pin_memory=True)
host.copy_(x)
dt, ft = dm.device_table(), fm.device_table()
for ramp in (1 << 17, 1 << 16):
    _device.RAMP_PIECE = ramp
    for c in (1 << 18, 1 << 19, 1 << 20, 1 << 21):
        _device.align_host(host, dt, ft, 20, 0.025, chunk=c); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); _device.align_host(host, dt, ft, 20, 0.025, chunk=c); torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"ramp 2^{ramp.bit_length()-1} chunk 2^{c.bit_length()-1}: median {sorted(ts)[2]:.1f} ms  min {min(ts):.1f}", flush=True)
