"""Where the end-to-end (host frames) alignment time goes: H2D / D2H copy rates alone, the device-resident
alignment, and align_frames on pinned host frames for several pipeline piece sizes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
def t(f, reps=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
print(f"H2D 2.4 GB pinned: {t(lambda: x.copy_(host, non_blocking=True)):.1f} ms")
d = torch.empty(n * 5, dtype=torch.float64, device='cuda'); hp = torch.empty(n * 5, dtype=torch.float64, pin_memory=True)
print(f"D2H 0.4 GB pinned: {t(lambda: hp.copy_(d, non_blocking=True)):.1f} ms")
print(f"device align: {t(lambda: _device.align(x, dm.device_table(), fm.device_table(), 20, 0.025)):.1f} ms")
for ch in (1 << 18, 1 << 19, 1 << 20):
    _device.STREAM_CHUNK = ch
    print(f"align_frames host, chunk {ch}: {t(lambda: pkg.align_frames(dm, fm, host, top_k=20, prune=0.025)):.1f} ms", flush=True)
