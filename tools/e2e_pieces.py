"""Per-piece device timing inside align_host: compute busy time vs wall (config 2, 1e7 frames)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _device, _lib
n = 10_000_000
w, mu, cov = bench.make_ubm(0)
dm = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
fm = pkg.GmmFull(w, mu, cov)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
host = torch.empty((n, 60), dtype=torch.float32, pin_memory=True)
host.copy_(x)
dt, ft = dm.device_table(), fm.device_table()
# device-only: same pieces, frames already resident
for ch in (1 << 19, 1 << 21, n):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for lo in range(0, n, ch):
        _device.align(x[lo:lo + ch], dt, ft, 20, 0.025, sync_count=False)
    torch.cuda.synchronize(); print(f"device-resident pieces of {ch}: {(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
orig = _device.align
evs = []
def timed_align(*a, **k):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); r = orig(*a, **k); e1.record(); evs.append((e0, e1)); return r
_device.align = timed_align
for rep in range(2):
    evs.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _device.align_host(host, dt, ft, 20, 0.025)
    torch.cuda.synchronize(); wall = (time.perf_counter() - t0) * 1e3
    busy = sum(a.elapsed_time(b) for a, b in evs)
    span = evs[0][0].elapsed_time(evs[-1][1])
    gaps = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(len(evs) - 1)]
    print(f"align_host wall {wall:.1f} ms, compute busy {busy:.1f} ms over span {span:.1f} ms, pieces {len(evs)}, "
          f"max gap {max(gaps):.2f} ms, first start after {0:.1f}", flush=True)
    print("  per-piece ms:", [round(a.elapsed_time(b), 2) for a, b in evs])
