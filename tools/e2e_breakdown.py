"""Where the end-to-end align_frames time goes (pinned host frames, config 2)."""
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
del x
torch.cuda.empty_cache()
def tm(name, f, reps=2):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): r = f()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / reps * 1e3:.1f} ms", flush=True)
    return r
tm("diag device_table", lambda: dm.device_table())
tm("full device_table", lambda: fm.device_table())
dt, ft = dm.device_table(), fm.device_table()
tm("H2D 2.4 GB pinned", lambda: host.to("cuda", non_blocking=True))
for ch in (1 << 19, 3 << 18, 1 << 20):
    tm(f"align_host chunk {ch}", lambda: _device.align_host(host, dt, ft, 20, 0.025, chunk=ch))
tm("align_frames (public)", lambda: pkg.align_frames(dm, fm, host, top_k=20, prune=0.025))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable(); pkg.align_frames(dm, fm, host, top_k=20, prune=0.025); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
