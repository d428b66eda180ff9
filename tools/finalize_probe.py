"""Per-kernel times of the finalize / scan / compact stage inside tvk_align_frames (config 2, 1e7 frames), and the step time."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import numpy as np, bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib
n = 10_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 1000, torch.device("cuda"))
dm = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))); fm = pkg.GmmFull(w, mu, cov)
dt, ft = dm.device_table(), fm.device_table()
off = _lib.empty((n + 1,), torch.int64); comps = _lib.empty((n * 20,), torch.int32); wts = _lib.empty((n * 20,), torch.float32)
wsb = int(_lib.load().tvk_align_workspace_bytes(n, 20, 2048)); ws = _lib.empty((wsb,), torch.uint8)
step = lambda: _lib.call("tvk_align_frames", _lib.ptr(x), 0, n, 60, _lib.ptr(dt.table), None, _lib.ptr(ft.prec), 2048, 20, 0.025, 0, _lib.ptr(ws), wsb, _lib.ptr(off), _lib.ptr(comps), _lib.ptr(wts), None, None, _lib.stream())
for _ in range(3): step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3): step()
    torch.cuda.synchronize()
tot = {}
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name.split("(")[0].split("<")[0].split("::")[-1]
        tot[k] = tot.get(k, 0.0) + ev.device_time / 3e3
for k in ("finalize_fixed_kernel", "compact_kernel", "scan_write_offsets", "scan_block_sums", "scan_block_prefix"):
    print(f"{tot.get(k, 0):.3f} ms {k}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): step()
e1.record(); torch.cuda.synchronize(); print(f"step {e0.elapsed_time(e1)/5:.2f} ms")
