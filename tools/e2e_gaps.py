"""Where the end-to-end frame-posterior time goes: align_frames on pinned host frames (config 2,
1e7 frames) under the torch profiler (CUPTI); prints the wall time, the busy time of the compute
kernels, the idle gaps between consecutive compute kernels (largest first, with the kernels either
side), and the copy engine busy time.

    python tools/e2e_gaps.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1906_08556_b200 as pkg  # noqa: E402

n = 10_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
dm = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
fm = pkg.GmmFull(w, mu, cov)
host = torch.empty((n, 60), dtype=torch.float32, pin_memory=True)
host.copy_(x)
run = lambda: pkg.align_frames(dm, fm, host, top_k=20, prune=0.025)
for _ in range(2):
    run()
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    run()
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
print("wall ms (3 runs):", [round(v, 1) for v in ts])
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    run()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = sorted([e for e in evs if "Memcpy" not in e.name and "Memset" not in e.name], key=lambda e: e.time_range.start)
cps = [e for e in evs if "Memcpy" in e.name]
t_lo = min(e.time_range.start for e in evs)
t_hi = max(e.time_range.end for e in evs)
print(f"profiled wall {wall:.1f} ms; device span {(t_hi - t_lo) / 1e3:.1f} ms")


def union(es):
    iv = sorted((e.time_range.start, e.time_range.end) for e in es)
    tot, cs, ce = 0, None, None
    for s, e in iv:
        if cs is None or s > ce:
            if cs is not None:
                tot += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if cs is not None:
        tot += ce - cs
    return tot / 1e3


print(f"kernel busy (union) {union(kern):.1f} ms, sum {sum(e.time_range.end - e.time_range.start for e in kern) / 1e3:.1f} ms")
for kind in ("HtoD", "DtoH"):
    sel = [e for e in cps if kind in e.name]
    print(f"{kind}: {len(sel)} copies, busy {union(sel):.1f} ms, first start {(min(e.time_range.start for e in sel) - t_lo) / 1e3:.2f} ms, last end {(max(e.time_range.end for e in sel) - t_lo) / 1e3:.2f} ms")
print(f"first kernel starts at {(kern[0].time_range.start - t_lo) / 1e3:.2f} ms, last kernel ends at {(kern[-1].time_range.end - t_lo) / 1e3:.2f} ms")
gaps = []
end = kern[0].time_range.end
prev = kern[0]
for e in kern[1:]:
    if e.time_range.start > end:
        gaps.append(((e.time_range.start - end) / 1e3, prev.name[:40], e.name[:40], (end - t_lo) / 1e3))
    if e.time_range.end > end:
        end = e.time_range.end
        prev = e
gaps.sort(reverse=True)
print(f"idle gaps between kernels: {len(gaps)}, total {sum(g[0] for g in gaps):.2f} ms")
for g in gaps[:15]:
    print(f"  {g[0]:.3f} ms at {g[3]:.2f} ms after {g[1]} before {g[2]}")
tot = {}
for e in kern:
    k = e.name.split("(")[0][-40:]
    tot[k] = tot.get(k, 0) + (e.time_range.end - e.time_range.start) / 1e3
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {v:7.2f} ms {k}")
