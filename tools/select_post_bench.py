"""Preselection stage on config-2 frames: per-kernel CUPTI times (select_tc / select_post /
select_exact) and the tensor-core selection checked index-for-index against the FP64 DMMA kernel.

    python tools/select_post_bench.py [frames]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1906_08556_b200 as pkg  # noqa: E402
from paper_1906_08556_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 1000, torch.device("cuda"))
tab = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))).device_table()


def run(mode, sel):
    os.environ["TVK_SELECT"] = mode
    _lib.call("tvk_select_topk", _lib.ptr(x), 0, n, 60, _lib.ptr(tab.table), 2048, 20, _lib.ptr(sel), None,
              _lib.stream())


sel = _lib.empty((n, 20), torch.int32)
for _ in range(2):
    run("tc", sel)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        run("tc", sel)
    torch.cuda.synchronize()
tot = {}
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        k = ev.name.split("(")[0].split("<")[0].split("::")[-1]
        tot[k] = tot.get(k, 0.0) + ev.device_time / 3e3
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:8.3f} ms  {k}")
print(f"stage total {sum(tot.values()):.3f} ms per {n} frames")
ref = _lib.empty((n, 20), torch.int32)
run("dmma", ref)
os.environ.pop("TVK_SELECT")
torch.cuda.synchronize()
print("mismatched frames vs FP64 DMMA:", int((sel != ref).any(dim=1).sum().item()))
