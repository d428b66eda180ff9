"""Time the tcgen05 preselection for several B-ring geometries (TVK_SEL_PIPE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib
n = 2_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
tab = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))).device_table()
sel = _lib.empty((n, 20), torch.int32)
def t(reps=5):
    f = lambda: _lib.call("tvk_select_topk", _lib.ptr(x), 0, n, 60, _lib.ptr(tab.table), 2048, 20, _lib.ptr(sel), None, _lib.stream())
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for cfg in sys.argv[1:]:
    os.environ["TVK_SEL_PIPE"] = cfg
    full = t()
    os.environ["TVK_SELECT_DEBUG"] = "2"; pipe = t(); os.environ.pop("TVK_SELECT_DEBUG")
    print(f"{cfg:>22s}: full {full:6.2f} ms  pipeline-only {pipe:6.2f} ms", flush=True)
