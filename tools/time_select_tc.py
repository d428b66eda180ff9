"""Quick timing of the tcgen05 preselection on 2e6 config-2 frames (full, pipeline-only, copies-only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib, _device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
tab = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))).device_table()
sel = _lib.empty((n, 20), torch.int32)
def t(mode, dbg=None, reps=3):
    os.environ["TVK_SELECT"] = mode
    if dbg: os.environ["TVK_SELECT_DEBUG"] = dbg
    f = lambda: _lib.call("tvk_select_topk", _lib.ptr(x), 0, n, 60, _lib.ptr(tab.table), 2048, 20, _lib.ptr(sel), None, _lib.stream())
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    os.environ.pop("TVK_SELECT_DEBUG", None)
    return e0.elapsed_time(e1) / reps
print(f"full {t('tc'):.2f} ms, no-exact {t('tc_noexact'):.2f}, pipeline {t('tc_noexact', '2'):.2f}, copies {t('tc_noexact', '3'):.2f}")
t("tc", reps=1); a = sel.clone(); t("dmma", reps=1)
print("identical to dmma:", bool(torch.equal(a, sel)))
