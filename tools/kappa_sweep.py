"""Preselection cost vs the 3xFP16 error margin kappa (config-2 frames; needs a -DTVK_SELECT_DIAG build
with a TVK_SELECT_KAPPA read added): select time, frames
handed to the exact kernel, and identity with the FP64 DMMA selection."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
tab = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))).device_table()
sel = _lib.empty((n, 20), torch.int32)
f = lambda: _lib.call("tvk_select_topk", _lib.ptr(x), 0, n, 60, _lib.ptr(tab.table), 2048, 20, _lib.ptr(sel), None, _lib.stream())
os.environ["TVK_SELECT"] = "dmma"
f(); torch.cuda.synchronize(); ref = sel.clone()
for kap in ["0.0000152587890625", "0.00006103515625", "0.0001220703125", "0.000244140625"]:
    os.environ["TVK_SELECT_KAPPA"] = kap
    os.environ["TVK_SELECT"] = "tc_noexact"
    f(); torch.cuda.synchronize()
    flagged = int((sel[:, 0] == -1).sum().item())
    os.environ["TVK_SELECT"] = "tc"
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    same = bool(torch.equal(sel, ref))
    print(f"kappa=2^{np.log2(float(kap)):.0f}: {ms:.2f} ms / {n} frames ({ms * 1e7 / n:.1f} ms per 1e7), "
          f"flagged {flagged} ({100 * flagged / n:.3f}%), identical to dmma: {same}", flush=True)
