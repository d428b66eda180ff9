"""Per-phase timeline (clock64) of the tcgen05 preselection epilogue, CTA 0 (diagnostics build, TVK_SELECT_DEBUG=6;
7: scores not consumed, 12: no pass-1 append, 13: next A not built in pass 0, 14: no pass-0 bound)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from build_diag import use_diag
use_diag()
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib, _device
n = 2_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
tab = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))).device_table()
for dbg in (sys.argv[1:] or ["6", "7"]):
    os.environ["TVK_SELECT_DEBUG"] = dbg
    os.environ["TVK_SELECT"] = "tc_noexact"
    sel, val = _device.select_topk(x, tab, 20, values=True)
    sel, val = _device.select_topk(x, tab, 20, values=True)
    torch.cuda.synchronize()
    v = val.view(-1)[:64 * 8].cpu().numpy().reshape(64, 8)
    names = ["start", "pass0 done", "thr ready", "next A built", "pass1 done", "-", "merge done", "tile end"]
    d = np.diff(v[2:12], axis=1)
    print("debug", dbg, "mean cycles per phase (tiles 2-11):")
    for i in range(7):
        print(f"  {names[i]:>12s} -> {names[i + 1]:<12s}: {d[:, i].mean():9.0f}")
    print("  tile total:", np.diff(v[2:12, 0]).mean())
