"""Fraction of config-2 frames the tcgen05 preselection hands to select_exact_kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _device
n = 2_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
tab = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2))).device_table()
os.environ["TVK_SELECT"] = "tc_noexact"
sel, _ = _device.select_topk(x, tab, 20)
flag = (sel[:, 0] == -1).sum().item()
print(f"flagged {flag} of {n} frames ({100 * flag / n:.3f}%)")
