"""One config-2 alignment (select + grouped whitening + finalize) on n frames resident in HBM, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
dm = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
fm = pkg.GmmFull(w, mu, cov)
res = _device.align(x, dm.device_table(), fm.device_table(), 20, 0.025)
torch.cuda.synchronize()
print("entries", res.n_entries)
