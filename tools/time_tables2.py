import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib, _device
w, mu, cov = bench.make_ubm(0)
fm = pkg.GmmFull(w, mu, cov)
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    d = _lib.to_dev(cov); torch.cuda.synchronize(); t1 = time.perf_counter()
    tab = _device.FullTable(w, mu, cov); torch.cuda.synchronize(); t2 = time.perf_counter()
    bad = tab.bad_components(); t3 = time.perf_counter()
    print(f"to_dev(cov) {1e3*(t1-t0):.2f} ms, FullTable {1e3*(t2-t1):.2f} ms, status check {1e3*(t3-t2):.2f} ms", flush=True)
