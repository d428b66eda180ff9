"""Debug helper: run the top-K preselection alone on a small frame batch and compare with the oracle."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import tvkit_oracle as orc
from paper_1906_08556_b200 import _device, _lib
import paper_1906_08556_b200 as pkg
T = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
C = int(sys.argv[2]) if len(sys.argv) > 2 else 256
diag, full, x = orc.posterior_ubm(C, 60, 0.3, seed=5, n_frames=T)
dm = pkg.GmmDiag(*diag)
xd = _device.frames_to_device(x)
t0 = time.time()
sel, val = _device.select_topk(xd, dm.device_table(), 20, values=True)
torch.cuda.synchronize()
print("select ok", time.time() - t0, flush=True)
ll = orc.diag_loglik(*diag, x)
want = np.argsort(-ll, axis=1, kind="stable")[:, :20]
got = _lib.to_host(sel)
print("mismatched frames", int(np.sum(np.any(got != want, axis=1))), "of", T)
