"""Small align_frames + select + sparse path run for compute-sanitizer (memcheck / racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1906_08556_b200 as pkg
from oracle import tvkit_oracle as orc
for C, F, T in [(300, 40, 700), (64, 20, 260)]:
    (w, mu, var), full, x = orc.posterior_ubm(C, F, 0.5, seed=1, n_frames=T)
    dm, fm = pkg.GmmDiag(w, mu, var), pkg.GmmFull(*full)
    for sparse in ("0", "1"):
        os.environ["TVK_ALIGN_SPARSE"] = sparse
        a = pkg.align_frames(dm, fm, x, top_k=20, prune=0.025)
    torch.cuda.synchronize()
print("ok")
