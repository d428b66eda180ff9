"""One config-3-shaped E-step batch (C=2048, F=60, R=400, --utts utterances): workspace, BW stats,
L / b GEMMs, posterior_kernel, A / B GEMMs.  Driver for ncu captures of the EM kernels:

    ncu --set full --clock-control none --import-source on -k regex:"posterior_kernel|gemm_kernel" \
        -c 8 -o gpurun_out/em python tools/profile_em.py --utts 1024
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _estep, pipeline as P

ap = argparse.ArgumentParser()
ap.add_argument("--utts", type=int, default=1024)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
dev = torch.device("cuda")
gen = bench.generator("augmented")
tr, align_diag, align_cov, store, model = bench.em_setup(
    pkg, gen, a.utts, 0, dev, dict(iterations=10 ** 6, min_div=True, sigma_update=True, realign_interval=0))
tr.align(align_diag, align_cov)
dm = tr.dm
ws = _estep.Workspace(dm)
acc = _estep.DeviceAcc(dm.C, dm.F, dm.D)
n, f = P._stats_batch(tr.corpus, tr.alignment, 0, a.utts, dm.C, None, acc.Ssum)
torch.cuda.synchronize()
for _ in range(a.reps):
    _estep.accumulate_batch(dm, ws, acc, n, f)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
phi, Mpk, logdet, bphi, status, _ = _estep.posterior_batch(dm, ws, n, f)
e1.record()
torch.cuda.synchronize()
print(f"posterior_batch ({a.utts} utts, L/b GEMMs + posterior_kernel): {e0.elapsed_time(e1):.2f} ms")
