"""One train_gmm_full iteration (T=262144, F=60, C=2048) for an ncu launch list."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1906_08556_b200 as pkg  # noqa: E402

T, F, C = int(os.environ.get("T", 262144)), 60, 2048
rng = np.random.default_rng(0)
x = rng.normal(0.0, 1.0, (T, F)) + rng.normal(0.0, 3.0, (64, F))[rng.integers(0, 64, T)]
d = pkg.GmmDiag(np.full(C, 1.0 / C), x[rng.choice(T, C, replace=False)], np.ones((C, F)))
for it in range(int(os.environ.get("REPS", 1))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pkg.train_gmm_full(x, d, n_iters=1)
    torch.cuda.synchronize()
    print("full iter", time.perf_counter() - t0, flush=True)
