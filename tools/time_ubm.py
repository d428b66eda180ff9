"""Time UBM EM training (train_gmm_diag + train_gmm_full) on the device against the numpy oracle
(the reference's own algorithm) on the same synthetic frames.  Usage: python tools/time_ubm.py"""

import json
import os
import sys
import time
import warnings

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1906_08556_b200 as pkg  # noqa: E402
from oracle import tvkit_oracle as orc  # noqa: E402


def frames(T, F, k=64, seed=0):
    rng = np.random.default_rng(seed)
    centres = rng.normal(0.0, 3.0, (k, F))
    lab = rng.integers(0, k, T)
    return centres[lab] + rng.normal(0.0, 1.0, (T, F)) * rng.uniform(0.5, 2.0, F)


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def main():
    warnings.simplefilter("ignore", RuntimeWarning)
    rows = []
    for T, F, C, di, fi, cpu in [(200_000, 20, 256, 3, 2, True), (1_000_000, 39, 512, 2, 1, False),
                                 (1_000_000, 60, 2048, 1, 1, False)]:
        x = frames(T, F)
        pkg.train_gmm_diag(x[:20000], 8, n_iters=1)  # warm-up (library load, kernels)
        d, td_seed = timed(lambda: pkg.train_gmm_diag(x, C, n_iters=0, seed=1))
        d, td = timed(lambda: pkg.train_gmm_diag(x, C, n_iters=di, seed=1))
        f, tf = timed(lambda: pkg.train_gmm_full(x, d, n_iters=fi))
        row = {"T": T, "F": F, "C": C, "diag_iters": di, "full_iters": fi, "gpu_seed_s": td_seed,
               "gpu_diag_iter_s": (td - td_seed) / di, "gpu_full_iter_s": tf / fi}
        if cpu:
            t0 = time.perf_counter()
            od = orc.train_gmm_diag(x, C, n_iters=0, seed=1)
            t1 = time.perf_counter()
            od = orc.train_gmm_diag(x, C, n_iters=di, seed=1)
            t2 = time.perf_counter()
            of = orc.train_gmm_full(x, od.weights, od.means, od.variances, n_iters=fi)
            t3 = time.perf_counter()
            row.update(cpu_seed_s=t1 - t0, cpu_diag_iter_s=(t2 - t1 - (t1 - t0)) / di, cpu_full_iter_s=(t3 - t2) / fi,
                       max_rel_cov_diff=float(np.max(np.abs(f.covariances - of.covariances)) /
                                              np.max(np.abs(of.covariances))))
        print(json.dumps(row), flush=True)
        rows.append(row)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/time_ubm.json", "w") as fh:
        json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
