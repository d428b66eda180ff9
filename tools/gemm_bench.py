"""Time the E-step DGEMMs of one 1024-utterance batch at the config-3 shape (C=2048, F=60, D=400).

python tools/gemm_bench.py [Ub]  -- ms and TFLOP/s per GEMM (CUDA events, median of 5), vs torch (cuBLAS)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_08556_b200 import _lib  # noqa: E402

Ub = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
C, F, D = 2048, 60, 400
P = D * (D + 1) // 2
dev = _lib.device()
r = lambda *s: torch.rand(s, device=dev, dtype=torch.float64)  # noqa: E731
N, U, Mpk = r(Ub, C), r(C, P), r(Ub, P)
Fm, W, phi = r(Ub, C * F), r(C * F, D), r(Ub, D)
Lpk, Apk, b, B = torch.empty(Ub, P, device=dev, dtype=torch.float64), r(C, P), r(Ub, D), r(C * F, D)
splits = max(1, min(16, C * F // 2048)) if Ub * D < 148 * 128 * 128 else 1
work = torch.empty(splits * Ub * D, device=dev, dtype=torch.float64) if splits > 1 else None


def timeit(fn, reps=5):
    ts = []
    for i in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


cases = [
    ("L = N U", 2.0 * Ub * C * P, lambda: _lib.dgemm(N, U, Lpk, Ub, P, C), lambda: torch.mm(N, U)),
    ("A += N' M", 2.0 * Ub * C * P, lambda: _lib.dgemm(N, Mpk, Apk, C, P, Ub, trans_a=True, beta=1.0),
     lambda: torch.mm(N.t(), Mpk)),
    (f"b = F W (split {splits})", 2.0 * Ub * C * F * D,
     lambda: _lib.dgemm(Fm, W, b, Ub, D, C * F, beta=1.0, splits=splits, work=work), lambda: torch.mm(Fm, W)),
    ("B += F' phi", 2.0 * Ub * C * F * D, lambda: _lib.dgemm(Fm, phi, B, C * F, D, Ub, trans_a=True, beta=1.0),
     lambda: torch.mm(Fm.t(), phi)),
]
tot = 0.0
for name, flop, ours, ref in cases:
    t = timeit(ours)
    tr = timeit(ref)
    tot += t
    print(f"{name:24s} ours {t:7.3f} ms {flop / t / 1e9:6.2f} TF ({flop / t / 1e9 / 37.15:.2f})   cuBLAS {tr:7.3f} ms "
          f"{flop / tr / 1e9:6.2f} TF")
print(f"total {tot:.3f} ms per {Ub}-utterance batch")
