"""Ozaki GEMM kernel time with and without the epilogue arithmetic (diagnostics build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from build_diag import use_diag
use_diag()
import torch
from paper_1906_08556_b200 import _lib
from paper_1906_08556_b200._lib import dgemm_i8 as dgemm
dev = torch.device("cuda")
Ub, C, D = 1024, 2048, 400
P = D * (D + 1) // 2
r = lambda *s: torch.randn(*s, device=dev, dtype=torch.float64)
n, U, out = r(Ub, C), r(C, P), r(Ub, P)
M, A = r(Ub, P), r(C, P)
for dbg in ("0", "1"):
    os.environ["TVK_OZ_DEBUG"] = dbg
    for name, fn in (("L = N U", lambda: dgemm(n, U, out, Ub, P, C)),
                     ("A += N'M", lambda: dgemm(n, M, A, C, P, Ub, trans_a=True, beta=1.0))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        print(f"dbg {dbg} {name}: {e0.elapsed_time(e1):.2f} ms (split + gemm)", flush=True)
