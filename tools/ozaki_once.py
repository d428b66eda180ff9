"""One Ozaki GEMM at an E-step shape (for ncu): python tools/ozaki_once.py {L|A|b|B} [digits]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_08556_b200 import _lib
from paper_1906_08556_b200._lib import dgemm_i8 as dgemm
which = sys.argv[1] if len(sys.argv) > 1 else "L"
dev = torch.device("cuda")
Ub, C, F, D = 1024, 2048, 60, 400
P = D * (D + 1) // 2
r = lambda *s: torch.randn(*s, device=dev, dtype=torch.float64)
if which == "L":
    n, U, out = r(Ub, C), r(C, P), r(Ub, P); dgemm(n, U, out, Ub, P, C)
elif which == "A":
    n, M, out = r(Ub, C), r(Ub, P), r(C, P); dgemm(n, M, out, C, P, Ub, trans_a=True, beta=1.0)
elif which == "b":
    fm, W, out = r(Ub, C * F), r(C * F, D), r(Ub, D); dgemm(fm, W, out, Ub, D, C * F, beta=1.0)
else:
    fm, phi, out = r(Ub, C * F), r(Ub, D), r(C * F, D); dgemm(fm, phi, out, C * F, D, Ub, trans_a=True, beta=1.0)
torch.cuda.synchronize()
print("ok")
