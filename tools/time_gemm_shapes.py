"""tvk_dgemm TFLOP/s at the EM shapes (L = N U, A += N^T M) and at 8192^3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1906_08556_b200 import _lib
dev = torch.device("cuda")
def run(m, n, k, ta=False, reps=3):
    a = torch.randn((k, m) if ta else (m, k), dtype=torch.float64, device=dev)
    b = torch.randn((k, n), dtype=torch.float64, device=dev)
    c = torch.zeros((m, n), dtype=torch.float64, device=dev)
    f = lambda: _lib.dgemm(a, b, c, m, n, k, trans_a=ta, beta=1.0)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"M={m} N={n} K={k} ta={ta}: {ms:.2f} ms, {2*m*n*k/ms/1e9:.1f} TF", flush=True)
run(8192, 8192, 8192)
run(1024, 80200, 2048)
run(2048, 80200, 1024, ta=True)
run(1024, 80256, 2048)
