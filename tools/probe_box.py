"""One-shot probe of a GPU box: FP64 cuBLAS peak (torch.matmul float64), our DMMA GEMM, host info."""
import json
import os
import time

import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1906_08556_b200 import _lib

out = {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
try:
    with open("/proc/cpuinfo") as fh:
        out["cpu_model"] = next(l.split(":", 1)[1].strip() for l in fh if l.startswith("model name"))
except Exception:
    pass
dev = torch.device("cuda")
out["gpu"] = torch.cuda.get_device_name(0)
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = torch.empty(n, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); torch.matmul(a, b, out=c); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    out[f"cublas_dgemm_{n}_tflops"] = 2 * n**3 / best / 1e9
    for _ in range(2):
        _lib.dgemm(a, b, c, n, n, n)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); _lib.dgemm(a, b, c, n, n, n); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    out[f"tvk_dgemm_{n}_tflops"] = 2 * n**3 / best / 1e9
    ref = torch.matmul(a, b)
    _lib.dgemm(a, b, c, n, n, n)
    out[f"tvk_dgemm_{n}_maxrel"] = float(((c - ref).abs().max() / ref.abs().max()).item())
print(json.dumps(out, indent=1))
