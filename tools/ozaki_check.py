"""Int8 tensor-core FP64 emulation (Ozaki, csrc/ozaki.cu) vs the FP64 DMMA GEMM at the E-step shapes of
the config-3 EM iteration (C=2048, F=60, D=400, 1024-utterance batch): time and error.

python tools/ozaki_check.py [digits]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1906_08556_b200 import _lib
from paper_1906_08556_b200._lib import dgemm, dgemm_i8

digits = int(sys.argv[1]) if len(sys.argv) > 1 else 7
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
Ub, C, F, D = 1024, 2048, 60, 400
P = D * (D + 1) // 2
# occupancies: sparse non-negative rows summing to ~300 frames; features, model-like operands
n = torch.rand(Ub, C, device=dev, dtype=torch.float64, generator=g) ** 8 * 3.0
U = torch.randn(C, P, device=dev, dtype=torch.float64, generator=g) * (torch.rand(C, 1, device=dev, dtype=torch.float64, generator=g) + 0.1)
M = torch.randn(Ub, P, device=dev, dtype=torch.float64, generator=g) * 0.01
fm = torch.randn(Ub, C * F, device=dev, dtype=torch.float64, generator=g) * n.repeat_interleave(F, 1)
W = torch.randn(C * F, D, device=dev, dtype=torch.float64, generator=g) * 0.1
phi = torch.randn(Ub, D, device=dev, dtype=torch.float64, generator=g)
cases = [
    ("L = N U", lambda g, out: g(n, U, out, Ub, P, C), (Ub, P)),
    ("A += N'M", lambda g, out: g(n, M, out, C, P, Ub, trans_a=True, beta=1.0), (C, P)),
    ("b = F W", lambda g, out: g(fm, W, out, Ub, D, C * F, beta=1.0), (Ub, D)),
    ("B += F'phi", lambda g, out: g(fm, phi, out, C * F, D, Ub, trans_a=True, beta=1.0), (C * F, D)),
]
DMMA, I8 = "dmma", "i8"
eng = {DMMA: dgemm, I8: lambda *a, **k: dgemm_i8(*a, digits=digits, **k)}
for name, fn, shape in cases:
    res = {}
    for mode in (DMMA, I8):
        init = torch.randn(*shape, device=dev, dtype=torch.float64, generator=torch.Generator(device=dev).manual_seed(1))
        out = init.clone()
        fn(eng[mode], out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            o2 = init.clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(eng[mode], o2); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        assert torch.equal(o2, out), "not bit-reproducible"
        res[mode] = (out, min(ts))
    ref, t_ref = res[DMMA]
    got, t_oz = res[I8]
    err = (got - ref).abs()
    scale = ref.abs().max().item()
    rel = (err / ref.abs().clamp_min(1e-300)).max().item()
    flop = 2.0 * np.prod(shape) * {"L = N U": C, "A += N'M": Ub, "b = F W": C * F, "B += F'phi": Ub}[name]
    print(f"{name:11s} dmma {t_ref:7.2f} ms ({flop / t_ref / 1e9:5.1f} TF)  ozaki{digits} {t_oz:7.2f} ms "
          f"({flop / t_oz / 1e9:6.1f} TF-equiv)  max|err|/max|C| {err.max().item() / scale:.2e}  "
          f"median rel {torch.median(err / ref.abs().clamp_min(1e-300)).item():.2e}", flush=True)
