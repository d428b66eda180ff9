"""Small runs of the round-2 kernels for compute-sanitizer: int8 FP64 emulation (inline split, pre-split
operand, split-K, digits 6-8), the DMMA BW second-order sum, an E-step batch on the int8 engine, the
sweep-based update_T, and the preselection / alignment path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib, _estep, _device, tvm
from oracle import tvkit_oracle as orc
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
for M, N, K, d in [(200, 130, 77, 7), (129, 70, 3000, 8), (64, 64, 32, 6)]:
    A = torch.randn(M, K, device=dev, dtype=torch.float64, generator=g)
    B = torch.randn(K, N, device=dev, dtype=torch.float64, generator=g)
    C = torch.zeros(M, N, device=dev, dtype=torch.float64)
    _lib.dgemm_i8(A, B, C, M, N, K, beta=1.0, digits=d)
    _lib.dgemm_i8(A, None, C, M, N, K, digits=d, b_split=_lib.i8_split_b(B, K, N, digits=d))
    _lib.dgemm_i8(A.t().contiguous(), B, C, M, N, K, trans_a=True, digits=d)
rng = np.random.default_rng(0)
Cc, F, D, U = 96, 24, 40, 60
model = tvm.TvModel(formulation="augmented", T=rng.standard_normal((Cc, F, D)) * 0.3,
                    Sigma=np.tile(np.eye(F), (Cc, 1, 1)), ubm_weights=np.full(Cc, 1.0 / Cc),
                    ubm_means=rng.standard_normal((Cc, F)), prior_offset=10.0)
_estep.I8_MIN_WORK = 0
dm = _estep.DeviceModel(model)
ws = _estep.Workspace(dm)
acc = _estep.DeviceAcc(Cc, F, D)
n = rng.gamma(0.3, 2.0, (U, Cc))
_estep.accumulate_batch(dm, ws, acc, _lib.to_dev(n), _lib.to_dev(rng.standard_normal((U, Cc * F)) * n.repeat(F, 1)))
_estep.update_T_device(dm.T, acc.Apk, acc.B, acc.N, Cc, F, D)
for C2, F2, T2 in [(300, 40, 700), (64, 20, 260)]:
    (w, mu, var), full, x = orc.posterior_ubm(C2, F2, 0.5, seed=1, n_frames=T2)
    a = pkg.align_frames(pkg.GmmDiag(w, mu, var), pkg.GmmFull(*full), x, top_k=20, prune=0.025)
    utt = _lib.to_dev(np.array([0, 100, T2], np.int64), torch.int64)
    ssum = _lib.zeros((C2, F2, F2))
    _device.bw_stats(_device.frames_to_device(x), utt, _lib.to_dev(a.offsets, torch.int64),
                     _lib.to_dev(a.components.astype(np.int32), torch.int32), _lib.to_dev(a.weights, torch.float32),
                     C2, ssum_acc=ssum)
torch.cuda.synchronize()
print("ok")
