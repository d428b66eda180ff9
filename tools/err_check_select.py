import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _device
from oracle import tvkit_oracle as orc
for (C, F, sd, T) in [(256, 40, 0.4, 6000), (256, 60, 0.4, 6000), (2048, 40, 0.4, 6000), (256, 40, 0.3, 6000), (256, 48, 0.4, 6000), (320, 40, 0.4, 6000)]:
    (w, mu, var), _, x = orc.posterior_ubm(C, F, sd, seed=T, n_frames=T)
    dm = pkg.GmmDiag(w, mu, var)
    xd = _device.frames_to_device(x)
    os.environ["TVK_SELECT"] = "tc_noexact"; os.environ["TVK_SELECT_DEBUG"] = "1"
    sel, val = _device.select_topk(xd, dm.device_table(), 20, values=True)
    torch.cuda.synchronize()
    os.environ.pop("TVK_SELECT_DEBUG")
    sel = sel.cpu().numpy(); d = np.abs(val.cpu().numpy())
    ok = sel[:, 0] >= 0
    a = 0.5 / var; b = np.abs(mu / var)
    c = np.abs(np.log(w) - 0.5 * (F * np.log(2 * np.pi) + np.log(var).sum(1)) - 0.5 * (mu * mu / var).sum(1))
    xd64 = x.astype(np.float64)
    St = (xd64 ** 2) @ a.max(0) + np.abs(xd64) @ b.max(0) + c.max()
    r = (d / St[:, None])[ok]
    worst = np.argsort(-r.max(1))[:5]
    print(C, F, "max err/S", r.max(), "log2", np.log2(r.max()), "frames over 2^-16:", (r.max(1) > 2**-16).sum(), "of", ok.sum())
    idx = np.flatnonzero(ok)[worst]
    print("   worst frames", idx, "tile", idx // 128, "row", idx % 128, r.max(1)[worst])
