"""Repeat the tcgen05 preselection and report frames whose result differs between runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _device
from oracle import tvkit_oracle as orc
T = int(sys.argv[1]) if len(sys.argv) > 1 else 60000
C = int(sys.argv[2]) if len(sys.argv) > 2 else 256
(w, mu, var), _, x = orc.posterior_ubm(C, 40, 0.4, seed=T, n_frames=T)
dm = pkg.GmmDiag(w, mu, var)
xd = _device.frames_to_device(x)
tab = dm.device_table()
ll = orc.diag_loglik(w, mu, var, x.astype(np.float64))
ref = np.argsort(-ll, axis=1, kind="stable")[:, :20]
runs = []
for mode in ("tc_noexact",) * 6 + ("tc",) * 6:
    os.environ["TVK_SELECT"] = mode
    s, _ = _device.select_topk(xd, tab, 20)
    torch.cuda.synchronize()
    runs.append((mode, s.cpu().numpy()))
for mode in ("tc_noexact", "tc"):
    rs = [r for m, r in runs if m == mode]
    diff = set()
    for r in rs[1:]:
        diff |= set(np.flatnonzero((r != rs[0]).any(1)).tolist())
    print(mode, "frames differing between runs:", sorted(diff)[:20], "count", len(diff))
    for t in sorted(diff)[:5]:
        print("  t", t, "tile", t // 128, "row", t % 128, "flagged", [int(r[t, 0] == -1) for r in rs])
        for r in rs[:3]: print("   ", r[t][:20])
        print("  ref", ref[t])
    bad = np.flatnonzero((rs[0] != ref).any(1) & (rs[0][:, 0] >= 0))
    print(mode, "frames != oracle (unflagged):", bad[:10], len(bad))
s = runs[-1][1]
bad = np.flatnonzero((s != ref).any(1))
for t in bad[:4]:
    a, b = s[t], ref[t]
    print("t", t, "ours", a.tolist())
    print("   ref ", b.tolist())
    print("   ours ll", np.round(ll[t, a], 6).tolist())
    print("   ref  ll", np.round(ll[t, b], 6).tolist())
    print("   ours set == ref set:", set(a.tolist()) == set(b.tolist()), "21st ref:", np.argsort(-ll[t], kind='stable')[20], ll[t, np.argsort(-ll[t], kind='stable')[20]])
