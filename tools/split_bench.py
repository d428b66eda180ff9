"""Operand split (row_exp_kernel + split_tile_kernel, csrc/ozaki.cu) at the E-step shapes of one
2048-utterance batch of the config-3 EM iteration: per-kernel CUPTI times and effective HBM GB/s.

    python tools/split_bench.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_08556_b200 import _lib  # noqa: E402

U, C, F, D = 2048, 2048, 60, 400
P = D * (D + 1) // 2
# (name, rows, k, rs, ks, row tile, digits): fm for b = F W (rows = utterances, k contiguous),
# fm' for B += F' phi (rows = (c, f), contiguous), M for A += N' M (rows = packed entries, contiguous)
SHAPES = [("fm (b = F W)", U, C * F, C * F, 1, 128, 8),
          ("fm' (B += F' phi)", C * F, U, 1, C * F, 128, 8),
          ("M (A += N' M)", P, U, 1, P, 64, 7)]


def main():
    for name, R, K, rs, ks, RT, S in SHAPES:
        x = torch.randn(R * K, dtype=torch.float64, device="cuda")
        out = torch.empty(int(_lib.load().tvk_i8_operand_bytes(R, K, RT, S)), dtype=torch.uint8, device="cuda")
        run = lambda: _lib.call("tvk_i8_split", _lib.ptr(x), R, K, rs, ks, RT, S, _lib.ptr(out), _lib.stream())
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            for _ in range(5):
                run()
            torch.cuda.synchronize()
        tot = {}
        for ev in prof.events():
            if ev.device_type == torch.autograd.DeviceType.CUDA:
                tot[ev.name] = tot.get(ev.name, 0.0) + ev.device_time / 5
        rd = R * K * 8
        for k, us in sorted(tot.items(), key=lambda kv: -kv[1]):
            nm = k.split("(")[0].split("<")[0][-28:]
            gbs = (rd + (out.numel() if "split_tile" in k else 0)) / (us * 1e-6) / 1e9
            print(f"{name:20s} {nm:28s} {us / 1e3:8.3f} ms  {gbs:7.0f} GB/s")
        del x, out


if __name__ == "__main__":
    main()
