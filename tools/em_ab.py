import os, sys, argparse
sys.path.insert(0, "/root/repo")
import torch, bench, paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _lib
args = argparse.Namespace(em_utts=20000, em_steps=3, em_warmup=1)
for stage in (True, False, True):
    _lib._STAGE_MIN = (8 << 20) if stage else (1 << 62)
    r = bench.bench_em(args, pkg, torch.device("cuda"), 0, 1, torch.cuda.synchronize, lambda v: v)
    print("pinned staging" if stage else "pageable", r["value"], flush=True)
