"""Kernel-time breakdown of one augmented EM iteration (config-3 shape, 8192 utterances) with the torch
profiler (CUDA activity timestamps, kernels not serialized)."""
import os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1906_08556_b200 as pkg
from torch.profiler import profile, ProfilerActivity

n_utt = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
orig = bench.bench_em
holder = {}


class Hook:
    pass


# reuse bench_em's corpus/model construction, then profile one extra iteration
import types
src = open(bench.__file__).read()
args = argparse.Namespace(em_utts=n_utt, em_steps=1, em_warmup=1)
dev = torch.device("cuda")
import paper_1906_08556_b200.pipeline as P
orig_iter = P.DeviceTrainer.iteration
state = {"n": 0}


def prof_iter(self):
    state["n"] += 1
    if state["n"] != 2:
        return orig_iter(self)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = orig_iter(self)
        torch.cuda.synchronize()
    ev = [e for e in prof.key_averages() if e.device_type.name == "CUDA" or e.self_device_time_total > 0]
    tot = sum(e.self_device_time_total for e in ev)
    print(f"EM iteration ({n_utt} utts): kernel time {tot / 1e3:.1f} ms")
    for e in sorted(ev, key=lambda e: -e.self_device_time_total)[:14]:
        print(f"  {e.self_device_time_total / 1e3:8.1f} ms {e.count:5d}  {e.key[:100]}")
    return r


P.DeviceTrainer.iteration = prof_iter
res = bench.bench_em(args, pkg, dev, 0, 1, lambda: None, lambda v: v)
print("s/iter", res["value"])
