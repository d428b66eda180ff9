"""Seconds per config-3 EM iteration (20k utterances, C=2048, F=60, R=400) for several E-step batch
sizes (_estep.E_STEP_BATCH): one setup, then per batch size 1 warm-up + 3 timed iterations.

    python tools/estep_batch_probe.py [2048 4096 ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1906_08556_b200 as pkg  # noqa: E402
from paper_1906_08556_b200 import _estep  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [2048, 3072, 4096]
dev = torch.device("cuda")
gen = bench.generator("augmented")
tr, ad, ac, store, model = bench.em_setup(pkg, gen, 20000, 0, dev, dict(iterations=10 ** 6, min_div=True,
                                                                      sigma_update=True, realign_interval=0))
tr.align(ad, ac)
for bs in sizes:
    _estep.E_STEP_BATCH = bs
    tr.iteration()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        aux = tr.iteration()
    e1.record()
    torch.cuda.synchronize()
    print(f"E_STEP_BATCH {bs}: {e0.elapsed_time(e1) / 3e3:.4f} s/iter  aux {aux:.10e}  "
          f"peak mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB", flush=True)
