"""e2e tail probe: align_frames on pinned host frames (config 2, 1e7 frames) with the returned numpy
arrays freshly allocated (default), pre-faulted, or backed by transparent huge pages (madvise)."""
import mmap, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_1906_08556_b200 as pkg
from paper_1906_08556_b200 import _device
print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      "| defrag:", open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip(), "| cpus:", os.cpu_count())
n = 10_000_000
w, mu, cov = bench.make_ubm(0)
x = bench.sample_frames(w, mu, cov, n, 5, torch.device("cuda"))
dm = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
fm = pkg.GmmFull(w, mu, cov)
host = torch.empty((n, 60), dtype=torch.float32, pin_memory=True)
host.copy_(x)
orig_empty = np.empty


def t(f, reps=3):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    return sorted(ts)[len(ts) // 2]


run = lambda: pkg.align_frames(dm, fm, host, top_k=20, prune=0.025)
print(f"device align: {t(lambda: _device.align(x, dm.device_table(), fm.device_table(), 20, 0.025)):.1f} ms")
print(f"host e2e default: {t(run):.1f} ms")
cache = {}


def prefaulted(shape, dtype=float, *a, **k):
    key = (shape if isinstance(shape, tuple) else (shape,), np.dtype(dtype).str)
    if key not in cache:
        arr = orig_empty(shape, dtype, *a, **k)
        arr.fill(0)
        cache[key] = arr
    return cache[key]


def huge(shape, dtype=float, *a, **k):
    nb = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if nb < (1 << 22):
        return orig_empty(shape, dtype, *a, **k)
    m = mmap.mmap(-1, nb + (1 << 21))
    m.madvise(mmap.MADV_HUGEPAGE)
    return np.frombuffer(m, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


for name, fn in (("prefaulted outputs", prefaulted), ("THP-advised outputs", huge)):
    _device.np.empty = fn
    try:
        print(f"host e2e {name}: {t(run):.1f} ms", flush=True)
    finally:
        _device.np.empty = orig_empty
