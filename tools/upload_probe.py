import time, numpy as np, torch, concurrent.futures as cf, os
cov = np.random.default_rng(0).standard_normal((2048, 60, 60))
t = torch.from_numpy(cov)
pin = torch.empty(cov.nbytes, dtype=torch.uint8, pin_memory=True).view(torch.float64).view(cov.shape)
out = torch.empty(cov.shape, dtype=torch.float64, device="cuda")
pool = cf.ThreadPoolExecutor(8)
print("cpus", os.cpu_count())
def tm(name, f, reps=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:40s} {min(ts):7.2f} ms (median {sorted(ts)[reps//2]:.2f})")
d, s = pin.numpy().reshape(-1), cov.reshape(-1)
n = d.shape[0]
def mc(nt):
    step = -(-n // nt)
    list(pool.map(lambda lo: np.copyto(d[lo:lo + step], s[lo:lo + step]), range(0, n, step)))
tm("memcpy 1 thread", lambda: np.copyto(d, s))
tm("memcpy 8 threads", lambda: mc(8))
tm("memcpy 16 chunks/8 threads", lambda: mc(16))
tm("H2D from pinned", lambda: out.copy_(pin, non_blocking=True))
tm("pageable .to(cuda)", lambda: t.to("cuda"))
tm("pageable copy_ into out", lambda: out.copy_(t))
tm("memcpy8 + H2D", lambda: (mc(8), out.copy_(pin, non_blocking=True)))

# page-lock the numpy buffer in place (no staging copy), upload, unlock
from cuda.bindings import runtime as rt  # noqa: E402


def registered():
    ptr = cov.ctypes.data
    err, = rt.cudaHostRegister(ptr, cov.nbytes, 0)
    assert err == rt.cudaError_t.cudaSuccess, err
    out.copy_(torch.from_numpy(cov), non_blocking=True)
    torch.cuda.synchronize()
    rt.cudaHostUnregister(ptr)


try:
    tm("cudaHostRegister + H2D + unregister", registered)
except Exception as exc:  # cuda-python missing or registration refused
    print("cudaHostRegister probe failed:", exc)
