"""Benchmark of the GPU i-vector hot path (BASELINE.json metric).

Headline (``value``): UBM frame posteriors (BASELINE config 2): 2048-component full-covariance
UBM, 60-dim frames, 1e7 synthetic frames per GPU per step, top-20 preselection + prune 0.025,
frames resident in HBM (2.4 GB per GPU, larger than L2).  ``e2e``: the same through the public
``align_frames`` API from pinned host frames to a host SparseAlignment.  A second object
(``em_iteration``) reports seconds per EM iteration of the Kaldi augmented-bias extractor at
2048 x 60, R=400 (BASELINE config 3 shape) on ``--em-utts`` synthetic utterances per GPU.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--no-em]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU)

``--impl reference`` times the reference algorithm on the host cores (the CPU oracle restating
tvkit.gmm.align_frames, since the reference tree does not exist on the GPU box) on a bounded
frame sample per step.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = json.load(open(os.path.join(REPO, "BASELINE.json")))["metric"]
C, F, K_TOP, PRUNE = 2048, 60, 20, 0.025
FRAMES_PER_GPU = 10_000_000
Q = 1 + F + F * (F + 1) // 2
FLOP_FULL_PER_FRAME = 2 * C * Q            # dominant kernel (quadratic-feature GEMM)
FLOP_DIAG_PER_FRAME = 2 * C * (2 * F + 1)   # preselection GEMM [x^2, x, 1] . Wdiag
FLOP_PER_FRAME = FLOP_DIAG_PER_FRAME + FLOP_FULL_PER_FRAME   # 8,241,152 (dense)
FLOP_GROUPED_PER_FRAME = 2 * K_TOP * Q                       # quadratic-feature count for the K selected
KP_TC = (2 * F + 1 + 15) // 16 * 16                          # [x^2, x, 1] padded to the f16 MMA K step
F16_EXEC_PER_FRAME = 4 * 2 * KP_TC * C                       # 1xFP16 bound pass + 3xFP16 collection pass
# whiten_ll: per 128-pair tile, 8 warps x sum over k4-steps kk < ceil(F/4) of 2 * (8 - kk // 2) DMMA.8x8x4
DMMA_EXEC_PER_FRAME = K_TOP * 8 * sum(2 * (8 - kk // 2) for kk in range((F + 3) // 4)) * 512 // 128
WINDOW_FRAMES = 131072                                       # grouped full-LL frame window (align_grouped.cu)


def f16_peak():
    """Dense f16/bf16 tensor peak (tcgen05 kind::f16): MEASURED_PEAKS.json's cuBLAS bf16 figure."""
    try:
        m = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
        return m["bf16_tflops"], "measured bf16 (MEASURED_PEAKS.json)"
    except Exception:
        return 1590.0, "fallback bf16 1.59 PF (B200_PROFILING.md)"
FP64_PEAK_FILE = os.path.join(REPO, "profiles", "r01_fp64_pipe_peak.txt")
I8_PEAK_FILE = os.path.join(REPO, "profiles", "r02_i8_peak.txt")


def i8_peak():
    """Measured tcgen05 kind::i8 issue rate (SS operands, N >= 128) on this pool's B200 (tools/i8_probe.cu)."""
    try:
        vals = [float(l.split()[-2]) for l in open(I8_PEAK_FILE) if l.startswith("i8 SS")]
        return max(vals), "measured tcgen05 kind::i8 SS issue rate (profiles/r02_i8_peak.txt)"
    except Exception:
        return 4500.0, "nominal B200 dense int8 4.5 POPS"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def fp64_peak():
    """Measured FP64 tensor-pipe (DMMA.8x8x4) issue ceiling on this pool's B200 (tools/fp64_peak.cu)."""
    try:
        vals = [float(l.split()[-2]) for l in open(FP64_PEAK_FILE) if l.startswith("DMMA")]
        return max(vals), "measured DMMA.8x8x4 issue ceiling (profiles/r01_fp64_pipe_peak.txt)"
    except Exception:
        return 37.2, "nominal 148 SM x 64 FP64 FMA/clk x 1.965 GHz"


def make_ubm(seed=0):
    """SURVEY §8(d) config 2 recipe: w ~ Dir(10), mu ~ N(0, 0.3^2), Sigma = A A'/2F + 0.5 I."""
    rng = np.random.default_rng(seed)
    w = rng.dirichlet(np.full(C, 10.0))
    mu = rng.normal(0.0, 0.3, (C, F))
    a = rng.normal(0.0, 1.0, (C, F, 2 * F))
    cov = np.einsum("cik,cjk->cij", a, a) / (2 * F) + 0.5 * np.eye(F)
    return w, mu, cov


def sample_frames(w, mu, cov, n, seed, device):
    """n frames from the full GMM, generated on the device (not timed), returned as f32."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    wt = torch.from_numpy(w).to(device)
    counts = torch.bincount(torch.multinomial(wt, n, replacement=True, generator=g), minlength=C).cpu().numpy()
    chol = torch.linalg.cholesky(torch.from_numpy(cov).to(device))
    mut = torch.from_numpy(mu).to(device)
    out = torch.empty((n, F), dtype=torch.float32, device=device)
    pos = 0
    for c0 in range(0, C, 256):
        c1 = min(C, c0 + 256)
        mx = int(counts[c0:c1].max())
        z = torch.randn((c1 - c0, mx, F), dtype=torch.float64, device=device, generator=g)
        x = torch.bmm(z, chol[c0:c1].transpose(1, 2)) + mut[c0:c1, None, :]
        for i, c in enumerate(range(c0, c1)):
            k = int(counts[c])
            out[pos:pos + k] = x[i, :k].to(torch.float32)
            pos += k
    perm = torch.randperm(n, device=device, generator=g)
    return out[perm].contiguous()


class Clocks:
    """nvidia-smi sampler (the recipe's clocks line).  Started before the warm-up so it is already
    sampling when the timed region begins; only samples stamped inside [mark(), stop()] are kept."""

    def __init__(self, index):
        self.proc = None
        self.t0 = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), "--query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def mark(self):
        self.t0 = time.time()

    def stop(self):
        if self.proc is None:
            return None
        t1 = time.time()
        time.sleep(0.15)  # let the sample covering the end of the region land
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        import datetime
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                if self.t0 is not None and not (self.t0 <= ts <= t1 + 0.1):
                    continue
                rows.append((float(parts[1]), float(parts[2]), parts[4:8]))
            except ValueError:
                pass
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        load = [r[0] for r in rows]
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": rows[0][1], "reasons": reasons,
                "samples": len(rows)}


def bench_reference(args):
    """CPU reference arm: the reference align_frames algorithm (oracle port) on host cores."""
    from oracle import tvkit_oracle as orc
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w, mu, cov = make_ubm(0)
    rng = np.random.default_rng(1)
    comp = rng.choice(C, p=w, size=args.ref_frames)
    L = np.linalg.cholesky(cov)
    x = (mu[comp] + np.einsum("tij,tj->ti", L[comp], rng.standard_normal((args.ref_frames, F)))).astype(np.float32)
    diag = (w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
    full = (w, mu, cov)
    for _ in range(args.warmup):
        orc.align(diag, full, x, K_TOP, PRUNE)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        orc.align(diag, full, x, K_TOP, PRUNE)
    dt = (time.perf_counter() - t0) / args.steps
    fps = args.ref_frames / dt
    cores = len(os.sched_getaffinity(0))
    sample = f"{args.ref_frames} frames of the config-2 workload per step (one align_frames chunk)"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2 frame posteriors: 2048-comp full-cov UBM, 60-dim, top-20, prune 0.025",
                   "frames_per_step": args.ref_frames},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "x_realtime": fps / 100.0,
    }), flush=True)


def cpu_baseline_sample(n_frames=4000):
    """Oracle timing on rank 0 (reported baseline, not the target)."""
    from oracle import tvkit_oracle as orc
    w, mu, cov = make_ubm(0)
    rng = np.random.default_rng(2)
    comp = rng.choice(C, p=w, size=n_frames)
    L = np.linalg.cholesky(cov)
    x = (mu[comp] + np.einsum("tij,tj->ti", L[comp], rng.standard_normal((n_frames, F)))).astype(np.float32)
    diag = (w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
    t0 = time.perf_counter()
    orc.align(diag, (w, mu, cov), x, K_TOP, PRUNE)
    dt = time.perf_counter() - t0
    return {"value": n_frames / dt, "unit": "frames/s", "cores": len(os.sched_getaffinity(0)), "kind": "port",
            "sample": f"{n_frames} frames (one chunk) of the config-2 workload, oracle restatement of "
                      f"tvkit.gmm.align_frames, numpy/OpenBLAS on all host cores"}


def bench_ours(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local % torch.cuda.device_count())
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    import paper_1906_08556_b200 as pkg
    from paper_1906_08556_b200 import _device, _lib

    w, mu, cov = make_ubm(0)
    diag_m = pkg.GmmDiag(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)))
    full_m = pkg.GmmFull(w, mu, cov)
    n = args.frames
    x = sample_frames(w, mu, cov, n, 1000 + rank, dev)
    log(f"[bench] rank {rank}: {n} frames generated")
    dtab, ftab = diag_m.device_table(), full_m.device_table()
    k = K_TOP
    offsets = _lib.empty((n + 1,), torch.int64)
    comps = _lib.empty((n * k,), torch.int32)
    wts = _lib.empty((n * k,), torch.float32)
    ws_bytes = int(_lib.load().tvk_align_workspace_bytes(n, k, C))
    ws = _lib.empty((ws_bytes,), torch.uint8)
    quad = None

    def step(dense=False):
        nonlocal quad
        if dense and quad is None:
            quad = ftab.table
        _lib.call("tvk_align_frames", _lib.ptr(x), 0, n, F, _lib.ptr(dtab.table), _lib.ptr(quad) if dense else None,
                  _lib.ptr(ftab.prec), C, k, PRUNE, 1 if dense else 0, _lib.ptr(ws), ws_bytes, _lib.ptr(offsets),
                  _lib.ptr(comps), _lib.ptr(wts), None, None, _lib.stream())

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.current_stream()

    def timed(fn, reps):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(reps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / reps

    clocks = Clocks(local)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    log("[bench] warm-up done")
    clocks.mark()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    entries = int(offsets[n].item())
    value = world * n / (ms / 1e3)
    ref_offsets = offsets.clone()
    ref_comps = comps[:entries].clone()

    log(f"[bench] timed region: {ms:.1f} ms/step")
    # per-stage kernel times (CUDA events on the launching stream)
    sel = _lib.empty((n, k), torch.int32)
    sll = _lib.empty((n, k))
    gws_bytes = int(_lib.load().tvk_full_loglik_workspace_bytes(n, k, C))
    gws = _lib.empty((gws_bytes,), torch.uint8)

    def stage1():
        _lib.call("tvk_select_topk", _lib.ptr(x), 0, n, F, _lib.ptr(dtab.table), C, k, _lib.ptr(sel), None,
                  _lib.stream())

    def stage2(dense=False):
        _lib.call("tvk_full_loglik_selected", _lib.ptr(x), 0, n, F, _lib.ptr(quad) if dense else None,
                  _lib.ptr(ftab.prec), C, k, 1 if dense else 0, _lib.ptr(sel), _lib.ptr(sll), _lib.ptr(gws),
                  gws_bytes, _lib.stream())

    stage1()
    s1_ms = timed(stage1, 3)
    stage2()
    s2_ms = timed(stage2, 3)
    peak, peak_src = fp64_peak()
    tpeak, tpeak_src = f16_peak()
    s1_tf = FLOP_DIAG_PER_FRAME * n / (s1_ms / 1e3) / 1e12
    s1_exec = F16_EXEC_PER_FRAME * n / (s1_ms / 1e3) / 1e12
    s2_tf = FLOP_GROUPED_PER_FRAME * n / (s2_ms / 1e3) / 1e12
    s2_exec = DMMA_EXEC_PER_FRAME * n / (s2_ms / 1e3) / 1e12
    # dense north-star variant: quadratic-feature GEMM over all C components (the reference's own work)
    dense = None
    if args.dense_steps > 0:
        step(dense=True)
        torch.cuda.synchronize()
        dense_ms = timed(lambda: step(dense=True), args.dense_steps)
        same = bool(torch.equal(offsets, ref_offsets)) and bool(torch.equal(comps[:entries], ref_comps))
        stage2(dense=True)
        d2_ms = timed(lambda: stage2(dense=True), 1)
        dense = {"value": world * n / (max_over_ranks(dense_ms) / 1e3), "unit": "frames/s",
                 "ms_per_step": dense_ms, "steps": args.dense_steps,
                 "alignment_identical_to_grouped": same,
                 "full_ll_kernel": {"launch_ms": d2_ms, "flop_per_frame": FLOP_FULL_PER_FRAME,
                                    "achieved_tflops": FLOP_FULL_PER_FRAME * n / (d2_ms / 1e3) / 1e12,
                                    "frac_of_peak": FLOP_FULL_PER_FRAME * n / (d2_ms / 1e3) / 1e12 / peak}}
    prof = os.path.join(REPO, "profiles", "r02_ncu_summary.json")
    traffic = None
    if os.path.exists(prof):
        try:  # DRAM bytes/frame of the dominant kernel from the committed ncu --set full capture
            reps = json.load(open(prof))["reports"]
            per_frame = [k["dram_bytes_per_frame"] for r in reps.values() for k in r
                         if k["kernel"].startswith("whiten_ll_kernel") and "dram_bytes_per_frame" in k][0]
            traffic = per_frame * n
        except Exception:
            traffic = None
    del sel, sll, gws

    log("[bench] stage timing done")
    # e2e through the public API: pinned host frames -> align_frames -> host SparseAlignment
    host = torch.empty((n, F), dtype=torch.float32, pin_memory=True)
    host.copy_(x)
    xs_check = x[:max(0, min(n, args.exact_frames))].clone()
    del x, ws, comps, wts
    torch.cuda.empty_cache()
    e2e_steps = max(1, min(args.steps, 3))
    pkg.align_frames(diag_m, full_m, host, top_k=k, prune=PRUNE)
    barrier()
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(e2e_steps):
        ali = pkg.align_frames(diag_m, full_m, host, top_k=k, prune=PRUNE)
        d2h = ali.offsets.nbytes + ali.components.nbytes + ali.weights.nbytes
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e_value = world * n / e2e_s
    del host, ali

    log("[bench] e2e done")
    exact = selection_exactness(xs_check, dtab, args.exact_frames, pkg) if args.exact_frames > 0 else None
    del xs_check
    torch.cuda.empty_cache()
    em = c5 = c4 = None
    if args.em_utts > 0:  # config 3: augmented, min-div + Sigma update, no realignment
        em, _ = bench_em_leg(args, pkg, dev, rank, world, barrier, max_over_ranks, "augmented", args.em_utts,
                             args.em_steps, args.em_warmup,
                             dict(iterations=10 ** 6, min_div=True, sigma_update=True, realign_interval=0),
                             "config 3: augmented (Kaldi) TVM, C=2048, F=60, R=400, min-div + Sigma update")
        log(f"[bench] config 3 EM: {em['value']:.3f} s/iter")
    if args.c5_utts > 0:  # config 5: standard, min-div + UBM-mean update + realignment every iteration
        c5, _ = bench_em_leg(args, pkg, dev, rank, world, barrier, max_over_ranks, "standard", args.c5_utts,
                             args.em_steps, args.em_warmup,
                             dict(iterations=10 ** 6, min_div=True, sigma_update=False, update_mean=True,
                                  realign_interval=1),
                             "config 5 training: standard TVM, C=2048, F=60, R=400, min-div + UBM-mean (bias) "
                             "update + realignment of every frame each iteration", profile_kernels=False)
        log(f"[bench] config 5 EM: {c5['value']:.3f} s/iter")
        if args.extract_utts > 0:
            c5["extraction"] = bench_extract_leg(args, pkg, dev, rank, world, barrier, max_over_ranks,
                                                 args.extract_utts)
            log(f"[bench] config 5 extraction: {c5['extraction']['value']:.0f} utts/s")
    c1 = None
    if args.config1 and world == 1 and not args.no_cpu:
        try:
            c1 = bench_config1(pkg)
            log(f"[bench] config 1: {c1['value']:.2f} s/run (reference algorithm on the host: "
                f"{c1['cpu_baseline']['value']:.1f} s)")
        except Exception as exc:  # reported leg: never kill the headline line
            c1 = {"error": str(exc)}
    if args.config4_utts > 0:  # config 4: VoxCeleb scale (opt-in: ~1 min per iteration on one GPU)
        c4, _ = bench_em_leg(args, pkg, dev, rank, world, barrier, max_over_ranks, "augmented", args.config4_utts,
                             1, 0, dict(iterations=10 ** 6, min_div=True, sigma_update=True, realign_interval=0),
                             "config 4: VoxCeleb-scale augmented TVM, C=2048, F=60, R=400, min-div + residual "
                             "covariance update", profile_kernels=False)
        log(f"[bench] config 4 EM: {c4['value']:.3f} s/iter")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config2 frame posteriors: 2048-comp full-cov UBM, 60-dim MFCC-shaped "
                                   "frames, top-20 diag preselection, prune 0.025",
                       "frames_per_gpu_per_step": n, "global_frames_per_step": world * n,
                       "parallelism": f"dp{world} (frames sharded, no collective)",
                       "l2": "inputs (2.4 GB/GPU) larger than L2"},
            "x_realtime": value / 100.0,
            "entries_per_frame": entries / n,
            # per step: select_tc + select_post + select_exact, 8 per grouped-LL frame window (hist
            # memset/count/scan/scatter, tile count/scan/build, whiten_ll), finalize + 3 scans + compact
            "gpu_launches": args.steps * (3 + 8 * ((n + WINDOW_FRAMES - 1) // WINDOW_FRAMES) + 5),
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": n * F * 4,
                    "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                    "path": "paper_1906_08556_b200.align_frames(pinned host f32 frames) -> SparseAlignment"},
            # dominant kernel: whiten_ll (FP64 DMMA); the preselection stage is reported beside it
            "roofline": {"bound": "tensor", "kernel": "whiten_ll_kernel (FP64 DMMA full-cov LL of the top-20 pairs)",
                         "achieved": s2_tf, "peak": peak, "unit": "TFLOP/s", "frac": s2_tf / peak,
                         "peak_source": peak_src, "flop_per_frame": FLOP_GROUPED_PER_FRAME, "launch_ms": s2_ms,
                         "share_of_step": s2_ms / ms, "traffic": traffic,
                         "executed_tflops": s2_exec, "executed_frac": s2_exec / peak,
                         "executed_flop_per_frame": DMMA_EXEC_PER_FRAME,
                         "note": "achieved = algorithmic 2*K*Q flop/frame (Q = 1+F+F(F+1)/2: the quadratic-feature "
                                 "count of SURVEY 8(d) restricted to the K selected components, 8(f) row 3); the kernel "
                                 "executes the triangular U = L^-T product in 8x8x4 DMMA blocks (executed_flop_per_frame)"},
            "stages": {"select_ms": s1_ms, "whiten_ll_ms": s2_ms,
                       "select": {"bound": "tensor (tcgen05 kind::f16)",
                                  "kernels": "select_tc_kernel (3xFP16 scores, candidate windows) + "
                                             "select_post_kernel (window merge, FP64 cluster order) + "
                                             "select_exact_kernel (flagged frames)",
                                  "achieved": s1_tf, "peak": tpeak, "unit": "TFLOP/s", "frac": s1_tf / tpeak,
                                  "peak_source": tpeak_src, "flop_per_frame": FLOP_DIAG_PER_FRAME,
                                  "executed_f16_tflops": s1_exec, "executed_frac": s1_exec / tpeak,
                                  "executed_flop_per_frame": F16_EXEC_PER_FRAME},
                       "rest_ms": ms - s1_ms - s2_ms},
            "dense_variant": dense,
            "clocks": clk,
        }
        line["selection_exactness"] = exact
        if not args.no_cpu:
            try:
                line["cpu_baseline"] = cpu_baseline_sample(args.cpu_frames)
            except Exception as exc:  # never let the reported baseline kill the bench line
                line["cpu_baseline"] = {"error": str(exc)}
            log("[bench] cpu baselines")
            for leg, fn in ((em, em_cpu_baseline), (c5, extract_cpu_baseline)):
                if leg is None or world > 1:
                    continue
                try:
                    cb = fn()
                    tgt = leg if fn is em_cpu_baseline else leg.get("extraction")
                    if tgt is not None:
                        tgt["cpu_baseline"] = cb
                        tgt["vs_cpu"] = (cb["value"] / tgt["value"]) if fn is em_cpu_baseline else \
                            (tgt["value"] / cb["value"])
                except Exception as exc:
                    (leg if fn is em_cpu_baseline else leg.setdefault("extraction", {}))["cpu_baseline"] = \
                        {"error": str(exc)}
        if em is not None:
            line["em_iteration"] = em
        if c5 is not None:
            line["config5"] = c5
        if c4 is not None:
            line["config4"] = c4
        if c1 is not None:
            line["config1"] = c1
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------------------------ EM legs (configs 3-5)

D_TVM, P_OFF, FR_UTT = 400, 100.0, 300
FLOP_EM_UTT = 2 * C * D_TVM * (D_TVM + 1) + 4 * C * F * D_TVM + D_TVM ** 3   # 917.6 MFLOP
FLOP_EM_GEMM_UTT = 2 * C * D_TVM * (D_TVM + 1) + 4 * C * F * D_TVM          # L, A (2CP each), b, B (2CFD each)
# per-iteration fixed GEMM work: workspace W (2CF^2D) + U (CF D(D+1)), Sigma update T B' (2CF^2D), T.R (2CFD^2)
FLOP_EM_GEMM_FIXED = 2 * C * F * F * D_TVM + C * F * D_TVM * (D_TVM + 1) + 2 * C * F * F * D_TVM \
    + 2 * C * F * D_TVM * D_TVM
FLOP_EXTRACT_UTT = C * D_TVM * (D_TVM + 1) + 2 * C * F * D_TVM + D_TVM ** 3 // 3  # L + b + Cholesky


def generator(form, seed=7):
    """synth.py:90-104 recipe at C=2048, F=60, R=400 (host, numpy): w ~ Dir(10), mu ~ N(0, 8^2),
    Sigma = A A'/2F + 0.5 I, T ~ N(0, 1); augmented: T[:, :, 0] = mu / p; standard: bias = mu."""
    rng = np.random.default_rng(seed)
    w = rng.dirichlet(np.full(C, 10.0))
    mu = rng.normal(0.0, 8.0, (C, F))
    a = rng.normal(0.0, 1.0, (C, F, 2 * F))
    sig = np.einsum("cik,cjk->cij", a, a) / (2 * F) + 0.5 * np.eye(F)
    Tg = rng.normal(0.0, 1.0, (C, F, D_TVM))
    if form == "augmented":
        Tg[:, :, 0] = mu / P_OFF
    return dict(w=w, mu=mu, sig=sig, T=Tg, form=form)


def device_utterances(gen, n_utt, seed, dev):
    """n_utt synthetic utterances x 300 frames drawn on the device from the generator (synth.py:107-147
    recipe: augmented x = T_c z + Sigma_c^(1/2) e with z = p e1 + N(0, I); standard x = mu_c + T_c w + ...)."""
    import torch
    g = torch.Generator(device=dev).manual_seed(seed)
    Td = torch.from_numpy(gen["T"]).to(dev).view(C * F, D_TVM)
    L = torch.linalg.cholesky(torch.from_numpy(gen["sig"]).to(dev))
    mu = torch.from_numpy(gen["mu"]).to(dev)
    x = torch.empty((n_utt * FR_UTT, F), dtype=torch.float32, device=dev)
    wt = torch.from_numpy(gen["w"]).to(dev)
    for u0 in range(0, n_utt, 64):
        u1 = min(n_utt, u0 + 64)
        z = torch.randn((u1 - u0, D_TVM), dtype=torch.float64, device=dev, generator=g)
        if gen["form"] == "augmented":
            z[:, 0] += P_OFF
        M = (Td @ z.T).T.reshape(u1 - u0, C, F)  # latent-shifted mean supervectors
        if gen["form"] == "standard":
            M += mu
        cu = torch.multinomial(wt, (u1 - u0) * FR_UTT, replacement=True, generator=g).view(u1 - u0, FR_UTT)
        means = torch.gather(M, 1, cu[:, :, None].expand(-1, -1, F))
        e = torch.randn((u1 - u0, FR_UTT, F), dtype=torch.float64, device=dev, generator=g)
        x[u0 * FR_UTT:u1 * FR_UTT] = (means + torch.einsum("utij,utj->uti", L[cu], e)).reshape(-1, F).float()
    return x


def em_setup(pkg, gen, n_local, rank, dev, cfg_kw, first_utt=0):
    """(trainer, align_diag, align_cov, store) for this rank's utterances [first_utt, first_utt + n_local)."""
    from paper_1906_08556_b200 import pipeline as P
    x = device_utterances(gen, n_local, 11 + rank, dev)
    ids = [f"u{first_utt + i:08d}" for i in range(n_local)]
    store = P.DeviceFeatureStore(x, np.arange(0, (n_local + 1) * FR_UTT, FR_UTT), ids)
    T, Sg, form = gen["T"], gen["sig"], gen["form"]
    bias = gen["mu"] if form == "standard" else None
    genm = pkg.TvModel(form, T, Sg, gen["w"], gen["mu"], bias, P_OFF if form == "augmented" else 0.0)
    ubm_full, ubm_diag = genm.alignment_ubm_full(), genm.alignment_ubm_diag()
    model = pkg.init_model(ubm_full, D_TVM, form, seed=0, prior_offset=P_OFF)
    cfg = P.TrainConfig(formulation=form, latent_dim=D_TVM, top_k=K_TOP, prune=PRUNE, seeds=(0,), **cfg_kw)
    tr = P.DeviceTrainer(model, store.device_corpus(ids), cfg)
    return tr, ubm_diag.copy(), ubm_full.covariances, store, model


def estep_i8_work(n_utts):
    """(executed int8 ops, FP64-equivalent 2MNK flops) of the four E-step contractions of one EM
    iteration over n_utts utterances, batched as _estep does."""
    from paper_1906_08556_b200 import _estep
    P = D_TVM * (D_TVM + 1) // 2
    up = lambda v, t: -(-v // t) * t
    ops = eq = 0
    left = n_utts
    while left > 0:
        ub = min(left, _estep.E_STEP_BATCH)
        left -= ub
        for (m, n, k, s) in ((ub, P, C, _estep.I8_DIGITS), (C, P, ub, _estep.I8_DIGITS),
                             (ub, D_TVM, C * F, _estep.I8_DIGITS_F), (C * F, D_TVM, ub, _estep.I8_DIGITS_F)):
            if m * n * k < _estep.I8_MIN_WORK:
                continue
            ops += 2 * up(m, 128) * up(n, 64) * up(k, 32) * s * (s + 1) // 2
            eq += 2 * m * n * k
    return ops, eq


def em_kernel_breakdown(tr, it, align_diag, align_cov):
    """One extra EM iteration under the torch profiler (CUPTI kernel timestamps; outside every timed
    region): device time per kernel, and the achieved rate of the dominant kernel (gemm_i8_kernel)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        if tr.alignment is None:
            tr.align(align_diag, align_cov)
        tr.iteration()
        tr.realign_point(it, align_diag)
        torch.cuda.synchronize()
    ev = [e for e in prof.key_averages() if e.self_device_time_total > 0]
    tot = sum(e.self_device_time_total for e in ev) / 1e6
    kern = {}
    for e in ev:
        name = e.key.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        k = kern.setdefault(name, [0.0, 0])
        k[0] += e.self_device_time_total / 1e6
        k[1] += e.count
    top = sorted(kern.items(), key=lambda kv: -kv[1][0])[:8]
    return tot, {n: {"s": round(v[0], 5), "share": round(v[0] / tot, 4), "launches": v[1]} for n, v in top}


def bench_em_leg(args, pkg, dev, rank, world, barrier, max_over_ranks, form, n_global, steps, warmup, cfg_kw,
                 label, profile_kernels=True):
    """Seconds per EM iteration on n_global utterances sharded over the ranks (strong scaling): each
    timed iteration = E-step over the corpus (BW stats, posteriors, accumulators) + one all-reduce +
    M-step (update_T, update_sigma, min-divergence), plus realignment of every frame where the config
    asks for it (CUDA events on the launching stream, max over ranks)."""
    import torch
    from paper_1906_08556_b200 import _dist
    lo, hi = _dist.shard_range(n_global, rank, world)
    gen = generator(form)
    tr, align_diag, align_cov, store, model = em_setup(pkg, gen, hi - lo, rank, dev, cfg_kw, first_utt=lo)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr.align(align_diag, align_cov)
    barrier()
    align_s = max_over_ranks(time.perf_counter() - t0)
    it = 0

    def one():
        nonlocal it
        it += 1
        if tr.alignment is None:
            tr.align(align_diag, align_cov)
        a = tr.iteration()
        tr.realign_point(it, align_diag)
        return a

    for _ in range(warmup):
        one()
    barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    auxes = [one() for _ in range(steps)]
    e1.record(stream)
    barrier()
    sec = max_over_ranks(e0.elapsed_time(e1) / 1e3 / steps)
    out = {"value": sec, "unit": "s/iter", "higher_is_better": False, "global_utts": n_global,
           "utts_per_gpu": hi - lo, "frames_per_utt": FR_UTT, "steps": steps, "warmup": warmup,
           "scaling": "strong", "alignment_s": align_s, "config": label,
           "achieved_tflops": n_global * FLOP_EM_UTT / sec / 1e12, "flop_per_utt": FLOP_EM_UTT,
           "aux_last": auxes[-1]}
    if profile_kernels:  # every rank: the extra iteration's all-reduce needs all of them
        tot, kern = em_kernel_breakdown(tr, it + 1, align_diag, align_cov)
        g = kern.get("gemm_i8_kernel")
        if g:
            ops, fp64_eq = estep_i8_work(hi - lo)
            peak, src = i8_peak()
            dpeak, dsrc = fp64_peak()
            ach = ops / g["s"] / 1e12
            out["roofline"] = {"bound": "tensor", "kernel": "gemm_i8_kernel (FP64 emulated on the int8 tensor cores: "
                                                            "L = N U, A += N'M, b = F W, B += F'phi)",
                               "achieved": ach, "peak": peak, "unit": "TOP/s", "frac": ach / peak,
                               "peak_source": src, "int8_ops_per_iter": ops, "kernel_s_per_iter": g["s"],
                               "share_of_kernel_time": g["share"],
                               "fp64_equivalent_tflops": fp64_eq / g["s"] / 1e12,
                               "fp64_equivalent_vs_dmma_ceiling": fp64_eq / g["s"] / 1e12 / dpeak,
                               "dmma_ceiling": dpeak, "dmma_ceiling_source": dsrc,
                               "note": "achieved = executed int8 multiply-adds x 2 of the digit products "
                                       "(S(S+1)/2 per tile, S = 7 for the N contractions, 8 for the F ones, "
                                       "padded tiles) / CUPTI kernel time; fp64_equivalent = 2MNK of the four "
                                       "contractions / the same time",
                               "method": "torch.profiler (CUPTI) kernel durations of one extra iteration"}
        out["kernel_breakdown"] = {"kernel_s_per_iter": tot, "top": kern}
    del tr, store
    torch.cuda.empty_cache()
    return out, model


def bench_extract_leg(args, pkg, dev, rank, world, barrier, max_over_ranks, n_global):
    """Config 5 extraction: i-vectors of n_global fresh standard-formulation utterances through the
    public extract_corpus (alignment with the predictive-covariance UBM, BW stats, posterior means),
    frames resident in HBM (DeviceFeatureStore), embeddings returned to the host; median of three
    passes."""
    import torch
    from paper_1906_08556_b200 import _dist, pipeline as P
    gen = generator("standard", seed=9)
    lo, hi = _dist.shard_range(n_global, rank, world)
    x = device_utterances(gen, hi - lo, 211 + rank, dev)
    # each rank holds only its shard; extract_corpus shards the global id list the same way
    all_ids = [f"e{i:08d}" for i in range(n_global)]
    store = P.DeviceFeatureStore(x, np.arange(0, (hi - lo + 1) * FR_UTT, FR_UTT), all_ids[lo:hi], all_ids)
    T, Sg = gen["T"], gen["sig"]
    model = pkg.TvModel("standard", T, Sg, gen["w"], gen["mu"], gen["mu"].copy(), 0.0)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world == 1:  # warm-up on a slice (tables, allocator); a rank-sharded store has no such slice
        P.extract_corpus(model, store, top_k=K_TOP, prune=PRUNE, ids=all_ids[:min(n_global, 2048)])
    runs = []
    for _ in range(3):  # median of three timed passes over the whole corpus
        barrier()
        e0.record(stream)
        _, emb = P.extract_corpus(model, store, top_k=K_TOP, prune=PRUNE)
        e1.record(stream)
        barrier()
        runs.append(max_over_ranks(e0.elapsed_time(e1) / 1e3))
    sec = sorted(runs)[1]
    ups = n_global / sec
    ok = bool(np.all(np.isfinite(emb)))
    del x, store
    torch.cuda.empty_cache()
    return {"value": ups, "unit": "utterances/s", "global_utts": n_global, "utts_per_gpu": hi - lo,
            "seconds": sec, "seconds_runs": runs, "x_realtime": ups * FR_UTT / 100.0, "scaling": "strong",
            "achieved_tflops_posterior": n_global * FLOP_EXTRACT_UTT / sec / 1e12, "finite": ok,
            "path": "pipeline extract (alignment + BW stats + posterior mean), frames in HBM, i-vectors to host"}


C1 = dict(C=64, F=20, R=100, spk=50, upc=4, frames=300, iters=5, within=0.3)


def config1_corpus(seed=1):
    """BASELINE config 1 shape (64-comp UBM, 20-dim, R=100, 50 speakers x 4 utts x 300 frames), host
    numpy, synth.py:90-147 recipe (augmented): w ~ Dir(10), mu ~ N(0, 8^2), Sigma = AA'/2F + 0.5 I,
    T ~ N(0, 1) with T[:, :, 0] = mu / p; x = T_c (p e1 + w_spk) + Sigma_c^(1/2) e."""
    c, f, r = C1["C"], C1["F"], C1["R"]
    rng = np.random.default_rng(seed)
    w = rng.dirichlet(np.full(c, 10.0))
    mu = rng.normal(0.0, 8.0, (c, f))
    a = rng.normal(0.0, 1.0, (c, f, 2 * f))
    sig = np.einsum("cik,cjk->cij", a, a) / (2 * f) + 0.5 * np.eye(f)
    T = rng.normal(0.0, 1.0, (c, f, r))
    T[:, :, 0] = mu / P_OFF
    L = np.linalg.cholesky(sig)
    feats, ids = {}, []
    for s_ in range(C1["spk"]):
        zs = rng.normal(0.0, 1.0, r)
        zs[0] += P_OFF
        for u in range(C1["upc"]):
            z = zs + C1["within"] * rng.normal(0.0, 1.0, r)
            comp = rng.choice(c, p=w, size=C1["frames"])
            m = np.einsum("cfr,r->cf", T, z)
            x = m[comp] + np.einsum("tij,tj->ti", L[comp], rng.standard_normal((C1["frames"], f)))
            uid = f"s{s_:03d}u{u}"
            feats[uid] = x.astype(np.float32)
            ids.append(uid)
    return dict(w=w, mu=mu, sig=sig, T=T, feats=feats, ids=ids)


def bench_config1(pkg):
    """Config 1 end to end through the public API (train_extractor: 5 EM iterations with min-div and
    Sigma update, then extract_corpus), host features in (InMemoryFeatureStore: every H2D copy inside
    the timing) and the trained model / i-vectors out, against the reference algorithm (oracle
    restatement of pipeline.train_extractor) on the host cores on the same corpus, with a parity check."""
    import warnings
    from types import SimpleNamespace
    from oracle import tvkit_oracle as orc
    from paper_1906_08556_b200 import pipeline as P
    cor = config1_corpus()
    genm = pkg.TvModel("augmented", cor["T"], cor["sig"], cor["w"], cor["mu"], None, P_OFF)
    full, diag = genm.alignment_ubm_full(), genm.alignment_ubm_diag()
    cfg = P.TrainConfig(formulation="augmented", latent_dim=C1["R"], iterations=C1["iters"], min_div=True,
                        sigma_update=True, update_mean=False, realign_interval=0, top_k=K_TOP, prune=PRUNE,
                        seeds=(0,), batch_size_utts=8, workers=1)
    store = P.InMemoryFeatureStore(cor["feats"])

    def run():
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            model, metrics = P.train_extractor(cfg, store, diag, full, seed=0)
            _, emb = P.extract_corpus(model, store, top_k=K_TOP, prune=PRUNE)
        return model, metrics, emb

    run()  # warm-up (tables, allocator)
    t0 = time.perf_counter()
    model, metrics, emb = run()
    ours = time.perf_counter() - t0
    ns = SimpleNamespace(formulation="augmented", latent_dim=C1["R"], iterations=C1["iters"], min_div=True,
                         sigma_update=True, update_mean=False, realign_interval=0, top_k=K_TOP, prune=PRUNE,
                         prior_offset=P_OFF, batch_size_utts=8)
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref, ref_aux = orc.train(ns, cor["feats"], cor["ids"], (diag.weights, diag.means, diag.variances),
                                 (full.weights, full.means, full.covariances), seed=0)
    cpu = time.perf_counter() - t0
    rel = lambda a, b: float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))  # noqa: E731
    aux = np.array([r.aux for r in metrics.records])
    return {"value": ours, "unit": "s/run", "higher_is_better": False, "iterations": C1["iters"],
            "s_per_iter": ours / C1["iters"], "utts": len(cor["ids"]), "frames_per_utt": C1["frames"],
            "config": "config 1: augmented TVM, C=64, F=20, R=100, 200 utts x 300 frames, 5 EM iterations "
                      "(min-div + Sigma update) + extract_corpus",
            "path": "pipeline.train_extractor + extract_corpus (public API, host features, models/i-vectors to host)",
            "cpu_baseline": {"value": cpu, "unit": "s/run (training only)", "cores": len(os.sched_getaffinity(0)),
                             "kind": "port", "sample": "the whole config-1 training run, oracle restatement of "
                                                       "tvkit.pipeline.train_extractor (numpy/OpenBLAS, all host cores)"},
            "vs_cpu": cpu / ours,
            "parity_vs_reference_algorithm": {"T_rel": rel(model.T, ref.T), "Sigma_rel": rel(model.Sigma, ref.Sigma),
                                              "aux_rel": float(np.max(np.abs(aux - np.array(ref_aux))
                                                                      / np.abs(np.array(ref_aux)))),
                                              "tolerance": "T, Sigma 1e-4 relative; aux 1e-9",
                                              "ivectors_finite": bool(np.all(np.isfinite(emb)))}}


def em_cpu_baseline(n_utts=6, comp_sample=128):
    """The reference EM iteration on the host cores (oracle restatement of tvm.py/pipeline.py), timed on
    a bounded sample and extrapolated per BASELINE.md §4: sec/iter = workspace + 20k x (BW stats +
    posterior + accumulate per utterance) + per-batch accumulator merges + update_T + update_sigma +
    min-div.  Per-component work (workspace, update_T, update_sigma) is timed on ``comp_sample``
    components and scaled by C / comp_sample; the per-utterance work on ``n_utts`` utterances."""
    from oracle import tvkit_oracle as orc
    gen = generator("augmented")
    rng = np.random.default_rng(5)
    model = orc.make_model("augmented", rng.normal(0, 1, (C, F, D_TVM)), gen["sig"], gen["w"], gen["mu"], None,
                           P_OFF)
    model.T[:, :, 0] = gen["mu"] / P_OFF
    gm = orc.make_model("augmented", gen["T"], gen["sig"], gen["w"], gen["mu"], None, P_OFF)
    ids, feats, _ = orc.sample_utterances(gm, n_utts, 1, (FR_UTT, FR_UTT), 0.3, rng)
    pc = orc.predictive_covariances(gm)
    diag = (gen["w"], gen["mu"], np.ascontiguousarray(np.diagonal(pc, axis1=1, axis2=2)))
    alis = [orc.align(diag, (gen["w"], gen["mu"], pc), feats[u], K_TOP, PRUNE) for u in ids]  # untimed
    sub = orc.make_model("augmented", model.T[:comp_sample], model.Sigma[:comp_sample], gen["w"][:comp_sample],
                         gen["mu"][:comp_sample], None, P_OFF)
    t0 = time.perf_counter()
    orc.workspace(sub)
    t_ws = (time.perf_counter() - t0) * C / comp_sample
    # full-size workspace arrays for the per-utterance timing (values do not change the work)
    ws = orc.workspace(sub)
    reps = -(-C // comp_sample)
    ws.W = np.concatenate([ws.W] * reps)[:C]
    ws.U = np.concatenate([ws.U] * reps)[:C]
    ws.Sinv = np.concatenate([ws.Sinv] * reps)[:C]
    ws.logdet = np.concatenate([ws.logdet] * reps)[:C]
    t0 = time.perf_counter()
    stats = [orc.bw_stats(feats[u], *alis[i], C) for i, u in enumerate(ids)]
    acc = orc.accumulate(model, stats, ws)
    t_utt = (time.perf_counter() - t0) / n_utts
    other = orc.zero_acc(C, F, D_TVM)
    t0 = time.perf_counter()
    orc.merge_acc(other, acc)
    t_merge = time.perf_counter() - t0  # once per batch of 8 utterances (pipeline.py:406-413)
    suba = orc.zero_acc(comp_sample, F, D_TVM)
    for k in ("A", "B", "N", "Ssum"):
        setattr(suba, k, getattr(acc, k)[:comp_sample])
    suba.U, suba.phi_sum, suba.moment_sum = acc.U, acc.phi_sum, acc.moment_sum
    import warnings
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        newT = orc.update_T(sub, suba)
        orc.update_sigma(sub, suba, newT)
    t_m = (time.perf_counter() - t0) * C / comp_sample
    t0 = time.perf_counter()
    tr = orc.min_div(acc, "augmented")
    sub.T = sub.T.copy()
    orc.apply_min_div(sub, tr, acc.phi_sum / acc.U)
    t_md = (time.perf_counter() - t0) * C / comp_sample
    n_glob = 20000
    sec = t_ws + n_glob * t_utt + (n_glob / 8) * t_merge + t_m + t_md
    return {"value": sec, "unit": "s/iter", "cores": len(os.sched_getaffinity(0)), "kind": "port",
            "sample": f"{n_utts} utterances (BW stats + posterior + accumulate) and {comp_sample} of {C} components "
                      f"(workspace, update_T, update_sigma, min-div) of the config-3 shape, oracle restatement of "
                      f"tvkit (numpy/OpenBLAS, all host cores), extrapolated to 20k utterances per BASELINE.md §4",
            "parts_s": {"workspace": t_ws, "per_utt": t_utt, "merge_per_batch_of_8": t_merge, "mstep": t_m,
                        "min_div": t_md}}


def extract_cpu_baseline(n_utts=3, comp_sample=128):
    """Reference extraction per utterance on the host (align + BW stats + posterior mean) plus the
    one-off workspace, extrapolated to 150k utterances."""
    from oracle import tvkit_oracle as orc
    gen = generator("standard", seed=9)
    rng = np.random.default_rng(6)
    gm = orc.make_model("standard", gen["T"], gen["sig"], gen["w"], gen["mu"], gen["mu"].copy(), 0.0)
    ids, feats, _ = orc.sample_utterances(gm, n_utts, 1, (FR_UTT, FR_UTT), 0.3, rng)
    sub = orc.make_model("standard", gm.T[:comp_sample], gm.Sigma[:comp_sample], gen["w"][:comp_sample],
                         gen["mu"][:comp_sample], gen["mu"][:comp_sample].copy(), 0.0)
    t0 = time.perf_counter()
    ws = orc.workspace(sub)
    t_ws = (time.perf_counter() - t0) * C / comp_sample
    reps = -(-C // comp_sample)
    for k in ("W", "U", "Sinv", "logdet"):
        setattr(ws, k, np.concatenate([getattr(ws, k)] * reps)[:C])
    pc = orc.predictive_covariances(gm)
    diag = (gen["w"], gen["mu"], np.ascontiguousarray(np.diagonal(pc, axis1=1, axis2=2)))
    t0 = time.perf_counter()
    for u in ids:
        off, comp, w = orc.align(diag, (gen["w"], gen["mu"], pc), feats[u], K_TOP, PRUNE)
        n, f, S = orc.bw_stats(feats[u], off, comp, w, C, center=gm.bias)
        orc.posterior(gm, n, f, S, ws)
    t_utt = (time.perf_counter() - t0) / n_utts
    n_glob = 150000
    sec = t_ws + n_glob * t_utt
    return {"value": n_glob / sec, "unit": "utterances/s", "cores": len(os.sched_getaffinity(0)), "kind": "port",
            "sample": f"{n_utts} utterances (align + BW stats + posterior) and the workspace on {comp_sample} of "
                      f"{C} components, oracle restatement of tvkit.extract_corpus, extrapolated to 150k utterances",
            "parts_s": {"workspace": t_ws, "per_utt": t_utt}}


def selection_exactness(x, dtab, n, pkg):
    """tcgen05 3xFP16 preselection vs the FP64 DMMA kernel on n bench frames (identical indices
    required), and vs the oracle's stable argsort on a 2000-frame sample (outside the timed region)."""
    import torch
    from paper_1906_08556_b200 import _lib
    from oracle import tvkit_oracle as orc
    n = min(n, x.shape[0])
    out = {}
    for mode in ("tc", "dmma"):
        os.environ["TVK_SELECT"] = mode
        sel = _lib.empty((n, K_TOP), torch.int32)
        _lib.call("tvk_select_topk", _lib.ptr(x), 0, n, F, _lib.ptr(dtab.table), C, K_TOP, _lib.ptr(sel), None,
                  _lib.stream())
        out[mode] = sel
    os.environ.pop("TVK_SELECT", None)
    mism = int((out["tc"] != out["dmma"]).any(dim=1).sum().item())
    w, mu, cov = make_ubm(0)
    xs = x[:2000].double().cpu().numpy()
    ll = orc.diag_loglik(w, mu, np.ascontiguousarray(np.diagonal(cov, axis1=1, axis2=2)), xs)
    ref = np.argsort(-ll, axis=1, kind="stable")[:, :K_TOP]
    omism = int((out["tc"][:2000].cpu().numpy() != ref).any(axis=1).sum())
    return {"frames": n, "mismatched_frames_vs_fp64_dmma": mism, "oracle_sample_frames": 2000,
            "mismatched_frames_vs_oracle_stable_argsort": omism,
            "margin": "kappa = 2^-14 (proof: csrc/select_tc.cu header; DESIGN.md §2)"}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=FRAMES_PER_GPU)
    ap.add_argument("--em-utts", type=int, default=20000, help="config 3: utterances (global, sharded)")
    ap.add_argument("--em-steps", type=int, default=3)
    ap.add_argument("--em-warmup", type=int, default=1)
    ap.add_argument("--c5-utts", type=int, default=20000, help="config 5 training utterances (global)")
    ap.add_argument("--extract-utts", type=int, default=150000, help="config 5 extraction utterances (global)")
    ap.add_argument("--config4-utts", type=int, default=0, help="config 4 (opt-in): 1100000 utterances")
    ap.add_argument("--no-config1", dest="config1", action="store_false",
                    help="skip the config-1 end-to-end training leg (and its host reference run)")
    ap.add_argument("--exact-frames", type=int, default=2_000_000,
                    help="frames of the tcgen05-vs-FP64 preselection identity check")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (one GPU per rank) or gloo (test: ranks may share a GPU)")
    ap.add_argument("--no-em", action="store_true")
    ap.add_argument("--dense-steps", type=int, default=1, help="steps of the dense quadratic-feature variant")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-frames", type=int, default=4000)
    ap.add_argument("--ref-frames", type=int, default=2000)
    args = ap.parse_args()
    if args.no_em:
        args.em_utts = args.c5_utts = args.extract_utts = args.config4_utts = 0
    if args.warmup < 3 and args.impl == "ours":
        log("note: fewer than 3 warm-up steps")
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
