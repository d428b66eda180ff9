"""Device-resident building blocks shared by the API functions and the corpus drivers.

Every function here takes/returns torch CUDA tensors and calls libtvk; shapes
follow the reference (C components, F feature dims, D latent dims).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream


def _f64(a):
    return _lib.to_dev(a, torch.float64)


class DiagTable:
    """(2F+1) x C coefficient table of a diagonal GMM (gmm.py:56-67), followed in the same device
    buffer by the tensor-core operands of the top-K preselection (``tvk_diag_table_bytes``)."""

    def __init__(self, weights, means, variances):
        w, mu, var = _f64(weights), _f64(means), _f64(variances)
        self.C, self.F = mu.shape
        nbytes = int(_lib.load().tvk_diag_table_bytes(self.C, self.F))
        self.buf = _lib.empty(((nbytes + 7) // 8,))
        self.table = self.buf[: (2 * self.F + 1) * self.C].view(2 * self.F + 1, self.C)
        call("tvk_diag_table", ptr(w), ptr(mu), ptr(var), self.C, self.F, ptr(self.buf), stream())


class FullTable:
    """Device tables of a full-covariance GMM (gmm.py:106-119): the per-component precision table
    used by the grouped (default) path and, on demand, the Q x C quadratic-feature table used by
    the dense path and the dense T x C log-likelihood API."""

    def __init__(self, weights, means, covariances):
        self._w, self._mu, self._cov = _f64(weights), _f64(means), _f64(covariances)
        self.C, self.F = self._mu.shape
        stride = int(_lib.load().tvk_precision_table_stride(self.F))
        self.prec = _lib.empty((self.C, stride))
        self.status = _lib.empty((self.C,), torch.int32)
        call("tvk_precision_table", ptr(self._w), ptr(self._mu), ptr(self._cov), self.C, self.F, ptr(self.prec),
             ptr(self.status), stream())
        self._quad = None

    @property
    def table(self):
        """Q x C quadratic-feature table (built on first use)."""
        if self._quad is None:
            q = 1 + self.F + self.F * (self.F + 1) // 2
            self._quad = _lib.empty((q, self.C))
            st = _lib.empty((self.C,), torch.int32)
            call("tvk_full_table", ptr(self._w), ptr(self._mu), ptr(self._cov), self.C, self.F, ptr(self._quad),
                 ptr(st), stream())
        return self._quad

    def bad_components(self):
        return np.flatnonzero(_lib.to_host(self.status) != _lib.ITEM_OK)


def frames_to_device(features):
    """Frames as a device matrix; float32 stays float32 (exact in f64), anything else f64."""
    if isinstance(features, torch.Tensor):
        x = features
        if x.dtype not in (torch.float32, torch.float64):
            x = x.to(torch.float64)
        return x.to(_lib.device(), non_blocking=True).contiguous()
    arr = np.asarray(features)
    if arr.dtype != np.float32:
        arr = arr.astype(np.float64, copy=False)
    return _lib.to_dev(np.atleast_2d(arr), torch.float32 if arr.dtype == np.float32 else torch.float64)


def dense_loglik(x, table, kind):
    """T x C log-likelihoods = features(x) . table (kind 0 diag, 1 full)."""
    T, F = x.shape
    q, C = table.shape
    feats = _lib.empty((T, q))
    xp, xf = _lib.x_args(x)
    call("tvk_frame_features", xp, xf, T, F, kind, ptr(feats), stream())
    out = _lib.empty((T, C))
    _lib.dgemm(feats, table, out, T, C, q)
    return out


def select_topk(x, diag_tab, k, values=False):
    T, F = x.shape
    sel = _lib.empty((T, k), torch.int32)
    val = _lib.empty((T, k)) if values else None
    xp, xf = _lib.x_args(x)
    call("tvk_select_topk", xp, xf, T, F, ptr(diag_tab.table), diag_tab.C, k, ptr(sel), ptr(val), stream())
    return sel, val


class AlignResult:
    """Device CSR alignment of a frame batch."""

    def __init__(self, offsets, components, weights, n_entries):
        self.offsets = offsets
        self.components = components
        self.weights = weights
        self.n_entries = n_entries


ALIGN_DENSE = 1  # TVK_ALIGN_DENSE
DEFAULT_DENSE = os.environ.get("TVK_ALIGN_MODE", "grouped") == "dense"


def align(x, diag_tab, full_tab, top_k, prune, debug=False, sync_count=True, dense=None):
    """Frame posteriors for a device frame matrix (gmm.py:389-439), all on device.

    ``dense`` selects the dense quadratic-feature GEMM over all C components (the reference's
    own work, gmm.py:412) instead of the grouped evaluation of the K selected ones; both give
    the same alignment (see tests/test_gpu_align.py).
    """
    if dense is None:
        dense = DEFAULT_DENSE
    T, F = x.shape
    C = diag_tab.C
    k = min(top_k, C)
    if k > 32 and T * k > WIDE_PAIRS and not debug:
        # wide top_k: bound the (T x k) workspace by aligning frame chunks and joining the CSRs
        step = max(1, WIDE_PAIRS // k)
        parts = [align(x[i:i + step], diag_tab, full_tab, k, prune, dense=dense) for i in range(0, T, step)]
        bases = np.cumsum([0] + [p.n_entries for p in parts])
        offsets = torch.cat([p.offsets[:-1] + int(b) for p, b in zip(parts, bases[:-1])] +
                            [torch.tensor([int(bases[-1])], dtype=torch.int64, device=x.device)])
        comps = torch.cat([p.components[:p.n_entries] for p in parts])
        wts = torch.cat([p.weights[:p.n_entries] for p in parts])
        return AlignResult(offsets, comps, wts, int(bases[-1]))
    offsets = _lib.empty((T + 1,), torch.int64)
    comps = _lib.empty((max(T * k, 1),), torch.int32)
    wts = _lib.empty((max(T * k, 1),), torch.float32)
    ws_bytes = int(_lib.load().tvk_align_workspace_bytes(T, k, C))
    ws = _lib.empty((max(ws_bytes, 1),), torch.uint8)
    sel = _lib.empty((T, k), torch.int32) if debug else None
    sll = _lib.empty((T, k)) if debug else None
    xp, xf = _lib.x_args(x)
    quad = ptr(full_tab.table) if dense else None
    call("tvk_align_frames", xp, xf, T, F, ptr(diag_tab.table), quad, ptr(full_tab.prec), C, k, float(prune),
         ALIGN_DENSE if dense else 0, ptr(ws), ws_bytes, ptr(offsets), ptr(comps), ptr(wts), ptr(sel), ptr(sll),
         stream())
    n = int(offsets[T].item()) if sync_count else None
    res = AlignResult(offsets, comps, wts, n)
    if debug:
        res.selected, res.sel_ll = sel, sll
    return res


STREAM_CHUNK = 1 << 19  # frames per chunk of the host-input alignment pipeline
WIDE_PAIRS = 1 << 24    # (frame, component) pairs per align() call / host piece when top_k > 32
N_SLOTS = 4             # pinned result staging slots = pieces whose host unstaging may run concurrently
RAMP_PIECE = 1 << 17    # first / last pieces of the host pipeline (only their copies cannot overlap)
_staging = {}             # (chunk, k) -> pinned host staging slots, reused across calls
_copier = None


def _pinned_slots(chunk, k):
    key = (chunk, k)
    if key not in _staging:
        _staging.clear()
        _staging[key] = [(torch.empty(chunk + 1, dtype=torch.int64, pin_memory=True),
                          torch.empty(chunk * k, dtype=torch.int32, pin_memory=True),
                          torch.empty(chunk * k, dtype=torch.float32, pin_memory=True)) for _ in range(N_SLOTS)]
    return _staging[key]


def align_host(features, diag_tab, full_tab, top_k, prune, chunk=STREAM_CHUNK, tables=None):
    """Frame posteriors of HOST frames with every copy overlapped (align_frames' host path).

    The frames are cut into ``chunk``-frame pieces.  Piece i+1's host->device copy (copy stream),
    piece i's alignment kernels (compute stream), piece i-1's device->host copy of its CSR into
    pinned staging (drain stream) and piece i-2's copy from staging into the returned arrays (a
    host worker thread) all run concurrently.  Returns host (offsets, components, weights).

    ``tables``: instead of ``diag_tab`` / ``full_tab``, a callable returning them that is run once
    the first piece's host->device copy is queued, so the model upload and table builds (and their
    checks) overlap that copy; ``top_k`` must then already be at most C.
    """
    global _copier
    import concurrent.futures as cf
    T, F = features.shape
    if isinstance(features, torch.Tensor):
        host = features if features.dtype in (torch.float32, torch.float64) else features.to(torch.float64)
    else:
        arr = np.asarray(features)
        if arr.dtype != np.float32:
            arr = arr.astype(np.float64, copy=False)
        host = torch.from_numpy(np.ascontiguousarray(arr))
    host = host.contiguous()
    k = min(top_k, diag_tab.C) if tables is None else top_k
    chunk = min(chunk, T, max(1, WIDE_PAIRS // k))
    offsets = np.empty(T + 1, np.int64)
    comps = np.empty(T * k, np.int32)   # untouched capacity is never paged in
    wts = np.empty(T * k, np.float32)
    offsets[0] = 0
    if _copier is None:
        # first-touch page faults of the returned arrays dominate the unstaging: run pieces in parallel
        _copier = cf.ThreadPoolExecutor(max_workers=N_SLOTS, thread_name_prefix="tvk-copy")
    slots = _pinned_slots(chunk, k)
    slot_busy = [None] * N_SLOTS
    comp_stream = torch.cuda.current_stream()
    copy_stream, drain_stream = torch.cuda.Stream(), torch.cuda.Stream()
    bufs = [_lib.empty((chunk, F), host.dtype) for _ in range(2)]
    free = [None, None]
    pending = None
    base = 0

    def unstage(lo, n, e, base, st, ev):
        ev.synchronize()
        off_st, c_st, w_st = st
        np.add(off_st[1:n + 1].numpy(), base, out=offsets[lo + 1:lo + n + 1])
        comps[base:base + e] = c_st[:e].numpy()
        wts[base:base + e] = w_st[:e].numpy()

    def drain(item, base, slot):
        lo, n, res, done = item
        if slot_busy[slot] is not None:
            slot_busy[slot].result()  # staging slot free again
        st = slots[slot]
        with torch.cuda.stream(drain_stream):
            drain_stream.wait_event(done)
            # the piece's outputs were allocated on the compute stream: keep the caching allocator
            # from handing their memory to a later piece until these copies have run
            for t in (res.offsets, res.components, res.weights):
                t.record_stream(drain_stream)
            st[0][:n + 1].copy_(res.offsets, non_blocking=True)
            got = torch.cuda.Event()
            got.record(drain_stream)
            got.synchronize()
            e = int(st[0][n])
            st[1][:e].copy_(res.components[:e], non_blocking=True)
            st[2][:e].copy_(res.weights[:e], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(drain_stream)
        slot_busy[slot] = _copier.submit(unstage, lo, n, e, base, st, ev)
        return base + e

    # piece sizes ramp up and down (chunk/4, chunk/2, chunk, ..., chunk/2, chunk/4) so that the first
    # host->device copy and the last copy-out, which cannot overlap anything, are short
    sizes, rest, q = [], T, max(1, min(chunk // 4, RAMP_PIECE))
    for c in (q, 2 * q):
        if rest > 0:
            sizes.append(min(c, rest))
            rest -= sizes[-1]
    tail = []
    for c in (q, 2 * q):
        if rest > 4 * chunk:
            tail.insert(0, c)
            rest -= c
    while rest > 0:
        sizes.append(min(chunk, rest))
        rest -= sizes[-1]
    sizes += tail
    nd = 0
    lo = 0
    for i, n in enumerate(sizes):
        buf = bufs[i % 2][:n]
        with torch.cuda.stream(copy_stream):
            if free[i % 2] is not None:
                copy_stream.wait_event(free[i % 2])
            buf.copy_(host[lo:lo + n], non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(copy_stream)
        if i == 0 and tables is not None:
            try:
                diag_tab, full_tab = tables()
            except BaseException:
                copy_stream.synchronize()  # the queued copy still writes into bufs: let it land first
                raise
        comp_stream.wait_event(copied)
        res = align(buf, diag_tab, full_tab, k, prune, sync_count=False)
        done = torch.cuda.Event()
        done.record(comp_stream)
        free[i % 2] = done
        if pending is not None:
            base = drain(pending, base, nd % N_SLOTS)
            nd += 1
        pending = (lo, n, res, done)
        lo += n
    if pending is not None:
        base = drain(pending, base, nd % N_SLOTS)
    for f in slot_busy:
        if f is not None:
            f.result()
    torch.cuda.current_stream().wait_stream(drain_stream)
    return offsets, comps[:base], wts[:base]


def bw_stats(x, utt_frames, ali_offsets, comps, wts, C, center=None, want_S=False, ssum_acc=None,
             entry_capacity=None):
    """Per-utterance n (U x C), f (U x C x F) [, S (U x C x F x F)] on device (gmm.py:442-492).

    ``utt_frames`` (U+1, int64 device) delimits utterances in ``x``; the alignment CSR covers
    the same frames.  ``ssum_acc`` (C x F x F) is added to in place when given.
    """
    F = x.shape[1]
    U = utt_frames.shape[0] - 1
    if entry_capacity is None:
        entry_capacity = comps.shape[0]
    n = _lib.empty((U, C))
    f = _lib.empty((U, C, F))
    S = _lib.empty((U, C, F, F)) if want_S else None
    ws_bytes = int(_lib.load().tvk_bw_workspace_bytes(entry_capacity, U, C))
    ws = _lib.empty((max(ws_bytes, 1),), torch.uint8)
    xp, xf = _lib.x_args(x)
    call("tvk_bw_stats", xp, xf, F, ptr(utt_frames), U, ptr(ali_offsets), ptr(comps), ptr(wts), C, ptr(center),
         ptr(n), ptr(f), ptr(S), ptr(ssum_acc), int(entry_capacity), ptr(ws), ws_bytes, stream())
    return n, f, S


# ---------------------------------------------------------------------------- UBM EM training

EM_CHUNK_ELEMS = 1 << 27  # doubles in each per-chunk T x max(C, Q) buffer (1 GiB)


def seed_means(x, frames, n_components, rng):
    """k-means++-style seeding (_seed_means, gmm.py:228-243).

    The whole draw loop runs on the device (``tvk_seed_means``): distance updates bit-identical
    to numpy, inverse-CDF draws against uniforms taken from the caller's Generator up front (one
    ``rng.random()`` per ``rng.choice``, exactly what the reference consumes).  If the device
    stops early (all distances zero -> the reference's ``rng.integers`` branch, or non-finite
    distances -> ``rng.choice``'s ValueError) the random stream is rewound and the remaining
    draws follow the reference step by step on the host.
    """
    T, F = x.shape
    C = n_components
    chosen = np.empty((C, F))
    first = int(rng.integers(T))
    chosen[0] = frames[first]
    if C == 1:
        return chosen
    state = rng.bit_generator.state
    u = _lib.to_dev(rng.random(C - 1))
    idx = _lib.empty((C,), torch.int64)
    idx[:1].fill_(first)
    dist2 = _lib.empty((T,))
    stop = _lib.empty((2,), torch.int32)
    ws_bytes = int(_lib.load().tvk_seed_workspace_bytes(T))
    ws = _lib.empty((ws_bytes // 8,))
    xp, xf = _lib.x_args(x)
    call("tvk_seed_means", xp, xf, T, F, C, ptr(u), ptr(idx), ptr(dist2), ptr(stop), ptr(ws), ws_bytes, stream())
    idx_h, stop_h = _lib.to_host(idx), _lib.to_host(stop)
    s = int(stop_h[0])
    if s == 0:
        chosen[1:] = frames[idx_h[1:]]
        return chosen
    chosen[1:s] = frames[idx_h[1:s]]
    rng.bit_generator.state = state
    if s > 1:
        rng.random(s - 1)
    _seed_host_steps(x, frames, chosen, dist2, s, rng)
    return chosen


def _seed_host_steps(x, frames, chosen, dist2, start, rng):
    """Steps ``start..C-1`` of _seed_means with the draws on the host (gmm.py:235-242)."""
    T, F = x.shape
    xp, xf = _lib.x_args(x)
    center = _lib.empty((F,))
    host = torch.empty((T,), dtype=torch.float64, pin_memory=True)
    for c in range(start, chosen.shape[0]):
        host.copy_(dist2)
        d = host.numpy()
        total = d.sum()
        if total <= 0:
            chosen[c] = frames[rng.integers(T)]
            continue
        chosen[c] = frames[rng.choice(T, p=d / total)]
        center.copy_(torch.from_numpy(chosen[c]))
        call("tvk_seed_dist2", xp, xf, T, F, ptr(center), ptr(dist2), 0, stream())


class EmEStep:
    """GMM E-step over a device frame matrix (gmm.py:283-292 diagonal, 344-349 full).

    Per chunk of frames: features (kind 0 ``[x^2, x, 1]``, kind 1 ``[1, x_i, x_i x_j]``) ->
    log-likelihoods as one DMMA GEMM against the model's coefficient table -> row softmax
    (responsibilities in place, log-normalisers out) -> one ``resp^T x features`` GEMM that
    accumulates every sufficient statistic at once (C x Q: occupancy, first and second
    moments).  The total log-likelihood is a fixed-order device reduction of the normalisers.
    """

    def __init__(self, x, kind, C):
        self.x = x
        self.T, self.F = x.shape
        F = self.F
        self.kind, self.C = kind, C
        self.q = 2 * F + 1 if kind == 0 else 1 + F + F * (F + 1) // 2
        self.rows = int(max(256, min(self.T, EM_CHUNK_ELEMS // max(C, self.q))))
        self.feats = _lib.empty((self.rows, self.q))
        self.ll = _lib.empty((self.rows, C))
        self.norm = _lib.empty((self.rows,))
        self.stats = _lib.empty((C, self.q))
        self.total = _lib.empty((1,))
        self.dot_ws = _lib.empty((max(int(_lib.load().tvk_ddot_workspace_bytes()) // 8, 1),))
        tiles = -(-C // 128) * -(-self.q // 128)
        self.splits = int(max(1, min(32, (2 * 148) // tiles, self.rows // 1024)))
        self.work = _lib.empty((self.splits * C * self.q,)) if self.splits > 1 else None

    def run(self, table):
        """Accumulate the statistics for the model whose table is ``table``; returns (stats, total)."""
        T, F, C, q = self.T, self.F, self.C, self.q
        for lo in range(0, T, self.rows):
            n = min(self.rows, T - lo)
            xp, xf = _lib.x_args(self.x[lo:lo + n])
            feats, ll = self.feats[:n], self.ll[:n]
            call("tvk_frame_features", xp, xf, n, F, self.kind, ptr(feats), stream())
            _lib.dgemm(feats, table, ll, n, C, q)
            call("tvk_row_softmax", ptr(ll), n, C, ptr(self.norm), stream())
            beta = 0.0 if lo == 0 else 1.0
            call("tvk_ddot", ptr(self.norm), None, n, 1.0, beta, ptr(self.total), ptr(self.dot_ws), stream())
            splits = self.splits if n >= 1024 * self.splits else 1
            _lib.dgemm(ll, feats, self.stats, C, q, n, trans_a=True, beta=beta, splits=splits,
                       work=self.work if splits > 1 else None)
        return self.stats, self.total


def full_moments(stats, mean_old, C, F, occ_min=1.0):
    """(mean, S2, s1 s1^T/occ, N (0 when starved), trace) from a kind-1 statistics matrix."""
    mean = _lib.empty((C, F))
    s2 = _lib.empty((C, F, F))
    tb = _lib.empty((C, F, F))
    n = _lib.empty((C,))
    tr = _lib.empty((C,))
    call("tvk_full_moments", ptr(stats), C, F, float(occ_min), ptr(mean_old), ptr(mean), ptr(s2), ptr(tb), ptr(n),
         ptr(tr), stream())
    return mean, s2, tb, n, tr


def sigma_floor(s2, tb, n, sigma_old, C, F, floor_scale):
    out = _lib.empty((C, F, F))
    status = _lib.empty((C,), torch.int32)
    call("tvk_sigma_floor", ptr(s2), ptr(tb), ptr(n), ptr(sigma_old), C, F, float(floor_scale), ptr(out),
         ptr(status), stream())
    return out, status


def spd_status(a, C, F):
    status = _lib.empty((C,), torch.int32)
    call("tvk_spd_small", ptr(a), C, F, None, None, None, ptr(status), stream())
    return status
