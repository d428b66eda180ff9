"""Corpus drivers on the B200: alignment, E-step accumulation, extraction, EM training.

Drop-in for the hot-path drivers of the reference ``tvkit.pipeline`` (pipeline.py:364-655):
``align_corpus``, ``accumulate_corpus``, ``extract_corpus``, ``train_extractor`` with
``TrainConfig``, feature stores, run metrics and checkpoint/resume.  Instead of the
reference's thread pool over per-utterance numpy calls, each driver moves the (rank's
share of the) corpus into HBM once and runs device batches:

    frames (T x F) --align--> CSR (offsets, comps, f32 weights)          [no collective]
    per batch of 1024 utts: BW stats -> L/b GEMMs -> Cholesky/inverse -> A/B GEMMs
    one all-reduce of the flat accumulator per iteration (multi-GPU), then the M-step
    (replicated on every rank; identical inputs give identical outputs).

``workers`` only parallelizes host-side feature loading; results do not depend on it.
Everything is deterministic for a fixed GPU count (fixed-order reductions, no atomics).
"""

from __future__ import annotations

import hashlib
import logging
import os
import time
import warnings
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field, fields, replace

import numpy as np
import torch

from . import _device, _dist, _estep, _lib
from . import gmm
from .gmm import GmmDiag, GmmFull, SparseAlignment
from .io_formats import load_model, read_alignment, read_matrix, save_model, write_alignment, write_matrix
from .tvm import (AUGMENTED, DEFAULT_PRIOR_OFFSET, SIGMA_FLOOR_SCALE, STANDARD, EmAccumulators, TvModel,
                  _raise_collapsed, _warn_singular, compute_min_div, init_model)

logger = logging.getLogger(__name__)

ALIGN_CHUNK_FRAMES = 1 << 21  # frames per device alignment launch
ENTRY_CAPACITY_PER_FRAME = 8  # initial corpus CSR capacity (entries per frame; grows on demand)


class PipelineError(RuntimeError):
    """A training or extraction run could not complete."""


# ----------------------------------------------------------------------------- feature stores


class DirectoryFeatureStore:
    """Features as one ``<utterance id>.fmx`` matrix file per utterance (pipeline.py:60-78)."""

    def __init__(self, root):
        self.root = root
        self._ids = sorted(n[:-4] for n in os.listdir(root) if n.endswith(".fmx"))
        if not self._ids:
            raise PipelineError(f"no .fmx feature files under {root}")

    def ids(self):
        return list(self._ids)

    def load(self, utt_id):
        path = os.path.join(self.root, f"{utt_id}.fmx")
        if not os.path.exists(path):
            raise KeyError(f"missing features for utterance {utt_id!r}")
        return read_matrix(path)


class InMemoryFeatureStore:
    """Features from a {utterance id: (T, F) array} mapping (pipeline.py:81-94)."""

    def __init__(self, mapping):
        self._mapping = dict(mapping)

    def ids(self):
        return sorted(self._mapping)

    def load(self, utt_id):
        try:
            return self._mapping[utt_id]
        except KeyError:
            raise KeyError(f"missing features for utterance {utt_id!r}") from None


# ----------------------------------------------------------------------------- host batch pool


def _map_batches(batches, fn, workers, deterministic):
    """Yield ``(index, fn(batch))`` over a bounded pool of host threads (pipeline.py:279-350).

    With ``deterministic`` results come out in batch order, otherwise in completion order; at most
    ``2 * workers`` batches are submitted ahead of the consumer.  The GPU drivers do not run their
    arithmetic through it (device batching replaces it); it remains for host-side
    work such as feature loading.  A failing batch stops the pool and raises ``PipelineError``.
    """
    import concurrent.futures as cf

    n = len(batches)
    if workers <= 1 or n <= 1:
        for i in range(n):
            yield i, fn(batches[i])
        return
    window = 2 * workers
    with cf.ThreadPoolExecutor(max_workers=workers) as pool:
        live = {}
        nxt = 0

        def refill():
            nonlocal nxt
            while nxt < n and len(live) < window:
                live[pool.submit(fn, batches[nxt])] = nxt
                nxt += 1

        def result(fut):
            try:
                return fut.result()
            except Exception as exc:
                for f in live:
                    f.cancel()
                raise PipelineError("a loader worker failed") from exc

        refill()
        if deterministic:
            order = {i: f for f, i in live.items()}
            for i in range(n):
                fut = order.pop(i)
                payload = result(fut)
                del live[fut]
                yield i, payload
                refill()
                order.update({j: f for f, j in live.items() if j not in order})
        else:
            while live:
                done, _ = cf.wait(list(live), return_when=cf.FIRST_COMPLETED)
                for fut in sorted(done, key=live.get):
                    payload = result(fut)
                    i = live.pop(fut)
                    yield i, payload
                refill()


# ----------------------------------------------------------------------------- configuration

_TRUE = {"true", "1", "yes"}
_FALSE = {"false", "0", "no"}


@dataclass
class TrainConfig:
    """Knobs of one extractor training run; flat ``key = value`` file (pipeline.py:105-209)."""

    formulation: str = AUGMENTED
    latent_dim: int = 400
    iterations: int = 22
    min_div: bool = True
    sigma_update: bool = True
    update_mean: bool = False
    realign_interval: int = 0
    top_k: int = 20
    prune: float = 0.025
    prior_offset: float = DEFAULT_PRIOR_OFFSET
    seeds: tuple = (0, 1, 2, 3, 4)
    batch_size_utts: int = 8
    workers: int = 1
    deterministic: bool = True

    def validate(self):
        checks = [
            (self.formulation in (STANDARD, AUGMENTED), f"unknown formulation {self.formulation!r}"),
            (self.iterations >= 1, "iterations must be >= 1"),
            (self.realign_interval >= 0, "realign_interval must be >= 0"),
            (bool(self.seeds), "at least one seed is required"),
            (self.latent_dim >= 1 and not (self.formulation == AUGMENTED and self.latent_dim < 2),
             "latent_dim too small for the formulation"),
            (self.top_k >= 1, "top_k must be >= 1"),
            (0.0 <= self.prune < 1.0, "prune must be in [0, 1)"),
            (self.batch_size_utts >= 1 and self.workers >= 1, "batch_size_utts and workers must be >= 1"),
            (not (self.update_mean and self.formulation != STANDARD),
             "update_mean applies to the standard formulation only"),
            (not (self.update_mean and not self.min_div), "update_mean requires min_div"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)
        if self.update_mean and self.sigma_update:
            warnings.warn("bias updates combined with residual covariance updates are known to train poorly",
                          RuntimeWarning, stacklevel=2)

    def to_text(self):
        out = []
        for f in fields(self):
            v = getattr(self, f.name)
            if f.name == "seeds":
                v = ",".join(str(s) for s in v)
            elif isinstance(v, bool):
                v = "true" if v else "false"
            out.append(f"{f.name} = {v}")
        return "\n".join(out) + "\n"

    def save(self, path):
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(self.to_text())

    @classmethod
    def load(cls, path):
        with open(path, encoding="utf-8") as fh:
            return cls.from_text(fh.read())

    @classmethod
    def from_text(cls, text):
        kinds = {f.name: type(getattr(cls(), f.name)) for f in fields(cls)}
        kw = {}
        for no, raw in enumerate(text.splitlines(), 1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ValueError(f"line {no}: expected 'key = value'")
            key, value = (p.strip() for p in line.split("=", 1))
            if key not in kinds:
                raise ValueError(f"line {no}: unknown config key {key!r}")
            kw[key] = _parse(kinds[key], value, key)
        return cls(**kw)

    def config_hash(self):
        return hashlib.sha256(self.to_text().encode("utf-8")).hexdigest()[:16]

    def with_seed(self, seed):
        return replace(self, seeds=(seed,))


def _parse(kind, value, key):
    if kind is tuple:
        return tuple(int(p) for p in value.split(",") if p.strip())
    if kind is bool:
        v = value.lower()
        if v in _TRUE:
            return True
        if v in _FALSE:
            return False
        raise ValueError(f"{key}: expected a boolean, got {value!r}")
    if kind is float:
        return float(value)
    if kind is int:
        return int(value)
    return value


# ----------------------------------------------------------------------------- run metrics


@dataclass
class IterationRecord:
    seed: int
    iteration: int
    aux: float
    eer: float = float("nan")
    wall_seconds: float = 0.0


@dataclass
class RunMetrics:
    """Per-iteration records across seeds plus the seed-averaged series (pipeline.py:225-268)."""

    records: list = field(default_factory=list)
    complete: bool = True

    def seeds(self):
        return sorted({r.seed for r in self.records})

    def series(self, seed):
        return sorted((r for r in self.records if r.seed == seed), key=lambda r: r.iteration)

    def averaged(self):
        by_iter = {}
        for r in self.records:
            by_iter.setdefault(r.iteration, []).append(r)
        out = []
        for it in sorted(by_iter):
            rows = by_iter[it]
            eers = [r.eer for r in rows]
            eer = float(np.mean(eers)) if not any(np.isnan(e) for e in eers) else float("nan")
            out.append(IterationRecord(-1, it, float(np.mean([r.aux for r in rows])), eer,
                                       float(np.mean([r.wall_seconds for r in rows]))))
        return out

    def write_csv(self, path):
        with open(path, "w", encoding="utf-8") as fh:
            fh.write("seed,iteration,aux,eer,wall_seconds\n")
            for seed in self.seeds():
                for r in self.series(seed):
                    fh.write(f"{seed},{r.iteration},{r.aux!r},{r.eer!r},{r.wall_seconds!r}\n")
            for r in self.averaged():
                fh.write(f"avg,{r.iteration},{r.aux!r},{r.eer!r},{r.wall_seconds!r}\n")


# ----------------------------------------------------------------------------- device corpus


STAGE_BYTES = 64 << 20  # pinned staging buffer size of the corpus upload (two buffers)
_corpus_stage = []


def _stream_to_device(mats, n_frames, dim, dtype):
    """Upload a list of (T_u, F) host matrices into one device (n_frames, F) tensor through two
    reused pinned staging buffers (copy stream, double-buffered), so the host never holds a
    concatenated or pinned copy of the whole shard (host memory stays ~1x the corpus)."""
    tdt = torch.float32 if dtype == np.float32 else torch.float64
    esize = np.dtype(dtype).itemsize
    x = _lib.empty((n_frames, dim), tdt)
    rows_per = max(1, STAGE_BYTES // (dim * esize))
    if not _corpus_stage:
        _corpus_stage.extend(torch.empty(STAGE_BYTES, dtype=torch.uint8, pin_memory=True) for _ in range(2))
    copy_stream = torch.cuda.Stream()
    copy_stream.wait_stream(torch.cuda.current_stream())  # x allocated on the current stream
    done = [None, None]
    b, fill, row0 = 0, 0, 0
    view = None

    def flush():
        nonlocal b, fill, row0
        with torch.cuda.stream(copy_stream):
            x[row0:row0 + fill].copy_(view[:fill], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        done[b] = ev
        row0 += fill
        fill = 0
        b ^= 1

    for m in mats:
        m = m.reshape(-1, dim)
        pos = 0
        while pos < m.shape[0]:
            if fill == 0:
                if done[b] is not None:
                    done[b].synchronize()  # this staging buffer's previous copy has landed
                view = torch.from_numpy(_corpus_stage[b].numpy()[: rows_per * dim * esize].view(dtype)).view(rows_per, dim)
            n = min(rows_per - fill, m.shape[0] - pos)
            view.numpy()[fill:fill + n] = m[pos:pos + n]
            fill += n
            pos += n
            if fill == rows_per:
                flush()
    if fill:
        flush()
    for ev in done:  # the staging buffers are reused by the next upload
        if ev is not None:
            ev.synchronize()
    torch.cuda.current_stream().wait_stream(copy_stream)
    x.record_stream(copy_stream)
    return x


class DeviceCorpus:
    """The (rank's share of the) corpus resident in HBM: concatenated frames + utterance bounds."""

    def __init__(self, store, ids, workers=1):
        self.ids = list(ids)
        if workers > 1 and len(self.ids) > 1:
            with ThreadPoolExecutor(workers) as ex:
                mats = list(ex.map(lambda u: np.atleast_2d(np.asarray(store.load(u))), self.ids))
        else:
            mats = [np.atleast_2d(np.asarray(store.load(u))) for u in self.ids]
        lens = np.array([m.shape[0] for m in mats], dtype=np.int64)
        self.dim = mats[0].shape[1] if mats else 0
        for m in mats:
            if m.shape[0] and m.shape[1] != self.dim:
                raise PipelineError("utterances disagree on the feature dimension")
        dtype = np.float32 if all(m.dtype == np.float32 for m in mats) else np.float64
        self.n_frames = int(lens.sum())
        self.x = _stream_to_device(mats, self.n_frames, self.dim, dtype) if self.n_frames else \
            _lib.empty((0, max(self.dim, 1)), torch.float32 if dtype == np.float32 else torch.float64)
        self.utt_frames_host = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        self.utt_frames = _lib.to_dev(self.utt_frames_host, torch.int64)

    @classmethod
    def from_device(cls, x, utt_frames_host, ids):
        self = cls.__new__(cls)
        self.ids = list(ids)
        self.x = x
        self.dim = x.shape[1]
        self.n_frames = x.shape[0]
        self.utt_frames_host = np.asarray(utt_frames_host, dtype=np.int64)
        self.utt_frames = _lib.to_dev(self.utt_frames_host, torch.int64)
        return self


class DeviceFeatureStore:
    """A feature store whose frames are already resident in HBM: one (T, F) device matrix plus
    utterance bounds (e.g. frames produced on the device, or a corpus loaded once and reused by
    several drivers).  The drivers use its frames in place; ``load`` returns a host copy for
    callers that want one utterance.  ``ids()`` keeps construction order.

    Under torch.distributed a rank may hold only its shard: pass the corpus-wide id list as
    ``global_ids`` (the rank's ``ids`` must be its ``_dist.shard`` of it); the drivers then shard
    ``global_ids`` exactly as they would shard a host store and find every local id resident."""

    def __init__(self, x, utt_frames, ids, global_ids=None):
        self.x = x
        self.utt_frames_host = np.asarray(utt_frames, dtype=np.int64)
        self._ids = list(ids)
        self._global = list(global_ids) if global_ids is not None else None
        self._pos = {u: i for i, u in enumerate(self._ids)}
        if len(self._pos) != len(self._ids) or self.utt_frames_host.shape[0] != len(self._ids) + 1:
            raise ValueError("DeviceFeatureStore: ids must be unique and match the utterance bounds")

    def ids(self):
        return list(self._global if self._global is not None else self._ids)

    def load(self, utt_id):
        try:
            i = self._pos[utt_id]
        except KeyError:
            raise KeyError(f"missing features for utterance {utt_id!r}") from None
        lo, hi = self.utt_frames_host[i], self.utt_frames_host[i + 1]
        return _lib.to_host(self.x[lo:hi])

    def device_corpus(self, ids):
        """DeviceCorpus over ``ids``: a view when they are a contiguous run of the store, else a
        device gather of their frames."""
        try:
            idx = np.array([self._pos[u] for u in ids], dtype=np.int64)
        except KeyError as exc:
            raise KeyError(f"utterance {exc.args[0]!r} is not resident on this rank") from None
        if idx.size and np.all(np.diff(idx) == 1):
            lo, hi = int(idx[0]), int(idx[-1]) + 1
            b = self.utt_frames_host[lo:hi + 1]
            return DeviceCorpus.from_device(self.x[b[0]:b[-1]], b - b[0], ids)
        lens = self.utt_frames_host[idx + 1] - self.utt_frames_host[idx]
        rows = np.concatenate([np.arange(self.utt_frames_host[i], self.utt_frames_host[i + 1]) for i in idx]) \
            if idx.size else np.zeros(0, np.int64)
        x = self.x[_lib.to_dev(rows, torch.int64)] if rows.size else self.x[:0]
        return DeviceCorpus.from_device(x, np.concatenate([[0], np.cumsum(lens)]), ids)


def _device_corpus(store, ids, workers):
    if hasattr(store, "device_corpus"):
        return store.device_corpus(list(ids))
    return DeviceCorpus(store, ids, workers)


class DeviceAlignment:
    """Corpus alignment in device CSR form plus per-utterance entry bounds (host)."""

    def __init__(self, offsets, comps, weights, utt_entries_host):
        self.offsets, self.comps, self.weights = offsets, comps, weights
        self.utt_entries = utt_entries_host

    @classmethod
    def compute(cls, corpus, diag_tab, full_tab, top_k, prune):
        """Align the corpus chunk by chunk into one CSR sized by the entries actually kept.

        The CSR starts at ENTRY_CAPACITY_PER_FRAME entries per frame (prune 0.025 keeps <= 40 by
        construction and ~4.5 on speech-like data) and grows geometrically only if a chunk needs
        more, so HBM holds ~44 B/frame instead of a top_k-sized 8*top_k B/frame.
        """
        T = corpus.n_frames
        k = min(top_k, diag_tab.C)
        gmm._check_envelope(k, diag_tab.F, diag_tab.C, "align_corpus")
        offsets = _lib.empty((T + 1,), torch.int64)
        cap = max(1, min(T * k, int(T * ENTRY_CAPACITY_PER_FRAME)))
        comps = _lib.empty((cap,), torch.int32)
        wts = _lib.empty((cap,), torch.float32)
        offsets[:1].zero_()
        ebase = 0
        for lo in range(0, T, ALIGN_CHUNK_FRAMES):
            hi = min(T, lo + ALIGN_CHUNK_FRAMES)
            res = _device.align(corpus.x[lo:hi], diag_tab, full_tab, k, prune)
            e = res.n_entries
            if ebase + e > cap:  # grow: at least 1.5x, enough for the rest at this chunk's density
                need = ebase + e + int((T - hi) * (e / max(hi - lo, 1)) * 1.1)
                cap = min(T * k, max(need, int(cap * 1.5)))
                comps = torch.cat([comps[:ebase], _lib.empty((cap - ebase,), torch.int32)])
                wts = torch.cat([wts[:ebase], _lib.empty((cap - ebase,), torch.float32)])
            offsets[lo + 1:hi + 1] = res.offsets[1:] + ebase
            comps[ebase:ebase + e] = res.components[:e]
            wts[ebase:ebase + e] = res.weights[:e]
            ebase += e
            del res
        ue = _lib.to_host(offsets[corpus.utt_frames])
        return cls(offsets, comps, wts, ue)

    @classmethod
    def from_host(cls, corpus, alignments):
        offs, comps, wts = [np.zeros(1, np.int64)], [], []
        base = 0
        for u, (lo, hi) in zip(corpus.ids, zip(corpus.utt_frames_host[:-1], corpus.utt_frames_host[1:])):
            try:
                a = alignments[u]
            except KeyError:
                raise KeyError(f"missing alignment for utterance {u!r}") from None
            if a.n_frames != hi - lo:
                raise ValueError("alignment frame count does not match features")
            offs.append(a.offsets[1:] - a.offsets[0] + base)
            comps.append(a.components)
            wts.append(a.weights)
            base += int(a.offsets[-1] - a.offsets[0])
        o = np.concatenate(offs)
        c = np.concatenate(comps) if comps else np.zeros(0, np.int32)
        w = np.concatenate(wts) if wts else np.zeros(0, np.float32)
        return cls(_lib.to_dev(o, torch.int64), _lib.to_dev(c.astype(np.int32), torch.int32),
                   _lib.to_dev(w.astype(np.float32), torch.float32), o[corpus.utt_frames_host])

    def to_host(self, corpus):
        off = _lib.to_host(self.offsets)
        comps = _lib.to_host(self.comps[: int(off[-1])]) if off[-1] else np.zeros(0, np.int32)
        wts = _lib.to_host(self.weights[: int(off[-1])]) if off[-1] else np.zeros(0, np.float32)
        out = {}
        for i, u in enumerate(corpus.ids):
            lo, hi = corpus.utt_frames_host[i], corpus.utt_frames_host[i + 1]
            e0, e1 = off[lo], off[hi]
            out[u] = SparseAlignment((off[lo:hi + 1] - e0).astype(np.int64), comps[e0:e1].astype(np.int32),
                                     wts[e0:e1].astype(np.float32))
        return out


def _batches(n, size):
    return [(i, min(n, i + size)) for i in range(0, n, size)]


def _stats_batch(corpus, ali, lo, hi, C, center, ssum):
    """Device BW stats for utterances [lo, hi): n (Ub, C), f (Ub, C*F); ssum accumulated."""
    F = corpus.dim
    utt = corpus.utt_frames[lo:hi + 1]
    cap = int(ali.utt_entries[hi] - ali.utt_entries[lo]) + 1
    n, f, _ = _device.bw_stats(corpus.x, utt, ali.offsets, ali.comps, ali.weights, C, center=center,
                               ssum_acc=ssum, entry_capacity=cap)
    return n, f.view(hi - lo, C * F)


def _accumulate(dm, ws, corpus, ali, center):
    """E-step over a device corpus into a fresh device accumulator (merged across ranks)."""
    acc = _estep.DeviceAcc(dm.C, dm.F, dm.D)
    n_utt = len(corpus.ids)
    statuses = []  # checked once after the last batch: no host synchronization inside the E-step
    for lo, hi in _batches(n_utt, _estep.E_STEP_BATCH):
        n, f = _stats_batch(corpus, ali, lo, hi, dm.C, center, acc.Ssum)
        _estep.accumulate_batch(dm, ws, acc, n, f, S=None, statuses=statuses)
    _estep.check_status(statuses)
    _dist.allreduce_sum_(acc.flat)
    return acc


# ----------------------------------------------------------------------------- corpus operations


def align_corpus(store, ubm_diag, ubm_full, top_k=20, prune=0.025, workers=1, batch_size=8, ids=None):
    """Align every utterance of a store; returns {utterance id: SparseAlignment} (pipeline.py:364-382)."""
    if ids is None:
        ids = store.ids()
    corpus = _device_corpus(store, ids, workers)
    if corpus.n_frames == 0:
        return {u: SparseAlignment.from_frames([]) for u in ids}
    full_tab = ubm_full.device_table()
    from .gmm import _raise_if_not_spd
    _raise_if_not_spd(full_tab)
    ali = DeviceAlignment.compute(corpus, ubm_diag.device_table(), full_tab, top_k, prune)
    return ali.to_host(corpus)


def accumulate_corpus(model, store, alignments, config, ids=None, workspace=None):
    """Full-corpus E-step from features and given alignments (pipeline.py:385-415)."""
    if ids is None:
        ids = store.ids()
    if not ids:
        raise PipelineError("empty corpus")
    dm = _estep.DeviceModel(model)
    ws = _estep.Workspace(dm) if workspace is None or workspace.model is not model else workspace.dev
    if getattr(ws, "bad", np.zeros(0)).size:
        from ._linalg import NumericError
        raise NumericError(f"Sigma[{int(ws.bad[0])}] is not SPD")
    # under torch.distributed each rank accumulates its contiguous shard and the all-reduce in
    # _accumulate sums the shards, so every rank returns the full-corpus statistics
    rank, world_size = _dist.world()
    corpus = _device_corpus(store, _dist.shard(list(ids), rank, world_size), config.workers)
    ali = DeviceAlignment.from_host(corpus, alignments)
    center = dm.bias if model.formulation == STANDARD else None
    acc = _accumulate(dm, ws, corpus, ali, center)
    return EmAccumulators(**_estep.to_host_acc(acc, _estep.finalize_aux(dm, ws, acc)))


def extract_corpus(model, store, top_k=20, prune=0.025, workers=1, batch_size=8, ids=None, out_path=None):
    """One embedding per utterance, aligned with the model's predictive-covariance UBM
    (pipeline.py:418-459).  Returns (ids, (U, D) array)."""
    if ids is None:
        ids = store.ids()
    dm = _estep.DeviceModel(model)
    ws = _estep.Workspace(dm)
    if ws.bad.size:
        from ._linalg import NumericError
        raise NumericError(f"Sigma[{int(ws.bad[0])}] is not SPD")
    rank, world_size = _dist.world()
    local = _dist.shard(list(ids), rank, world_size)
    emb = _extract_device(dm, ws, model, _device_corpus(store, local, workers), top_k, prune)
    counts = [_dist.shard_range(len(ids), r, world_size)[1] - _dist.shard_range(len(ids), r, world_size)[0]
              for r in range(world_size)]
    emb = _lib.to_host(_dist.gather_rows(emb, counts))
    if out_path is not None and rank == 0:
        save_embeddings(out_path, list(ids), emb)
    return list(ids), emb


def _extract_device(dm, ws, model, corpus, top_k, prune):
    D = dm.D
    out = _lib.empty((len(corpus.ids), D))
    if not corpus.ids:
        return out
    pc = _estep.predictive_covariances_device(dm.T, dm.Sigma, dm.C, dm.F, D)
    diag_var = torch.diagonal(pc, dim1=1, dim2=2).contiguous()
    diag_tab = _device.DiagTable(model.ubm_weights, model.ubm_means, diag_var)
    full_tab = _device.FullTable(model.ubm_weights, model.ubm_means, pc)
    from .gmm import _raise_if_not_spd
    _raise_if_not_spd(full_tab)
    center = dm.bias if model.formulation == STANDARD else None
    if corpus.n_frames:
        ali = DeviceAlignment.compute(corpus, diag_tab, full_tab, top_k, prune)
    else:
        ali = DeviceAlignment(_lib.zeros((1,), torch.int64), _lib.zeros((1,), torch.int32),
                              _lib.zeros((1,), torch.float32), np.zeros(len(corpus.ids) + 1, np.int64))
    statuses = []
    for lo, hi in _batches(len(corpus.ids), _estep.E_STEP_BATCH):
        n, f = _stats_batch(corpus, ali, lo, hi, dm.C, center, None)
        phi, _, _, _, status, _ = _estep.posterior_batch(dm, ws, n, f, want_moment=False)
        statuses.append(status)
        out[lo:hi] = phi
    _estep.check_status(statuses)
    return out


def save_embeddings(path, ids, embeddings):
    """Embedding store: f64 matrix file plus a ``<path>.ids`` text sidecar."""
    write_matrix(embeddings, "f64", path)
    with open(path + ".ids", "w", encoding="utf-8") as fh:
        fh.writelines(f"{u}\n" for u in ids)


def load_embeddings(path):
    emb = read_matrix(path)
    with open(path + ".ids", encoding="utf-8") as fh:
        ids = [ln.strip() for ln in fh if ln.strip()]
    if len(ids) != emb.shape[0]:
        raise PipelineError("embedding ids do not match matrix rows")
    return ids, emb


# ----------------------------------------------------------------------------- checkpoints

_STATE_FILE = "state.txt"
_ALIGN_CACHE = "alignments.aln"


def _ckpt_model(d, it):
    return os.path.join(d, f"model_iter_{it:04d}.tvm")


def _save_ubm_aux(d, ubm_diag, ubm_full):
    write_matrix(ubm_diag.weights[None, :], "f64", os.path.join(d, "ubm_diag_weights.fmx"))
    write_matrix(ubm_diag.means, "f64", os.path.join(d, "ubm_diag_means.fmx"))
    write_matrix(ubm_diag.variances, "f64", os.path.join(d, "ubm_diag_vars.fmx"))
    c, f, _ = ubm_full.covariances.shape
    write_matrix(ubm_full.covariances.reshape(c * f, f), "f64", os.path.join(d, "ubm_full_covs.fmx"))


def _load_ubm_aux(d, c):
    w = read_matrix(os.path.join(d, "ubm_diag_weights.fmx"))[0]
    mu = read_matrix(os.path.join(d, "ubm_diag_means.fmx"))
    var = read_matrix(os.path.join(d, "ubm_diag_vars.fmx"))
    covs = read_matrix(os.path.join(d, "ubm_full_covs.fmx"))
    return GmmDiag(w, mu, var), covs.reshape(c, mu.shape[1], mu.shape[1])


def _write_state(d, it, h, seed):
    with open(os.path.join(d, _STATE_FILE), "w", encoding="utf-8") as fh:
        fh.write(f"iteration = {it}\nconfig_hash = {h}\nseed = {seed}\n")


def _read_state(d):
    st = {}
    with open(os.path.join(d, _STATE_FILE), encoding="utf-8") as fh:
        for line in fh:
            if "=" in line:
                k, v = (p.strip() for p in line.split("=", 1))
                st[k] = v
    return int(st["iteration"]), st["config_hash"], int(st["seed"])


def _realign_points(config, upto):
    if config.realign_interval <= 0:
        return []
    return [it for it in range(1, upto + 1) if it % config.realign_interval == 0 and it != config.iterations]


# ----------------------------------------------------------------------------- EM training


class _HostMoments:
    """The slice of EmAccumulators that compute_min_div reads (h, H, U)."""

    def __init__(self, acc):
        self.U = acc.U
        self.phi_sum = _lib.to_host(acc.phi_sum)
        self.moment_sum = _estep.unpack_host(_lib.to_host(acc.moment), acc.D)

    @classmethod
    def start(cls, acc):
        """Asynchronous variant: device->pinned copies queued now, ``finish()`` waits for them only."""
        self = cls.__new__(cls)
        self.U = acc.U
        self._D = acc.D
        self._phi = torch.empty(acc.phi_sum.shape, dtype=torch.float64, pin_memory=True)
        self._mom = torch.empty(acc.moment.shape, dtype=torch.float64, pin_memory=True)
        self._phi.copy_(acc.phi_sum, non_blocking=True)
        self._mom.copy_(acc.moment, non_blocking=True)
        self._ev = torch.cuda.Event()
        self._ev.record()
        return self

    def finish(self):
        self._ev.synchronize()
        self.phi_sum = self._phi.numpy().copy()
        self.moment_sum = _estep.unpack_host(self._mom.numpy(), self._D)

    @property
    def h(self):
        return self.phi_sum / self.U

    @property
    def H(self):
        return self.moment_sum / self.U


class DeviceTrainer:
    """Device-resident EM loop state (pipeline.py:597-653 semantics)."""

    def __init__(self, model: TvModel, corpus: DeviceCorpus, config: TrainConfig):
        self.model = model
        self.config = config
        self.corpus = corpus
        self.dm = _estep.DeviceModel(model)
        self.alignment = None
        self.host_dirty = False

    def sync_host(self):
        """Copy the device parameters back into the host TvModel."""
        if not self.host_dirty:
            return self.model
        m, dm = self.model, self.dm
        m.T = _lib.to_host(dm.T)
        m.Sigma = _lib.to_host(dm.Sigma)
        if dm.bias is not None:
            m.bias = _lib.to_host(dm.bias)
        m.prior_offset = dm.prior_offset
        self.host_dirty = False
        return m

    def align(self, align_diag, align_cov):
        m = self.model
        diag_tab = _device.DiagTable(align_diag.weights, align_diag.means, align_diag.variances)
        full_tab = _device.FullTable(m.ubm_weights, m.ubm_means, align_cov)
        from .gmm import _raise_if_not_spd
        _raise_if_not_spd(full_tab)
        self.alignment = DeviceAlignment.compute(self.corpus, diag_tab, full_tab, self.config.top_k,
                                                 self.config.prune)

    def realign_point(self, it, align_diag):
        """UBM-mean feedback after iteration ``it`` (pipeline.py:628-638): at a realignment point the
        alignment means become p*T[:, :, 0] (augmented) or the bias (standard) and the corpus
        alignment is dropped so the next iteration realigns every frame.  Returns True if so."""
        cfg = self.config
        if not (cfg.realign_interval > 0 and it % cfg.realign_interval == 0 and it != cfg.iterations):
            return False
        dm = self.dm
        if dm.formulation == AUGMENTED:
            means = dm.prior_offset * _lib.to_host(dm.T[:, :, 0])
        else:
            means = _lib.to_host(dm.bias)
        self.model.ubm_means = means.copy()
        align_diag.means = means.copy()
        self.alignment = None
        return True

    def iteration(self):
        """E-step + M-step (+ min-div); returns the aux of the E-step."""
        cfg, dm = self.config, self.dm
        C, F, D = dm.C, dm.F, dm.D
        ws = _estep.Workspace(dm)
        if ws.bad.size:
            from ._linalg import NumericError
            raise NumericError(f"Sigma[{int(ws.bad[0])}] is not SPD")
        center = dm.bias if dm.formulation == STANDARD else None
        acc = _accumulate(dm, ws, self.corpus, self.alignment, center)
        if acc.U < 1:
            raise PipelineError("empty corpus")
        aux_dev = _estep.finalize_aux_dev(dm, ws, acc)
        # the min-divergence moments go to pinned host memory ahead of the M-step kernels, so the host
        # eigh of compute_min_div runs while the GPU computes update_T / update_sigma; the results are
        # checked (warnings, errors) and applied in the reference's order afterwards
        mom = _HostMoments.start(acc) if cfg.min_div else None
        T_new, st = _estep.update_T_device(dm.T, acc.Apk, acc.B, acc.N, C, F, D)
        if cfg.sigma_update:
            S_new, st2 = _estep.update_sigma_device(dm.Sigma, T_new, acc.B, acc.N, acc.Ssum, C, F, D,
                                                    SIGMA_FLOOR_SCALE)
        tr = tr_err = None
        if mom is not None:
            mom.finish()
            try:
                tr = compute_min_div(mom, dm.formulation)
            except Exception as exc:  # raised after the M-step's own checks, as the reference orders them
                tr_err = exc
        aux = _estep.aux_value(dm, acc, aux_dev)
        _warn_singular(_lib.to_host(st))
        if cfg.sigma_update:
            _raise_collapsed(_lib.to_host(st2))
            dm.Sigma = S_new
        dm.T = T_new
        if cfg.min_div:
            if tr_err is not None:
                raise tr_err
            h = mom.h
            if cfg.update_mean and dm.formulation == STANDARD:
                hb = _lib.to_dev(h)
                bias = dm.bias.reshape(C * F, 1)
                _lib.dgemm(dm.T, hb, bias, C * F, 1, D, beta=1.0)
            from .tvm import _right_factor
            right = _right_factor(tr, dm.formulation)
            dm.T = _estep.right_multiply(dm.T, right, C, F, D)
            if dm.formulation == AUGMENTED:
                projected = tr.P2 @ (tr.P1 @ h)
                tail = np.max(np.abs(projected[1:])) if projected.shape[0] > 1 else 0.0
                if tail > 1e-8 * max(1.0, abs(projected[0])):
                    from ._linalg import NumericError
                    raise NumericError("projected prior mean not aligned with the first axis")
                dm.prior_offset = float(projected[0])
                dm.prior_mean = np.zeros(D)
                dm.prior_mean[0] = dm.prior_offset
        self.host_dirty = True
        self.last_acc = acc
        return aux


def train_extractor(config, store, ubm_diag, ubm_full, seed=None, checkpoint_dir=None, resume=False,
                    iteration_hook=None):
    """Train one extractor; returns (model, RunMetrics for this seed) (pipeline.py:539-655).

    Under torch.distributed each rank holds a contiguous shard of the utterances and the
    E-step statistics are summed with one all-reduce per iteration; rank 0 writes checkpoints.
    """
    config.validate()
    if seed is None:
        seed = config.seeds[0]
    ids = store.ids()
    if not ids:
        raise PipelineError("empty corpus")
    if ubm_diag.n_components != ubm_full.n_components or ubm_diag.dim != ubm_full.dim:
        raise PipelineError("diagonal and full background models disagree")
    config_hash = config.config_hash()
    rank, world_size = _dist.world()

    start = 1
    model = None
    align_diag = None
    align_cov = ubm_full.covariances.copy()
    if resume:
        if checkpoint_dir is None:
            raise PipelineError("resume requires a checkpoint directory")
        if os.path.exists(os.path.join(checkpoint_dir, _STATE_FILE)):
            done, saved_hash, saved_seed = _read_state(checkpoint_dir)
            if saved_hash != config_hash:
                raise PipelineError("checkpoint config hash does not match")
            if saved_seed != seed:
                raise PipelineError("checkpoint seed does not match")
            model = load_model(_ckpt_model(checkpoint_dir, done))
            align_diag, align_cov = _load_ubm_aux(checkpoint_dir, model.n_components)
            if _realign_points(config, done):
                align_diag.means = model.ubm_means.copy()
            start = done + 1
            logger.info("resuming at iteration %d", start)
    if model is None:
        model = init_model(ubm_full, config.latent_dim, config.formulation, seed=seed,
                           prior_offset=config.prior_offset)
        align_diag = ubm_diag.copy()
        if checkpoint_dir is not None and rank == 0:
            os.makedirs(checkpoint_dir, exist_ok=True)
            config.save(os.path.join(checkpoint_dir, "config.cfg"))
            _save_ubm_aux(checkpoint_dir, ubm_diag, ubm_full)
            stale = os.path.join(checkpoint_dir, _ALIGN_CACHE)
            if os.path.exists(stale):
                os.remove(stale)

    metrics = RunMetrics()
    local_ids = _dist.shard(ids, rank, world_size)
    corpus = _device_corpus(store, local_ids, config.workers)
    trainer = DeviceTrainer(model, corpus, config)
    cache = os.path.join(checkpoint_dir, _ALIGN_CACHE) if checkpoint_dir is not None else None
    have_alignment = False

    for it in range(start, config.iterations + 1):
        t0 = time.perf_counter()
        if not have_alignment:
            if cache is not None and os.path.exists(cache) and world_size == 1:
                trainer.alignment = DeviceAlignment.from_host(corpus, read_alignment(cache))
            else:
                trainer.align(align_diag, align_cov)
                if cache is not None and world_size == 1:
                    write_alignment(cache, [(u, a) for u, a in trainer.alignment.to_host(corpus).items()],
                                    top_k=config.top_k)
            have_alignment = True

        aux = trainer.iteration()

        if trainer.realign_point(it, align_diag):
            have_alignment = False
            if cache is not None and rank == 0 and os.path.exists(cache):
                os.remove(cache)

        eer = float("nan")
        if iteration_hook is not None:
            res = iteration_hook(trainer.sync_host(), it)
            if res is not None:
                eer = float(res)
        wall = time.perf_counter() - t0
        metrics.records.append(IterationRecord(seed, it, aux, eer, wall))
        logger.info("seed %d iteration %d: aux %.6f eer %s (%.2fs)", seed, it, aux, eer, wall)
        if checkpoint_dir is not None and rank == 0:
            save_model(trainer.sync_host(), _ckpt_model(checkpoint_dir, it))
            _write_state(checkpoint_dir, it, config_hash, seed)
    return trainer.sync_host(), metrics


# ----------------------------------------------------------------------------- out of scope
# The reference pipeline module also hosts the verification back-end drivers (pipeline.py:660-757:
# EvalProtocol, evaluate_model, ensemble_run).  They score embeddings with the PLDA/LDA back-end,
# which is outside the GPU hot path.  The names resolve so that code importing them
# from the drop-in still imports; using one raises and points at the reference package.

_OUT_OF_SCOPE = ("EvalProtocol", "evaluate_model", "ensemble_run")


class _OutOfScope:
    def __init__(self, name):
        self.__name__ = self.__qualname__ = name

    def __call__(self, *args, **kwargs):
        raise NotImplementedError(f"tvkit.{self.__name__} is verification back-end scoring, outside the GPU "
                                  f"i-vector path of this package; use the reference tvkit for it")

    def __repr__(self):
        return f"<out-of-scope {self.__name__}>"


def __getattr__(name):
    if name in _OUT_OF_SCOPE:
        return _OutOfScope(name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
