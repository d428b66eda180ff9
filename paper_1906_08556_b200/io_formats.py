"""Binary containers used by the drivers: FMX1 matrices, TVM1 models, ALN1 alignments.

Byte-compatible with the reference ``io_formats.py`` (layouts at io_formats.py:1-15,
59-98, 104-233, 240-295) so checkpoints and alignment caches interoperate with it.
The ALN1 encoder is vectorized (one numpy scatter per utterance instead of a per-frame
``struct.pack`` loop); the decoder walks the frame records with
numpy cumulative sums over the u32 stream.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass

import numpy as np

MATRIX_MAGIC = b"FMX1"
ALIGNMENT_MAGIC = b"ALN1"
MODEL_MAGIC = b"TVM1"
_CODES = {"f32": 0, "f64": 1}
_DTYPES = {0: np.dtype("<f4"), 1: np.dtype("<f8")}


class FormatError(ValueError):
    """A file does not conform to its declared container layout."""


def _need(fh, n, what):
    b = fh.read(n)
    if len(b) != n:
        raise FormatError(f"truncated file while reading {what}")
    return b


def _fits(fh, n, what):
    left = os.fstat(fh.fileno()).st_size - fh.tell()
    if n > left:
        raise FormatError(f"declared {what} size {n} exceeds remaining {left} bytes")


def write_matrix(matrix, dtype, path):
    """2-D array -> FMX1 file with dtype "f32" or "f64"."""
    m = np.asarray(matrix)
    if m.ndim != 2:
        raise ValueError("matrix files hold 2-D arrays")
    if m.shape[0] < 1 or m.shape[1] < 1:
        raise ValueError("matrix must have at least one row and column")
    if dtype not in _CODES:
        raise ValueError(f"unknown dtype {dtype!r}, expected 'f32' or 'f64'")
    code = _CODES[dtype]
    with open(path, "wb") as fh:
        fh.write(MATRIX_MAGIC + struct.pack("<BQQ", code, m.shape[0], m.shape[1]))
        fh.write(np.ascontiguousarray(m, dtype=_DTYPES[code]).tobytes())


def read_matrix(path):
    with open(path, "rb") as fh:
        if _need(fh, 4, "magic") != MATRIX_MAGIC:
            raise FormatError("bad magic, expected b'FMX1'")
        code, rows, cols = struct.unpack("<BQQ", _need(fh, 17, "header"))
        if code not in _DTYPES:
            raise FormatError(f"unknown dtype code {code}")
        dt = _DTYPES[code]
        _fits(fh, rows * cols * dt.itemsize, "matrix payload")
        raw = _need(fh, rows * cols * dt.itemsize, "payload")
        if fh.read(1):
            raise FormatError("trailing bytes after matrix payload")
    return np.frombuffer(raw, dtype=dt).reshape(rows, cols).copy()


# ------------------------------------------------------------------------ models


def save_model(model, path):
    """TVM1: tag, C, F, D, prior offset, then weights, means, T, Sigma[, bias] as <f8."""
    model.validate()
    c, f, d = model.T.shape
    tag = 0 if model.formulation == "standard" else 1
    with open(path, "wb") as fh:
        fh.write(MODEL_MAGIC + struct.pack("<BQQQd", tag, c, f, d, model.prior_offset))
        parts = [model.ubm_weights, model.ubm_means, model.T, model.Sigma]
        if tag == 0:
            parts.append(model.bias)
        for p in parts:
            fh.write(np.ascontiguousarray(p, dtype="<f8").tobytes())


def load_model(path):
    from .tvm import TvModel

    with open(path, "rb") as fh:
        if _need(fh, 4, "magic") != MODEL_MAGIC:
            raise FormatError("bad magic, expected b'TVM1'")
        tag, c, f, d, p = struct.unpack("<BQQQd", _need(fh, 33, "header"))
        if tag not in (0, 1):
            raise FormatError(f"unknown formulation tag {tag}")

        def take(shape, what):
            k = int(np.prod(shape))
            _fits(fh, 8 * k, what)
            return np.frombuffer(_need(fh, 8 * k, what), dtype="<f8").reshape(shape).copy()

        w = take((c,), "weights")
        mu = take((c, f), "means")
        T = take((c, f, d), "T")
        S = take((c, f, f), "Sigma")
        bias = take((c, f), "bias") if tag == 0 else None
        if fh.read(1):
            raise FormatError("trailing bytes after model tensors")
    model = TvModel("standard" if tag == 0 else "augmented", T, S, w, mu, bias=bias, prior_offset=p)
    model.validate()
    return model


# ------------------------------------------------------------------------ alignments


def _encode_frames(ali):
    """u32 stream [count_t, (comp, weight bits) * count_t] for every frame, vectorized."""
    counts = np.diff(ali.offsets).astype(np.int64)
    T = counts.shape[0]
    E = int(ali.offsets[-1] - ali.offsets[0]) if T else 0
    out = np.empty(T + 2 * E, dtype="<u4")
    start = np.arange(T, dtype=np.int64) + 2 * (ali.offsets[:-1] - ali.offsets[0])
    out[start] = counts
    if E:
        frame_of = np.repeat(np.arange(T, dtype=np.int64), counts)
        pos = frame_of + 1 + 2 * np.arange(E, dtype=np.int64)
        out[pos] = ali.components.astype("<u4")
        out[pos + 1] = np.ascontiguousarray(ali.weights, dtype="<f4").view("<u4")
    return out


def write_alignment(path, alignments, top_k):
    """Per-utterance sparse alignments -> one ALN1 corpus file (given order)."""
    items = list(alignments.items()) if hasattr(alignments, "items") else list(alignments)
    index = []
    with open(path, "wb") as fh:
        fh.write(ALIGNMENT_MAGIC + struct.pack("<IQQ", top_k, len(items), 0))
        for utt, ali in items:
            ali.validate(top_k=top_k)
            index.append((utt, fh.tell()))
            uid = utt.encode("utf-8")
            fh.write(struct.pack("<I", len(uid)) + uid + struct.pack("<Q", ali.n_frames))
            fh.write(_encode_frames(ali).tobytes())
        index_offset = fh.tell()
        for utt, off in index:
            uid = utt.encode("utf-8")
            fh.write(struct.pack("<I", len(uid)) + uid + struct.pack("<Q", off))
        fh.seek(4 + 4 + 8)
        fh.write(struct.pack("<Q", index_offset))


def _decode_frames(words, n_frames):
    """Inverse of _encode_frames; frame starts found by walking the count words."""
    from .gmm import SparseAlignment

    import ctypes

    from . import _lib

    words = np.ascontiguousarray(words, dtype="<u4")
    if n_frames > words.shape[0]:  # every frame needs its count word: reject before allocating
        raise FormatError("frame record shorter than declared (entry count)")
    starts = np.empty(n_frames, dtype=np.int64)
    counts = np.empty(n_frames, dtype=np.int64)
    end = ctypes.c_int64(0)
    # the sequential count-word walk runs in libtvk's host code (tvk_aln1_scan)
    st = _lib.load().tvk_aln1_scan(words.ctypes.data_as(ctypes.c_void_p), words.shape[0], n_frames,
                                   starts.ctypes.data_as(ctypes.c_void_p), counts.ctypes.data_as(ctypes.c_void_p),
                                   ctypes.byref(end))
    if st != _lib.TVK_OK:
        raise FormatError(_lib.last_error().replace("aln1: ", ""))
    pos = int(end.value)
    E = int(counts.sum())
    offsets = np.zeros(n_frames + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    if E:
        frame_of = np.repeat(np.arange(n_frames), counts)
        within = np.arange(E) - offsets[:-1][frame_of]
        idx = starts[frame_of] + 1 + 2 * within
        comps = words[idx].astype(np.int32)
        wts = words[idx + 1].view("<f4").astype(np.float32)
    else:
        comps, wts = np.zeros(0, np.int32), np.zeros(0, np.float32)
    return SparseAlignment(offsets, comps, wts), pos


class AlignmentReader:
    """Random access to an ALN1 corpus file through its index (io_formats.py:155-227).

    Each record is bounded by the next record's start (or the index); the count-word walk and the
    entry gather are vectorized (``_decode_frames``).  One file handle per reader.
    """

    def __init__(self, path):
        self.path = path
        self._fh = open(path, "rb")
        try:
            fh = self._fh
            magic = _need(fh, 4, "magic")
            if magic != ALIGNMENT_MAGIC:
                raise FormatError(f"bad magic {magic!r}, expected {ALIGNMENT_MAGIC!r}")
            self.top_k, n_utts, index_offset = struct.unpack("<IQQ", _need(fh, 20, "header"))
            if index_offset > os.fstat(fh.fileno()).st_size:
                raise FormatError("index offset beyond end of file")
            self._index_offset = index_offset
            fh.seek(index_offset)
            self._index, self._order = {}, []
            for _ in range(n_utts):
                (n,) = struct.unpack("<I", _need(fh, 4, "index"))
                _fits(fh, n, "index id")
                uid = _need(fh, n, "index id").decode("utf-8")
                (off,) = struct.unpack("<Q", _need(fh, 8, "index offset"))
                self._index[uid] = off
                self._order.append(uid)
            # record end = next record start in file order (one sort, O(U log U))
            starts = np.unique(np.array(list(self._index.values()) + [index_offset], dtype=np.uint64))
            self._bounds = starts
        except Exception:
            self._fh.close()
            raise

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def close(self):
        self._fh.close()

    def ids(self):
        return list(self._order)

    def _end_of(self, off):
        b = self._bounds
        i = int(np.searchsorted(b, np.uint64(off), side="right"))
        return int(b[i]) if i < b.shape[0] else self._index_offset

    def read(self, utt_id):
        try:
            off = self._index[utt_id]
        except KeyError:
            raise KeyError(f"utterance {utt_id!r} not in alignment file") from None
        fh = self._fh
        end = min(self._end_of(off), self._index_offset)
        fh.seek(off)

        def bounded(count, what):
            if fh.tell() + count > self._index_offset:
                raise FormatError(f"frame record shorter than declared ({what})")
            return _need(fh, count, what)

        (n,) = struct.unpack("<I", bounded(4, "utterance id"))
        stored = bounded(n, "utterance id").decode("utf-8")
        if stored != utt_id:
            raise FormatError("alignment index does not match record")
        (n_frames,) = struct.unpack("<Q", bounded(8, "frame count"))
        body = max(0, end - fh.tell())
        words = np.frombuffer(_need(fh, body - body % 4, "frame entries"), dtype="<u4")
        ali, _ = _decode_frames(words, n_frames)
        return ali


def read_alignment(path):
    """Whole ALN1 file -> {utterance id: SparseAlignment} (io_formats.py:230-233)."""
    with AlignmentReader(path) as reader:
        return {u: reader.read(u) for u in reader.ids()}


# ----------------------------------------------------------------------------- trial lists
# Verification trial files (io_formats.py:299-327): one "enrol test target|nontarget" line per trial.
# Not on the GPU path; kept so the drop-in's io_formats surface matches the reference's.

_LABELS = {"target": True, "nontarget": False}


@dataclass
class TrialList:
    """Verification trials: enrol/test id pairs with target flags."""

    enrol_ids: list
    test_ids: list
    is_target: np.ndarray

    def __len__(self):
        return len(self.enrol_ids)

    def validate(self):
        if len(self.enrol_ids) != len(self.test_ids) or len(self.test_ids) != self.is_target.shape[0]:
            raise ValueError("trial field lengths differ")


def write_trials(path, trials):
    trials.validate()
    lines = [f"{e} {t} {'target' if flag else 'nontarget'}\n"
             for e, t, flag in zip(trials.enrol_ids, trials.test_ids, trials.is_target)]
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(lines)


def read_trials(path):
    enrol, test, flags = [], [], []
    with open(path, encoding="utf-8") as fh:
        for n, raw in enumerate(fh, 1):
            parts = raw.split()
            if not parts:
                continue
            if len(parts) != 3:
                raise FormatError(f"{path}:{n}: expected 'enrol test label'")
            if parts[2] not in _LABELS:
                raise FormatError(f"{path}:{n}: unknown label {parts[2]!r}")
            enrol.append(parts[0])
            test.append(parts[1])
            flags.append(_LABELS[parts[2]])
    return TrialList(enrol, test, np.asarray(flags, dtype=bool))
