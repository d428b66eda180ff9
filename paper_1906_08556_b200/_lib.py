"""ctypes binding of libtvk.so (the C ABI declared in include/tvk.h).

The product path has exactly one implementation: these CUDA kernels.  If the
library or a CUDA device is missing every entry point raises; there is no CPU
fallback.  Device memory, streams and host<->device copies are torch
(plumbing); all arithmetic of the hot path happens inside libtvk.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtvk.so")

TVK_OK = 0
TVK_OUT_DENSE = 0
TVK_OUT_PACKED_LOWER = 1
ITEM_OK = 0
ITEM_NOT_SPD = 1
ITEM_CLAMPED = 2
ITEM_SKIPPED = 4

_p = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_d = ctypes.c_double

# name -> (restype, argtypes); mirrors include/tvk.h
SIGNATURES = {
    "tvk_version": (_i, []),
    "tvk_aln1_scan": (_i, [_p, _i64, _i64, _p, _p, _p]),
    "tvk_last_error": (_i, [ctypes.c_char_p, _i64]),
    "tvk_dgemm": (_i, [_i, _i, _i, _i, _i, _d, _p, _i64, _i64, _p, _i64, _i64, _d, _p, _i64, _i64, _i, _i, _i,
                       _p, _p]),
    "tvk_dgemm_i8": (_i, [_i, _i, _i, _i, _i, _d, _p, _i64, _p, _p, _i64, _p, _d, _p, _i64, _i, _p]),
    "tvk_i8_operand_bytes": (_i64, [_i, _i, _i, _i]),
    "tvk_i8_split": (_i, [_p, _i, _i, _i64, _i64, _i, _i, _p, _p]),
    "tvk_colsum": (_i, [_p, _i64, _i64, _i64, _d, _d, _p, _p]),
    "tvk_ddot_workspace_bytes": (_i64, []),
    "tvk_ddot": (_i, [_p, _p, _i64, _d, _d, _p, _p, _p]),
    "tvk_spd_small": (_i, [_p, _i, _i, _p, _p, _p, _p, _p]),
    "tvk_diag_table": (_i, [_p, _p, _p, _i, _i, _p, _p]),
    "tvk_diag_table_bytes": (_i64, [_i, _i]),
    "tvk_row_softmax": (_i, [_p, _i64, _i, _p, _p]),
    "tvk_seed_dist2": (_i, [_p, _i, _i64, _i, _p, _p, _i, _p]),
    "tvk_seed_workspace_bytes": (_i64, [_i64]),
    "tvk_seed_means": (_i, [_p, _i, _i64, _i, _i, _p, _p, _p, _p, _p, _i64, _p]),
    "tvk_full_moments": (_i, [_p, _i, _i, _d, _p, _p, _p, _p, _p, _p, _p]),
    "tvk_full_table": (_i, [_p, _p, _p, _i, _i, _p, _p, _p]),
    "tvk_precision_table": (_i, [_p, _p, _p, _i, _i, _p, _p, _p]),
    "tvk_precision_table_stride": (_i64, [_i]),
    "tvk_align_workspace_bytes": (_i64, [_i64, _i, _i]),
    "tvk_align_frames": (_i, [_p, _i, _i64, _i, _p, _p, _p, _i, _i, _d, _i, _p, _i64, _p, _p, _p, _p, _p, _p]),
    "tvk_select_topk": (_i, [_p, _i, _i64, _i, _p, _i, _i, _p, _p, _p]),
    "tvk_frame_features": (_i, [_p, _i, _i64, _i, _i, _p, _p]),
    "tvk_full_loglik_workspace_bytes": (_i64, [_i64, _i, _i]),
    "tvk_full_loglik_selected": (_i, [_p, _i, _i64, _i, _p, _p, _i, _i, _i, _p, _p, _p, _i64, _p]),
    "tvk_bw_workspace_bytes": (_i64, [_i64, _i, _i]),
    "tvk_bw_stats": (_i, [_p, _i, _i, _p, _i, _p, _p, _p, _i, _p, _p, _p, _p, _p, _i64, _p, _i64, _p]),
    "tvk_posterior_workspace_bytes": (_i64, [_i, _i]),
    "tvk_posterior": (_i, [_p, _p, _i, _i, _i, _p, _p, _p, _p, _p, _p, _i64, _p]),
    "tvk_spd_solve_rows": (_i, [_p, _p, _i, _i, _i, _p, _p, _p, _p, _i64, _p]),
    "tvk_sigma_floor": (_i, [_p, _p, _p, _p, _i, _i, _d, _p, _p, _p]),
}

_lib = None
_lock = threading.Lock()


class TvkError(RuntimeError):
    """A libtvk call failed (bad argument or CUDA error)."""


def load():
    """Load libtvk.so (raises if it is missing: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing; build it with `python -m paper_1906_08556_b200.build`")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name, None)
                if fn is None:
                    raise ImportError(f"{LIB_PATH} does not export {name}; rebuild the library")
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error():
    buf = ctypes.create_string_buffer(512)
    load().tvk_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def call(name, *args):
    """Invoke a status-returning entry point; raise TvkError on failure."""
    fn = getattr(load(), name)
    st = fn(*args)
    if fn.restype is _i and st != TVK_OK:
        raise TvkError(f"{name} failed (status {st}): {last_error()}")
    return st


_DEVICE = None


def device():
    """The CUDA device the kernels run on (rank-local under torch.distributed)."""
    global _DEVICE
    if _DEVICE is None:
        if not torch.cuda.is_available():
            raise TvkError("libtvk needs a CUDA device (B200); no CPU fallback exists")
        _DEVICE = torch.device("cuda", torch.cuda.current_device())
    return _DEVICE


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream(device()).cuda_stream)


def ptr(t):
    """Raw device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


_STAGE_MIN = 8 << 20          # host arrays at least this large go through the pinned staging buffer
_stage = {"buf": None, "ev": None}
_stage_pool = None


def _stage_copy(dst, src):
    """dst[:] = src for equal-shape CPU tensors, row blocks copied by a small thread pool (numpy copies
    release the GIL), so a large host array reaches pinned memory at memory bandwidth.  (Queuing each
    block's upload as soon as it is staged measured slower: 7 vs 5 ms for a 59 MB covariance stack.)"""
    global _stage_pool
    import concurrent.futures as cf
    if _stage_pool is None:
        _stage_pool = cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1), thread_name_prefix="tvk-stage")
    d, s_ = dst.numpy().reshape(-1), src.numpy().reshape(-1)
    n = d.shape[0]
    step = -(-n // (2 * _stage_pool._max_workers))
    list(_stage_pool.map(lambda lo: np.copyto(d[lo:lo + step], s_[lo:lo + step]), range(0, n, step)))


def to_dev(a, dtype=torch.float64):
    """Host array -> contiguous device tensor.  Large arrays (>= 8 MiB, e.g. a 2048 x 60 x 60 covariance
    stack) are staged through one reused pinned buffer and copied asynchronously (small ones through
    pinned blocks of torch's host allocator measured no faster end to end)."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    if t.numel() * t.element_size() < _STAGE_MIN:
        return t.to(device(), non_blocking=False).contiguous()
    nbytes = t.numel() * t.element_size()
    if _stage["ev"] is not None:
        _stage["ev"].synchronize()  # the previous staged copy has left the buffer
    buf = _stage["buf"]
    if buf is None or buf.numel() < nbytes:
        buf = _stage["buf"] = torch.empty(max(nbytes, 64 << 20), dtype=torch.uint8, pin_memory=True)
    view = buf[:nbytes].view(t.dtype).view(t.shape)
    _stage_copy(view, t)
    out = torch.empty(t.shape, dtype=t.dtype, device=device())
    out.copy_(view, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    _stage["ev"] = ev
    return out


def empty(shape, dtype=torch.float64):
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype=torch.float64):
    return torch.zeros(shape, dtype=dtype, device=device())


def to_host(t):
    return t.detach().cpu().numpy()


# ---------------------------------------------------------------------------- thin typed wrappers


def dgemm(a, b, c, m, n, k, *, trans_a=False, trans_b=False, alpha=1.0, beta=0.0, lda=None, ldb=None, ldc=None,
          batch=1, stride_a=0, stride_b=0, stride_c=0, out_mode=TVK_OUT_DENSE, splits=1, work=None):
    """C = alpha op(A) op(B) + beta C (row-major, FP64, DMMA tensor pipe)."""
    if lda is None:
        lda = m if trans_a else k
    if ldb is None:
        ldb = k if trans_b else n
    if ldc is None:
        ldc = n
    call("tvk_dgemm", int(trans_a), int(trans_b), m, n, k, alpha, ptr(a), lda, stride_a, ptr(b), ldb, stride_b,
         beta, ptr(c), ldc, stride_c, batch, out_mode, splits, ptr(work), stream())
    return c


def dgemm_i8(a, b, c, m, n, k, *, trans_a=False, trans_b=False, alpha=1.0, beta=0.0, lda=None, ldb=None, ldc=None,
             digits=7, a_split=None, b_split=None):
    """C = alpha op(A) op(B) + beta C (row-major, FP64) emulated on the int8 tensor cores (Ozaki digits,
    exact int32 products; include/tvk.h tvk_dgemm_i8).  a_split / b_split: operands pre-split with
    i8_split (then a / b may be None)."""
    if lda is None:
        lda = m if trans_a else k
    if ldb is None:
        ldb = k if trans_b else n
    if ldc is None:
        ldc = n
    call("tvk_dgemm_i8", int(trans_a), int(trans_b), m, n, k, alpha, ptr(a), lda, ptr(a_split), ptr(b), ldb,
         ptr(b_split), beta, ptr(c), ldc, int(digits), stream())
    return c


def i8_split_b(b, k, n, *, trans_b=False, ldb=None, digits=7):
    """Split op(B) (k x n, row-major B or B^T) once for repeated dgemm_i8(..., b_split=...) calls."""
    if ldb is None:
        ldb = k if trans_b else n
    nbytes = int(load().tvk_i8_operand_bytes(n, k, 64, digits))
    out = empty((nbytes,), torch.uint8)
    rs, ks = (ldb, 1) if trans_b else (1, ldb)
    call("tvk_i8_split", ptr(b), n, k, rs, ks, 64, int(digits), ptr(out), stream())
    return out


def x_args(x):
    """(pointer, is_f64) for a float32/float64 device frame matrix."""
    if x.dtype == torch.float64:
        return ptr(x), 1
    if x.dtype == torch.float32:
        return ptr(x), 0
    raise TypeError("frames must be float32 or float64")
