"""Device engine of the total-variability E-step and M-step (tvm.py:146-463 on libtvk).

Data layout in HBM (FP64 throughout, C components, F dims, D latent dims, P = D(D+1)/2):
  model      T (C, F, D) == (C*F, D) row-major;  Sigma (C, F, F)
  workspace  W = Sigma^-1 T (C*F, D);  Upk = packed T_c' Sigma_c^-1 T_c (C, P);
             Sinv (C, F, F);  logdet (C,)                                  [tvm.py:155-171]
  batch      N (Ub, C), Fm (Ub, C*F)  -> Lpk = N Upk (Ub, P),  b = Fm W + p e1 (Ub, D)
             posterior kernel -> phi (Ub, D), Mpk = packed(Phi + phi phi') (Ub, P)
  acc        Apk (C, P) += N' Mpk;  B (C*F, D) += Fm' phi;  Nsum, phi_sum, moment (P), Ssum
The four large E-step contractions (L = N U, b = F W, A += N'M, B += F' phi) run as FP64 emulated on
the int8 tensor cores (tvk_dgemm_i8: 7 Ozaki digits, exact int32 products, error <= 2^-45.8 K
max|row| max|col|); every other contraction is a tvk_dgemm call (FP64 DMMA tensor pipe).  Vector
sums are fixed-order reductions (bit-reproducible, no atomics).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import call, dgemm, dgemm_i8, i8_split_b, ptr, stream

LOG_2PI = float(np.log(2.0 * np.pi))
E_STEP_BATCH = 2048  # utterances per device E-step batch
# engine of the large E-step contractions: "int8" (tvk_dgemm_i8, FP64 emulated on the int8 tensor
# cores) or "dmma" (tvk_dgemm); products below I8_MIN_WORK multiply-adds stay on DMMA (the digit
# split is O((M + N) K) and not worth it for small shapes)
GEMM_ENGINE = "int8"
I8_DIGITS = 7     # contractions over the occupancies N (L = N U, A += N'M)
I8_DIGITS_F = 8   # contractions over the first-order statistics (b = F W, B += F' phi): a row of F spans
                  # components of very different occupancy, so it carries one more digit
I8_MIN_WORK = 1 << 30


def egemm(a, b, c, m, n, k, *, trans_a=False, beta=0.0, splits=1, work=None, digits=None, cache=None):
    """One of the E-step contractions C = op(A) B + beta C on the configured engine.  ``cache``: a dict
    that keeps B's int8 digits for later calls (B constant within an EM iteration: U, W)."""
    if GEMM_ENGINE == "int8" and m * n * k >= I8_MIN_WORK:
        digits = digits or I8_DIGITS
        b_split = None
        if cache is not None:
            key = (digits, k, n)
            if key not in cache:
                cache[key] = i8_split_b(b, k, n, digits=digits)
            b_split = cache[key]
        return dgemm_i8(a, b, c, m, n, k, trans_a=trans_a, beta=beta, digits=digits, b_split=b_split)
    return dgemm(a, b, c, m, n, k, trans_a=trans_a, beta=beta, splits=splits, work=work)


def packed_size(d):
    return d * (d + 1) // 2


_TRIL_CACHE = {}


def tril(d):
    """Row-major lower-triangle index pair (packed order of libtvk)."""
    if d not in _TRIL_CACHE:
        _TRIL_CACHE[d] = np.tril_indices(d)
    return _TRIL_CACHE[d]


def pack_host(a):
    """(..., D, D) symmetric -> (..., P) packed lower (host, layout only)."""
    i, j = tril(a.shape[-1])
    return np.ascontiguousarray(a[..., i, j])


def unpack_host(p, d):
    """(..., P) packed lower -> (..., D, D) symmetric (host, layout only)."""
    i, j = tril(d)
    out = np.empty(p.shape[:-1] + (d, d))
    out[..., i, j] = p
    out[..., j, i] = p
    return out


def ones(n):
    return torch.ones(n, dtype=torch.float64, device=_lib.device())


def col_sum_into(out_row, mat, rows, cols, beta=1.0, alpha=1.0):
    """out (cols) = beta*out + alpha * sum over the rows of mat (rows x cols)  [fixed order]."""
    call("tvk_colsum", ptr(mat), rows, cols, cols, alpha, beta, ptr(out_row), stream())
    return out_row


_DOT_WS = {}


def dot_into(out, x, y, n, alpha=1.0, beta=1.0):
    """out[0] = beta*out[0] + alpha * x.y over n elements (fixed-order reduction; y None: sum)."""
    dev = _lib.device()
    if dev not in _DOT_WS:
        _DOT_WS[dev] = _lib.empty((int(_lib.load().tvk_ddot_workspace_bytes()) // 8,))
    call("tvk_ddot", ptr(x), ptr(y), n, alpha, beta, ptr(out), ptr(_DOT_WS[dev]), stream())
    return out


class DeviceModel:
    """Device mirror of a TvModel's arrays."""

    def __init__(self, model):
        self.formulation = model.formulation
        self.C, self.F, self.D = model.T.shape
        self.T = _lib.to_dev(model.T)
        self.Sigma = _lib.to_dev(model.Sigma)
        pm = np.zeros(self.D)
        if model.formulation == "augmented" and self.D:
            pm[0] = model.prior_offset
        self.prior_mean = pm
        self.prior_offset = float(model.prior_offset)
        self.bias = _lib.to_dev(model.bias) if model.bias is not None else None


class Workspace:
    """PosteriorWorkspace on device (tvm.py:146-171)."""

    def __init__(self, dm: DeviceModel):
        C, F, D = dm.C, dm.F, dm.D
        self.C, self.F, self.D = C, F, D
        self.Sinv = _lib.empty((C, F, F))
        self.logdet = _lib.empty((C,))
        self.status = _lib.empty((C,), torch.int32)
        call("tvk_spd_small", ptr(dm.Sigma), C, F, None, ptr(self.Sinv), ptr(self.logdet), ptr(self.status),
             stream())
        bad = np.flatnonzero(_lib.to_host(self.status) != _lib.ITEM_OK)
        self.bad = bad
        self.W = _lib.empty((C, F, D))
        self.Upk = _lib.empty((C, packed_size(D)))
        self.i8_U = {}  # int8 digits of Upk / W for the E-step contractions (built on first use)
        self.i8_W = {}
        if D:
            # W_c = Sigma_c^-1 T_c   (C x [F x F . F x D])
            dgemm(self.Sinv, dm.T, self.W, F, D, F, batch=C, stride_a=F * F, stride_b=F * D, stride_c=F * D)
            # U_c = T_c' W_c packed lower   (C x [D x F . F x D])
            dgemm(dm.T, self.W, self.Upk, D, D, F, trans_a=True, batch=C, stride_a=F * D, stride_b=F * D,
                  stride_c=packed_size(D), out_mode=_lib.TVK_OUT_PACKED_LOWER)
        # per-component constant of the data term: F log 2pi + log|Sigma_c|
        self.const = self.logdet + F * LOG_2PI


class DeviceAcc:
    """Device EmAccumulators (tvm.py:232-280) with A in packed-lower storage."""

    def __init__(self, C, F, D, with_A=True):
        P = packed_size(D)
        self.C, self.F, self.D = C, F, D
        shapes = [("Apk", (C, P) if with_A else None), ("B", (C, F, D)), ("N", (C,)), ("Ssum", (C, F, F)),
                  ("phi_sum", (D,)), ("moment", (P,)), ("aux_post", (1,)), ("count", (1,))]
        total = sum(int(np.prod(s)) for _, s in shapes if s is not None)
        # one flat FP64 buffer: the multi-GPU merge is a single all-reduce over it
        self.flat = _lib.zeros((total,))
        off = 0
        for name, shape in shapes:
            if shape is None:
                setattr(self, name, None)
                continue
            k = int(np.prod(shape))
            setattr(self, name, self.flat[off:off + k].view(shape))
            off += k
        # aux pieces: sum_u [0.5 b.phi - 0.5 log|L|]; -0.5 sum_c N_c const_c, -0.5 <Sinv, Ssum> and
        # -0.5 U |mu0|^2 are added at finalize from corpus-level sums

    @property
    def U(self):
        return int(round(float(self.count.item())))

    @U.setter
    def U(self, value):
        self.count.fill_(float(value))


POST_ADD_IDENTITY = 1
POST_MOMENT = 2


def prior_mean_dev(dm):
    """Device copy of dm.prior_mean, refreshed only when the host vector changes (a pageable host->device
    copy per batch would synchronize the stream)."""
    key = dm.prior_mean.tobytes()
    cached = getattr(dm, "_prior_dev", None)
    if cached is None or cached[0] != key:
        dm._prior_dev = (key, _lib.to_dev(np.ascontiguousarray(dm.prior_mean, dtype=np.float64)))
    return dm._prior_dev[1]


def posterior_batch(dm: DeviceModel, ws: Workspace, n, fm, want_moment=True, status_out=None, covariance=False):
    """Posterior of a batch: phi (Ub, D), packed Phi + phi phi' (or Phi if ``covariance``) or None,
    logdet (Ub), bphi (Ub), status, b."""
    Ub = n.shape[0]
    C, F, D = dm.C, dm.F, dm.D
    P = packed_size(D)
    Lpk = _lib.empty((Ub, P))
    egemm(n, ws.Upk, Lpk, Ub, P, C, cache=ws.i8_U)  # L - I = sum_c n_c U_c
    b = _lib.empty((Ub, D))
    b.copy_(prior_mean_dev(dm).expand(Ub, D))
    K = C * F
    splits = max(1, min(16, K // 2048)) if Ub * D < 148 * 128 * 128 else 1
    work = _lib.empty((splits * Ub * D,)) if splits > 1 else None
    egemm(fm, ws.W, b, Ub, D, K, beta=1.0, splits=splits, work=work, digits=I8_DIGITS_F,
          cache=ws.i8_W)  # b = p e1 + sum_c W_c' f_c
    phi = _lib.empty((Ub, D))
    Mpk = Lpk if want_moment else None  # factored in place: M overwrites L (L2-resident working set)
    logdet = _lib.empty((Ub,))
    bphi = _lib.empty((Ub,))
    status = status_out if status_out is not None else _lib.empty((Ub,), torch.int32)
    flags = POST_ADD_IDENTITY | (0 if covariance else POST_MOMENT)
    call("tvk_posterior", ptr(Lpk), ptr(b), Ub, D, flags, ptr(phi), ptr(Mpk), ptr(logdet), ptr(bphi), ptr(status),
         None, 0, stream())
    return phi, Mpk, logdet, bphi, status, b


def check_status(status, what="posterior precision not SPD (corrupted Sigma?)"):
    from ._linalg import NumericError
    if isinstance(status, (list, tuple)):
        if not status:
            return
        status = torch.cat(status)
    st = _lib.to_host(status)
    if np.any(st != _lib.ITEM_OK):
        raise NumericError(what)


def accumulate_batch(dm: DeviceModel, ws: Workspace, acc: DeviceAcc, n, fm, S=None, statuses=None):
    """One E-step batch into the device accumulators (tvm.py:283-309).

    n (Ub, C), fm (Ub, C*F) device; S (Ub, C*F*F) device or None (Ssum accumulated elsewhere).
    ``statuses``: a list that collects the batch's posterior status for one check after the last batch
    (no host synchronization between batches); None checks it here.
    """
    Ub = n.shape[0]
    if Ub == 0:
        return
    C, F, D = dm.C, dm.F, dm.D
    P = packed_size(D)
    phi, Mpk, logdet, bphi, status, _ = posterior_batch(dm, ws, n, fm, want_moment=True)
    if statuses is None:
        check_status(status)
    else:
        statuses.append(status)
    if acc.Apk is not None:
        egemm(n, Mpk, acc.Apk, C, P, Ub, trans_a=True, beta=1.0)  # A_c += sum_u n_uc M_u
    egemm(fm, phi, acc.B, C * F, D, Ub, trans_a=True, beta=1.0, digits=I8_DIGITS_F)  # B_c += sum_u f_uc phi_u'
    col_sum_into(acc.N.view(1, C), n, Ub, C)
    col_sum_into(acc.phi_sum.view(1, D), phi, Ub, D)
    col_sum_into(acc.moment.view(1, P), Mpk, Ub, P)
    if S is not None:
        col_sum_into(acc.Ssum.view(1, C * F * F), S, Ub, C * F * F)
    # sum_u (0.5 b.phi - 0.5 log|L|)
    dot_into(acc.aux_post, bphi, None, Ub, alpha=0.5)
    dot_into(acc.aux_post, logdet, None, Ub, alpha=-0.5)
    acc.count += Ub


def finalize_aux(dm: DeviceModel, ws: Workspace, acc: DeviceAcc):
    """aux = sum_u loglik_u (tvm.py:202-214) from corpus-level sums."""
    return aux_value(dm, acc, finalize_aux_dev(dm, ws, acc))


def aux_value(dm: DeviceModel, acc: DeviceAcc, out):
    """Host value of finalize_aux_dev's device scalar."""
    mu0 = dm.prior_mean
    return float(out.item()) - 0.5 * float(mu0 @ mu0) * acc.U


def finalize_aux_dev(dm: DeviceModel, ws: Workspace, acc: DeviceAcc):
    """The device part of finalize_aux (fixed-order dot products), no host synchronization."""
    C, F = dm.C, dm.F
    out = acc.aux_post.clone()
    # -0.5 sum_c N_c (F log 2pi + log|Sigma_c|)
    dot_into(out, acc.N, ws.const, C, alpha=-0.5)
    # -0.5 <Sinv, Ssum>
    dot_into(out, ws.Sinv, acc.Ssum, C * F * F, alpha=-0.5)
    return out


def to_host_acc(acc: DeviceAcc, aux):
    """Device accumulators -> host EmAccumulators fields (A unpacked to (C, D, D))."""
    D = acc.D
    A = unpack_host(_lib.to_host(acc.Apk), D) if acc.Apk is not None else None
    return dict(A=A, B=_lib.to_host(acc.B), N=_lib.to_host(acc.N), Ssum=_lib.to_host(acc.Ssum),
                phi_sum=_lib.to_host(acc.phi_sum), moment_sum=unpack_host(_lib.to_host(acc.moment), D),
                U=acc.U, aux=aux)


# ------------------------------------------------------------------------------- M-step


SWEEP_MAX_D = 416  # tvk_posterior's block-sweep kernel (csrc/posterior.cu)
_TRIL_DEV = {}


def unpack_dev(pk, d):
    """(n, P) packed lower -> (n, D, D) symmetric dense on device (layout only)."""
    key = (d, pk.device)
    if key not in _TRIL_DEV:
        i, j = tril(d)
        _TRIL_DEV[key] = (torch.from_numpy(i).to(pk.device), torch.from_numpy(j).to(pk.device))
    i, j = _TRIL_DEV[key]
    out = torch.empty((pk.shape[0], d, d), dtype=pk.dtype, device=pk.device)
    out[:, i, j] = pk
    out[:, j, i] = pk
    return out


def update_T_device(T_old, Apk, B, N, C, F, D):
    """T_c = B_c A_c^-1 for N_c > 0 (tvm.py:317-334); returns (T_new, status).

    D <= 416: A_c^-1 for all components from one block-sweep pass (the EM posterior kernel without the
    identity and without b: it returns -(-A^-1)), then one batched DGEMM B_c A_c^-1; components that are
    starved (N_c <= 0) or whose A_c is not SPD (a non-positive sweep pivot, the Cholesky failure of the
    reference) keep T_c."""
    if 0 < D <= SWEEP_MAX_D:
        P = packed_size(D)
        inv = _lib.empty((C, P))
        zb = _lib.zeros((C, D))
        phi, ld, bp = _lib.empty((C, D)), _lib.empty((C,)), _lib.empty((C,))
        status = _lib.empty((C,), torch.int32)
        call("tvk_posterior", ptr(Apk), ptr(zb), C, D, 0, ptr(phi), ptr(inv), ptr(ld), ptr(bp), ptr(status), None, 0,
             stream())
        dense = unpack_dev(inv, D)
        del inv
        X = _lib.empty((C, F, D))
        dgemm(B, dense, X, F, D, D, batch=C, stride_a=F * D, stride_b=D * D, stride_c=F * D)
        skip = N.view(-1) <= 0
        status = torch.where(skip, torch.full_like(status, _lib.ITEM_SKIPPED), status)
        keep = (status != _lib.ITEM_OK).view(C, 1, 1)
        X = torch.where(keep, T_old.view(C, F, D), X)
        return X, status
    X = T_old.clone()
    skip = (N <= 0).to(torch.int32)
    status = _lib.empty((C,), torch.int32)
    ws_bytes = int(_lib.load().tvk_posterior_workspace_bytes(D, C))
    ws = _lib.empty((max(ws_bytes, 8),), torch.uint8)
    call("tvk_spd_solve_rows", ptr(Apk), ptr(B), C, D, F, ptr(skip), ptr(X), ptr(status), ptr(ws), ws_bytes,
         stream())
    return X, status


def update_sigma_device(Sigma_old, T_new, B, N, Ssum, C, F, D, floor_scale):
    """Residual covariances with eigen floor (tvm.py:337-358); returns (Sigma_new, status)."""
    TB = _lib.empty((C, F, F))
    if D:
        dgemm(T_new, B, TB, F, F, D, trans_b=True, batch=C, stride_a=F * D, stride_b=F * D, stride_c=F * F)
    else:
        TB.zero_()
    out = _lib.empty((C, F, F))
    status = _lib.empty((C,), torch.int32)
    call("tvk_sigma_floor", ptr(Ssum), ptr(TB), ptr(N), ptr(Sigma_old), C, F, float(floor_scale), ptr(out),
         ptr(status), stream())
    return out, status


def right_multiply(T, R, C, F, D):
    """T (C*F, D) @ R (D, D) on the tensor pipe (apply_min_div, tvm.py:436-444)."""
    out = _lib.empty((C, F, D))
    dgemm(T, R, out, C * F, D, D)
    return out


def predictive_covariances_device(T, Sigma, C, F, D):
    """Sigma_c + T_c T_c' (tvm.py:78-86)."""
    out = Sigma.clone()
    if D:
        dgemm(T, T, out, F, F, D, trans_b=True, beta=1.0, batch=C, stride_a=F * D, stride_b=F * D, stride_c=F * F)
    return out

