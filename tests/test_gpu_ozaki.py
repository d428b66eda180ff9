"""FP64 GEMM emulated on the int8 tensor cores (tvk_dgemm_i8, csrc/ozaki.cu) against a torch FP64
reference of the same product.

Every element must satisfy the scheme's rigorous bound (include/tvk.h):
    |C~ - C| <= (2 + S) 2^(-7 S) K max_k|op(A)_mk| max_k|op(B)_kn|   (+ FP64 rounding of the reference)
Shapes cover partial tiles (M, N not multiples of 128 / 64, K not a multiple of 32), all transposes,
alpha / beta, the split-K path (long K, few tiles), zero and non-finite rows, 6/7/8 digits, bit
reproducibility, and the E-step engine switch end to end.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(gpu, M, N, K, ta, tb, alpha=1.0, beta=0.0, digits=7, seed=0, scale_rows=True):
    from paper_1906_08556_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(seed)
    dev = torch.device("cuda")
    A = torch.randn(*(K, M) if ta else (M, K), device=dev, dtype=torch.float64, generator=g)
    B = torch.randn(*(N, K) if tb else (K, N), device=dev, dtype=torch.float64, generator=g)
    if scale_rows:  # rows / columns spanning many binades
        A = A * torch.exp2(torch.randint(-20, 20, (A.shape[0], 1), device=dev, generator=g).double())
        B = B * torch.exp2(torch.randint(-20, 20, (1, B.shape[1]), device=dev, generator=g).double())
    C0 = torch.randn(M, N, device=dev, dtype=torch.float64, generator=g)
    C = C0.clone()
    _lib.dgemm_i8(A, B, C, M, N, K, trans_a=ta, trans_b=tb, alpha=alpha, beta=beta, digits=digits)
    opA = A.t() if ta else A
    opB = B.t() if tb else B
    ref = alpha * (opA @ opB) + beta * C0
    bound = (2 + digits) * 2.0 ** (-7 * digits) * K * opA.abs().amax(1, keepdim=True) * opB.abs().amax(0, keepdim=True)
    bound = abs(alpha) * bound + 1e-15 * (abs(alpha) * (opA.abs() @ opB.abs()) + abs(beta) * C0.abs())
    return C, ref, bound


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K", [(200, 130, 77), (128, 64, 32), (1, 1, 1), (300, 700, 1000)])
def test_dgemm_i8_within_bound(gpu, M, N, K, ta, tb):
    C, ref, bound = _run(gpu, M, N, K, ta, tb, alpha=-1.5, beta=1.0)
    err = (C - ref).abs()
    assert bool((err <= bound).all()), float((err / bound).max())


@pytest.mark.parametrize("digits", [6, 7, 8])
def test_dgemm_i8_digits_and_split_k(gpu, digits):
    # few output tiles and a long K: the kernel splits K and sums the partials in fixed order
    C, ref, bound = _run(gpu, 100, 90, 40000, False, False, beta=1.0, digits=digits)
    err = (C - ref).abs()
    assert bool((err <= bound).all()), float((err / bound).max())
    rel = float(err.max() / ref.abs().max())
    assert rel < {6: 1e-9, 7: 1e-11, 8: 1e-13}[digits], rel


def test_dgemm_i8_reproducible_and_zero_nan_rows(gpu):
    from paper_1906_08556_b200 import _lib
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(3)
    M, N, K = 257, 129, 300
    A = torch.randn(M, K, device=dev, dtype=torch.float64, generator=g)
    B = torch.randn(K, N, device=dev, dtype=torch.float64, generator=g)
    A[5] = 0.0          # all-zero row -> exact zeros
    B[:, 7] = 0.0       # all-zero column -> exact zeros
    A[9, 3] = float("nan")
    B[11, 20] = float("inf")
    outs = []
    for _ in range(2):
        C = torch.full((M, N), 7.0, device=dev, dtype=torch.float64)
        _lib.dgemm_i8(A, B, C, M, N, K)
        outs.append(C)
    a, b = outs
    assert torch.equal(torch.nan_to_num(a, nan=1.5), torch.nan_to_num(b, nan=1.5))  # bit-reproducible
    # (IEEE agrees: 0 * inf = NaN in the non-finite column, NaN * 0 = NaN in the non-finite row)
    assert bool((a[5][torch.arange(N, device=dev) != 20] == 0).all())
    assert bool((a[:, 7][torch.arange(M, device=dev) != 9] == 0).all())
    assert bool(torch.isnan(a[9]).all()) and bool(torch.isnan(a[:, 20]).all())
    ok = torch.ones(M, N, dtype=torch.bool, device=dev)
    ok[9] = False
    ok[:, 20] = False
    ref = A.nan_to_num(0.0) @ B.nan_to_num(0.0, posinf=0.0)
    assert torch.allclose(a[ok], ref[ok], rtol=1e-11, atol=1e-11)


def test_presplit_operand_matches_inline_split(gpu):
    from paper_1906_08556_b200 import _lib
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(5)
    M, N, K = 300, 200, 1000
    A = torch.randn(M, K, device=dev, dtype=torch.float64, generator=g)
    B = torch.randn(K, N, device=dev, dtype=torch.float64, generator=g)
    for digits in (7, 8):
        c1 = torch.zeros(M, N, device=dev, dtype=torch.float64)
        c2 = torch.zeros(M, N, device=dev, dtype=torch.float64)
        _lib.dgemm_i8(A, B, c1, M, N, K, digits=digits)
        bs = _lib.i8_split_b(B, K, N, digits=digits)
        _lib.dgemm_i8(A, None, c2, M, N, K, digits=digits, b_split=bs)
        assert torch.equal(c1, c2)


def test_estep_engine_int8_matches_dmma(gpu, monkeypatch):
    """One E-step accumulation at C=256, F=24, D=96 on both engines (all four contractions forced onto
    the int8 emulation): accumulators agree to 1e-11 relative."""
    from paper_1906_08556_b200 import _estep, _lib, tvm
    rng = np.random.default_rng(0)
    C, F, D, U = 256, 24, 96, 300
    T = rng.standard_normal((C, F, D)) * 0.3
    Sigma = np.tile(np.eye(F), (C, 1, 1)) * rng.uniform(0.5, 2.0, (C, 1, 1))
    model = tvm.TvModel(formulation="augmented", T=T, Sigma=Sigma, ubm_weights=np.full(C, 1.0 / C),
                        ubm_means=rng.standard_normal((C, F)), prior_offset=10.0)
    n = rng.gamma(0.3, 2.0, (U, C))
    fm = rng.standard_normal((U, C * F)) * n.repeat(F, 1)
    res = {}
    for eng in ("dmma", "int8"):
        monkeypatch.setattr(_estep, "GEMM_ENGINE", eng)
        monkeypatch.setattr(_estep, "I8_MIN_WORK", 0)
        dm = _estep.DeviceModel(model)
        ws = _estep.Workspace(dm)
        acc = _estep.DeviceAcc(C, F, D)
        _estep.accumulate_batch(dm, ws, acc, _lib.to_dev(n), _lib.to_dev(fm))
        res[eng] = {k: _lib.to_host(getattr(acc, k)) for k in ("Apk", "B", "N", "phi_sum", "moment", "aux_post")}
    for k in res["dmma"]:
        a, b = res["int8"][k], res["dmma"][k]
        rel = float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
        assert rel < 1e-11, (k, rel)


def _split_ref(X, RT, S):
    """numpy restatement of the operand split (csrc/ozaki.cu header): row exponents e_r = max frexp
    exponent, digits by the FP64 recurrence d_s = trunc(128 r_{s-1}) on x 2^-e, K-major core-matrix
    tiles [row tile][k-step][digit][RT x 32]."""
    R, K = X.shape
    KST = (K + 31) // 32
    Rp = (R + RT - 1) // RT * RT
    fin = np.isfinite(X).all(1)
    nz = (X != 0).any(1)
    e = np.full(R, np.int32(-1061109568), dtype=np.int64)  # 0xC0C0C0C0
    with np.errstate(invalid="ignore"):
        ex = np.frexp(np.where(np.isfinite(X), X, 0.0))[1]
    ex = np.where(X != 0, ex, -(1 << 30)).max(1)
    e[nz] = ex[nz]
    e[~fin] = 1 << 20
    ok = fin & nz
    V = np.zeros((Rp, KST * 32))
    V[:R, :K] = np.where(ok[:, None], np.ldexp(np.nan_to_num(X), -np.where(ok, e, 0)[:, None].astype(np.int32)), 0.0)
    D = np.zeros((S, Rp, KST * 32), dtype=np.int8)
    for s in range(S):
        V = V * 128.0
        d = np.trunc(V)
        V = V - d
        D[s] = d.astype(np.int8)
    blob = np.zeros((Rp // RT, KST, S, RT * 32), dtype=np.int8)
    rr = np.arange(RT)[:, None]
    kk = np.arange(32)[None, :]
    off = (rr // 8) * 256 + (kk // 16) * 128 + (rr % 8) * 16 + kk % 16
    for rb in range(Rp // RT):
        for ks in range(KST):
            for s in range(S):
                blob[rb, ks, s, off] = D[s, rb * RT:(rb + 1) * RT, ks * 32:(ks + 1) * 32]
    return blob.reshape(-1), e.astype(np.int32)


@pytest.mark.parametrize("digits", [6, 7, 8])
@pytest.mark.parametrize("rows_contiguous", [False, True])
def test_split_digits_match_fp64_recurrence(gpu, digits, rows_contiguous):
    """The integer digit cut is bit-identical to the FP64 recurrence it replaces, signs, zero rows,
    non-finite rows, subnormals and rows spanning many binades included."""
    from paper_1906_08556_b200 import _lib
    rng = np.random.default_rng(11 + digits)
    R, K = 150, 77
    X = rng.standard_normal((R, K)) * np.exp2(rng.integers(-40, 40, (R, 1)))
    X *= np.exp2(rng.integers(-30, 1, (R, K)))  # elements far below their row maximum
    X[3] = 0.0
    X[4, 5] = np.nan
    X[6, 7] = -np.inf
    X[8] = rng.standard_normal(K) * 2.0 ** -1060  # subnormal row
    X[9, :40] = 5e-324
    X[10] = -X[10]
    X[11, 0] = 1.0
    X[11, 1:] = 2.0 ** -60  # digits beyond the last -> 0
    for RT in (64, 128):
        nbytes = int(_lib.load().tvk_i8_operand_bytes(R, K, RT, digits))
        out = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
        if rows_contiguous:  # element (r, k) at r + k R
            src = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
            rs, ks = 1, R
        else:
            src = torch.from_numpy(X).cuda()
            rs, ks = K, 1
        _lib.call("tvk_i8_split", _lib.ptr(src), R, K, rs, ks, RT, digits, _lib.ptr(out), _lib.stream())
        got = out.cpu().numpy()
        blob, e = _split_ref(X, RT, digits)
        assert np.array_equal(got[:blob.size].view(np.int8), blob)
        eoff = (blob.size + 255) // 256 * 256
        assert np.array_equal(got[eoff:eoff + 4 * R].view(np.int32), e)


def test_colsum_paths_bit_identical_and_match_torch(gpu):
    """tvk_colsum: the two-column (16-byte) kernel and the scalar kernel sum every column in the same
    fixed order (bit-identical), and both agree with torch's FP64 sum."""
    from paper_1906_08556_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(9)
    R, Cn = 1037, 4002
    A = torch.randn(R, Cn, device="cuda", dtype=torch.float64, generator=g)
    out_vec = torch.full((Cn,), 0.5, device="cuda", dtype=torch.float64)
    _lib.call("tvk_colsum", _lib.ptr(A), R, Cn, Cn, 2.0, 1.0, _lib.ptr(out_vec), _lib.stream())
    sub = A[:, 1:]  # 8-byte aligned start, odd width: the scalar kernel
    out_sc = torch.full((Cn - 1,), 0.5, device="cuda", dtype=torch.float64)
    _lib.call("tvk_colsum", _lib.ptr(sub), R, Cn - 1, Cn, 2.0, 1.0, _lib.ptr(out_sc), _lib.stream())
    assert torch.equal(out_vec[1:], out_sc)
    assert torch.allclose(out_vec, 0.5 + 2.0 * A.sum(0), rtol=1e-12, atol=1e-12)
