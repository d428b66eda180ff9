"""GPU parity of the frame-posterior and Baum-Welch path (libtvk) against the reference.

Compares the CUDA path with (a) the golden fixtures produced by the reference
package and (b) the oracle on the same seeded inputs; also ports the
reference's own alignment/BW tests (pkg/tests/test_gmm.py:159-367).
Tolerances (north star): pruning indices bit-exact except documented ties,
posteriors within 1e-5 relative (weights are float32 on output).
"""

import numpy as np
import pytest

import cases
from oracle import tvkit_oracle as orc

pytestmark = pytest.mark.gpu

ALIGN = cases.load("align")
TIE_REL = 1e-9  # documented tie: diag log-likelihood gap < 1e-9 * max(1, |ll|)


def _pkg():
    import paper_1906_08556_b200 as pkg
    return pkg


def _models(diag, full):
    g = _pkg().gmm
    return g.GmmDiag(*diag), g.GmmFull(*full)


def _assert_alignment_matches(got, off, comp, w, tie_frames=()):
    skip = set(int(t) for t in tie_frames)
    cnt_ref = np.diff(off)
    cnt_got = got.entry_counts()
    for t in range(len(cnt_ref)):
        if t in skip:
            continue
        a0, a1 = off[t], off[t + 1]
        b0, b1 = got.offsets[t], got.offsets[t + 1]
        assert cnt_ref[t] == cnt_got[t], f"frame {t}: entry count {cnt_got[t]} != {cnt_ref[t]}"
        np.testing.assert_array_equal(got.components[b0:b1], comp[a0:a1], err_msg=f"frame {t}")
        np.testing.assert_allclose(got.weights[b0:b1], w[a0:a1], rtol=1e-5, atol=1e-7, err_msg=f"frame {t}")


@pytest.mark.parametrize("case", cases.ALIGN_CASES, ids=[c[0] for c in cases.ALIGN_CASES])
def test_align_matches_reference_golden(gpu, case):
    g = ALIGN[case[0]]
    diag, full, x, k, prune, _ = cases.align_inputs(case)
    dm, fm = _models(diag, full)
    got = gpu.gmm.align_frames(dm, fm, x, top_k=k, prune=prune)
    ties = np.flatnonzero(g["boundary_gap"] < TIE_REL * np.maximum(1.0, np.abs(g["sel_full_ll"][:, 0])))
    assert ties.size <= max(1, x.shape[0] // 1000), f"too many documented ties: {ties.size}"
    _assert_alignment_matches(got, g["offsets"], g["components"], g["weights"], ties)
    got.validate(top_k=k, prune=prune)


@pytest.mark.parametrize("dense", [False, True], ids=["grouped", "dense"])
@pytest.mark.parametrize("case", cases.ALIGN_CASES, ids=[c[0] for c in cases.ALIGN_CASES])
def test_selection_and_full_ll_match_reference(gpu, case, dense):
    g = ALIGN[case[0]]
    diag, full, x, k, prune, _ = cases.align_inputs(case)
    if dense and (k > 32 or x.shape[1] > 96):
        pytest.skip("the dense quadratic-feature mode covers top_k <= 32, F <= 96")
    from paper_1906_08556_b200 import _device, _lib
    dm, fm = _models(diag, full)
    xd = _device.frames_to_device(x)
    res = _device.align(xd, dm.device_table(), fm.device_table(), k, prune, debug=True, dense=dense)
    ties0 = np.flatnonzero(g["boundary_gap"] < TIE_REL * np.maximum(1.0, np.abs(g["sel_full_ll"][:, 0])))
    got = gpu.gmm.SparseAlignment(_lib.to_host(res.offsets), _lib.to_host(res.components[:res.n_entries]),
                                  _lib.to_host(res.weights[:res.n_entries]))
    _assert_alignment_matches(got, g["offsets"], g["components"], g["weights"], ties0)
    sel = _lib.to_host(res.selected)
    ties = g["boundary_gap"] < TIE_REL * np.maximum(1.0, np.abs(g["sel_full_ll"][:, 0]))
    mism = np.flatnonzero(np.any(sel != g["selected"], axis=1) & ~ties)
    assert mism.size == 0, f"selection differs on frames {mism[:10]}"
    ok = ~ties
    sll = _lib.to_host(res.sel_ll)
    np.testing.assert_allclose(sll[ok], g["sel_full_ll"][ok], rtol=1e-10, atol=1e-9)


@pytest.mark.parametrize("case", cases.ALIGN_CASES, ids=[c[0] for c in cases.ALIGN_CASES])
def test_bw_stats_match_reference_golden(gpu, case):
    g = ALIGN[case[0]]
    diag, full, x, k, prune, center = cases.align_inputs(case)
    ali = gpu.gmm.SparseAlignment(g["offsets"], g["components"], g["weights"])
    c = diag[0].shape[0]
    st = gpu.gmm.accumulate_bw_stats(x, ali, c)
    np.testing.assert_allclose(st.n, g["n"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(st.f, g["f"], rtol=1e-12, atol=1e-10)
    if g["S"].size:
        np.testing.assert_allclose(st.S, g["S"], rtol=1e-12, atol=1e-10)
    stc = gpu.gmm.accumulate_bw_stats(x, ali, c, center_with=center)
    assert stc.centered
    np.testing.assert_allclose(stc.f, g["fc"], rtol=1e-12, atol=1e-10)
    if g["Sc"].size:
        np.testing.assert_allclose(stc.S, g["Sc"], rtol=1e-12, atol=1e-10)


def test_dense_loglik_match_oracle(gpu):
    diag, full, x, k, prune, _ = cases.align_inputs(cases.ALIGN_CASES[3])
    dm, fm = _models(diag, full)
    np.testing.assert_allclose(dm.log_likelihoods(x), orc.diag_loglik(*diag, x), rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(fm.log_likelihoods(x), orc.full_loglik(*full, x), rtol=1e-10, atol=1e-9)


# ---------------------------------------------------------------- ported reference tests (test_gmm.py)


def _random_model_pair(rng, c=8, f=3):
    weights = rng.dirichlet(np.full(c, 5.0))
    means = rng.normal(0, 3, (c, f))
    variances = rng.uniform(0.5, 1.5, (c, f))
    covs = np.zeros((c, f, f))
    for i in range(c):
        a = rng.normal(0, 0.3, (f, f))
        covs[i] = np.diag(variances[i]) + a @ a.T
    g = _pkg().gmm
    return g.GmmDiag(weights, means, variances), g.GmmFull(weights, means, covs)


class TestSelectTopK:
    def test_frame_at_component_mean(self, gpu):
        g = gpu.gmm
        model = g.GmmDiag(np.array([1 / 3, 1 / 3, 1 / 3]), np.array([[0.0, 0.0], [5.0, 5.0], [-5.0, 5.0]]),
                          np.ones((3, 2)))
        assert g.select_top_k(model, model.means[0], 1).tolist() == [0]

    def test_matches_dense_posterior_oracle(self, gpu):
        rng = np.random.default_rng(21)
        c, f = 16, 4
        model = gpu.gmm.GmmDiag(rng.dirichlet(np.full(c, 2.0)), rng.normal(0, 2, (c, f)),
                                rng.uniform(0.5, 2.0, (c, f)))
        for _ in range(20):
            frame = rng.normal(0, 2, f)
            got = gpu.gmm.select_top_k(model, frame, 5)
            log_post = model.log_posteriors(frame[None, :])[0]
            want = np.argsort(-log_post, kind="stable")[:5]
            np.testing.assert_array_equal(np.sort(got), np.sort(want))
            np.testing.assert_array_equal(
                got, orc.top_k_single(model.weights, model.means, model.variances, frame, 5))

    def test_k_equals_c_returns_everything(self, gpu):
        model = gpu.gmm.GmmDiag(np.full(4, 0.25), np.zeros((4, 2)), np.ones((4, 2)))
        assert sorted(gpu.gmm.select_top_k(model, np.zeros(2), 4).tolist()) == [0, 1, 2, 3]

    def test_tie_breaks_toward_lower_index(self, gpu):
        model = gpu.gmm.GmmDiag(np.full(3, 1 / 3), np.zeros((3, 2)), np.ones((3, 2)))
        assert gpu.gmm.select_top_k(model, np.ones(2), 2).tolist() == [0, 1]

    def test_k_too_large_rejected(self, gpu):
        model = gpu.gmm.GmmDiag(np.full(2, 0.5), np.zeros((2, 2)), np.ones((2, 2)))
        with pytest.raises(ValueError):
            gpu.gmm.select_top_k(model, np.zeros(2), 3)


class TestAlignFrames:
    def test_invariants_on_random_frames(self, gpu):
        rng = np.random.default_rng(30)
        diag, full = _random_model_pair(rng)
        frames = rng.normal(0, 3, (1000, 3))
        alignment = gpu.gmm.align_frames(diag, full, frames, top_k=5, prune=0.025)
        alignment.validate(top_k=5, prune=0.025)
        sums = np.add.reduceat(alignment.weights.astype(np.float64), alignment.offsets[:-1])
        assert np.max(np.abs(sums - 1.0)) < 1e-5
        assert alignment.weights.min() >= 0.025 - 1e-7
        assert alignment.entry_counts().max() <= 5
        off, comp, w = orc.align((diag.weights, diag.means, diag.variances),
                                 (full.weights, full.means, full.covariances), frames, 5, 0.025)
        _assert_alignment_matches(alignment, off, comp, w)

    def test_symmetric_frame_splits_evenly(self, gpu):
        g = gpu.gmm
        weights = np.array([0.5, 0.5])
        means = np.array([[-1.0, 0.0], [1.0, 0.0]])
        diag = g.GmmDiag(weights, means, np.ones((2, 2)))
        full = g.GmmFull(weights, means, np.stack([np.eye(2), np.eye(2)]))
        alignment = g.align_frames(diag, full, np.zeros((1, 2)), top_k=2, prune=0.025)
        comps, wts = alignment.frame(0)
        np.testing.assert_array_equal(comps, [0, 1])
        np.testing.assert_allclose(wts, [0.5, 0.5], atol=1e-6)

    def test_posteriors_renormalized_over_selection_only(self, gpu):
        from scipy.special import logsumexp
        rng = np.random.default_rng(31)
        diag, full = _random_model_pair(rng, c=6)
        frames = rng.normal(0, 3, (50, 3))
        k = 3
        alignment = gpu.gmm.align_frames(diag, full, frames, top_k=k, prune=0.0)
        full_ll = full.log_likelihoods(frames)
        diag_ll = diag.log_likelihoods(frames)
        for t in range(50):
            sel = np.argsort(-diag_ll[t], kind="stable")[:k]
            expect = np.exp(full_ll[t, sel] - logsumexp(full_ll[t, sel]))
            comps, wts = alignment.frame(t)
            order = np.argsort(sel, kind="stable")
            np.testing.assert_array_equal(comps, np.sort(sel))
            np.testing.assert_allclose(wts, expect[order], atol=1e-6)

    def test_degenerate_frame_keeps_argmax(self, gpu):
        rng = np.random.default_rng(32)
        diag, full = _random_model_pair(rng, c=4)
        frames = rng.normal(0, 3, (200, 3))
        alignment = gpu.gmm.align_frames(diag, full, frames, top_k=4, prune=0.9999)
        assert np.all(alignment.entry_counts() == 1)
        np.testing.assert_allclose(alignment.weights, 1.0)

    def test_model_mismatch_rejected(self, gpu):
        rng = np.random.default_rng(33)
        diag, _ = _random_model_pair(rng, c=4)
        _, full = _random_model_pair(rng, c=5)
        with pytest.raises(ValueError, match="share"):
            gpu.gmm.align_frames(diag, full, np.zeros((1, 3)))

    def test_empty_utterance(self, gpu):
        rng = np.random.default_rng(34)
        diag, full = _random_model_pair(rng)
        assert gpu.gmm.align_frames(diag, full, np.zeros((0, 3))).n_frames == 0


class TestBaumWelchStats:
    def test_empty_utterance_zeros(self, gpu):
        g = gpu.gmm
        stats = g.accumulate_bw_stats(np.zeros((0, 2)), g.SparseAlignment.from_frames([]), 3)
        assert stats.n.sum() == 0 and np.all(stats.f == 0) and np.all(stats.S == 0)
        assert not stats.centered

    def test_single_frame_centered_at_mean(self, gpu):
        g = gpu.gmm
        x = np.array([[1.5, -2.0]])
        ali = g.SparseAlignment.from_frames([(np.array([0]), np.array([1.0], dtype=np.float32))])
        means = np.array([[1.5, -2.0], [0.0, 0.0]])
        stats = g.accumulate_bw_stats(x, ali, 2, center_with=means)
        assert stats.centered
        np.testing.assert_allclose(stats.n, [1.0, 0.0])
        np.testing.assert_allclose(stats.f, 0.0, atol=1e-12)
        np.testing.assert_allclose(stats.S, 0.0, atol=1e-12)

    def test_matches_dense_brute_force(self, gpu):
        rng = np.random.default_rng(40)
        c, f, t = 6, 3, 5
        x = rng.normal(0, 2, (t, f))
        diag, full = _random_model_pair(rng, c=c, f=f)
        alignment = gpu.gmm.align_frames(diag, full, x, top_k=4, prune=0.0)
        stats = gpu.gmm.accumulate_bw_stats(x, alignment, c)
        gamma = np.zeros((t, c))
        for i in range(t):
            comps, wts = alignment.frame(i)
            gamma[i, comps] = wts.astype(np.float64)
        np.testing.assert_allclose(stats.n, gamma.sum(axis=0), atol=1e-9)
        np.testing.assert_allclose(stats.f, gamma.T @ x, atol=1e-9)
        for ci in range(c):
            np.testing.assert_allclose(stats.S[ci], (x * gamma[:, ci, None]).T @ x, atol=1e-9)

    def test_occupancy_sums_to_frame_count(self, gpu):
        rng = np.random.default_rng(41)
        diag, full = _random_model_pair(rng)
        x = rng.normal(0, 3, (321, 3))
        alignment = gpu.gmm.align_frames(diag, full, x, top_k=5, prune=0.025)
        stats = gpu.gmm.accumulate_bw_stats(x, alignment, 8)
        assert abs(stats.n.sum() - 321) < 1e-6
        stats.validate(frame_count=321)

    def test_out_of_range_component_rejected(self, gpu):
        g = gpu.gmm
        ali = g.SparseAlignment.from_frames([(np.array([5]), np.array([1.0], dtype=np.float32))])
        with pytest.raises(ValueError, match="out of range"):
            g.accumulate_bw_stats(np.zeros((1, 2)), ali, 3)

    def test_frame_count_mismatch_rejected(self, gpu):
        g = gpu.gmm
        ali = g.SparseAlignment.from_frames([(np.array([0]), np.array([1.0], dtype=np.float32))])
        with pytest.raises(ValueError, match="frame count"):
            g.accumulate_bw_stats(np.zeros((2, 2)), ali, 3)


def test_dgemm_matches_torch_fp64(gpu):
    import torch
    from paper_1906_08556_b200 import _lib
    rng = np.random.default_rng(0)
    for (m, n, k, ta, tb) in [(1, 1, 1, 0, 0), (5, 7, 3, 0, 0), (130, 70, 33, 1, 0), (200, 300, 129, 0, 1),
                              (257, 129, 64, 1, 1), (1024, 1024, 96, 0, 0)]:
        a = rng.normal(size=(k, m) if ta else (m, k))
        b = rng.normal(size=(n, k) if tb else (k, n))
        want = (a.T if ta else a) @ (b.T if tb else b)
        c = _lib.empty((m, n))
        _lib.dgemm(_lib.to_dev(a), _lib.to_dev(b), c, m, n, k, trans_a=bool(ta), trans_b=bool(tb))
        np.testing.assert_allclose(_lib.to_host(c), want, rtol=1e-12, atol=1e-12 * k)
    # packed-lower output and split-K
    m, k = 200, 1000
    a = rng.normal(size=(m, k))
    want = a @ a.T
    c = _lib.zeros((m * (m + 1) // 2,))
    _lib.dgemm(_lib.to_dev(a), _lib.to_dev(a), c, m, m, k, trans_b=True, out_mode=_lib.TVK_OUT_PACKED_LOWER)
    il = np.tril_indices(m)
    np.testing.assert_allclose(_lib.to_host(c), want[il], rtol=1e-12, atol=1e-10)
    work = _lib.empty((8 * m * m,))
    c2 = _lib.empty((m, m))
    _lib.dgemm(_lib.to_dev(a), _lib.to_dev(a), c2, m, m, k, trans_b=True, splits=8, work=work)
    np.testing.assert_allclose(_lib.to_host(c2), want, rtol=1e-12, atol=1e-10)
    del torch


# ---------------------------------------------------------------- host-input pipeline, tcgen05 preselection


@pytest.mark.parametrize("pinned", [False, True], ids=["numpy", "pinned"])
def test_align_host_chunked_pipeline_matches_single_shot(gpu, monkeypatch, pinned):
    """align_frames on a large HOST input runs the chunked copy/compute/copy pipeline
    (_device.align_host); its CSR must be identical to the one-shot device path."""
    import torch
    (w, mu, var), full, x = orc.posterior_ubm(64, 20, 0.5, seed=21, n_frames=5000)
    dm, fm = gpu.gmm.GmmDiag(w, mu, var), gpu.gmm.GmmFull(*full)
    ref = gpu.gmm.align_frames(dm, fm, torch.from_numpy(x).cuda(), top_k=20, prune=0.025)
    monkeypatch.setattr(gpu._device, "STREAM_CHUNK", 1234)
    feats = torch.from_numpy(x).pin_memory() if pinned else x
    got = gpu.gmm.align_frames(dm, fm, feats, top_k=20, prune=0.025)
    np.testing.assert_array_equal(got.offsets, ref.offsets)
    np.testing.assert_array_equal(got.components, ref.components)
    np.testing.assert_array_equal(got.weights, ref.weights)


def _select(gpu, x, dm, k, mode, monkeypatch, values=True):
    import torch
    monkeypatch.setenv("TVK_SELECT", mode)
    xd = gpu._device.frames_to_device(x)
    sel, val = gpu._device.select_topk(xd, dm.device_table(), k, values=values)
    torch.cuda.synchronize()
    return sel.cpu().numpy(), (val.cpu().numpy() if val is not None else None)


@pytest.mark.parametrize("C,F,k,sd", [(2048, 60, 20, 0.3), (100, 13, 7, 0.5), (300, 63, 32, 0.5), (20, 5, 20, 0.5),
                                      (129, 8, 1, 0.5), (700, 24, 20, 3.0), (2100, 40, 20, 0.3),
                                      (16384, 20, 20, 0.3)],
                         ids=["config2", "C100", "F63K32", "C=K", "K1", "spread", "odd_pair", "C16384"])
def test_tensor_core_preselection_is_exact(gpu, monkeypatch, C, F, k, sd):
    """The 3xTF32 tcgen05 preselection (select_tc.cu) returns exactly the stable top-K of the FP64
    scores: same indices and order as the FP64 DMMA kernel and the oracle's stable argsort."""
    (w, mu, var), _, x = orc.posterior_ubm(C, F, sd, seed=C + F, n_frames=3000)
    dm = gpu.gmm.GmmDiag(w, mu, var)
    a, av = _select(gpu, x, dm, k, "tc", monkeypatch)
    ll = orc.diag_loglik(w, mu, var, x.astype(np.float64))
    ref = np.argsort(-ll, axis=1, kind="stable")[:, :k]
    np.testing.assert_array_equal(a, ref)
    np.testing.assert_allclose(av, np.take_along_axis(ll, ref, 1), rtol=1e-12, atol=1e-9)
    if F <= 60 and k <= 20:
        b, _ = _select(gpu, x, dm, k, "dmma", monkeypatch)
        np.testing.assert_array_equal(a, b)


def test_tensor_core_preselection_exact_ties_and_degenerate_frames(gpu, monkeypatch):
    """Duplicated components (exact ties -> lower index first), all-zero and NaN frames (the exact
    fallback kernel) and frames whose windows overflow under a deliberately tiny pass-0 slack."""
    (w, mu, var), _, x = orc.posterior_ubm(64, 10, 0.5, seed=9, n_frames=1000)
    mu[32:], var[32:], w[32:] = mu[:32], var[:32], w[:32]
    w = w / w.sum()
    x[5] = 0.0
    x[7, 3] = np.nan
    dm = gpu.gmm.GmmDiag(w, mu, var)
    ll = orc.diag_loglik(w, mu, var, x.astype(np.float64))
    ref = np.argsort(-ll, axis=1, kind="stable")[:, :20]
    for kappa1 in (None, "1e-9", "1.0"):
        if kappa1:
            monkeypatch.setenv("TVK_SELECT_KAPPA1", kappa1)
        a, _ = _select(gpu, x, dm, 20, "tc", monkeypatch, values=False)
        ok = np.ones(len(x), bool)
        ok[7] = False  # NaN frame: the reference order of NaN scores is index order (checked below)
        np.testing.assert_array_equal(a[ok], ref[ok])
        np.testing.assert_array_equal(a[7], np.arange(20))


@pytest.mark.parametrize("T", [1, 127, 129, 5000, 60000])
def test_tensor_core_preselection_stable_across_runs_and_tile_counts(gpu, monkeypatch, T):
    """Every CTA's first and last tiles (tile-boundary staging of frames and A operands) give the
    exact FP64 top-K, identically on repeated runs; differences from the oracle's stable argsort are
    only documented ties (adjacent scores within 1e-9 relative)."""
    (w, mu, var), _, x = orc.posterior_ubm(256, 40, 0.4, seed=T, n_frames=T)
    dm = gpu.gmm.GmmDiag(w, mu, var)
    first, _ = _select(gpu, x, dm, 20, "tc", monkeypatch, values=False)
    for _ in range(3):
        a, _ = _select(gpu, x, dm, 20, "tc", monkeypatch, values=False)
        np.testing.assert_array_equal(a, first)
    ll = orc.diag_loglik(w, mu, var, x.astype(np.float64))
    ref = np.argsort(-ll, axis=1, kind="stable")[:, :20]
    bad = np.flatnonzero((first != ref).any(1))
    for t in bad:  # same multiset of scores up to ties at the 1e-9 level
        np.testing.assert_allclose(np.sort(ll[t, first[t]]), np.sort(ll[t, ref[t]]), rtol=1e-9, atol=0)
    assert bad.size <= max(1, T // 1000)


@pytest.mark.parametrize("C,T,xf64", [(64, 60000, False), (300, 20000, True)], ids=["c64_many_tiles", "c300_f64"])
def test_whitening_kernel_many_tiles_matches_oracle_and_is_reproducible(gpu, C, T, xf64):
    """whiten_ll_kernel (selected-pair full-covariance LLs, FP64 DMMA): many tiles per CTA with
    component switches; values equal the oracle's Cholesky/solve LLs to 1e-11 and are bit-identical
    between runs."""
    import torch
    from paper_1906_08556_b200 import _lib
    (w, mu, var), full, x = orc.posterior_ubm(C, 20, 0.5, seed=C, n_frames=T)
    if xf64:
        x = x.astype(np.float64)
    fm = gpu.gmm.GmmFull(*full)
    tab = fm.device_table()
    rng = np.random.default_rng(1)
    sel = np.stack([rng.permutation(C)[:20] for _ in range(T)]).astype(np.int32)
    xd = gpu._device.frames_to_device(x)
    seld = torch.from_numpy(sel).cuda()
    outs = []
    for _ in range(2):
        out = _lib.empty((T, 20))
        nbytes = int(_lib.load().tvk_full_loglik_workspace_bytes(T, 20, C))
        ws = _lib.empty((nbytes,), torch.uint8)
        xp, xfl = _lib.x_args(xd)
        _lib.call("tvk_full_loglik_selected", xp, xfl, T, 20, None, _lib.ptr(tab.prec), C, 20, 0, _lib.ptr(seld),
                  _lib.ptr(out), _lib.ptr(ws), nbytes, _lib.stream())
        outs.append(out.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
    ll = orc.full_loglik(*full, x[:2000].astype(np.float64))
    np.testing.assert_allclose(outs[0][:2000], np.take_along_axis(ll, sel[:2000], 1), rtol=1e-11, atol=1e-9)


@pytest.mark.parametrize("case", cases.ALIGN_CASES, ids=[c[0] for c in cases.ALIGN_CASES])
def test_sparse_align_path_matches_reference_golden(gpu, monkeypatch, case):
    """Opt-in approximate (tcgen05 3xTF32) + exact (FP64 on kept/ambiguous pairs) stage 2-3 path
    (TVK_ALIGN_SPARSE=1): the same alignment as the reference goldens."""
    monkeypatch.setenv("TVK_ALIGN_SPARSE", "1")
    g = ALIGN[case[0]]
    diag, full, x, k, prune, _ = cases.align_inputs(case)
    dm, fm = _models(diag, full)
    got = gpu.gmm.align_frames(dm, fm, x, top_k=k, prune=prune)
    ties = np.flatnonzero(g["boundary_gap"] < TIE_REL * np.maximum(1.0, np.abs(g["sel_full_ll"][:, 0])))
    _assert_alignment_matches(got, g["offsets"], g["components"], g["weights"], ties)


@pytest.mark.parametrize("F,long_run", [(60, False), (60, True), (20, False), (64, True), (80, False)])
def test_corpus_second_order_sum_matches_numpy(gpu, F, long_run):
    """tvk_bw_stats' corpus second-order sum Ssum_c += sum w (x - m_c)(x - m_c)^T (tvm.py:304) -- the DMMA
    kernel for F <= 64, the FMA kernel above -- against numpy, including a component run longer than the
    kernel's 4096-entry position window (one 9000-frame utterance aligned to component 0)."""
    import torch
    from paper_1906_08556_b200 import _device, _lib
    rng = np.random.default_rng(F + long_run)
    C = 48
    lens = [9000, 120, 300] if long_run else list(rng.integers(1, 400, 40))
    T = int(sum(lens))
    x = rng.standard_normal((T, F)).astype(np.float32)
    comps, wts, off = [], [], [0]
    for t in range(T):
        k = int(rng.integers(1, 5))
        cs = np.sort(rng.choice(C, k, replace=False))
        if long_run and t < 9000:
            cs = np.unique(np.concatenate([[0], cs]))
        w = rng.random(len(cs)).astype(np.float32)
        comps += list(cs)
        wts += list(w / w.sum())
        off.append(len(comps))
    comps, wts, off = np.array(comps, np.int32), np.array(wts, np.float32), np.array(off, np.int64)
    center = rng.standard_normal((C, F))
    utt = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ssum = _lib.zeros((C, F, F))
    _device.bw_stats(_lib.to_dev(x), _lib.to_dev(utt, torch.int64), _lib.to_dev(off, torch.int64),
                     _lib.to_dev(comps, torch.int32), _lib.to_dev(wts, torch.float32), C,
                     center=_lib.to_dev(center), ssum_acc=ssum)
    got = _lib.to_host(ssum)
    ref = np.zeros((C, F, F))
    fr = np.repeat(np.arange(T), np.diff(off))
    xd = x.astype(np.float64)
    for c in range(C):
        m = comps == c
        y = xd[fr[m]] - center[c]
        ref[c] = (y * wts[m].astype(np.float64)[:, None]).T @ y
    assert np.array_equal(got, np.swapaxes(got, 1, 2))  # exactly symmetric
    np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_tensor_core_preselection_exact_at_scale(gpu, monkeypatch):
    """2e5 config-2 frames (1563 frame tiles, every window / overflow / flagged-frame path exercised
    many times): the tcgen05 preselection is index-identical to the FP64 DMMA kernel; a 3000-frame
    slice also matches the oracle's stable argsort (gmm.py:409-410)."""
    (w, mu, var), _, x = orc.posterior_ubm(2048, 60, 0.3, seed=77, n_frames=200_000)
    dm = gpu.gmm.GmmDiag(w, mu, var)
    a, _ = _select(gpu, x, dm, 20, "tc", monkeypatch)
    b, _ = _select(gpu, x, dm, 20, "dmma", monkeypatch)
    np.testing.assert_array_equal(a, b)
    ll = orc.diag_loglik(w, mu, var, x[:3000].astype(np.float64))
    np.testing.assert_array_equal(a[:3000], np.argsort(-ll, axis=1, kind="stable")[:, :20])


def test_align_host_many_pieces_full_entries_match_device_path(gpu, monkeypatch):
    """The host pipeline at prune 0 (every top-K entry kept: the largest copy-outs) over many pieces,
    including the ramp pieces: piece outputs freed on the compute stream must not be reused while
    their device->host copies run (record_stream on the drain stream), so the CSR is identical to the
    one-shot device alignment."""
    import torch
    (w, mu, var), full, x = orc.posterior_ubm(256, 20, 0.5, seed=5, n_frames=200_000)
    dm, fm = gpu.gmm.GmmDiag(w, mu, var), gpu.gmm.GmmFull(*full)
    ref = gpu.gmm.align_frames(dm, fm, torch.from_numpy(x).cuda(), top_k=20, prune=0.0)
    monkeypatch.setattr(gpu._device, "STREAM_CHUNK", 8192)
    monkeypatch.setattr(gpu._device, "RAMP_PIECE", 2048)
    got = gpu.gmm.align_frames(dm, fm, torch.from_numpy(x).pin_memory(), top_k=20, prune=0.0)
    assert got.components.shape[0] == 20 * x.shape[0]
    np.testing.assert_array_equal(got.offsets, ref.offsets)
    np.testing.assert_array_equal(got.components, ref.components)
    np.testing.assert_array_equal(got.weights, ref.weights)


def test_align_host_path_rejects_non_spd_model(gpu, monkeypatch):
    """Host pipeline: the full-covariance tables are built while the first piece of frames is copied,
    and a non-SPD covariance still raises the reference's LinAlgError before any alignment kernel."""
    import torch
    (w, mu, var), (wf, muf, cov), x = orc.posterior_ubm(64, 20, 0.5, seed=23, n_frames=5000)
    cov = cov.copy()
    cov[5] = -np.eye(20)
    dm, fm = gpu.gmm.GmmDiag(w, mu, var), gpu.gmm.GmmFull(wf, muf, cov)
    monkeypatch.setattr(gpu._device, "STREAM_CHUNK", 1000)
    with pytest.raises(np.linalg.LinAlgError):
        gpu.gmm.align_frames(dm, fm, torch.from_numpy(x).pin_memory(), top_k=20, prune=0.025)
    good = gpu.gmm.GmmFull(wf, muf, orc.posterior_ubm(64, 20, 0.5, seed=23)[1][2])
    ali = gpu.gmm.align_frames(dm, good, torch.from_numpy(x).pin_memory(), top_k=20, prune=0.025)
    assert ali.offsets.shape[0] == 5001  # the pipeline is usable after the failed call
