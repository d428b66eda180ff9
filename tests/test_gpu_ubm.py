"""GPU parity of UBM EM training (train_gmm_diag / train_gmm_full, gmm.py:228-373).

(a) Golden fixtures of the reference's own training runs (tests/golden/ubm.npz): models,
    per-iteration log-likelihoods, starvation warnings and the collapse error.
(b) Bit-exact k-means++ seeding against the oracle at sizes where a 1-ulp distance error
    would show up as a different frame draw.
(c) Larger runs against the oracle, with the E-step forced through many frame chunks and
    split-K statistics GEMMs.
"""

import warnings

import numpy as np
import pytest

import cases
from oracle import tvkit_oracle as orc

pytestmark = pytest.mark.gpu

UBM = cases.load("ubm")


def _check_diag(d, g, rtol=1e-9, ll_rtol=1e-11):
    np.testing.assert_allclose(d.weights, g["diag_w"], rtol=rtol, atol=1e-12)
    np.testing.assert_allclose(d.means, g["diag_mu"], rtol=rtol, atol=1e-9)
    np.testing.assert_allclose(d.variances, g["diag_var"], rtol=rtol, atol=1e-12)
    np.testing.assert_allclose(d.training_loglik, g["diag_ll"], rtol=ll_rtol)


def _check_full(f, g, rtol=1e-9, ll_rtol=1e-11):
    np.testing.assert_allclose(f.weights, g["full_w"], rtol=rtol, atol=1e-12)
    np.testing.assert_allclose(f.means, g["full_mu"], rtol=rtol, atol=1e-9)
    np.testing.assert_allclose(f.covariances, g["full_cov"], rtol=rtol, atol=1e-9)
    np.testing.assert_allclose(f.training_loglik, g["full_ll"], rtol=ll_rtol)


@pytest.mark.parametrize("case", cases.UBM_CASES, ids=[c[0] for c in cases.UBM_CASES])
def test_ubm_training_matches_reference_golden(gpu, case):
    name, c, di, fi, seed = case[0], case[6], case[7], case[8], case[9]
    g = UBM[name]
    x = cases.ubm_frames(case)
    assert g["x_digest"][0] == cases.digest(x)
    d = gpu.train_gmm_diag(x, c, n_iters=di, seed=seed)
    _check_diag(d, g)
    f = gpu.train_gmm_full(x, d, n_iters=fi)
    _check_full(f, g)
    assert isinstance(f, gpu.GmmFull) and len(f.training_loglik) == fi


@pytest.mark.parametrize("name,seed", cases.UBM_EDGE_CASES, ids=[c[0] for c in cases.UBM_EDGE_CASES])
def test_ubm_starvation_and_collapse_match_reference(gpu, name, seed):
    g = UBM[name]
    x, c = cases.ubm_edge_frames(seed)
    di, fi = cases.UBM_EDGE_ITERS
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        d = gpu.train_gmm_diag(x, c, n_iters=di, seed=seed)
        nd = len(w)
        # near-singular outlier components (variance at the floor) amplify the rounding of the
        # quadratic-feature log-likelihood; the models themselves still agree to 1e-8
        _check_diag(d, g, rtol=1e-8, ll_rtol=1e-9)
        if "error" in g:
            with pytest.raises(gpu.NumericError) as exc:
                gpu.train_gmm_full(x, d, n_iters=fi)
            assert str(g["error"][0]) == f"NumericError: {exc.value}"
        else:
            _check_full(gpu.train_gmm_full(x, d, n_iters=fi), g, rtol=1e-8, ll_rtol=1e-9)
    assert [nd, len(w) - nd] == list(g["warnings"])
    assert all(issubclass(m.category, RuntimeWarning) and "starved" in str(m.message) for m in w)


def test_ubm_input_validation(gpu):
    with pytest.raises(ValueError, match="n_components"):
        gpu.train_gmm_diag(np.zeros((100, 3)), 0)
    with pytest.raises(ValueError, match="at least 40 frames"):
        gpu.train_gmm_diag(np.zeros((39, 3)), 4)
    with pytest.raises(ValueError, match="empty feature collection"):
        gpu.train_gmm_diag([], 2)
    # a list of utterances is stacked like one matrix
    x = cases.ubm_frames(cases.UBM_CASES[0])
    a = gpu.train_gmm_diag([x[:700], x[700:]], 4, n_iters=3)
    b = gpu.train_gmm_diag(x, 4, n_iters=3)
    np.testing.assert_array_equal(a.means, b.means)
    # zero iterations: the seeded initial model / the expanded diagonal model
    d0 = gpu.train_gmm_diag(x, 4, n_iters=0)
    o0 = orc.train_gmm_diag(x, 4, n_iters=0)
    np.testing.assert_array_equal(d0.means, o0.means)
    f0 = gpu.train_gmm_full(x, d0, n_iters=0)
    np.testing.assert_array_equal(f0.covariances[1], np.diag(d0.variances[1]))


@pytest.mark.parametrize("T,F,C", [(20000, 39, 64), (3000, 7, 300), (50000, 1, 5)])
def test_seeding_is_bit_exact(gpu, T, F, C):
    from paper_1906_08556_b200 import _device, _lib
    rng = np.random.default_rng(T + F)
    x = rng.normal(0.0, 1.0, (T, F)) * rng.uniform(0.1, 10.0, F) + rng.normal(0.0, 5.0, F)
    ours = _device.seed_means(_lib.to_dev(x), x, C, np.random.default_rng(9))
    ref = orc.seed_means(x, C, np.random.default_rng(9))
    np.testing.assert_array_equal(ours, ref)
    # the host-draw fallback steps agree too (dist2 after the first device step)
    rng = np.random.default_rng(9)
    chosen = np.empty((C, F))
    chosen[0] = x[rng.integers(T)]
    dist2 = _lib.to_dev(np.sum((x - chosen[0]) ** 2, axis=1))
    _device._seed_host_steps(_lib.to_dev(x), x, chosen, dist2, 1, rng)
    np.testing.assert_array_equal(chosen, ref)


@pytest.mark.parametrize("chunk", [None, 1 << 14])
def test_larger_training_matches_oracle(gpu, chunk, monkeypatch):
    from paper_1906_08556_b200 import _device
    if chunk is not None:  # force many frame chunks (and split-K statistics GEMMs)
        monkeypatch.setattr(_device, "EM_CHUNK_ELEMS", chunk)
    rng = np.random.default_rng(5)
    centres = rng.normal(0.0, 3.0, (24, 12))
    x = np.concatenate([m + rng.normal(0.0, 1.0, (1500, 12)) * rng.uniform(0.5, 2.0, 12) for m in centres])
    x = x[rng.permutation(len(x))] + 20.0  # an offset like log-energy features
    C = 32
    d = gpu.train_gmm_diag(x, C, n_iters=4, seed=2)
    od = orc.train_gmm_diag(x, C, n_iters=4, seed=2)
    np.testing.assert_allclose(d.means, od.means, rtol=1e-8, atol=1e-8)
    np.testing.assert_allclose(d.variances, od.variances, rtol=1e-8)
    np.testing.assert_allclose(d.training_loglik, od.training_loglik, rtol=1e-11)
    f = gpu.train_gmm_full(x, d, n_iters=3)
    of = orc.train_gmm_full(x, od.weights, od.means, od.variances, n_iters=3)
    np.testing.assert_allclose(f.weights, of.weights, rtol=1e-8)
    np.testing.assert_allclose(f.means, of.means, rtol=1e-8, atol=1e-8)
    np.testing.assert_allclose(f.covariances, of.covariances, rtol=1e-7, atol=1e-9)
    np.testing.assert_allclose(f.training_loglik, of.training_loglik, rtol=1e-11)
    # EM never decreases the likelihood
    assert np.all(np.diff(d.training_loglik) > -1e-6 * abs(d.training_loglik[0]))
    assert np.all(np.diff(f.training_loglik) > -1e-6 * abs(f.training_loglik[0]))


def test_seeding_degenerate_inputs(gpu):
    """All distances zero mid-loop (the reference's rng.integers branch) and NaN frames
    (rng.choice's ValueError): the device loop stops and the host finishes like the reference."""
    from paper_1906_08556_b200 import _device, _lib
    pts = np.array([[0.0, 1.0], [3.0, -2.0], [5.0, 5.0]])
    x = np.repeat(pts, 20, axis=0)[np.random.default_rng(0).permutation(60)]
    for C in (3, 4, 6):
        ours = _device.seed_means(_lib.to_dev(x), x, C, np.random.default_rng(4))
        ref = orc.seed_means(x, C, np.random.default_rng(4))
        np.testing.assert_array_equal(ours, ref)
    # the random stream after seeding is where the reference leaves it
    r1, r2 = np.random.default_rng(4), np.random.default_rng(4)
    _device.seed_means(_lib.to_dev(x), x, 6, r1)
    orc.seed_means(x, 6, r2)
    assert r1.random() == r2.random()
    xn = x.copy()
    xn[7, 1] = np.nan
    with pytest.raises(ValueError, match="Probabilities contain NaN"):
        orc.seed_means(xn, 4, np.random.default_rng(1))
    with pytest.raises(ValueError, match="Probabilities contain NaN"):
        _device.seed_means(_lib.to_dev(xn), xn, 4, np.random.default_rng(1))
