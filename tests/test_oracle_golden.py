"""Pin the CPU oracle to the real reference through the committed golden fixtures.

CPU only.  If these pass, every GPU parity test that compares against the
oracle is (transitively) a comparison against the reference package.
"""

import warnings

import numpy as np
import pytest

import cases
from oracle import tvkit_oracle as orc

ALIGN = cases.load("align")
TVM = cases.load("tvm")
TRAIN = cases.load("train")


@pytest.mark.parametrize("case", cases.ALIGN_CASES, ids=[c[0] for c in cases.ALIGN_CASES])
def test_align_and_bw_match_reference(case):
    g = ALIGN[case[0]]
    diag, full, x, k, prune, center = cases.align_inputs(case)
    assert cases.digest(diag[0], diag[1], diag[2], full[2], x) == str(g["input_digest"])
    off, comp, w = orc.align(diag, full, x, k, prune)
    np.testing.assert_array_equal(off, g["offsets"])
    np.testing.assert_array_equal(comp, g["components"])
    np.testing.assert_allclose(w, g["weights"], rtol=1e-6, atol=1e-7)
    c = diag[0].shape[0]
    n, f, S = orc.bw_stats(x, off, comp, w, c)
    np.testing.assert_allclose(n, g["n"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(f, g["f"], rtol=1e-12, atol=1e-10)
    if g["S"].size:
        np.testing.assert_allclose(S, g["S"], rtol=1e-12, atol=1e-10)
    n2, f2, S2 = orc.bw_stats(x, off, comp, w, c, center)
    np.testing.assert_allclose(f2, g["fc"], rtol=1e-12, atol=1e-10)
    if g["Sc"].size:
        np.testing.assert_allclose(S2, g["Sc"], rtol=1e-12, atol=1e-10)


@pytest.mark.parametrize("case", cases.TVM_CASES, ids=[c[0] for c in cases.TVM_CASES])
def test_tvm_steps_match_reference(case):
    g = TVM[case[0]]
    cor, model, k = cases.tvm_inputs(case)
    assert cases.digest(*[cor.features[u] for u in cor.ids]) == str(g["feat_digest"])
    np.testing.assert_array_equal(model.T, g["init_T"])
    c = model.T.shape[0]
    center = model.bias if model.formulation == "standard" else None
    stats = []
    for u in cor.ids:
        ali = orc.align(cor.diag, cor.full, cor.features[u], k, 0.025)
        stats.append(orc.bw_stats(cor.features[u], *ali, c, center))
    ws = orc.workspace(model)
    np.testing.assert_allclose(ws.U, g["ws_U"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ws.W, g["ws_W"], rtol=1e-12, atol=1e-12)
    posts = [orc.posterior(model, *s, ws) for s in stats]
    np.testing.assert_allclose(np.stack([p[0] for p in posts]), g["Phi"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(np.stack([p[1] for p in posts]), g["phi"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose([p[2] for p in posts], g["loglik"], rtol=1e-10)
    acc = orc.accumulate(model, stats, ws)
    for key in ("A", "B", "N", "Ssum", "phi_sum", "moment_sum"):
        np.testing.assert_allclose(getattr(acc, key), g[key], rtol=1e-10, atol=1e-9)
    assert acc.U == int(g["U"])
    np.testing.assert_allclose(acc.aux, float(g["aux"]), rtol=1e-12)
    T1 = orc.update_T(model, acc)
    np.testing.assert_allclose(T1, g["T1"], rtol=1e-9, atol=1e-10)
    S1 = orc.update_sigma(model, acc, T1)
    np.testing.assert_allclose(S1, g["S1"], rtol=1e-9, atol=1e-10)
    tr = orc.min_div(acc, model.formulation)
    np.testing.assert_allclose(tr.P1, g["P1"], rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(tr.P2, g["P2"], rtol=1e-8, atol=1e-9)
    model.T, model.Sigma = T1, S1
    if model.formulation == "standard":
        orc.update_mean_standard(model, acc.phi_sum / acc.U)
        np.testing.assert_allclose(model.bias, g["bias2"], rtol=1e-9, atol=1e-9)
    orc.apply_min_div(model, tr, acc.phi_sum / acc.U)
    np.testing.assert_allclose(model.T, g["T2"], rtol=1e-8, atol=1e-9)
    np.testing.assert_allclose(model.prior_offset, float(g["prior2"]), rtol=1e-10)


@pytest.mark.parametrize("case", cases.TRAIN_CASES, ids=[c[0] for c in cases.TRAIN_CASES])
def test_training_loop_matches_reference(case):
    g = TRAIN[case[0]]
    cor, cfg = cases.train_inputs(case)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        model, aux = orc.train(cfg, cor.features, cor.ids, cor.diag, cor.full, seed=0)
        emb = orc.extract_corpus(model, cor.features, cor.ids, 4, 0.025)
    np.testing.assert_allclose(aux, g["aux"], rtol=1e-9)
    np.testing.assert_allclose(model.T, g["T"], rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(model.Sigma, g["Sigma"], rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(emb, g["ivectors"], rtol=1e-6, atol=1e-6)


@pytest.mark.slow
def test_config1_training_matches_reference():
    g = np.load(cases.HERE + "/config1.npz")
    ids, feats, cfg = cases.config1_inputs()
    assert cases.digest(*[feats[u] for u in ids]) == str(g["feat_digest"])
    diag = (g["diag_w"], g["diag_mu"], g["diag_var"])
    full = (g["full_w"], g["full_mu"], g["full_cov"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        model, aux = orc.train(cfg, feats, ids, diag, full, seed=0)
    np.testing.assert_allclose(aux, g["aux"], rtol=1e-9)
    np.testing.assert_allclose(model.T, g["T"], rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(model.Sigma, g["Sigma"], rtol=1e-6, atol=1e-8)


def test_householder_and_min_div_properties():
    rng = np.random.default_rng(0)
    for d in (2, 5, 40):
        v = rng.normal(0, 3, d)
        p2 = orc.householder(v)
        np.testing.assert_allclose(p2 @ p2, np.eye(d), atol=1e-10)
        np.testing.assert_allclose((p2 @ v)[1:], 0.0, atol=1e-10 * max(1, np.linalg.norm(v)))
    np.testing.assert_array_equal(orc.householder(np.array([2.5, 0.0, 0.0])), np.eye(3))


UBM = cases.load("ubm")


@pytest.mark.parametrize("case", cases.UBM_CASES, ids=[c[0] for c in cases.UBM_CASES])
def test_ubm_training_matches_reference(case):
    """Oracle UBM EM (gmm.py:246-373) against the reference's own run."""
    name, c, di, fi, seed = case[0], case[6], case[7], case[8], case[9]
    x = cases.ubm_frames(case)
    assert UBM[name]["x_digest"][0] == cases.digest(x)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        d = orc.train_gmm_diag(x, c, n_iters=di, seed=seed)
        f = orc.train_gmm_full(x, d.weights, d.means, d.variances, n_iters=fi)
    np.testing.assert_allclose(d.weights, UBM[name]["diag_w"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(d.means, UBM[name]["diag_mu"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(d.variances, UBM[name]["diag_var"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(d.training_loglik, UBM[name]["diag_ll"], rtol=1e-12)
    np.testing.assert_allclose(f.weights, UBM[name]["full_w"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(f.means, UBM[name]["full_mu"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(f.covariances, UBM[name]["full_cov"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(f.training_loglik, UBM[name]["full_ll"], rtol=1e-12)


@pytest.mark.parametrize("name,seed", cases.UBM_EDGE_CASES, ids=[c[0] for c in cases.UBM_EDGE_CASES])
def test_ubm_edge_cases_match_reference(name, seed):
    """Starved components and collapsed covariances: warnings, re-seeding and errors as the reference."""
    g = UBM[name]
    x, c = cases.ubm_edge_frames(seed)
    assert g["x_digest"][0] == cases.digest(x)
    di, fi = cases.UBM_EDGE_ITERS
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        d = orc.train_gmm_diag(x, c, n_iters=di, seed=seed)
        nd = len(w)
        np.testing.assert_allclose(d.means, g["diag_mu"], rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(d.variances, g["diag_var"], rtol=1e-10, atol=1e-12)
        if "error" in g:
            with pytest.raises(orc.OracleNumericError) as exc:
                orc.train_gmm_full(x, d.weights, d.means, d.variances, n_iters=fi)
            assert str(exc.value) in str(g["error"][0])
        else:
            f = orc.train_gmm_full(x, d.weights, d.means, d.variances, n_iters=fi)
            np.testing.assert_allclose(f.covariances, g["full_cov"], rtol=1e-9, atol=1e-10)
    assert [nd, len(w) - nd] == list(g["warnings"])
