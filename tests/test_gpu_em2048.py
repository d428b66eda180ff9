"""Parity at the EM metric's configuration: C=2048 components, F=60, R=400 (BASELINE configs 3/5).

Goldens (tests/golden/em2048.npz) are the REFERENCE's own ``train_extractor`` + ``extract_corpus``
on 48 utterances x 300 frames drawn by its generator (make_golden.py: make_em2048):

* ``aug2048``: augmented (Kaldi) formulation, 2 EM iterations, min-divergence + Sigma update;
* ``std2048``: standard formulation, 2 iterations, min-divergence + UBM-mean (bias) update and
  realignment after iteration 1 (config 5's per-iteration realignment), no Sigma update.

The device E-step batch is forced down to 16 utterances, so every code path the 20k-utterance
bench runs is exercised here: three accumulation batches, the split-K b-GEMM (K = C*F = 122,880),
``posterior_kernel`` at D=400 (12.5 panels of 32), ``spd_solve_rows`` at D=400 and the F=60
``tvk_spd_small`` of the workspace.  North-star tolerance: T, Sigma and i-vectors within 1e-4
relative, aux within 1e-9.  The goldens hold T/Sigma rows of 8 components verbatim plus per-
component norms / traces and the column sums of T (``cases.em2048_summary``).
"""

import warnings

import numpy as np
import pytest

import cases

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GOLD = cases.load("em2048")
TOL = 1e-4


def _rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("engine", ["int8-all", "default"])
@pytest.mark.parametrize("case", cases.EM2048_CASES, ids=[c[0] for c in cases.EM2048_CASES])
def test_em_at_metric_shape_matches_reference(gpu, monkeypatch, case, engine):
    """``int8-all``: all four E-step contractions on the int8 tensor-core FP64 emulation (the 16-
    utterance batches fall below the size cut for b = F W and B += F' phi otherwise)."""
    from paper_1906_08556_b200 import _estep, pipeline as P
    if engine == "int8-all":
        monkeypatch.setattr(_estep, "I8_MIN_WORK", 0)
    g = GOLD[case[0]]
    cor, kw = cases.em2048_inputs(case)
    assert cases.digest(*[cor.features[u] for u in cor.ids]) == str(g["feat_digest"][0]), "generator drifted"
    monkeypatch.setattr(_estep, "E_STEP_BATCH", 16)
    store = P.InMemoryFeatureStore(cor.features)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        model, metrics = P.train_extractor(P.TrainConfig(**kw), store, gpu.GmmDiag(*cor.diag),
                                           gpu.GmmFull(*cor.full), seed=0)
        ids, emb = P.extract_corpus(model, store, top_k=20, prune=0.025)
    got = cases.em2048_summary(model.T, model.Sigma)
    errs = {k: _rel(got[k], g[k]) for k in got}
    errs["ivectors"] = _rel(emb, g["ivectors"])
    errs["ubm_means"] = _rel(model.ubm_means, g["ubm_means"])
    if model.bias is not None:
        errs["bias"] = _rel(model.bias, g["bias"])
    aux_rel = np.abs(np.array([r.aux for r in metrics.records]) - g["aux"]) / np.abs(g["aux"])
    print(case[0], {k: f"{v:.1e}" for k, v in errs.items()}, "aux", aux_rel)
    assert ids == sorted(cor.ids)
    assert np.all(aux_rel < 1e-9), aux_rel
    np.testing.assert_allclose(model.prior_offset, float(g["prior"]), rtol=1e-9)
    bad = {k: v for k, v in errs.items() if not v < TOL}
    assert not bad, bad
