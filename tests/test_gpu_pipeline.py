"""GPU parity of the corpus drivers (train_extractor / extract_corpus / align_corpus).

Golden fixtures come from the reference's own ``train_extractor`` + ``extract_corpus``
(tests/golden/train.npz, config1.npz = BASELINE config 1).  North-star tolerance: i-vectors,
T and Sigma within 1e-4 relative after a fixed number of EM iterations.
"""

import os
import warnings

import numpy as np
import pytest

import cases

pytestmark = pytest.mark.gpu

TRAIN = cases.load("train")


def _ubms(pkg, cor):
    return pkg.GmmDiag(*cor.diag), pkg.GmmFull(*cor.full)


def _cfg(pkg, cfg_ns, **over):
    from paper_1906_08556_b200.pipeline import TrainConfig
    kw = dict(formulation=cfg_ns.formulation, latent_dim=cfg_ns.latent_dim, iterations=cfg_ns.iterations,
              min_div=cfg_ns.min_div, sigma_update=cfg_ns.sigma_update, update_mean=cfg_ns.update_mean,
              realign_interval=cfg_ns.realign_interval, top_k=cfg_ns.top_k, prune=cfg_ns.prune, seeds=(0,),
              batch_size_utts=cfg_ns.batch_size_utts, workers=1)
    kw.update(over)
    return TrainConfig(**kw)


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("case", cases.TRAIN_CASES, ids=[c[0] for c in cases.TRAIN_CASES])
def test_train_and_extract_match_reference_golden(gpu, case):
    from paper_1906_08556_b200 import pipeline as P
    g = TRAIN[case[0]]
    cor, cfg_ns = cases.train_inputs(case)
    diag, full = _ubms(gpu, cor)
    store = P.InMemoryFeatureStore(cor.features)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        model, metrics = P.train_extractor(_cfg(gpu, cfg_ns), store, diag, full, seed=0)
    np.testing.assert_allclose([r.aux for r in metrics.records], g["aux"], rtol=1e-9)
    assert _rel(model.T, g["T"]) < 1e-6
    assert _rel(model.Sigma, g["Sigma"]) < 1e-6
    np.testing.assert_allclose(model.prior_offset, float(g["prior"]), rtol=1e-9)
    np.testing.assert_allclose(model.ubm_means, g["ubm_means"], rtol=1e-6, atol=1e-9)
    ids, emb = P.extract_corpus(model, store, top_k=cfg_ns.top_k, prune=cfg_ns.prune)
    assert ids == sorted(cor.ids)
    assert _rel(emb, g["ivectors"]) < 1e-6


@pytest.mark.slow
def test_config1_training_matches_reference(gpu):
    """BASELINE config 1: 64-comp UBM, 20-dim, 200 utts x 300 frames, R=100, 5 EM iterations."""
    from paper_1906_08556_b200 import pipeline as P
    g = np.load(os.path.join(cases.HERE, "config1.npz"))
    ids, feats, cfg_ns = cases.config1_inputs()
    diag = gpu.GmmDiag(g["diag_w"], g["diag_mu"], g["diag_var"])
    full = gpu.GmmFull(g["full_w"], g["full_mu"], g["full_cov"])
    store = P.InMemoryFeatureStore(feats)
    model, metrics = P.train_extractor(_cfg(gpu, cfg_ns), store, diag, full, seed=0)
    np.testing.assert_allclose([r.aux for r in metrics.records], g["aux"], rtol=1e-9)
    assert _rel(model.T, g["T"]) < 1e-4
    assert _rel(model.Sigma, g["Sigma"]) < 1e-4
    _, emb = P.extract_corpus(model, store, top_k=20, prune=0.025)
    assert _rel(emb, g["ivectors"]) < 1e-4


@pytest.fixture(scope="module")
def small_world(gpu):
    cor = cases.corpus("augmented", 0, 3, 5, 4, 12, 4, (60, 90), 0.5)
    from paper_1906_08556_b200 import pipeline as P
    return cor, P.InMemoryFeatureStore(cor.features), gpu.GmmDiag(*cor.diag), gpu.GmmFull(*cor.full)


def _config(**overrides):
    from paper_1906_08556_b200.pipeline import TrainConfig
    base = dict(formulation="augmented", latent_dim=4, iterations=3, min_div=True, sigma_update=True,
                realign_interval=0, top_k=3, prune=0.025, seeds=(0,), batch_size_utts=4, workers=1)
    base.update(overrides)
    return TrainConfig(**base)


class TestDrivers:
    def test_align_corpus_equals_per_utterance(self, gpu, small_world):
        from paper_1906_08556_b200 import pipeline as P
        cor, store, diag, full = small_world
        got = P.align_corpus(store, diag, full, top_k=3, prune=0.025)
        for u in cor.ids[:10]:
            want = gpu.align_frames(diag, full, cor.features[u], top_k=3, prune=0.025)
            np.testing.assert_array_equal(got[u].offsets, want.offsets)
            np.testing.assert_array_equal(got[u].components, want.components)
            np.testing.assert_array_equal(got[u].weights, want.weights)

    def test_accumulate_corpus_equals_em_accumulate(self, gpu, small_world):
        from paper_1906_08556_b200 import pipeline as P
        cor, store, diag, full = small_world
        model = gpu.init_model(full, 4, "augmented", seed=0)
        alis = P.align_corpus(store, diag, full, top_k=3, prune=0.025)
        acc = P.accumulate_corpus(model, store, alis, _config())
        stats = [gpu.accumulate_bw_stats(cor.features[u], alis[u], 3) for u in store.ids()]
        want = gpu.em_accumulate(model, stats)
        for key in ("A", "B", "N", "Ssum", "phi_sum", "moment_sum"):
            np.testing.assert_allclose(getattr(acc, key), getattr(want, key), rtol=1e-11, atol=1e-9)
        np.testing.assert_allclose(acc.aux, want.aux, rtol=1e-11)

    def test_metrics_and_monotone_aux(self, gpu, small_world):
        from paper_1906_08556_b200 import pipeline as P
        _, store, diag, full = small_world
        _, metrics = P.train_extractor(_config(iterations=4, min_div=False), store, diag, full)
        aux = np.array([r.aux for r in metrics.records])
        assert len(aux) == 4 and np.all(np.diff(aux) / np.abs(aux[:-1]) > -1e-8)

    def test_two_runs_bit_identical(self, gpu, small_world):
        from paper_1906_08556_b200 import pipeline as P
        _, store, diag, full = small_world
        m1, _ = P.train_extractor(_config(), store, diag, full)
        m2, _ = P.train_extractor(_config(workers=4), store, diag, full)
        assert m1.T.tobytes() == m2.T.tobytes() and m1.Sigma.tobytes() == m2.Sigma.tobytes()
        e1 = P.extract_corpus(m1, store, top_k=3)[1]
        e2 = P.extract_corpus(m1, store, top_k=3)[1]
        assert e1.tobytes() == e2.tobytes()

    def test_checkpoint_resume_bit_exact(self, gpu, small_world, tmp_path):
        from paper_1906_08556_b200 import pipeline as P
        _, store, diag, full = small_world
        ref, _ = P.train_extractor(_config(iterations=3), store, diag, full)
        ck = str(tmp_path / "ck")

        def boom(model, it):
            if it == 2:
                raise RuntimeError("injected failure")

        with pytest.raises(RuntimeError, match="injected"):
            P.train_extractor(_config(iterations=3), store, diag, full, checkpoint_dir=ck, iteration_hook=boom)
        assert os.path.exists(os.path.join(ck, "model_iter_0001.tvm"))
        resumed, metrics = P.train_extractor(_config(iterations=3), store, diag, full, checkpoint_dir=ck,
                                             resume=True)
        assert [r.iteration for r in metrics.records] == [2, 3]
        assert resumed.T.tobytes() == ref.T.tobytes()

    def test_resume_rejects_modified_config(self, gpu, small_world, tmp_path):
        from paper_1906_08556_b200 import pipeline as P
        _, store, diag, full = small_world
        ck = str(tmp_path / "ck")
        P.train_extractor(_config(iterations=1), store, diag, full, checkpoint_dir=ck)
        with pytest.raises(P.PipelineError, match="hash"):
            P.train_extractor(_config(iterations=2), store, diag, full, checkpoint_dir=ck, resume=True)

    def test_alignment_cache_written_and_invalidated(self, gpu, small_world, tmp_path):
        from paper_1906_08556_b200 import pipeline as P
        from paper_1906_08556_b200.io_formats import read_alignment
        cor, store, diag, full = small_world
        ck = str(tmp_path / "ck")
        P.train_extractor(_config(iterations=2), store, diag, full, checkpoint_dir=ck)
        cached = read_alignment(os.path.join(ck, "alignments.aln"))
        want = P.align_corpus(store, diag, full, top_k=3, prune=0.025)
        for u in cor.ids[:5]:
            np.testing.assert_array_equal(cached[u].components, want[u].components)
        # each realignment point (after iterations 1 and 2) removes the cache; iteration 3 writes the
        # realigned one, which must be the alignment under the UBM means updated at iteration 2
        ck2 = str(tmp_path / "ck2")
        seen = {}

        def probe(model, it):
            seen[it] = os.path.exists(os.path.join(ck2, "alignments.aln"))
            seen[f"means{it}"] = model.ubm_means.copy()

        P.train_extractor(_config(iterations=3, realign_interval=1), store, diag, full, checkpoint_dir=ck2,
                          iteration_hook=probe)
        assert seen[1] is False and seen[2] is False and seen[3] is True
        cached2 = read_alignment(os.path.join(ck2, "alignments.aln"))
        m2 = seen["means2"]
        realigned = P.align_corpus(store, gpu.GmmDiag(diag.weights, m2, diag.variances),
                                   gpu.GmmFull(full.weights, m2, full.covariances), top_k=3, prune=0.025)
        assert not np.array_equal(m2, full.means)  # the realignment means did move
        for u in cor.ids:
            np.testing.assert_array_equal(cached2[u].components, realigned[u].components)
            np.testing.assert_array_equal(cached2[u].weights, realigned[u].weights)

    def test_realignment_skipped_on_final_iteration(self, gpu, small_world):
        from paper_1906_08556_b200 import pipeline as P
        _, store, diag, full = small_world
        model, _ = P.train_extractor(_config(iterations=1, realign_interval=1), store, diag, full)
        np.testing.assert_array_equal(model.ubm_means, full.means)

    def test_empty_corpus_rejected(self, gpu, small_world):
        from paper_1906_08556_b200 import pipeline as P
        _, _, diag, full = small_world
        with pytest.raises(P.PipelineError):
            P.train_extractor(_config(), P.InMemoryFeatureStore({}), diag, full)

    def test_empty_utterance_maps_to_prior_mean(self, gpu, small_world):
        from paper_1906_08556_b200 import pipeline as P
        cor, store, diag, full = small_world
        model, _ = P.train_extractor(_config(iterations=1), store, diag, full)
        feats = dict(cor.features)
        feats["zz_empty"] = np.zeros((0, 5), dtype=np.float32)
        ids, emb = P.extract_corpus(model, P.InMemoryFeatureStore(feats), top_k=3)
        np.testing.assert_allclose(emb[ids.index("zz_empty")], model.prior_mean, atol=1e-12)

    def test_standard_with_bias_update(self, gpu, small_world):
        from paper_1906_08556_b200 import pipeline as P
        _, store, diag, full = small_world
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            model, metrics = P.train_extractor(_config(formulation="standard", update_mean=True,
                                                       sigma_update=False, iterations=4), store, diag, full)
        assert np.all(np.isfinite(model.bias)) and len(metrics.records) == 4

    def test_embedding_store_round_trip(self, gpu, small_world, tmp_path):
        from paper_1906_08556_b200 import pipeline as P
        _, store, diag, full = small_world
        model, _ = P.train_extractor(_config(iterations=1), store, diag, full)
        path = str(tmp_path / "emb.fmx")
        ids, emb = P.extract_corpus(model, store, top_k=3, out_path=path)
        ids2, emb2 = P.load_embeddings(path)
        assert ids2 == ids and emb2.tobytes() == emb.tobytes()
