"""Generate the golden parity fixtures from the REAL reference package.

Runs only in the build container, where the reference tree exists at
``/root/reference`` (read-only).  It imports the reference ``tvkit`` package,
builds seeded synthetic inputs with the oracle's generator recipes (whose
bit-equality with the reference generator is asserted here), runs the
reference hot-path functions and stores their outputs as ``.npz`` fixtures.
Inputs that are cheap to regenerate are stored as seeds plus a checksum; the
tests rebuild them on any box and check the checksum first.

    python tests/golden/make_golden.py        # rewrites tests/golden/*.npz
"""

from __future__ import annotations

import os
import warnings
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import tvkit as ref  # noqa: E402  (the reference, read-only)
from tvkit import gmm as rgmm, pipeline as rpipe, synth as rsynth, tvm as rtvm  # noqa: E402

from oracle import tvkit_oracle as orc  # noqa: E402
sys.path.insert(0, HERE)
from cases import (ALIGN_CASES, TRAIN_CASES, TRAIN_TOPK, TVM_CASES, UBM_CASES, UBM_EDGE_CASES, UBM_EDGE_ITERS,  # noqa: E402
                   digest, ubm_edge_frames, ubm_frames)


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB)")


def ubm_pair(seed, n_comp, dim, mean_sd):
    (w, mu, var), (_, _, cov), _ = orc.posterior_ubm(n_comp, dim, mean_sd, seed)
    return rgmm.GmmDiag(w, mu, var), rgmm.GmmFull(w, mu, cov)


def frames_for(seed, n, dim, scale):
    return np.random.default_rng(seed).normal(0.0, scale, (n, dim))


def make_align():
    out = {}
    for name, us, c, f, sd, fs, n, sc, k, pr in ALIGN_CASES:
        diag, full = ubm_pair(us, c, f, sd)
        x = frames_for(fs, n, f, sc).astype(np.float32)
        ali = rgmm.align_frames(diag, full, x, top_k=k, prune=pr)
        bw = rgmm.accumulate_bw_stats(x, ali, c)
        center = np.random.default_rng(us + 1000).normal(0.0, 1.0, (c, f))
        bwc = rgmm.accumulate_bw_stats(x, ali, c, center_with=center)
        dll = diag.log_likelihoods(x)
        sel = np.argsort(-dll, axis=1, kind="stable")[:, :k]
        srt = -np.sort(-dll, axis=1)
        # the boundary gap between the k-th and (k+1)-th diag log-likelihood (tie diagnostics)
        gap = (srt[:, k - 1] - srt[:, k]) if k < c else np.full(n, np.inf)
        out[name] = dict(
            input_digest=digest(diag.weights, diag.means, diag.variances, full.covariances, x),
            offsets=ali.offsets, components=ali.components, weights=ali.weights,
            selected=sel.astype(np.int32), boundary_gap=gap,
            sel_full_ll=np.take_along_axis(full.log_likelihoods(x), sel, axis=1),
            n=bw.n, f=bw.f, S=bw.S if c * f * f <= 100_000 else np.zeros(0),
            nc=bwc.n, fc=bwc.f, Sc=bwc.S if c * f * f <= 100_000 else np.zeros(0),
        )
    flat = {f"{case}__{k}": v for case, d in out.items() for k, v in d.items()}
    save("align", **flat)


def small_corpus(formulation, seed, c, f, d, spk, ups, frames, within):
    spec = rsynth.SynthSpec(n_components=c, feat_dim=f, latent_dim=d, n_speakers=spk,
                            utts_per_speaker=ups, frames_range=frames, seed=seed,
                            formulation=formulation, within_noise=within, mean_scale=8.0)
    corpus = rsynth.sample_corpus(spec)
    rng = np.random.default_rng(seed)
    gm = orc.generator_model(c, f, d, formulation, 8.0, 100.0, rng)
    ids, feats, _ = orc.sample_utterances(gm, spk, ups, frames, within, rng)
    assert ids == corpus.ids
    for u in ids:
        assert feats[u].tobytes() == corpus.features[u].tobytes(), "oracle generator drifted"
    return corpus


def make_tvm():
    flat = {}
    for name, form, seed, c, f, d, spk, ups, frames, within, rank in TVM_CASES:
        corpus = small_corpus(form, seed, c, f, d, spk, ups, frames, within)
        gen = corpus.model
        ubm_full = gen.alignment_ubm_full()
        ubm_diag = gen.alignment_ubm_diag()
        model = rtvm.init_model(ubm_full, rank, form, seed=seed + 1)
        center = model.bias if form == "standard" else None
        stats = []
        for u in corpus.ids:
            x = np.asarray(corpus.features[u], dtype=np.float64)
            ali = rgmm.align_frames(ubm_diag, ubm_full, x, top_k=min(4, c), prune=0.025)
            stats.append(rgmm.accumulate_bw_stats(x, ali, c, center_with=center))
        ws = rtvm.PosteriorWorkspace(model)
        posts = [rtvm._posterior_terms(model, s, ws) for s in stats]
        acc = rtvm.em_accumulate(model, stats, ws)
        T1 = rtvm.update_T(model, acc)
        S1 = rtvm.update_sigma(model, acc, T1)
        tr = rtvm.compute_min_div(acc, form)
        m2 = model.copy()
        m2.T, m2.Sigma = T1, S1
        if form == "standard":
            rtvm.update_mean_standard(m2, acc.h)
        rtvm.apply_min_div(m2, tr, acc.h)
        d_ = dict(
            feat_digest=digest(*[corpus.features[u] for u in corpus.ids]),
            init_T=model.T,
            ws_W=ws.sinv_T, ws_U=ws.T_sinv_T, ws_Sinv=ws.sigma_inv, ws_logdet=ws.logdet,
            Phi=np.stack([p.Phi for p, _ in posts]), phi=np.stack([p.phi for p, _ in posts]),
            loglik=np.array([ll for _, ll in posts]),
            A=acc.A, B=acc.B, N=acc.N, Ssum=acc.Ssum, phi_sum=acc.phi_sum,
            moment_sum=acc.moment_sum, U=np.array(acc.U), aux=np.array(acc.aux),
            T1=T1, S1=S1, P1=tr.P1, P2=tr.P2, G=tr.G,
            T2=m2.T, prior2=np.array(m2.prior_offset),
            bias2=m2.bias if m2.bias is not None else np.zeros(0),
        )
        for k, v in d_.items():
            flat[f"{name}__{k}"] = v
    save("tvm", **flat)


def make_train():
    flat = {}
    for (name, form, seed, c, f, d, spk, upc, frames, rank, iters, md, su, um, ri) in TRAIN_CASES:
        corpus = small_corpus(form, seed, c, f, d, spk, upc, frames, 0.5)
        gen = corpus.model
        ubm_full = gen.alignment_ubm_full()
        ubm_diag = gen.alignment_ubm_diag()
        cfg = rpipe.TrainConfig(formulation=form, latent_dim=rank, iterations=iters, min_div=md,
                                sigma_update=su, update_mean=um, realign_interval=ri,
                                top_k=TRAIN_TOPK.get(name, 4), prune=0.025, seeds=(0,), batch_size_utts=4,
                                workers=1)
        store = rpipe.InMemoryFeatureStore(corpus.features)
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            model, metrics = rpipe.train_extractor(cfg, store, ubm_diag, ubm_full, seed=0)
        ids, emb = rpipe.extract_corpus(model, store, top_k=TRAIN_TOPK.get(name, 4), prune=0.025)
        d_ = dict(T=model.T, Sigma=model.Sigma, prior=np.array(model.prior_offset),
                  ubm_means=model.ubm_means,
                  bias=model.bias if model.bias is not None else np.zeros(0),
                  aux=np.array([r.aux for r in metrics.records]), ivectors=emb)
        for k, v in d_.items():
            flat[f"{name}__{k}"] = v
    save("train", **flat)


def make_config1():
    """BASELINE config 1: 64-comp UBM, 20-dim, 200 utts x 300 frames, R=100, 5 EM iters.

    The UBM comes from the reference's own UBM trainer (out of scope for the
    GPU build), so its parameters are stored as fixture inputs.
    """
    spec = rsynth.SynthSpec(n_components=64, feat_dim=20, latent_dim=100, n_speakers=50,
                            utts_per_speaker=4, frames_range=(300, 300), seed=0,
                            formulation="augmented", mean_scale=8.0, within_noise=0.3)
    corpus = rsynth.sample_corpus(spec)
    frames = [corpus.features[u] for u in corpus.ids]
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        diag = rgmm.train_gmm_diag(frames, 64, n_iters=10, seed=0)
        full = rgmm.train_gmm_full(frames, diag, n_iters=5)
        cfg = rpipe.TrainConfig(formulation="augmented", latent_dim=100, iterations=5,
                                min_div=True, sigma_update=True, top_k=20, prune=0.025,
                                seeds=(0,), batch_size_utts=8, workers=1, deterministic=True)
        store = rpipe.InMemoryFeatureStore(corpus.features)
        model, metrics = rpipe.train_extractor(cfg, store, diag, full, seed=0)
        ids, emb = rpipe.extract_corpus(model, store, top_k=20, prune=0.025)
    save("config1",
         feat_digest=digest(*frames),
         diag_w=diag.weights, diag_mu=diag.means, diag_var=diag.variances,
         full_w=full.weights, full_mu=full.means, full_cov=full.covariances,
         T=model.T, Sigma=model.Sigma, prior=np.array(model.prior_offset),
         aux=np.array([r.aux for r in metrics.records]), ivectors=emb)


def make_ubm():
    """Reference UBM EM training (gmm.py:246-373) on seeded cluster data."""
    out = {}
    for case in UBM_CASES:
        name, c, di, fi, seed = case[0], case[6], case[7], case[8], case[9]
        x = ubm_frames(case)
        diag = rgmm.train_gmm_diag(x, c, n_iters=di, seed=seed)
        full = rgmm.train_gmm_full(x, diag, n_iters=fi)
        od = orc.train_gmm_diag(x, c, n_iters=di, seed=seed)
        of = orc.train_gmm_full(x, od.weights, od.means, od.variances, n_iters=fi)
        assert np.allclose(od.means, diag.means, rtol=1e-10, atol=1e-10), name
        assert np.allclose(of.covariances, full.covariances, rtol=1e-10, atol=1e-10), name
        out[f"{name}__x_digest"] = np.array([digest(x)])
        out[f"{name}__diag_w"], out[f"{name}__diag_mu"], out[f"{name}__diag_var"] = diag.weights, diag.means, diag.variances
        out[f"{name}__diag_ll"] = np.array(diag.training_loglik)
        out[f"{name}__full_w"], out[f"{name}__full_mu"], out[f"{name}__full_cov"] = full.weights, full.means, full.covariances
        out[f"{name}__full_ll"] = np.array(full.training_loglik)
    di, fi = UBM_EDGE_ITERS
    for name, seed in UBM_EDGE_CASES:
        x, c = ubm_edge_frames(seed)
        out[f"{name}__x_digest"] = np.array([digest(x)])
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            diag = rgmm.train_gmm_diag(x, c, n_iters=di, seed=seed)
            nd = len(w)
            out[f"{name}__diag_w"], out[f"{name}__diag_mu"] = diag.weights, diag.means
            out[f"{name}__diag_var"], out[f"{name}__diag_ll"] = diag.variances, np.array(diag.training_loglik)
            try:
                full = rgmm.train_gmm_full(x, diag, n_iters=fi)
                out[f"{name}__full_w"], out[f"{name}__full_mu"] = full.weights, full.means
                out[f"{name}__full_cov"], out[f"{name}__full_ll"] = full.covariances, np.array(full.training_loglik)
            except Exception as exc:  # the reference's own error is the golden output
                out[f"{name}__error"] = np.array([f"{type(exc).__name__}: {exc}"])
        out[f"{name}__warnings"] = np.array([nd, len(w) - nd])
    save("ubm", **out)


def make_em2048():
    """Reference train_extractor + extract_corpus at C=2048, F=60, D=400 (EM2048_CASES)."""
    import time
    from cases import EM2048_CASES, em2048_inputs, em2048_summary
    out = {}
    for case in EM2048_CASES:
        name = case[0]
        t0 = time.time()
        cor, kw = em2048_inputs(case)
        # the oracle generator must reproduce the reference's sample_corpus bit for bit
        spec = rsynth.SynthSpec(n_components=2048, feat_dim=60, latent_dim=400, n_speakers=case[3],
                                utts_per_speaker=1, frames_range=(300, 300), seed=case[2],
                                formulation=case[1], within_noise=0.3, mean_scale=8.0)
        ref_cor = rsynth.sample_corpus(spec)
        assert ref_cor.ids == cor.ids
        for u in cor.ids:
            assert ref_cor.features[u].tobytes() == cor.features[u].tobytes(), "generator drifted"
        gen = ref_cor.model
        ubm_full, ubm_diag = gen.alignment_ubm_full(), gen.alignment_ubm_diag()
        assert np.array_equal(ubm_full.covariances, cor.full[2])
        cfg = rpipe.TrainConfig(**kw)
        store = rpipe.InMemoryFeatureStore(ref_cor.features)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            model, metrics = rpipe.train_extractor(cfg, store, ubm_diag, ubm_full, seed=0)
            ids, emb = rpipe.extract_corpus(model, store, top_k=20, prune=0.025)
        d = dict(feat_digest=np.array([digest(*[cor.features[u] for u in cor.ids])]),
                 aux=np.array([r.aux for r in metrics.records]), prior=np.array(model.prior_offset),
                 ubm_means=model.ubm_means, bias=model.bias if model.bias is not None else np.zeros(0),
                 ivectors=emb, **em2048_summary(model.T, model.Sigma))
        for k, v in d.items():
            out[f"{name}__{k}"] = v
        print(f"{name}: {time.time() - t0:.0f} s, aux {d['aux']}", flush=True)
    save("em2048", **out)



def make_io():
    """Files written by the reference's own writers (io_formats.py): an ALN1 alignment corpus (from
    reference align_frames on seeded data, including an empty utterance), a TVM1 model of each
    formulation, FMX1 matrices in f32 and f64 and a trial list.  Committed as bytes under
    tests/golden/io/; the drop-in must read them and write byte-identical files."""
    from tvkit import io_formats as rio
    d = os.path.join(HERE, "io")
    os.makedirs(d, exist_ok=True)
    diag, full = ubm_pair(80, 16, 5, 1.0)
    rng = np.random.default_rng(81)
    alis = []
    for u, n in (("spk1-utt1", 40), ("spk1-utt2", 0), ("spk2-utt1", 25), ("spk3-utt7", 57)):
        x = rng.normal(0.0, 1.5, (n, 5)).astype(np.float32)
        alis.append((u, rgmm.align_frames(diag, full, x, top_k=6, prune=0.025)))
    rio.write_alignment(os.path.join(d, "ref.aln"), alis, top_k=6)
    for form, seed in (("augmented", 82), ("standard", 83)):
        m = rtvm.init_model(full, 3, form, seed=seed)
        rio.save_model(m, os.path.join(d, f"ref_{form}.tvm"))
    rio.write_matrix(rng.normal(size=(7, 3)), "f64", os.path.join(d, "ref_f64.fmx"))
    rio.write_matrix(rng.normal(size=(4, 9)).astype(np.float32), "f32", os.path.join(d, "ref_f32.fmx"))
    t = rio.TrialList(["a", "a", "b"], ["x", "y", "x"], np.array([True, False, True]))
    rio.write_trials(os.path.join(d, "ref.trials"), t)
    print("wrote", sorted(os.listdir(d)))


if __name__ == "__main__":
    which = sys.argv[1:] or ["align", "tvm", "train", "config1", "ubm"]
    for w in which:
        globals()[f"make_{w}"]()
