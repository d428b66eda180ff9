"""Golden-case tables and oracle-only input builders.

Shared by ``make_golden.py`` (build container, runs the reference) and the
tests (any box).  Inputs are rebuilt from seeds with the oracle's generator
recipes; each fixture stores a digest of its inputs so a drifting generator is
caught before any comparison.
"""

from __future__ import annotations

import hashlib
import os
from types import SimpleNamespace

import numpy as np

from oracle import tvkit_oracle as orc

HERE = os.path.dirname(os.path.abspath(__file__))

ALIGN_CASES = [
    # name, ubm seed, C, F, mean sd, frame seed, n frames, frame scale, top_k, prune
    ("c8f3", 30, 8, 3, 3.0, 31, 1000, 3.0, 5, 0.025),
    ("c8f3_noprune", 30, 8, 3, 3.0, 32, 200, 3.0, 4, 0.0),
    ("c8f3_degenerate", 30, 8, 3, 3.0, 33, 200, 3.0, 8, 0.9999),
    ("c64f20", 40, 64, 20, 0.5, 41, 2000, 1.5, 20, 0.025),
    ("c256f60", 50, 256, 60, 0.3, 51, 600, 1.2, 20, 0.025),
    ("c2048f60", 60, 2048, 60, 0.3, 61, 300, 1.2, 20, 0.025),
    # outside the fast kernels' envelope (align_wide.cu): top_k > 32, F > 64, top_k == C, no pruning
    ("c128f20_k40", 42, 128, 20, 0.5, 43, 1000, 1.5, 40, 0.025),
    ("c64f80", 44, 64, 80, 0.3, 45, 500, 1.2, 20, 0.025),
    ("c96f80_k48_noprune", 46, 96, 80, 0.3, 47, 300, 1.2, 48, 0.0),
    ("c40f12_kall", 48, 40, 12, 1.0, 49, 400, 2.0, 40, 0.01),
]
WIDE_ALIGN = ("c128f20_k40", "c64f80", "c96f80_k48_noprune", "c40f12_kall")

TVM_CASES = [
    # name, formulation, seed, C, F, D, speakers, utts/spk, frames, within, rank
    ("aug_c4f6", "augmented", 3, 4, 6, 4, 6, 2, (80, 140), 1.0, 4),
    ("std_c4f6", "standard", 4, 4, 6, 4, 6, 2, (80, 140), 1.0, 3),
    ("aug_c16f8", "augmented", 5, 16, 8, 6, 10, 2, (60, 120), 0.5, 6),
]

TRAIN_CASES = [
    # name, formulation, seed, C, F, D, spk, upc, frames, rank, iters, min_div, sigma, update_mean, realign
    ("aug", "augmented", 7, 8, 6, 4, 10, 3, (60, 100), 5, 3, True, True, False, 0),
    ("aug_realign", "augmented", 8, 8, 6, 4, 10, 3, (60, 100), 4, 3, True, True, False, 1),
    ("std_mean", "standard", 9, 8, 6, 4, 10, 3, (60, 100), 4, 3, True, False, True, 1),
    # outside the fast kernels' envelope: 80-dim features (wide selection/whitening, F > 63 BW second
    # order, F > 64 Sigma floor) and top_k = 40 (wide selection + finalize)
    ("aug_f80", "augmented", 10, 8, 80, 4, 6, 2, (40, 60), 4, 2, True, True, False, 1),
    ("aug_k40", "augmented", 11, 48, 6, 4, 6, 2, (60, 100), 4, 2, True, True, False, 1),
]
TRAIN_TOPK = {"aug_k40": 40}  # top_k of the training runs (default 4)

CONFIG1 = dict(n_comp=64, dim=20, rank=100, speakers=50, upc=4, frames=(300, 300), seed=0,
               within=0.3, iterations=5)


UBM_CASES = [
    # name, frame seed, frames per cluster, dim, clusters, spread, C, diag iters, full iters, diag seed
    ("ubm_c4f3", 70, 400, 3, 4, 6.0, 4, 8, 5, 0),
    ("ubm_c16f8", 71, 300, 8, 6, 4.0, 16, 6, 4, 3),
]


def ubm_frames(case):
    """Gaussian clusters around seeded centres (UBM training inputs)."""
    _, fs, per, f, k, spread = case[:6]
    rng = np.random.default_rng(fs)
    centres = rng.normal(0.0, spread, (k, f))
    x = np.concatenate([c + rng.normal(0.0, 1.0, (per, f)) for c in centres])
    return x[rng.permutation(x.shape[0])]


# Outlier-laden inputs (name, seed): starved components (re-seeded in the diagonal EM, frozen in
# the full EM) and a single-frame component whose covariance collapses (NumericError).
UBM_EDGE_CASES = [("ubm_starve7", 7), ("ubm_starve21", 21), ("ubm_collapse0", 0)]
UBM_EDGE_ITERS = (8, 5)


def ubm_edge_frames(seed):
    """(frames, C): a unit cluster of 10*C frames plus 1-5 scattered outliers."""
    rng = np.random.default_rng(seed)
    F, C = 2, int(rng.integers(6, 14))
    nout = int(rng.integers(1, 6))
    x = np.concatenate([rng.normal(0, 1, (10 * C, F)), rng.normal(0, 1, (nout, F)) * rng.uniform(5, 40)])
    return x[rng.permutation(len(x))], C


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def load(name):
    """Fixture ``name`` as {case: {key: array}}."""
    raw = np.load(os.path.join(HERE, f"{name}.npz"))
    out = {}
    for k in raw.files:
        case, key = k.split("__", 1)
        out.setdefault(case, {})[key] = raw[k]
    return out


def align_inputs(case):
    """(diag, full, frames f32, top_k, prune, center) for an ALIGN_CASES row."""
    name, us, c, f, sd, fs, n, sc, k, pr = case
    diag, full, _ = orc.posterior_ubm(c, f, sd, us)
    x = np.random.default_rng(fs).normal(0.0, sc, (n, f)).astype(np.float32)
    center = np.random.default_rng(us + 1000).normal(0.0, 1.0, (c, f))
    return diag, full, x, k, pr, center


def corpus(formulation, seed, c, f, d, spk, ups, frames, within):
    """Oracle restatement of ``synth.sample_corpus`` (bit-identical, asserted at generation)."""
    rng = np.random.default_rng(seed)
    gen = orc.generator_model(c, f, d, formulation, 8.0, 100.0, rng)
    ids, feats, spk_of = orc.sample_utterances(gen, spk, ups, frames, within, rng)
    pc = orc.predictive_covariances(gen)
    diag = (gen.ubm_weights, gen.ubm_means, np.ascontiguousarray(np.diagonal(pc, axis1=1, axis2=2)))
    full = (gen.ubm_weights, gen.ubm_means, pc)
    return SimpleNamespace(ids=ids, features=feats, speakers=spk_of, gen=gen, diag=diag, full=full)


def tvm_inputs(case):
    name, form, seed, c, f, d, spk, ups, frames, within, rank = case
    cor = corpus(form, seed, c, f, d, spk, ups, frames, within)
    model = orc.init_model(cor.full[0], cor.full[1], cor.full[2], rank, form, seed + 1)
    return cor, model, min(4, c)


def train_inputs(case):
    (name, form, seed, c, f, d, spk, upc, frames, rank, iters, md, su, um, ri) = case
    cor = corpus(form, seed, c, f, d, spk, upc, frames, 0.5)
    cfg = SimpleNamespace(formulation=form, latent_dim=rank, iterations=iters, min_div=md,
                          sigma_update=su, update_mean=um, realign_interval=ri, top_k=TRAIN_TOPK.get(name, 4),
                          prune=0.025, prior_offset=100.0, batch_size_utts=4)
    return cor, cfg


def config1_inputs():
    p = CONFIG1
    rng = np.random.default_rng(p["seed"])
    gen = orc.generator_model(p["n_comp"], p["dim"], p["rank"], "augmented", 8.0, 100.0, rng)
    ids, feats, _ = orc.sample_utterances(gen, p["speakers"], p["upc"], p["frames"], p["within"], rng)
    cfg = SimpleNamespace(formulation="augmented", latent_dim=p["rank"], iterations=p["iterations"],
                          min_div=True, sigma_update=True, update_mean=False, realign_interval=0,
                          top_k=20, prune=0.025, prior_offset=100.0, batch_size_utts=8)
    return ids, feats, cfg


# BASELINE config-3 / config-5 shape (C=2048, F=60, D=400) at a corpus size the reference
# finishes in minutes: the EM metric's arithmetic (D=400 posteriors, split-K b-GEMM, multi-batch
# accumulation, update_T at D=400, F=60 workspace) checked against the reference itself.
EM2048_CASES = [
    # name, formulation, generator seed, utterances, iterations, min_div, sigma, update_mean, realign
    ("aug2048", "augmented", 0, 48, 2, True, True, False, 0),
    ("std2048", "standard", 1, 48, 2, True, False, True, 1),
]
EM2048_SHAPE = dict(n_comp=2048, dim=60, rank=400, frames=(300, 300), within=0.3)
# components whose T / Sigma rows are stored verbatim (the rest is pinned by per-component norms)
EM2048_SAMPLE_COMPS = (0, 1, 17, 333, 1024, 1500, 2046, 2047)


def em2048_inputs(case):
    """(corpus namespace, TrainConfig kwargs) for an EM2048_CASES row."""
    name, form, seed, n_utts, iters, md, su, um, ri = case
    p = EM2048_SHAPE
    cor = corpus(form, seed, p["n_comp"], p["dim"], p["rank"], n_utts, 1, p["frames"], p["within"])
    kw = dict(formulation=form, latent_dim=p["rank"], iterations=iters, min_div=md, sigma_update=su,
              update_mean=um, realign_interval=ri, top_k=20, prune=0.025, prior_offset=100.0,
              seeds=(0,), batch_size_utts=8, workers=1)
    return cor, kw


def em2048_summary(T, Sigma):
    """Rotation-sensitive fingerprints of a trained (T, Sigma) small enough to commit."""
    s = list(EM2048_SAMPLE_COMPS)
    return dict(T_rows=T[s], Sigma_rows=Sigma[s], T_norm=np.sqrt(np.einsum("cfd,cfd->c", T, T)),
                T_colsum=T.sum(axis=0), Sigma_trace=np.trace(Sigma, axis1=1, axis2=2))
