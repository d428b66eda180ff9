"""Shapes outside the fast kernels' envelope (csrc/align_wide.cu): top_k > 32, 80-dim features,
top_k == C, negative / zero top_k semantics of the reference (gmm.py:376-439).

The golden alignment and training cases of these shapes (cases.WIDE_ALIGN, ``aug_f80``,
``aug_k40``) run in test_gpu_align.py / test_gpu_pipeline.py against the reference's outputs; this
file adds the oracle comparisons and the argument semantics.
"""

import numpy as np
import pytest

import cases
from oracle import tvkit_oracle as orc

pytestmark = pytest.mark.gpu
TIE_REL = 1e-9


def _models(gpu, seed, c, f, sd=0.3):
    (w, mu, var), (_, _, cov), _ = orc.posterior_ubm(c, f, sd, seed)
    return gpu.gmm.GmmDiag(w, mu, var), gpu.gmm.GmmFull(w, mu, cov), (w, mu, var), (w, mu, cov)


@pytest.mark.parametrize("c,f,k", [(128, 20, 40), (64, 80, 20), (200, 8, 150), (40, 12, 40)])
def test_select_top_k_wide_matches_stable_argsort(gpu, c, f, k):
    dm, _, diag, _ = _models(gpu, 3, c, f)
    rng = np.random.default_rng(c + f + k)
    for _ in range(5):
        x = rng.normal(0.0, 1.2, f)
        ll = orc.diag_loglik(*diag, x[None, :])[0]
        want = np.argsort(-ll, kind="stable")[:k]
        got = gpu.gmm.select_top_k(dm, x, k)
        srt = -np.sort(-ll)
        # documented ties: equal-within-rounding neighbours may swap
        d = np.abs(np.diff(srt[: min(k + 1, c)]))
        tie = d < TIE_REL * np.maximum(1.0, np.abs(srt[: d.size]))
        if not tie.any():
            np.testing.assert_array_equal(got, want)
        else:
            assert set(got[: np.argmax(tie)]) == set(want[: np.argmax(tie)])


def test_select_top_k_negative_and_zero_k_follow_numpy_slicing(gpu):
    dm, _, diag, _ = _models(gpu, 4, 16, 5)
    x = np.random.default_rng(0).normal(0.0, 1.0, 5)
    ll = orc.diag_loglik(*diag, x[None, :])[0]
    order = np.argsort(-ll, kind="stable")
    assert gpu.gmm.select_top_k(dm, x, 0).size == 0
    np.testing.assert_array_equal(gpu.gmm.select_top_k(dm, x, -3), order[:-3])
    assert gpu.gmm.select_top_k(dm, x, -16).size == 0


def test_align_frames_zero_top_k_raises_like_reference(gpu):
    dm, fm, _, _ = _models(gpu, 5, 8, 3)
    x = np.random.default_rng(1).normal(0.0, 1.0, (4, 3))
    with pytest.raises(ValueError):
        gpu.gmm.align_frames(dm, fm, x, top_k=0)
    with pytest.raises(ValueError):
        gpu.gmm.align_frames(dm, fm, x, top_k=-8)


def test_align_frames_beyond_envelope_raises_value_error(gpu, monkeypatch):
    from paper_1906_08556_b200 import gmm
    dm, fm, _, _ = _models(gpu, 6, 40, 4)
    x = np.random.default_rng(2).normal(0.0, 1.0, (4, 4))
    monkeypatch.setattr(gmm, "MAX_TOP_K", 16)
    with pytest.raises(ValueError, match="top_k"):
        gmm.align_frames(dm, fm, x, top_k=20)


@pytest.mark.parametrize("c,f,k,prune,n", [(128, 20, 40, 0.025, 3000), (64, 80, 20, 0.025, 2000),
                                          (96, 80, 48, 0.0, 500), (48, 100, 33, 0.01, 300)])
def test_wide_alignment_matches_oracle(gpu, c, f, k, prune, n):
    dm, fm, diag, full = _models(gpu, 7 + f, c, f)
    x = np.random.default_rng(c * f).normal(0.0, 1.2, (n, f)).astype(np.float32)
    off, comp, w = orc.align(diag, full, x, k, prune)
    got = gpu.gmm.align_frames(dm, fm, x, top_k=k, prune=prune)
    dll = orc.diag_loglik(*diag, x.astype(np.float64))
    srt = -np.sort(-dll, axis=1)
    gap = srt[:, k - 1] - srt[:, k] if k < c else np.full(n, np.inf)
    ties = set(np.flatnonzero(gap < TIE_REL * np.maximum(1.0, np.abs(srt[:, 0]))).tolist())
    assert len(ties) <= max(1, n // 1000)
    for t in range(n):
        if t in ties:
            continue
        a0, a1, b0, b1 = off[t], off[t + 1], got.offsets[t], got.offsets[t + 1]
        np.testing.assert_array_equal(got.components[b0:b1], comp[a0:a1], err_msg=f"frame {t}")
        np.testing.assert_allclose(got.weights[b0:b1], w[a0:a1], rtol=1e-5, atol=1e-7, err_msg=f"frame {t}")
    got.validate(top_k=k, prune=prune)


def test_wide_alignment_chunked_device_and_host_paths_agree(gpu, monkeypatch):
    from paper_1906_08556_b200 import _device
    dm, fm, _, _ = _models(gpu, 9, 96, 16)
    x = np.random.default_rng(3).normal(0.0, 1.2, (5000, 16)).astype(np.float32)
    one = gpu.gmm.align_frames(dm, fm, x, top_k=64, prune=0.01)
    monkeypatch.setattr(_device, "WIDE_PAIRS", 64 * 700)  # several device chunks / host pieces
    monkeypatch.setattr(_device, "STREAM_CHUNK", 1024)
    host = gpu.gmm.align_frames(dm, fm, x, top_k=64, prune=0.01)
    dev = gpu.gmm.align_frames(dm, fm, _device.frames_to_device(x), top_k=64, prune=0.01)
    for other in (host, dev):
        np.testing.assert_array_equal(other.offsets, one.offsets)
        np.testing.assert_array_equal(other.components, one.components)
        np.testing.assert_array_equal(other.weights, one.weights)


def test_bw_second_order_f80_matches_oracle(gpu):
    """Corpus second-order statistics at F = 80 (the F <= 128 variant of bw_second_order_kernel)."""
    from paper_1906_08556_b200 import _device, _lib
    import torch
    dm, fm, diag, full = _models(gpu, 11, 16, 80)
    rng = np.random.default_rng(5)
    lens = [37, 80, 1, 55]
    x = rng.normal(0.0, 1.2, (sum(lens), 80)).astype(np.float32)
    off, comp, w = orc.align(diag, full, x, 6, 0.0)
    want = np.zeros((16, 80, 80))
    for t in range(x.shape[0]):
        for e in range(off[t], off[t + 1]):
            xt = x[t].astype(np.float64)
            want[comp[e]] += float(w[e]) * np.outer(xt, xt)
    xd = _device.frames_to_device(x)
    uf = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64, device=xd.device)
    ssum = torch.zeros(16 * 80 * 80, dtype=torch.float64, device=xd.device)
    _device.bw_stats(xd, uf, _lib.to_dev(off, torch.int64), _lib.to_dev(comp, torch.int32),
                     _lib.to_dev(w, torch.float32), 16, ssum_acc=ssum)
    got = _lib.to_host(ssum).reshape(16, 80, 80)
    np.testing.assert_allclose(got, want, rtol=1e-11, atol=1e-9)
