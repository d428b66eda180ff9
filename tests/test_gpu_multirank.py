"""Multi-rank drivers on one B200: ``train_extractor``, ``extract_corpus`` and ``accumulate_corpus``
at world_size 2 (gloo over CUDA tensors, both ranks on cuda:0), against the single-process run.

The sharded trainer keeps a contiguous utterance shard per rank, sums the flat E-step accumulator
with one all-reduce per iteration and replicates the M-step; the reference merges per-batch
accumulators by addition (tvm.py:271-280, ``EmAccumulators.merge``), so the results agree up to
the summation order of the two shard sums.  Rank 0 alone writes checkpoints; a world-2 run that
fails mid-training resumes from them bit-exactly.
"""

import os
import socket
import warnings

import numpy as np
import pytest
import torch.multiprocessing as mp

import cases

pytestmark = pytest.mark.gpu

CASE = ("aug_realign", "augmented", 8, 8, 6, 4, 10, 3, (60, 100), 4, 3, True, True, False, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _config(P, cfg_ns, **over):
    kw = dict(formulation=cfg_ns.formulation, latent_dim=cfg_ns.latent_dim, iterations=cfg_ns.iterations,
              min_div=cfg_ns.min_div, sigma_update=cfg_ns.sigma_update, update_mean=cfg_ns.update_mean,
              realign_interval=cfg_ns.realign_interval, top_k=cfg_ns.top_k, prune=cfg_ns.prune, seeds=(0,),
              batch_size_utts=cfg_ns.batch_size_utts, workers=1)
    kw.update(over)
    return P.TrainConfig(**kw)


def _run(P, pkg, cor, cfg_ns, ckpt=None, fail_at=None, resume=False):
    """train_extractor + extract_corpus + accumulate_corpus on the current process group."""
    store = P.InMemoryFeatureStore(cor.features)
    diag, full = pkg.GmmDiag(*cor.diag), pkg.GmmFull(*cor.full)

    def hook(model, it):
        if fail_at is not None and it == fail_at:
            raise RuntimeError("injected failure")

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        model, metrics = P.train_extractor(_config(P, cfg_ns), store, diag, full, seed=0, checkpoint_dir=ckpt,
                                           resume=resume, iteration_hook=hook)
        ids, emb = P.extract_corpus(model, store, top_k=cfg_ns.top_k, prune=cfg_ns.prune)
        alis = P.align_corpus(store, diag, full, top_k=cfg_ns.top_k, prune=cfg_ns.prune)
        acc = P.accumulate_corpus(model, store, alis, _config(P, cfg_ns))
    return dict(T=model.T, Sigma=model.Sigma, prior=np.array(model.prior_offset), ubm_means=model.ubm_means,
                aux=np.array([r.aux for r in metrics.records]), iters=np.array([r.iteration for r in metrics.records]),
                ivectors=emb, ids=np.array(ids), acc_B=acc.B, acc_N=acc.N, acc_A=acc.A, acc_aux=np.array(acc.aux),
                acc_U=np.array(acc.U))


def _worker(rank, world, port, out_dir, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1906_08556_b200 as pkg
    from paper_1906_08556_b200 import pipeline as P
    cor, cfg_ns = cases.train_inputs(CASE)
    ckpt = os.path.join(out_dir, "ckpt")
    try:
        if mode == "plain":
            res = _run(P, pkg, cor, cfg_ns)
        elif mode == "fail":
            try:
                _run(P, pkg, cor, cfg_ns, ckpt=ckpt, fail_at=2)
                res = dict(failed=np.array(False))
            except RuntimeError:
                res = dict(failed=np.array(True))
        else:  # resume
            res = _run(P, pkg, cor, cfg_ns, ckpt=ckpt, resume=True)
        np.savez(os.path.join(out_dir, f"{mode}_rank{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


def _spawn(tmp_path, mode):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), mode), nprocs=2, join=True)
    return [dict(np.load(tmp_path / f"{mode}_rank{r}.npz")) for r in range(2)]


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_two_rank_training_extraction_and_accumulation_match_single_rank(gpu, tmp_path):
    from paper_1906_08556_b200 import pipeline as P
    cor, cfg_ns = cases.train_inputs(CASE)
    single = _run(P, gpu, cor, cfg_ns)
    ranks = _spawn(tmp_path, "plain")
    # the replicated M-step gives bit-identical models on both ranks
    for k in ("T", "Sigma", "ivectors", "acc_B", "acc_A", "aux"):
        assert ranks[0][k].tobytes() == ranks[1][k].tobytes(), k
    r = ranks[0]
    assert list(r["ids"]) == list(single["ids"])
    np.testing.assert_allclose(r["aux"], single["aux"], rtol=1e-12)
    for k in ("T", "Sigma", "ubm_means", "ivectors", "acc_B", "acc_N", "acc_A"):
        assert _rel(r[k], single[k]) < 1e-10, (k, _rel(r[k], single[k]))
    # (the all-reduce changes the accumulators' summation order: 1e-16-level differences that the EM
    # iterations amplify, hence the same 1e-10 as the model arrays)
    np.testing.assert_allclose(r["prior"], single["prior"], rtol=1e-10)
    # accumulate_corpus on an initialised group sums the shards once (not world_size times)
    assert int(r["acc_U"]) == int(single["acc_U"]) == len(cor.ids)
    np.testing.assert_allclose(r["acc_aux"], single["acc_aux"], rtol=1e-12)


def test_two_rank_checkpoint_resume_is_bit_exact(gpu, tmp_path):
    plain = _spawn(tmp_path, "plain")
    failed = _spawn(tmp_path, "fail")
    assert all(bool(f["failed"]) for f in failed)
    ck = tmp_path / "ckpt"
    assert (ck / "model_iter_0001.tvm").exists() and not (ck / "model_iter_0002.tvm").exists()
    resumed = _spawn(tmp_path, "resume")
    for r in range(2):
        assert list(resumed[r]["iters"]) == [2, 3]
        for k in ("T", "Sigma", "ivectors", "prior"):
            assert resumed[r][k].tobytes() == plain[r][k].tobytes(), k


def test_bench_torchrun_two_ranks(gpu):
    """bench.py's multi-rank path as the driver launches it (torchrun, one process per rank; gloo here
    so both ranks can share the one GPU): frames sharded with no collective, the EM leg's one
    all-reduce per iteration, max-over-ranks timing, and ONE JSON line from rank 0 whose whole-job
    value counts both ranks' frames."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--frames", "300000", "--em-utts", "512", "--em-steps", "1", "--c5-utts", "256",
           "--extract-utts", "1024", "--exact-frames", "0", "--dense-steps", "0", "--no-cpu", "--no-config1",
           "--dist-backend", "gloo"]
    env = dict(os.environ, OMP_NUM_THREADS="4")
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["config"]["global_frames_per_step"] == 600000
    assert abs(rec["value"] - 600000 / (rec["ms_per_step"] / 1e3)) <= 1e-6 * rec["value"]
    em = rec["em_iteration"]
    assert em["global_utts"] == 512 and em["utts_per_gpu"] == 256 and em["value"] > 0
    assert np.isfinite(em["aux_last"])
    assert rec["config5"]["extraction"]["global_utts"] == 1024
