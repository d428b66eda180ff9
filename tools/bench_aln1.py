"""ALN1 alignment-cache throughput: this package's writer/reader against the
reference's (imported from /root/reference in the build container only), same synthetic corpus.
Checks byte-identical files and identical decoded alignments.  CPU only."""
import os, sys, tempfile, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1906_08556_b200 import io_formats as ours
from paper_1906_08556_b200.gmm import SparseAlignment

REF = "/root/reference/pkg/src"


def corpus(n_utts=400, frames=300, C=2048, K=20, seed=0):
    rng = np.random.default_rng(seed)
    out = {}
    for u in range(n_utts):
        cnt = rng.integers(1, 9, frames)
        off = np.zeros(frames + 1, np.int64)
        np.cumsum(cnt, out=off[1:])
        comps = np.concatenate([np.sort(rng.choice(C, c, replace=False)) for c in cnt]).astype(np.int32)
        w = rng.random(off[-1]).astype(np.float32) + 0.1
        for t in range(frames):
            w[off[t]:off[t + 1]] /= w[off[t]:off[t + 1]].sum()
        out[f"utt{u:05d}"] = (off, comps, w)
    return out


def main():
    raw = corpus()
    T = sum(len(v[0]) - 1 for v in raw.values())
    mine = {k: SparseAlignment(*v) for k, v in raw.items()}
    d = tempfile.mkdtemp()
    p1, p2 = os.path.join(d, "ours.aln"), os.path.join(d, "ref.aln")
    t0 = time.perf_counter(); ours.write_alignment(p1, mine, 20); t1 = time.perf_counter()
    t2 = time.perf_counter(); back = ours.read_alignment(p1); t3 = time.perf_counter()
    print(f"ours: write {T / (t1 - t0) / 1e6:.2f} M frames/s, read {T / (t3 - t2) / 1e6:.2f} M frames/s ({T} frames)")
    if os.path.isdir(REF):
        sys.path.insert(0, REF)
        from tvkit import gmm as rg, io_formats as rio
        theirs = {k: rg.SparseAlignment(*v) for k, v in raw.items()}
        t0 = time.perf_counter(); rio.write_alignment(p2, theirs, 20); t1 = time.perf_counter()
        t2 = time.perf_counter(); rback = rio.read_alignment(p2); t3 = time.perf_counter()
        print(f"reference: write {T / (t1 - t0) / 1e6:.3f} M frames/s, read {T / (t3 - t2) / 1e6:.3f} M frames/s")
        print("byte-identical files:", open(p1, "rb").read() == open(p2, "rb").read())
        same = all(np.array_equal(back[k].offsets, rback[k].offsets) and np.array_equal(back[k].components, rback[k].components)
                   and np.array_equal(back[k].weights, rback[k].weights) for k in raw)
        print("identical decoded alignments:", same)


if __name__ == "__main__":
    main()
