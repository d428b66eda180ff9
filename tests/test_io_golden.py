"""Container formats against files written by the REFERENCE's own writers (tests/golden/io/,
make_golden.py: make_io): the drop-in reads them and writes them back byte for byte.  Plus the
ALN1 reader's corrupt-header and large-index behaviour.  CPU except the TVM1 model check."""

import os
import struct
import time

import numpy as np
import pytest

from paper_1906_08556_b200 import io_formats as io
from paper_1906_08556_b200.gmm import SparseAlignment

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


def test_reference_aln1_reads_and_rewrites_identically(tmp_path):
    src = os.path.join(GOLD, "ref.aln")
    alis = io.read_alignment(src)
    assert list(alis) == ["spk1-utt1", "spk1-utt2", "spk2-utt1", "spk3-utt7"]
    assert alis["spk1-utt2"].n_frames == 0
    for a in alis.values():
        a.validate(top_k=6)
    out = str(tmp_path / "back.aln")
    io.write_alignment(out, list(alis.items()), top_k=6)
    assert _bytes(out) == _bytes(src)
    with io.AlignmentReader(src) as r:  # random access in reverse order
        assert r.top_k == 6 and r.ids() == list(alis)
        for u in reversed(r.ids()):
            got = r.read(u)
            np.testing.assert_array_equal(got.offsets, alis[u].offsets)
            np.testing.assert_array_equal(got.components, alis[u].components)
            assert got.weights.tobytes() == alis[u].weights.tobytes()
        with pytest.raises(KeyError, match="not in alignment file"):
            r.read("nope")


@pytest.mark.gpu  # load_model validates Sigma with the device Cholesky
@pytest.mark.parametrize("form", ["augmented", "standard"])
def test_reference_tvm1_model_round_trip(gpu, tmp_path, form):
    src = os.path.join(GOLD, f"ref_{form}.tvm")
    m = io.load_model(src)
    assert m.formulation == form and m.T.shape == (16, 5, 3)
    out = str(tmp_path / "m.tvm")
    io.save_model(m, out)
    assert _bytes(out) == _bytes(src)


@pytest.mark.parametrize("name,dtype", [("ref_f64.fmx", "f64"), ("ref_f32.fmx", "f32")])
def test_reference_fmx1_round_trip(tmp_path, name, dtype):
    src = os.path.join(GOLD, name)
    m = io.read_matrix(src)
    out = str(tmp_path / "m.fmx")
    io.write_matrix(m, dtype, out)
    assert _bytes(out) == _bytes(src)


def test_reference_trial_list_round_trip(tmp_path):
    src = os.path.join(GOLD, "ref.trials")
    t = io.read_trials(src)
    assert t.enrol_ids == ["a", "a", "b"] and list(t.is_target) == [True, False, True]
    out = str(tmp_path / "t.trials")
    io.write_trials(out, t)
    assert _bytes(out) == _bytes(src)
    open(out, "a").write("a b maybe\n")
    with pytest.raises(io.FormatError, match="unknown label"):
        io.read_trials(out)


def test_aln1_huge_frame_count_raises_format_error_before_allocating(tmp_path):
    ali = SparseAlignment.from_frames([(np.array([1]), np.array([1.0], np.float32))])
    p = str(tmp_path / "z.aln")
    io.write_alignment(p, {"u": ali}, top_k=1)
    raw = bytearray(_bytes(p))
    raw[24 + 4 + 1:24 + 4 + 1 + 8] = struct.pack("<Q", 1 << 60)
    open(p, "wb").write(bytes(raw))
    with pytest.raises(io.FormatError, match="shorter than declared"):
        io.read_alignment(p)


def test_aln1_index_walk_scales_to_large_corpora(tmp_path):
    """20k utterances: the record bounds come from one sort (the old per-record list.index walk was
    O(U^2), tens of seconds here)."""
    one = SparseAlignment.from_frames([(np.array([0, 2]), np.array([0.5, 0.5], np.float32))] * 3)
    p = str(tmp_path / "big.aln")
    io.write_alignment(p, [(f"u{i:06d}", one) for i in range(20000)], top_k=2)
    t0 = time.perf_counter()
    back = io.read_alignment(p)
    assert len(back) == 20000 and back["u019999"].n_frames == 3
    assert time.perf_counter() - t0 < 20.0
