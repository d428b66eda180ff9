"""The reference's own hot-path tests (pkg/tests/test_gmm.py, test_tvm.py, test_pipeline.py), run
unchanged against the drop-in through the ``tvkit`` alias.

Each file runs in a child pytest (fresh ``sys.modules``: the alias and the reference generator
are registered there, not in this session).  The files come from ``tests/ref_suite/_vendor.tgz``,
packed by ``__graft_entry__.build()`` in the build container (see ``vendor.py``); every test in
them is on the GPU path, so the whole check is ``gpu``-marked.
"""

import os
import re
import shutil
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
import vendor  # noqa: E402

# passed counts of these files in the reference run (pkg/test_output.txt), minus its 4 TestEnsemble tests
EXPECTED_MIN_PASSED = {"test_gmm.py": 30, "test_tvm.py": 46, "test_pipeline.py": 30}


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(EXPECTED_MIN_PASSED))
def test_reference_file_passes_unchanged(gpu, tmp_path, name):
    if not os.path.exists(vendor.ARCHIVE):
        pytest.fail("tests/ref_suite/_vendor.tgz missing: run __graft_entry__.build() in the build container")
    vendor.unpack(str(tmp_path))
    shutil.copy(os.path.join(HERE, "alias_conftest.py"), tmp_path / "conftest.py")
    env = dict(os.environ, TVK_REPO=REPO, PYTHONDONTWRITEBYTECODE="1")
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir",
                           str(tmp_path), str(tmp_path / name)], cwd=str(tmp_path), env=env,
                          capture_output=True, text=True, timeout=1800)
    out = proc.stdout + proc.stderr
    print(out[-3000:])
    assert proc.returncode == 0, out[-6000:]
    passed = int(re.search(r"(\d+) passed", out).group(1))
    assert passed >= EXPECTED_MIN_PASSED[name], out[-2000:]
