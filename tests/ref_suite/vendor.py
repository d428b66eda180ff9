"""Packs the reference's own hot-path test files for the drop-in check (build container only).

``pack()`` (called by ``__graft_entry__.build()`` when ``/root/reference`` exists) stores the
reference's ``pkg/tests/test_{gmm,tvm,pipeline}.py`` and the synthetic-corpus generator
``pkg/src/tvkit/synth.py`` (their input generator; outside this package's scope) UNCHANGED in
``tests/ref_suite/_vendor.tgz``.  The archive is git-ignored (reference files never enter the
history) but travels with the working tree to the GPU box, where
``test_reference_suite.py`` unpacks it into a temporary directory and runs the files with
pytest against the ``tvkit`` alias of this package.
"""

from __future__ import annotations

import io
import os
import tarfile

HERE = os.path.dirname(os.path.abspath(__file__))
ARCHIVE = os.path.join(HERE, "_vendor.tgz")
REF = "/root/reference/pkg"
FILES = {
    "test_gmm.py": "tests/test_gmm.py",
    "test_tvm.py": "tests/test_tvm.py",
    "test_pipeline.py": "tests/test_pipeline.py",
    "synth.py": "src/tvkit/synth.py",
}


def pack(ref=REF):
    """Archive the reference files (no-op without the reference tree)."""
    if not all(os.path.exists(os.path.join(ref, p)) for p in FILES.values()):
        return None
    buf = io.BytesIO()
    with tarfile.open(fileobj=buf, mode="w:gz") as tar:
        for name, rel in sorted(FILES.items()):
            data = open(os.path.join(ref, rel), "rb").read()
            info = tarfile.TarInfo(name)
            info.size = len(data)
            info.mtime = 0
            tar.addfile(info, io.BytesIO(data))
    tmp = ARCHIVE + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(buf.getvalue())
    os.replace(tmp, ARCHIVE)
    return ARCHIVE


def unpack(dest):
    with tarfile.open(ARCHIVE, "r:gz") as tar:
        tar.extractall(dest, filter="data")
    return dest


if __name__ == "__main__":
    print(pack())
