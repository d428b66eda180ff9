"""Build tools/libtvk_diag.so: libtvk with the -DTVK_SELECT_DIAG diagnostics (TVK_SELECT_DEBUG modes,
TVK_SEL_PIPE, TVK_SELECT=tc_noexact).  Tools load it with use_diag() before the first libtvk call; the
product library never contains these hooks."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_08556_b200 import build as B, _lib

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtvk_diag.so")


def build_diag():
    objdir = os.path.join(B.HERE, "build_diag")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for s in B.SOURCES:
        src = os.path.join(B.CSRC, s)
        o = os.path.join(objdir, s + ".o")
        objs.append(o)
        procs.append(subprocess.Popen([B.nvcc(), *B.ARCH, *B.FLAGS, "-DTVK_SELECT_DIAG", "-c", src, "-o", o]))
    if any(p.wait() for p in procs):
        raise RuntimeError("nvcc failed")
    subprocess.check_call([B.nvcc(), *B.ARCH, "-shared", "-o", OUT, *objs, "-lcudart"])
    return OUT


def use_diag():
    if not os.path.exists(OUT):
        build_diag()
    _lib.LIB_PATH = OUT


if __name__ == "__main__":
    print(build_diag())
