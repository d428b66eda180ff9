"""``import tvkit`` alias of the B200 drop-in (``paper_1906_08556_b200``).

Code written against the reference package (``from tvkit.gmm import align_frames``,
``import tvkit.pipeline as pipeline``, ...) runs unchanged on the GPU path: the package root and
its hot-path submodules (gmm, tvm, io_formats, pipeline, _linalg) are the drop-in's own modules,
registered under the reference names.  See INTEGRATION.md.
"""

import sys as _sys

import paper_1906_08556_b200 as _impl
from paper_1906_08556_b200 import _linalg, gmm, io_formats, pipeline, tvm  # noqa: F401
from paper_1906_08556_b200 import *  # noqa: F401,F403
from paper_1906_08556_b200 import __version__  # noqa: F401

for _name in ("_linalg", "gmm", "tvm", "io_formats", "pipeline"):
    _sys.modules[f"{__name__}.{_name}"] = getattr(_impl, _name)


def __getattr__(name):
    return getattr(_impl, name)
