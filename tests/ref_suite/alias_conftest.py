"""conftest for the reference's own test files, run UNCHANGED against the drop-in.

Copied next to the unpacked reference tests by ``test_reference_suite.py``.  It makes ``tvkit``
the drop-in (``import tvkit`` -> paper_1906_08556_b200 with its hot-path submodules), loads the
reference generator ``synth.py`` as ``tvkit.synth`` (its ``from .tvm import TvModel`` etc. then
bind to the drop-in's classes), and deselects the classes that exercise the back-end scoring
outside this package's scope.
"""

import importlib.util
import os
import sys

REPO = os.environ["TVK_REPO"]
sys.path.insert(0, REPO)

import tvkit  # noqa: E402  (the drop-in alias)

_spec = importlib.util.spec_from_file_location("tvkit.synth", os.path.join(os.path.dirname(__file__), "synth.py"))
_synth = importlib.util.module_from_spec(_spec)
sys.modules["tvkit.synth"] = _synth
_spec.loader.exec_module(_synth)
tvkit.synth = _synth

# back-end scoring (PLDA/LDA/EER via ensemble_run / evaluate_model): outside the GPU path
OUT_OF_SCOPE = {"TestEnsemble"}


def pytest_collection_modifyitems(config, items):
    keep, drop = [], []
    for it in items:
        (drop if it.cls is not None and it.cls.__name__ in OUT_OF_SCOPE else keep).append(it)
    if drop:
        config.hook.pytest_deselected(items=drop)
        items[:] = keep
