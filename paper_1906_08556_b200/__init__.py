"""B200-native GPU i-vector hot path (arXiv 1906.08556), drop-in for the reference ``tvkit``
hot-path API: UBM frame posteriors, Baum-Welch statistics, i-vector extractor training and
extraction (augmented and standard formulations).  Arithmetic runs in libtvk.so (sm_100a).

The names below are the reference package root's (``tvkit/__init__.py:3-75``) for the modules
on the hot path (gmm, tvm, io_formats, pipeline).  The verification back-end (``backend``),
the synthetic-corpus generator (``synth``) and the back-end drivers of ``pipeline`` are outside
this package's scope: their names resolve to placeholders that raise when used.
"""

from ._linalg import NumericError
from .gmm import (
    BaumWelchStats,
    GmmDiag,
    GmmFull,
    SparseAlignment,
    accumulate_bw_stats,
    align_frames,
    select_top_k,
    train_gmm_diag,
    train_gmm_full,
)
from .tvm import (
    AUGMENTED,
    STANDARD,
    EmAccumulators,
    LatentPosterior,
    MinDivTransforms,
    PosteriorWorkspace,
    TvModel,
    apply_min_div,
    aux_objective,
    compute_min_div,
    em_accumulate,
    extract_ivector,
    householder_to_e1,
    init_model,
    latent_posterior,
    model_covariance,
    update_mean_standard,
    update_sigma,
    update_T,
    update_ubm_means_augmented,
)
from .io_formats import (
    FormatError,
    TrialList,
    load_model,
    read_alignment,
    read_matrix,
    read_trials,
    save_model,
    write_alignment,
    write_matrix,
    write_trials,
)
from .pipeline import (
    DirectoryFeatureStore,
    InMemoryFeatureStore,
    PipelineError,
    RunMetrics,
    TrainConfig,
    align_corpus,
    accumulate_corpus,
    extract_corpus,
    train_extractor,
)

__version__ = "0.1.0"

# reference root names outside the GPU path (backend.py, synth.py, pipeline.py:660-757)
_OUT_OF_SCOPE = (
    "GaussianizerChain", "LdaModel", "PldaModel", "compute_eer", "det_points", "fit_chain", "fit_lda",
    "fit_plda", "length_normalize", "score_cosine", "score_plda", "score_plda_trials",
    "EvalProtocol", "ensemble_run", "evaluate_model",
    "SynthCorpus", "SynthSpec", "make_trials", "sample_corpus", "subspace_angles",
)


def __getattr__(name):
    if name in _OUT_OF_SCOPE:
        from .pipeline import _OutOfScope
        return _OutOfScope(name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
