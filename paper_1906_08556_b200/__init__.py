"""B200-native GPU i-vector hot path (arXiv 1906.08556), drop-in for the reference ``tvkit``
hot-path API: UBM frame posteriors, Baum-Welch statistics, i-vector extractor training and
extraction (augmented and standard formulations).  Arithmetic runs in libtvk.so (sm_100a).
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

__version__ = "0.1.0"
