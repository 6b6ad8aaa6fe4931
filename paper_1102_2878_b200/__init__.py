"""B200-native (sm_100a) dual-tree fast Gauss transform (arXiv:1102.2878 hot path).

Gaussian kernel sums G(q) = sum_r exp(-|q-r|^2 / 2h^2) with a per-query relative
error bound eps, and the likelihood / least-squares cross-validation sweeps they
drive.  The compute path is libdfgtb.so (hand-written CUDA for sm_100a) behind the
C ABI in include/dfgtb.h; this package is the thin host mirror of the reference's
interface.  Importing it loads the CUDA library and fails loudly if it is missing.
"""
from .engine import (  # noqa: F401
    Algorithm, CostModel, CvOptions, CvRow, CvScore, DualTreeEngine, EngineConfig, Mode,
    RelativeErrorReport, ScoreResult, TraversalStats, bandwidth_sweep, compute_sums,
    convolution_bandwidth, dfd_kde, dfgt_kde, gaussian_normalizer, lkcv_from_sums, lkcv_score,
    lscv_from_sums, lscv_score, naive_kde, pilot_bandwidth, verify_relative_error)

__all__ = [
    "Algorithm", "CostModel", "CvOptions", "CvRow", "CvScore", "DualTreeEngine", "EngineConfig",
    "Mode", "RelativeErrorReport", "ScoreResult", "TraversalStats", "bandwidth_sweep",
    "compute_sums", "convolution_bandwidth", "dfd_kde", "dfgt_kde", "gaussian_normalizer",
    "lkcv_from_sums", "lkcv_score", "lscv_from_sums", "lscv_score", "naive_kde",
    "pilot_bandwidth", "verify_relative_error",
]
