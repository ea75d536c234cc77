"""B200-native sFFT-DT (arXiv 1407.8315): drop-in for the reference
package's recovery entry points, computed by hand-written sm_100a kernels
(libsfdt_b200.so).  See DESIGN.md."""

from .exact import (EstimateResult, ExactBatch, ExactConfig, IterationStats, SolverTrace,
                    estimate_sparsity_and_solve, exact_batch, solve_iterative,
                    solve_iterative_batch, solve_noniterative, solve_noniterative_batch)
from .general import (CollisionEstimate, GeneralBatch, GeneralConfig, GeneralPlan, GeneralTrace,
                      SensingMatrix, draw_shifts, estimate_collisions, prune_columns, sensing_matrix,
                      solve_general, solve_general_batch, subspace_pursuit)
from .graph import SolveGraph, SolvePipeline
from .host import HostBatchResult, solve_host_batch
from .syndrome import (DecodedBin, DecodedBins, DegenerateBranch, IllConditioned, NearSingular,
                       PolyCoefficients, decode_bin, decode_bins, root_to_location, roots_closed_form,
                       solve_coefficients, solve_values)
from .spectral import (AliasedSpectrum, DownsampleView, SparseSpectrum, SyndromeSet, aliased_values,
                       aliased_values_batch, as_signal, downsample, fft, forward_dft_oracle, rms, snr,
                       syndromes_for_bin, synthesize, transform_view)

from ._lib import tuning

BACKEND = "b200"
__version__ = "0.1.0"


def using_compiled() -> bool:
    """The CUDA library is the only backend."""
    return True


__all__ = [
    "DecodedBin", "DegenerateBranch", "IllConditioned", "NearSingular", "PolyCoefficients",
    "decode_bin", "root_to_location", "roots_closed_form", "solve_coefficients", "solve_values",
    "fft", "snr", "synthesize", "AliasedSpectrum", "DownsampleView", "SyndromeSet", "aliased_values",
    "aliased_values_batch", "downsample", "forward_dft_oracle", "rms", "syndromes_for_bin",
    "transform_view", "DecodedBins", "decode_bins", "SensingMatrix", "prune_columns", "sensing_matrix",
    "subspace_pursuit", "tuning",
    "BACKEND", "EstimateResult", "ExactBatch", "ExactConfig", "HostBatchResult",
    "IterationStats", "SolverTrace", "SolveGraph", "SolvePipeline", "solve_host_batch",
    "SparseSpectrum", "as_signal", "estimate_sparsity_and_solve", "exact_batch",
    "solve_iterative", "solve_iterative_batch", "solve_noniterative",
    "solve_noniterative_batch", "using_compiled", "CollisionEstimate", "GeneralBatch",
    "GeneralConfig", "GeneralPlan", "GeneralTrace", "draw_shifts", "estimate_collisions", "solve_general", "solve_general_batch",
]
