"""B200-native sFFT-DT (arXiv 1407.8315): drop-in for the reference
package's recovery entry points, computed by hand-written sm_100a kernels
(libsfdt_b200.so).  See DESIGN.md."""

from .exact import (EstimateResult, ExactBatch, ExactConfig, IterationStats, SolverTrace,
                    estimate_sparsity_and_solve, exact_batch, solve_iterative,
                    solve_iterative_batch, solve_noniterative, solve_noniterative_batch)
from .general import (CollisionEstimate, GeneralBatch, GeneralConfig, GeneralPlan, GeneralTrace,
                      draw_shifts, estimate_collisions,
                      solve_general, solve_general_batch)
from .graph import SolveGraph, SolvePipeline
from .host import HostBatchResult, solve_host_batch
from .syndrome import (DecodedBin, DegenerateBranch, IllConditioned, NearSingular,
                       PolyCoefficients, decode_bin, root_to_location, roots_closed_form,
                       solve_coefficients, solve_values)
from .spectral import SparseSpectrum, as_signal, fft, snr, synthesize

BACKEND = "b200"
__version__ = "0.1.0"


def using_compiled() -> bool:
    """The CUDA library is the only backend."""
    return True


__all__ = [
    "DecodedBin", "DegenerateBranch", "IllConditioned", "NearSingular", "PolyCoefficients",
    "decode_bin", "root_to_location", "roots_closed_form", "solve_coefficients", "solve_values",
    "fft", "snr", "synthesize",
    "BACKEND", "EstimateResult", "ExactBatch", "ExactConfig", "HostBatchResult",
    "IterationStats", "SolverTrace", "SolveGraph", "SolvePipeline", "solve_host_batch",
    "SparseSpectrum", "as_signal", "estimate_sparsity_and_solve", "exact_batch",
    "solve_iterative", "solve_iterative_batch", "solve_noniterative",
    "solve_noniterative_batch", "using_compiled", "CollisionEstimate", "GeneralBatch",
    "GeneralConfig", "GeneralPlan", "GeneralTrace", "draw_shifts", "estimate_collisions", "solve_general", "solve_general_batch",
]
