"""B200-native polygrain fit hot path (arXiv 2605.20816, "polynomial diagrams").

Drop-in for the reference package's hot-path API (polygrain/__init__.py:62-86):
``evaluate_objective``, ``objective``, ``gradient``, ``hard_assign``, ``fit``
and the descriptors they take.  All arithmetic of the hot path runs in the
hand-written sm_100a kernels of ``libpgx.so`` (C ABI: ``include/pgx.h``).
"""

from .basis import (
    BASIS_KINDS,
    GAUGE_FREE,
    GAUGE_LAST_ZERO,
    LEGENDRE,
    MONOMIAL,
    ORDERING_CONVENTION,
    DesignBasis,
    DesignMatrix,
    MultiIndexSet,
    ParamMatrix,
    assemble_design_matrix,
    feature_count,
)
from .errors import InputFormatError, NumericalError, ResourceError
from .geometry import TIE_RTOL, GrainMap, PixelGrid, accuracy_and_error, make_grid
from .objective import (
    EvalResult,
    EvalStats,
    Problem,
    SoftAssignment,
    energy_eps,
    energy_zero,
    evaluate_objective,
    gradient,
    hard_assign,
    hessian_block,
    objective,
    soft_assign,
)
from .heuristics import MomentSummary, heuristic_theta, moments
from .optimizer import FitConfig, FitReport, fit, init_zero, line_search
from . import binio  # noqa: E402,F401  (binary sidecars of the grain-map / theta text formats)

__version__ = "0.1.0"

__all__ = [
    "BASIS_KINDS", "GAUGE_FREE", "GAUGE_LAST_ZERO", "LEGENDRE", "MONOMIAL",
    "ORDERING_CONVENTION", "DesignBasis", "DesignMatrix", "MultiIndexSet", "ParamMatrix",
    "assemble_design_matrix", "feature_count", "InputFormatError", "NumericalError",
    "ResourceError", "TIE_RTOL", "GrainMap", "PixelGrid", "accuracy_and_error", "make_grid",
    "EvalResult", "EvalStats", "Problem", "energy_eps", "energy_zero", "evaluate_objective",
    "gradient", "hard_assign", "objective", "soft_assign", "hessian_block", "SoftAssignment", "FitConfig", "FitReport", "fit", "init_zero",
    "line_search", "MomentSummary", "heuristic_theta", "moments",
]
