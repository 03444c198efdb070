"""B200-native pseudo-hermitian ChASE (arXiv 2601.10557) — drop-in for the
reference package ``bsesolve``'s solve path.

Host control logic in Python; every numerical step in the sm_100a CUDA
library ``libbse200.so`` behind the C ABI of ``include/bse200.h``.
"""

__version__ = "0.1.0"

from .errors import (
    BseSolveError,
    HermitianRqError,
    IndefiniteError,
    LanczosBreakdownError,
    NumericalError,
    RankDeficiencyError,
    ValidationError,
)
from .hamiltonian import (
    BseHamiltonian,
    Definiteness,
    apply_h,
    apply_h_via_adjoint,
    apply_j,
    apply_k,
    apply_s,
    is_definite,
    materialize,
    materialize_sh,
    validate_pseudo_hermitian,
)
from .metrics import PhaseLedger
from .lanczos import SpectralBounds, estimate_bounds, update_cutoff
from .chebyshev import FilterConfig, chebyshev_filter, scalar_filter_value
from .ortho import SearchSpace, cholqr_with_fallback, fix_column_phases, s_orthonormalize
from .rayleigh_ritz import (
    ReducedProblem,
    RitzSet,
    build_backup_rq,
    build_hermitian_rq,
    lock_converged,
    residuals,
)
from .solver import (
    CompletedSpectrum,
    SolveResult,
    SolverConfig,
    TraceRecord,
    complete_spectrum,
    mirror_largest,
    set_mixed_precision,
    solve,
)
from .generate import GeneratorSpec, generate
from ._lib import filter_algorithm, filter_precision, set_filter_algorithm, set_filter_precision
from . import fileio

__all__ = [n for n in dir() if not n.startswith("_")]
