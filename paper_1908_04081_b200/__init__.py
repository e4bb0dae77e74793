"""B200-native drop-in for the adaptive s-step CG hot path (arXiv 1908.04081).

`adaptive_solve(problem, cfg)` and `sstep_solve(problem, s, eps_star, ...)` have
the reference's signatures and return types (/root/reference/pkg/src/sstepcg/
adaptive.py:111, sstep.py:79); every outer iteration runs
as sm_100a CUDA kernels behind the C-ABI in include/sscg.h.  The CUDA library
is loaded on first use and its absence is an error, never a CPU fallback.
"""

from .types import (  # noqa: F401
    DEFAULT_LEJA_GRID,
    MACHINE_UNIT,
    AdaptiveConfig,
    BasisBreakdownError,
    BasisParams,
    BreakdownSignal,
    CgCoefficients,
    CoordState,
    OuterLoopRecord,
    ParameterError,
    ProblemInstance,
    SolveTrace,
    SparseMatrix,
    SStepBlock,
)
from .adaptive import adaptive_solve, attained_accuracy_report, select_s_tilde  # noqa: F401
from .sstep import sstep_solve  # noqa: F401
from .classic import assemble_tridiag, hscg_attainable_accuracy, hscg_solve  # noqa: F401
from .kernels import (  # noqa: F401
    RitzState,
    assemble_change_of_basis,
    build_block,
    chebyshev_params,
    gram,
    leja_points,
    monomial_params,
    nested_basis_conds,
    newton_params,
    params_for,
    recover_iterates,
    spmv,
)
