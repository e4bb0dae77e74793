"""Boundary data model of the drop-in.

Field-for-field mirrors of the reference types so callers of
`sstepcg.adaptive.adaptive_solve` (adaptive.py:111) keep working unchanged:

  SparseMatrix     matio.py:28-84     (CSR input; `_plan` caches the device copy,
                                       as `_csr` caches the scipy copy, matio.py:47-53)
  ProblemInstance  matio.py:278-288
  AdaptiveConfig   adaptive.py:36-71  (same defaults, same ValueError checks)
  OuterLoopRecord  adaptive.py:74-86
  BasisParams      basis.py:39-55
  SStepBlock       basis.py:198-207
  CoordState       sstep.py:19-34
  SolveTrace       trace.py:25-81
  CgCoefficients   trace.py:10-22

The solver also accepts the reference's own objects (duck typing on the same
field names).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MACHINE_UNIT = 2.0 ** -53  # ritz.py:25
DEFAULT_LEJA_GRID = 10000  # basis.py:24
STAGNATION_WINDOW = 200  # trace.py:85
DIVERGENCE_LIMIT = 1e5  # trace.py:86
C_STRATEGIES = ("adaptive", "unit", "kappa-estimate", "full-bound")  # ritz.py:161
BASIS_KINDS = ("monomial", "newton", "chebyshev")


class ParameterError(ValueError):
    """basis.py:31."""


class BasisBreakdownError(RuntimeError):
    """basis.py:35."""


class BreakdownSignal(ValueError):
    """ritz.py:28."""


@dataclass
class SparseMatrix:
    """matio.py:28-84: symmetric CSR; the device plan is cached on it like the
    reference caches its scipy view (`_csr`)."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    n_a: int
    is_symmetric: bool = True
    _plan: object = field(default=None, repr=False, compare=False)
    _csr: object = field(default=None, repr=False, compare=False)

    @property
    def nnz(self):
        return len(self.values)

    def as_csr(self):
        """scipy CSR view, built once and cached (host helper)."""
        if self._csr is None:
            import scipy.sparse as sp
            self._csr = sp.csr_matrix((self.values, self.col_idx, self.row_ptr),
                                      shape=(self.n, self.n))
        return self._csr

    def row_max(self):
        """Largest stored entry of each row (signed; -inf for an empty row)."""
        out = np.full(self.n, -np.inf)
        lens = np.diff(self.row_ptr)
        nz = lens > 0
        if np.any(nz):
            out[nz] = np.maximum.reduceat(np.asarray(self.values), np.asarray(self.row_ptr)[:-1][nz])
        return out

    def to_dense(self):
        return self.as_csr().toarray()

    def pattern_is_symmetric(self):
        c = self.as_csr()
        return ((c != 0) - (c.T != 0)).nnz == 0

    def validate(self):
        """matio.py:70-84 structural invariants; raises ValueError."""
        if len(self.row_ptr) != self.n + 1:
            raise ValueError("row_ptr length must be n+1")
        if np.any(np.diff(self.row_ptr) < 0):
            raise ValueError("row_ptr must be monotone nondecreasing")
        if len(self.col_idx) and (self.col_idx.min() < 0 or self.col_idx.max() >= self.n):
            raise ValueError("col_idx out of range")
        true_na = int(np.diff(self.row_ptr).max()) if self.n else 0
        if self.n_a != true_na:
            raise ValueError(f"n_a={self.n_a} but true max row population is {true_na}")
        if self.is_symmetric and not self.pattern_is_symmetric():
            raise ValueError("flagged symmetric but stored pattern is not")


@dataclass
class ProblemInstance:
    a: SparseMatrix
    b: np.ndarray
    x0: np.ndarray
    norm_a: float
    norm_abs_a: float
    kappa_a: float
    label: str = ""


@dataclass
class AdaptiveConfig:
    """adaptive.py:36-71 (s_bar0 = f = sigma by default)."""

    sigma: int
    eps_star: float
    s_bar0: int | None = None
    f: int | None = None
    basis_kind: str = "newton"
    c_strategy: str = "adaptive"
    variant: str = "improved"
    max_outer: int = 5000
    leja_grid: int = DEFAULT_LEJA_GRID
    spectral_bounds: tuple | None = None

    def __post_init__(self):
        if self.sigma < 1:
            raise ValueError("sigma must be >= 1")
        if self.s_bar0 is None:
            self.s_bar0 = self.sigma
        if self.f is None:
            self.f = self.sigma
        if not (1 <= self.s_bar0 <= self.sigma):
            raise ValueError("need 1 <= s_bar0 <= sigma")
        if self.f < 0:
            raise ValueError("f must be >= 0")
        if self.eps_star <= 0:
            raise ValueError("eps_star must be positive")
        if self.variant not in ("old", "improved"):
            raise ValueError(f"unknown variant {self.variant!r}")


@dataclass
class BasisParams:
    kind: str
    thetas: np.ndarray
    gammas: np.ndarray
    mus: np.ndarray
    generated_from: tuple | None = None

    def degree_capacity(self):
        return len(self.thetas)


@dataclass
class SStepBlock:
    s: int
    y: np.ndarray
    b_mat: np.ndarray
    g: np.ndarray
    cond_estimates: np.ndarray


@dataclass
class CoordState:
    xp: np.ndarray
    rp: np.ndarray
    pp: np.ndarray
    j: int = 0

    @classmethod
    def initial(cls, s):
        dim = 2 * s + 1
        pp = np.zeros(dim)
        rp = np.zeros(dim)
        pp[0] = 1.0
        rp[s + 1] = 1.0
        return cls(xp=np.zeros(dim), rp=rp, pp=pp)


@dataclass
class OuterLoopRecord:
    k: int
    s_bar: int
    s_tilde: int
    s_actual: int
    phi: float
    cond_used: np.ndarray
    basis_params_used: object
    break_j: int | None = None
    break_lhs: float = float("nan")
    break_rhs: float = float("nan")


@dataclass
class CgCoefficients:
    alphas: list = field(default_factory=list)
    betas: list = field(default_factory=list)

    def append(self, alpha, beta):
        self.alphas.append(float(alpha))
        self.betas.append(float(beta))

    def __len__(self):
        return len(self.alphas)


@dataclass
class SolveTrace:
    """trace.py:25-81.  `trace_level` says where the residual columns came from:

    "full"  reference semantics (adaptive.py:205-215): every inner iteration's
            true residual ||b - A x_j|| / ||b||, updated ||Y r'_j|| / ||b||, gap.
    "fast"  the hot path: upd_resid is the Gram quadrature sqrt(r'^T G r')/||b||
            (what the solver itself steers by), true_resid equals it inside a
            block and is the exact ||b - A x|| / ||b|| on every block-final
            iteration (computed at the next outer boundary anyway), resid_gap
            is |true - upd| there and NaN elsewhere.
    """

    true_resid: list = field(default_factory=list)
    upd_resid: list = field(default_factory=list)
    resid_gap: list = field(default_factory=list)
    outer_marks: list = field(default_factory=list)
    s_schedule: list = field(default_factory=list)
    c_values: list = field(default_factory=list)
    psi: list = field(default_factory=list)
    lambda_min: list = field(default_factory=list)
    lambda_max: list = field(default_factory=list)
    converged: bool = False
    stagnated: bool = False
    diverged: bool = False
    total_iters: int = 0
    total_outer: int = 0
    outer_records: list = field(default_factory=list)
    trace_level: str = "full"
    outer_true_resid: list = field(default_factory=list)
    truncated: bool = False  # device log capacity ran out (the solve itself is complete)

    def record_iteration(self, true_rel, upd_rel, gap, c_val, lmin, lmax, psi=float("nan")):
        self.true_resid.append(float(true_rel))
        self.upd_resid.append(float(upd_rel))
        self.resid_gap.append(float(gap))
        self.c_values.append(float(c_val))
        self.lambda_min.append(float(lmin))
        self.lambda_max.append(float(lmax))
        self.psi.append(float(psi))
        self.total_iters += 1

    def mark_outer(self, s_k):
        self.outer_marks.append(self.total_iters)
        self.s_schedule.append(int(s_k))
        self.total_outer += 1

    @property
    def final_true_resid(self):
        return self.true_resid[-1] if self.true_resid else np.inf

    @property
    def min_true_resid(self):
        return min(self.true_resid) if self.true_resid else np.inf

    def check_consistency(self):
        n = self.total_iters
        assert len(self.true_resid) == n
        assert len(self.upd_resid) == n
        assert len(self.resid_gap) == n
        assert len(self.c_values) == n
        assert all(b > a for a, b in zip(self.outer_marks, self.outer_marks[1:]))
        assert len(self.outer_marks) == self.total_outer == len(self.s_schedule)
