"""Problem setup (reference: /root/reference/pkg/src/sstepcg/matio.py; SURVEY.md
8(f) row 3): Matrix Market ingest, two-sided Jacobi scaling, operator norms,
`load_problem`.

The text parse and CSR assembly run in native code (`sscg_mm_parse`,
csrc/setup.cu), the power iterations for ||A||, || |A| || and lambda_min on
the GPU (`sscg_power_iteration`), so setup at c5 scale is not host-bound;
the O(nnz) diagonal scaling is vectorised numpy with the reference's exact
arithmetic.  Names, signatures, return types and errors follow the
reference."""

from __future__ import annotations

import ctypes as C
import gzip
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .kernels import _plan
from .types import ProblemInstance, SparseMatrix


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input; carries the offending line number (matio.py:14-21)."""

    def __init__(self, message, line_no=None):
        if line_no is not None:
            message = f"{message} (line {line_no})"
        super().__init__(message)
        self.line_no = line_no


class DegenerateMatrixError(ValueError):
    """matio.py:24-25."""


def from_coo(n, rows, cols, vals, is_symmetric=True):
    """Build a SparseMatrix from coordinate data, summing duplicates (matio.py:87-101)."""
    import scipy.sparse as sp
    coo = sp.coo_matrix((vals, (rows, cols)), shape=(n, n))
    csr = coo.tocsr()
    csr.sum_duplicates()
    csr.sort_indices()
    n_a = int(np.diff(csr.indptr).max()) if n else 0
    return SparseMatrix(n=n, row_ptr=csr.indptr.copy(), col_idx=csr.indices.copy(),
                        values=csr.data.copy(), n_a=n_a, is_symmetric=is_symmetric)


def read_matrix_market(path):
    """Read a real square Matrix Market coordinate file into full symmetric CSR
    (matio.py:104-184): symmetric files mirrored, general files must have a
    structurally symmetric pattern, duplicates summed."""
    opener = gzip.open if str(path).endswith(".gz") else open
    with opener(path, "rb") as f:
        text = f.read()
    lib = L.load()
    h, n, nnz, sym = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int32()
    rc = lib.sscg_mm_parse(text, len(text), C.byref(h), C.byref(n), C.byref(nnz), C.byref(sym))
    if rc == L.EFORMAT:
        line = int(lib.sscg_mm_error_line())
        msg = lib.sscg_last_error().decode(errors="replace")
        suffix = f" (line {line})"
        if line and msg.endswith(suffix):
            msg = msg[: -len(suffix)]
        raise MatrixMarketError(msg, line or None)
    L.check(rc)
    try:
        row_ptr = np.empty(n.value + 1, dtype=np.int64)
        col = np.empty(nnz.value, dtype=np.int32)
        val = np.empty(nnz.value)
        L.check(lib.sscg_mm_take(h, row_ptr.ctypes.data_as(C.POINTER(C.c_int64)), L.iptr(col),
                                 L.dptr(val)))
    finally:
        lib.sscg_mm_free(h)
    n_a = int(np.diff(row_ptr).max()) if n.value else 0
    return SparseMatrix(n=int(n.value), row_ptr=row_ptr, col_idx=col, values=val, n_a=n_a,
                        is_symmetric=True)


def jacobi_precondition(a):
    """Two-sided diagonal scaling A_hat = D^{-1/2} A D^{-1/2} (matio.py:187-209):
    D = the largest signed stored entry of each row; each value is divided by
    root[min(i,j)] * root[max(i,j)], so A_hat is bitwise symmetric.
    Returns (A_hat, d^{-1/2})."""
    d = a.row_max()
    if np.any(~np.isfinite(d)) or np.any(d <= 0.0):
        bad = int(np.argmin(d))
        raise DegenerateMatrixError(f"row {bad} has nonpositive maximum {d[bad]!r}")
    root = np.sqrt(d)
    n = a.n
    row_ptr = np.asarray(a.row_ptr)
    cols = np.asarray(a.col_idx)
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    lo = np.minimum(rows, cols)
    hi = np.maximum(rows, cols)
    scaled = np.asarray(a.values) / (root[lo] * root[hi])
    # a canonical CSR (sorted, duplicate-free rows -- what read_matrix_market and
    # from_coo return) is its own from_coo image; anything else goes through it
    keyed = rows.astype(np.int64) * max(n, 1) + cols
    canonical = bool(np.all(np.diff(keyed) > 0)) if len(keyed) > 1 else True
    if canonical:
        out = SparseMatrix(n=n, row_ptr=row_ptr.copy(), col_idx=cols.copy(), values=scaled,
                           n_a=int(np.diff(row_ptr).max()) if n else 0, is_symmetric=True)
    else:
        out = from_coo(n, rows, cols, scaled, is_symmetric=True)
    return out, 1.0 / root


def build_rhs(n):
    """Right-hand side with all entries 1/sqrt(n) (matio.py:212-217)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    return np.full(n, 1.0 / np.sqrt(n))


@dataclass
class NormEstimates:
    norm_a: float
    norm_abs_a: float
    kappa_a: float
    lambda_min: float
    iters_used: int
    converged: bool


def _power_iteration(plan, mode, shift, n, iters, tol, seed=0):
    """matio.py:229-244 on the device: the seeded start vector is drawn and
    normalised here exactly as the reference does, the iteration runs on the GPU."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    v /= np.linalg.norm(v)
    lam, used, conv = C.c_double(), C.c_int32(), C.c_int32()
    L.check(L.load().sscg_power_iteration(plan.handle, int(mode), float(shift), L.dptr(v),
                                          int(iters), float(tol), C.byref(lam), C.byref(used),
                                          C.byref(conv)))
    return float(lam.value), int(used.value), bool(conv.value)


def estimate_operator_norms(a, iters=500, tol=1e-10, *, device=0):
    """||A||_2, || |A| ||_2 and kappa(A) for symmetric A (matio.py:247-276):
    power iteration (on the GPU) for the norms; lambda_min from a dense
    eigensolve for n <= 2000, else power iteration on ||A|| I - A."""
    plan = _plan(a, device)
    norm_a, it1, c1 = _power_iteration(plan, 0, 0.0, a.n, iters, tol)
    norm_abs_a, it2, c2 = _power_iteration(plan, 1, 0.0, a.n, iters, tol)
    if a.n <= 2000:
        w = np.linalg.eigvalsh(a.to_dense())
        lam_min = float(w[0])
        it3, c3 = 0, True
    else:
        shifted, it3, c3 = _power_iteration(plan, 2, norm_a, a.n, iters, tol, seed=1)
        lam_min = norm_a - shifted
    kappa = np.inf if lam_min <= 0 else norm_a / lam_min
    return NormEstimates(norm_a=float(norm_a), norm_abs_a=float(norm_abs_a), kappa_a=float(kappa),
                         lambda_min=lam_min, iters_used=it1 + it2 + it3,
                         converged=c1 and c2 and c3)


def load_problem(path, label=None, norm_iters=500, norm_tol=1e-10, *, device=0):
    """Ingest, precondition and assemble the standard test problem (matio.py:291-307)."""
    raw = read_matrix_market(path)
    a, _ = jacobi_precondition(raw)
    est = estimate_operator_norms(a, iters=norm_iters, tol=norm_tol, device=device)
    b = build_rhs(a.n)
    if label is None:
        label = str(path)
    return ProblemInstance(a=a, b=b, x0=np.zeros(a.n), norm_a=est.norm_a,
                           norm_abs_a=est.norm_abs_a, kappa_a=est.kappa_a, label=label)
