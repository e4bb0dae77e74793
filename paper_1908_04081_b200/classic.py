"""Drop-in `hscg_solve` -- Hestenes-Stiefel CG on the GPU (reference:
/root/reference/pkg/src/sstepcg/classic.py), the
classic-CG baseline s-step CG is measured against.

`hscg_solve(problem, eps_star, max_iters=None)` keeps the reference's
semantics: the true residual b - A x is recomputed every iteration and drives
the stopping decisions; breakdown and NaN are recorded on the trace, never
raised.  Each iteration is three fused row-streaming kernels on the plan's
operator (csrc/hscg.cu), replayed in CUDA graphs of 16 iterations.
`assemble_tridiag` / `hscg_attainable_accuracy` are the module's host helpers.
"""

from __future__ import annotations

import numpy as np

from . import _lib as L
from .kernels import _plan
from .types import CgCoefficients, SolveTrace


def assemble_tridiag(coeffs, i):
    """The Lanczos tridiagonal T_i that the first i CG coefficient pairs define
    (classic.py:12-30): diagonal 1/alpha_l (+ beta_{l-1}/alpha_{l-1} for
    l >= 1), off-diagonal sqrt(beta_{l-1})/alpha_{l-1}; built from whole
    coefficient vectors (the same per-entry operations)."""
    if i < 1:
        raise ValueError("need at least one coefficient pair")
    if i > len(coeffs.alphas):
        raise ValueError(f"only {len(coeffs.alphas)} coefficient pairs stored")
    al = np.asarray(coeffs.alphas[:i], dtype=float)
    be = np.asarray(coeffs.betas[:i - 1], dtype=float)
    diag = 1.0 / al
    diag[1:] += be / al[:-1]
    off = np.sqrt(be) / al[:-1]
    return np.diag(diag) + np.diag(off, 1) + np.diag(off, -1)


def hscg_logs(max_iters):
    """Host log buffers of an HSCG run (one row per iteration)."""
    cap = int(min(max(int(max_iters), 0), 1 << 20)) + 2
    iters = np.full((cap, L.IT_N), np.nan)
    logs = L.SscgLogs()
    logs.cap_iters, logs.cap_outer = cap, 0
    logs.iters = L.dptr(iters)
    return iters, logs


def hscg_trace(iters, logs):
    """SolveTrace / CgCoefficients of an HSCG run: one record and one outer
    mark per iteration (classic.py:93-103)."""
    tr = SolveTrace(trace_level="full")
    co = CgCoefficients()
    n = min(int(logs.total_iters), len(iters))
    for row in iters[:n]:
        co.append(float(row[L.IT_ALPHA]), float(row[L.IT_BETA]))
        tr.mark_outer(1)
        tr.record_iteration(row[L.IT_TRUE], row[L.IT_UPD], row[L.IT_GAP], row[L.IT_XI],
                            row[L.IT_LMIN], row[L.IT_LMAX], row[L.IT_PSI])
    tr.converged = logs.status == L.CONVERGED
    tr.stagnated = logs.status == L.STAGNATED
    tr.diverged = logs.status == L.DIVERGED
    return tr, co


def hscg_solve(problem, eps_star, max_iters=None, *, device=0, mode="reference", info=None):
    """Classic CG on the GPU (classic.py:33-104).  Returns (x, SolveTrace,
    CgCoefficients); one trace record and one outer mark per iteration.

    mode="reference" keeps classic.py's semantics (the true residual every
    iteration drives the verdicts); mode="production" is the CG a user would
    run at scale -- one SpMV per iteration, convergence on the updated residual,
    the true residual formed once for the last trace row (the other rows' true
    residual is NaN)."""
    a = problem.a
    if mode not in L.HSCG_MODES:
        raise ValueError(f"unknown HSCG mode {mode!r}")
    if max_iters is None:
        max_iters = 100 * a.n
    b, x0 = L.f64(problem.b), L.f64(problem.x0)
    if b.shape != (a.n,) or x0.shape != (a.n,):
        raise ValueError("b / x0 do not match the matrix dimension")
    plan = _plan(a, device)
    iters, logs = hscg_logs(max_iters)
    x = L.result_pool.vector(a.n)
    L.check(L.load().sscg_hscg_ex(plan.handle, L.dptr(b), L.dptr(x0), float(eps_star),
                                  int(max_iters), L.HSCG_MODES[mode], L.dptr(x), logs))
    tr, co = hscg_trace(iters, logs)
    if isinstance(info, dict):
        info.update(device_ms=logs.device_ms, status=int(logs.status))
    return x, tr, co


def hscg_attainable_accuracy(problem, max_iters=None, *, device=0):
    """Smallest relative true residual HSCG reaches before stagnating
    (classic.py:107-110)."""
    _, trace, _ = hscg_solve(problem, eps_star=0.0, max_iters=max_iters, device=device)
    return trace.min_true_resid
