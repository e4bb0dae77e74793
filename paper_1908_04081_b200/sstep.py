"""Drop-in `sstep_solve` -- fixed s-step CG on the GPU (reference:
/root/reference/pkg/src/sstepcg/sstep.py:79-174).

Same signature, return types and errors as the reference.  It runs on the same
plan, kernels and CUDA graph as `adaptive_solve` with the C-ABI's fixed solver
(`sscg_config.solver = SSCG_SOLVER_FIXED`): s~ = s every outer loop (no
condition estimates), basis parameters fixed for the whole solve -- the
caller's `params`, or params_for(basis_kind, s, spectral_bounds) built once on
the device -- only the estimated-residual exit inside a block, and no
"stagnated" verdict when max_outer runs out.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np

from . import _lib as L
from .adaptive import LogBuffers, build_trace, clamp_i32
from .kernels import _plan
from .types import DEFAULT_LEJA_GRID, ParameterError


def sstep_solve(problem, s, eps_star, max_outer=None, params=None, basis_kind="monomial",
                spectral_bounds=None, *, trace="full", device=0, info=None):
    """Fixed s-step CG (sstep.py:79-174).  Returns (x, SolveTrace, CgCoefficients).

    trace="full" reproduces the reference's per-inner-iteration true residual
    (sstep.py:146-156); trace="fast" keeps every decision and coefficient and
    takes the residual columns from the Gram quadrature (see SolveTrace)."""
    a, b = problem.a, problem.b
    if s < 1:
        raise ValueError("s must be >= 1")
    if s > L.MAX_SIGMA:
        raise ValueError(f"s={s} exceeds the device limit {L.MAX_SIGMA}")
    if trace not in ("full", "fast"):
        raise ValueError("trace must be 'full' or 'fast'")
    if max_outer is None:
        max_outer = max(1, (100 * a.n) // s)  # sstep.py:95-96
    if params is None and basis_kind not in L.BASIS:
        raise ParameterError(f"unknown basis kind {basis_kind!r}")  # basis.py:175-176
    if params is not None and params.degree_capacity() < s:  # basis.py:235-236
        raise ParameterError(f"params cover degree {params.degree_capacity()}, need {s}")
    c = L.SscgConfig()
    c.sigma, c.s_bar0, c.f = s, s, 0
    c.basis_kind = L.BASIS[params.kind if params is not None and params.kind in L.BASIS
                           else basis_kind]
    c.c_strategy = L.CSTRAT["adaptive"]  # only the trace's xi estimate, as sstep.py:151
    c.variant = 1
    c.max_outer = clamp_i32(max_outer)
    c.leja_grid = DEFAULT_LEJA_GRID
    if spectral_bounds and spectral_bounds[0] is not None and spectral_bounds[1] is not None:
        c.has_bounds = 1
        c.bound_lo, c.bound_hi = float(spectral_bounds[0]), float(spectral_bounds[1])
    c.trace_full = 1 if trace == "full" else 0
    c.n_a = int(a.n_a)
    c.solver = L.SOLVER_FIXED
    c.eps_star = float(eps_star)
    c.norm_a, c.norm_abs_a = float(problem.norm_a), float(problem.norm_abs_a)
    c.kappa_a = float(problem.kappa_a)
    plan = _plan(a, device)
    lib = L.load()
    bv, x0 = L.f64(b), L.f64(problem.x0)
    if bv.shape != (a.n,) or x0.shape != (a.n,):
        raise ValueError("b / x0 do not match the matrix dimension")
    shape = SimpleNamespace(sigma=s, s_bar0=s, max_outer=clamp_i32(max_outer))
    logs = LogBuffers(shape)
    x = L.result_pool.vector(a.n)
    if params is not None:
        th, ga = L.f64(params.thetas), L.f64(params.gammas)
        mu = L.f64(params.mus) if len(params.mus) else np.zeros(1)
        L.check(lib.sscg_set_basis_params(plan.handle, int(len(th)), L.dptr(th), L.dptr(ga),
                                          L.dptr(mu)))
    try:
        L.check(lib.sscg_solve(plan.handle, c, L.dptr(bv), L.dptr(x0), L.dptr(x), logs.s))
    finally:
        if params is not None:
            lib.sscg_set_basis_params(plan.handle, 0, None, None, None)
    tr, co = build_trace(shape, logs, trace, records=False)
    tr.check_consistency()
    if isinstance(info, dict):
        info.update(device_ms=logs.s.device_ms, outer_launched=logs.s.outer_launched,
                    first_gram=logs.first_gram, logs=logs)
    return x, tr, co
