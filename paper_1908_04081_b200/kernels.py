"""The reference's hot-path helpers, each backed by one sm_100a kernel family.

Same names, argument meaning and error behaviour as the reference functions
they replace, so the parity tests read like the reference's own tests:

  spmv                  lacore.py:25-34      -> sscg_spmv          (K_mpk row kernel)
  gram                  lacore.py:37-47      -> sscg_gram          (K_gram, DMMA)
  nested_basis_conds    lacore.py:135-148    -> sscg_nested_conds  (K_small Jacobi)
  leja_points           basis.py:91-127      -> sscg_leja_points   (K_small Leja)
  monomial/newton/chebyshev_params, params_for  basis.py:58-177 -> sscg_params_for
  assemble_change_of_basis  basis.py:180-195 (host: a (2s+1)^2 layout helper)
  build_block           basis.py:228-248     -> sscg_build_block   (K_mpk + K_gram)
  recover_iterates      sstep.py:37-44       -> sscg_recover       (K_rec)
  RitzState             ritz.py:108-158      -> sscg_ritz_sequence (K_small Ritz)
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .types import (
    DEFAULT_LEJA_GRID,
    MACHINE_UNIT,
    BasisBreakdownError,
    BasisParams,
    BreakdownSignal,
    ParameterError,
    SStepBlock,
)


def _plan(a, device=0):
    """Device plan cached on the matrix object (like SparseMatrix._csr)."""
    plan = getattr(a, "_sscg_plan", None)
    if plan is None or plan.handle is None or plan.device != device:
        plan = L.Plan(a.n, a.row_ptr, a.col_idx, a.values, device=device)
        try:
            object.__setattr__(a, "_sscg_plan", plan)
        except Exception:
            pass
    return plan


def spmv(a, x, device=0):
    x = np.asarray(x, dtype=float)
    if x.shape != (a.n,):
        raise ValueError(f"dimension mismatch: matrix is {a.n}x{a.n}, vector has shape {x.shape}")
    plan = _plan(a, device)
    xin = L.f64(x)
    y = np.empty(a.n)
    L.check(L.load().sscg_spmv(plan.handle, L.dptr(xin), L.dptr(y)))
    return y


def gram(y, device=0):
    y = np.asarray(y, dtype=float)
    if y.ndim != 2:
        raise ValueError("gram expects a 2-D block")
    n, k = y.shape
    ycm = np.ascontiguousarray(y.T)  # column-major block
    g = np.empty((k, k))
    L.require_device(device)
    L.check(L.load().sscg_gram(device, n, k, L.dptr(ycm), L.dptr(g)))
    return g


def nested_basis_conds(g, s_bar, device=0):
    g = L.f64(g)
    if g.shape != (2 * s_bar + 1, 2 * s_bar + 1):
        raise ValueError("Gram matrix does not match s_bar")
    conds = np.empty(s_bar + 1)
    L.require_device(device)
    L.check(L.load().sscg_nested_conds(device, L.dptr(g), int(s_bar), L.dptr(conds)))
    return conds


def select_s_tilde(g, s_bar, c, eps, eps_star, r_norm, device=0):
    """adaptive.py:89-104."""
    g = L.f64(g)
    conds = np.empty(s_bar + 1)
    st = C.c_int32(0)
    L.require_device(device)
    L.check(L.load().sscg_select_s_tilde(device, L.dptr(g), int(s_bar), float(c), float(eps),
                                         float(eps_star), float(r_norm), C.byref(st),
                                         L.dptr(conds)))
    return int(st.value), conds


def leja_points(lmin, lmax, count, grid_points=DEFAULT_LEJA_GRID, device=0):
    if not (0.0 <= lmin < lmax):
        raise ParameterError(f"need 0 <= lmin < lmax, got ({lmin}, {lmax})")
    if count > L.MAX_SIGMA:
        raise ValueError(f"count={count} exceeds the device limit {L.MAX_SIGMA}")
    if count <= 0:
        return np.array([lmax, lmin])[:max(count, 0)]
    out = np.empty(count)
    L.require_device(device)
    L.check(L.load().sscg_leja_points(device, float(lmin), float(lmax), int(count),
                                      int(grid_points), L.dptr(out)))
    return out


def params_for(kind, s, lmin=None, lmax=None, grid_points=DEFAULT_LEJA_GRID, device=0):
    if kind not in L.BASIS:
        raise ParameterError(f"unknown basis kind {kind!r}")
    if s < 1:
        raise ParameterError("s must be >= 1")
    if s > L.MAX_SIGMA:
        raise ValueError(f"s={s} exceeds the device limit {L.MAX_SIGMA}")
    has = lmin is not None and lmax is not None
    th, ga, mu = np.empty(s), np.empty(s), np.empty(max(1, s - 1))
    ko = C.c_int32(0)
    L.require_device(device)
    L.check(L.load().sscg_params_for(device, L.BASIS[kind], int(s), int(has),
                                     float(lmin) if has else 0.0, float(lmax) if has else 0.0,
                                     int(grid_points), L.dptr(th), L.dptr(ga), L.dptr(mu),
                                     C.byref(ko)))
    name = L.BASIS_NAMES[ko.value]
    gen = (lmin, lmax) if name != "monomial" else None
    return BasisParams(kind=name, thetas=th, gammas=ga, mus=mu[: max(0, s - 1)].copy(),
                       generated_from=gen)


def monomial_params(s):
    if s < 1:
        raise ParameterError("s must be >= 1")
    return params_for("monomial", s)


def newton_params(lmin, lmax, s, grid_points=DEFAULT_LEJA_GRID):
    if s < 1:
        raise ParameterError("s must be >= 1")
    if not (0.0 <= lmin < lmax):
        raise ParameterError(f"need 0 <= lmin < lmax, got ({lmin}, {lmax})")
    th = leja_points(lmin, lmax, s, grid_points)
    return BasisParams(kind="newton", thetas=th, gammas=np.ones(s), mus=np.zeros(max(0, s - 1)),
                       generated_from=(lmin, lmax))


def chebyshev_params(lmin, lmax, s):
    if not (0.0 < lmin < lmax):
        raise ParameterError(f"need 0 < lmin < lmax, got ({lmin}, {lmax})")
    if s < 1:
        raise ParameterError("s must be >= 1")
    return params_for("chebyshev", s, lmin, lmax)


def assemble_change_of_basis(s, params):
    th, ga, mu = params.thetas, params.gammas, params.mus
    b = np.zeros((2 * s + 1, 2 * s + 1))
    for start, size in ((0, s + 1), (s + 1, s)):
        j = np.arange(size - 1)
        b[start + j, start + j] = th[: size - 1]
        b[start + j + 1, start + j] = ga[: size - 1]
        if size > 2:
            b[start + j[1:] - 1, start + j[1:]] = mu[: size - 2]
    return b


def build_block(a, p, r, params, s, device=0):
    if len(params.thetas) < s:
        raise ParameterError(f"params cover degree {len(params.thetas)}, need {s}")
    if s > L.MAX_SIGMA:
        raise ValueError(f"s={s} exceeds the device limit {L.MAX_SIGMA}")
    plan = _plan(a, device)
    k = 2 * s + 1
    ycm = np.empty((k, a.n))
    g = np.empty((k, k))
    th, ga = L.f64(params.thetas), L.f64(params.gammas)
    mu = L.f64(params.mus) if len(params.mus) else np.zeros(1)
    rc = L.load().sscg_build_block(plan.handle, L.dptr(L.f64(p)), L.dptr(L.f64(r)), int(s),
                                   L.dptr(th), L.dptr(ga), L.dptr(mu), L.dptr(ycm), L.dptr(g))
    if rc == L.EBREAKDOWN:
        raise BasisBreakdownError("non-finite basis column")
    L.check(rc)
    return SStepBlock(s=s, y=np.ascontiguousarray(ycm.T), b_mat=assemble_change_of_basis(s, params),
                      g=g, cond_estimates=nested_basis_conds(g, s, device))


def recover_iterates(block, coords, x_base, device=0):
    if len(coords.xp) != 2 * block.s + 1:
        raise ValueError("coordinate length does not match block size")
    y = np.asarray(block.y, dtype=float)
    n, k = y.shape
    ycm = np.ascontiguousarray(y.T)
    x, r, p = np.empty(n), np.empty(n), np.empty(n)
    L.require_device(device)
    L.check(L.load().sscg_recover(device, n, k, L.dptr(ycm), L.dptr(L.f64(coords.xp)),
                                  L.dptr(L.f64(coords.rp)), L.dptr(L.f64(coords.pp)),
                                  L.dptr(L.f64(x_base)), L.dptr(x), L.dptr(r), L.dptr(p)))
    return x, r, p


def ritz_sequence(alphas, betas, device=0):
    """Device RitzState replay: rows (lambda_min, lambda_max, psi, c, xi, count)."""
    a, b = L.f64(alphas), L.f64(betas)
    m = len(a)
    rec = np.empty((m, 6))
    if m:
        L.require_device(device)
        L.check(L.load().sscg_ritz_sequence(device, m, L.dptr(a), L.dptr(b), L.dptr(rec)))
    return rec


class RitzState:
    """ritz.py:108-158 with the estimator arithmetic evaluated by the device code
    K_small runs (replayed over the absorbed (alpha, beta) history)."""

    def __init__(self):
        self._a, self._b = [], []
        self._rec = None

    def absorb_step(self, alpha, beta):
        if not (alpha > 0.0 and beta > 0.0):
            raise BreakdownSignal(f"nonpositive coefficients alpha={alpha!r} beta={beta!r}")
        self._a.append(float(alpha))
        self._b.append(float(beta))
        self._rec = None

    def _last(self):
        if not self._a:
            return None
        if self._rec is None:
            self._rec = ritz_sequence(self._a, self._b)
        return self._rec[-1]

    @property
    def count(self):
        return len(self._a)

    @property
    def lambda_min(self):
        r = self._last()
        return float("nan") if r is None else float(r[0])

    @property
    def lambda_max(self):
        r = self._last()
        return float("nan") if r is None else float(r[1])

    @property
    def psi(self):
        r = self._last()
        return 1.0 if r is None else float(r[2])

    @property
    def c(self):
        r = self._last()
        return MACHINE_UNIT ** -0.5 if r is None else float(r[3])

    def current_c(self):
        return self.c

    def xi_estimate(self):
        r = self._last()
        return 1.0 if r is None else float(r[4])
