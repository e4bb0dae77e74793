"""Drop-in `adaptive_solve` (reference: /root/reference/pkg/src/sstepcg/adaptive.py:111).

Same signature, same return types, same validation errors.  The whole solve
runs on the GPU through `sscg_solve` (include/sscg.h): per outer loop the
matrix-powers levels, the Gram matrix, the O(s^2) control kernel and the fused
recovery are replayed as one CUDA graph with no host round trip; this module
only marshals the inputs and rebuilds `SolveTrace` / `CgCoefficients` /
`OuterLoopRecord` from the device logs.

trace="full" (default) reproduces the reference's per-inner-iteration
diagnostics (adaptive.py:205-215: one extra SpMV + recovery per inner
iteration).  trace="fast" is the hot path the benchmark times: every decision,
alpha/beta, Ritz value, c, x and count is the same; only the residual
columns differ as documented on `SolveTrace`.
"""

from __future__ import annotations

import math
import warnings

import numpy as np

from . import _lib as L
from .kernels import _plan
from .kernels import select_s_tilde  # noqa: F401  (re-exported like the reference)
from .types import (
    AdaptiveConfig,
    BasisParams,
    CgCoefficients,
    OuterLoopRecord,
    ParameterError,
    SolveTrace,
)


def _validate(cfg):
    """AdaptiveConfig.__post_init__ (adaptive.py:57-71) for duck-typed configs."""
    if isinstance(cfg, AdaptiveConfig):
        return cfg
    return AdaptiveConfig(
        sigma=cfg.sigma, eps_star=cfg.eps_star, s_bar0=cfg.s_bar0, f=cfg.f,
        basis_kind=cfg.basis_kind, c_strategy=cfg.c_strategy, variant=cfg.variant,
        max_outer=cfg.max_outer, leja_grid=cfg.leja_grid, spectral_bounds=cfg.spectral_bounds)


def make_config(cfg, problem, trace="full"):
    cfg = _validate(cfg)
    if cfg.basis_kind not in L.BASIS:
        raise ParameterError(f"unknown basis kind {cfg.basis_kind!r}")
    if cfg.c_strategy not in L.CSTRAT:
        raise ValueError(f"unknown c strategy {cfg.c_strategy!r}")
    if cfg.sigma > L.MAX_SIGMA:
        raise ValueError(f"sigma={cfg.sigma} exceeds the device limit {L.MAX_SIGMA}")
    if trace not in ("full", "fast"):
        raise ValueError("trace must be 'full' or 'fast'")
    c = L.SscgConfig()
    c.sigma, c.s_bar0, c.f = cfg.sigma, cfg.s_bar0, cfg.f
    c.basis_kind = L.BASIS[cfg.basis_kind]
    c.c_strategy = L.CSTRAT[cfg.c_strategy]
    c.variant = 1 if cfg.variant == "improved" else 0
    c.max_outer = clamp_i32(cfg.max_outer)
    c.leja_grid = int(cfg.leja_grid)
    if cfg.spectral_bounds:
        c.has_bounds = 1
        lo, hi = cfg.spectral_bounds
        c.has_bounds = 0 if (lo is None or hi is None) else 1
        c.bound_lo = float(lo) if lo is not None else 0.0
        c.bound_hi = float(hi) if hi is not None else 0.0
    c.trace_full = 1 if trace == "full" else 0
    c.n_a = int(problem.a.n_a)
    c.eps_star = float(cfg.eps_star)
    c.norm_a = float(problem.norm_a)
    c.norm_abs_a = float(problem.norm_abs_a)
    c.kappa_a = float(problem.kappa_a)
    return cfg, c


INT32_LOOP_MAX = 2**31 - 2


def clamp_i32(v):
    """A loop bound for the ABI's int32 fields: the reference's defaults (e.g.
    sstep's 100 n / s) can exceed int32 on huge operators; the solve ends on
    its verdict long before such a bound, so clamping changes nothing."""
    return int(min(max(int(v), 0), INT32_LOOP_MAX))


class LogBuffers:
    """Host arrays the device logs are copied into (caller-owned per the ABI)."""

    def __init__(self, cfg):
        sig = cfg.sigma
        mo = clamp_i32(cfg.max_outer)
        co = min(mo + 2, L.LOG_CAP_OUTER)
        ci = min((mo + 1) * sig + 1, L.LOG_CAP_ITERS)
        self.iters = np.full((ci, L.IT_N), np.nan)
        self.rec_i = np.zeros((co, L.REC_NI), dtype=np.int32)
        self.rec_d = np.full((co, L.RECD_ND), np.nan)
        self.conds = np.full((co, L.MAX_SIGMA + 1), np.nan)
        self.thetas = np.full((co, L.MAX_SIGMA), np.nan)
        self.gammas = np.full((co, L.MAX_SIGMA), np.nan)
        self.mus = np.full((co, L.MAX_SIGMA), np.nan)
        self.outer_true = np.full(co + 1, np.nan)
        d = 2 * cfg.s_bar0 + 1
        self.first_gram = np.full((d, d), np.nan)
        s = L.SscgLogs()
        s.cap_iters, s.cap_outer = ci, co
        s.iters, s.rec_i, s.rec_d = L.dptr(self.iters), L.iptr(self.rec_i), L.dptr(self.rec_d)
        s.conds, s.thetas = L.dptr(self.conds), L.dptr(self.thetas)
        s.gammas, s.mus = L.dptr(self.gammas), L.dptr(self.mus)
        s.outer_true, s.first_gram = L.dptr(self.outer_true), L.dptr(self.first_gram)
        self.s = s


def build_trace(cfg, logs, trace_level, records=True):
    """SolveTrace / CgCoefficients from the device logs (trace.py:25-81).
    records=False: no OuterLoopRecords (the fixed s-step solver keeps none)."""
    s = logs.s
    tr = SolveTrace(trace_level=trace_level)
    co = CgCoefficients()
    # runs longer than the log capacity keep their first rows (trace truncated)
    nrec = min(int(s.n_records), len(logs.rec_i))
    nit = min(int(s.total_iters), len(logs.iters))
    it = logs.iters[:nit]
    sig = cfg.sigma
    for r in range(nrec):
        ri, rd = logs.rec_i[r], logs.rec_d[r]
        tr.outer_marks.append(int(ri[L.REC_MARK]))
        tr.s_schedule.append(int(ri[L.REC_SACTUAL]))
        tr.total_outer += 1
        if not records:
            continue
        kind = L.BASIS_NAMES[int(ri[L.REC_PKIND])]
        gen = None
        if not math.isnan(rd[L.RECD_GEN_LO]):
            gen = (float(rd[L.RECD_GEN_LO]), float(rd[L.RECD_GEN_HI]))
        bp = BasisParams(kind=kind, thetas=logs.thetas[r, :sig].copy(),
                         gammas=logs.gammas[r, :sig].copy(),
                         mus=logs.mus[r, : max(0, sig - 1)].copy(), generated_from=gen)
        s_bar = int(ri[L.REC_SBAR])
        bj = int(ri[L.REC_BREAKJ])
        tr.outer_records.append(OuterLoopRecord(
            k=int(ri[L.REC_K]), s_bar=s_bar, s_tilde=int(ri[L.REC_STILDE]),
            s_actual=int(ri[L.REC_SACTUAL]), phi=float(rd[L.RECD_PHI]),
            cond_used=logs.conds[r, : s_bar + 1].copy(), basis_params_used=bp,
            break_j=None if bj < 0 else bj, break_lhs=float(rd[L.RECD_BLHS]),
            break_rhs=float(rd[L.RECD_BRHS])))
    for i in range(nit):
        row = it[i]
        tr.record_iteration(row[L.IT_TRUE], row[L.IT_UPD], row[L.IT_GAP], row[L.IT_XI],
                            row[L.IT_LMIN], row[L.IT_LMAX], row[L.IT_PSI])
        co.append(row[L.IT_ALPHA], row[L.IT_BETA])
    tr.converged = s.status == L.CONVERGED
    tr.stagnated = s.status == L.STAGNATED
    tr.diverged = s.status == L.DIVERGED
    nt = min(len(logs.outer_true), nrec + 1)
    tr.outer_true_resid = [float(v) for v in logs.outer_true[:nt] if not math.isnan(v)]
    # the device logs keep at most SSCG_LOG_CAP_ITERS iterations and
    # SSCG_LOG_CAP_OUTER outer loops; a longer solve is complete but its trace
    # holds only the first rows -- say so instead of returning it silently
    tr.truncated = nit < int(s.total_iters) or nrec < int(s.n_records)
    if tr.truncated:
        warnings.warn(f"trace truncated: {nit} of {int(s.total_iters)} iterations and {nrec} of "
                      f"{int(s.n_records)} outer loops logged (device log capacity)",
                      RuntimeWarning, stacklevel=3)
    return tr, co


def _group(a, devices, depth):
    """Multi-GPU plans cached on the matrix object (like the single plan)."""
    from .dist import DeviceGroup
    from .partition import CsrRows
    key = (tuple(int(d) for d in devices), int(depth))
    cache = getattr(a, "_sscg_groups", None)
    if cache is None:
        cache = {}
        try:
            object.__setattr__(a, "_sscg_groups", cache)
        except Exception:
            pass
    grp = cache.get(key)
    if grp is None:
        grp = cache[key] = DeviceGroup(CsrRows.of(a), list(devices), depth)
    return grp


def adaptive_solve(problem, cfg, *, trace=None, device=0, devices=None, info=None):
    """Run improved / old adaptive s-step CG on the GPU (adaptive.py:111-268).

    Returns (x, SolveTrace, CgCoefficients) like the reference.  `info`, if a
    dict, receives device_ms / outer_launched / first_gram / device logs.
    `devices=[d0, d1, ...]` (two or more GPUs) row-partitions the operator over
    them from this one process (one halo exchange and one
    NCCL allreduce per outer loop); trace defaults to "full" on one GPU
    (reference semantics) and must be "fast" on several.
    """
    if devices is not None and len(devices) > 1:
        trace = "fast" if trace is None else trace
        if trace != "fast":
            raise ValueError("a multi-GPU solve records trace='fast' (per-iteration true "
                             "residuals are a single-GPU diagnostic)")
        cfg, ccfg = make_config(cfg, problem, trace)
        a = problem.a
        if np.asarray(problem.b).shape != (a.n,) or np.asarray(problem.x0).shape != (a.n,):
            raise ValueError("b / x0 do not match the matrix dimension")
        grp = _group(a, devices, cfg.sigma)
        x, tr, co = grp.solve(problem, cfg, info=info)
        tr.check_consistency()
        return x, tr, co
    if devices is not None and len(devices) == 1:
        device = int(devices[0])
    trace = "full" if trace is None else trace
    cfg, ccfg = make_config(cfg, problem, trace)
    a = problem.a
    plan = _plan(a, device)
    b = L.f64(problem.b)
    x0 = L.f64(problem.x0)
    if b.shape != (a.n,) or x0.shape != (a.n,):
        raise ValueError("b / x0 do not match the matrix dimension")
    logs = LogBuffers(cfg)
    x = L.result_pool.vector(a.n)  # page-locked for large n: one DMA brings x back
    L.check(L.load().sscg_solve(plan.handle, ccfg, L.dptr(b), L.dptr(x0), L.dptr(x), logs.s))
    tr, co = build_trace(cfg, logs, trace)
    tr.check_consistency()
    if isinstance(info, dict):
        info.update(device_ms=logs.s.device_ms, outer_launched=logs.s.outer_launched,
                    first_gram=logs.first_gram, logs=logs)
    return x, tr, co


class AccuracyReport:
    def __init__(self, outcome, cell, total_outer=0, total_iters=0, attained=float("nan")):
        self.outcome, self.cell = outcome, cell
        self.total_outer, self.total_iters, self.attained = total_outer, total_iters, attained


def attained_accuracy_report(trace):
    """adaptive.py:282-305 (host-side formatting of a finished trace)."""
    if trace.converged:
        return AccuracyReport("converged", f"{trace.total_outer} ({trace.total_iters})",
                              trace.total_outer, trace.total_iters, trace.final_true_resid)
    if trace.diverged:
        return AccuracyReport("diverged", "–", attained=trace.min_true_resid)
    attained = trace.min_true_resid
    return AccuracyReport("stagnated", f"– [{attained:.1e}]", attained=attained)
