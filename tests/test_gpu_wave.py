"""GPU tier: the wavefront matrix-powers kernel (mpk.cu k_mpk_wave).

Opt-in (SSCG_WAVE=1).  The wavefront schedule only changes WHEN each (level, row tile) is computed,
never the arithmetic of a row, so a solve through it must be bit-identical to
the one-launch-per-level path (SSCG_WAVE=0) -- basis, Gram, every alpha and
the iterate.  Forced schedules stress the dependency waits: one level per pass,
two levels per pass, all levels in one pass, and a single CTA per SM (deep
waits on items other CTAs hold)."""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import cfg_of, golden
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems
from paper_1908_04081_b200.kernels import _plan
from paper_1908_04081_b200.types import ProblemInstance, SparseMatrix

pytestmark = pytest.mark.gpu

ENV_KEYS = ("SSCG_WAVE", "SSCG_WAVE_NL", "SSCG_WAVE_CTAS", "SSCG_WAVE_L2_MB", "SSCG_WAVE_SLACK",
            "SSCG_PATTERN", "SSCG_STAGE_MIN_CTAS")


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in ENV_KEYS}
    try:
        for k in ENV_KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _random_spd(n, seed):
    m = sp.random(n, n, density=6.0 / n, random_state=seed, format="csr")
    m = (m + m.T + sp.identity(n) * 14.0).tocsr()
    m.sort_indices()
    a = SparseMatrix(n=n, row_ptr=m.indptr.astype(np.int64), col_idx=m.indices.astype(np.int32),
                     values=m.data.copy(), n_a=7)
    rng = np.random.default_rng(seed)
    norm = float(np.linalg.norm(m.toarray(), 2))
    ev = np.linalg.eigvalsh(m.toarray())
    return ProblemInstance(a=a, b=rng.standard_normal(n), x0=np.zeros(n), norm_a=norm,
                           norm_abs_a=float(np.linalg.norm(abs(m).toarray(), 2)),
                           kappa_a=float(ev[-1] / ev[0]), label=f"rand{n}")


CASES = [
    ("c1", lambda: problems.make_problem("c1"), dict(sigma=8, eps_star=1e-10, basis_kind="newton")),
    ("c3", lambda: problems.make_problem("c3", scale=24),
     dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev")),
    ("c5", lambda: problems.make_problem("c5", scale=28),
     dict(sigma=12, eps_star=1e-10, basis_kind="newton")),
    ("rand", lambda: _random_spd(1500, 5), dict(sigma=6, eps_star=1e-9, basis_kind="monomial")),
]
# the wavefront streams staged CSR tiles: force staging even where the direct
# kernels would be chosen (long rows, few CTAs per SM)
ON = {"SSCG_WAVE": "1", "SSCG_PATTERN": "0", "SSCG_STAGE_MIN_CTAS": "1"}
SCHEDULES = [
    dict(ON),                                         # the L2-budgeted schedule
    dict(ON, SSCG_WAVE_NL="1"),                       # one level per pass
    dict(ON, SSCG_WAVE_NL="2"),
    dict(ON, SSCG_WAVE_NL="16"),                      # every level in one pass
    dict(ON, SSCG_WAVE_CTAS="1", SSCG_WAVE_NL="16"),  # few CTAs: long dependency waits
]


@pytest.mark.parametrize("name,make,kw", CASES, ids=[c[0] for c in CASES])
def test_wavefront_bit_identical_to_level_launches(gpu_ready, name, make, kw):
    cfg = AdaptiveConfig(**kw)
    ref = _with_env({}, lambda: adaptive_solve(make(), cfg, trace="fast"))
    assert ref[1].converged
    for env in SCHEDULES:
        def run():
            prob = make()
            sched = _plan(prob.a).mpk_schedule(cfg.sigma)
            return sched, adaptive_solve(prob, cfg, trace="fast")
        sched, (x, tr, co) = _with_env(env, run)
        assert sched["wavefront"], (name, env, sched)
        np.testing.assert_array_equal(co.alphas, ref[2].alphas, err_msg=f"{name} {env} {sched}")
        np.testing.assert_array_equal(x, ref[0], err_msg=f"{name} {env} {sched}")
        assert tr.total_outer == ref[1].total_outer


def test_wavefront_full_trace_matches_golden_counts(gpu_ready):
    """Full diagnostics (per-iteration true residual) through the wavefront path."""
    ref = golden("solve_c1")
    prob = problems.make_problem("c1")
    def run():
        return _plan(prob.a).mpk_schedule(cfg_of(ref)["sigma"]), \
            adaptive_solve(prob, AdaptiveConfig(**cfg_of(ref)))
    sched, (x, tr, co) = _with_env(ON, run)
    assert sched["wavefront"]
    recs = ref["rec_int"]
    got = [(r.s_tilde, r.s_actual) for r in tr.outer_records[:5]]
    assert got == [tuple(v) for v in recs[:5, 2:4]]
    assert tr.converged


def test_schedule_shape(gpu_ready):
    """Pass planning: levels add up to sigma, every lag exceeds the dependency
    reach (the deadlock-freedom condition), forced one-level passes."""
    mk = lambda: _plan(problems.make_problem("c5", scale=64).a).mpk_schedule(12)
    s = _with_env(ON, mk)
    assert s["wavefront"] and sum(nl for nl, _ in s["passes"]) == 12
    assert s["reach_tiles"] == 16  # 64 x 64 plane = 4096 rows = 16 tiles of 256
    assert all(d > s["reach_tiles"] for _, d in s["passes"])
    assert len(_with_env(dict(ON, SSCG_WAVE_NL="1"), mk)["passes"]) == 12
    assert not _with_env({}, mk)["wavefront"]  # opt-in
