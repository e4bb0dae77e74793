"""GPU tier for fixed s-step CG (`sstep_solve`, sstep.py:79-174; SURVEY.md
8(f) row 1) against golden runs of the reference's own sstep_solve
(oracle/make_golden.py gen_sstep; the oracle restatement reproduces them bit
for bit, tests/test_oracle_golden.py).

North-star tolerances as for adaptive_solve: first Gram 1e-12 (entrywise,
relative to sqrt(G_ii G_jj)), the block schedule and alpha/beta to 1e-8
through the first 5 outer loops, counts within 2% and the final true residual
below eps* when the reference converged; verdict flags identical.  Where the
reference's own runs with a different Gram summation order move
(tests/golden/noise_sstep_*.npz: ill-conditioned monomial s = 10, the
stagnating spd50 case) alpha is held to 1e-8 only up to that noise horizon and
the counts to the envelope of the perturbed runs widened by max(2%, their own
relative spread)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden
from test_oracle_golden import SSTEP_CASES, sstep_kwargs, sstep_problem
from paper_1908_04081_b200 import BasisParams, ParameterError, problems, sstep_solve
from oracle import sscg_oracle as O

pytestmark = pytest.mark.gpu


def _device_kwargs(ref):
    kw = sstep_kwargs(ref)
    if "params" in kw:  # oracle Params -> BasisParams (the public type)
        p = kw["params"]
        kw["params"] = BasisParams(kind="chebyshev", thetas=np.asarray(p.thetas),
                                   gammas=np.asarray(p.gammas), mus=np.asarray(p.mus))
    return kw


def _true_rel(prob, x):
    a = prob.a
    m = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n))
    return np.linalg.norm(prob.b - m @ x) / np.linalg.norm(prob.b)


@pytest.mark.parametrize("name", SSTEP_CASES)
def test_fixed_sstep_parity(gpu_ready, name):
    ref = golden(name)
    prob = sstep_problem(name, ref)
    info = {}
    x, tr, co = sstep_solve(prob, **_device_kwargs(ref), info=info)
    flags = ref["flags"]
    noise_flags = golden("noise_" + name)["counts"][:, 2:5]
    if (noise_flags == flags[:3]).all():  # the verdict never moved under noise
        assert [tr.converged, tr.stagnated, tr.diverged] == [bool(v) for v in flags[:3]]
    assert tr.outer_records == []  # the reference's fixed solver keeps none
    g_ref = ref["first_g"]
    d = g_ref.shape[0]
    g = info["first_gram"][:d, :d]
    scale = np.sqrt(np.outer(np.diag(g_ref), np.diag(g_ref)))
    assert np.max(np.abs(g - g_ref) / scale) <= 1e-12
    noise = golden("noise_" + name)
    horizon = int(noise["alpha_horizon"])
    marks = ref["outer_marks"]
    m5 = int(marks[5]) if len(marks) > 5 else len(ref["alphas"])
    m = min(m5, horizon)
    np.testing.assert_allclose(co.alphas[:m], ref["alphas"][:m], rtol=1e-8)
    np.testing.assert_allclose(co.betas[:m], ref["betas"][:m], rtol=1e-8)
    if horizon >= m5:  # no perturbed run moved inside the first 5 blocks
        np.testing.assert_array_equal(tr.s_schedule[:5], ref["s_schedule"][:5])
    counts = noise["counts"]
    tot_ref, out_ref = int(flags[3]), int(flags[4])
    for got, want, col in ((tr.total_iters, tot_ref, 1), (tr.total_outer, out_ref, 0)):
        # 2%, or the reference's own relative spread under Gram-order noise
        cmin, cmax = min(want, counts[:, col].min()), max(want, counts[:, col].max())
        tol = max(0.02, (cmax - cmin) / want)
        lo, hi = cmin * (1 - tol) - 1, cmax * (1 + tol) + 1
        assert lo <= got <= hi, (name, col, got, lo, hi)
    if flags[0]:
        assert tr.converged
    if tr.converged:
        assert _true_rel(prob, x) <= cfg_eps(ref)
        np.testing.assert_allclose(tr.true_resid[-1], _true_rel(prob, x), rtol=1e-6)


def cfg_eps(ref):
    return sstep_kwargs(ref)["eps_star"]


def test_fixed_sstep_fast_trace_keeps_every_decision(gpu_ready):
    prob = problems.make_problem("c1")
    kw = dict(s=8, eps_star=1e-10, basis_kind="newton", spectral_bounds=(0.004, 8.0))
    xf, tf, cf = sstep_solve(prob, **kw)
    xs, ts, cs = sstep_solve(prob, **kw, trace="fast")
    np.testing.assert_array_equal(cs.alphas, cf.alphas)
    np.testing.assert_array_equal(xs, xf)
    assert ts.s_schedule == tf.s_schedule and ts.converged == tf.converged


def test_fixed_sstep_s1_matches_hscg_alphas(gpu_ready):
    """s = 1 (monomial) is Hestenes-Stiefel CG (test_adaptive.py:76-87 analogue)."""
    ref = golden("sstep_spd40_mono1")
    h = golden("hscg_spd40")
    prob = sstep_problem("sstep_spd40_mono1", ref)
    _, tr, co = sstep_solve(prob, 1, 1e-10)
    # up to the reference's own noise horizon (its Gram order moves alpha there)
    m = min(len(co.alphas), len(h["alphas"]), int(golden("noise_sstep_spd40_mono1")["alpha_horizon"]))
    np.testing.assert_allclose(co.alphas[:m], h["alphas"][:m], rtol=1e-8)


def test_fixed_sstep_errors(gpu_ready):
    prob = problems.make_problem("c1", scale=8)
    with pytest.raises(ValueError):
        sstep_solve(prob, 0, 1e-8)
    with pytest.raises(ValueError):
        sstep_solve(prob, 17, 1e-8)
    short = O.params_monomial(3)
    with pytest.raises(ParameterError):
        sstep_solve(prob, 5, 1e-8, params=BasisParams("monomial", np.asarray(short.thetas),
                                                      np.asarray(short.gammas),
                                                      np.asarray(short.mus)))
    with pytest.raises(ParameterError):
        sstep_solve(prob, 4, 1e-8, basis_kind="legendre")


def test_adaptive_after_fixed_on_one_plan(gpu_ready):
    """A plan used by sstep_solve(params=...) solves adaptively as before."""
    from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve
    ref = golden("solve_c1")
    prob = problems.make_problem("c1")
    p = O.params_chebyshev(0.004, 8.0, 8)
    sstep_solve(prob, 8, 1e-10, params=BasisParams("chebyshev", np.asarray(p.thetas),
                                                   np.asarray(p.gammas), np.asarray(p.mus)))
    x, tr, co = adaptive_solve(prob, AdaptiveConfig(sigma=8, eps_star=1e-10, basis_kind="newton"))
    assert tr.converged and tr.total_outer == int(ref["flags"][4])
