"""GPU tier for Hestenes-Stiefel CG (`hscg_solve`, classic.py:33-104; SURVEY.md
8(f) row 2) against golden runs of the reference (oracle/make_golden.py
gen_hscg; the oracle restatement reproduces them bit for bit).

The device sums its dots in a fixed tree order, not BLAS ddot's, so alpha /
beta are held to 1e-8 up to the reference's own noise horizon (the first
iteration where its runs with a chunked dot move by more than 1e-8; 1e-8 to
80% of it, 1e-6 up to it) and the
iteration count to max(2%, the spread of those runs).  Covers the pattern
kernels (c1, c3 proxy) and the CSR kernels (dense spd40/spd50, 494_bus)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import cfg_of, golden
from test_oracle_golden import HSCG_CASES, hscg_problem
from paper_1908_04081_b200 import CgCoefficients, assemble_tridiag, hscg_solve, problems
from paper_1908_04081_b200.kernels import _plan

pytestmark = pytest.mark.gpu


def _true_rel(prob, x):
    a = prob.a
    m = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n))
    return np.linalg.norm(prob.b - m @ x) / np.linalg.norm(prob.b)


@pytest.mark.parametrize("name", HSCG_CASES)
def test_hscg_parity(gpu_ready, name):
    ref = golden(name)
    prob = hscg_problem(name, ref)
    kw = cfg_of(ref)
    x, tr, co = hscg_solve(prob, **kw)
    flags = ref["flags"]
    noise = ref["noise_counts"]
    if (noise[:, 1:4] == flags[:3]).all():
        assert [tr.converged, tr.stagnated, tr.diverged] == [bool(v) for v in flags[:3]]
    # the device's tree order is one more perturbation of the same kind as the
    # sampled ones, so it may cross 1e-8 a little before their horizon
    hz = min(int(ref["alpha_horizon"]), len(ref["alphas"]))
    h = hz if hz == len(ref["alphas"]) else int(0.8 * hz)
    np.testing.assert_allclose(co.alphas[:h], ref["alphas"][:h], rtol=1e-8)
    np.testing.assert_allclose(co.betas[:h], ref["betas"][:h], rtol=1e-8)
    np.testing.assert_allclose(co.alphas[:hz], ref["alphas"][:hz], rtol=1e-6)
    np.testing.assert_allclose(tr.true_resid[:h], ref["true_resid"][:h], rtol=1e-6)
    np.testing.assert_allclose(tr.lambda_max[:h], ref["lambda_max"][:h], rtol=1e-8)
    want = int(flags[3])
    cmin, cmax = min(want, noise[:, 0].min()), max(want, noise[:, 0].max())
    tol = max(0.02, (cmax - cmin) / max(want, 1))
    assert cmin * (1 - tol) - 1 <= tr.total_iters <= cmax * (1 + tol) + 1
    assert tr.total_outer == tr.total_iters and tr.s_schedule == [1] * tr.total_iters
    if tr.converged:
        assert _true_rel(prob, x) <= kw["eps_star"]
        np.testing.assert_allclose(tr.true_resid[-1], _true_rel(prob, x), rtol=1e-6)


@pytest.mark.parametrize("env,cases", [
    ({"SSCG_PATTERN": "0"}, (("c1", None),)),
    ({"SSCG_HS_SS": "0"}, (("c1", None), ("c5", 28))),
], ids=["csr", "table_walk"])
def test_hscg_kernel_modes_agree(gpu_ready, env, cases):
    """Superset-mask pattern rows (default), table-walk pattern rows and CSR
    rows give the same solve bit for bit: the row sums are identical, and the
    dots too where both plans use the same grid (c1 for CSR; the pattern forms
    of one plan always do, c5 proxy for the 7-slot union)."""
    import os
    for key, scale in cases:
        prob = problems.make_problem(key, scale=scale)
        assert _plan(prob.a).mpk_schedule(8)["kind"] == "pattern"
        x1, t1, c1 = hscg_solve(prob, 1e-10)
        os.environ.update(env)
        try:
            prob2 = problems.make_problem(key, scale=scale)
            x2, t2, c2 = hscg_solve(prob2, 1e-10)
        finally:
            for k in env:
                os.environ.pop(k, None)
        np.testing.assert_array_equal(c1.alphas, c2.alphas)
        np.testing.assert_array_equal(x1, x2)


def test_hscg_max_iters_zero_and_tridiag(gpu_ready):
    prob = problems.make_problem("c1", scale=16)
    x, tr, co = hscg_solve(prob, 1e-10, max_iters=0)
    assert tr.total_iters == 0 and not (tr.converged or tr.stagnated or tr.diverged)
    np.testing.assert_array_equal(x, prob.x0)
    _, tr, co = hscg_solve(prob, 1e-10)
    t = assemble_tridiag(co, 5)
    assert np.allclose(t, t.T) and t.shape == (5, 5)


def test_hscg_production_mode(gpu_ready):
    """Production HSCG (one SpMV per iteration, verdicts on the updated
    residual, the true residual formed once at the end): the same alphas as the
    reference-semantics run while both iterate, and the final true residual
    meets eps*."""
    prob = problems.make_problem("c3", scale=24)
    x1, t1, c1 = hscg_solve(prob, 1e-10)
    x2, t2, c2 = hscg_solve(prob, 1e-10, mode="production")
    assert t1.converged and t2.converged
    m = min(len(c1.alphas), len(c2.alphas))
    # the production SpMV kernel runs a larger grid (one row sum per row), so its
    # p.Ap partials group differently: the same coefficients to rounding
    np.testing.assert_allclose(c2.alphas[:m], c1.alphas[:m], rtol=1e-11)
    assert abs(t2.total_iters - t1.total_iters) <= 2
    a = prob.a
    m_ = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n))
    rel = np.linalg.norm(prob.b - m_ @ x2) / np.linalg.norm(prob.b)
    assert t2.true_resid[-1] == pytest.approx(rel, rel=1e-8) and rel <= 1e-9


@pytest.mark.parametrize("mode", ["reference", "production"])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_hscg_distributed(gpu_ready, mode, world):
    """Distributed HSCG (§8(f)2): row slabs with depth-1 ghosts, per iteration
    one halo exchange and two reductions (virtual group: device copies and
    fixed-order sums).  P = 1 equals the single-GPU run bit for bit; P > 1
    agrees to reduction order (alphas 1e-10 early, same verdict, counts +-2)."""
    from paper_1908_04081_b200.dist import VirtualGroup
    from paper_1908_04081_b200.partition import CsrRows
    prob = problems.make_problem("c5", scale=20)
    x1, t1, c1 = hscg_solve(prob, 1e-10, mode=mode)
    g = VirtualGroup(CsrRows.of(prob.a), world, depth=1)
    xg, tg, cg = g.hscg(prob, 1e-10, mode=mode)
    if world == 1:
        np.testing.assert_array_equal(cg.alphas, c1.alphas)
        np.testing.assert_array_equal(xg, x1)
        return
    np.testing.assert_allclose(cg.alphas[:20], c1.alphas[:20], rtol=1e-10)
    assert tg.converged == t1.converged and abs(tg.total_iters - t1.total_iters) <= 2
    assert tg.true_resid[-1] <= 1e-10


def test_hscg_nccl_world1(gpu_ready):
    """The NCCL transport of distributed HSCG at world size 1 (halo and both
    allreduces captured in the iteration graph) reproduces the single GPU."""
    from paper_1908_04081_b200.dist import hscg_partitioned
    from paper_1908_04081_b200.partition import CsrRows
    prob = problems.make_problem("c3", scale=24)
    for mode in ("reference", "production"):
        x1, t1, c1 = hscg_solve(prob, 1e-10, mode=mode)
        xo, tr, co, plan = hscg_partitioned(CsrRows.of(prob.a), prob.b, prob.x0, 1e-10, 0, 1, 0,
                                            exchange=lambda o: [o], broadcast_bytes=lambda b: b,
                                            mode=mode)
        np.testing.assert_array_equal(xo, x1)
        np.testing.assert_array_equal(co.alphas, c1.alphas)
