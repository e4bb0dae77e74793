"""GPU tier: behaviour the reference's own solver tests pin (test_classic.py,
test_sstep.py, test_adaptive.py), restated against this package's three GPU
solvers -- finite termination, identity systems, residual orthogonality of the
returned coefficients, s-step agreeing with classic CG early, block-mark
spacing, the paper's nos1 counts, and the degenerate inputs (b = 0,
x0 = the exact solution) with the reference's verdicts."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_problem
from paper_1908_04081_b200 import (AdaptiveConfig, ProblemInstance, SparseMatrix, adaptive_solve,
                                   hscg_solve, sstep_solve)

pytestmark = pytest.mark.gpu


def dense_problem(a, b=None, x0=None):
    a = np.asarray(a, dtype=float)
    n = a.shape[0]
    m = sp.csr_matrix(a)
    m.sort_indices()
    w = np.linalg.eigvalsh(a)
    return ProblemInstance(
        a=SparseMatrix(n=n, row_ptr=m.indptr.astype(np.int64), col_idx=m.indices.astype(np.int32),
                       values=m.data.copy(), n_a=int(np.diff(m.indptr).max())),
        b=np.full(n, 1.0 / np.sqrt(n)) if b is None else np.asarray(b, dtype=float),
        x0=np.zeros(n) if x0 is None else np.asarray(x0, dtype=float),
        norm_a=float(w[-1]), norm_abs_a=float(np.linalg.norm(abs(a), 2)),
        kappa_a=float(w[-1] / w[0]))


def spd(n, kappa, seed):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return (q * np.geomspace(1.0, kappa, n)) @ q.T


def test_identity_and_finite_termination(gpu_ready):
    rng = np.random.default_rng(0)
    b = rng.standard_normal(8)
    x, tr, _ = hscg_solve(dense_problem(np.eye(8), b), 1e-12)
    assert tr.converged and tr.total_iters == 1
    np.testing.assert_allclose(x, b, rtol=1e-14)
    d = np.repeat([1.0, 2.0, 5.0], 10)
    b = rng.standard_normal(30)
    prob = dense_problem(np.diag(d), b)
    x, tr, _ = hscg_solve(prob, 1e-12)
    assert tr.converged and tr.total_iters <= 5
    np.testing.assert_allclose(x, b / d, rtol=1e-10)
    for solve in (lambda p: adaptive_solve(p, AdaptiveConfig(sigma=4, eps_star=1e-12)),
                  lambda p: sstep_solve(p, 3, 1e-12)):
        x, tr, _ = solve(prob)
        assert tr.converged
        np.testing.assert_allclose(x, b / d, rtol=1e-9)


def test_hscg_coefficients_replay_orthogonal_residuals(gpu_ready):
    a = spd(60, 100.0, 2)
    prob = dense_problem(a)
    _, tr, co = hscg_solve(prob, 1e-10)
    tr.check_consistency()
    assert tr.total_outer == tr.total_iters
    r = prob.b.copy()
    p = r.copy()
    for i in range(min(10, len(co))):
        rn = r - co.alphas[i] * (a @ p)
        assert abs(rn @ r) / (np.linalg.norm(rn) * np.linalg.norm(r)) <= 1e-6
        p = rn + co.betas[i] * p
        r = rn


def test_sstep_matches_hscg_early_and_mark_spacing(gpu_ready):
    prob = dense_problem(spd(60, 80.0, 34))
    _, _, ref = hscg_solve(prob, 1e-13)
    for s in (2, 3):
        _, _, co = sstep_solve(prob, s, 1e-13)
        m = min(15, len(co), len(ref))
        np.testing.assert_allclose(co.alphas[:m], ref.alphas[:m], rtol=1e-6)
        np.testing.assert_allclose(co.betas[:m], ref.betas[:m], rtol=1e-6)
    _, tr, _ = sstep_solve(dense_problem(spd(50, 30.0, 37)), 4, 1e-10)
    assert tr.converged
    assert all(b - a == 4 for a, b in zip(tr.outer_marks, tr.outer_marks[1:]))
    assert tr.total_outer == int(np.ceil(tr.total_iters / 4))


def test_paper_counts_on_nos1(gpu_ready):
    """HSCG ~510 iterations on Jacobi-scaled nos1 at 1e-6
    (reference: 508); fixed s = 10, ~714 outer (7134 total) in the paper, 706
    (7058) in the reference -- but the reference's own count moves from ~3700
    to ~11600 iterations when only its Gram summation order changes
    (tests/golden/nos1_counts.npz), so the GPU is held to that envelope."""
    from conftest import golden
    g = golden("nos1_counts")
    prob = golden_problem("problem_nos1")
    _, tr, _ = hscg_solve(prob, 1e-6)
    assert tr.converged and tr.total_iters == pytest.approx(int(g["hscg"][0]), rel=0.02)
    assert tr.total_iters == pytest.approx(510, rel=0.15)
    _, tr, _ = sstep_solve(prob, 10, 1e-6)
    assert tr.converged
    env = g["sstep10"]
    assert env[:, 1].min() * 0.98 <= tr.total_iters <= env[:, 1].max() * 1.02
    assert env[:, 0].min() * 0.98 <= tr.total_outer <= env[:, 0].max() * 1.02


def test_degenerate_inputs(gpu_ready):
    """b = 0: ||b|| = 0 makes the relative residual NaN -> diverged after 0
    iterations (the reference's verdict); x0 = the exact solution: converged
    after 0 iterations, x returned unchanged."""
    m = np.diag(4.0 * np.ones(20)) - np.diag(np.ones(19), 1) - np.diag(np.ones(19), -1)
    zero = dense_problem(m, b=np.zeros(20))
    exact = dense_problem(m, b=m @ np.ones(20), x0=np.ones(20))
    cfg = AdaptiveConfig(sigma=4, eps_star=1e-10)
    for solve in (lambda p: adaptive_solve(p, cfg), lambda p: sstep_solve(p, 4, 1e-10),
                  lambda p: hscg_solve(p, 1e-10)):
        _, tr, _ = solve(zero)
        assert tr.diverged and not tr.converged and tr.total_iters == 0
        x, tr, _ = solve(exact)
        assert tr.converged and tr.total_iters == 0
        np.testing.assert_array_equal(x, np.ones(20))
