"""GPU tier for problem setup: operator norms by device power iteration
(matio.py:229-276) against the reference's estimates, and load_problem end to
end on the synthetic Matrix Market files (oracle/make_golden.py gen_matio).

Norms and dots are tree sums on the device, so the estimates match the
reference to the power method's resolution, not bit for bit: rtol 1e-8 where
it converged (tol 1e-10), 1e-9 after the same 500 unconverged iterations."""

import os

import numpy as np
import pytest

from conftest import ROOT, golden, golden_problem
from test_matio_host import MM, _files
from paper_1908_04081_b200.matio import (estimate_operator_norms, jacobi_precondition,
                                         load_problem, read_matrix_market)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k,name", _files())
def test_operator_norms_match_reference(gpu_ready, k, name):
    g = golden("matio")
    ref = g[f"f{k}_norms"]
    ah, _ = jacobi_precondition(read_matrix_market(os.path.join(MM, name)))
    est = estimate_operator_norms(ah)
    assert est.converged == bool(ref[5])
    rt = 1e-8 if est.converged else 1e-9
    np.testing.assert_allclose(est.norm_a, ref[0], rtol=rt)
    np.testing.assert_allclose(est.norm_abs_a, ref[1], rtol=rt)
    if np.isfinite(ref[2]):
        np.testing.assert_allclose(est.kappa_a, ref[2], rtol=1e-6)
        np.testing.assert_allclose(est.lambda_min, ref[3], rtol=1e-6)
    else:
        assert not np.isfinite(est.kappa_a)
    assert abs(est.iters_used - int(ref[4])) <= 3


@pytest.mark.parametrize("name", ["problem_nos1", "problem_494bus"])
def test_acceptance_problem_norms(gpu_ready, name):
    """The reference's load_problem norms of its acceptance matrices."""
    prob = golden_problem(name)
    est = estimate_operator_norms(prob.a)
    np.testing.assert_allclose(est.norm_a, prob.norm_a, rtol=1e-8)
    np.testing.assert_allclose(est.norm_abs_a, prob.norm_abs_a, rtol=1e-8)
    np.testing.assert_allclose(est.kappa_a, prob.kappa_a, rtol=1e-6)


def test_load_problem_end_to_end(gpu_ready):
    g = golden("matio")
    k, name = _files()[0]
    prob = load_problem(os.path.join(MM, name), label="p48")
    np.testing.assert_array_equal(prob.a.values, g[f"f{k}_jvalues"])
    np.testing.assert_allclose(prob.norm_a, g[f"f{k}_norms"][0], rtol=1e-9)
    assert prob.label == "p48" and np.all(prob.x0 == 0) and prob.b.shape == (prob.a.n,)
