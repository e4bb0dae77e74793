"""GPU tier for the row-partitioned solve.

With one GPU the multi-rank algorithm is exercised two ways:
  * VirtualGroup: P = 1..4 rank plans in one process on one device, halo by
    device copies and the Gram allreduce as a fixed-order sum (no kernel waits
    on another -- the ranks run in lock step on one stream);
  * the NCCL transport at world size 1: a real communicator, the halo exchange
    and the allreduce captured in the outer-loop CUDA graph.
Both must reproduce the single-GPU solve: P = 1 bit for bit, P > 1 up to the
Gram summation order (first Gram 1e-12, s sequence, convergence)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import cfg_of, golden
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems
from paper_1908_04081_b200.dist import VirtualGroup, solve_partitioned
from paper_1908_04081_b200.partition import CsrRows, Stencil7Rows

pytestmark = pytest.mark.gpu


def true_rel(prob, x):
    a = prob.a
    m = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n))
    return np.linalg.norm(prob.b - m @ x) / np.linalg.norm(prob.b)


@pytest.mark.parametrize("case,key,scale", [("solve_c1", "c1", None), ("solve_c3p", "c3", 24),
                                            ("solve_c5p", "c5", 24)])
@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_virtual_group_matches_single_gpu(gpu_ready, case, key, scale, world):
    ref = golden(case)
    kw = cfg_of(ref)
    prob = problems.make_problem(key, scale=scale)
    x1, t1, c1 = adaptive_solve(prob, AdaptiveConfig(**kw), trace="fast")
    grp = VirtualGroup(CsrRows.of(prob.a), world, depth=kw["sigma"])
    xg, tg, cg, logs = grp.solve(prob, AdaptiveConfig(**kw))
    assert tg.converged and true_rel(prob, xg) <= kw["eps_star"]
    if world == 1:  # no ghosts, same arithmetic: bit for bit
        np.testing.assert_array_equal(xg, x1)
        np.testing.assert_array_equal(cg.alphas, c1.alphas)
        return
    recs = ref["rec_int"]
    got = [(r.s_tilde, r.s_actual) for r in tg.outer_records[:5]]
    assert got == [tuple(v) for v in recs[:5, 2:4]]
    m = int(ref["outer_marks"][4] + recs[4, 3]) if len(recs) >= 5 else len(cg.alphas)
    np.testing.assert_allclose(cg.alphas[:m], c1.alphas[:m], rtol=1e-8)
    assert abs(tg.total_outer - t1.total_outer) <= max(1, 0.02 * t1.total_outer)


def test_virtual_group_stencil_rows_generator(gpu_ready):
    """Slabs built from the on-demand stencil generator (what the weak-scaled
    bench uses) give the same solve as the global CSR."""
    prob = problems.make_problem("c5", scale=20)
    kw = dict(sigma=12, eps_star=1e-10, basis_kind="newton")
    a = VirtualGroup(CsrRows.of(prob.a), 3, 12).solve(prob, AdaptiveConfig(**kw))
    b = VirtualGroup(Stencil7Rows(20, 20, 20), 3, 12).solve(prob, AdaptiveConfig(**kw))
    np.testing.assert_array_equal(a[0], b[0])


def test_nccl_world1_matches_single_gpu(gpu_ready):
    prob = problems.make_problem("c3", scale=24)
    kw = dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev")
    x1, t1, c1 = adaptive_solve(prob, AdaptiveConfig(**kw), trace="fast")
    xo, tr, co, plan = solve_partitioned(
        CsrRows.of(prob.a), prob, prob.b, prob.x0, AdaptiveConfig(**kw), rank=0, world=1,
        device=0, exchange=lambda obj: [obj], broadcast_bytes=lambda b: b)
    np.testing.assert_array_equal(xo, x1)
    np.testing.assert_array_equal(co.alphas, c1.alphas)
    assert tr.converged and tr.total_outer == t1.total_outer


def test_partitioned_rejects_sigma_above_depth(gpu_ready):
    prob = problems.make_problem("c1", scale=16)
    grp = VirtualGroup(CsrRows.of(prob.a), 2, depth=4)
    with pytest.raises(Exception):
        grp.solve(prob, AdaptiveConfig(sigma=6, eps_star=1e-8))


@pytest.mark.parametrize("world", [2, 3, 4])
def test_partitioned_slabs_keep_the_plane_march(gpu_ready, world):
    """Every rank of a stencil slab partition runs the plane-march kernels:
    patterns in global offsets, the owned and ghost planes walked through a
    plane table (sscg_part.global_rows), not only the bottom slab whose local
    rows happen to be in grid order."""
    from paper_1908_04081_b200.dist import VirtualGroup
    g = VirtualGroup(Stencil7Rows(32, 32, 32 * world), world, 12)
    assert [pl.mpk_schedule(12)["form"] for pl in g.plans] == ["march"] * world



@pytest.mark.parametrize("shape,world", [((40, 9, 15), 3), ((17, 16, 12), 2), ((33, 33, 8), 4)],
                         ids=["40x9x15-3", "17x16x12-2", "33x33x8-4"])
def test_partitioned_march_edge_shapes(gpu_ready, shape, world):
    """Odd slab shapes through the plane table (x-lines not a multiple of 32,
    thin slabs whose ghost planes reach past the neighbour): every rank marches
    and the partitioned solve converges like the single-GPU one."""
    from paper_1908_04081_b200.problems import poisson3d
    prob = poisson3d(*shape)
    kw = dict(sigma=6, eps_star=1e-10, basis_kind="newton")
    x1, t1, c1 = adaptive_solve(prob, AdaptiveConfig(**kw), trace="fast")
    grp = VirtualGroup(CsrRows.of(prob.a), world, depth=kw["sigma"])
    assert [pl.mpk_schedule(6)["form"] for pl in grp.plans] == ["march"] * world
    xg, tg, cg, _ = grp.solve(prob, AdaptiveConfig(**kw))
    assert tg.converged and true_rel(prob, xg) <= kw["eps_star"]
    np.testing.assert_allclose(cg.alphas[:5], c1.alphas[:5], rtol=1e-8)
