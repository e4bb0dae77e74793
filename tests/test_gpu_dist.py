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
    # the captured outer-loop graph holds exactly one allreduce (the algorithm's
    # one synchronisation per outer loop) and one grouped halo exchange
    coll = plan.collectives()
    assert coll["allreduce_per_outer"] == 1 and coll["halo_exchanges_per_outer"] == 1, coll
    assert coll["kernel_nodes"] >= kw["sigma"] + 3, coll  # levels, Gram, K_small, recovery


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
    assert [pl.mpk_schedule(12)["form"] for pl in g.plans] == ["tma march"] * world
    # x lines of 28: the register march (the TMA boxes need 32-column tiles)
    g = VirtualGroup(Stencil7Rows(28, 28, 28 * world), world, 12)
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


@pytest.mark.parametrize("key,jacobi", [("c4", False), ("c4j", True)])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_partitioned_value_stream(gpu_ready, key, jacobi, world):
    """Row-varying 27-point slabs (c4 / c4j) keep the value-stream kernels on
    every rank: values slot-major in GLOBAL offsets, neighbours through the
    plane tables.  P = 1 is bit-identical to the single-GPU value stream (and
    so to CSR); P > 1 agrees up to the Gram summation order."""
    from paper_1908_04081_b200.partition import Varcoef27Rows
    n = 12
    prob = problems.make_problem(key, scale=n)
    kw = dict(sigma=10, eps_star=1e-8, basis_kind="newton", max_outer=30)
    info = {}
    x1, t1, c1 = adaptive_solve(prob, AdaptiveConfig(**kw), trace="fast", info=info)
    grp = VirtualGroup(Varcoef27Rows(n, jacobi=jacobi), world, depth=kw["sigma"])
    assert [pl.mpk_schedule(10)["kind"] for pl in grp.plans] == ["stencil values"] * world
    xg, tg, cg, logs = grp.solve(prob, AdaptiveConfig(**kw))
    if world == 1:
        np.testing.assert_array_equal(xg, x1)
        np.testing.assert_array_equal(cg.alphas, c1.alphas)
        return
    # the first block's Gram differs only in summation order (per-rank partials)
    g1, gg = info["first_gram"], logs.first_gram
    scale = np.sqrt(np.outer(np.diag(g1), np.diag(g1)))
    assert np.all(np.abs(gg - g1) <= 1e-12 * scale)
    # decisions agree until the noise horizon of this ill-conditioned operator
    # (c4j 12^3 moves s~ at outer loop 3 under a reordered Gram sum)
    got = [(r.s_tilde, r.s_actual) for r in tg.outer_records[:2]]
    assert got == [(r.s_tilde, r.s_actual) for r in t1.outer_records[:2]]
    m = sum(r.s_actual for r in t1.outer_records[:2])
    np.testing.assert_allclose(cg.alphas[:m], c1.alphas[:m], rtol=1e-8)


def test_device_group_single_process(gpu_ready):
    """The single-process multi-GPU drop-in (DeviceGroup: ncclCommInitAll, one
    host thread + stream per GPU) at the one GPU this box has: bit-identical to
    the single-GPU solve, one allreduce per outer loop in its graph, and
    adaptive_solve(devices=[...]) reaches it."""
    from paper_1908_04081_b200.dist import DeviceGroup
    prob = problems.make_problem("c3", scale=24)
    kw = dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev")
    x1, t1, c1 = adaptive_solve(prob, AdaptiveConfig(**kw), trace="fast")
    g = DeviceGroup(CsrRows.of(prob.a), [0], depth=10)
    info = {}
    x, tr, co = g.solve(prob, AdaptiveConfig(**kw), info=info)
    np.testing.assert_array_equal(x, x1)
    np.testing.assert_array_equal(co.alphas, c1.alphas)
    assert tr.converged and tr.total_outer == t1.total_outer and info["device_ms"] > 0
    coll = g.collectives()[0]
    assert coll["allreduce_per_outer"] == 1 and coll["halo_exchanges_per_outer"] == 1, coll
    g.close()
    # devices=[0] is the single-GPU path; duplicate devices are refused
    x2, _, _ = adaptive_solve(prob, AdaptiveConfig(**kw), trace="fast", devices=[0])
    np.testing.assert_array_equal(x2, x1)
    with pytest.raises(ValueError):
        adaptive_solve(prob, AdaptiveConfig(**kw), devices=[0, 0])
    with pytest.raises(ValueError):
        adaptive_solve(prob, AdaptiveConfig(**kw), trace="full", devices=[0, 1])


def test_group_create_refuses_duplicate_devices_in_c(gpu_ready):
    """sscg_group_create itself rejects a device listed twice (NCCL cannot put
    two ranks of one communicator on one GPU)."""
    import ctypes as C

    from paper_1908_04081_b200 import _lib as L
    from paper_1908_04081_b200.dist import _part_struct
    from paper_1908_04081_b200.partition import partition_all
    prob = problems.make_problem("c1", scale=16)
    parts = partition_all(CsrRows.of(prob.a), 2, 4)
    st = [_part_struct(p, r, 2, None, None) for r, p in enumerate(parts)]
    arr = (L.SscgPart * 2)(*[s for s, _ in st])
    hs = (C.c_void_p * 2)()
    devs = np.array([0, 0], dtype=np.int32)
    rc = L.load().sscg_group_create(C.cast(hs, C.POINTER(C.c_void_p)), 2, L.iptr(devs), arr)
    assert rc == L.EINVAL and b"distinct" in L.load().sscg_last_error()
