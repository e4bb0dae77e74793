"""GPU tier: pattern-compressed level kernels (mpk.cu k_level_pat, k_level_ss,
k_level_zm).

A plan whose rows reduce to a small table of (relative column, value)
patterns streams 1- or 2-byte row ids instead of CSR.  Columns, values and
stored order are A's, so every solve must be bit-identical to the CSR
kernels (SSCG_PATTERN=0): basis, Gram, alphas and the iterate."""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems
from paper_1908_04081_b200.kernels import _plan
from paper_1908_04081_b200.types import ProblemInstance, SparseMatrix

pytestmark = pytest.mark.gpu


_KEYS = ("SSCG_PATTERN", "SSCG_PAT_SS", "SSCG_ZM", "SSCG_ZM_ZC", "SSCG_ZM_2D", "SSCG_VS",
         "SSCG_ZM_DYN", "SSCG_TM", "SSCG_TM_EXACT", "SSCG_VS_SYM")


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in _KEYS}
    try:
        for k in _KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _instance(m, seed, label):
    m = m.tocsr()
    m.sort_indices()
    n = m.shape[0]
    a = SparseMatrix(n=n, row_ptr=m.indptr.astype(np.int64), col_idx=m.indices.astype(np.int32),
                     values=m.data.astype(np.float64), n_a=int(np.diff(m.indptr).max()))
    dense = m.toarray()
    ev = np.linalg.eigvalsh(dense)
    rng = np.random.default_rng(seed)
    return ProblemInstance(a=a, b=rng.standard_normal(n), x0=np.zeros(n),
                           norm_a=float(ev[-1]), norm_abs_a=float(np.linalg.norm(abs(dense), 2)),
                           kappa_a=float(ev[-1] / ev[0]), label=label)


def _tridiag_many_patterns(n=1200, distinct=300, seed=3):
    """Tridiagonal SPD matrix with `distinct` diagonal values: > 256 patterns,
    so the plan uses 2-byte row ids."""
    rng = np.random.default_rng(seed)
    diag = 2.5 + rng.integers(0, distinct, n) / distinct
    return _instance(sp.diags([-np.ones(n - 1), diag, -np.ones(n - 1)], [-1, 0, 1]), seed, "tri")


def _random_spd(n=800, seed=5):
    m = sp.random(n, n, density=6.0 / n, random_state=seed, format="csr")
    return _instance(m + m.T + sp.identity(n) * 14.0, seed, "rand")


CASES = [
    ("c1", lambda: problems.make_problem("c1"), dict(sigma=8, eps_star=1e-10, basis_kind="newton"),
     "pattern"),
    ("c3", lambda: problems.make_problem("c3", scale=24),
     dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev"), "pattern"),
    ("c5", lambda: problems.make_problem("c5", scale=28),
     dict(sigma=12, eps_star=1e-10, basis_kind="newton"), "pattern"),
    ("tri300", _tridiag_many_patterns, dict(sigma=6, eps_star=1e-9, basis_kind="newton"), "pattern"),
    ("rand", _random_spd, dict(sigma=6, eps_star=1e-9, basis_kind="monomial"), "csr"),
]


@pytest.mark.parametrize("name,make,kw,kind", CASES, ids=[c[0] for c in CASES])
def test_pattern_bit_identical_to_csr(gpu_ready, name, make, kw, kind):
    cfg = AdaptiveConfig(**kw)

    def run():
        prob = make()
        return _plan(prob.a).mpk_schedule(cfg.sigma), adaptive_solve(prob, cfg, trace="fast")

    s0, ref = _with_env({"SSCG_PATTERN": "0"}, run)
    s1, got = _with_env({}, run)
    assert s0["kind"] == "csr" and s1["kind"] == kind, (s0, s1)
    assert ref[1].converged
    np.testing.assert_array_equal(got[2].alphas, ref[2].alphas)
    np.testing.assert_array_equal(got[0], ref[0])
    assert got[1].total_outer == ref[1].total_outer


def test_pattern_counts(gpu_ready):
    """Translation classes of the stencils: 2D 5-point 3x3 = 9, 3D 7-point 27;
    the 300-value tridiagonal needs 2-byte ids."""
    assert _plan(problems.make_problem("c1").a).mpk_schedule(8)["patterns"] == 9
    assert _plan(problems.make_problem("c5", scale=16).a).mpk_schedule(8)["patterns"] == 27
    s = _plan(_tridiag_many_patterns().a).mpk_schedule(6)
    assert s["kind"] == "pattern" and 256 < s["patterns"] <= 900


def test_pattern_kernel_forms(gpu_ready):
    """Which pattern kernel a plan takes: the plane march for stencils whose
    plane stride S >= 256 (c3, c5), the superset mask for small strides (c1:
    S = 64; the tridiagonal), the table walk when disabled."""
    def form(prob, env=None):
        return _with_env(env or {}, lambda: _plan(prob().a).mpk_schedule(8)["form"])
    assert form(lambda: problems.make_problem("c5", scale=28)) == "march"
    assert form(lambda: problems.make_problem("c5", scale=32)) == "tma march"
    assert form(lambda: problems.make_problem("c5", scale=32), {"SSCG_TM": "0"}) == "march"
    assert form(lambda: problems.make_problem("c3", scale=24)) == "march"
    assert form(lambda: problems.make_problem("c1")) == "superset"
    assert form(_tridiag_many_patterns) == "superset"
    assert form(lambda: problems.make_problem("c5", scale=28), {"SSCG_ZM": "0"}) == "superset"
    assert form(lambda: problems.make_problem("c5", scale=28), {"SSCG_PAT_SS": "0"}) == "table"


@pytest.mark.parametrize("env", [{"SSCG_ZM": "0"}, {"SSCG_PAT_SS": "0"}, {"SSCG_ZM_ZC": "3"},
                                 {"SSCG_ZM_2D": "0"}, {"SSCG_ZM_DYN": "0"}, {"SSCG_TM": "0"},
                                 {"SSCG_TM": "0", "SSCG_ZM_DYN": "0"}, {"SSCG_TM_EXACT": "0"}],
                         ids=["superset", "table", "march_zc3", "march_1d", "static_items",
                              "register_march", "register_march_static", "tma_mul_then_add"])
def test_pattern_forms_bit_identical(gpu_ready, env):
    """Plane march (default), its opt-in variants, superset mask and table
    walk run the same rounded operations in the same order: identical solves
    (Newton and Chebyshev bases, unit and non-unit gamma, mu != 0).  The 32^3
    grids give whole 32 x 8 column tiles: the default there is the TMA march,
    so the reference run and every variant compare the TMA-fed and register
    marches too; the TMA march's exact-product form (one fma per 0 / +-1 entry,
    the default on these Poisson operators) against its mul-then-add form."""
    for key, scale, kw in (("c5", 28, dict(sigma=12, eps_star=1e-10, basis_kind="newton")),
                           ("c3", 24, dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev")),
                           ("c5", 32, dict(sigma=12, eps_star=1e-10, basis_kind="newton")),
                           ("c3", 32, dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev"))):
        cfg = AdaptiveConfig(**kw)
        ref = adaptive_solve(problems.make_problem(key, scale=scale), cfg, trace="fast")
        got = _with_env(env, lambda: adaptive_solve(problems.make_problem(key, scale=scale), cfg,
                                                    trace="fast"))
        np.testing.assert_array_equal(got[2].alphas, ref[2].alphas)
        np.testing.assert_array_equal(got[0], ref[0])


def test_pattern_full_trace_and_partitioned_agree(gpu_ready):
    """Full diagnostics and the virtual-group (row-slab) path through the
    pattern kernels reproduce the CSR single-GPU solve."""
    from paper_1908_04081_b200.dist import VirtualGroup
    from paper_1908_04081_b200.partition import CsrRows
    kw = dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev")
    ref = _with_env({"SSCG_PATTERN": "0"},
                    lambda: adaptive_solve(problems.make_problem("c3", scale=24), AdaptiveConfig(**kw)))
    x, tr, co = adaptive_solve(problems.make_problem("c3", scale=24), AdaptiveConfig(**kw))
    np.testing.assert_array_equal(x, ref[0])
    # ||b - A x|| per outer loop: the same rows, summed in the kernel's own
    # order (the plane-march level 0 groups rows by column), so only the
    # rounding of the norm may differ
    np.testing.assert_allclose(tr.true_resid, ref[1].true_resid, rtol=1e-14, atol=0)
    prob = problems.make_problem("c3", scale=24)
    xg, tg, cg, _ = VirtualGroup(CsrRows.of(prob.a), 1, depth=10).solve(prob, AdaptiveConfig(**kw))
    np.testing.assert_array_equal(xg, ref[0])


@pytest.mark.parametrize("key,kw", [
    ("c4", dict(sigma=10, eps_star=1e-8, basis_kind="newton", max_outer=60)),
    ("c4j", dict(sigma=10, eps_star=1e-8, basis_kind="newton")),
    ("c4j", dict(sigma=8, eps_star=1e-8, basis_kind="chebyshev")),
], ids=["c4", "c4j", "c4j_cheb"])
def test_value_stream_bit_identical_to_csr(gpu_ready, key, kw):
    """Row-varying 27-point operators (c4) run the value-stream stencil kernels
    (k_level_vs: union offsets as parameters, values slot-major): the same
    rounded operations in stored order as csr_matvec, so the solve is
    identical to the CSR kernels' (SSCG_VS=0)."""
    cfg = AdaptiveConfig(**kw)

    def run():
        prob = problems.make_problem(key, scale=16)
        return _plan(prob.a).mpk_schedule(cfg.sigma), adaptive_solve(prob, cfg, trace="fast")

    s0, ref = _with_env({"SSCG_VS": "0"}, run)
    s1, got = _with_env({}, run)
    assert s0["kind"] == "csr" and s1["kind"] == "stencil values" and s1["slots"] == 27, (s0, s1)
    np.testing.assert_array_equal(got[2].alphas, ref[2].alphas)
    np.testing.assert_array_equal(got[0], ref[0])
    assert got[1].total_outer == ref[1].total_outer
    # these operators are bitwise symmetric: the default streams the diagonal's
    # and the upper offsets' planes only; the full-plane form must agree too
    assert s1["form"] == "symmetric" and s1["planes"] == 14, s1
    s2, full = _with_env({"SSCG_VS_SYM": "0"}, run)
    assert s2["form"] is None and s2["planes"] == 27, s2
    np.testing.assert_array_equal(full[2].alphas, ref[2].alphas)
    np.testing.assert_array_equal(full[0], ref[0])


def test_value_stream_symmetric_form_needs_bitwise_symmetry(gpu_ready):
    """One entry one ulp away from its mirror image: the plan must keep every
    plane (the symmetric form would read the mirror's bits), and the solve
    stays the CSR kernels'."""
    cfg = AdaptiveConfig(sigma=8, eps_star=1e-8, basis_kind="newton", max_outer=12)

    def run():
        prob = problems.make_problem("c4j", scale=16)
        a = prob.a
        a.values = np.array(a.values, copy=True)
        i = a.n // 2
        j = int(a.row_ptr[i])  # the row's first (a lower) entry
        assert a.col_idx[j] < i
        a.values[j] = np.nextafter(a.values[j], np.inf)
        return _plan(a).mpk_schedule(cfg.sigma), adaptive_solve(prob, cfg, trace="fast")

    s0, ref = _with_env({"SSCG_VS": "0"}, run)
    s1, got = _with_env({}, run)
    assert s1["kind"] == "stencil values" and s1["form"] is None and s1["planes"] == 27, s1
    np.testing.assert_array_equal(got[2].alphas, ref[2].alphas)
    np.testing.assert_array_equal(got[0], ref[0])



def test_staged_host_copies_round_trip(gpu_ready):
    """Vectors of >= 16 MB move through the per-thread pinned chunk pipelines
    (plan.cu staged_copy; all-zero chunks of an upload are set on the device),
    and x comes back into a page-locked block of the result pool by one DMA;
    every combination must be bit-identical to plain cudaMemcpy transfers
    (SSCG_STAGE_COPY=0) into a plain numpy array."""
    import gc
    from paper_1908_04081_b200 import _lib as L
    kw = dict(sigma=12, eps_star=1e-10, basis_kind="newton", max_outer=3)

    def run(env, pool):
        old = os.environ.get("SSCG_STAGE_COPY")
        old_pool = L.result_pool
        os.environ["SSCG_STAGE_COPY"] = env
        L.result_pool = pool
        try:
            prob = problems.make_problem("c5", scale=136)  # 2.5 M rows: 20 MB vectors
            n = prob.a.n
            prob.x0[n // 2:] = np.linspace(-1e-3, 1e-3, n - n // 2)  # zero chunks, then data
            return adaptive_solve(prob, AdaptiveConfig(**kw), trace="fast")
        finally:
            L.result_pool = old_pool
            if old is None:
                os.environ.pop("SSCG_STAGE_COPY", None)
            else:
                os.environ["SSCG_STAGE_COPY"] = old

    plain = L.PinnedPool(max_bytes=0)  # hands out numpy arrays only
    ref = run("0", plain)
    assert ref[0].nbytes >= 16 << 20 and ref[0].base is None
    staged = run("1", plain)           # staged both ways
    pool = L.PinnedPool()
    pinned = run("1", pool)            # staged upload, x by one DMA into the pool's block
    assert pinned[0].base is not None and pool._pinned == 2 * pinned[0].nbytes  # + the spare
    for got in (staged, pinned):
        np.testing.assert_array_equal(got[0], ref[0])
        np.testing.assert_array_equal(got[2].alphas, ref[2].alphas)
    # the block returns to the pool only when the last view of x is gone
    del got
    ptr = pinned[0].ctypes.data
    view = pinned[0][5:10]
    nb = pinned[0].nbytes
    pinned = None
    gc.collect()
    assert pool._free[nb] and ptr not in pool._free[nb]  # only the spare is free
    view = None
    gc.collect()
    assert ptr in pool._free[nb] and pool._pinned == 2 * nb


def test_staged_upload_covers_every_byte(gpu_ready):
    """The CSR arrays of a plan go up through the staged chunk pipelines, one
    contiguous range per copy thread.  4 (n + 1) bytes of row_ptr with n a
    multiple of 8 * 4096 / 4 is the size whose last word falls off a partition
    rounded down: the last row would end at 0 (found by bench.py's CSR line on
    c5w).  A bidiagonal operator of 2^22 rows: y = A x must be right at the
    last row."""
    from paper_1908_04081_b200.kernels import spmv
    n = 1 << 22
    row_ptr = np.concatenate([[0], np.cumsum(np.r_[1, np.full(n - 1, 2)])]).astype(np.int64)
    col = np.empty(2 * n - 1, dtype=np.int64)
    col[0] = 0
    col[1::2] = np.arange(n - 1)
    col[2::2] = np.arange(1, n)
    val = np.empty(2 * n - 1)
    val[0] = 2.0
    val[1::2] = -0.5
    val[2::2] = 2.0
    a = SparseMatrix(n=n, row_ptr=row_ptr, col_idx=col, values=val, n_a=2, is_symmetric=False)
    assert 4 * (n + 1) >= 16 << 20  # staged
    x = np.linspace(1.0, 2.0, n)
    y = spmv(a, x)
    ref = 2.0 * x
    ref[1:] += -0.5 * x[:-1]
    np.testing.assert_array_equal(y[-4:], ref[-4:])
    np.testing.assert_array_equal(y[:4], ref[:4])
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("shape", [(17, 16, 5), (40, 9, 13), (33, 33, 3), (256, 1, 6),
                                   (64, 8, 2), (32, 16, 40), (96, 24, 7)],
                         ids=lambda s: "x".join(map(str, s)))
def test_march_edge_shapes_bit_identical(gpu_ready, shape):
    """Plane-march edge cases against the CSR kernels: x-lines that are not a
    multiple of 32 (no 2-D tiles), planes of a single line (the 5-slot union),
    two or three planes, more planes per item than the grid has, partial last
    items -- Newton (Leja chain: per-CTA claiming) and Chebyshev (fixed
    stripes, two-back term)."""
    from paper_1908_04081_b200.problems import poisson3d
    for kw in (dict(sigma=6, eps_star=1e-10, basis_kind="newton", max_outer=8),
               dict(sigma=5, eps_star=1e-10, basis_kind="chebyshev", max_outer=8)):
        cfg = AdaptiveConfig(**kw)

        def run():
            prob = poisson3d(*shape)
            return _plan(prob.a).mpk_schedule(cfg.sigma), adaptive_solve(prob, cfg, trace="fast")

        s0, ref = _with_env({"SSCG_PATTERN": "0"}, run)
        s1, got = _with_env({}, run)
        assert s0["kind"] == "csr" and s1["kind"] == "pattern", (s0, s1)
        np.testing.assert_array_equal(got[2].alphas, ref[2].alphas)
        np.testing.assert_array_equal(got[0], ref[0])
