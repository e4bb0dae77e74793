"""Generate tests/golden/*.npz by running the REFERENCE package itself.

Test infrastructure only.  Run in the build container, where the reference is
importable (it does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python oracle/make_golden.py

Every fixture records the reference's outputs for seeded inputs built by
`paper_1908_04081_b200.problems` (or inline seeded numpy), so that
  * tests/test_oracle_golden.py pins oracle/sscg_oracle.py to the reference, and
  * the -m gpu parity tests compare the CUDA path with the reference's own
    numbers without needing the reference at run time.
The nos1 / 494_bus fixtures store the *preconditioned* problem exactly as the
reference's `load_problem` builds it (matio.py:291-307), as input vectors.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

import sstepcg  # noqa: E402  (the reference)
from sstepcg import adaptive as ref_adaptive  # noqa: E402
from sstepcg import basis as ref_basis  # noqa: E402
from sstepcg import lacore as ref_lacore  # noqa: E402
from sstepcg import ritz as ref_ritz  # noqa: E402
from sstepcg.matio import ProblemInstance as RefProblem  # noqa: E402
from sstepcg.matio import SparseMatrix as RefSparse  # noqa: E402

from paper_1908_04081_b200 import problems  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"  wrote {name}.npz ({os.path.getsize(path) / 1024:.1f} KB)")


def to_ref(prob):
    a = prob.a
    ra = RefSparse(n=a.n, row_ptr=np.asarray(a.row_ptr), col_idx=np.asarray(a.col_idx),
                   values=np.asarray(a.values), n_a=a.n_a)
    return RefProblem(a=ra, b=prob.b.copy(), x0=prob.x0.copy(), norm_a=prob.norm_a,
                      norm_abs_a=prob.norm_abs_a, kappa_a=prob.kappa_a, label=prob.label)


def spd_dense(n, kappa, seed):
    """tests/conftest.py:49-54 style: QR-rotated geomspace spectrum."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return (q * np.geomspace(1.0, kappa, n)) @ q.T


def dense_problem(a_dense, label):
    from scipy import sparse as sp
    a_dense = np.asarray(a_dense, dtype=float)
    n = a_dense.shape[0]
    rows, cols = np.nonzero(a_dense)
    m = sp.coo_matrix((a_dense[rows, cols], (rows, cols)), shape=(n, n)).tocsr()
    m.sum_duplicates()
    m.sort_indices()
    w = np.linalg.eigvalsh(a_dense)
    ra = RefSparse(n=n, row_ptr=m.indptr.copy(), col_idx=m.indices.copy(),
                   values=m.data.copy(), n_a=int(np.diff(m.indptr).max()))
    return RefProblem(a=ra, b=np.full(n, 1.0 / np.sqrt(n)), x0=np.zeros(n),
                      norm_a=float(w[-1]), norm_abs_a=float(np.linalg.norm(np.abs(a_dense), 2)),
                      kappa_a=float(w[-1] / w[0]), label=label)


# ---------------------------------------------------------------------------
def gen_leja():
    cases = [(1.0, 3.0, 2, 10000), (1.0, 3.0, 5, 10000), (0.0, 4.0, 4, 10**5),
             (0.5, 2.5, 5, 20000), (1e-6, 2.0, 10, 10000), (0.25, 1.75, 6, 20000)]
    rng = np.random.default_rng(7001)
    for _ in range(40):
        lo = float(10 ** rng.uniform(-4, 1))
        hi = lo + float(10 ** rng.uniform(-2, 3))
        cases.append((lo, hi, int(rng.integers(3, 16)), int(rng.choice([1000, 10000]))))
    lo_a, hi_a, cnt, grid, pts = [], [], [], [], []
    for lo, hi, c, g in cases:
        lo_a.append(lo); hi_a.append(hi); cnt.append(c); grid.append(g)
        p = np.full(16, np.nan)
        p[:c] = ref_basis.leja_points(lo, hi, c, g)
        pts.append(p)
    save("leja", lo=np.array(lo_a), hi=np.array(hi_a), count=np.array(cnt),
         grid=np.array(grid), points=np.array(pts))


def gen_params():
    rng = np.random.default_rng(7002)
    rows = []
    for kind in ("monomial", "newton", "chebyshev"):
        for _ in range(6):
            s = int(rng.integers(1, 13))
            lo = float(rng.uniform(0.01, 1.0))
            hi = lo + float(rng.uniform(0.1, 10.0))
            p = ref_basis.params_for(kind, s, lo, hi)
            b = ref_basis.assemble_change_of_basis(s, p)
            rows.append((kind, s, lo, hi, p, b))
    out = {}
    for i, (kind, s, lo, hi, p, b) in enumerate(rows):
        out[f"c{i}_meta"] = np.array([["monomial", "newton", "chebyshev"].index(kind), s, lo, hi])
        out[f"c{i}_thetas"] = p.thetas
        out[f"c{i}_gammas"] = p.gammas
        out[f"c{i}_mus"] = p.mus
        out[f"c{i}_bmat"] = b
    out["ncases"] = np.array(len(rows))
    save("params", **out)


def gen_ritz():
    rng = np.random.default_rng(7003)
    seqs = []
    for _ in range(30):
        m = int(rng.integers(1, 40))
        al = rng.uniform(1e-3, 1e3, m)
        be = rng.uniform(1e-3, 1e3, m)
        if rng.random() < 0.3:
            k = int(rng.integers(0, m))
            be[k] = -be[k]  # breakdown entries are skipped by the caller
        seqs.append((al, be))
    out = {}
    for i, (al, be) in enumerate(seqs):
        st = ref_ritz.RitzState()
        rec = []
        for a_, b_ in zip(al, be):
            try:
                st.absorb_step(a_, b_)
            except ref_ritz.BreakdownSignal:
                pass
            rec.append([st.lambda_min, st.lambda_max, st.psi, st.c, st.xi_estimate(), st.count])
        out[f"s{i}_alpha"] = al
        out[f"s{i}_beta"] = be
        out[f"s{i}_rec"] = np.array(rec)
    out["nseq"] = np.array(len(seqs))
    out["full_bound"] = np.array([ref_ritz.full_bound_c(1, 1, 1.0, 1.0, 1.0),
                                  ref_ritz.full_bound_c(7, 27, 1.3, 2.5, 1e4)])
    save("ritz", **out)


def gen_gram_conds():
    rng = np.random.default_rng(7004)
    out = {}
    cases = []
    for t in range(24):
        n = int(rng.integers(20, 400))
        s_bar = int(rng.integers(1, 13))
        y = np.empty((n, 2 * s_bar + 1))
        d = np.geomspace(1.0, float(rng.uniform(2, 1e6)), n)
        y[:, 0] = rng.standard_normal(n)
        for k in range(1, s_bar + 1):
            y[:, k] = d * y[:, k - 1] / np.linalg.norm(d * y[:, k - 1])
        y[:, s_bar + 1] = rng.standard_normal(n)
        for k in range(1, s_bar):
            y[:, s_bar + 1 + k] = d * y[:, s_bar + k]
        g = ref_lacore.gram(y)
        conds = ref_lacore.nested_basis_conds(g, s_bar)
        c = float(10 ** rng.uniform(0, 8))
        eps_star = float(10 ** rng.uniform(-12, -4))
        rn = float(10 ** rng.uniform(-8, 0))
        st, _ = ref_adaptive.select_s_tilde(g, s_bar, c, ref_ritz.MACHINE_UNIT, eps_star, rn)
        out[f"t{t}_y"] = y
        out[f"t{t}_g"] = g
        out[f"t{t}_conds"] = conds
        out[f"t{t}_sel"] = np.array([s_bar, c, eps_star, rn, st])
        cases.append(t)
    # Jacobi eigensolver (full-bound c path)
    for t in range(6):
        m = rng.standard_normal((2 * t + 3, 2 * t + 3))
        m = m + m.T
        out[f"j{t}_m"] = m
        out[f"j{t}_w"] = ref_lacore.sym_eig(m)
    out["ncases"] = np.array(len(cases))
    save("gram_conds", **out)


def gen_blocks():
    rng = np.random.default_rng(7005)
    out = {}
    nc = 0
    for kind in ("monomial", "newton", "chebyshev"):
        for t in range(4):
            n = int(rng.integers(30, 300))
            s = int(rng.integers(1, 13))
            a_dense = spd_dense(n, float(rng.uniform(10, 1e4)), seed=9000 + nc)
            a_dense[np.abs(a_dense) < 0.05 * np.abs(a_dense).max()] = 0.0
            a_dense = 0.5 * (a_dense + a_dense.T) + n * 0.01 * np.eye(n)
            prob = dense_problem(a_dense, "blk")
            p = rng.standard_normal(n)
            r = rng.standard_normal(n)
            prm = ref_basis.params_for(kind, s, 0.5, 2.0)
            blk = ref_basis.build_block(prob.a, p, r, prm, s)
            out[f"b{nc}_rowptr"] = prob.a.row_ptr
            out[f"b{nc}_col"] = prob.a.col_idx
            out[f"b{nc}_val"] = prob.a.values
            out[f"b{nc}_p"] = p
            out[f"b{nc}_r"] = r
            out[f"b{nc}_thetas"] = prm.thetas
            out[f"b{nc}_gammas"] = prm.gammas
            out[f"b{nc}_mus"] = prm.mus
            out[f"b{nc}_y"] = blk.y
            out[f"b{nc}_g"] = blk.g
            out[f"b{nc}_s"] = np.array(s)
            nc += 1
    out["ncases"] = np.array(nc)
    save("blocks", **out)


def run_ref(prob, cfg_kwargs, store_x=True):
    cfg = ref_adaptive.AdaptiveConfig(**cfg_kwargs)
    first_g = {}
    orig = ref_basis.gram

    def spy(y):
        g = orig(y)
        if "g" not in first_g:
            first_g["g"] = g.copy()
        return g

    ref_basis.gram = spy
    try:
        t0 = time.perf_counter()
        x, trace, coeffs = ref_adaptive.adaptive_solve(prob, cfg)
        dt = time.perf_counter() - t0
    finally:
        ref_basis.gram = orig
    recs = trace.outer_records
    d = dict(
        alphas=np.array(coeffs.alphas), betas=np.array(coeffs.betas),
        s_schedule=np.array(trace.s_schedule), outer_marks=np.array(trace.outer_marks),
        true_resid=np.array(trace.true_resid), upd_resid=np.array(trace.upd_resid),
        resid_gap=np.array(trace.resid_gap), c_values=np.array(trace.c_values),
        psi=np.array(trace.psi), lambda_min=np.array(trace.lambda_min),
        lambda_max=np.array(trace.lambda_max),
        flags=np.array([trace.converged, trace.stagnated, trace.diverged,
                        trace.total_iters, trace.total_outer]),
        rec_int=np.array([[r.k, r.s_bar, r.s_tilde, r.s_actual,
                           -1 if r.break_j is None else r.break_j] for r in recs]).reshape(-1, 5),
        rec_float=np.array([[r.phi, r.break_lhs, r.break_rhs] for r in recs]).reshape(-1, 3),
        rec_thetas=np.array([np.asarray(r.basis_params_used.thetas) for r in recs]),
        first_g=first_g.get("g", np.zeros((0, 0))),
        wall=np.array(dt),
        cfg=np.array(json.dumps(cfg_kwargs)),
    )
    if store_x:
        d["x"] = x
    else:
        d["x_digest"] = np.array([float(np.sum(x)), float(np.linalg.norm(x))])
        d["x_head"] = np.asarray(x[:256]).copy()
    d["final_true"] = np.array(trace.final_true_resid)
    # conds of the first 8 outer loops (ragged -> padded)
    k8 = min(8, len(recs))
    if k8:
        w = max(len(r.cond_used) for r in recs[:k8])
        cm = np.full((k8, w), np.nan)
        for i in range(k8):
            cm[i, : len(recs[i].cond_used)] = recs[i].cond_used
        d["conds8"] = cm
    print(f"    {prob.label} {cfg_kwargs}: outer={trace.total_outer} total={trace.total_iters} "
          f"conv={trace.converged} final={trace.final_true_resid:.3e} ({dt:.2f}s)")
    return d


def problem_arrays(prob):
    a = prob.a
    return dict(n=np.array(a.n), row_ptr=np.asarray(a.row_ptr), col_idx=np.asarray(a.col_idx),
                values=np.asarray(a.values), n_a=np.array(a.n_a), b=prob.b, x0=prob.x0,
                norms=np.array([prob.norm_a, prob.norm_abs_a, prob.kappa_a]))


def gen_solves():
    # BASELINE configs that the reference finishes quickly (c1, c2) -- inputs are
    # regenerated from the seed, so only outputs are stored
    c1 = to_ref(problems.make_problem("c1"))
    save("solve_c1", **run_ref(c1, dict(sigma=8, eps_star=1e-10, basis_kind="newton")))
    c2 = to_ref(problems.make_problem("c2"))
    save("solve_c2_cheb", **run_ref(c2, dict(sigma=10, eps_star=1e-8, basis_kind="chebyshev")))
    save("solve_c2_newton", **run_ref(c2, dict(sigma=10, eps_star=1e-8, basis_kind="newton")))
    # small proxies of c3 / c4 / c5 (same generators, reduced edge)
    c3p = to_ref(problems.make_problem("c3", scale=24))
    save("solve_c3p", **run_ref(c3p, dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev")))
    c5p = to_ref(problems.make_problem("c5", scale=24))
    save("solve_c5p", **run_ref(c5p, dict(sigma=12, eps_star=1e-10, basis_kind="newton")))
    c4p = to_ref(problems.make_problem("c4", scale=12))
    save("solve_c4p", **run_ref(c4p, dict(sigma=10, eps_star=1e-8, basis_kind="newton",
                                           max_outer=400)),
         **{"in_" + k: v for k, v in problem_arrays(c4p).items()})

    # the reference's own acceptance matrices (preconditioned by its load_problem)
    from sstepcg.matio import load_problem
    data = "/root/reference/pkg/data/matrices"
    nos1 = load_problem(os.path.join(data, "nos1.mtx"), label="nos1")
    bus = load_problem(os.path.join(data, "494_bus.mtx"), label="494bus")
    save("problem_nos1", **problem_arrays(nos1))
    save("problem_494bus", **problem_arrays(bus))
    for kind in ("newton", "chebyshev"):
        for strat in ("adaptive", "unit", "kappa-estimate"):
            save(f"solve_nos1_{kind}_{strat}",
                 **run_ref(nos1, dict(sigma=10, eps_star=1e-6, basis_kind=kind, c_strategy=strat)))
        save(f"solve_494bus_s15_{kind}",
             **run_ref(bus, dict(sigma=15, eps_star=1e-6, basis_kind=kind)))
    save("solve_494bus_old", **run_ref(bus, dict(sigma=5, eps_star=1e-6, variant="old",
                                                 basis_kind="monomial", c_strategy="unit")))
    save("solve_494bus_cheb6", **run_ref(bus, dict(sigma=6, eps_star=1e-8, basis_kind="chebyshev")))

    # tests/test_adaptive.py-style dense problems
    p44 = dense_problem(spd_dense(50, 1e4, 44), "spd50")
    for kind in ("newton", "chebyshev"):
        save(f"solve_spd50_{kind}", **run_ref(p44, dict(sigma=6, eps_star=1e-10, basis_kind=kind)),
             **{"in_" + k: v for k, v in problem_arrays(p44).items()})
    p43 = dense_problem(spd_dense(40, 50.0, 43), "spd40")
    for variant in ("old", "improved"):
        save(f"solve_spd40_s1_{variant}",
             **run_ref(p43, dict(sigma=1, eps_star=1e-10, variant=variant, basis_kind="monomial")),
             **{"in_" + k: v for k, v in problem_arrays(p43).items()})
    p45 = dense_problem(spd_dense(40, 1e3, 45), "spd40fb")
    save("solve_spd40_fullbound",
         **run_ref(p45, dict(sigma=4, eps_star=1e-8, basis_kind="newton", c_strategy="full-bound")),
         **{"in_" + k: v for k, v in problem_arrays(p45).items()})
    # HSCG alphas for the sigma = 1 cross-check (classic.py:33-104)
    from sstepcg.classic import hscg_solve
    _, _, co = hscg_solve(p43, 1e-10)
    save("hscg_spd40", alphas=np.array(co.alphas), betas=np.array(co.betas))


# ---------------------------------------------------------------------------
# Fixed s-step CG (sstep.py:79-174), SURVEY.md 8(f) row 1
def sstep_cases():
    """name -> (problem factory, sstep_solve kwargs); explicit `params` are
    given as (kind, s, lo, hi) and built with the reference's params_for."""
    c1 = lambda: to_ref(problems.make_problem("c1"))
    c3p = lambda: to_ref(problems.make_problem("c3", scale=24))
    p44 = dense_problem(spd_dense(50, 1e4, 44), "spd50")
    p43 = dense_problem(spd_dense(40, 50.0, 43), "spd40")
    from sstepcg.matio import load_problem
    data = "/root/reference/pkg/data/matrices"
    bus = load_problem(os.path.join(data, "494_bus.mtx"), label="494bus")
    return {
        "sstep_c1_mono4": (c1, dict(s=4, eps_star=1e-10)),
        "sstep_c1_newton8": (c1, dict(s=8, eps_star=1e-10, basis_kind="newton",
                                      spectral_bounds=(0.004, 8.0))),
        "sstep_c1_mono10": (c1, dict(s=10, eps_star=1e-10, max_outer=60)),
        "sstep_c3p_cheb8": (c3p, dict(s=8, eps_star=1e-10, basis_kind="chebyshev",
                                      spectral_bounds=(0.04, 12.0))),
        "sstep_spd50_newton6": (lambda: p44, dict(s=6, eps_star=1e-10, basis_kind="newton",
                                                  spectral_bounds=(1.0, 1e4))),
        "sstep_spd40_mono1": (lambda: p43, dict(s=1, eps_star=1e-10)),
        "sstep_spd40_mono3": (lambda: p43, dict(s=3, eps_star=1e-10)),
        "sstep_spd40_params5": (lambda: p43, dict(s=5, eps_star=1e-10,
                                                  params=("chebyshev", 5, 1.0, 50.0))),
        "sstep_494bus_mono5": (lambda: bus, dict(s=5, eps_star=1e-6)),
        "sstep_494bus_cheb6": (lambda: bus, dict(s=6, eps_star=1e-8, basis_kind="chebyshev",
                                                 spectral_bounds=(1e-3, 2.0))),
    }


def gen_sstep():
    from sstepcg.sstep import sstep_solve
    orig = ref_basis.gram
    for name, (mk, kw) in sstep_cases().items():
        prob = mk()
        kw = dict(kw)
        spec = kw.get("params")
        if spec is not None:
            kw["params"] = ref_basis.params_for(*spec)
        first = {}

        def spy(y):
            g = orig(y)
            first.setdefault("g", g.copy())
            return g

        ref_basis.gram = spy
        try:
            t0 = time.perf_counter()
            x, tr, co = sstep_solve(prob, **kw)
            dt = time.perf_counter() - t0
        finally:
            ref_basis.gram = orig
        meta = {k: v for k, v in kw.items() if k != "params"}
        if spec is not None:
            meta["params"] = list(spec)
        save(name, alphas=np.array(co.alphas), betas=np.array(co.betas),
             s_schedule=np.array(tr.s_schedule), outer_marks=np.array(tr.outer_marks),
             true_resid=np.array(tr.true_resid), upd_resid=np.array(tr.upd_resid),
             resid_gap=np.array(tr.resid_gap), c_values=np.array(tr.c_values),
             psi=np.array(tr.psi), lambda_min=np.array(tr.lambda_min),
             lambda_max=np.array(tr.lambda_max),
             flags=np.array([tr.converged, tr.stagnated, tr.diverged, tr.total_iters,
                             tr.total_outer]),
             x=x, first_g=first.get("g", np.zeros((0, 0))), wall=np.array(dt),
             cfg=np.array(json.dumps(meta)),
             **({"in_" + k: v for k, v in problem_arrays(prob).items()}
                if name.startswith(("sstep_spd", "sstep_494")) else {}))
        print(f"    {name}: outer={tr.total_outer} total={tr.total_iters} conv={tr.converged} "
              f"stag={tr.stagnated} div={tr.diverged} final={tr.final_true_resid:.3e} ({dt:.2f}s)")


# ---------------------------------------------------------------------------
# Rounding-noise floor of the reference itself: the same solve
# with only the Gram summation order changed.  Counts / s-sequences that move
# under these perturbations cannot be demanded bit-exactly of any other
# implementation; tests/test_gpu_parity.py holds the GPU to this floor.
def _gram_chunked(y):
    y = np.asarray(y, dtype=float)
    g = np.zeros((y.shape[1], y.shape[1]))
    for s0 in range(0, y.shape[0], 512):
        c = y[s0:s0 + 512]
        g += c.T @ c
    il = np.tril_indices(g.shape[0], -1)
    g[il[1], il[0]] = g[il]
    return g


def _gram_reversed(y):
    y = np.ascontiguousarray(np.asarray(y, dtype=float)[::-1])
    g = y.T @ y
    il = np.tril_indices(g.shape[0], -1)
    g[il[1], il[0]] = g[il]
    return g


def _gram_einsum(y):
    y = np.asarray(y, dtype=float)
    g = np.einsum("ij,ik->jk", y, y, optimize=False)
    il = np.tril_indices(g.shape[0], -1)
    g[il[1], il[0]] = g[il]
    return g


def _gram_chunk(size):
    def g(y):
        y = np.asarray(y, dtype=float)
        out = np.zeros((y.shape[1], y.shape[1]))
        for s0 in range(0, y.shape[0], size):
            c = y[s0:s0 + size]
            out += c.T @ c
        il = np.tril_indices(out.shape[0], -1)
        out[il[1], il[0]] = out[il]
        return out
    return g


def _conds_jacobi(g, s_bar):
    """nested_basis_conds with the reference's own cyclic Jacobi instead of LAPACK."""
    g = np.asarray(g, dtype=float)
    conds = np.full(s_bar + 1, np.nan)
    for i in range(1, s_bar + 1):
        cols = list(range(0, i + 1)) + list(range(s_bar + 1, s_bar + 1 + i))
        try:
            w = ref_lacore.sym_eig(g[np.ix_(cols, cols)])
        except ref_lacore.EigenConvergenceError:
            w = np.linalg.eigvalsh(g[np.ix_(cols, cols)])
        conds[i] = ref_lacore._cond_from_eigvals(w)
    return conds


class _NoisyLogNumpy:
    """numpy shim for basis.py whose log() is off by up to 1 ulp (seeded): the
    Leja objective's golden-section maximum is then located differently at the
    ~sqrt(u) level, as with any other libm (CUDA's log vs numpy's SIMD log)."""

    def __init__(self, seed):
        self._rng = np.random.default_rng(seed)

    def __getattr__(self, k):
        return getattr(np, k)

    def log(self, x):
        y = np.log(x)
        k = self._rng.integers(-1, 2, size=np.shape(y))
        return np.where(k == 0, y, np.where(k > 0, np.nextafter(y, np.inf),
                                            np.nextafter(y, -np.inf)))


# (Gram summation order, eigensolver, libm) perturbations of the reference
PERTURBATIONS = {"chunked512": (_gram_chunked, None), "reversed": (_gram_reversed, None),
                 "einsum": (_gram_einsum, None), "chunked64": (_gram_chunk(64), None),
                 "chunked4096": (_gram_chunk(4096), None),
                 "chunked16": (_gram_chunk(16), None), "chunked2": (_gram_chunk(2), None),
                 "jacobi-eig": (None, _conds_jacobi),
                 "leja-log-ulp-1": (None, None, 1), "leja-log-ulp-2": (None, None, 2)}


def solve_cases():
    from sstepcg.matio import load_problem
    data = "/root/reference/pkg/data/matrices"
    nos1 = load_problem(os.path.join(data, "nos1.mtx"), label="nos1")
    bus = load_problem(os.path.join(data, "494_bus.mtx"), label="494bus")
    cases = {
        "solve_c1": (lambda: to_ref(problems.make_problem("c1")),
                     dict(sigma=8, eps_star=1e-10, basis_kind="newton")),
        "solve_c2_cheb": (lambda: to_ref(problems.make_problem("c2")),
                          dict(sigma=10, eps_star=1e-8, basis_kind="chebyshev")),
        "solve_c2_newton": (lambda: to_ref(problems.make_problem("c2")),
                            dict(sigma=10, eps_star=1e-8, basis_kind="newton")),
        "solve_c3p": (lambda: to_ref(problems.make_problem("c3", scale=24)),
                      dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev")),
        "solve_c5p": (lambda: to_ref(problems.make_problem("c5", scale=24)),
                      dict(sigma=12, eps_star=1e-10, basis_kind="newton")),
        "solve_c4p": (lambda: to_ref(problems.make_problem("c4", scale=12)),
                      dict(sigma=10, eps_star=1e-8, basis_kind="newton", max_outer=400)),
        "solve_c4jp": (lambda: to_ref(problems.make_problem("c4j", scale=12)),
                       dict(sigma=10, eps_star=1e-8, basis_kind="newton")),
        # full-size c4j (192^3, 5 outer loops): its third block's nested condition
        # estimates sit at the noise level (~1/sqrt(u)), so the reference's own
        # perturbed runs show how far its decisions are determined
        "full_c4j": (lambda: to_ref(problems.make_problem("c4j")),
                     dict(sigma=10, eps_star=1e-8, basis_kind="newton", max_outer=5)),
        "solve_494bus_old": (lambda: bus, dict(sigma=5, eps_star=1e-6, variant="old",
                                               basis_kind="monomial", c_strategy="unit")),
        "solve_494bus_cheb6": (lambda: bus, dict(sigma=6, eps_star=1e-8, basis_kind="chebyshev")),
    }
    for kind in ("newton", "chebyshev"):
        for strat in ("adaptive", "unit", "kappa-estimate"):
            cases[f"solve_nos1_{kind}_{strat}"] = (
                lambda: nos1, dict(sigma=10, eps_star=1e-6, basis_kind=kind, c_strategy=strat))
        cases[f"solve_494bus_s15_{kind}"] = (lambda: bus, dict(sigma=15, eps_star=1e-6,
                                                               basis_kind=kind))
    p44 = dense_problem(spd_dense(50, 1e4, 44), "spd50")
    for kind in ("newton", "chebyshev"):
        cases[f"solve_spd50_{kind}"] = (lambda: p44, dict(sigma=6, eps_star=1e-10,
                                                          basis_kind=kind))
    p43 = dense_problem(spd_dense(40, 50.0, 43), "spd40")
    for variant in ("old", "improved"):
        cases[f"solve_spd40_s1_{variant}"] = (lambda: p43, dict(
            sigma=1, eps_star=1e-10, variant=variant, basis_kind="monomial"))
    p45 = dense_problem(spd_dense(40, 1e3, 45), "spd40fb")
    cases["solve_spd40_fullbound"] = (lambda: p45, dict(sigma=4, eps_star=1e-8,
                                                        basis_kind="newton",
                                                        c_strategy="full-bound"))
    return cases


def gen_c4j():
    """c4 Jacobi-scaled proxy (the secondary c4 run): the solve
    with its inputs, and its Gram-order noise runs."""
    c4jp = to_ref(problems.make_problem("c4j", scale=12))
    save("solve_c4jp", **run_ref(c4jp, dict(sigma=10, eps_star=1e-8, basis_kind="newton")),
         **{"in_" + k: v for k, v in problem_arrays(c4jp).items()})
    os.environ["NOISE_ONLY"] = "solve_c4jp"
    gen_noise()


def gen_noise():
    orig = ref_basis.gram
    orig_conds = ref_lacore.nested_basis_conds
    only = os.environ.get("NOISE_ONLY")
    for name, (mk, kw) in solve_cases().items():
        if only and only not in name:
            continue
        prob = mk()
        rows, seqs, lmins, lmaxs = [], [], [], []
        keep = os.environ.get("NOISE_PERTS")
        perts = {k: v for k, v in PERTURBATIONS.items() if not keep or k in keep.split(",")}
        for pname, spec in perts.items():
            gfn, cfn = spec[0], spec[1]
            ref_basis.gram = gfn or orig
            ref_lacore.nested_basis_conds = cfn or orig_conds
            if len(spec) > 2:
                ref_basis.np = _NoisyLogNumpy(spec[2])
            try:
                cfg = ref_adaptive.AdaptiveConfig(**kw)
                _, tr, _ = ref_adaptive.adaptive_solve(prob, cfg)
            finally:
                ref_basis.gram = orig
                ref_lacore.nested_basis_conds = orig_conds
                ref_basis.np = np
            rows.append([tr.total_outer, tr.total_iters, tr.converged, tr.final_true_resid])
            sq = np.zeros((8, 2), dtype=np.int64)
            for i, r in enumerate(tr.outer_records[:8]):
                sq[i] = (r.s_tilde, r.s_actual)
            seqs.append(sq)
            lmins.append(tr.lambda_min[-1] if tr.lambda_min else np.nan)
            lmaxs.append(tr.lambda_max[-1] if tr.lambda_max else np.nan)
        save("noise_" + name, counts=np.array(rows, dtype=float), seq8=np.array(seqs),
             lmin_end=np.array(lmins), lmax_end=np.array(lmaxs),
             names=np.array(list(perts)))
        print(f"    noise {name}: outer/total {[(int(r[0]), int(r[1])) for r in rows]}")


def gen_sstep_noise():
    """Noise floor of the reference's fixed s-step CG: the same runs with only
    the Gram summation order changed.  alpha_horizon = the first iteration at
    which any perturbed run's alpha moves by more than 1e-8 relative (parity of
    alpha beyond it cannot be demanded of another implementation)."""
    from sstepcg.sstep import sstep_solve
    orig = ref_basis.gram
    grams = {k: v[0] for k, v in PERTURBATIONS.items() if v[0] is not None}
    for name, (mk, kw) in sstep_cases().items():
        prob = mk()
        kw = dict(kw)
        if kw.get("params") is not None:
            kw["params"] = ref_basis.params_for(*kw["params"])
        _, tr0, co0 = sstep_solve(prob, **kw)
        a0 = np.array(co0.alphas)
        rows, horizon = [], len(a0)
        for pname, gfn in grams.items():
            ref_basis.gram = gfn
            try:
                _, tr, co = sstep_solve(prob, **kw)
            finally:
                ref_basis.gram = orig
            a = np.array(co.alphas)
            m = min(len(a), len(a0))
            bad = np.nonzero(np.abs(a[:m] - a0[:m]) > 1e-8 * np.abs(a0[:m]))[0]
            h = int(bad[0]) if len(bad) else (m if len(a) == len(a0) else m)
            horizon = min(horizon, h)
            rows.append([tr.total_outer, tr.total_iters, tr.converged, tr.stagnated, tr.diverged])
        save("noise_" + name, counts=np.array(rows, dtype=float), alpha_horizon=np.array(horizon),
             names=np.array(list(grams)))
        print(f"    noise {name}: horizon={horizon} outer/total "
              f"{sorted(set((int(r[0]), int(r[1])) for r in rows))}")


# ---------------------------------------------------------------------------
# Hestenes-Stiefel CG (classic.py:33-104), SURVEY.md 8(f) row 2
def hscg_cases():
    c1 = lambda: to_ref(problems.make_problem("c1"))
    c3p = lambda: to_ref(problems.make_problem("c3", scale=24))
    p44 = dense_problem(spd_dense(50, 1e4, 44), "spd50")
    p43 = dense_problem(spd_dense(40, 50.0, 43), "spd40")
    from sstepcg.matio import load_problem
    data = "/root/reference/pkg/data/matrices"
    bus = load_problem(os.path.join(data, "494_bus.mtx"), label="494bus")
    return {
        "hscg_c1": (c1, dict(eps_star=1e-10)),
        "hscg_c1_cap50": (c1, dict(eps_star=1e-10, max_iters=50)),
        "hscg_c3p": (c3p, dict(eps_star=1e-10)),
        "hscg_spd40": (lambda: p43, dict(eps_star=1e-10)),
        "hscg_spd50": (lambda: p44, dict(eps_star=1e-12)),
        "hscg_494bus": (lambda: bus, dict(eps_star=1e-8)),
    }


class _DotShim:
    """numpy stand-in for classic.py whose dot sums in chunks (another order)."""

    def __init__(self, chunk):
        self.chunk = chunk

    def dot(self, a, b):
        a, b = np.asarray(a), np.asarray(b)
        return float(sum(np.dot(a[i:i + self.chunk], b[i:i + self.chunk])
                         for i in range(0, len(a), self.chunk)))

    def __getattr__(self, name):
        return getattr(np, name)


def gen_hscg():
    from sstepcg import classic as ref_classic
    for name, (mk, kw) in hscg_cases().items():
        prob = mk()
        t0 = time.perf_counter()
        x, tr, co = ref_classic.hscg_solve(prob, **kw)
        dt = time.perf_counter() - t0
        rows = []
        a0 = np.array(co.alphas)
        horizon = len(a0)
        for chunk in (7, 64, 1000):
            ref_classic.np = _DotShim(chunk)
            try:
                _, tq, cq = ref_classic.hscg_solve(prob, **kw)
            finally:
                ref_classic.np = np
            aq = np.array(cq.alphas)
            m = min(len(aq), len(a0))
            bad = np.nonzero(np.abs(aq[:m] - a0[:m]) > 1e-8 * np.abs(a0[:m]))[0]
            horizon = min(horizon, int(bad[0]) if len(bad) else m)
            rows.append([tq.total_iters, tq.converged, tq.stagnated, tq.diverged])
        save(name, alphas=a0, betas=np.array(co.betas), true_resid=np.array(tr.true_resid),
             upd_resid=np.array(tr.upd_resid), resid_gap=np.array(tr.resid_gap),
             c_values=np.array(tr.c_values), psi=np.array(tr.psi),
             lambda_min=np.array(tr.lambda_min), lambda_max=np.array(tr.lambda_max),
             flags=np.array([tr.converged, tr.stagnated, tr.diverged, tr.total_iters,
                             tr.total_outer]),
             x=x, wall=np.array(dt), cfg=np.array(json.dumps(kw)),
             noise_counts=np.array(rows, dtype=float), alpha_horizon=np.array(horizon),
             **({"in_" + k: v for k, v in problem_arrays(prob).items()}
                if name.startswith(("hscg_spd", "hscg_494")) else {}))
        print(f"    {name}: iters={tr.total_iters} conv={tr.converged} stag={tr.stagnated} "
              f"div={tr.diverged} final={tr.final_true_resid:.3e} horizon={horizon} "
              f"noise iters {sorted(set(int(r[0]) for r in rows))} ({dt:.2f}s)")


# ---------------------------------------------------------------------------
# Problem setup (matio.py:104-307): synthetic Matrix
# Market files written here, parsed / scaled / normed by the reference
MM_DIR = os.path.join(OUT, "mm")


def _write_mm(path, n, rows, cols, vals, sym="symmetric", field="real", comments=True,
              fmt="{:.17g}"):
    lines = [f"%%MatrixMarket matrix coordinate {field} {sym}"]
    if comments:
        lines += ["% synthetic test matrix (oracle/make_golden.py gen_matio)", "%", ""]
    lines.append(f"{n} {n} {len(vals)}")
    for r, c, v in zip(rows, cols, vals):
        lines.append(f"{r + 1} {c + 1} " + (str(int(v)) if field == "integer" else fmt.format(v)))
    text = "\n".join(lines) + "\n"
    if path.endswith(".gz"):
        import gzip
        with gzip.open(path, "wt") as f:
            f.write(text)
    else:
        with open(path, "w") as f:
            f.write(text)


def gen_matio():
    from scipy import sparse as sp
    from sstepcg import matio as ref_matio
    os.makedirs(MM_DIR, exist_ok=True)
    rng = np.random.default_rng(9001)
    files = {}
    # 2-D Poisson 48x48 (n > 2000: shifted power iteration), lower triangle, with comments
    t = sp.diags([-np.ones(47), 2 * np.ones(48), -np.ones(47)], [-1, 0, 1])
    lap = (sp.kron(sp.identity(48), t) + sp.kron(t, sp.identity(48))).tocoo()
    low = lap.row >= lap.col
    files["poisson48_sym.mtx"] = (2304, lap.row[low], lap.col[low], lap.data[low], "symmetric", "real")
    # random SPD, general format (both triangles), shuffled entry order
    m = sp.random(300, 300, density=0.02, random_state=5)
    m = (m + m.T + sp.identity(300) * 8.0).tocoo()
    perm = rng.permutation(m.nnz)
    files["rand300_gen.mtx"] = (300, m.row[perm], m.col[perm], m.data[perm], "general", "real")
    # integer field, with a duplicated diagonal entry (summed)
    r = np.array([0, 1, 1, 2, 2, 0, 3, 3])
    c = np.array([0, 0, 1, 1, 2, 0, 2, 3])
    v = np.array([4.0, -1.0, 5.0, -2.0, 6.0, 3.0, -1.0, 7.0])
    files["int4_dup.mtx"] = (4, r, c, v, "symmetric", "integer")
    # gzipped, values with many digits
    d = sp.random(120, 120, density=0.05, random_state=7)
    d = (d + d.T + sp.identity(120) * 3.5).tocoo()
    lo = d.row >= d.col
    files["rand120_sym.mtx.gz"] = (120, d.row[lo], d.col[lo], d.data[lo] * np.pi, "symmetric", "real")
    out = {}
    for k, (name, (n, rr, cc, vv, sym, fld)) in enumerate(files.items()):
        path = os.path.join(MM_DIR, name)
        _write_mm(path, n, rr, cc, vv, sym, fld)
        a = ref_matio.read_matrix_market(path)
        ah, dinv = ref_matio.jacobi_precondition(a)
        est = ref_matio.estimate_operator_norms(ah)
        out[f"f{k}_name"] = np.array(name)
        out[f"f{k}_row_ptr"] = a.row_ptr
        out[f"f{k}_col_idx"] = a.col_idx
        out[f"f{k}_values"] = a.values
        out[f"f{k}_jvalues"] = ah.values
        out[f"f{k}_dinv"] = dinv
        out[f"f{k}_norms"] = np.array([est.norm_a, est.norm_abs_a, est.kappa_a, est.lambda_min,
                                       est.iters_used, est.converged])
        print(f"    {name}: n={a.n} nnz={a.nnz} norms {est.norm_a:.6g} {est.norm_abs_a:.6g} "
              f"kappa {est.kappa_a:.6g} iters {est.iters_used}")
    out["nfiles"] = np.array(len(files))
    save("matio", **out)


def gen_grid():
    """The reference's run_grid (harness.py:103-154) on a synthetic MM file:
    rows and summary tables for tests/test_gpu_harness.py."""
    import tempfile
    from sstepcg import harness as ref_harness
    spec = ref_harness.ExperimentSpec(
        matrices=[(os.path.join(MM_DIR, "rand300_gen.mtx"), "rand300")], s_values=[4, 8],
        eps_modes=["hscg-attainable", 1e-8], basis_kinds=["newton", "chebyshev"],
        c_strategies=["adaptive"])
    with tempfile.TemporaryDirectory() as tmp:
        rows = ref_harness.run_grid(spec, tmp)
        md = ref_harness.emit_summary_table(rows, "markdown", os.path.join(tmp, "t.md"))
        table = open(md).read()
    save("grid_rand300",
         keys=np.array([f"{r.algorithm}|{r.basis}|{r.c_strategy}|{r.s}" for r in rows]),
         eps=np.array([r.eps_star for r in rows]), outcome=np.array([r.outcome for r in rows]),
         iters=np.array([r.total_iters for r in rows]), outer=np.array([r.total_outer for r in rows]),
         cell=np.array([r.cell for r in rows]), table=np.array(table))
    for r in rows:
        print(f"    {r.algorithm:18s} {r.basis:9s} s={r.s:2d} eps={r.eps_star:.2e} {r.outcome:10s} "
              f"{r.cell}")


def gen_nos1_counts():
    """The paper's nos1 rows on the reference: HSCG and fixed
    s = 10 at 1e-6, plus the fixed-s run under every Gram-order perturbation
    (its count moves by 3x: a degree-10 monomial basis at nos1's conditioning)."""
    from sstepcg.classic import hscg_solve
    from sstepcg.matio import load_problem
    from sstepcg.sstep import sstep_solve
    prob = load_problem("/root/reference/pkg/data/matrices/nos1.mtx", label="nos1")
    _, th, _ = hscg_solve(prob, 1e-6)
    orig = ref_basis.gram
    rows = []
    for name, spec in [("reference", (None,))] + [(k, v) for k, v in PERTURBATIONS.items()
                                                  if v[0] is not None]:
        ref_basis.gram = spec[0] or orig
        try:
            _, tr, _ = sstep_solve(prob, 10, 1e-6)
        finally:
            ref_basis.gram = orig
        rows.append([tr.total_outer, tr.total_iters, tr.converged])
    save("nos1_counts", hscg=np.array([th.total_iters, th.converged]),
         sstep10=np.array(rows, dtype=float),
         names=np.array(["reference"] + [k for k, v in PERTURBATIONS.items() if v[0] is not None]))
    print(f"    hscg {th.total_iters}; sstep s=10 outer/total {[(int(r[0]), int(r[1])) for r in rows]}")


def _full_record(prob, cfg_kwargs, name, keep_outer=5):
    """Run the reference's adaptive_solve (as shipped, diagnostics on) on a
    BASELINE config at its full size and keep what the -m gpu tests compare:
    counts, flags, the per-outer (s_bar, s_tilde, s_actual) records, the first
    Gram, alphas / betas / Ritz values of every iteration (small: ~1k iters),
    the final true residual and a checksum of x (x itself is 134 MB at 256^3).
    The wall time of the reference run is kept too (the as-shipped CPU figure
    on this 8-core container; bench.py re-times the port on the GPU host)."""
    d = run_ref(prob, cfg_kwargs, store_x=False)
    d["keep_outer"] = np.array(keep_outer)
    d["n"] = np.array(prob.a.n)
    d["nnz"] = np.array(int(np.asarray(prob.a.row_ptr)[-1]))
    d["threads"] = np.array(os.cpu_count())
    save(name, **d)


def gen_full():
    """Full-size reference goldens (pin parity at the headline size).

    c3 128^3 Chebyshev, full run; c4 192^3 Newton and c4j (Jacobi-scaled),
    max_outer = 5; c5w 256^3 sigma = 12 Newton, full run (~20-30 min here).
    Selected with FULL=c3,c4,c4j,c5w (default all)."""
    which = os.environ.get("FULL", "c3,c4,c4j,c5w").split(",")
    jobs = {
        "c3": ("c3", dict(sigma=10, eps_star=1e-10, basis_kind="chebyshev")),
        "c4": ("c4", dict(sigma=10, eps_star=1e-8, basis_kind="newton", max_outer=5)),
        "c4j": ("c4j", dict(sigma=10, eps_star=1e-8, basis_kind="newton", max_outer=5)),
        "c5w": ("c5w", dict(sigma=12, eps_star=1e-10, basis_kind="newton")),
        "c5w2": ("c5w2", dict(sigma=12, eps_star=1e-10, basis_kind="newton", max_outer=5)),
    }
    for key in which:
        cname, kw = jobs[key]
        t0 = time.perf_counter()
        if cname == "c5w2":
            prob = problems.make_problem("c5w", world=2)
        else:
            prob = problems.make_problem(cname)
        print(f"  built {cname} n={prob.a.n} in {time.perf_counter() - t0:.1f}s", flush=True)
        _full_record(to_ref(prob), kw, f"full_{key}")
        del prob


def first_block_cases():
    """x0 = 0 problems (the first block's P and R columns are bitwise
    duplicates: p = r): 2-D / 3-D Poisson with random x*, random dense SPD
    spectra, Strakos diagonals -- with Newton, Chebyshev and monomial bases."""
    cases = []
    for seed in range(6):
        cases.append((f"p2d_{seed}", lambda s=seed: to_ref(problems.poisson2d(24 + 4 * s, seed=s)),
                      dict(sigma=8, eps_star=1e-10, basis_kind="newton")))
        cases.append((f"p3d_{seed}", lambda s=seed: to_ref(problems.poisson3d(10 + s, seed=s)),
                      dict(sigma=10, eps_star=1e-10, basis_kind=("chebyshev" if seed % 2 else "newton"))))
        kap = [1e2, 1e4, 1e6, 1e3, 1e5, 3e4][seed]
        cases.append((f"spd_{seed}", lambda s=seed, k=kap: dense_problem(spd_dense(60, k, 100 + s),
                                                                          f"spd{s}"),
                      dict(sigma=6 + seed % 3, eps_star=1e-9,
                           basis_kind=("newton", "chebyshev", "monomial")[seed % 3])))
        cases.append((f"strakos_{seed}", lambda s=seed: to_ref(problems.strakos(400 + 100 * s, seed=s)),
                      dict(sigma=10, eps_star=1e-8, basis_kind=("chebyshev" if seed % 2 else "newton"))))
    return cases


def _first_blocks_run():
    """(in a subprocess with OPENBLAS_CORETYPE set) the reference's first three
    outer loops of every first-block case: (s~, s_actual) and the first conds."""
    out = {}
    for name, mk, kw in first_block_cases():
        prob = mk()
        cfg = ref_adaptive.AdaptiveConfig(max_outer=3, **kw)
        _, tr, co = ref_adaptive.adaptive_solve(prob, cfg)
        out[name] = dict(seq=[[r.s_tilde, r.s_actual] for r in tr.outer_records],
                         conds=[float(v) for v in tr.outer_records[0].cond_used],
                         alphas=[float(a) for a in co.alphas[:6]])
    print("JSON" + json.dumps(out))


def gen_first_blocks():
    """The first-block decisions (p = r, duplicated Gram columns: the noise-level
    condition estimates DESIGN.md 5 discusses) of the reference under two
    OpenBLAS kernel choices (OPENBLAS_CORETYPE Haswell / SkylakeX): the
    decisions the GPU's calibrated noise floor must reproduce."""
    import subprocess
    res = {}
    for core in ("Haswell", "SkylakeX"):
        env = dict(os.environ, OPENBLAS_CORETYPE=core, PYTHONPATH=REF_SRC)
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "_first_blocks_run"],
                           env=env, capture_output=True, text=True, check=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("JSON")][-1]
        res[core] = json.loads(line[4:])
    cases = first_block_cases()
    names = [n for n, _, _ in cases]
    out = {"names": np.array(names), "cores": np.array(list(res))}
    for name, mk, kw in cases:  # dense SPD inputs are stored (their QR is BLAS-dependent)
        if name.startswith("spd_"):
            out.update({f"{name}_in_" + k: v for k, v in problem_arrays(mk()).items()})
    for ci, core in enumerate(res):
        for name in names:
            d = res[core][name]
            seq = np.full((3, 2), -1, dtype=np.int64)
            seq[:len(d["seq"])] = d["seq"]
            out[f"{name}_{core}_seq"] = seq
            out[f"{name}_{core}_conds"] = np.array(d["conds"])
            out[f"{name}_{core}_alphas"] = np.array(d["alphas"])
    save("first_blocks", **out)
    same = sum(np.array_equal(out[f"{n}_Haswell_seq"], out[f"{n}_SkylakeX_seq"]) for n in names)
    print(f"    {len(names)} cases; the two kernel choices agree on {same}")


def main():
    if sys.argv[1:] == ["_first_blocks_run"]:
        _first_blocks_run()
        return
    os.makedirs(OUT, exist_ok=True)
    print("reference:", sstepcg.__file__)
    which = sys.argv[1:] or ["leja", "params", "ritz", "gram_conds", "blocks", "solves"]
    for w in which:
        print(w)
        globals()["gen_" + w]()
    meta = dict(numpy=np.__version__, generated_by="oracle/make_golden.py",
                reference="/root/reference/pkg/src/sstepcg")
    import scipy
    meta["scipy"] = scipy.__version__
    with open(os.path.join(OUT, "META.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
