"""Pin the CPU oracle (oracle/sscg_oracle.py) to the REFERENCE's own outputs.

tests/golden/*.npz were produced by oracle/make_golden.py running the reference
package (/root/reference/pkg/src/sstepcg) in the build container.  Every oracle
function is checked against them; on the generating host the match is bit for
bit (same numpy / scipy / OpenBLAS), elsewhere to rounding noise.
"""

import numpy as np
import pytest

from conftest import cfg_of, golden, golden_problem, problem_from_arrays
from oracle import sscg_oracle as O
from paper_1908_04081_b200 import problems


def test_leja_points_match_reference():
    d = golden("leja")
    for i in range(len(d["lo"])):
        c = int(d["count"][i])
        got = O.leja_sequence(float(d["lo"][i]), float(d["hi"][i]), c, int(d["grid"][i]))
        ref = d["points"][i, :c]
        span = float(d["hi"][i] - d["lo"][i])
        assert np.max(np.abs(got - ref)) <= 1e-12 * span, i


def test_leja_known_answers():
    # test_basis.py:56-60, :68-76
    np.testing.assert_array_equal(O.leja_sequence(1.0, 3.0, 2), [3.0, 1.0])
    p = O.leja_sequence(0.0, 4.0, 4, 10**5)
    assert p[0] == 4.0 and p[1] == 0.0
    assert abs(p[2] - 2.0) <= 4.0 / 10**5
    assert abs(p[3] - (2.0 - 2.0 / np.sqrt(3))) <= 2 * 4.0 / 10**5
    with pytest.raises(O.OracleParamError):
        O.leja_sequence(2.0, 1.0, 3)


def test_params_and_change_of_basis_match_reference():
    d = golden("params")
    kinds = ["monomial", "newton", "chebyshev"]
    for i in range(int(d["ncases"])):
        meta = d[f"c{i}_meta"]
        kind, s, lo, hi = kinds[int(meta[0])], int(meta[1]), float(meta[2]), float(meta[3])
        p = O.params_select(kind, s, lo, hi)
        np.testing.assert_allclose(p.thetas, d[f"c{i}_thetas"], rtol=1e-13, atol=0)
        np.testing.assert_array_equal(p.gammas, d[f"c{i}_gammas"])
        np.testing.assert_array_equal(p.mus, d[f"c{i}_mus"])
        np.testing.assert_allclose(O.change_of_basis(s, p), d[f"c{i}_bmat"], rtol=1e-13, atol=0)
    # Chebyshev KATs (test_basis.py:97-107): mu = w/8 as coded
    p = O.params_chebyshev(1.0, 3.0, 3)
    np.testing.assert_array_equal(p.thetas, [2, 2, 2])
    np.testing.assert_array_equal(p.gammas, [2, 1, 1])
    np.testing.assert_array_equal(p.mus, [0.25, 0.25])
    assert O.params_select("newton", 4, 2.0, 2.0).kind == "monomial"


def test_ritz_matches_reference_bitwise():
    d = golden("ritz")
    for i in range(int(d["nseq"])):
        rz = O.RitzTracker()
        rec = []
        for a, b in zip(d[f"s{i}_alpha"], d[f"s{i}_beta"]):
            rz.absorb(float(a), float(b))
            rec.append([rz.lam_min, rz.lam_max, rz.psi, rz.c, rz.xi(), rz.count])
        np.testing.assert_array_equal(np.array(rec), d[f"s{i}_rec"])
    fb = d["full_bound"]
    assert O.full_bound(1, 1, 1.0, 1.0, 1.0) == fb[0]
    assert O.full_bound(7, 27, 1.3, 2.5, 1e4) == fb[1]


def test_gram_conds_select_match_reference():
    d = golden("gram_conds")
    for t in range(int(d["ncases"])):
        y, g = d[f"t{t}_y"], d[f"t{t}_g"]
        np.testing.assert_array_equal(O.gram_matrix(y), g)
        s_bar, c, eps_star, rn, st = d[f"t{t}_sel"]
        s_bar = int(s_bar)
        np.testing.assert_array_equal(O.nested_conds(g, s_bar), d[f"t{t}_conds"])
        got, _ = O.choose_s(g, s_bar, c, O.UNIT, eps_star, rn)
        assert got == int(st)
    for t in range(6):
        np.testing.assert_allclose(O.jacobi_eigvals(d[f"j{t}_m"]), d[f"j{t}_w"], rtol=1e-13,
                                   atol=1e-13)


def test_krylov_blocks_match_reference():
    d = golden("blocks")
    for i in range(int(d["ncases"])):
        n = len(d[f"b{i}_p"])
        mat = O.csr_of(n, d[f"b{i}_rowptr"], d[f"b{i}_col"], d[f"b{i}_val"])
        s = int(d[f"b{i}_s"])
        prm = O.Params("x", d[f"b{i}_thetas"], d[f"b{i}_gammas"], d[f"b{i}_mus"])
        y = np.hstack([O.krylov_columns(mat, d[f"b{i}_p"], s, prm),
                       O.krylov_columns(mat, d[f"b{i}_r"], s - 1, prm)])
        np.testing.assert_array_equal(y, d[f"b{i}_y"])
        np.testing.assert_array_equal(O.gram_matrix(y), d[f"b{i}_g"])


def _check_solve(ref, x, tr, alphas, betas, exact=True):
    flags = ref["flags"]
    assert [tr.converged, tr.stagnated, tr.diverged] == [bool(v) for v in flags[:3]]
    assert tr.total_iters == int(flags[3]) and tr.total_outer == int(flags[4])
    np.testing.assert_array_equal(tr.s_schedule, ref["s_schedule"])
    np.testing.assert_array_equal(tr.outer_marks, ref["outer_marks"])
    ri = np.array([[r.k, r.s_bar, r.s_tilde, r.s_actual, -1 if r.break_j is None else r.break_j]
                   for r in tr.outer_records]).reshape(-1, 5)
    np.testing.assert_array_equal(ri, ref["rec_int"])
    cmp = np.testing.assert_array_equal if exact else (
        lambda a, b: np.testing.assert_allclose(a, b, rtol=1e-10, atol=0))
    cmp(np.array(alphas), ref["alphas"])
    cmp(np.array(betas), ref["betas"])
    for key in ("true_resid", "upd_resid", "resid_gap", "c_values", "psi", "lambda_min",
                "lambda_max"):
        cmp(np.array(getattr(tr, key)), ref[key])
    if "x" in ref:
        cmp(x, ref["x"])
    if ref["first_g"].size:
        cmp(tr.first_gram, ref["first_g"])


@pytest.mark.parametrize("name,gen", [
    ("solve_c1", ("c1", None)),
    ("solve_c2_cheb", ("c2", None)),
    ("solve_c3p", ("c3", 24)),
    ("solve_c5p", ("c5", 24)),
])
def test_solves_on_baseline_configs_match_reference(name, gen):
    ref = golden(name)
    prob = problems.make_problem(gen[0], scale=gen[1])
    x, tr, al, be = O.solve_problem(prob, O.OracleConfig(**cfg_of(ref)))
    _check_solve(ref, x, tr, al, be)


@pytest.mark.slow
def test_solve_c2_newton_matches_reference():
    ref = golden("solve_c2_newton")
    prob = problems.make_problem("c2")
    x, tr, al, be = O.solve_problem(prob, O.OracleConfig(**cfg_of(ref)))
    _check_solve(ref, x, tr, al, be)


def test_solve_c4_proxy_matches_reference():
    ref = golden("solve_c4p")
    prob = problem_from_arrays(ref, "in_")
    gen = problems.make_problem("c4", scale=12)
    np.testing.assert_array_equal(gen.a.values, prob.a.values)  # generator is pinned too
    np.testing.assert_array_equal(gen.b, prob.b)
    x, tr, al, be = O.solve_problem(prob, O.OracleConfig(**cfg_of(ref)))
    _check_solve(ref, x, tr, al, be)


def test_solve_c4_jacobi_proxy_matches_reference():
    ref = golden("solve_c4jp")
    prob = problem_from_arrays(ref, "in_")
    gen = problems.make_problem("c4j", scale=12)
    np.testing.assert_array_equal(gen.a.values, prob.a.values)  # scaling pinned too
    np.testing.assert_array_equal(gen.b, prob.b)
    x, tr, al, be = O.solve_problem(prob, O.OracleConfig(**cfg_of(ref)))
    _check_solve(ref, x, tr, al, be)


@pytest.mark.parametrize("kind", ["newton", "chebyshev"])
@pytest.mark.parametrize("strat", ["adaptive", "unit", "kappa-estimate"])
def test_nos1_acceptance_runs_match_reference(kind, strat):
    prob = golden_problem("problem_nos1")
    ref = golden(f"solve_nos1_{kind}_{strat}")
    x, tr, al, be = O.solve_problem(prob, O.OracleConfig(**cfg_of(ref)))
    _check_solve(ref, x, tr, al, be)


@pytest.mark.parametrize("name", ["solve_494bus_s15_newton", "solve_494bus_s15_chebyshev",
                                  "solve_494bus_old", "solve_494bus_cheb6"])
def test_494bus_runs_match_reference(name):
    prob = golden_problem("problem_494bus")
    ref = golden(name)
    x, tr, al, be = O.solve_problem(prob, O.OracleConfig(**cfg_of(ref)))
    _check_solve(ref, x, tr, al, be)


@pytest.mark.parametrize("name", ["solve_spd50_newton", "solve_spd50_chebyshev",
                                  "solve_spd40_s1_old", "solve_spd40_s1_improved",
                                  "solve_spd40_fullbound"])
def test_dense_problem_runs_match_reference(name):
    ref = golden(name)
    prob = problem_from_arrays(ref, "in_")
    x, tr, al, be = O.solve_problem(prob, O.OracleConfig(**cfg_of(ref)))
    _check_solve(ref, x, tr, al, be)


def test_fast_trace_mode_keeps_every_decision():
    """diagnostics=False (the 'fast' trace) changes no decision, coefficient or x."""
    ref = golden("solve_c1")
    prob = problems.make_problem("c1")
    cfg = O.OracleConfig(**cfg_of(ref))
    x, tr, al, be = O.solve_problem(prob, cfg, diagnostics=False)
    np.testing.assert_array_equal(x, ref["x"])
    np.testing.assert_array_equal(al, ref["alphas"])
    np.testing.assert_array_equal(tr.s_schedule, ref["s_schedule"])
    ends = np.array(tr.outer_marks[1:] + [tr.total_iters]) - 1
    # block-final true residuals equal the reference's per-iteration ones
    np.testing.assert_array_equal(np.array(tr.true_resid)[ends], ref["true_resid"][ends])


def test_sigma_one_reduces_to_hscg():
    """test_adaptive.py:76-87 on the oracle: sigma=1 monomial == HSCG alphas."""
    ref = golden("hscg_spd40")
    prob = problem_from_arrays(golden("solve_spd40_s1_old"), "in_")
    a = prob.a
    _, al, be, conv = O.hscg(a.n, a.row_ptr, a.col_idx, a.values, prob.b, prob.x0, 1e-10)
    np.testing.assert_array_equal(al, ref["alphas"])
    for variant in ("old", "improved"):
        _, tr, al2, _ = O.solve_problem(prob, O.OracleConfig(
            sigma=1, eps_star=1e-10, variant=variant, basis_kind="monomial"))
        m = min(20, len(al2), len(al))
        np.testing.assert_allclose(al2[:m], al[:m], rtol=1e-8)


# ---- fixed s-step CG (sstep.py:79-174), SURVEY.md 8(f) row 1 -----------------
SSTEP_CASES = ["sstep_c1_mono4", "sstep_c1_newton8", "sstep_c1_mono10", "sstep_c3p_cheb8",
               "sstep_spd50_newton6", "sstep_spd40_mono1", "sstep_spd40_mono3",
               "sstep_spd40_params5", "sstep_494bus_mono5", "sstep_494bus_cheb6"]


def sstep_problem(name, ref):
    if name.startswith("sstep_c1"):
        return problems.make_problem("c1")
    if name.startswith("sstep_c3p"):
        return problems.make_problem("c3", scale=24)
    return problem_from_arrays(ref, "in_")


def sstep_kwargs(ref):
    kw = cfg_of(ref)
    if "params" in kw:
        kind, s, lo, hi = kw.pop("params")
        kw["params"] = O.params_select(kind, int(s), lo, hi)
    if "spectral_bounds" in kw:
        kw["spectral_bounds"] = tuple(kw["spectral_bounds"])
    return kw


@pytest.mark.parametrize("name", SSTEP_CASES)
def test_fixed_sstep_matches_reference(name):
    ref = golden(name)
    prob = sstep_problem(name, ref)
    a = prob.a
    x, tr, al, be = O.sstep(a.n, a.row_ptr, a.col_idx, a.values, prob.b, prob.x0,
                            **sstep_kwargs(ref))
    flags = ref["flags"]
    assert [tr.converged, tr.stagnated, tr.diverged] == [bool(v) for v in flags[:3]]
    assert tr.total_iters == int(flags[3]) and tr.total_outer == int(flags[4])
    np.testing.assert_array_equal(tr.s_schedule, ref["s_schedule"])
    np.testing.assert_array_equal(tr.outer_marks, ref["outer_marks"])
    np.testing.assert_array_equal(al, ref["alphas"])
    np.testing.assert_array_equal(be, ref["betas"])
    for key in ("true_resid", "upd_resid", "resid_gap", "c_values", "psi", "lambda_min",
                "lambda_max"):
        np.testing.assert_array_equal(np.array(getattr(tr, key)), ref[key])
    np.testing.assert_array_equal(x, ref["x"])
    np.testing.assert_array_equal(tr.first_gram, ref["first_g"])


def test_fixed_sstep_validation():
    prob = problems.make_problem("c1", scale=8)
    a = prob.a
    with pytest.raises(ValueError):
        O.sstep(a.n, a.row_ptr, a.col_idx, a.values, prob.b, prob.x0, 0, 1e-8)
    with pytest.raises(O.OracleParamError):
        O.sstep(a.n, a.row_ptr, a.col_idx, a.values, prob.b, prob.x0, 5, 1e-8,
                params=O.params_monomial(3))


# ---- Hestenes-Stiefel CG (classic.py:33-104), SURVEY.md 8(f) row 2 -----------
HSCG_CASES = ["hscg_c1", "hscg_c1_cap50", "hscg_c3p", "hscg_spd40", "hscg_spd50", "hscg_494bus"]


def hscg_problem(name, ref):
    if name.startswith("hscg_c1"):
        return problems.make_problem("c1")
    if name.startswith("hscg_c3p"):
        return problems.make_problem("c3", scale=24)
    return problem_from_arrays(ref, "in_")


@pytest.mark.parametrize("name", HSCG_CASES)
def test_hscg_matches_reference(name):
    ref = golden(name)
    prob = hscg_problem(name, ref)
    a = prob.a
    x, tr, al, be = O.hscg_trace(a.n, a.row_ptr, a.col_idx, a.values, prob.b, prob.x0,
                                 **cfg_of(ref))
    flags = ref["flags"]
    assert [tr.converged, tr.stagnated, tr.diverged] == [bool(v) for v in flags[:3]]
    assert tr.total_iters == int(flags[3]) and tr.total_outer == int(flags[4])
    np.testing.assert_array_equal(al, ref["alphas"])
    np.testing.assert_array_equal(be, ref["betas"])
    for key in ("true_resid", "upd_resid", "resid_gap", "c_values", "psi", "lambda_min",
                "lambda_max"):
        np.testing.assert_array_equal(np.array(getattr(tr, key)), ref[key])
    np.testing.assert_array_equal(x, ref["x"])
