"""CPU tier: the C-ABI library builds, loads and exports every symbol in
include/sscg.h; the ctypes mirror matches the C layout; host-side logic
(problem generators, config validation, trace assembly) is right.  No compute
call reaches the GPU here."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import ROOT
from paper_1908_04081_b200 import _lib as L
from paper_1908_04081_b200 import build, problems
from paper_1908_04081_b200.adaptive import LogBuffers, build_trace, make_config
from paper_1908_04081_b200.types import AdaptiveConfig

HEADER = os.path.join(ROOT, "include", "sscg.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return L.load()


def header_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sscg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol(lib):
    names = header_functions()
    assert len(names) >= 20
    assert set(names) == set(L.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (sscg_\w+)", out))
    assert set(names) <= exported


def test_abi_version_and_constants(lib):
    assert lib.sscg_abi_version() == L.ABI_VERSION
    txt = open(HEADER).read()
    assert f"#define SSCG_ABI_VERSION {L.ABI_VERSION}" in txt
    assert f"#define SSCG_MAX_SIGMA {L.MAX_SIGMA}" in txt
    for name, val in [("SSCG_IT_N", L.IT_N), ("SSCG_REC_NI", L.REC_NI),
                      ("SSCG_RECD_ND", L.RECD_ND), ("SSCG_EBREAKDOWN", L.EBREAKDOWN),
                      ("SSCG_DIVERGED", L.DIVERGED), ("SSCG_BASIS_CHEBYSHEV", 2),
                      ("SSCG_C_FULLBOUND", 3), ("SSCG_EXHAUSTED", L.EXHAUSTED),
                      ("SSCG_SOLVER_FIXED", L.SOLVER_FIXED)]:
        assert re.search(rf"#define {name} {val}\b", txt), name
    for name, val in [("SSCG_LOG_CAP_OUTER", "(1 << 18)"), ("SSCG_LOG_CAP_ITERS", "(1 << 21)")]:
        assert f"#define {name} {val}" in txt and eval(val) == getattr(L, name[5:])
    for name, val in []:
        assert re.search(rf"#define {name} {val}\b", txt), name


def test_struct_layouts_match_c(tmp_path):
    src = tmp_path / "probe.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "sscg.h"\n'
                   "int main(void){printf(\"%zu %zu %zu %zu %zu\\n\", sizeof(sscg_config),"
                   " sizeof(sscg_logs), offsetof(sscg_config, eps_star),"
                   " offsetof(sscg_logs, status), offsetof(sscg_logs, device_ms));return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                           check=True).stdout.split()]
    assert vals == [ctypes.sizeof(L.SscgConfig), ctypes.sizeof(L.SscgLogs),
                    L.SscgConfig.eps_star.offset, L.SscgLogs.status.offset,
                    L.SscgLogs.device_ms.offset]


def test_error_paths_without_gpu(lib):
    """Argument validation answers before touching a device; with no device the
    plan refuses (no CPU fallback)."""
    h = ctypes.c_void_p()
    rp = np.array([0, 1], dtype=np.int64)
    ci = np.array([0], dtype=np.int32)
    va = np.array([1.0])
    rc = lib.sscg_plan_create(ctypes.byref(h), 0, 0, 1, rp.ctypes.data_as(
        ctypes.POINTER(ctypes.c_int64)), L.iptr(ci), L.dptr(va))
    assert rc == L.EINVAL
    assert b"n must be" in lib.sscg_last_error()
    rc = lib.sscg_leja_points(0, 2.0, 1.0, 3, 100, L.dptr(np.zeros(3)))
    assert rc == L.EPARAM
    if L.device_count() == 0:
        rc = lib.sscg_plan_create(ctypes.byref(h), 0, 1, 1, rp.ctypes.data_as(
            ctypes.POINTER(ctypes.c_int64)), L.iptr(ci), L.dptr(va))
        assert rc in (L.ENODEV, L.ECUDA)
        with pytest.raises(L.SscgError):
            L.require_device(0)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1908_04081_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "import sstepcg" not in txt and "from sstepcg" not in txt, f


# ---- problem generators -----------------------------------
def test_stencil7_equals_kron_construction():
    n = 5
    t = sp.diags([-np.ones(n - 1), 2 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1])
    i = sp.identity(n)
    ref = (sp.kron(sp.kron(i, i), t) + sp.kron(sp.kron(i, t), i) + sp.kron(sp.kron(t, i), i)).tocsr()
    ref.eliminate_zeros()
    ref.sort_indices()
    a = problems.stencil7(n, n, n)
    np.testing.assert_array_equal(a.row_ptr, ref.indptr)
    np.testing.assert_array_equal(a.col_idx, ref.indices)
    np.testing.assert_array_equal(a.values, ref.data)
    assert a.n_a == 7
    nnz = (3 * 128 - 2) * 128 * 128 * 3 - 2 * 128 ** 3  # sanity of the c3 count formula
    assert 7 * 128 ** 3 - 6 * 128 ** 2 == 14_581_760 and nnz > 0


def test_c1_and_c2_generators():
    p = problems.make_problem("c1")
    assert p.a.n == 4096 and p.a.nnz == 20_224
    assert np.all(np.diff(p.a.col_idx[p.a.row_ptr[0]:p.a.row_ptr[1]]) > 0)
    q = problems.make_problem("c2")
    assert q.a.n == 10_000 and q.a.nnz == 10_000
    assert abs(np.linalg.norm(q.b) - 1.0) < 1e-14
    lam = q.a.values
    assert lam[0] == 1e-3 and abs(lam[-1] - 1e2) < 1e-12


def test_varcoef27_is_symmetric_spd_like():
    p = problems.varcoef27(6, seed=3)
    m = sp.csr_matrix((p.a.values, p.a.col_idx, p.a.row_ptr), shape=(p.a.n, p.a.n))
    assert abs(m - m.T).max() == 0.0
    assert p.a.n_a == 27 and p.a.nnz == (3 * 6 - 2) ** 3
    w = np.linalg.eigvalsh(m.toarray())
    assert w[0] > 0
    d = m.diagonal()
    off = np.asarray(abs(m).sum(axis=1)).ravel() - d
    assert np.all(d >= off - 1e-12)  # diagonally dominant (Dirichlet surplus)


def test_weak_scaled_c5_grows_in_z():
    p = problems.make_problem("c5w", scale=4, world=2)
    assert p.a.n == 4 * 4 * 8


# ---- config + trace assembly -------------------------------------------------
def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        AdaptiveConfig(sigma=0, eps_star=1e-6)
    with pytest.raises(ValueError):
        AdaptiveConfig(sigma=5, eps_star=-1.0)
    with pytest.raises(ValueError):
        AdaptiveConfig(sigma=5, eps_star=1e-6, s_bar0=9)
    with pytest.raises(ValueError):
        AdaptiveConfig(sigma=5, eps_star=1e-6, variant="bogus")
    c = AdaptiveConfig(sigma=7, eps_star=1e-8)
    assert c.s_bar0 == 7 and c.f == 7


def test_make_config_maps_fields():
    prob = problems.make_problem("c1")
    cfg, c = make_config(AdaptiveConfig(sigma=8, eps_star=1e-10, basis_kind="chebyshev",
                                        c_strategy="kappa-estimate", variant="old",
                                        spectral_bounds=(0.1, 7.9)), prob, "fast")
    assert (c.sigma, c.s_bar0, c.f, c.basis_kind, c.c_strategy, c.variant) == (8, 8, 8, 2, 2, 0)
    assert c.has_bounds == 1 and c.bound_lo == 0.1 and c.trace_full == 0
    assert c.n_a == 5 and c.leja_grid == 10000 and c.max_outer == 5000
    with pytest.raises(ValueError):
        make_config(AdaptiveConfig(sigma=17, eps_star=1e-8), prob)
    with pytest.raises(ValueError):
        make_config(AdaptiveConfig(sigma=4, eps_star=1e-8, c_strategy="bogus"), prob)


def test_build_trace_from_synthetic_logs():
    cfg = AdaptiveConfig(sigma=3, eps_star=1e-8, max_outer=10)
    lb = LogBuffers(cfg)
    lb.s.status, lb.s.total_iters, lb.s.n_records = L.CONVERGED, 4, 2
    lb.rec_i[0, :7] = [0, 3, 3, 3, -1, 0, 0]
    lb.rec_i[1, :7] = [1, 3, 2, 1, 0, 3, 1]
    lb.rec_d[1, L.RECD_GEN_LO], lb.rec_d[1, L.RECD_GEN_HI] = 0.5, 2.0
    for i in range(4):
        lb.iters[i, :] = [1.0 + i, 0.5, 1e-3, 1e-3, np.nan, 2.0, 0.1, 3.0, 0.2, 1e-3]
    tr, co = build_trace(cfg, lb, "fast")
    tr.check_consistency()
    assert tr.converged and tr.total_outer == 2 and tr.outer_marks == [0, 3]
    assert tr.s_schedule == [3, 1] and co.alphas == [1.0, 2.0, 3.0, 4.0]
    r1 = tr.outer_records[1]
    assert r1.break_j == 0 and r1.s_tilde == 2 and r1.basis_params_used.kind == "newton"
    assert r1.basis_params_used.generated_from == (0.5, 2.0)
    assert tr.outer_records[0].break_j is None


def test_assemble_tridiag_host():
    """classic.py:12-30 on a hand-checked pair list (host helper, no GPU)."""
    from paper_1908_04081_b200 import CgCoefficients, assemble_tridiag
    co = CgCoefficients()
    for a, b in [(0.5, 0.25), (0.25, 4.0), (1.0, 1.0)]:
        co.append(a, b)
    t = assemble_tridiag(co, 3)
    want = np.array([[2.0, 1.0, 0.0],
                     [1.0, 4.0 + 0.5, 8.0],
                     [0.0, 8.0, 1.0 + 16.0]])
    np.testing.assert_allclose(t, want)
    with pytest.raises(ValueError):
        assemble_tridiag(co, 0)
    with pytest.raises(ValueError):
        assemble_tridiag(co, 4)


def test_harness_formats_host(tmp_path):
    """emit_trace_csv / emit_summary_table / round_up_2sig (harness.py) on a
    hand-built trace -- host formatting, no GPU."""
    from paper_1908_04081_b200 import SolveTrace
    from paper_1908_04081_b200.harness import (ExperimentSpec, ResultRow, emit_summary_table,
                                               emit_trace_csv, round_up_2sig)
    assert round_up_2sig(2.31e-16) == pytest.approx(2.4e-16)
    assert round_up_2sig(0.0) == 0.0
    tr = SolveTrace()
    for s_k in (2, 1):
        tr.mark_outer(s_k)
        for _ in range(s_k):
            tr.record_iteration(0.5, 0.25, 1e-3, 2.0, 0.1, 3.0, 0.9)
    path = emit_trace_csv(tr, str(tmp_path / "t.csv"))
    lines = open(path).read().splitlines()
    assert lines[1] == "1,1,2,0.5,0.25,0.001,0.10000000000000001,3,2"
    assert lines[3].startswith("3,2,1,")
    rows = [ResultRow("m", "hscg", "", "", 0, 1e-8, "9 (9)", "converged", 9, 9, 1e-9),
            ResultRow("m", "sstep", "monomial", "", 4, 1e-8, "3 (10)", "converged", 10, 3, 1e-9)]
    md = open(emit_summary_table(rows, "markdown", str(tmp_path / "s.md"))).read()
    assert md.splitlines()[0] == "| m eps*=1.00e-08 | s=4 |"
    assert "| sstep monomial | 3 (10) |" in md and "| hscg | 9 (9) |" in md
    with pytest.raises(ValueError):
        ExperimentSpec(matrices=[])
    with pytest.raises(ValueError):
        ExperimentSpec(matrices=["x"], algorithms=["cg"])
