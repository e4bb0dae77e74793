"""GPU tier for the experiment harness (harness.py):
run_grid over every algorithm on a synthetic Matrix Market file, against the
reference's own run_grid (oracle/make_golden.py gen_grid).  Rows come in the
reference's order; at eps* = 1e-8 every outcome matches and the counts agree
to one iteration / one outer loop (at 4-5 outer loops a single s~ decision
moved by Gram rounding is the noise floor); at the HSCG-attainable tolerance
(~2e-16, machine precision) only the tolerance is compared -- verdicts there
are rounding noise in either implementation."""

import os

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_1908_04081_b200.harness import ExperimentSpec, emit_summary_table, run_grid

pytestmark = pytest.mark.gpu


def test_run_grid_matches_reference(gpu_ready, tmp_path):
    g = golden("grid_rand300")
    spec = ExperimentSpec(
        matrices=[(os.path.join(ROOT, "tests", "golden", "mm", "rand300_gen.mtx"), "rand300")],
        s_values=[4, 8], eps_modes=["hscg-attainable", 1e-8], basis_kinds=["newton", "chebyshev"],
        c_strategies=["adaptive"])
    rows = run_grid(spec, str(tmp_path))
    keys = [f"{r.algorithm}|{r.basis}|{r.c_strategy}|{r.s}" for r in rows]
    assert keys == [str(k) for k in g["keys"]]
    for r, eps, out, it, ou, cell in zip(rows, g["eps"], g["outcome"], g["iters"], g["outer"],
                                         g["cell"]):
        if eps == 1e-8:
            assert r.eps_star == eps
            assert r.outcome == str(out), r
            assert abs(r.total_iters - int(it)) <= 1 and abs(r.total_outer - int(ou)) <= 1, r
        else:
            assert abs(r.eps_star - eps) <= 0.1 * eps
        lines = open(r.trace_file).read().splitlines()
        assert lines[0].startswith("global_iter,outer_iter,s_k,") and len(lines) == r.total_iters + 1
    md = emit_summary_table(rows, "markdown", str(tmp_path / "t.md"))
    ours = open(md).read().split("\n\n")
    ref = str(g["table"]).split("\n\n")
    assert len(ours) == len(ref)
    for a, b in zip(ours, ref):  # same blocks, headers and row labels
        la, lb = a.splitlines(), b.splitlines()
        assert len(la) == len(lb)
        assert [l.split(" | ")[0] for l in la[2:]] == [l.split(" | ")[0] for l in lb[2:]]
