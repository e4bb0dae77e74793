"""Diagnostics: first outer loops' cond estimates, GPU vs the reference golden."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import cfg_of, golden, golden_problem  # noqa
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, nested_basis_conds  # noqa
np.set_printoptions(precision=6, linewidth=200)
for name, pname in [("solve_494bus_old", "problem_494bus"), ("solve_nos1_chebyshev_unit", "problem_nos1"),
                    ("solve_nos1_newton_adaptive", "problem_nos1")]:
    ref = golden(name)
    prob = golden_problem(pname)
    info = {}
    x, tr, co = adaptive_solve(prob, AdaptiveConfig(**cfg_of(ref)), info=info)
    print(name, "gpu", tr.total_outer, tr.total_iters, tr.converged, "ref", ref["flags"])
    g0 = info["first_gram"]
    sb = (g0.shape[0] - 1) // 2
    print("  conds(first G) gpu-kernel on ref G:", nested_basis_conds(ref["first_g"], sb))
    for k in range(min(6, len(tr.outer_records))):
        r = tr.outer_records[k]
        print(f"  outer {k}: gpu s~={r.s_tilde} s={r.s_actual} brk={r.break_j} lhs={r.break_lhs:.6g} rhs={r.break_rhs:.6g}")
        print("     gpu conds", np.asarray(r.cond_used))
        if k < len(ref["conds8"]):
            print("     ref conds", ref["conds8"][k], " ref s~,s", ref["rec_int"][k][2:4], "brk", ref["rec_int"][k][4], ref["rec_float"][k][1:])
