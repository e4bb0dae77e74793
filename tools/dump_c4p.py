import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import cfg_of, golden, problem_from_arrays  # noqa
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve  # noqa
np.set_printoptions(precision=4, linewidth=220)
ref = golden("solve_c4p")
prob = problem_from_arrays(ref, "in_")
info = {}
x, tr, co = adaptive_solve(prob, AdaptiveConfig(**cfg_of(ref)), info=info)
lg = info["logs"]
ri = ref["rec_int"]
g = np.array([[r.s_bar, r.s_tilde, r.s_actual, -1 if r.break_j is None else r.break_j] for r in tr.outer_records])
n = min(len(g), len(ri))
d = np.nonzero(np.any(g[:n, 1:3] != ri[:n, 2:4], axis=1))[0]
print("gpu", tr.total_outer, tr.total_iters, "ref", ref["flags"][3:], "first diff outer", d[:10])
k = d[0] if len(d) else 0
for j in range(max(0, k - 1), min(n, k + 3)):
    r = tr.outer_records[j]
    print(j, "gpu s~,s,brk", g[j, 1:], "lhs/rhs", r.break_lhs, r.break_rhs, "c", lg.rec_d[j, 7], "rrel", lg.rec_d[j, 6])
    print("   gpu conds", np.asarray(r.cond_used))
    print("   ref s~,s,brk", ri[j, 2:], ref["rec_float"][j])
    if j < len(ref["conds8"]):
        print("   ref conds", ref["conds8"][j])
hist = np.bincount(g[:, 2], minlength=11), np.bincount(ri[:, 3], minlength=11)
print("s_actual histogram gpu", hist[0][:11], "\n                    ref", hist[1][:11])
print("s_tilde hist gpu", np.bincount(g[:, 1], minlength=11)[:11], "\n             ref", np.bincount(ri[:, 2], minlength=11)[:11])
print("breaks gpu", np.sum(g[:, 3] >= 0), "ref", np.sum(ri[:, 4] >= 0))
