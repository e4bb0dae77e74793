"""Compare the first outer loops of a full-size GPU solve with the reference's
own run (tests/golden/full_<key>.npz): s~, conds, phi, break data, r_rel, c."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems, _lib as L

key = sys.argv[1] if len(sys.argv) > 1 else "c4j"
ref = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"full_{key}.npz"))
cfg = json.loads(str(ref["cfg"]))
prob = problems.make_problem(key)
info = {}
x, tr, co = adaptive_solve(prob, AdaptiveConfig(**cfg), trace="fast", info=info)
g = info["first_gram"]
rg = ref["first_g"]
print("first gram max rel", np.max(np.abs(g - rg) / np.sqrt(np.outer(np.diag(rg), np.diag(rg)))))
logs = info["logs"]
for k in range(min(5, len(tr.outer_records))):
    r = tr.outer_records[k]
    print(f"outer {k}: ours s~={r.s_tilde} s={r.s_actual} phi={r.phi:.6e} brk={r.break_j} "
          f"lhs={r.break_lhs:.6e} rhs={r.break_rhs:.6e} rrel={logs.rec_d[k, L.RECD_RREL]:.6e} "
          f"c={logs.rec_d[k, L.RECD_C]:.6e}")
    print("   ours conds", np.array2string(np.asarray(r.cond_used), precision=6))
    ri, rf = ref["rec_int"][k], ref["rec_float"][k]
    print(f"   ref  s~={ri[2]} s={ri[3]} brk={ri[4]} phi={rf[0]:.6e} lhs={rf[1]:.6e} rhs={rf[2]:.6e}")
    if k < len(ref["conds8"]):
        print("   ref  conds", np.array2string(ref["conds8"][k], precision=6))
m = int(ref["outer_marks"][min(4, len(ref["outer_marks"]) - 1)])
print("alphas ours", co.alphas[:m])
print("alphas ref ", ref["alphas"][:m])
print("lmin ours", tr.lambda_min[:m])
print("lmin ref ", ref["lambda_min"][:m])
print("lmax ours", tr.lambda_max[:m])
print("lmax ref ", ref["lambda_max"][:m])
