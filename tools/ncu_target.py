"""A short c5w solve (first outer loops only) as an ncu target:
    ncu ... -k regex:k_level_tm python tools/ncu_target.py [max_outer] [config]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems  # noqa: E402
import bench  # noqa: E402

mo = int(sys.argv[1]) if len(sys.argv) > 1 else 2
key, sigma, basis, eps, _, _ = bench.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c5w"]
prob = problems.make_problem(key)
x, tr, co = adaptive_solve(prob, AdaptiveConfig(sigma=sigma, eps_star=eps, basis_kind=basis,
                                                max_outer=mo), trace="fast")
print("outer", tr.total_outer, "iters", tr.total_iters)
