import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems
from paper_1908_04081_b200.kernels import _plan
import bench
key, sigma, basis, eps, _, _ = bench.CONFIGS["c5w"]
cfg = AdaptiveConfig(sigma=sigma, eps_star=eps, basis_kind=basis)
for rep in range(3):
    prob = problems.make_problem(key)
    t0 = time.perf_counter(); plan = _plan(prob.a, 0); t1 = time.perf_counter()
    adaptive_solve(prob, cfg, trace="fast"); t2 = time.perf_counter()
    adaptive_solve(prob, cfg, trace="fast"); t3 = time.perf_counter()
    print(f"rep {rep}: plan {t1-t0:.3f}s first solve {t2-t1:.3f}s second solve {t3-t2:.3f}s", flush=True)
    del plan, prob
