import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems
from paper_1908_04081_b200.kernels import _plan
import bench
for cfgname in sys.argv[1:] or ["c5w"]:
    key, sigma, basis, eps, _, _ = bench.CONFIGS[cfgname]
    prob = problems.make_problem(key)
    t0 = time.perf_counter(); plan = _plan(prob.a, 0); t1 = time.perf_counter()
    adaptive_solve(prob, AdaptiveConfig(sigma=sigma, eps_star=eps, basis_kind=basis), trace="fast"); t2 = time.perf_counter()
    adaptive_solve(prob, AdaptiveConfig(sigma=sigma, eps_star=eps, basis_kind=basis), trace="fast"); t3 = time.perf_counter()
    print(cfgname, f"plan {t1-t0:.3f}s first solve {t2-t1:.3f}s second solve {t3-t2:.3f}s")
