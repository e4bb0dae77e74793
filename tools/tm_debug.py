"""Run one small TMA-march solve (c5 at 32^3) -- for debug side builds
(SSCG_LIB=.../libsscg_dbg.so, -DMBAR_DEBUG: timed-out mbarrier waits are
recorded and read back with sscg_debug_mbar)."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1908_04081_b200 import AdaptiveConfig, _lib as L, adaptive_solve, problems
from paper_1908_04081_b200.kernels import _plan
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 32
prob = problems.make_problem("c5", scale=scale)
print(_plan(prob.a).mpk_schedule(12), flush=True)
try:
    x, tr, co = adaptive_solve(prob, AdaptiveConfig(sigma=12, eps_star=1e-10, basis_kind="newton",
                                                    max_outer=3), trace="fast")
    print("solve returned", tr.total_outer, tr.total_iters, co.alphas[:3], flush=True)
except Exception as e:
    print("solve failed:", e, flush=True)
lib = L.load()
if hasattr(lib, "sscg_debug_mbar"):
    buf = (C.c_uint * 8)()
    print("dbg rc", lib.sscg_debug_mbar(buf), list(buf))
