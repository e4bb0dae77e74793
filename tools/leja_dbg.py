"""Leja-point phase cycles (side build with -DLEJA_DBG): grid objective,
local maxima, candidate sort, golden refinement, tie rule."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems, _lib as L
prob = problems.make_problem(sys.argv[1] if len(sys.argv) > 1 else "c1")
adaptive_solve(prob, AdaptiveConfig(sigma=int(sys.argv[2]) if len(sys.argv) > 2 else 8, eps_star=1e-10, basis_kind="newton"), trace="fast")
buf = (C.c_ulonglong * 8)()
L.load().sscg_debug_leja(buf)
n = max(1, buf[7])
print("points", n, "cycles/point:", {k: round(buf[i] / n) for i, k in enumerate(["grid", "maxima", "sort", "golden", "tie"])})

if buf[6]:
    print("golden_refine2 (warp 0): rounds", buf[6], "cycles per round", round(buf[5] / buf[6]))
    print("per round: log", round(buf[0] / buf[6]), "group sum", round(buf[1] / buf[6]), "broadcasts", round(buf[4] / buf[6]))
