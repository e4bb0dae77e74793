"""Where the end-to-end time of adaptive_solve goes (GPU box):
host->device copies, device run, device->host copies, trace assembly."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1908_04081_b200 import AdaptiveConfig, _lib as L, adaptive_solve, problems
from paper_1908_04081_b200.adaptive import LogBuffers, build_trace, make_config
from paper_1908_04081_b200.kernels import _plan

prob = problems.make_problem("c5w")
cfg = AdaptiveConfig(sigma=12, eps_star=1e-10, basis_kind="newton")
for _ in range(2):
    adaptive_solve(prob, cfg, trace="fast")
lib = L.load()
c2, ccfg = make_config(cfg, prob, "fast")
plan = _plan(prob.a, 0)
for rep in range(3):
    t = [time.perf_counter()]
    b, x0 = L.f64(prob.b), L.f64(prob.x0)
    logs = LogBuffers(c2)
    x = np.empty(prob.a.n)
    t.append(time.perf_counter())
    L.check(lib.sscg_load(plan.handle, L.dptr(b), L.dptr(x0)))
    L.check(lib.sscg_run(plan.handle, ccfg, logs.s))
    t.append(time.perf_counter())
    L.check(lib.sscg_fetch(plan.handle, L.dptr(x), logs.s))
    t.append(time.perf_counter())
    tr, co = build_trace(c2, logs, "fast")
    tr.check_consistency()
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"prep {d[0]:.1f} ms  load+run {d[1]:.1f} ms (device {logs.s.device_ms:.1f})  "
          f"fetch {d[2]:.1f} ms  trace {d[3]:.1f} ms  total {sum(d):.1f}")
    t0 = time.perf_counter()
    adaptive_solve(prob, cfg, trace="fast")
    print(f"adaptive_solve {1e3 * (time.perf_counter() - t0):.1f} ms")
