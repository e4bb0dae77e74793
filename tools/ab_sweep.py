"""A/B sweep of matrix-powers schedules on one problem (GPU box).

    python tools/ab_sweep.py [--config c5w] [--outer 12] ENV1 ENV2 ...

Each ENV is a comma list like "SSCG_ZM=0" or "SSCG_ZM_ZC=16,SSCG_ZM_DYN=0"
(empty string = defaults).  For every ENV a fresh plan is created with that
environment, one solve capped at --outer outer loops runs unprofiled (device
time) and once profiled (per-class kernel ms); prints one JSON line per ENV.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1908_04081_b200 import AdaptiveConfig, _lib as L, problems  # noqa: E402
from paper_1908_04081_b200.adaptive import LogBuffers, make_config  # noqa: E402

KEYS = ("SSCG_PATTERN", "SSCG_STAGE_MAX_KB", "SSCG_LEJA_HEAD", "SSCG_PAT_SS", "SSCG_PF",
        "SSCG_PF_AHEAD", "SSCG_ZM", "SSCG_ZM_ZC", "SSCG_ZM_2D", "SSCG_ZM_DYN", "SSCG_LEJA_AFTER0",
        "SSCG_ZM_ZC0", "SSCG_VS", "SSCG_TM", "SSCG_TM_TAIL")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5w")
    ap.add_argument("--outer", type=int, default=12)
    ap.add_argument("envs", nargs="*")
    args = ap.parse_args()
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    key, sigma, basis, eps, _, desc = bench.CONFIGS[args.config]
    prob = problems.make_problem(key)
    lib = L.load()
    cfg = AdaptiveConfig(sigma=sigma, eps_star=eps, basis_kind=basis, max_outer=args.outer)
    cfg, ccfg = make_config(cfg, prob, "fast")
    logs = LogBuffers(cfg)
    b, x0 = L.f64(prob.b), L.f64(prob.x0)
    for env in args.envs or [""]:
        for k in KEYS:
            os.environ.pop(k, None)
        for kv in filter(None, env.split(",")):
            k, v = kv.split("=")
            os.environ[k] = v
        plan = L.Plan(prob.a.n, prob.a.row_ptr, prob.a.col_idx, prob.a.values)
        sched = plan.mpk_schedule(sigma)
        L.check(lib.sscg_load(plan.handle, L.dptr(b), L.dptr(x0)))
        ms = []
        for _ in range(3):
            L.check(lib.sscg_run(plan.handle, ccfg, logs.s))
            ms.append(logs.s.device_ms)
        L.check(lib.sscg_fetch(plan.handle, None, logs.s))
        outer = int(logs.s.total_outer)
        dbg = None
        L.check(lib.sscg_set_profiling(plan.handle, 1))
        L.check(lib.sscg_run(plan.handle, ccfg, logs.s))
        L.check(lib.sscg_set_profiling(plan.handle, 0))
        pms = np.zeros(5)
        pcnt = np.zeros(5, dtype=np.int64)
        L.check(lib.sscg_get_profile(plan.handle, L.dptr(pms), pcnt.ctypes.data_as(C.POINTER(C.c_int64))))
        act = max(1, int(pcnt[1]))
        print(json.dumps({"env": env, "sched": sched, "outer": outer, "iters": int(logs.s.total_iters),
                          "dev_ms": min(ms), "ms_per_outer": min(ms) / act,
                          "mpk_ms_per_outer": pms[0] / act, "gram": pms[1] / act,
                          "small": pms[2] / act, "rec": pms[3] / act, "other": pms[4] / act, "dbg": dbg}),
              flush=True)
        plan.close()


if __name__ == "__main__":
    main()
