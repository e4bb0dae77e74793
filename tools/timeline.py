"""Timeline of the outer-loop graph from the kernels' own clocks (GPU box).

    python tools/build_variants.py tl:SSCG_TIMELINE=1
    SSCG_LIB=paper_1908_04081_b200/_lib/libsscg_tl.so python tools/timeline.py [--config c5w]

The SSCG_TIMELINE side build makes every kernel of the outer-loop graph record
the globaltimer of its first CTA's start and its last warp's end, per outer
loop.  This prints, averaged over the steady outer loops of one solve, each
node's start (relative to level 0's start), duration and the gap to the node
before it on the main chain -- what a timeline view would show (no nsys here).
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5w")
    ap.add_argument("--lo", type=int, default=5)
    ap.add_argument("--hi", type=int, default=60)
    ap.add_argument("--dump", type=int, default=-1, help="also print this outer loop's raw rows")
    ap.add_argument("--steady", action="store_true",
                    help="also time the Gram / recovery alone, cool and in a long back-to-back run")
    args = ap.parse_args()
    import bench
    key, sigma, basis, eps, _, desc = bench.CONFIGS[args.config]
    prob = problems.make_problem(key)
    lib = L.load()
    fn = lib.sscg_debug_timeline
    fn.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    cfg = AdaptiveConfig(sigma=sigma, eps_star=eps, basis_kind=basis)
    cfg, ccfg = make_config(cfg, prob, "fast")
    logs = LogBuffers(cfg)
    b, x0 = L.f64(prob.b), L.f64(prob.x0)
    plan = L.Plan(prob.a.n, prob.a.row_ptr, prob.a.col_idx, prob.a.values)
    L.check(lib.sscg_load(plan.handle, L.dptr(b), L.dptr(x0)))
    reps, nodes = C.c_int(), C.c_int()
    for _ in range(2):
        L.check(lib.sscg_run(plan.handle, ccfg, logs.s))
    fn(None, C.byref(reps), C.byref(nodes))
    buf = np.zeros((reps.value, nodes.value, 2), dtype=np.uint64)
    fn(buf.ctypes.data, C.byref(reps), C.byref(nodes))  # read + reset (drops the warm solves)
    L.check(lib.sscg_run(plan.handle, ccfg, logs.s))
    ms = logs.s.device_ms
    fn(buf.ctypes.data, C.byref(reps), C.byref(nodes))
    L.check(lib.sscg_fetch(plan.handle, None, logs.s))
    outer = int(logs.s.total_outer)
    t0 = buf[:, :, 0].astype(np.float64)
    t1 = buf[:, :, 1].astype(np.float64)
    valid = (buf[:, :, 0] != np.uint64(0xFFFFFFFFFFFFFFFF)) & (buf[:, :, 1] != 0)
    names = {l: f"level{l}" for l in range(16)}
    names.update({16: "gram", 17: "small", 18: "recover", 19: "params"})
    names.update({20 + n: f"leja{n}" for n in range(2, 16)})
    lo, hi = args.lo, min(args.hi, outer - 2)
    # reference node: level 0 of the TMA march, else (other level kernels are
    # not instrumented) the parameter kernel that opens the outer loop
    ref = 0 if valid[lo:hi, 0].any() else 19
    valid[:, 19] = buf[:, 19, 0] != np.uint64(0xFFFFFFFFFFFFFFFF)
    t1[:, 19] = np.where(buf[:, 19, 1] != 0, t1[:, 19], t0[:, 19])
    chain = [l for l in range(sigma)] + [16, 17, 18]
    rows = []
    for nd in sorted(names):
        ks = [k for k in range(lo, hi) if valid[k, nd] and valid[k, ref]]
        if not ks:
            continue
        st = np.mean([t0[k, nd] - t0[k, ref] for k in ks]) / 1e3
        du = np.mean([t1[k, nd] - t0[k, nd] for k in ks]) / 1e3
        gap = None
        if nd in chain and chain.index(nd) > 0:
            pv = chain[chain.index(nd) - 1]
            g = [t0[k, nd] - t1[k, pv] for k in ks if valid[k, pv]]
            gap = float(np.mean(g)) / 1e3 if g else None
        elif nd == 0:
            g = [t0[k, 0] - t1[k - 1, 18] for k in ks if k >= 1 and valid[k - 1, 18]]
            gap = float(np.mean(g)) / 1e3 if g else None
        rows.append({"node": names[nd], "start_us": round(st, 1), "dur_us": round(du, 1),
                     "gap_before_us": None if gap is None else round(gap, 1), "n": len(ks)})
    period = np.mean([t0[k + 1, ref] - t0[k, ref] for k in range(lo, hi) if valid[k, ref] and valid[k + 1, ref]]) / 1e3
    print(json.dumps({"config": args.config, "device_ms": ms, "outer": outer,
                      "period_us": round(float(period), 1)}))
    for r in rows:
        print(json.dumps(r))
    if args.steady:
        import time
        sd = lib.sscg_debug_steady
        sd.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
        out = C.c_float()
        k = 2 * sigma + 1
        for which, nm in ((0, "gram"), (1, "recover")):
            res = {}
            for reps, pause in ((3, 3.0), (20, 3.0), (400, 0.0), (400, 0.0)):
                time.sleep(pause)
                sd(plan.handle, which, k, reps, C.byref(out))
                res[f"{reps}{'_cool' if pause else ''}"] = round(out.value * 1e3, 1)
            print(json.dumps({"steady": nm, "cols": k, "us_per_launch": res}))
    if args.dump >= 0:
        k = args.dump
        for nd in sorted(names):
            if valid[k, nd]:
                print(names[nd], (t0[k, nd] - t0[k, 0]) / 1e3, (t1[k, nd] - t0[k, 0]) / 1e3)


if __name__ == "__main__":
    main()
