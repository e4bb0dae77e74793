"""Outer / total iteration counts of the c5 weak-scaled global problems
(256 x 256 x 256N) for N = 1, 2, 4, 8, solved on one GPU with adaptive_solve
(trace="fast"), written to profiles/counts.json: the reference arm of bench.py
extrapolates its one-outer-loop CPU sample with them (the reference itself
would need hours per global solve).

    python tools/measure_counts.py [N ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    worlds = [int(w) for w in sys.argv[1:]] or [1, 2, 4, 8]
    path = os.path.join(ROOT, "profiles", "counts.json")
    counts = json.load(open(path)) if os.path.exists(path) else {}
    for w in worlds:
        t0 = time.perf_counter()
        prob = problems.make_problem("c5w", world=w)
        tg = time.perf_counter() - t0
        _, tr, _ = adaptive_solve(prob, AdaptiveConfig(sigma=12, eps_star=1e-10,
                                                       basis_kind="newton"), trace="fast")
        counts[f"c5w_w{w}"] = {"outer": tr.total_outer, "total": tr.total_iters,
                               "converged": tr.converged,
                               "source": f"GPU solve of the global 256x256x{256 * w} problem "
                                         "(adaptive_solve, trace='fast', parity-tested)"}
        print(f"N={w}: n={prob.a.n} outer={tr.total_outer} total={tr.total_iters} "
              f"conv={tr.converged} gen={tg:.1f}s solve={time.perf_counter() - t0 - tg:.1f}s",
              flush=True)
        del prob
        json.dump(counts, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
