"""Benchmark: adaptive s-step CG (arXiv 1908.04081) on B200 -- BASELINE.json metric
"s-step CG iterations/sec & HBM GB/s (frac of peak) at 1/2/4/8 B200; syncs to tol".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5w] [--impl reference]

One step = one full solve to eps* (the hot path: every outer loop's matrix-powers
levels, Gram, O(s^2) control kernel and recovery, on the device).  Workload at
N=1: config c5 weak-scaled, a 256^3 7-point Poisson slab per GPU, sigma=12,
dynamic Newton basis, eps*=1e-10 (BASELINE.json configs[4]); --config picks the
other partitioned configs (c4 / c4j 192^3 and c5 512^3 strong-scaled, c3 128^3).

--gpus N > 1 runs the row-partitioned solve, one process per GPU: under
torchrun (WORLD_SIZE set, it must equal N) or, without it, bench.py re-launches
itself under torch.distributed.run with N ranks.  --partitioned takes the
partitioned (NCCL) path at N = 1 too.

value   CG iterations/s, device time (CUDA events on the solver stream) with b,
        x0 and A resident in HBM; max over ranks.  Weak scaling (c5w): N x
        total_iters / time (one unit = one CG iteration on one 256^3 slab);
        strong scaling (c3 / c4 / c4j / c5): total_iters / time.
e2e     the same metric through the public API with host buffers (H2D of b, x0
        and D2H of x and the logs inside the timed region).
roofline  dominant kernel = the matrix-powers levels: algorithmic bytes
         / their CUDA-event time from one profiled
        solve after the timed region, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the reference's CPU arithmetic (oracle/sscg_oracle.py, a port of
        its numpy/scipy calls) as shipped -- per-iteration diagnostics on --
        timed on this host for one outer loop of the same problem and
        extrapolated to the solve's counts.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# name: (problem key, sigma, basis, eps*, scaling, description)
CONFIGS = {
    "c5w": ("c5w", 12, "newton", 1e-10, "weak",
            "c5 weak-scaled: 3D Poisson 7-pt 256^3 per GPU, sigma=12 Newton, eps*=1e-10"),
    "c5": ("c5", 12, "newton", 1e-10, "strong",
           "c5: 3D Poisson 7-pt 512^3 row-slab partitioned, sigma=12 Newton, eps*=1e-10"),
    "c3": ("c3", 10, "chebyshev", 1e-10, "strong",
           "c3: 3D Poisson 7-pt 128^3, sigma=10 Chebyshev, eps*=1e-10"),
    "c4": ("c4", 10, "newton", 1e-8, "strong",
           "c4: 27-pt var-coef 192^3 (lognormal 1.5), sigma=10 Newton, eps*=1e-8"),
    "c4j": ("c4j", 10, "newton", 1e-8, "strong",
            "c4 Jacobi-scaled (secondary run, SURVEY.md H6): 27-pt var-coef 192^3, "
            "sigma=10 Newton, eps*=1e-8"),
    "c1": ("c1", 8, "newton", 1e-10, "strong", "c1: 2D Poisson 64^2, sigma=8 Newton, eps*=1e-10"),
    "c2": ("c2", 10, "chebyshev", 1e-8, "strong", "c2: Strakos 1e4, sigma=10 Chebyshev, eps*=1e-8"),
}
GOLDEN_COUNTS = {"c5w": "full_c5w", "c3": "full_c3"}  # reference runs at the full size


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


# ---------------------------------------------------------------------------
# algorithmic bytes
def kernel_name(sched):
    """The level kernel (levels >= 1) a matrix-powers schedule runs."""
    if sched["kind"] == "pattern":
        return {"tma march": "k_level_tm", "march": "k_level_zm",
                "superset": "k_level_ss"}.get(sched.get("form"), "k_level_pat")
    return {"csr": "k_level_staged", "stencil values": "k_level_vs"}[sched["kind"]]


def a_bytes_per_level(n, nnz, sched):
    """Bytes of the operator one matrix-powers level must stream: CSR
    (12 nnz + 4 (n+1)) or, for a pattern-compressed plan, the
    1- or 2-byte row ids (the pattern table lives in shared memory), or the
    value stream's 8 bytes per stored plane and row (every union slot, or the
    diagonal and the upper offsets of a bitwise symmetric operator)."""
    if sched and sched.get("kind") == "pattern":
        return (1 if sched["patterns"] <= 256 else 2) * n
    if sched and sched.get("kind") == "stencil values":
        return 8 * sched.get("planes", sched["slots"]) * n  # symmetric form: half the planes
    return 12 * nnz + 4 * (n + 1)


def mpk_bytes_per_outer(n, nnz, sigma, mu_nonzero, sched=None):
    """Algorithmic bytes of the sigma matrix-powers levels of one outer loop:
    A once per level, 16 n per generated column (in + out), +8 n for the
    Chebyshev two-back term (levels >= 1), x and b on level 0 (true residual)."""
    s_a = a_bytes_per_level(n, nnz, sched)
    gen = 2 * sigma - 1
    two_back = (2 * sigma - 3) if mu_nonzero else 0
    return sigma * s_a + 16 * n * gen + 8 * n * two_back + 16 * n


def outer_bytes(n, nnz, sigma, s_t, mu_nonzero, sched=None):
    """One outer loop: the levels, the Gram (one read of Y), the recovery."""
    return (mpk_bytes_per_outer(n, nnz, sigma, mu_nonzero, sched) + 8 * n * (2 * sigma + 1)
            + 8 * n * (2 * s_t + 1) + 8 * n + 24 * n)


def cpu_threads():
    """(threads the CPU path may use, description): OpenBLAS' pool (dgemm/dgemv
    of the Gram and recovery) -- scipy csr_matvec and numpy element-wise work
    run on one core."""
    try:
        import threadpoolctl
        np.ones(2) @ np.ones(2)
        pools = [(d["internal_api"], int(d["num_threads"]), d.get("version"))
                 for d in threadpoolctl.threadpool_info()]
    except Exception:
        pools = []
    blas = max([t for _, t, _ in pools] or [1])
    return blas, (f"os.cpu_count()={os.cpu_count()}; BLAS pools {pools}; scipy csr_matvec "
                  "and numpy element-wise work (most of the time) are single-threaded")


def workload_config(args, world):
    """The `config` dict -- identical in both arms (same workload)."""
    key, sigma, basis, eps, scaling, desc = CONFIGS[args.config]
    c = {"workload": desc, "config": args.config, "sigma": sigma, "basis": basis,
         "eps_star": eps, "scaling": scaling, "x0": "0",
         "l2": "inputs larger than L2 (each vector >= 16 MB; Y >= 0.35 GB)"
               if key not in ("c1", "c2") else "L2-resident (latency-bound)"}
    if args.scale:
        c["scale"] = args.scale
    c["parallelism"] = (f"dp{world} row slabs (ghost depth sigma; one halo exchange + one "
                        "allreduce per outer loop)") if (world > 1 or args.partitioned) else "dp1"
    return c


def global_shape(args, world):
    """(problem key, nx, ny, nz) of the global problem of a partitioned run."""
    key = CONFIGS[args.config][0]
    if key == "c5w":
        e = args.scale or 256
        return key, e, e, e * world
    e = args.scale or {"c5": 512, "c3": 128, "c4": 192, "c4j": 192}.get(key, 0)
    if not e:
        raise SystemExit(f"--config {args.config} is not a partitioned 3-D workload")
    return key, e, e, e


# ---------------------------------------------------------------------------
def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n):
    """--gpus N > 1 without torchrun: run this same command as N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    return subprocess.call(cmd)


def init_gloo(rank, world):
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29533))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


# ---------------------------------------------------------------------------
def profile_solve(lib, L, handle, run):
    """One profiled solve (per-kernel-class event times) outside the timed region."""
    import ctypes as C
    L.check(lib.sscg_set_profiling(handle, 1))
    run()
    L.check(lib.sscg_set_profiling(handle, 0))
    pms = np.zeros(5)
    pcnt = np.zeros(5, dtype=np.int64)
    L.check(lib.sscg_get_profile(handle, L.dptr(pms), pcnt.ctypes.data_as(C.POINTER(C.c_int64))))
    return pms, pcnt


def roofline(n, nnz, sigma, basis, sched, pms, pcnt, outer_active, traffic=None):
    """roofline object of the matrix-powers levels: algorithmic bytes of the
    profiled solve's active outer loops / their CUDA-event time."""
    mu_nz = basis == "chebyshev"
    mpk_bytes = outer_active * mpk_bytes_per_outer(n, nnz, sigma, mu_nz, sched)
    peak, peak_kind = peaks()
    launches = max(1, outer_active * sigma)
    ach = mpk_bytes / (float(pms[0]) / 1e3) / 1e9
    tot = max(float(pms.sum()), 1e-9)
    return {
        "bound": "hbm", "kernel": kernel_name(sched), "schedule": sched,
        "a_bytes_per_level": a_bytes_per_level(n, nnz, sched),
        "a_bytes_per_level_csr": a_bytes_per_level(n, nnz, None),
        "achieved": ach, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
        "frac": ach / peak, "traffic": traffic,
        "algorithmic_bytes_per_launch": mpk_bytes / launches,
        "avg_launch_ms": float(pms[0]) / launches,
        "kernel_ms": {"mpk": pms[0], "gram": pms[1], "small": pms[2], "recovery": pms[3],
                      "other": pms[4]},
        "kernel_launches": {"mpk_outer_loops": int(pcnt[0]), "gram": int(pcnt[1]),
                            "small": int(pcnt[2]), "recovery": int(pcnt[3])},
        "share_of_step": {k: float(v) / tot for k, v in
                          zip(("mpk", "gram", "small", "recovery", "other"), pms)},
    }


def traffic_for(config, kname):
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(tpath)).get(config, {}).get(kname)
    except Exception:
        return None


def single_plan_line(prob, cfg_kw, steps, warmup, env=None, label=None, traffic_config=None):
    """Device-time solves of one problem on a single-GPU plan (optionally under
    an environment override, e.g. SSCG_PATTERN=0 for the CSR kernels)."""
    from paper_1908_04081_b200 import AdaptiveConfig, _lib as L
    from paper_1908_04081_b200.adaptive import LogBuffers, make_config
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        t0 = time.perf_counter()
        plan = L.Plan(prob.a.n, prob.a.row_ptr, prob.a.col_idx, prob.a.values, device=0)
        t_plan = time.perf_counter() - t0
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    lib = L.load()
    cfg, ccfg = make_config(AdaptiveConfig(**cfg_kw), prob, "fast")
    logs = LogBuffers(cfg)
    b, x0 = L.f64(prob.b), L.f64(prob.x0)
    L.check(lib.sscg_load(plan.handle, L.dptr(b), L.dptr(x0)))
    ms = []
    for k in range(warmup + steps):
        L.check(lib.sscg_run(plan.handle, ccfg, logs.s))
        if k >= warmup:
            ms.append(logs.s.device_ms)
    L.check(lib.sscg_fetch(plan.handle, None, logs.s))
    tot, outer = int(logs.s.total_iters), int(logs.s.total_outer)
    pms, pcnt = profile_solve(lib, L, plan.handle,
                              lambda: L.check(lib.sscg_run(plan.handle, ccfg, logs.s)))
    sched = plan.mpk_schedule(cfg.sigma)
    dev = sum(ms) / len(ms)
    n, nnz = prob.a.n, prob.a.nnz
    line = {"workload": label, "value": tot / (dev / 1e3), "unit": "iter/s", "ms_per_step": dev,
            "steps": steps, "syncs_to_tol": outer, "total_iters": tot,
            "converged": int(logs.s.status) == L.CONVERGED, "plan_create_s": round(t_plan, 2),
            "roofline": roofline(n, nnz, cfg.sigma, cfg.basis_kind, sched, pms, pcnt, outer + 1,
                                 traffic_for(traffic_config, kernel_name(sched))
                                 if traffic_config else None)}
    plan.close()
    return line


# ---------------------------------------------------------------------------
def run_single(args):
    """N = 1 on the single-GPU plan (the default headline line)."""
    import ctypes as C

    import scipy.sparse as sp

    from paper_1908_04081_b200 import AdaptiveConfig, _lib as L, adaptive_solve, problems
    from paper_1908_04081_b200.adaptive import LogBuffers, make_config
    from paper_1908_04081_b200.kernels import _plan

    key, sigma, basis, eps, scaling, desc = CONFIGS[args.config]
    t0 = time.perf_counter()
    prob = problems.make_problem(key, scale=args.scale)
    t_gen = time.perf_counter() - t0
    cfg_kw = dict(sigma=sigma, eps_star=eps, basis_kind=basis)
    if os.environ.get("SSCG_BENCH_LEJA_GRID"):  # experiments only (another grid = other shifts)
        cfg_kw["leja_grid"] = int(os.environ["SSCG_BENCH_LEJA_GRID"])
    n, nnz = prob.a.n, prob.a.nnz
    # first call through the public API on a matrix with no cached plan: plan
    # creation (upload, pattern compression) + the solve, host buffers in / out
    t0 = time.perf_counter()
    adaptive_solve(prob, AdaptiveConfig(**cfg_kw), trace="fast")
    t_first = time.perf_counter() - t0
    plan = _plan(prob.a, 0)
    lib = L.load()
    cfg, ccfg = make_config(AdaptiveConfig(**cfg_kw), prob, "fast")
    logs = LogBuffers(cfg)
    b, x0 = L.f64(prob.b), L.f64(prob.x0)
    L.check(lib.sscg_load(plan.handle, L.dptr(b), L.dptr(x0)))
    sched = plan.mpk_schedule(sigma)

    def dev_solve():
        L.check(lib.sscg_run(plan.handle, ccfg, logs.s))
        return logs.s.device_ms, int(logs.s.outer_launched)

    for _ in range(args.warmup):
        dev_solve()
    ms_list, launches = [], 0
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            ms, ol = dev_solve()
            ms_list.append(ms)
            # per outer loop: sigma levels, gram, small, params + (sigma-2) Leja, recovery
            launches += 2 + ol * (sigma + sigma + 2)
    L.check(lib.sscg_fetch(plan.handle, None, logs.s))
    total_iters, total_outer = int(logs.s.total_iters), int(logs.s.total_outer)
    converged = int(logs.s.status) == L.CONVERGED
    x = np.empty(n)
    L.check(lib.sscg_fetch(plan.handle, L.dptr(x), logs.s))
    a = prob.a
    rel = float(np.linalg.norm(prob.b - sp.csr_matrix((a.values, a.col_idx, a.row_ptr),
                                                      shape=(n, n)) @ x) / np.linalg.norm(prob.b))
    dev_ms = sum(ms_list) / len(ms_list)
    value = total_iters / (dev_ms / 1e3)

    pms, pcnt = profile_solve(lib, L, plan.handle, dev_solve)
    ph = np.zeros(8, dtype=np.int64)
    L.check(lib.sscg_get_small_phases(plan.handle, ph.ctypes.data_as(C.POINTER(C.c_int64))))
    calls = max(1, int(ph[7]))
    names = ["classify", "gram_extract_c", "nested_conds", "select_truncate", "inner_loop",
             "next_params"]
    small_phases = {nm: round(float(ph[i]) / calls / 1965.0, 2) for i, nm in enumerate(names)}
    s_t = [int(v) for v in logs.rec_i[:total_outer, L.REC_STILDE]]
    mu_nz = basis == "chebyshev"
    solve_bytes = sum(outer_bytes(n, nnz, sigma, st, mu_nz, sched) for st in s_t) + \
        mpk_bytes_per_outer(n, nnz, sigma, mu_nz, sched) + 8 * (2 * sigma + 1) * n
    hbm_peak, _ = peaks()
    solve_gbs = solve_bytes / (dev_ms / 1e3) / 1e9
    rl = roofline(n, nnz, sigma, basis, sched, pms, pcnt, total_outer + 1,
                  traffic_for(args.config, kernel_name(sched)))
    rl["small_phases_us_per_call"] = small_phases

    # end to end through the public API (host buffers), plan cached on the matrix
    e2e_times = []
    for _ in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        xe, tr, co = adaptive_solve(prob, AdaptiveConfig(**cfg_kw), trace="fast")
        e2e_times.append(time.perf_counter() - t0)
    e2e_value = tr.total_iters / (sum(e2e_times) / len(e2e_times))
    log_bytes = int(logs.iters.nbytes + logs.rec_i.nbytes + logs.rec_d.nbytes +
                    logs.conds.nbytes + 3 * logs.thetas.nbytes + logs.outer_true.nbytes)

    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline_sample(prob, cfg_kw, total_outer, total_iters)

    secondary = []
    if args.config == "c5w" and not args.no_secondary:
        # the general CSR kernels on the same operator (no pattern compression)
        secondary.append(single_plan_line(
            prob, cfg_kw, min(args.steps, 3), 1, env={"SSCG_PATTERN": "0"},
            label="c5w through the general CSR kernels (SSCG_PATTERN=0): " + desc,
            traffic_config=None if args.scale else "c5w"))
        # the value-stream kernels on c4j (27-point, row-varying values)
        _, s4, b4, e4, _, d4 = CONFIGS["c4j"]
        p4 = problems.make_problem("c4j", scale=args.scale and max(16, args.scale * 3 // 4))
        secondary.append(single_plan_line(p4, dict(sigma=s4, eps_star=e4, basis_kind=b4),
                                          min(args.steps, 3), 1, label=d4,
                                          traffic_config=None if args.scale else "c4j"))
        del p4

    line = {
        "metric": "cg_iterations_per_sec", "value": value, "unit": "iter/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded (np.random.default_rng(0)): x*~U[-1,1], b=A x*, x0=0",
        "config": workload_config(args, 1),
        "solve": {"n": n, "nnz": nnz, "syncs_to_tol": total_outer, "total_iters": total_iters,
                  "converged": converged, "final_true_rel_resid": rel, "trace": "fast",
                  "problem_gen_s": round(t_gen, 2), "collectives": plan.collectives(),
                  "syncs_note": "one global reduction point (the Gram) per outer loop; a "
                                "single-GPU plan needs no NCCL call for it"},
        "hbm": {"solve_gbs": solve_gbs, "frac_of_measured": solve_gbs / hbm_peak,
                "frac_of_8tbs": solve_gbs / 8000.0, "algorithmic_bytes_per_solve": solve_bytes},
        "roofline": rl,
        "e2e": {"value": e2e_value, "unit": "iter/s", "h2d_bytes_per_step": 16 * n,
                "d2h_bytes_per_step": 8 * n + log_bytes,
                "first_call_s": round(t_first, 3),
                "first_call_iter_per_s": total_iters / t_first,
                "note": "adaptive_solve(problem, cfg, trace='fast') with the plan cached on the "
                        "matrix like SparseMatrix._csr; first_call_s = the first call on a fresh "
                        "matrix: plan creation (upload + pattern compression) + the solve",
                "h2d_note": "h2d_bytes_per_step = the host buffers handed over (b and x0); the "
                            "staging threads read both, and chunks that are all zero (x0 = 0: "
                            "8 n bytes) are set on the device instead of crossing PCIe"},
        "cpu_baseline": cpu,
        "secondary": secondary,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line))


def partition_rows(key, nx, ny, nz):
    from paper_1908_04081_b200.partition import Stencil7Rows, Varcoef27Rows
    if key in ("c4", "c4j"):
        return Varcoef27Rows(nx, jacobi=key == "c4j")
    return Stencil7Rows(nx, ny, nz)


def run_partitioned(args, rank, world):
    """One rank of the row-partitioned solve (one process per GPU): gloo
    carries the setup plumbing (ghost requests, the NCCL id, the final
    max-over-ranks time), NCCL the per-outer-loop halo exchange and the one
    Gram allreduce inside the CUDA graph."""
    import types

    import scipy.sparse as sp
    import torch

    from paper_1908_04081_b200 import AdaptiveConfig, _lib as L
    from paper_1908_04081_b200.dist import check_ranks_agree, logs_digest, solve_partitioned
    from paper_1908_04081_b200.partition import slab_bounds

    dist = init_gloo(rank, world)
    key, sigma, basis, eps, scaling, desc = CONFIGS[args.config]
    local = int(os.environ.get("LOCAL_RANK", rank))
    key, nx, ny, nz = global_shape(args, world)
    rows = partition_rows(key, nx, ny, nz)
    n = rows.n
    t0 = time.perf_counter()
    bnd = slab_bounds(n, world)
    lo, hi = int(bnd[rank]), int(bnd[rank + 1])
    ip, cols, vals = rows.rows(np.arange(lo, hi))
    a_own = sp.csr_matrix((vals, cols, ip), shape=(hi - lo, n))
    if key in ("c4", "c4j"):
        b_glob = rows.rhs()
        b_own = b_glob[lo:hi]
    else:  # b = A x*, x* ~ U[-1, 1] from seed 0 (problems.poisson3d)
        xs = np.random.default_rng(0).uniform(-1.0, 1.0, n)
        b_own = a_own @ xs
        del xs
        b_glob = np.zeros(n)
        b_glob[lo:hi] = b_own
    nb2 = torch.tensor([float(b_own @ b_own)], dtype=torch.float64)
    dist.all_reduce(nb2)
    lam = [2.0 - 2.0 * math.cos(math.pi / (m + 1)) for m in (nx, ny, nz)]
    lmax = sum(2.0 + 2.0 * math.cos(math.pi / (m + 1)) for m in (nx, ny, nz))
    scal = types.SimpleNamespace(a=types.SimpleNamespace(n_a=27 if key.startswith("c4") else 7),
                                 norm_a=lmax, norm_abs_a=lmax, kappa_a=lmax / sum(lam))
    cfg = AdaptiveConfig(sigma=sigma, eps_star=eps, basis_kind=basis)

    def exchange(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def bcast(b):
        obj = [b]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    info = {}
    xo, tr, co, plan = solve_partitioned(rows, scal, b_glob, np.zeros(n), cfg, rank, world, local,
                                         exchange, bcast, info=info)
    t_setup = time.perf_counter() - t0
    del b_glob
    lib = L.load()
    logs, ccfg = info["logs"], info["ccfg"]
    sched = plan.mpk_schedule(sigma)

    def dev_solve():
        L.check(lib.sscg_run(plan.handle, ccfg, logs.s))
        return logs.s.device_ms, int(logs.s.outer_launched)

    for _ in range(args.warmup):
        dev_solve()
    dist.barrier()
    ms_list, launches = [], 0
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            dist.barrier()
            ms, ol = dev_solve()
            ms_list.append(ms)
            # per outer loop: halo pack/unpack, sigma levels, gram, small,
            # params + (sigma-2) Leja points, recovery (+ NCCL's own kernels)
            launches += 3 + ol * (2 * sigma + 4)
    dev_ms = sum(ms_list) / len(ms_list)
    tmax = torch.tensor([dev_ms], dtype=torch.float64)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    # end to end through the C ABI with host buffers, max over ranks
    b_loc, x0_loc = info["b"], info["x0"]
    x_host = L.result_pool.vector(hi - lo)  # page-locked (sscg_host_alloc): x back by one DMA
    e2e = []
    for _ in range(max(1, min(args.steps, 3))):
        dist.barrier()
        t1 = time.perf_counter()
        L.check(lib.sscg_solve(plan.handle, ccfg, L.dptr(b_loc), L.dptr(x0_loc), L.dptr(x_host),
                               logs.s))
        e2e.append(time.perf_counter() - t1)
    te = torch.tensor([sum(e2e) / len(e2e)], dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    L.check(lib.sscg_fetch(plan.handle, None, logs.s))
    total_iters, total_outer = int(logs.s.total_iters), int(logs.s.total_outer)
    # every rank decided the same: compare the decision hash across ranks
    check_ranks_agree(exchange(logs_digest(logs)))
    coll = plan.collectives()
    pms, pcnt = profile_solve(lib, L, plan.handle, dev_solve)
    mpk_ms_t = torch.tensor([float(pms[0])], dtype=torch.float64)
    dist.all_reduce(mpk_ms_t, op=dist.ReduceOp.MAX)
    L.check(lib.sscg_fetch(plan.handle, None, logs.s))
    # global true residual from the owned pieces (independent host SpMV)
    x_glob = torch.zeros(n, dtype=torch.float64)
    x_glob[lo:hi] = torch.from_numpy(x_host)
    dist.all_reduce(x_glob)
    resid = a_own @ x_glob.numpy() - b_own
    rr = torch.tensor([float(resid @ resid)], dtype=torch.float64)
    dist.all_reduce(rr)
    rel = math.sqrt(rr.item() / nb2.item())
    ms = tmax.item()
    units = world if scaling == "weak" else 1
    value = units * total_iters / (ms / 1e3)
    if rank == 0:
        n_own = hi - lo
        pms[0] = mpk_ms_t.item()
        rl = roofline(n_own, int(ip[-1]), sigma, basis, sched, pms, pcnt, total_outer + 1)
        rl["kernel"] += " (owned rows; ghost-row levels are redundant work, not counted)"
        cpu = None
        if not args.no_cpu and world == 1:
            from paper_1908_04081_b200 import problems
            prob = problems.make_problem(key, scale=args.scale, world=1)
            cpu = cpu_baseline_sample(prob, dict(sigma=sigma, eps_star=eps, basis_kind=basis),
                                      total_outer, total_iters)
        line = {
            "metric": "cg_iterations_per_sec", "value": value, "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic, seeded (np.random.default_rng(0))",
            "config": workload_config(args, world),
            "solve": {"global_shape": [nx, ny, nz], "n": n, "n_per_gpu": n_own,
                      "syncs_to_tol": total_outer, "total_iters": total_iters,
                      "converged": int(logs.s.status) == L.CONVERGED,
                      "final_true_rel_resid": rel, "trace": "fast",
                      "value_definition": ("world x total_iters / max-over-ranks device time "
                                           "(one unit = a CG iteration on one slab)"
                                           if scaling == "weak" else
                                           "total_iters / max-over-ranks device time"),
                      "global_iters_per_sec": total_iters / (ms / 1e3),
                      "setup_s": round(t_setup, 2), "collectives": coll,
                      "ranks_agree": True},
            "roofline": rl,
            "e2e": {"value": units * total_iters / te.item(), "unit": "iter/s",
                    "h2d_bytes_per_step": int(8 * (len(b_loc) + len(x0_loc))),
                    "d2h_bytes_per_step": int(8 * (hi - lo) + logs.iters.nbytes),
                    "note": "sscg_solve per rank (host b, x0 -> x, logs), max over ranks"},
            "cpu_baseline": cpu,
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line))
    dist.barrier()


# ---------------------------------------------------------------------------
# CPU: the reference's arithmetic (oracle port) on this host
def reference_counts(config, world):
    """(outer, total, source) of the global solve the CPU figure extrapolates to:
    the reference's own full-size run when one is committed (tests/golden/
    full_*.npz, made by running the reference here), else the GPU counts."""
    name = GOLDEN_COUNTS.get(config) if world == 1 else None
    if name:
        path = os.path.join(ROOT, "tests", "golden", name + ".npz")
        if os.path.exists(path):
            f = np.load(path)["flags"]
            return int(f[4]), int(f[3]), f"the reference's own full run ({name}.npz)"
    cpath = os.path.join(ROOT, "profiles", "counts.json")
    if os.path.exists(cpath):
        c = json.load(open(cpath)).get(f"{config}_w{world}")
        if c:
            return int(c["outer"]), int(c["total"]), "GPU solve of the global problem (counts.json)"
    return None


def time_outer(prob, cfg_kw, diagnostics):
    """Seconds of one outer loop (max_outer=1) of the oracle port, and the
    inner iterations it ran."""
    from oracle import sscg_oracle as O
    t0 = time.perf_counter()
    _, tr, _, _ = O.solve_problem(prob, O.OracleConfig(max_outer=1, **cfg_kw),
                                  diagnostics=diagnostics)
    return time.perf_counter() - t0, max(1, tr.total_iters)


def diag_unit_seconds(prob, s_avg, reps=2):
    """Seconds of the reference's per-inner-iteration diagnostics
    (adaptive.py:205-215: recover_iterates -- x_j, r_j, p_j from the block's
    2 s~ + 1 columns, sstep.py:37-44 -- then tv = b - A x_j and three norms),
    timed on this host with the reference's own numpy / scipy calls on a block
    of the problem's size (s~ = the solve's mean block length)."""
    import scipy.sparse as sp
    a = prob.a
    mat = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n))
    k = 2 * max(1, int(round(s_avg))) + 1
    yt = np.ones((a.n, k))
    coef = np.full(k, 1e-3)
    x, b = np.asarray(prob.x0, dtype=float), np.asarray(prob.b, dtype=float)
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        xj = x + yt @ coef
        rj = yt @ coef
        yt @ coef  # p_j (recover_iterates forms all three)
        tv = b - mat @ xj
        np.linalg.norm(tv), np.linalg.norm(rj), np.linalg.norm(tv - rj)
        best = min(best, time.perf_counter() - t0)
    del yt
    return best


def cpu_baseline_sample(prob, cfg_kw, outer, total):
    """The as-shipped reference (per-iteration diagnostics on, adaptive.py:205-215)
    on this host: one outer loop of the oracle port without the diagnostics
    (the per-outer cost) plus the diagnostics' per-iteration cost measured
    with the same numpy / scipy calls; the solve is (outer + 1) x per-outer +
    total x per-iteration."""
    t_off, _ = time_outer(prob, cfg_kw, False)
    unit = diag_unit_seconds(prob, total / max(1, outer))
    est = t_off * (outer + 1) + unit * total
    cores, tnote = cpu_threads()
    return {"value": total / est, "unit": "iter/s", "cores": cores, "kind": "port",
            "value_diagnostics_off": total / (t_off * (outer + 1)),
            "sample": f"oracle/sscg_oracle.py (the reference's numpy/scipy arithmetic) on the "
                      f"same {prob.a.n}-row problem: one outer loop {t_off:.2f}s; the "
                      f"per-iteration diagnostics {unit:.3f}s; solve = {outer}+1 outer loops + "
                      f"{total} iterations = {est:.1f}s",
            "threads_note": tnote}


def run_reference(args, rank, world):
    """The reference's CPU path (oracle port of its numpy/scipy arithmetic, as
    shipped: per-iteration diagnostics on) on this host, same config / metric;
    rank 0 only.  A step = one outer loop of it on one slab-sized problem (for
    c5w the 256^3 slab every rank owns; an outer loop of the global
    256x256x(256N) problem costs N x that, linear in rows); the value
    extrapolates to the global solve's counts."""
    if rank != 0:
        return
    from paper_1908_04081_b200 import problems
    key, sigma, basis, eps, scaling, desc = CONFIGS[args.config]
    prob = problems.make_problem(key, scale=args.scale, world=1)
    cfg_kw = dict(sigma=sigma, eps_star=eps, basis_kind=basis)
    if args.scale:  # a test-sized problem: the oracle's own full solve gives the counts
        from oracle import sscg_oracle as O
        _, otr, _, _ = O.solve_problem(prob, O.OracleConfig(**cfg_kw), diagnostics=False)
        counts = (otr.total_outer, otr.total_iters, "the oracle's full solve of this scaled problem")
    else:
        counts = reference_counts(args.config, world)
    if counts is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"no outer/total counts for {args.config} at N={world}"}))
        return
    outer, total, src = counts
    small = problems.make_problem(key, scale=24 if key in ("c5w", "c5", "c3") else 12,
                                  world=1) if key in ("c5w", "c5", "c3", "c4", "c4j") else prob
    for _ in range(args.warmup):  # warm imports / allocator on a small instance
        time_outer(small, cfg_kw, False)
    # the per-iteration diagnostics, once (the reference's own numpy/scipy calls)
    per_it = diag_unit_seconds(prob, total / max(1, outer))
    offs = []
    for _ in range(args.steps):
        t, _ = time_outer(prob, cfg_kw, False)
        offs.append(t)
    t_off = sum(offs) / len(offs)
    t_on = t_off + per_it * total / max(1, outer + 1)  # one outer loop as shipped, on average
    # the global problem is N slabs (weak scaling) or the problem itself (strong)
    slabs = world if scaling == "weak" else 1
    est = slabs * (t_off * (outer + 1) + per_it * total)
    units = world if scaling == "weak" else 1
    value = units * total / est
    cores, tnote = cpu_threads()
    line = {
        "metric": "cg_iterations_per_sec", "value": value, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_on * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded (np.random.default_rng(0))", "impl": "reference",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": cores, "kind": "port",
                         "threads_note": tnote,
                         "value_diagnostics_off": units * total / (slabs * t_off * (outer + 1)),
                         "sample": f"each step = one outer loop of the oracle port on one "
                                   f"{prob.a.n}-row problem ({t_off:.2f}s); the reference's "
                                   f"per-iteration diagnostics {per_it:.3f}s (as shipped, "
                                   f"adaptive.py:205-215); the global N={world} solve = {slabs} x "
                                   f"({outer}+1 outer loops + {total} iterations) = {est:.1f}s; "
                                   f"counts: {src}"},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_hscg_partitioned(args, rank, world):
    """Distributed HSCG (classic CG, §8(f)2) on the same row slabs: one NCCL halo
    exchange and two NCCL allreduces per iteration -- the baseline the s-step
    solver's one synchronisation per outer loop is compared with."""
    import scipy.sparse as sp
    import torch

    from paper_1908_04081_b200 import _lib as L
    from paper_1908_04081_b200.classic import hscg_logs
    from paper_1908_04081_b200.dist import hscg_partitioned
    from paper_1908_04081_b200.partition import slab_bounds

    dist = init_gloo(rank, world)
    key, sigma, basis, eps, scaling, desc = CONFIGS[args.config]
    local = int(os.environ.get("LOCAL_RANK", rank))
    key, nx, ny, nz = global_shape(args, world)
    rows = partition_rows(key, nx, ny, nz)
    n = rows.n
    bnd = slab_bounds(n, world)
    lo, hi = int(bnd[rank]), int(bnd[rank + 1])
    if key in ("c4", "c4j"):
        b_glob = rows.rhs()
    else:
        ip, cols, vals = rows.rows(np.arange(lo, hi))
        xs = np.random.default_rng(0).uniform(-1.0, 1.0, n)
        b_glob = np.zeros(n)
        b_glob[lo:hi] = sp.csr_matrix((vals, cols, ip), shape=(hi - lo, n)) @ xs
        del xs

    def exchange(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    def bcast(bb):
        obj = [bb]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    info = {}
    hscg_partitioned(rows, b_glob, np.zeros(n), eps, rank, world, local, exchange, bcast,
                     mode=args.hscg_mode, info=info)
    plan, bl, x0l = info["plan"], info["b"], info["x0"]
    lib = L.load()
    iters, logs = hscg_logs(0)
    mode = L.HSCG_MODES[args.hscg_mode]
    ms = []
    with ClockSampler(local) as clk:
        for k in range(args.warmup + args.steps):
            dist.barrier()
            L.check(lib.sscg_hscg_ex(plan.handle, L.dptr(bl), L.dptr(x0l), float(eps),
                                     info["max_iters"], mode, None, logs))
            if k >= args.warmup:
                ms.append(logs.device_ms)
    t = torch.tensor([sum(ms) / len(ms)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    it = int(logs.total_iters)
    status = {L.CONVERGED: "converged", L.STAGNATED: "stagnated",
              L.DIVERGED: "diverged"}.get(int(logs.status), "max_iters")
    units = world if scaling == "weak" else 1
    if rank == 0:
        print(json.dumps({
            "metric": "cg_iterations_per_sec", "value": units * it / (t.item() / 1e3),
            "unit": "iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t.item(), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic, seeded", "impl": "ours",
            "solver": "hscg", "config": workload_config(args, world),
            "solve": {"n": n, "global_shape": [nx, ny, nz], "total_iters": it,
                      "syncs_to_tol": 2 * it, "status": status, "hscg_mode": args.hscg_mode,
                      "collectives": plan.collectives() if hasattr(plan, "collectives") else None},
            "clocks": clk.summary()}))
    dist.barrier()


# ---------------------------------------------------------------------------
def run_solver_compare(args):
    """--solver sstep|hscg (one GPU, informational, not the driver's headline):
    the same workload through fixed s-step CG (s = sigma, the config's basis
    with the stencil's exact spectral bounds) or Hestenes-Stiefel CG,
    device time per solve.  `syncs_to_tol` counts the global reductions a
    multi-GPU run would need: one per outer loop for s-step, two per iteration
    for HSCG (p.Ap, r.r)."""
    from paper_1908_04081_b200 import _lib as L, problems
    from paper_1908_04081_b200.kernels import _plan
    from paper_1908_04081_b200.sstep import sstep_solve
    key, sigma, basis, eps, scaling, desc = CONFIGS[args.config]
    prob = problems.make_problem(key, scale=args.scale)
    n = prob.a.n
    plan = _plan(prob.a, 0)
    lib = L.load()
    b, x0 = L.f64(prob.b), L.f64(prob.x0)
    ms, iters, syncs, status = [], 0, 0, None
    with ClockSampler(0) as clk:
        for k in range(args.warmup + args.steps):
            if args.solver == "hscg":
                logs = L.SscgLogs()
                logs.cap_iters, logs.iters = 0, None
                L.check(lib.sscg_hscg_ex(plan.handle, L.dptr(b), L.dptr(x0), float(eps), -1,
                                         L.HSCG_MODES[args.hscg_mode], None, logs))
                dev, it, sy = logs.device_ms, int(logs.total_iters), 2 * int(logs.total_iters)
                status = {L.CONVERGED: "converged", L.STAGNATED: "stagnated",
                          L.DIVERGED: "diverged"}.get(int(logs.status), "max_iters")
            else:
                nx = round(n ** (1.0 / 3.0)) if key in ("c3", "c5", "c5w") else None
                lam = (6 - 6 * math.cos(math.pi / (nx + 1)), 6 + 6 * math.cos(math.pi / (nx + 1))) \
                    if nx else None
                info = {}
                s_fixed = args.s or sigma
                _, tr, _ = sstep_solve(prob, s_fixed, eps, basis_kind=basis, spectral_bounds=lam,
                                       trace="fast", info=info)
                dev, it, sy = info["device_ms"], tr.total_iters, tr.total_outer
                status = ("converged" if tr.converged else "diverged" if tr.diverged
                          else "stagnated" if tr.stagnated else "max_outer")
            if k >= args.warmup:
                ms.append(dev)
                iters, syncs = it, sy
    dev_ms = sum(ms) / len(ms)
    print(json.dumps({
        "metric": "cg_iterations_per_sec", "value": iters / (dev_ms / 1e3), "unit": "iter/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded", "impl": "ours", "solver": args.solver,
        "config": workload_config(args, 1),
        "solve": {"n": n, "total_iters": iters, "syncs_to_tol": syncs, "status": status,
                  **({"s": args.s or sigma} if args.solver == "sstep" else {}),
                  **({"hscg_mode": args.hscg_mode} if args.solver == "hscg" else {})},
        "clocks": clk.summary()}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5w", choices=sorted(CONFIGS))
    ap.add_argument("--scale", type=int, default=None, help="override grid edge (testing)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the secondary (CSR path, value-stream c4j) lines at N=1")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the row-partitioned NCCL path even at one GPU")
    ap.add_argument("--solver", default="adaptive", choices=["adaptive", "sstep", "hscg"],
                    help="adaptive (the headline); sstep / hscg: one-GPU comparison lines")
    ap.add_argument("--s", type=int, default=None, help="fixed s for --solver sstep (default sigma)")
    ap.add_argument("--hscg-mode", default="production", choices=["reference", "production"],
                    help="--solver hscg: classic.py semantics (true residual every iteration) "
                         "or production CG (one SpMV per iteration)")
    ap.add_argument("--check-launch", action="store_true",
                    help="print this rank's (rank, world) and exit (launcher test)")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1 and args.impl == "ours":
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(env_world) if env_world is not None else args.gpus
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.check_launch:
        print(json.dumps({"rank": rank, "world": world}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.solver == "hscg" and (world > 1 or args.partitioned):
        run_hscg_partitioned(args, rank, world)
    elif args.solver != "adaptive":
        run_solver_compare(args)
    elif world > 1 or args.partitioned:
        run_partitioned(args, rank, world)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
