"""Benchmark: adaptive s-step CG (arXiv 1908.04081) on B200 -- BASELINE.json metric
"s-step CG iterations/sec & HBM GB/s (frac of peak) at 1/2/4/8 B200; syncs to tol".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5w] [--impl reference]

One step = one full solve to eps* (the hot path: every outer loop's matrix-powers
levels, Gram, O(s^2) control kernel and recovery, on the device).  Workload at
N=1: config c5 weak-scaled, a 256^3 7-point Poisson slab per GPU, sigma=12,
dynamic Newton basis, eps*=1e-10 (BASELINE.json configs[4]); the other configs
are parity-test cases (tests/), selectable with --config for reference.

value   CG iterations/s of the solve with b, x0 and A resident in HBM, device
        time (CUDA events on the solver stream) summed over the K timed solves.
e2e     the same metric through the public drop-in `adaptive_solve(problem, cfg,
        trace="fast")` with host buffers: H2D of b and x0 and D2H of x and the
        logs inside the timed region (wall clock, synchronised).
roofline  dominant kernel = K_mpk (matrix-powers levels): algorithmic bytes
        (12 nnz + 4 (n+1) per level of A, 16 n per generated
        column, + x, b on level 0) / its CUDA-event time, from one profiled solve
        after the timed region, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the CPU oracle port (oracle/sscg_oracle.py: the reference's
        numpy/scipy arithmetic, diagnostics off) timed on this host for a
        bounded sample (1 outer loop of the same problem), extrapolated to the
        solve's outer-loop count.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (problem key, scale override, sigma, basis, eps*, description)
    "c5w": ("c5w", None, 12, "newton", 1e-10,
            "c5 weak-scaled: 3D Poisson 7-pt 256^3 per GPU, sigma=12 Newton, eps*=1e-10"),
    "c3": ("c3", None, 10, "chebyshev", 1e-10, "c3: 3D Poisson 7-pt 128^3, sigma=10 Chebyshev, 1e-10"),
    "c4": ("c4", None, 10, "newton", 1e-8, "c4: 27-pt var-coef 192^3, sigma=10 Newton, 1e-8"),
    "c4j": ("c4j", None, 10, "newton", 1e-8,
            "c4 Jacobi-scaled (secondary run, SURVEY.md H6): 27-pt var-coef 192^3, sigma=10 Newton, 1e-8"),
    "c1": ("c1", None, 8, "newton", 1e-10, "c1: 2D Poisson 64^2, sigma=8 Newton, 1e-10"),
    "c2": ("c2", None, 10, "chebyshev", 1e-8, "c2: Strakos 1e4, sigma=10 Chebyshev, 1e-8"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


def kernel_name(sched):
    """The level kernel (levels >= 1) a matrix-powers schedule runs."""
    if sched["kind"] == "pattern":
        return {"tile march": "k_level_zt", "pair march": "k_level_zp", "march": "k_level_zm",
                "superset": "k_level_ss"}.get(sched.get("form"), "k_level_pat")
    return {"csr": "k_level_staged", "wavefront": "k_mpk_wave",
            "stencil values": "k_level_vs"}[sched["kind"]]


def a_bytes_per_level(n, nnz, sched):
    """Bytes of the operator one matrix-powers level must stream: CSR
    (12 nnz + 4 (n+1)) or, for a pattern-compressed plan, the
    1- or 2-byte row ids (the pattern table lives in shared memory)."""
    if sched and sched.get("kind") == "pattern":
        return (1 if sched["patterns"] <= 256 else 2) * n
    if sched and sched.get("kind") == "stencil values":  # 8 bytes per union slot and row
        return 8 * sched["slots"] * n
    return 12 * nnz + 4 * (n + 1)


def mpk_bytes_per_outer(n, nnz, sigma, mu_nonzero, sched=None):
    """Algorithmic bytes of the sigma matrix-powers levels of one outer loop
    (SURVEY.md 8(d)): A once per level, 16 n per generated column (+8 n for the
    Chebyshev two-back term), x and b on level 0 (true residual)."""
    s_a = a_bytes_per_level(n, nnz, sched)
    gen = 2 * sigma - 1
    two_back = (2 * sigma - 3) if mu_nonzero else 0  # columns with l >= 1
    return sigma * s_a + 16 * n * gen + 8 * n * two_back + 16 * n + 8 * n  # + r0 norm read


def outer_bytes(n, nnz, sigma, s_t, mu_nonzero, sched=None):
    return (mpk_bytes_per_outer(n, nnz, sigma, mu_nonzero, sched) + 8 * n * (2 * sigma + 1)
            + 8 * n * (2 * s_t + 1) + 8 * n + 24 * n)


def cpu_threads():
    """(threads the CPU path may use, description): OpenBLAS' pool (dgemm/dgemv
    of the Gram and recovery) -- scipy csr_matvec and numpy element-wise work
    run on one core."""
    try:
        import numpy
        import threadpoolctl
        numpy.ones(2) @ numpy.ones(2)
        pools = [(d["internal_api"], int(d["num_threads"]), d.get("version"))
                 for d in threadpoolctl.threadpool_info()]
    except Exception:
        pools = []
    blas = max([t for _, t, _ in pools] or [1])
    return blas, (f"os.cpu_count()={os.cpu_count()}; BLAS pools {pools}; scipy csr_matvec "
                  "and numpy element-wise work (most of the time) are single-threaded")


def cpu_sample(prob, cfg_kw, outer_count, total_iters):
    """Oracle port on this host: 1 outer loop of the same problem (bounded),
    per-outer time extrapolated to the solve's outer count."""
    from oracle import sscg_oracle as O
    t0 = time.perf_counter()
    O.solve_problem(prob, O.OracleConfig(max_outer=1, **cfg_kw), diagnostics=False)
    t1 = time.perf_counter() - t0
    est = t1 * (outer_count + 1)
    return total_iters / est, t1


def run_partitioned(args, rank, world):
    """One rank of the row-partitioned solve (torchrun, one process per GPU):
    gloo carries the setup plumbing (ghost requests, the NCCL id, the final
    max-over-ranks time), NCCL carries the per-outer-loop halo exchange and the
    one Gram allreduce inside the CUDA graph."""
    import ctypes as C
    import types

    import scipy.sparse as sp
    import torch
    import torch.distributed as dist

    from paper_1908_04081_b200 import AdaptiveConfig, _lib as L
    from paper_1908_04081_b200.adaptive import LogBuffers
    from paper_1908_04081_b200.dist import solve_partitioned
    from paper_1908_04081_b200.partition import Stencil7Rows

    key, scale, sigma, basis, eps, desc = CONFIGS[args.config]
    if key != "c5w":
        raise SystemExit("the partitioned bench runs the weak-scaled c5 slabs (--config c5w)")
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    local = int(os.environ.get("LOCAL_RANK", rank))
    edge = args.scale or 256
    nx = ny = edge
    nz = edge * world
    rows = Stencil7Rows(nx, ny, nz)
    n = rows.n
    t0 = time.perf_counter()
    xs = np.random.default_rng(0).uniform(-1.0, 1.0, n)  # same x* as problems.poisson3d
    from paper_1908_04081_b200.partition import slab_bounds
    bnd = slab_bounds(n, world)
    lo, hi = int(bnd[rank]), int(bnd[rank + 1])
    ip, cols, vals = rows.rows(np.arange(lo, hi))
    b_own = sp.csr_matrix((vals, cols, ip), shape=(hi - lo, n)) @ xs
    b_glob = np.zeros(n)
    b_glob[lo:hi] = b_own
    nb2 = torch.tensor([float(b_own @ b_own)], dtype=torch.float64)
    dist.all_reduce(nb2)
    lam = [2.0 - 2.0 * math.cos(math.pi / (m + 1)) for m in (nx, ny, nz)]
    lmax = sum(2.0 + 2.0 * math.cos(math.pi / (m + 1)) for m in (nx, ny, nz)) - 0.0
    scal = types.SimpleNamespace(a=types.SimpleNamespace(n_a=7), norm_a=lmax, norm_abs_a=lmax,
                                 kappa_a=lmax / sum(lam))
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
    lib = L.load()
    logs, ccfg = info["logs"], info["ccfg"]

    sched = plan.mpk_schedule(sigma)
    mpk_launches = len(sched["passes"])  # wavefront passes (or sigma level launches)

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
            launches += 3 + ol * (2 * sigma + 4)  # init 3; halo pack/unpack, params, Leja, levels, ...
    dev_ms = sum(ms_list) / len(ms_list)
    tmax = torch.tensor([dev_ms], dtype=torch.float64)
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    # end to end through the C ABI with host buffers: H2D of b and x0, D2H of x
    # and the logs inside the timed region, max over ranks
    b_loc, x0_loc = info["b"], info["x0"]
    x_host = np.empty(hi - lo)
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
    # roofline of the matrix-powers kernel on this rank's owned rows (SURVEY.md
    # 8(d): owned-row traffic only), from one profiled solve outside the timed
    # region (every rank runs it: the collectives are inside), max over ranks
    L.check(lib.sscg_set_profiling(plan.handle, 1))
    dev_solve()
    L.check(lib.sscg_set_profiling(plan.handle, 0))
    pms = np.zeros(5)
    pcnt = np.zeros(5, dtype=np.int64)
    L.check(lib.sscg_get_profile(plan.handle, L.dptr(pms), pcnt.ctypes.data_as(C.POINTER(C.c_int64))))
    mpk_ms_t = torch.tensor([float(pms[0])], dtype=torch.float64)
    dist.all_reduce(mpk_ms_t, op=dist.ReduceOp.MAX)
    L.check(lib.sscg_fetch(plan.handle, None, logs.s))
    # global true residual from the owned pieces (independent host SpMV)
    x_glob = torch.zeros(n, dtype=torch.float64)
    x_glob[lo:hi] = torch.from_numpy(xo)
    dist.all_reduce(x_glob)
    resid = sp.csr_matrix((vals, cols, ip), shape=(hi - lo, n)) @ x_glob.numpy() - b_own
    rr = torch.tensor([float(resid @ resid)], dtype=torch.float64)
    dist.all_reduce(rr)
    rel = math.sqrt(rr.item() / nb2.item())
    ms = tmax.item()
    value = world * total_iters / (ms / 1e3)
    if rank == 0:
        n_own = hi - lo
        line = {
            "metric": "cg_iterations_per_sec", "value": value, "unit": "iter/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic, seeded (np.random.default_rng(0)): x*~U[-1,1], b=A x*, x0=0",
            "config": {"workload": desc + f" (global {nx}x{ny}x{nz})", "n": n, "n_per_gpu": n_own,
                       "sigma": sigma, "basis": basis, "eps_star": eps,
                       "syncs_to_tol": total_outer, "total_iters": total_iters,
                       "converged": int(logs.s.status) == L.CONVERGED,
                       "final_true_rel_resid": rel, "trace": "fast",
                       "parallelism": f"dp{world} (row slabs, ghost depth {sigma}, one NCCL "
                                      "halo exchange + one NCCL allreduce per outer loop)",
                       "value_definition": "per-slab CG iterations/s summed over ranks = "
                                           "world x total_iters / max-over-ranks device time",
                       "global_iters_per_sec": total_iters / (ms / 1e3),
                       "setup_s": round(t_setup, 2),
                       "allreduce_per_outer": 1, "halo_exchanges_per_outer": 1},
            "e2e": {"value": world * total_iters / te.item(), "unit": "iter/s",
                    "h2d_bytes_per_step": int(8 * (len(b_loc) + len(x0_loc))),
                    "d2h_bytes_per_step": int(8 * (hi - lo) + logs.iters.nbytes),
                    "note": "sscg_solve per rank (host b, x0 -> x, logs), max over ranks"},
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        mu_nz = basis == "chebyshev"
        mpk_bytes = (total_outer + 1) * mpk_bytes_per_outer(n_own, 7 * n_own, sigma, mu_nz, sched)
        mpk_ms = mpk_ms_t.item()
        hbm_peak, peak_kind = peaks()
        ach = mpk_bytes / (mpk_ms / 1e3) / 1e9
        line["roofline"] = {
            "bound": "hbm", "kernel": kernel_name(sched) + " (owned rows; ghost-row levels are "
                                                          "redundant work, not counted)",
            "mpk_schedule": sched, "achieved": ach, "peak": hbm_peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": ach / hbm_peak, "traffic": None,
            "kernel_ms": {"mpk": pms[0], "gram": pms[1], "small": pms[2], "recovery": pms[3],
                          "other (halo, allreduce, Leja)": pms[4]}}
        print(json.dumps(line))
    dist.barrier()


def run_ours(args, rank, world):
    from paper_1908_04081_b200 import AdaptiveConfig, _lib as L, adaptive_solve, problems
    from paper_1908_04081_b200.adaptive import LogBuffers, make_config
    from paper_1908_04081_b200.kernels import _plan

    key, scale, sigma, basis, eps, desc = CONFIGS[args.config]
    if world > 1 or args.partitioned:
        return run_partitioned(args, rank, world)
    t0 = time.perf_counter()
    prob = problems.make_problem(key, scale=args.scale or scale, world=world)
    t_gen = time.perf_counter() - t0
    cfg_kw = dict(sigma=sigma, eps_star=eps, basis_kind=basis)
    cfg = AdaptiveConfig(**cfg_kw)
    n, nnz = prob.a.n, prob.a.nnz
    plan = _plan(prob.a, 0)
    lib = L.load()
    cfg, ccfg = make_config(cfg, prob, "fast")
    logs = LogBuffers(cfg)
    b = L.f64(prob.b)
    x0 = L.f64(prob.x0)
    L.check(lib.sscg_load(plan.handle, L.dptr(b), L.dptr(x0)))

    sched = plan.mpk_schedule(sigma)
    mpk_launches = len(sched["passes"])  # wavefront passes (or sigma level launches)

    def dev_solve():
        L.check(lib.sscg_run(plan.handle, ccfg, logs.s))
        return logs.s.device_ms, int(logs.s.outer_launched)

    for _ in range(args.warmup):
        dev_solve()
    # ---- timed region (device time, inputs resident in HBM)
    ms_list, launches = [], 0
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            ms, ol = dev_solve()
            ms_list.append(ms)
            # per outer: mpk passes, gram, small, params + (sigma-2) Leja, recovery
            launches += 2 + ol * (mpk_launches + sigma + 2)
    L.check(lib.sscg_fetch(plan.handle, None, logs.s))
    total_iters, total_outer = int(logs.s.total_iters), int(logs.s.total_outer)
    converged = int(logs.s.status) == L.CONVERGED
    x = np.empty(n)
    L.check(lib.sscg_fetch(plan.handle, L.dptr(x), logs.s))
    import scipy.sparse as sp
    a = prob.a
    rel = float(np.linalg.norm(prob.b - sp.csr_matrix((a.values, a.col_idx, a.row_ptr),
                                                      shape=(n, n)) @ x) / np.linalg.norm(prob.b))
    dev_ms = sum(ms_list) / len(ms_list)
    value = total_iters / (dev_ms / 1e3)

    # ---- profiled solve (per-kernel-class event times), outside the timed region
    L.check(lib.sscg_set_profiling(plan.handle, 1))
    dev_solve()
    L.check(lib.sscg_set_profiling(plan.handle, 0))
    import ctypes as C
    pms = np.zeros(5)
    pcnt = np.zeros(5, dtype=np.int64)
    L.check(lib.sscg_get_profile(plan.handle, L.dptr(pms),
                                 pcnt.ctypes.data_as(C.POINTER(C.c_int64))))
    ph = np.zeros(8, dtype=np.int64)
    L.check(lib.sscg_get_small_phases(plan.handle, ph.ctypes.data_as(C.POINTER(C.c_int64))))
    calls = max(1, int(ph[7]))
    names = ["classify", "gram_extract_c", "nested_conds", "select_truncate", "inner_loop",
             "next_params"]
    small_phases = {nm: round(float(ph[i]) / calls / 1965.0, 2) for i, nm in enumerate(names)}
    s_t = [int(v) for v in logs.rec_i[:total_outer, L.REC_STILDE]]
    mu_nz = basis == "chebyshev"
    active = total_outer + 1  # outer loops whose levels did real work
    mpk_bytes = active * mpk_bytes_per_outer(n, nnz, sigma, mu_nz, sched)
    mpk_ms = float(pms[0])
    hbm_peak, peak_kind = peaks()
    mpk_gbs = mpk_bytes / (mpk_ms / 1e3) / 1e9
    solve_bytes = sum(outer_bytes(n, nnz, sigma, st, mu_nz, sched) for st in s_t) + \
        mpk_bytes_per_outer(n, nnz, sigma, mu_nz, sched) + 8 * (2 * sigma + 1) * n
    solve_gbs = solve_bytes / (dev_ms / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            kname = kernel_name(sched)
            traffic = json.load(open(tpath)).get(args.config, {}).get(kname)
        except Exception:
            traffic = None

    # ---- end to end through the public API (host buffers)
    e2e_times = []
    for i in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        xe, tr, co = adaptive_solve(prob, AdaptiveConfig(**cfg_kw), trace="fast")
        e2e_times.append(time.perf_counter() - t0)
    e2e_value = tr.total_iters / (sum(e2e_times) / len(e2e_times))
    log_bytes = int(logs.iters.nbytes + logs.rec_i.nbytes + logs.rec_d.nbytes +
                    logs.conds.nbytes + 3 * logs.thetas.nbytes + logs.outer_true.nbytes)

    # ---- CPU baseline (oracle port, bounded sample)
    cpu = None
    if not args.no_cpu:
        cpu_v, t1 = cpu_sample(prob, cfg_kw, total_outer, total_iters)
        cores, tnote = cpu_threads()
        cpu = {"value": cpu_v, "unit": "iter/s", "cores": cores, "kind": "port",
               "sample": f"oracle/sscg_oracle.py (numpy/scipy, as the reference) on the same "
                         f"{n}-row problem, max_outer=1 took {t1:.2f}s; full solve extrapolated "
                         f"as (outer+1) x that = {t1 * (total_outer + 1):.1f}s for "
                         f"{total_iters} iterations",
               "threads_note": tnote}

    line = {
        "metric": "cg_iterations_per_sec", "value": value, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded (np.random.default_rng(0)): x*~U[-1,1], b=A x*, x0=0",
        "config": {"workload": desc, "n": n, "nnz": nnz, "sigma": sigma, "basis": basis,
                   "eps_star": eps, "syncs_to_tol": total_outer, "total_iters": total_iters,
                   "converged": converged, "final_true_rel_resid": rel,
                   "trace": "fast", "l2": "inputs larger than L2 (each vector "
                   f"{8 * n / 1e6:.0f} MB, Y {8 * n * (2 * sigma + 1) / 1e9:.2f} GB)",
                   "problem_gen_s": round(t_gen, 2), "parallelism": f"dp{world} (row slabs)"},
        "hbm": {"solve_gbs": solve_gbs, "frac_of_measured": solve_gbs / hbm_peak,
                "frac_of_8tbs": solve_gbs / 8000.0, "algorithmic_bytes_per_solve": solve_bytes},
        "roofline": {"bound": "hbm",
                     "kernel": kernel_name(sched) + " " + {
                         "wavefront": "(wavefront matrix powers + recurrence)",
                         "pattern": "(pattern-compressed matrix powers + recurrence, "
                                    f"{sched.get('form')} form)",
                         "csr": "(CSR matrix powers + recurrence)",
                         "stencil values": "(value-stream stencil matrix powers + recurrence)"}[sched["kind"]],
                     "a_bytes_per_level": a_bytes_per_level(n, nnz, sched),
                     "a_bytes_per_level_csr": a_bytes_per_level(n, nnz, None),
                     "mpk_schedule": sched,
                     "achieved": mpk_gbs, "peak": hbm_peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": mpk_gbs / hbm_peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": mpk_bytes / max(1, active * mpk_launches),
                     "avg_launch_ms": mpk_ms / max(1, active * mpk_launches),
                     "kernel_ms": {"mpk": pms[0], "gram": pms[1], "small": pms[2],
                                   "recovery": pms[3], "other": pms[4]},
                     "small_phases_us_per_call": small_phases,
                     "kernel_launches": {"mpk": int(pcnt[0]), "gram": int(pcnt[1]),
                                         "small": int(pcnt[2]), "recovery": int(pcnt[3])},
                     "share_of_step": {"mpk": pms[0] / max(pms.sum(), 1e-9),
                                       "gram": pms[1] / max(pms.sum(), 1e-9),
                                       "small": pms[2] / max(pms.sum(), 1e-9),
                                       "recovery": pms[3] / max(pms.sum(), 1e-9)}},
        "e2e": {"value": e2e_value, "unit": "iter/s", "h2d_bytes_per_step": 16 * n,
                "d2h_bytes_per_step": 8 * n + log_bytes,
                "note": "adaptive_solve(problem, cfg, trace='fast'); CSR plan cached on the "
                        "matrix like SparseMatrix._csr"},
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line))


def run_reference(args, rank, world):
    """The reference's CPU path (oracle port of its numpy/scipy arithmetic) on
    this host, same config / metric; rank 0 only."""
    if rank != 0:
        return
    from paper_1908_04081_b200 import problems
    from oracle import sscg_oracle as O
    key, scale, sigma, basis, eps, desc = CONFIGS[args.config]
    # One step = one outer loop of the CPU port on ONE slab-sized problem (for
    # c5w the 256^3 slab every rank owns): the CPU cost of an outer loop of the
    # global 256x256x(256N) problem is N times that (linear in rows), and the
    # metric, like ours, counts per-slab iterations summed over the N slabs:
    # value = N * total_N / ((outer_N + 1) * N * t_slab) = total_N / ((outer_N + 1) t_slab).
    prob = problems.make_problem(key, scale=args.scale or scale, world=1)
    cfg_kw = dict(sigma=sigma, eps_star=eps, basis_kind=basis)
    # outer / total counts of the full global solve (GPU-measured, parity-tested:
    # tools/measure_counts.py)
    counts = {}
    cpath = os.path.join(ROOT, "profiles", "counts.json")
    if os.path.exists(cpath):
        counts = json.load(open(cpath)).get(f"{args.config}_w{world}", {})
    outer = counts.get("outer", 90)
    total = counts.get("total", 1000)
    small = problems.make_problem(key, scale=32 if key.startswith("c5") else None, world=1) \
        if key in ("c5w", "c5", "c3", "c4") else prob
    for _ in range(args.warmup):  # warm imports / allocator on a small instance
        O.solve_problem(small, O.OracleConfig(max_outer=1, **cfg_kw), diagnostics=False)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.solve_problem(prob, O.OracleConfig(max_outer=1, **cfg_kw), diagnostics=False)
        times.append(time.perf_counter() - t0)
    t1 = sum(times) / len(times)
    value = total / (t1 * (outer + 1))
    line = {
        "metric": "cg_iterations_per_sec", "value": value, "unit": "iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t1 * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded", "impl": "reference",
        "config": {"workload": desc, "n": prob.a.n, "nnz": prob.a.nnz},
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": cpu_threads()[0], "kind": "port",
                         "threads_note": cpu_threads()[1],
                         "sample": f"each step = 1 outer loop of the oracle port on one "
                                   f"{prob.a.n}-row slab ({t1:.2f}s); the global N={world} "
                                   f"solve takes {outer}+1 outer loops of N x that; value = "
                                   f"N x {total} iters / its time (per-slab iterations summed, "
                                   "as the GPU arm); counts from profiles/counts.json"},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def run_solver_compare(args):
    """--solver sstep|hscg (one GPU, informational, not the driver's headline):
    the same workload through fixed s-step CG (s = sigma, the config's basis
    with Ritz-free spectral bounds of the stencil) or Hestenes-Stiefel CG
    (classic.py: true residual every iteration), device time per solve.
    `syncs_to_tol` counts the global reductions a multi-GPU run would need:
    one per outer loop for s-step, two per iteration for HSCG (p.Ap, r.r)."""
    from paper_1908_04081_b200 import _lib as L, problems
    from paper_1908_04081_b200.kernels import _plan
    from paper_1908_04081_b200.sstep import sstep_solve
    key, scale, sigma, basis, eps, desc = CONFIGS[args.config]
    prob = problems.make_problem(key, scale=args.scale or scale)
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
                L.check(lib.sscg_hscg(plan.handle, L.dptr(b), L.dptr(x0), float(eps), -1, None,
                                      logs))
                dev, it, sy = logs.device_ms, int(logs.total_iters), 2 * int(logs.total_iters)
                status = {L.CONVERGED: "converged", L.STAGNATED: "stagnated",
                          L.DIVERGED: "diverged"}.get(int(logs.status), "max_iters")
            else:
                nx = round(n ** (1.0 / 3.0)) if key in ("c3", "c5") else None
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
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, seeded", "impl": "ours", "solver": args.solver,
        "config": {"workload": desc, "n": n, "total_iters": iters, "syncs_to_tol": syncs,
                   "status": status, "eps_star": eps,
                   **({"s": args.s or sigma} if args.solver == "sstep" else {})},
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
    ap.add_argument("--partitioned", action="store_true",
                    help="use the row-partitioned NCCL path even at one GPU")
    ap.add_argument("--solver", default="adaptive", choices=["adaptive", "sstep", "hscg"],
                    help="adaptive (the headline); sstep / hscg: one-GPU comparison lines")
    ap.add_argument("--s", type=int, default=None, help="fixed s for --solver sstep (default sigma)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.solver != "adaptive":
        run_solver_compare(args)
    else:
        run_ours(args, rank, world)


if __name__ == "__main__":
    main()
