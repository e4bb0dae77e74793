"""Small solves through every kernel family, as a compute-sanitizer target:
    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_target.py
plane march (register and TMA forms), superset / table-walk patterns, value
stream, CSR (staged and direct), Gram / recovery / K_small / Leja, full-trace
diagnostics, fixed s-step, HSCG (both modes), the virtual group (halo and
fixed-order reductions), the unit entry points."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1908_04081_b200 import (AdaptiveConfig, adaptive_solve, hscg_solve, kernels,  # noqa: E402
                                   problems, sstep_solve)
from paper_1908_04081_b200.dist import VirtualGroup  # noqa: E402
from paper_1908_04081_b200.partition import CsrRows, Varcoef27Rows  # noqa: E402


def env(**kw):
    for k in ("SSCG_PATTERN", "SSCG_TM", "SSCG_ZM", "SSCG_PAT_SS", "SSCG_STAGE_MAX_KB"):
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in kw.items()})


def run(tag, prob, **cfg):
    mo = cfg.pop("max_outer", 6)
    trace = cfg.pop("trace", "fast")
    x, tr, co = adaptive_solve(prob, AdaptiveConfig(max_outer=mo, **cfg), trace=trace)
    print(f"{tag}: outer {tr.total_outer} iters {tr.total_iters}", flush=True)


newton = dict(sigma=8, eps_star=1e-10, basis_kind="newton")
cheb = dict(sigma=6, eps_star=1e-10, basis_kind="chebyshev")
env()
run("tma march newton", problems.make_problem("c5", scale=32), **newton)
run("tma march cheb", problems.make_problem("c3", scale=32), **cheb)
env(SSCG_TM=0)
run("register march", problems.make_problem("c5", scale=32), **newton)
env()
run("superset (2-D)", problems.make_problem("c1", scale=32), **newton)
run("full trace", problems.make_problem("c1", scale=32), trace="full", **newton)
env(SSCG_PAT_SS=0)
run("table walk", problems.make_problem("c1", scale=32), **newton)
env()
run("value stream", problems.make_problem("c4j", scale=10), **newton)
env(SSCG_PATTERN=0)
run("csr staged", problems.make_problem("c5", scale=16), **newton)
env(SSCG_PATTERN=0, SSCG_STAGE_MAX_KB=0)
run("csr direct", problems.make_problem("c5", scale=16), **newton)
env()
p = problems.make_problem("c5", scale=16)
sstep_solve(p, 4, 1e-10, basis_kind="newton", spectral_bounds=(0.1, 11.9), max_outer=4, trace="fast")
hscg_solve(p, 1e-10, max_iters=40)
hscg_solve(p, 1e-10, max_iters=40, mode="production")
print("sstep / hscg ok", flush=True)
g = VirtualGroup(CsrRows.of(p.a), 2, depth=8)
g.solve(p, AdaptiveConfig(max_outer=5, **newton))
g.hscg(p, 1e-10, max_iters=40)
VirtualGroup(Varcoef27Rows(10, jacobi=True), 2, depth=8).solve(
    problems.make_problem("c4j", scale=10), AdaptiveConfig(max_outer=4, **newton))
print("virtual groups ok", flush=True)
rng = np.random.default_rng(0)
y = rng.standard_normal((300, 9))
g_ = kernels.gram(y)
kernels.nested_basis_conds(g_, 4)
kernels.leja_points(0.1, 4.0, 6)
kernels.spmv(p.a, rng.standard_normal(p.a.n))
print("unit entries ok", flush=True)
from paper_1908_04081_b200 import _lib as L  # noqa: E402
lib = L.load()
if hasattr(lib, "sscg_debug_mbar"):  # checked side build: lost-transaction record
    import ctypes as C
    buf = (C.c_uint * 8)()
    rc = lib.sscg_debug_mbar(buf)
    print(f"mbarrier waits timed out: {buf[0]} (rc {rc})", flush=True)
print("library:", L.LIB_PATH)
