"""Diagnostics: run golden cases on the GPU and save full traces to gpurun_out/."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import cfg_of, golden, golden_problem, problem_from_arrays  # noqa
from paper_1908_04081_b200 import AdaptiveConfig, adaptive_solve, problems  # noqa

cases = {
    "solve_c2_cheb": lambda r: problems.make_problem("c2"),
    "solve_c2_newton": lambda r: problems.make_problem("c2"),
    "solve_c4p": lambda r: problem_from_arrays(r, "in_"),
    "solve_spd50_newton": lambda r: problem_from_arrays(r, "in_"),
    "solve_nos1_chebyshev_kappa-estimate": lambda r: golden_problem("problem_nos1"),
}
os.makedirs("gpurun_out", exist_ok=True)
for name, mk in cases.items():
    ref = golden(name)
    prob = mk(ref)
    info = {}
    x, tr, co = adaptive_solve(prob, AdaptiveConfig(**cfg_of(ref)), info=info)
    lg = info["logs"]
    nrec = len(tr.outer_records)
    np.savez_compressed(f"gpurun_out/trace_{name}.npz", alphas=np.array(co.alphas),
                        betas=np.array(co.betas), lmin=np.array(tr.lambda_min),
                        lmax=np.array(tr.lambda_max), psi=np.array(tr.psi),
                        s_schedule=np.array(tr.s_schedule), rec_i=lg.rec_i[:nrec],
                        rec_d=lg.rec_d[:nrec], conds=lg.conds[:nrec], thetas=lg.thetas[:nrec],
                        x=x, true_resid=np.array(tr.true_resid))
    print(name, tr.total_outer, tr.total_iters, tr.converged)
