"""Shared fixtures.  `-m gpu` tests need a B200 and the built libsscg.so; the
rest run on the CPU (oracle vs golden vectors, host logic, C-ABI symbols)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsscg.so")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.fail(f"golden fixture {name} missing (run oracle/make_golden.py)")
    return np.load(path, allow_pickle=False)


def golden_problem(name):
    """A ProblemInstance from a stored problem_* fixture (nos1 / 494bus)."""
    from paper_1908_04081_b200.types import ProblemInstance, SparseMatrix
    d = golden(name)
    return problem_from_arrays(d)


def problem_from_arrays(d, prefix=""):
    from paper_1908_04081_b200.types import ProblemInstance, SparseMatrix
    g = lambda k: d[prefix + k]  # noqa: E731
    a = SparseMatrix(n=int(g("n")), row_ptr=g("row_ptr"), col_idx=g("col_idx"),
                     values=g("values"), n_a=int(g("n_a")))
    nrm = g("norms")
    return ProblemInstance(a=a, b=g("b"), x0=g("x0"), norm_a=float(nrm[0]),
                           norm_abs_a=float(nrm[1]), kappa_a=float(nrm[2]))


def cfg_of(d):
    import json
    return json.loads(str(d["cfg"]))


@pytest.fixture(scope="session")
def gpu_ready():
    """Build (if needed) and load the CUDA library; skip-free: a GPU test with
    no device FAILS, so a silent CPU path can never pass the gpu tier."""
    from paper_1908_04081_b200 import _lib, build
    build.build()
    _lib.load()
    n = _lib.device_count()
    assert n >= 1, "gpu-marked test ran without a CUDA device"
    return n
