"""CPU tier for bench.py's launcher and bookkeeping (no GPU): --gpus N without
torchrun re-launches N ranks; a WORLD_SIZE that disagrees with --gpus is an
error; the algorithmic-byte formulas; the counts the
reference arm extrapolates with come from the reference's own runs."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(args, env_extra=None, drop=("WORLD_SIZE", "RANK", "LOCAL_RANK")):
    env = {k: v for k, v in os.environ.items() if k not in drop}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                          capture_output=True, text=True, timeout=300)


def test_gpus2_without_torchrun_spawns_two_ranks():
    p = _run(["--gpus", "2", "--check-launch"])
    assert p.returncode == 0, p.stderr[-2000:]
    got = sorted(json.loads(l)["rank"] for l in p.stdout.splitlines() if l.startswith("{"))
    worlds = {json.loads(l)["world"] for l in p.stdout.splitlines() if l.startswith("{")}
    assert got == [0, 1] and worlds == {2}, p.stdout


def test_world_size_must_match_gpus():
    p = _run(["--gpus", "2", "--check-launch"], {"WORLD_SIZE": "1", "RANK": "0"})
    assert p.returncode != 0 and "WORLD_SIZE" in (p.stderr + p.stdout)
    p = _run(["--gpus", "1", "--check-launch"])
    assert p.returncode == 0 and json.loads(p.stdout.strip()) == {"rank": 0, "world": 1}


def test_algorithmic_bytes():
    n, nnz = 1000, 6800
    march = {"kind": "pattern", "patterns": 27, "form": "march"}
    # Newton sigma = 12: A ids once per level (1 B/row), 23 generated columns
    # at 16 n, x and b on level 0
    assert bench.mpk_bytes_per_outer(n, nnz, 12, False, march) == 12 * n + 16 * n * 23 + 16 * n
    # Chebyshev adds the two-back read on levels >= 1 (2 sigma - 3 columns)
    assert bench.mpk_bytes_per_outer(n, nnz, 10, True, None) == \
        10 * (12 * nnz + 4 * (n + 1)) + 16 * n * 19 + 8 * n * 17 + 16 * n
    vs = {"kind": "stencil values", "slots": 27}
    assert bench.a_bytes_per_level(n, nnz, vs) == 8 * 27 * n


def test_same_config_in_both_arms():
    import argparse
    a = argparse.Namespace(config="c5w", scale=None, partitioned=False)
    assert bench.workload_config(a, 1) == bench.workload_config(a, 1)
    assert "solve" not in bench.workload_config(a, 1)


def test_reference_counts_from_the_reference_runs():
    got = bench.reference_counts("c3", 1)
    assert got is not None and got[:2] == (46, 425) and "reference" in got[2]
    if os.path.exists(os.path.join(ROOT, "tests", "golden", "full_c5w.npz")):
        assert "reference" in bench.reference_counts("c5w", 1)[2]
    assert bench.reference_counts("c5w", 8)[0] > 0  # GPU-measured global counts
