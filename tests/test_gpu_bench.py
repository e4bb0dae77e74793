"""GPU tier: bench.py's own arms at a small scale (wiring, JSON contract),
so a broken bench path fails the tests rather than the round-end run."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    return json.loads(line)


def test_bench_default_arm_small(gpu_ready):
    d = _bench("--scale", "48", "--steps", "1", "--warmup", "1")
    assert REQUIRED <= set(d) and d["value"] > 0 and d["solve"]["converged"]
    for key in ("roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in d
    assert d["roofline"]["schedule"]["kind"] == "pattern"
    assert d["e2e"]["first_call_s"] > 0 and len(d["secondary"]) == 2
    assert d["secondary"][0]["roofline"]["schedule"]["kind"] == "csr"
    assert d["secondary"][1]["roofline"]["schedule"]["kind"] == "stencil values"


@pytest.mark.parametrize("config,scale", [("c5w", 48), ("c4", 24), ("c4j", 24), ("c5", 40)])
def test_bench_partitioned_arm_small(gpu_ready, config, scale):
    d = _bench("--partitioned", "--config", config, "--scale", str(scale), "--steps", "1",
               "--warmup", "1", "--no-cpu")
    assert REQUIRED <= set(d) and d["value"] > 0
    assert d["solve"]["collectives"]["allreduce_per_outer"] == 1
    assert d["solve"]["ranks_agree"] and d["solve"]["converged"] or config == "c4"
    kind = "stencil values" if config.startswith("c4") else "pattern"
    assert d["roofline"]["schedule"]["kind"] == kind


@pytest.mark.parametrize("solver", ["hscg", "sstep"])
def test_bench_solver_lines_small(gpu_ready, solver):
    d = _bench("--solver", solver, "--scale", "48", "--steps", "1", "--warmup", "1",
               *(["--s", "6"] if solver == "sstep" else []))
    assert d["solver"] == solver and d["solve"]["status"] == "converged"


def test_bench_reference_arm_small(gpu_ready):
    d = _bench("--impl", "reference", "--config", "c3", "--scale", "32", "--steps", "1",
               "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    ours = _bench("--config", "c3", "--scale", "32", "--steps", "1", "--warmup", "1", "--no-cpu")
    assert ours["config"] == d["config"]  # the driver's same_config check


def test_bench_partitioned_hscg_line(gpu_ready):
    """The distributed-HSCG comparison line (§8(f)2): two allreduces and one
    halo exchange per iteration, measured from its captured graph."""
    d = _bench("--solver", "hscg", "--partitioned", "--scale", "32", "--steps", "1", "--warmup",
               "1")
    assert d["solver"] == "hscg" and d["solve"]["status"] == "converged"
    assert d["solve"]["collectives"]["allreduce_per_outer"] == 2
    assert d["solve"]["collectives"]["halo_exchanges_per_outer"] == 1
