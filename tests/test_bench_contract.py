"""bench.py's JSON line: the keys the driver and the judge read (contract in the task)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(*args, timeout=600):
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    """--impl reference times the CPU oracle (the tier's reference arm) on a bounded sample."""
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "3")
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("EDM n=65536")


@pytest.mark.gpu
def test_bench_line_edm():
    d = _run("--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu", "--only-edm")
    assert BASE_KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["unit"] == "cells/s" and d["config"]["cells_per_step"] == 65536 * 65537 // 2
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys()
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.5 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["gpu_launches"] == 3                      # one edm_kernel launch per step
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()


@pytest.mark.gpu
def test_bench_two_ranks_one_device():
    """The N-rank bench path (omega-range split, count / energy all-reduce, CA halo exchange,
    fused P2P halo stores) run as 2 torchrun ranks on one GPU over gloo: one JSON line from
    rank 0, n_gpus = 2, the halo exchange timed separately."""
    env = dict(os.environ, TRI_BENCH_BACKEND="gloo", TRI_BENCH_ONE_DEVICE="1")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout[-2000:]
    d = json.loads(lines[0])
    assert BASE_KEYS <= d.keys() and d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"] == "omega-range x2"
    ca = d["workloads"]["ca"]
    assert ca["halo_exchange_ms"] > 0 and ca["compute_only_ms"] > 0 and ca["p2p_ms"] > 0
    assert d["workloads"]["collide"]["tc_count"] == 123650
