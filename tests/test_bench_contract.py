"""bench.py keeps the driver's JSON contract (one line, required keys and types).

CPU: the reference arm (--impl reference times the oracle) on the small C1 workload.
GPU: the product arm on C1 with two steps.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "1"])
    assert d["impl"] == "reference"
    assert BASE_KEYS <= set(d)
    assert d["config"]["workload"] == "C1" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_product_arm_contract():
    d = _run(["--config", "C1", "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--no-variants"])
    assert BASE_KEYS - {"cpu_baseline"} <= set(d)
    assert {"roofline", "gpu_launches", "clocks", "e2e_cg"} <= set(d)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert d["gpu_launches"] > 0 and d["value"] > 0 and d["ms_per_step"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == d["e2e"]["d2h_bytes_per_step"] == 8 * 33 * 33
    assert d["dtype"] == "f64" and d["n_gpus"] == 1


@pytest.mark.gpu
def test_product_arm_multirank_code_path():
    """--dist: the bench's multi-rank branch (process group, NCCL id broadcast, the library's
    NCCL communicator, exchange + all-reduced CG, max over ranks) through a 1-rank group."""
    d = _run(["--config", "C1", "--steps", "2", "--warmup", "1", "--no-cpu-baseline", "--no-variants", "--dist"])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["ms_per_step"] > 0
    assert d["gpu_launches"] > 0 and 0 < d["roofline"]["frac"]


def test_gpus_flag_without_enough_devices_fails_clearly():
    """--gpus N outside torchrun self-launches N ranks, or exits non-zero with a clear message
    when fewer than N GPUs are visible (never silently times one GPU)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64", "--config", "C1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0
    assert "needs 64 visible GPUs" in r.stderr
    env = dict(os.environ, WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--config", "C1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr
