"""The driver's bench.py contract on CPU: the reference arm prints exactly one JSON line with the
metric, the CPU-baseline description and a zero-copy e2e block (the GPU arm is exercised on the
B200 by the driver; its keys are checked there)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_one_json_line():
    env = dict(os.environ, NUMBA_NUM_THREADS="2")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--ref-tokens", "20000"], capture_output=True, text=True, cwd=ROOT, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["metric"].startswith("token-layers scored/sec") and d["unit"] == "token-layers*placements/s"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["value_1thread"] > 0
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("config2")


import pytest  # noqa: E402


@pytest.mark.gpu
def test_gpu_arm_contract_keys():
    """One short GPU-arm run (1M tokens): the JSON line carries the contract keys, the roofline and
    clock objects, a positive launch count and a histogram that matched the setup pass."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3", "--tokens", "1000000",
                          "--e2e-steps", "1", "--cpu-tokens", "20000"], capture_output=True, text=True, cwd=ROOT,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["gpu_launches"] >= 3
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.2 and r["peak"] > 0 and r["unit"] == "GB/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 1_000_000 * 58 * 8 and d["e2e"]["value"] > 0
    assert d["clocks"]["samples"] >= 1 and d["cpu_baseline"]["cores"] >= 1
