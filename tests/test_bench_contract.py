"""bench.py's output contract: stdout carries exactly one JSON line with the keys the driver
reads (metric, value, unit, n_gpus, steps, warmup, ms_per_step, higher_is_better, scaling,
vs_baseline, dtype, data, config; the GPU arm adds e2e, gpu_launches, roofline, clocks).
Small configurations only (config 2)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=600):
    env = dict(os.environ, NCCL_DEBUG="WARN")  # NCCL's banner must not reach stdout
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.splitlines()
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_one_json_line():
    d = run_bench("--impl", "reference", "--config", "2", "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.2")
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["cpu_model"]
    # the GPU arm builds its config with the same function (same_config for the driver)
    sys.path.insert(0, ROOT)
    import argparse
    import bench
    args = argparse.Namespace(config=2, K=0, tick_ns=0.0, order4=False)
    p, K, _, m, S = bench.workload(args, 1)
    assert d["config"] == json.loads(json.dumps(bench.config_dict(args, p, K, m, S, 1)))
    # ms_per_step is the measured wall time of the step (not an extrapolation to K)
    assert 0 < d["ms_per_step"] < 60_000


@pytest.mark.gpu
def test_gpu_arm_one_json_line():
    d = run_bench("--config", "2", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert BASE_KEYS <= set(d) and d.get("impl", "dflop") != "reference"
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["config"]["workload"].startswith("cfg2")
    r = d["roofline"]
    assert r["bound"] == "issue" and 0 < r["frac"] <= 1 and r["achieved"] > 0 and r["peak"] > 0
    assert 0 < r["frac_alu_pipe"] <= 1 and "int_peaks.json" in r["peak_note"]
    assert d["cpu_baseline"] if "cpu_baseline" in d else True
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
