"""bench.py keeps its contract on every BASELINE config (B200): one JSON line
with the driver's keys, `roofline`, `e2e`, `cpu_baseline` and a `verify`
object whose check passed (zeta against NPB's official value, the device
outputs against the oracle)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline",
        "verify", "marshal_first_call")


def run_bench(*args, timeout=1200):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def check_line(line, config, steps, warmup):
    for k in KEYS:
        if config == "stencil" and k == "marshal_first_call":
            continue
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == steps and line["warmup"] == warmup and line["value"] > 0
    assert line["config"]["name"] == config
    rf = line["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1.3 and rf["peak"] > 0
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0 and "sm_mhz" in line["clocks"]
    cb = line["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    assert line["verify"]["verified"] is True, line["verify"]


@pytest.mark.gpu
def test_bench_npb_a_line():
    line = run_bench("--config", "npb_a", "--steps", "4", "--warmup", "3", "--spmv-reps", "20")
    check_line(line, "npb_a", 4, 3)
    for k in ("e2e", "e2e_lazy_pageable", "e2e_eager", "e2e_default"):
        assert line[k]["zeta_verified"] is True, (k, line[k])
    assert line["e2e_default"]["memory"] == "pageable" and line["e2e_default"]["writeback"] == "eager"
    assert line["marshal_first_call"]["s"] > 0


@pytest.mark.gpu
def test_bench_parboil_line():
    line = run_bench("--config", "parboil", "--steps", "5", "--warmup", "3", "--spmv-reps", "20")
    check_line(line, "parboil", 5, 3)


@pytest.mark.gpu
def test_bench_kron_line():
    line = run_bench("--config", "kron", "--steps", "4", "--warmup", "3", "--spmv-reps", "20")
    check_line(line, "kron", 4, 3)


@pytest.mark.gpu
def test_bench_stencil_line():
    line = run_bench("--config", "stencil", "--steps", "3", "--warmup", "3")
    check_line(line, "stencil", 3, 3)
    assert line["verify"]["spmv_within_1e-12"] is True


@pytest.mark.gpu
def test_bench_reference_arm_same_workload():
    ref = run_bench("--impl", "reference", "--config", "npb_a", "--steps", "1", "--warmup", "0")
    assert ref["impl"] == "reference" and ref["value"] > 0
    assert ref["cpu_baseline"]["kind"] in ("reference", "port") and ref["e2e"]["h2d_bytes_per_step"] == 0
    if ref["cpu_baseline"]["kind"] == "reference":
        assert ref["config"]["npb_zeta_verified"] is True
