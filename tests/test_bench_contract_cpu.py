# SPDX-License-Identifier: Apache-2.0
"""The bench.py JSON contract: the reference arm run here on the CPU (a tiny sample), and the
committed GPU bench line of the last measurement round checked key by key."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

import oracle

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _metric() -> str:
    return json.loads((ROOT / "BASELINE.json").read_text())["metric"]


def test_reference_arm_json_line():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "3", "--ref-ctx", "256"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT)
    assert res.returncode == 0, res.stderr
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["metric"] == _metric() and d["unit"] == "us/step" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["warmup"] >= 3 and d["steps"] == 2
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"] == "mla_decode_b16_ctx64k_h16_per_gpu"


def test_committed_bench_line_keeps_the_contract():
    lines = sorted((ROOT / "profiles").glob("r*/bench_r*.json"))
    lines = [p for p in lines if "_ref_" not in p.name]
    assert lines, "no committed bench line"
    d = json.loads(lines[-1].read_text())  # the latest round
    assert BASE_KEYS <= set(d)
    assert d["metric"] == _metric() and d["unit"] == "us/step" and d["higher_is_better"] is False
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["data"] == "synthetic" and d["dtype"] == "bf16"
    assert abs(d["ms_per_step"] * 1e3 - d["value"]) < 1e-6 * d["value"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0.9 < r["traffic"] / d["throughput"]["algorithmic_bytes_per_step_per_gpu"] < 1.1
    c = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(c) and c["kind"] in ("reference", "port")
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e) and e["h2d_bytes_per_step"] > 0
    assert e["value"] > d["value"]  # host buffers cross PCIe every step
    assert d["gpu_launches"] >= 2 * d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(d["clocks"]["reasons"])
