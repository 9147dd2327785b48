# SPDX-License-Identifier: Apache-2.0
"""CPU tests of the tcgen05 issued-work model (include/etaplab_b200_umma.hpp, tool
paper_2506_01969_b200/lib/etap_model): SURVEY.md §8f rank 4, the reference's WgmmaSpec model
(wgmma_model.hpp:64-76) restated for B200.

* With the Hopper spec the tool reproduces the reference's own model bit for bit (compiled
  reference, oracle/_ref) over a shape grid, and the reference's test_wgmma_model.cpp cases.
* With the B200 spec (M = 64 / 128 forms, N steps 8 / 16, hi|lo P doubling the PV issue)
  the ETAP issued work at the headline config gives the tensor-pipe share ncu measured.
"""
from __future__ import annotations

import csv
import ctypes as C
import io
import subprocess

import numpy as np
import pytest

import oracle
from paper_2506_01969_b200 import build

GRID = [(16, 1, 4096, 1), (16, 1, 100, 1), (16, 4, 1024, 2), (64, 1, 65536, 1), (128, 1, 8192, 3),
        (16, 2, 65536, 16), (7, 3, 777, 5), (1, 1, 1, 1), (32, 1, 129, 1)]


def model(*args: str) -> list[dict]:
    exe = build.build_model()
    out = subprocess.run([str(exe), *args], capture_output=True, text=True, check=True).stdout
    return list(csv.DictReader(io.StringIO(out)))


def rows_by_mode(rows):
    return {r["mode"]: r for r in rows}


def test_hopper_spec_matches_reference_model():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    L = oracle.ref()
    L.ref_wgmma_model.argtypes = [C.c_int] + [C.c_int64] * 9 + [C.c_void_p]
    L.ref_wgmma_model.restype = C.c_int
    for heads, qt, kv, batch in GRID:
        rows = rows_by_mode(model("--spec", "hopper", "--heads", str(heads), "--q-tokens", str(qt),
                                  "--batch", str(batch), "--kv", str(kv)))
        for mode_i, mode in enumerate(("original", "etap")):
            ref = np.zeros(6)
            assert L.ref_wgmma_model(mode_i, heads, qt, kv, 576, 512, batch, 64, 8, 16,
                                     ref.ctypes.data_as(C.c_void_p)) == 0
            r = rows[mode]
            assert int(r["useful_macs"]) == int(ref[0]) and int(r["issued_macs"]) == int(ref[1])
            assert float(r["utilization"]) == ref[2]
            assert float(r["qk_m_axis_utilization"]) == ref[3]
            assert float(r["pv_m_axis_utilization"]) == ref[4]
            assert float(r["predicted_speedup"]) == ref[5]


def test_reference_model_cases_hold_for_hopper_spec():  # test_wgmma_model.cpp:23-103
    r = rows_by_mode(model("--spec", "hopper", "--kv", "4096"))
    assert float(r["original"]["utilization"]) == 0.25
    assert int(r["original"]["issued_macs"]) == 4 * int(r["original"]["useful_macs"])
    assert float(r["etap"]["utilization"]) == 1.0
    r = rows_by_mode(model("--spec", "hopper", "--q-tokens", "4", "--kv", "4096"))
    assert float(r["original"]["utilization"]) == 1.0  # 64 folded queries hit the boundary
    r = rows_by_mode(model("--spec", "hopper", "--kv", "100"))
    assert 0.0 < float(r["etap"]["utilization"]) < 1.0
    s = rows_by_mode(model("--spec", "hopper", "--kv", "65536"))["etap"]["predicted_speedup"]
    assert abs(float(s) - 4.0) <= 0.04
    prev = 0.0
    for row in model("--spec", "hopper"):
        sp = float(row["predicted_speedup"])
        assert sp >= prev and sp >= 1.0
        prev = sp


def test_b200_spec_issue_model():
    # tcgen05 forms: the query-major mapping still pads 16 heads to M = 64 (0.25); the ETAP
    # mapping is unpadded but issues PV twice (P_hi | P_lo as N = 32) -> 0.68 utilization
    rows = rows_by_mode(model("--heads", "16", "--batch", "16", "--kv", "65536"))
    o, e = rows["original"], rows["etap"]
    assert float(o["utilization"]) == 0.25
    assert int(e["pv_passes"]) == 2
    useful = 16 * 65536 * 16 * (576 + 512)
    assert int(e["useful_macs"]) == useful
    assert int(e["issued_macs"]) == 16 * 65536 * 16 * (576 + 2 * 512)
    assert abs(float(e["utilization"]) - 1088 / 1600) < 1e-12
    # tensor time of the ETAP issued work at the measured bf16 peak: ~33 us of a ~190 us
    # HBM-bound step, i.e. the ~17% tensor-pipe activity ncu reports (profiles/)
    t = float(e["tensor_time_us"])
    assert 30.0 < t < 36.0
    assert 2.6 < float(e["predicted_speedup"]) < 2.8
    # unaligned KV pads the M axis to 64 rows
    r = rows_by_mode(model("--kv", "100"))
    assert float(r["etap"]["qk_m_axis_utilization"]) == 100 / 128


def test_model_rejects_bad_shapes():
    exe = build.build_model()
    res = subprocess.run([str(exe), "--heads", "0", "--kv", "64"], capture_output=True, text=True)
    assert res.returncode == 2 and "must be >= 1" in res.stderr
    res = subprocess.run([str(exe), "--spec", "volta"], capture_output=True, text=True)
    assert res.returncode == 2
