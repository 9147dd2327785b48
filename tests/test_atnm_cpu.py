# SPDX-License-Identifier: Apache-2.0
"""ATNM golden files (the reference's matrix_io format) — written by this repository, read by
the reference's own load_matrix and vice versa (oracle/_ref)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_2506_01969_b200 import atnm


def test_roundtrip_and_reference_compat(tmp_path):
    rng = np.random.default_rng(0)
    m = rng.normal(size=(16, 512)).astype(np.float32)
    p = tmp_path / "o.atnm"
    atnm.save(p, m)
    assert np.array_equal(atnm.load(p), m)
    assert np.array_equal(oracle.ref_load_matrix(p), m.astype(np.float64))  # reference reads ours
    q = tmp_path / "r.atnm"
    oracle.ref_save_matrix(q, m.astype(np.float64) * 3)  # we read the reference's
    assert np.array_equal(atnm.load(q), (m * 3).astype(np.float32))
    assert p.read_bytes()[:4] == b"ATNM" and len(p.read_bytes()) == 12 + 16 * 512 * 4


def test_error_behaviour(tmp_path):
    bad = tmp_path / "bad.atnm"
    bad.write_bytes(b"XXXX" + bytes(8))
    with pytest.raises(RuntimeError, match="magic"):
        atnm.load(bad)
    bad.write_bytes(b"ATNM" + bytes(3))
    with pytest.raises(RuntimeError, match="header"):
        atnm.load(bad)
    bad.write_bytes(b"ATNM" + (0).to_bytes(4, "little") + (3).to_bytes(4, "little"))
    with pytest.raises(RuntimeError, match="zero"):
        atnm.load(bad)
    bad.write_bytes(b"ATNM" + (2).to_bytes(4, "little") + (2).to_bytes(4, "little") + bytes(8))
    with pytest.raises(RuntimeError, match="payload"):
        atnm.load(bad)
    with pytest.raises(RuntimeError):
        oracle.ref_load_matrix(bad)


def test_committed_gpu_golden_matches_oracle():
    """The committed GPU dumps (made on a B200 by tests/golden/make_gpu_golden.py) agree with
    the CPU oracle on the same inputs, so the CPU suite also pins the GPU path's numerics."""
    import json
    from pathlib import Path

    gold = Path(__file__).resolve().parent / "golden"
    meta = json.loads((gold / "gpu_golden.json").read_text())
    for name, c in meta["cases"].items():
        go = atnm.load(gold / f"gpu_{name}_o.atnm").astype(np.float64)
        gl = atnm.load(gold / f"gpu_{name}_lse.atnm").astype(np.float64)
        H = c["heads"]
        for b, ctx in enumerate(c["seqlens"]):
            s = c["seed"] + 7919 * b
            q = oracle.bf16_round(oracle.matrix_from_seed(H, 576, 3 * s + 1))
            kv = oracle.bf16_round(oracle.matrix_from_seed(ctx, 576, 3 * s + 2))
            o_ref, l_ref = oracle.attention_ref(q, kv, kv[:, :512], 1.0 / 24.0)
            o = go[b * H:(b + 1) * H]
            assert np.sqrt(np.mean((o - o_ref) ** 2)) <= 2e-5, (name, b)
            assert np.abs(gl[b] - l_ref).max() <= 1e-4, (name, b)
