# SPDX-License-Identifier: Apache-2.0
"""CPU tests: pin the C restatement (oracle/) against the reference's own golden values and
against the reference itself (oracle/_ref, compiled from /root/reference/proj/src).

Mirrors the reference's test_oracle.cpp / test_etap.cpp cases (cited per test).
"""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle

GOLD = Path(__file__).resolve().parent / "golden"


def maxabs(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))))


# ------------------------------------------------------------------ reference inline goldens
def test_single_logit_passthrough():  # test_oracle.cpp:24-33, test_etap.cpp:127-135
    q = np.array([[1.0, 0.0]]); k = np.array([[1.0, 0.0]]); v = np.array([[3.0, 4.0]])
    o, l = oracle.attention_ref(q, k, v, 1.0)
    assert o.tolist() == [[3.0, 4.0]] and l.tolist() == [1.0]
    o, l = oracle.run_etap(q, k, v, 1.0, 1, 1)
    assert abs(o[0, 0] - 3.0) <= 1e-15 and abs(o[0, 1] - 4.0) <= 1e-15 and abs(l[0] - 1.0) <= 1e-15


def test_identical_keys_lse_is_s_plus_log2():  # test_oracle.cpp:35-45
    q = np.array([[0.5, -0.25]]); k = np.array([[1.0, 2.0], [1.0, 2.0]])
    v = np.array([[7.0, -1.0, 0.5], [7.0, -1.0, 0.5]])
    o, l = oracle.attention_ref(q, k, v, 1.0)
    assert maxabs(o[0], v[0]) <= 1e-14
    assert abs(l[0] - (0.5 * 1.0 - 0.25 * 2.0 + math.log(2.0))) <= 1e-14


def test_dense_brute_force():  # test_oracle.cpp:47-54 (materialized S, no max subtraction)
    q = oracle.matrix_from_seed(4, 8, 42 * 3 + 1); k = oracle.matrix_from_seed(37, 8, 42 * 3 + 2)
    v = oracle.matrix_from_seed(37, 8, 42 * 3 + 3)
    sc = 1.0 / math.sqrt(8.0)
    o, l = oracle.attention_ref(q, k, v, sc)
    e = np.exp(sc * (q @ k.T))
    o_d = (e / e.sum(1, keepdims=True)) @ v
    assert maxabs(o, o_d) <= 1e-12 and maxabs(l, np.log(e.sum(1))) <= 1e-12


def test_shift_invariance():  # test_oracle.cpp:56-80
    scale, shifts = 0.5, [0.0, 3.0, -2.0]
    q0 = oracle.matrix_from_seed(3, 4, 5); k0 = oracle.matrix_from_seed(6, 4, 6); v = oracle.matrix_from_seed(6, 5, 7)
    q1 = np.concatenate([q0, np.array(shifts)[:, None] / scale], 1)
    k1 = np.concatenate([k0, np.ones((6, 1))], 1)
    ob, lb = oracle.attention_ref(q0, k0, v, scale)
    os_, ls = oracle.attention_ref(q1, k1, v, scale)
    assert maxabs(ob, os_) <= 1e-12
    assert maxabs(ls - lb, shifts) <= 1e-12


def test_convex_hull_and_scale_zero():  # test_oracle.cpp:82-110
    q = oracle.matrix_from_seed(5, 6, 13 * 3 + 1); k = oracle.matrix_from_seed(9, 6, 13 * 3 + 2)
    v = oracle.matrix_from_seed(9, 4, 13 * 3 + 3)
    o, _ = oracle.attention_ref(q, k, v, 1 / math.sqrt(6))
    assert (o >= v.min(0) - 1e-12).all() and (o <= v.max(0) + 1e-12).all()
    o0, _ = oracle.attention_ref(q, k, v, 0.0)
    assert maxabs(o0, np.broadcast_to(v.mean(0), o0.shape)) <= 1e-13


def test_probability_rows_sum_to_one():  # test_oracle.cpp:112-126
    q = oracle.matrix_from_seed(4, 8, 21 * 3 + 1); k = oracle.matrix_from_seed(19, 8, 21 * 3 + 2)
    v = oracle.matrix_from_seed(19, 4, 21 * 3 + 3)
    sc = 1 / math.sqrt(8)
    _, l = oracle.attention_ref(q, k, v, sc)
    p = np.exp(sc * (q @ k.T) - l[:, None])
    assert maxabs(p.sum(1), 1.0) <= 1e-12


# ------------------------------------------------------------------ restatement == reference
def test_generator_matches_reference():  # matrix.cpp:23-48,153-165
    for seed, dist in [(1, "normal"), (42 * 3 + 2, "normal"), (7, "uniform"), (2**63 + 5, "normal")]:
        a = oracle.matrix_from_seed(13, 17, seed, dist)
        b = oracle.ref_matrix_from_seed(13, 17, seed, dist)
        assert np.array_equal(a, b)


def test_round_half_matches_reference():  # matrix.cpp:167-184, acceptance criterion 8
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.normal(size=3000) * 10.0 ** rng.integers(-9, 6, 3000),
                         [0.0, -0.0, 65504.0, 65519.99, 65520.0, 2.0**-24, 2.0**-25, 3 * 2.0**-26]])
    R = oracle.ref()
    L = oracle.lib()
    for x in xs:
        a, b = L.oracle_round_half(float(x)), R.ref_round_half(float(x))
        assert (a == b) or (math.isnan(a) and math.isnan(b)), x


def test_bf16_rounding_is_rne_and_single_rounding():
    import torch

    rng = np.random.default_rng(1)
    x32 = rng.normal(size=5000).astype(np.float32).astype(np.float64)
    # for binary32 inputs the direct rounding must equal torch's float32->bf16 RNE
    t = torch.from_numpy(x32).float().to(torch.bfloat16).double().numpy()
    assert np.array_equal(oracle.bf16_round(x32), t)
    # ties go to even; a value just above the tie rounds up even when its float32 image is a tie
    assert oracle.lib().oracle_bf16_round(1.0 + 2.0**-8) == 1.0
    assert oracle.lib().oracle_bf16_round(1.0 + 3 * 2.0**-8) == 1.0 + 2.0**-6
    assert oracle.lib().oracle_bf16_round(1.0 + 2.0**-8 + 2.0**-40) == 1.0 + 2.0**-7
    bits = oracle.bf16_bits(x32)
    assert np.array_equal(oracle.bf16_widen(bits), t)


@pytest.mark.parametrize("seed", [1, 2, 3])
@pytest.mark.parametrize("n_kv", [64, 257, 1024])
def test_restatement_equals_reference(seed, n_kv):  # acceptance.cpp:92-140 grid, cli.cpp:125-187
    q, k, v, sc = oracle.ref_make_problem(seed, 16, n_kv, 576, 512)
    o_ref, l_ref = oracle.ref_run("ref", q, k, v, sc)
    o, l = oracle.attention_ref(q, k, v, sc)
    assert np.array_equal(o, o_ref) and np.array_equal(l, l_ref)  # bit-exact restatement
    for b_c in (16, 64, 100):
        oe_ref, le_ref = oracle.ref_run("etap", q, k, v, sc, b_r=64, b_c=b_c)
        oe, le = oracle.run_etap(q, k, v, sc, 64, b_c)
        assert np.array_equal(oe, oe_ref) and np.array_equal(le, le_ref)
        assert maxabs(oe, o_ref) <= 1e-10 and maxabs(le, l_ref) <= 1e-10


def test_seed42_golden_fixture():  # test_etap.cpp:137-146 via the reference-generated fixture
    g = np.load(GOLD / "seed42_16x257.npz")
    q, k, v, sc = oracle.ref_make_problem(42, 16, 257, 576, 512)
    o, l = oracle.attention_ref(q, k, v, sc)
    assert np.array_equal(o, g["o"]) and np.array_equal(l, g["l"])
    oe, le = oracle.run_etap(q, k, v, sc, 16, 64)
    assert np.array_equal(oe, g["o_etap"]) and maxabs(oe, g["o"]) <= 1e-10 and maxabs(le, g["l"]) <= 1e-10


def test_partition_invariance_and_fault():  # test_etap.cpp:159-168, 242-249
    q = oracle.matrix_from_seed(4, 32, 42 * 3 + 1); k = oracle.matrix_from_seed(257, 32, 42 * 3 + 2)
    v = oracle.matrix_from_seed(257, 16, 42 * 3 + 3)
    outs = [oracle.run_etap(q, k, v, 0.3, 4, bc)[0] for bc in (5, 64, 100, 257)]
    for a, b in zip(outs, outs[1:]):
        assert maxabs(a, b) <= 1e-10
    good, _ = oracle.run_etap(q[:, :16], k[:64, :16], v[:64, :8], 0.25, 4, 16)
    bad, _ = oracle.run_etap(q[:, :16], k[:64, :16], v[:64, :8], 0.25, 4, 16, negate_rescale=True)
    assert maxabs(good, bad) > 1e-6
    with pytest.raises(ValueError):
        oracle.run_etap(q, k, v, 0.3, 0, 4)


def test_odd_and_unit_dv():  # test_etap.cpp:251-263
    for n_q, n_kv, d_qk, d_v, br, bc in [(3, 29, 8, 7, 2, 8), (2, 9, 4, 1, 2, 4)]:
        q = oracle.matrix_from_seed(n_q, d_qk, 5); k = oracle.matrix_from_seed(n_kv, d_qk, 6)
        v = oracle.matrix_from_seed(n_kv, d_v, 7)
        o_ref, _ = oracle.attention_ref(q, k, v, 1 / math.sqrt(d_qk))
        o, _ = oracle.run_etap(q, k, v, 1 / math.sqrt(d_qk), br, bc)
        assert maxabs(o, o_ref) <= 1e-11


# ------------------------------------------------------------------ MLA fixtures (bf16 inputs)
def _mla_inputs_from_seed(seed0, seqlens, heads):
    """Regenerate the fixture inputs with the restated generator, as bf16 bits, in a paged
    pool with an identity block table (pages padded with NaN)."""
    qs, kvs = [], []
    for b, ctx in enumerate(seqlens):
        s = seed0 + 7919 * b
        qs.append(oracle.bf16_round(oracle.matrix_from_seed(heads, 576, 3 * s + 1)))
        kvs.append(oracle.bf16_round(oracle.matrix_from_seed(ctx, 576, 3 * s + 2)))
    return qs, kvs


@pytest.mark.parametrize("name", ["mla_b1_h16_ctx1024", "mla_varlen_b4", "mla_b2_h32_ctx300"])
def test_mla_fixture_oracle(name):
    import hashlib

    g = np.load(GOLD / f"{name}.npz")
    seqlens = g["seqlens"].tolist()
    heads = int(g["heads"])
    qs, kvs = _mla_inputs_from_seed(int(g["seed"]), seqlens, heads)
    for b in range(len(seqlens)):
        assert hashlib.sha256(qs[b].tobytes()).hexdigest()[:16] == g["q_sha"][b]
        assert hashlib.sha256(kvs[b].tobytes()).hexdigest()[:16] == g["kv_sha"][b]
    # paged oracle on bf16 bits == the reference's attention_ref on the same values
    pages = [(s + 63) // 64 for s in seqlens]
    pool = np.full((sum(pages), 64, 576), 0x7FC0, dtype=np.uint16)  # NaN padding
    bt = np.zeros((len(seqlens), max(pages)), dtype=np.int32)
    off = 0
    for b, s in enumerate(seqlens):
        perm = np.arange(off, off + pages[b])[::-1]  # reversed pages: exercise the block table
        bt[b, :pages[b]] = perm
        rows = oracle.bf16_bits(kvs[b])
        for p in range(pages[b]):
            chunk = rows[p * 64:(p + 1) * 64]
            pool[perm[p], :chunk.shape[0]] = chunk
        off += pages[b]
    qb = np.stack([oracle.bf16_bits(q) for q in qs])
    o, l = oracle.mla_decode_bf16(qb, pool, bt, np.array(seqlens, np.int32), float(g["scale"]))
    assert np.array_equal(o, g["o"]) and np.array_equal(l, g["l"])


def test_golden_json_records_reference_fp16emu():  # test_etap.cpp:231-240
    meta = json.loads((GOLD / "golden.json").read_text())
    r = meta["fp16emu_8x512x64"]
    assert 0 < r["rmse_etap"] <= 1e-3 and r["rmse_etap"] <= 4 * r["rmse_standard"]
