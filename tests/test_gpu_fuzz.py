# SPDX-License-Identifier: Apache-2.0
"""Randomised decode configurations against the binary64 oracle (bf16 and FP8 latent caches):
batch, ragged / empty / page-aligned context lengths, heads (16..64), query tokens (MTP),
CTA counts 1..148 (the split schedule, lanes, K1 vs in-kernel schedule, combine). Fixed seeds,
so every run checks the same 40 cases (ETAP_FUZZ_CASES=N draws N per cache type instead).
Every case is also decoded with FLAG_EARLY_METADATA (schedule read before the grid
dependency) and must be bitwise the same."""
from __future__ import annotations

import os
import random

import numpy as np
import pytest
import torch

import oracle
from paper_2506_01969_b200 import inputs, mla

pytestmark = pytest.mark.gpu

RMSE_TOL = 2e-5
LSE_TOL = 1e-4
N_CASES = int(os.environ.get("ETAP_FUZZ_CASES", 20))


def bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def draw(case: int):
    rnd = random.Random(1000 + case)
    batch = rnd.choice([1, 2, 3, 5, 8, 17, 33])
    lens = []
    for _ in range(batch):
        kind = rnd.random()
        if kind < 0.1:
            lens.append(0)
        elif kind < 0.25:
            lens.append(64 * rnd.randint(1, 20))          # page-aligned
        elif kind < 0.35:
            lens.append(rnd.randint(1, 3))                # a few rows
        else:
            lens.append(rnd.randint(1, 2500))
    heads = rnd.choice([16, 16, 32, 48, 64])
    q_tokens = rnd.choice([1, 2, 3]) if heads == 16 else (rnd.choice([1, 2]) if heads == 32 else 1)
    parts = rnd.choice([1, 3, 16, 61, 148])
    return lens, heads, q_tokens, parts


def reference(inp, q_tokens, kv_bits):
    q = bits(inp.q)
    bt, sl = inp.block_table.cpu().numpy(), inp.seqlens.cpu().numpy()
    if q_tokens == 1:
        o, l = oracle.mla_decode_bf16(q[:, 0], kv_bits, bt, sl, inp.scale)
        return o[:, None], l[:, None]
    return oracle.mla_decode_bf16_tokens(q, kv_bits, bt, sl, inp.scale, True)


def check(out, lse, o_ref, l_ref, lens, q_tokens):
    o, l = out.double().cpu().numpy(), lse.double().cpu().numpy()
    assert np.isfinite(o).all()
    for j in range(q_tokens):
        vis = np.maximum(np.array(lens) - (q_tokens - 1 - j), 0)
        ne = vis > 0
        if ne.any():
            rmse = float(np.sqrt(np.mean((o[ne, j] - o_ref[ne, j]) ** 2)))
            assert rmse <= RMSE_TOL, rmse
            assert np.abs(l[ne, j] - l_ref[ne, j]).max() <= LSE_TOL
        if (~ne).any():
            assert (o[~ne, j] == 0).all() and np.isneginf(l[~ne, j]).all()


@pytest.mark.parametrize("case", range(N_CASES))
def test_fuzz_bf16(cuda_device, case):
    lens, heads, q_tokens, parts = draw(case)
    inp = inputs.make_mla_inputs(lens, heads=heads, seed=case, pad_value=float("nan"), q_tokens=q_tokens)
    plan = mla.MlaDecodePlan.create(len(lens), heads, "cuda", parts, q_tokens=q_tokens)
    out, lse = plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    o2, l2 = plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=mla.FLAG_EARLY_METADATA)
    torch.cuda.synchronize()
    assert torch.equal(out, o2) and torch.equal(lse, l2)
    o_ref, l_ref = reference(inp, q_tokens, bits(inp.kv_pool))
    check(out, lse, o_ref, l_ref, lens, q_tokens)


@pytest.mark.parametrize("case", range(N_CASES, 2 * N_CASES))
def test_fuzz_fp8(cuda_device, case):
    lens, heads, q_tokens, parts = draw(case)
    inp = inputs.make_mla_inputs(lens, heads=heads, seed=case, pad_value=float("nan"), q_tokens=q_tokens)
    kv_scale = 2.0 ** -3  # power of two: the dequantised cache is exact in bf16 for the oracle
    kv8 = (inp.kv_pool.float() / kv_scale).to(torch.float8_e4m3fn)
    deq = (kv8.float() * kv_scale).to(torch.bfloat16)
    plan = mla.MlaDecodePlan.create(len(lens), heads, "cuda", parts, q_tokens=q_tokens)
    out, lse = plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, kv_scale)
    o2, l2 = plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, kv_scale, flags=mla.FLAG_EARLY_METADATA)
    torch.cuda.synchronize()
    assert torch.equal(out, o2) and torch.equal(lse, l2)
    o_ref, l_ref = reference(inp, q_tokens, bits(deq))
    check(out, lse, o_ref, l_ref, lens, q_tokens)
