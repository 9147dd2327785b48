# SPDX-License-Identifier: Apache-2.0
"""GPU bring-up diagnostics: UMMA layout self-test, small parity cases, one timing.

Usage (on a B200 box): python scripts/gpu_check.py [--quick]
"""
from __future__ import annotations

import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import oracle
from paper_2506_01969_b200 import inputs, mla


def selftest():
    torch.manual_seed(0)
    k = torch.randn(64, 576, device="cuda").to(torch.bfloat16)
    q = torch.randn(16, 576, device="cuda").to(torch.bfloat16)
    p = torch.rand(64, 16, device="cuda")
    s_t, o_t = mla.selftest_umma(k, q, p)
    torch.cuda.synchronize()
    s_ref = k.double() @ q.double().T
    o_ref = k[:, :512].double().T @ p.double()
    o_t = o_t[:, :16] + o_t[:, 16:]
    es = (s_t.double() - s_ref).abs().max().item()
    eo = (o_t.double() - o_ref).abs().max().item()
    print(f"selftest: S^T max err {es:.3e} "
          f"(|S| max {s_ref.abs().max().item():.2f}), O^T max err {eo:.3e} (|O| max {o_ref.abs().max().item():.2f})")
    if es > 1e-2 or eo > 1e-2:
        # locate the error pattern
        d = (s_t.double() - s_ref).abs()
        print("  S err by row-block:", [round(d[i:i + 8].max().item(), 3) for i in range(0, 64, 8)])
        print("  S err by head:", [round(d[:, h].max().item(), 3) for h in range(16)])
        d = (o_t.double() - o_ref).abs()
        print("  O err by d-block(64):", [round(d[i:i + 64].max().item(), 3) for i in range(0, 512, 64)])
        print("  O err by head:", [round(d[:, h].max().item(), 3) for h in range(16)])
    return es, eo


def parity(seqlens, heads=16, pad=float("nan"), flags=0, seed=42, q_scale=1.0):
    inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=seed, pad_value=pad, q_scale=q_scale)
    out, lse = mla.mla_decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=flags)
    torch.cuda.synchronize()
    qb = inp.q.view(torch.int16).cpu().numpy().view(np.uint16)
    kvb = inp.kv_pool.view(torch.int16).cpu().numpy().view(np.uint16)
    o_ref, l_ref = oracle.mla_decode_bf16(qb, kvb, inp.block_table.cpu().numpy(), inp.seqlens.cpu().numpy(), inp.scale)
    o = out.double().cpu().numpy().reshape(o_ref.shape)
    l = lse.double().cpu().numpy().reshape(l_ref.shape)
    fin = np.isfinite(o_ref)
    rmse = math.sqrt(np.mean((o[fin] - o_ref[fin]) ** 2)) if fin.any() else 0.0
    mx = np.abs(o - o_ref)[fin].max() if fin.any() else 0.0
    lfin = np.isfinite(l_ref)
    lerr = np.abs(l - l_ref)[lfin].max() if lfin.any() else 0.0
    nonfinite = int((~np.isfinite(o)).sum())
    print(f"parity seqlens={seqlens[:4]}{'...' if len(seqlens) > 4 else ''} H={heads} flags={flags}: "
          f"rmse {rmse:.3e} maxabs {mx:.3e} lse maxabs {lerr:.3e} nonfinite {nonfinite}")
    return rmse


def timing(B=16, ctx=65536, iters=20):
    inp = inputs.make_mla_inputs([ctx] * B, heads=16, pad_value=0.0)
    plan = mla.MlaDecodePlan.create(B, 16, "cuda")
    for _ in range(3):
        plan.metadata(inp.seqlens)
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        plan.metadata(inp.seqlens)
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / iters
    nbytes = inputs.algorithmic_bytes(inp.seqlens_list, 16)
    print(f"timing B={B} ctx={ctx}: {us:.1f} us/step, {nbytes / us / 1e3:.1f} GB/s")


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), mla._lib.lib().etap_mla_version().decode())
    es, eo = selftest()
    if "--selftest" in sys.argv:
        sys.exit(0)
    parity([128])
    parity([64])
    parity([1000])
    parity([1024, 77, 4096, 129])
    parity([1024], flags=2)
    parity([4096] * 16)
    parity([1024], flags=1)
    if "--quick" not in sys.argv:
        timing()
