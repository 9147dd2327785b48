# SPDX-License-Identifier: Apache-2.0
"""Delivered KV bandwidth over time across consecutive decode launches (debug trace: per-tile
clock64 stamps of every CTA mapped onto %globaltimer with each CTA's own clock rate). Bins of
BIN us; a tile counts when its GEMM1 issuer first sees it (slot 2). Flags as the bench.

    [FP8=1] [BIN=2] python scripts/hbm_timeline.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2506_01969_b200 import _lib, inputs, mla

B, CTX, H = 16, 65536, int(os.environ.get("HEADS", 16))
BIN = float(os.environ.get("BIN", 2))
inp = inputs.make_mla_inputs([CTX] * B, heads=H, pad_value=0.0)
plan = mla.MlaDecodePlan.create(B, H, "cuda")
n, TT, STEPS = plan.num_sm_parts, 256, 4
fp8 = bool(os.environ.get("FP8"))
tile_bytes = 64 * 576 * (1 if fp8 else 2)
k2 = [torch.zeros(n * TT * 16, dtype=torch.int64, device="cuda") for _ in range(STEPS)]
L = _lib.lib()
FL = mla.FLAG_INDEPENDENT_INPUTS
f = lambda: plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=FL)
if fp8:
    kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
    f = lambda: plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125, flags=FL)
for _ in range(5):
    f()
torch.cuda.synchronize()
for i in range(STEPS):
    L.etap_mla_debug_trace(k2[i].data_ptr())
    f()
L.etap_mla_debug_trace(None)
torch.cuda.synchronize()
times, steps = [], []
gbase = None
for i in range(STEPS):
    raw = k2[i].view(n, TT, 16).cpu().numpy().astype(np.int64)
    g = raw[:, TT - 1]
    if gbase is None:
        gbase = g[:, 0][g[:, 0] > 0].min()
    ghz = (g[:, 6] - g[:, 5]) / np.maximum(1, g[:, 2] - g[:, 0])
    for c in range(n):
        t = raw[c, :TT - 2, 2]
        t = t[t > 0]
        times.append((g[c, 0] - gbase) + (t - g[c, 5]) / ghz[c])
        steps.append(np.full(len(t), i))
times = np.concatenate(times) / 1e3
steps = np.concatenate(steps)
edges = np.arange(0, times.max() + BIN, BIN)
print(f"{'fp8' if fp8 else 'bf16'}: delivered GB/s per {BIN:g} us bin (tiles seen by GEMM1), by launch")
for a, b in zip(edges[:-1], edges[1:]):
    sel = (times >= a) & (times < b)
    per = [int(((steps == i) & sel).sum()) for i in range(STEPS)]
    tot = sum(per) * tile_bytes / (BIN * 1e3)
    print(f"  {a:7.1f} {tot:7.0f} GB/s  " + " ".join(f"L{i}:{p:4d}" for i, p in enumerate(per) if p))
