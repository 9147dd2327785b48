# SPDX-License-Identifier: Apache-2.0
"""Is the FP8 decode's steady state memory- or SM-bound? Per-tile debug stamps (clock64) of
every CTA at B=16 x 64K x 16 heads: tile period, load latency (producer issue -> GEMM1 sees
the page), how long the producer waited for a free ring slot, and how long GEMM1 had the
page before it could take it. Medians over CTAs and tiles 8..-8.

    python scripts/fp8_tile_balance.py [--bf16]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2506_01969_b200 import _lib, inputs, mla

TT = 256
bf16 = "--bf16" in sys.argv
H = int(os.environ.get("HEADS", 16))  # bf16 head-group kernels: HEADS=32 -> head group 32
inp = inputs.make_mla_inputs([65536] * 16, heads=H, pad_value=0.0)
plan = mla.MlaDecodePlan.create(16, H, "cuda")
if bf16:
    f = lambda: plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
else:
    kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
    f = lambda: plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125)
n = plan.num_sm_parts
buf = torch.zeros(n * TT * 16, dtype=torch.int64, device="cuda")
for _ in range(3):
    f()
torch.cuda.synchronize()
_lib.lib().etap_mla_debug_trace(buf.data_ptr())
f()
torch.cuda.synchronize()
_lib.lib().etap_mla_debug_trace(None)
raw = buf.view(n, TT, 16).cpu().numpy().astype(np.int64)
ent = raw[:, TT - 1]
ghz = (ent[:, 6] - ent[:, 5]).astype(np.float64) / np.maximum(1, (ent[:, 2] - ent[:, 0]).astype(np.float64))
NPS = 5 if not bf16 else None
rows = {k: [] for k in ("period", "latency", "g1_after_prev_g1", "g2commit_to_issue", "issue_to_g1sees_minus_ring")}
for c in range(n):
    t = raw[c, :TT - 1]
    nt = int((t[:, 0] > 0).sum())
    if nt < 24:
        continue
    for g in range(8, nt - 8):
        rows["period"].append(t[g + 1, 0] - t[g, 0])
        rows.setdefault("TMA issue (5 boxes)", []).append(t[g, 1] - t[g, 0])
        rows["latency"].append(t[g, 2] - t[g, 0])
        rows["g1_after_prev_g1"].append(t[g, 2] - t[g - 1, 2])
        if NPS:
            rows["g2commit_to_issue"].append(t[g, 0] - t[g - NPS, 7])
        if True:
            # the tile's compute residency in its ring slot, stage by stage
            rows.setdefault("G1sees->Scommit", []).append(t[g, 3] - t[g, 2])
            rows.setdefault("Scommit->softmax sees S", []).append(t[g, 4] - t[g, 3])
            rows.setdefault("softmax sees S->exp done", []).append(t[g, 8] - t[g, 4])
            rows.setdefault("exp done->P buffer free", []).append(t[g, 9] - t[g, 8])
            rows.setdefault("P free->P written", []).append(t[g, 5] - t[g, 9])
            rows.setdefault("P written->G2 sees P", []).append(t[g, 6] - t[g, 5])
            rows.setdefault("G2 sees->G2 commit", []).append(t[g, 7] - t[g, 6])
            rows.setdefault("G1sees->G2commit (residency)", []).append(t[g, 7] - t[g, 2])
t = raw[:, :5]
print("first five tiles, TMA issue cycles (median over CTAs):", [int(np.median(t[:, j, 1] - t[:, j, 0])) for j in range(5)])
print(f"{'bf16' if bf16 else 'fp8'}: SM clock {np.median(ghz):.3f} GHz, CTAs {n}")
for k, v in rows.items():
    if v:
        v = np.array(v, dtype=np.float64)
        print(f"  {k:>28}: p10 {np.percentile(v, 10):8.0f}  median {np.median(v):8.0f}  p90 {np.percentile(v, 90):8.0f} cycles")
