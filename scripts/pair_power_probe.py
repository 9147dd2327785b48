# SPDX-License-Identifier: Apache-2.0
"""Probe: the pair kernel at 128 heads on fewer CTA pairs. If the time per page per pair drops as
fewer SMs run, the full-chip kernel is power-bound (the SM clock falls under load), not bound by
its own per-SM pipeline."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_01969_b200 import inputs, mla, _lib
seqlens = [65536] * 16
inp = inputs.make_mla_inputs(seqlens, heads=128, seed=1, pad_value=0.0)
for parts in (148, 96, 48, 24):
    plan = mla.MlaDecodePlan.create(16, 128, "cuda", parts)
    out = torch.empty((16, 1, 128, 512), dtype=torch.float32, device="cuda")
    lse = torch.empty((16, 1, 128), dtype=torch.float32, device="cuda")
    for _ in range(3): plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10 if parts >= 96 else 4
    e0.record()
    for _ in range(n): plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / n
    pages_per_pair = 16384 / (parts // 2)
    print(f"parts={parts} pairs={parts//2} us/step={us:.1f} us/page/pair={us/pages_per_pair:.3f}", flush=True)
