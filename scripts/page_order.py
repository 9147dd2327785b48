# SPDX-License-Identifier: Apache-2.0
"""Decode time with a shuffled vs contiguous page pool (same data volume)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import inputs, mla

def run(shuffle):
    inp = inputs.make_mla_inputs([65536] * 16, heads=16, pad_value=0.0, shuffle_pages=shuffle)
    plan = mla.MlaDecodePlan.create(16, 16, "cuda")
    f = lambda: plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    for _ in range(5): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): f()
    e1.record(); torch.cuda.synchronize()
    del inp
    return e0.elapsed_time(e1) * 1000 / 50
for rep in range(2):
    print(f"shuffled {run(True):.1f} us   contiguous {run(False):.1f} us")
