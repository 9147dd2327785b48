# SPDX-License-Identifier: Apache-2.0
"""Time the pieces of a decode step with CUDA events (stream launches and CUDA graphs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import inputs, mla

B, CTX = int(os.environ.get("B", 16)), int(os.environ.get("CTX", 65536))
inp = inputs.make_mla_inputs([CTX] * B, heads=16, pad_value=0.0)
plan = mla.MlaDecodePlan.create(B, 16, "cuda")
out = torch.empty((B, 1, 16, 512), dtype=torch.float32, device="cuda")
lse = torch.empty((B, 1, 16), dtype=torch.float32, device="cuda")
X = mla.FLAG_EXTERNAL_SCHEDULE
def dec(flags=0): plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse, flags=flags)
plan.metadata(inp.seqlens)
variants = [
    ("K1", lambda: plan.metadata(inp.seqlens)),
    ("K2 fused-sched", lambda: dec(mla.FLAG_SKIP_COMBINE)),
    ("K2 external", lambda: dec(mla.FLAG_SKIP_COMBINE | X)),
    ("K3", lambda: plan.combine(out, lse)),
    ("K2f+K3", lambda: dec()),
    ("K1+K2x+K3", lambda: (plan.metadata(inp.seqlens), dec(X))),
]
def timeit(fn, n=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / n
for rep in range(2):
    for name, fn in variants:
        print(f"B={B} ctx={CTX} {name:16s} {timeit(fn):8.2f} us")
g = plan.capture(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out, lse, with_metadata=False)
print(f"B={B} ctx={CTX} graph K2f+K3   {timeit(g.replay):8.2f} us")
