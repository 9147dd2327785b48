# SPDX-License-Identifier: Apache-2.0
"""Probe: 32 / 64 heads with and without the step overlap, per head-group setting (ETAP_HEAD_GROUP)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_01969_b200 import inputs, mla
for H in [int(x) for x in os.environ.get("HEADS_LIST", "32,64").split(",")]:
    inp = inputs.make_mla_inputs([65536] * 16, heads=H, seed=1, pad_value=0.0)
    plan = mla.MlaDecodePlan.create(16, H, "cuda")
    out = torch.empty((16, 1, H, 512), dtype=torch.float32, device="cuda"); lse = torch.empty((16, 1, H), dtype=torch.float32, device="cuda")
    for fl, name in ((mla.FLAG_INDEPENDENT_INPUTS, "indep"), (mla.FLAG_EARLY_METADATA, "early")) * int(os.environ.get("ROUNDS", 1)):
        for _ in range(10): plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse, flags=fl)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse, flags=fl)
        e1.record(); torch.cuda.synchronize()
        print(f"H={H} hg_env={os.environ.get('ETAP_HEAD_GROUP','auto')} {name} us/step={e0.elapsed_time(e1)*1000/50:.1f}", flush=True)
