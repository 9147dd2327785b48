# SPDX-License-Identifier: Apache-2.0
"""Start / exit distribution of consecutive decode launches (etap_mla_debug_span stamps) with
the bench's flags: how far the next step's CTAs start inside the previous step's tail."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2506_01969_b200 import _lib, inputs, mla

H = int(os.environ.get("HEADS", 16))
inp = inputs.make_mla_inputs([65536] * 16, heads=H, pad_value=0.0)
plan = mla.MlaDecodePlan.create(16, H, "cuda")
FL = mla.FLAG_INDEPENDENT_INPUTS if not os.environ.get("EARLY") else mla.FLAG_EARLY_METADATA
if os.environ.get("FP8"):  # FP8 (e4m3) latent cache: FP8=1
    kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
    step = lambda: plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125, flags=FL)
else:
    step = lambda: plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=FL)
n, STEPS = plan.num_sm_parts, 6
sp = torch.zeros((STEPS, n, 2), dtype=torch.int64, device="cuda")
L = _lib.lib()
for _ in range(5):
    step()
torch.cuda.synchronize()
for i in range(STEPS):
    L.etap_mla_debug_span(sp[i].data_ptr())
    step()
L.etap_mla_debug_span(None)
torch.cuda.synchronize()
a = sp.cpu().numpy().astype(np.int64)
g0 = a[a > 0].min()
a = (a - g0) / 1e3
for i in range(STEPS):
    st, ex = a[i, :, 0], a[i, :, 1]
    print(f"launch {i}: start min/p10/median/max {st.min():8.2f} {np.percentile(st, 10):8.2f} {np.median(st):8.2f} "
          f"{st.max():8.2f} | exit min/median/max {ex.min():8.2f} {np.median(ex):8.2f} {ex.max():8.2f} | "
          f"CTA busy mean {np.mean(ex - st):7.2f}")
    if os.environ.get("HIST"):
        print("   exits (sorted, every 8th):", " ".join(f"{x:.1f}" for x in np.sort(ex)[::8]))
        print("   starts (sorted, every 8th):", " ".join(f"{x:.1f}" for x in np.sort(st)[::8]))
