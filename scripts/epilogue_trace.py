# SPDX-License-Identifier: Apache-2.0
"""Where the last split's epilogue time goes (clock64 stamps in the last tile's trace row:
7 = GEMM2 committed (issuer), 10 = l reduced, 11 = after the reduction barrier, 12 = O rows
stored, 13 = LSE stored + final barrier)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2506_01969_b200 import _lib, inputs, mla

B, CTX = int(os.environ.get("B", 16)), int(os.environ.get("CTX", 8192))
inp = inputs.make_mla_inputs([CTX] * B, heads=16, pad_value=0.0)
plan = mla.MlaDecodePlan.create(B, 16, "cuda")
n, TT = plan.num_sm_parts, 256
buf = torch.zeros(n * TT * 16, dtype=torch.int64, device="cuda")
for _ in range(3):
    plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
torch.cuda.synchronize()
_lib.lib().etap_mla_debug_trace(buf.data_ptr())
plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
torch.cuda.synchronize()
_lib.lib().etap_mla_debug_trace(None)
t = buf.view(n, TT, 16).cpu().numpy().astype(np.int64)
rows = []
for c in range(n):
    last = [g for g in range(TT - 1) if t[c, g, 13] > 0]
    if not last:
        continue
    e = t[c, last[-1]]
    rows.append([e[10] - e[7], e[11] - e[10], e[12] - e[11], e[13] - e[12], e[13] - e[7], e[14] - e[11], e[15] - e[14]])
r = np.array(rows)
for i, lab in enumerate(["G2 commit -> l reduced", "reduction barrier", "O rows stored", "LSE + final barrier", "total", "  first TMEM loads", "  first 2 blocks stored"]):
    print(f"{lab:26s} cycles median {np.median(r[:, i]):7.0f}  p90 {np.percentile(r[:, i], 90):7.0f}")
