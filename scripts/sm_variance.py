# SPDX-License-Identifier: Apache-2.0
"""Is the per-CTA span variance systematic per SM? Repeated traced launches, span vs %smid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2506_01969_b200 import _lib, inputs, mla

TT = 256
inp = inputs.make_mla_inputs([65536] * 16, heads=16, pad_value=0.0)
plan = mla.MlaDecodePlan.create(16, 16, "cuda")
n = plan.num_sm_parts
buf = torch.zeros(n * TT * 16, dtype=torch.int64, device="cuda")
for _ in range(3):
    plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
torch.cuda.synchronize()
runs = []
for r in range(6):
    buf.zero_()
    _lib.lib().etap_mla_debug_trace(buf.data_ptr())
    plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    torch.cuda.synchronize()
    _lib.lib().etap_mla_debug_trace(None)
    t = buf.view(n, TT, 16).cpu().numpy()
    ent = (t[:, TT - 1] - t[:, TT - 1, 0].min()).astype(np.float64)  # int64 re-base: float64 ulp at 1.7e18 is 256
    span = (ent[:, 2] - ent[:, 0]) / 1e3
    smid = t[:, TT - 1, 3]
    runs.append((span, smid))
sched = plan.sched.view(n, 8).cpu().numpy()
full = np.array([s[0] == s[2] and s[3] - s[1] == 1024 // 1 * 0 + (s[3] - s[1]) for s in sched])
# per-SM average span over runs (only CTAs with 112-tile single splits)
ntile = np.array([(s[3] - s[1]) if s[0] == s[2] else -1 for s in sched])
sel = ntile == ntile.max()
per_sm = {}
for span, smid in runs:
    for c in np.nonzero(sel)[0]:
        per_sm.setdefault(int(smid[c]), []).append(span[c])
means = {k: np.mean(v) for k, v in per_sm.items()}
stds = {k: np.std(v) for k, v in per_sm.items()}
print("blockIdx->smid identical across runs:", all(np.array_equal(runs[0][1], r[1]) for r in runs))
m = np.array(list(means.values()))
print(f"per-SM mean span over {len(runs)} runs: min {m.min():.1f} median {np.median(m):.1f} max {m.max():.1f} us; "
      f"mean within-SM std {np.mean(list(stds.values())):.2f} us")
order = sorted(means, key=means.get)
print("slowest SMs:", [(k, round(means[k], 1)) for k in order[-12:]])
print("fastest SMs:", [(k, round(means[k], 1)) for k in order[:8]])
# correlation run-to-run
a = np.array([runs[0][0][c] for c in np.nonzero(sel)[0]]); b = np.array([runs[1][0][c] for c in np.nonzero(sel)[0]])
print("run0 vs run1 span corr:", np.corrcoef(a, b)[0, 1])
