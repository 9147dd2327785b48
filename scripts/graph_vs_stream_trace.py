# SPDX-License-Identifier: Apache-2.0
"""Per-CTA entry / exit stamps and SM ids of one decode step launched on a stream vs replayed
from a CUDA graph (debug instantiation), to see where the graph replay loses time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2506_01969_b200 import _lib, inputs, mla

H, CTX, B = int(os.environ.get("HEADS", 128)), int(os.environ.get("CTX", 65536)), 16
inp = inputs.make_mla_inputs([CTX] * B, heads=H, pad_value=0.0)
plan = mla.MlaDecodePlan.create(B, H, "cuda")
n, TT = plan.num_sm_parts, 256
L = _lib.lib()
out = torch.empty((B, 1, H, 512), dtype=torch.float32, device="cuda")
lse = torch.empty((B, 1, H), dtype=torch.float32, device="cuda")
buf = torch.zeros(n * TT * 16, dtype=torch.int64, device="cuda")
f = lambda: plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse)
L.etap_mla_debug_trace(buf.data_ptr())
for _ in range(3):
    f()
torch.cuda.synchronize()


def read(tag):
    g = buf.view(n, TT, 16).cpu().numpy()[:, TT - 1, :]
    ent, ex, sm = g[:, 0].astype(np.float64), g[:, 2].astype(np.float64), g[:, 3]
    t0 = ent.min()
    ent, ex = (ent - t0) / 1e3, (ex - t0) / 1e3
    lanes = 4 if H >= 128 else max(1, H // 32)
    per = n // lanes
    lane_ex = [np.median(ex[i * per:(i + 1) * per]) for i in range(lanes)]
    print(f"{tag}: entry spread {ent.max():.2f} us, exit med {np.median(ex):.2f} min {ex.min():.2f} max {ex.max():.2f}; "
          f"lane exit medians {[round(x, 1) for x in lane_ex]}")
    return sm, ex


buf.zero_()
f()
torch.cuda.synchronize()
sm_s, ex_s = read("stream")
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
gr = torch.cuda.CUDAGraph()
with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
    f()
torch.cuda.synchronize()
gr.replay()
torch.cuda.synchronize()
buf.zero_()
gr.replay()
torch.cuda.synchronize()
sm_g, ex_g = read("graph ")
print("same blockIdx->SM mapping:", bool((sm_s == sm_g).all()), " distinct SMs stream/graph:", len(set(sm_s)), len(set(sm_g)))
print("first 16 SM ids stream:", list(sm_s[:16]))
print("first 16 SM ids graph :", list(sm_g[:16]))
# SMs of the 4 CTAs that share pages (k, k+37, k+74, k+111)
if H >= 128:
    per = n // 4
    for k in (0, 1, 2):
        print(f"sharers of k={k}: stream {[int(sm_s[k + i * per]) for i in range(4)]} graph {[int(sm_g[k + i * per]) for i in range(4)]}")
L.etap_mla_debug_trace(None)
