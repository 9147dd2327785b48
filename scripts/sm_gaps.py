# SPDX-License-Identifier: Apache-2.0
"""Per-SM handover between consecutive decode launches (debug trace: %smid, entry, first KV
TMA, exit per CTA): how long each SM sits between its CTA of step i exiting and its CTA of
step i+1 entering / issuing its first KV load. Flags as the bench (independent inputs).

    [FP8=1] [CTX=65536] [HEADS=16] python scripts/sm_gaps.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2506_01969_b200 import _lib, inputs, mla

B, CTX, H = int(os.environ.get("B", 16)), int(os.environ.get("CTX", 65536)), int(os.environ.get("HEADS", 16))
inp = inputs.make_mla_inputs([CTX] * B, heads=H, pad_value=0.0)
plan = mla.MlaDecodePlan.create(B, H, "cuda")
n, TT, STEPS = plan.num_sm_parts, 256, 5
k2 = [torch.zeros(n * TT * 16, dtype=torch.int64, device="cuda") for _ in range(STEPS)]
L = _lib.lib()
FL = mla.FLAG_INDEPENDENT_INPUTS
f = lambda: plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=FL)
if os.environ.get("FP8"):
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
g = np.stack([k.view(n, TT, 16).cpu().numpy()[:, TT - 1, :] for k in k2])  # [step, cta, slot]
prol = np.stack([k.view(n, TT, 16).cpu().numpy()[:, TT - 2, :] for k in k2])  # prologue clock64 stamps
base = g[:, :, 0][g[:, :, 0] > 0].min()
ent, fkv, ext, sm = g[:, :, 0] - base, g[:, :, 9] - base, g[:, :, 2] - base, g[:, :, 3]
for i in range(STEPS - 1):
    prev = {int(sm[i, c]): c for c in range(n)}
    d_ent, d_kv, d_lag = [], [], []
    for c in range(n):
        p = prev.get(int(sm[i + 1, c]))
        if p is None:
            continue
        d_ent.append((ent[i + 1, c] - ext[i, p]) / 1e3)
        d_kv.append((fkv[i + 1, c] - ext[i, p]) / 1e3)
    d_ent, d_kv = np.array(d_ent), np.array(d_kv)
    q = lambda x: " / ".join(f"{v:6.2f}" for v in np.percentile(x, [10, 50, 90]))
    period = (np.median(ext[i + 1]) - np.median(ext[i])) / 1e3
    busy = np.median(ext[i + 1] - fkv[i + 1]) / 1e3
    pro = np.median(fkv[i + 1] - ent[i + 1]) / 1e3
    print(f"step {i}->{i + 1}: SMs matched {len(d_ent)}/{n}, distinct SMs {len(set(sm[i + 1].tolist()))} | "
          f"exit->next entry p10/p50/p90 {q(d_ent)} us | exit->next first KV {q(d_kv)} us | "
          f"entry->first KV med {pro:5.2f} | first KV->exit med {busy:6.2f} | exit-median period {period:6.2f} us")

# prologue milestones (clock64 after the CTA's entry stamp, median over CTAs of the last step)
i = STEPS - 1
clk0 = g[i, :, 5].astype(np.int64)
ghz = (g[i, :, 6] - g[i, :, 5]).astype(np.float64) / np.maximum(1, (g[i, :, 2] - g[i, :, 0]).astype(np.float64))
marks = {"seqlens in + scan (warp 0)": g[i, :, 13], "prev range + page ids (warp 2)": prol[i, :, 0],
         "schedule barrier passed": prol[i, :, 1], "first page ids in registers": prol[i, :, 2],
         "FP8 first Q terms in smem (GEMM1 issuer)": prol[i, :, 6],
         "FP8 producer entered": prol[i, :, 3], "FP8 producer policies made": prol[i, :, 4],
         "FP8 producer first split found": prol[i, :, 5],
         "producer at its first TMA": g[i, :, 12], "first TMA issued": g[i, :, 15]}
t0seen = np.stack([k.view(n, TT, 16).cpu().numpy()[:, 0, 2] for k in k2])[i].astype(np.int64)
marks["tile 0 seen by GEMM1"] = t0seen
print(f"prologue, step {i} (SM clock {np.median(ghz):.3f} GHz), us after entry:")
for k, v in marks.items():
    v = v.astype(np.int64)
    ok = v > 0
    if ok.any():
        print(f"  {k:>32}: {np.median((v[ok] - clk0[ok]) / ghz[ok]) / 1e3:6.2f}")
