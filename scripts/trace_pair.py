# SPDX-License-Identifier: Apache-2.0
"""Per-page pipeline trace of the CTA-pair decode (debug instantiation, %clock64 stamps per page,
see etap_mla_pair.cuh): medians over the pages of every leader / partner CTA.

    python scripts/trace_pair.py [--batch 16 --ctx 65536 --heads 128]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_2506_01969_b200 import _lib, inputs, mla

TT = 256
SLOTS = {0: "G1 TMA issued", 1: "V TMA issued", 2: "V landed", 3: "G1 data seen (leader)", 4: "G1 committed",
         5: "S seen (softmax)", 12: "S_FREE arrived", 6: "exp done", 7: "P buffer free", 8: "P_FULL arrived",
         9: "P seen (G2 issuer)", 10: "V ready seen", 11: "G2 committed", 13: "S in registers",
         14: "exchange barrier passed", 15: "P stores done"}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=65536)
    ap.add_argument("--heads", type=int, default=128)
    a = ap.parse_args()
    inp = inputs.make_mla_inputs([a.ctx] * a.batch, heads=a.heads, pad_value=0.0)
    plan = mla.MlaDecodePlan.create(a.batch, a.heads, "cuda")
    nparts = plan.num_sm_parts
    buf = torch.zeros(nparts * TT * 16, dtype=torch.int64, device="cuda")
    for _ in range(3):
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    torch.cuda.synchronize()
    _lib.lib().etap_mla_debug_trace(buf.data_ptr())
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
        e1.record()
        torch.cuda.synchronize()
    _lib.lib().etap_mla_debug_trace(None)
    print(f"traced step: {e0.elapsed_time(e1) * 1000:.1f} us")
    raw = buf.view(nparts, TT, 16).cpu().numpy().astype(np.int64)
    used = (raw[:, TT - 1, 2] > 0)
    print(f"CTAs that ran: {int(used.sum())} of {nparts}")
    ent = raw[:, TT - 1, 0]
    ext = raw[:, TT - 1, 2]
    g0 = ent[used].min()
    print(f"entry spread {(ent[used].max() - g0) / 1e3:.2f} us, exit min/median/max "
          f"{(ext[used].min() - g0) / 1e3:.1f} / {(np.median(ext[used]) - g0) / 1e3:.1f} / {(ext[used].max() - g0) / 1e3:.1f} us")
    # per pair: exit of the later CTA, pages streamed (stamped tile rows), sorted by exit
    pe = []
    for c in range(0, nparts, 2):
        if used[c]:
            n = int((raw[c, :TT - 1, 0] > 0).sum())
            pe.append(((max(ext[c], ext[c + 1]) - g0) / 1e3, n))
    pe.sort()
    print("pair exits (us, pages) fastest 5:", [(round(a, 1), b) for a, b in pe[:5]],
          "slowest 5:", [(round(a, 1), b) for a, b in pe[-5:]])
    ghz = (raw[:, TT - 1, 6] - raw[:, TT - 1, 5]) / np.maximum(1, ext - ent)
    print(f"SM clock {np.median(ghz[used]):.3f} GHz")
    for role, ctas in (("leader", [c for c in range(0, nparts, 2) if used[c]]),
                       ("partner", [c for c in range(1, nparts, 2) if used[c]])):
        rows = []
        for c in ctas:
            t = raw[c, :TT - 1]
            n = int((t[:, 0] > 0).sum())
            for g in range(4, min(n, TT - 2) - 1):
                rows.append(t[g].astype(np.float64) - t[g, 0])
                rows[-1] = np.append(rows[-1], t[g + 1, 5] - t[g, 5])  # softmax period
        if not rows:
            continue
        m = np.median(np.array(rows), axis=0)
        print(f"--- {role} (median over pages, cycles relative to its G1 TMA issue; period {m[16]:.0f} cycles)")
        for s in (0, 1, 2, 3, 4, 5, 13, 12, 6, 7, 14, 15, 8, 9, 10, 11):
            if role == "partner" and s in (3, 4, 9, 10, 11):
                continue
            print(f"  {SLOTS[s]:>24}: {m[s]:8.0f}")


if __name__ == "__main__":
    main()
