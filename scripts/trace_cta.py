# SPDX-License-Identifier: Apache-2.0
"""Per-tile stamps of a few CTAs (debug trace), to look at split boundaries:
    python scripts/trace_cta.py [--fp8] [--ctx 16384] [--heads 16]
Prints, for the CTAs with the most splits and one single-split CTA, every tile's stamps in us
after the CTA's entry: producer issue / last issue, G1 sees tile, S committed, softmax sees S,
exp done, P buffer free, P written, G2 sees P, G2 committed (+ the split epilogue's start / end
on a split's last tile, FP8 kernel)."""
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


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=16384)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--fp8", action="store_true")
    a = ap.parse_args()
    inp = inputs.make_mla_inputs([a.ctx] * a.batch, heads=a.heads, pad_value=0.0)
    plan = mla.MlaDecodePlan.create(a.batch, a.heads, "cuda")
    if a.fp8:
        kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
        f = lambda: plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125)  # noqa: E731
    else:
        f = lambda: plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)  # noqa: E731
    n = plan.num_sm_parts
    buf = torch.zeros(n * TT * 16, dtype=torch.int64, device="cuda")
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    _lib.lib().etap_mla_debug_trace(buf.data_ptr())
    f()
    torch.cuda.synchronize()
    _lib.lib().etap_mla_debug_trace(None)
    raw = buf.view(n, TT, 16).cpu().numpy()
    ent = raw[:, TT - 1]
    ghz = (ent[:, 6] - ent[:, 5]).astype(np.float64) / np.maximum(1, (ent[:, 2] - ent[:, 0]).astype(np.float64))
    sched = plan.sched.view(n, 8).cpu().numpy()
    nsplit = np.array([s[2] - s[0] + 1 if s[2] >= s[0] else 0 for s in sched])
    picks = list(np.argsort(-nsplit)[:2]) + [int(np.argmin(np.abs(nsplit - 1)))]
    names = ["issue", "issued", "G1sees", "Scommit", "SMsees", "expdone", "Pfree", "Pwritten", "G2sees", "G2commit",
             "epi_in", "epi_out"]
    order = [0, 1, 2, 3, 4, 8, 9, 5, 6, 7, 10, 11]  # epilogue stamps: last tile of a split (FP8 kernel)
    for c in picks:
        print(f"CTA {c}: sched {sched[c][:5].tolist()} splits {nsplit[c]}, clock {ghz[c]:.3f} GHz; "
              f"exit {(ent[c, 2] - ent[c, 0]) / 1e3:.2f} us; Q published {(ent[c, 4] - ent[c, 0]) / 1e3 if ent[c, 4] else float('nan'):.2f}; "
              f"last epilogue {(ent[c, 10] - ent[c, 0]) / 1e3:.2f}")
        print("   tile " + " ".join(f"{x:>8s}" for x in names))
        for g in range(TT - 1):
            row = raw[c, g]
            if not (row[:8] > 0).any():
                break
            us = [(row[k] - ent[c, 5]) / ghz[c] / 1e3 if row[k] > 0 else float("nan") for k in order]
            print(f"   {g:4d} " + " ".join(f"{x:8.2f}" for x in us))


if __name__ == "__main__":
    main()
