# SPDX-License-Identifier: Apache-2.0
"""The paper's central claim on B200: what the query-major order's head padding costs.

The reference models the claim (`/root/reference/proj/src/wgmma_model.cpp:56-86`,
`acceptance.cpp:142-185`): the query-major ("original") order puts the heads on the MMA M axis,
so 16 heads are padded to the 64-row minimum M and 3/4 of the QK^T and PV issued MACs are
padding; ETAP puts the KV rows on M and the 16 heads on N (steps of 8/16), with nothing padded.

Measured here with the same pipeline, schedule and HBM traffic: the ETAP decode of 16 heads
against the SAME decode with Q padded by zero heads to 32 / 64 / 128 columns. A padded column
costs what a query-major padded M row costs in tcgen05 work (M = 64 is the cta_group::1
minimum, M = 128 the full-rate shape), so the padded runs are a lower bound on a query-major
tcgen05 kernel's tensor work per byte. The 16 real heads of every padded run are checked
against the binary64 oracle (they must not change).

    python scripts/orientation_claim.py [--ctx 4096 16384 65536]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_2506_01969_b200 import inputs, mla

B, H = 16, 16


def timed(fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    res = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1000 / iters)
    return sorted(res)[1]


def model_issued(ctx: int) -> dict:
    """Issued / useful MACs of both orders from the tcgen05 restatement of the reference's
    WGMMA model (lib/etap_model, include/etaplab_b200_umma.hpp)."""
    exe = os.path.join(ROOT, "paper_2506_01969_b200", "lib", "etap_model")
    out = {}
    try:
        txt = subprocess.run([exe], capture_output=True, text=True, timeout=60).stdout.splitlines()
    except OSError:
        return out
    hdr = txt[0].split(",")
    for line in txt[1:]:
        row = dict(zip(hdr, line.split(",")))
        if int(row["heads"]) == H and int(row["kv_len"]) == ctx and int(row["batch"]) == 1:
            out[row["mode"]] = {"issued_over_useful": float(row["issued_macs"]) / float(row["useful_macs"]),
                                "predicted_speedup": float(row["predicted_speedup"])}
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, nargs="+", default=[4096, 16384, 65536])
    ap.add_argument("--check-ctx", type=int, default=4096, help="context of the oracle check of the padded arms")
    a = ap.parse_args()
    import oracle

    for ctx in a.ctx:
        inp = inputs.make_mla_inputs([ctx] * B, heads=H, seed=42, pad_value=0.0)
        line = {"config": f"B={B} ctx={ctx} 16 heads", "model": model_issued(ctx)}
        outs = {}
        for width in (16, 32, 64, 128):
            q = inp.q
            if width > H:  # zero heads appended: the query-major order's M padding
                q = torch.zeros((B, 1, width, 576), dtype=torch.bfloat16, device="cuda")
                q[:, :, :H] = inp.q
            plan = mla.MlaDecodePlan.create(B, width, "cuda")
            o = torch.empty((B, 1, width, 512), dtype=torch.float32, device="cuda")
            l = torch.empty((B, 1, width), dtype=torch.float32, device="cuda")
            f = lambda: plan.decode(q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=o, lse=l,  # noqa: E731
                                    flags=mla.FLAG_EARLY_METADATA)
            us = timed(f)
            f()
            torch.cuda.synchronize()
            outs[width] = (o[:, 0, :H].double().cpu().numpy(), l[:, 0, :H].double().cpu().numpy())
            line[f"us_width{width}"] = us
            line[f"head_group_width{width}"] = mla.head_group(width)
        line["padded64_over_etap"] = line["us_width64"] / line["us_width16"]
        line["padded128_over_etap"] = line["us_width128"] / line["us_width16"]
        if ctx == a.check_ctx:
            bits = lambda t: t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)  # noqa: E731
            o_ref, l_ref = oracle.mla_decode_bf16(bits(inp.q)[:, 0], bits(inp.kv_pool), inp.block_table.cpu().numpy(),
                                                  inp.seqlens.cpu().numpy(), inp.scale)
            line["rmse_vs_oracle"] = {w: math.sqrt(float(np.mean((oo - o_ref) ** 2))) for w, (oo, _) in outs.items()}
            line["lse_maxabs_vs_oracle"] = {w: float(np.abs(ll - l_ref).max()) for w, (_, ll) in outs.items()}
        print(json.dumps(line), flush=True)
        del inp
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
