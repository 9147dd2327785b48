# SPDX-License-Identifier: Apache-2.0
"""Run the decode step a few times on one config (for ncu launch lists / captures)."""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

from paper_2506_01969_b200 import inputs, mla


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=65536)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--fp8", action="store_true", help="FP8 (e4m3) latent cache, decode_fp8")
    a = ap.parse_args()
    inp = inputs.make_mla_inputs([a.ctx] * a.batch, heads=a.heads, pad_value=0.0)
    plan = mla.MlaDecodePlan.create(a.batch, a.heads, "cuda")
    if a.fp8:
        kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
        for _ in range(a.iters):
            plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125)
        torch.cuda.synchronize()
        print("ok")
        return
    for _ in range(a.iters):
        plan.metadata(inp.seqlens)
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
