# SPDX-License-Identifier: Apache-2.0
"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
bf16 with head groups of 16 and 32, MTP, the FP8 path, the combine and K1 paths.
    compute-sanitizer --tool memcheck python scripts/sanitize.py"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2506_01969_b200 import inputs, mla


def run() -> None:
    cases = [([300, 1, 0, 129], 16, 1, 148), ([700, 65], 32, 1, 7), ([200, 90], 16, 2, 148), ([5000], 64, 1, 148),
             ([70 * (i % 5 + 1) for i in range(20)], 16, 1, 3)]  # FP8: > 4 splits per CTA (warp-3 Q terms)
    for seqlens, heads, t, parts in cases:
        inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=3, pad_value=float("nan"), q_tokens=t)
        plan = mla.MlaDecodePlan.create(len(seqlens), heads, "cuda", parts, q_tokens=t)
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
        if heads == 16:
            kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
            plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125)
    seqlens = [64] * 140  # > 128 work units: K1 + K2 + K3
    inp = inputs.make_mla_inputs(seqlens, heads=16, seed=5, pad_value=0.0)
    plan = mla.MlaDecodePlan.create(len(seqlens), 16, "cuda")
    plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    run()
