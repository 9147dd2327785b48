# SPDX-License-Identifier: Apache-2.0
"""Step time vs the number of decode CTAs (num_sm_parts < SM count leaves SMs free for the
combine of the previous step under ETAP_FLAG_INDEPENDENT_INPUTS). Device-timed loop of K steps.

    python scripts/parts_probe.py [--kv fp8] [--heads 16] [--parts 148,144,140,136]
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2506_01969_b200 import inputs, mla


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--kv", default="bf16")
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--parts", default="148,146,144,142,140,136,132")
    a = ap.parse_args()
    inp = inputs.make_mla_inputs([a.ctx] * a.batch, heads=a.heads, pad_value=0.0)
    kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn) if a.kv == "fp8" else None
    fl = mla.FLAG_INDEPENDENT_INPUTS
    for rnd in range(2):
        for n in (int(x) for x in a.parts.split(",")):
            plan = mla.MlaDecodePlan.create(a.batch, a.heads, "cuda", num_parts=n)
            if kv8 is not None:
                f = lambda: plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125, flags=fl)
            else:
                f = lambda: plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=fl)
            for _ in range(10):
                f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                f()
            e1.record()
            torch.cuda.synchronize()
            print(f"round {rnd} kv={a.kv} heads={a.heads} parts={n}: {e0.elapsed_time(e1) * 1000 / a.steps:.2f} us/step",
                  flush=True)


if __name__ == "__main__":
    main()
