# SPDX-License-Identifier: Apache-2.0
"""Exit-time spread of the product K2's CTAs (per-CTA %globaltimer span stamps, programmatic
launch intact) over many back-to-back steps: is the tail systematic per CTA / SM?

    python scripts/tail_spread.py [--heads 16] [--fp8] [--steps 60]
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2506_01969_b200 import _lib, inputs, mla


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--fp8", action="store_true")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--rotate", type=int, default=0, help="rotate the sequences by this many slots")
    a = ap.parse_args()
    inp = inputs.make_mla_inputs([a.ctx] * 16, heads=a.heads, pad_value=0.0, seed=a.seed)
    if a.rotate:
        inp.block_table = torch.roll(inp.block_table, a.rotate, 0).contiguous()
    plan = mla.MlaDecodePlan.create(16, a.heads, "cuda")
    out = torch.empty((16, 1, a.heads, 512), dtype=torch.float32, device="cuda")
    lse = torch.empty((16, 1, a.heads), dtype=torch.float32, device="cuda")
    kv = inp.kv_pool
    if a.fp8:
        kv = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)

    def step():
        if a.fp8:
            plan.decode_fp8(inp.q, kv, inp.block_table, inp.seqlens, inp.scale, 0.125, out=out, lse=lse,
                            flags=mla.FLAG_EARLY_METADATA)
        else:
            plan.decode(inp.q, kv, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse,
                        flags=mla.FLAG_EARLY_METADATA)

    L = _lib.lib()
    n = plan.num_sm_parts
    sp = torch.zeros((a.steps, n, 2), dtype=torch.int64, device="cuda")
    for _ in range(10):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.steps):
        L.etap_mla_debug_span(sp[i].data_ptr())
        step()
    e1.record()
    torch.cuda.synchronize()
    L.etap_mla_debug_span(None)
    print(f"step {e0.elapsed_time(e1) * 1000 / a.steps:.1f} us (stream launches, span stamps on)")
    s = sp.cpu().numpy().astype(np.int64)
    t0 = s[:, :, 0].min(axis=1, keepdims=True)
    ex = (s[:, :, 1] - t0) / 1e3           # exit of each CTA after the launch's first dependency resolution
    dep = (s[:, :, 0] - t0) / 1e3
    k2 = ex.max(axis=1)
    print(f"K2 span us: median {np.median(k2):.1f} min {k2.min():.1f} max {k2.max():.1f}")
    q = np.percentile(ex, [0, 10, 50, 90, 100], axis=1).mean(axis=1)
    print("CTA exit us (mean over launches of per-launch percentiles) p0/p10/p50/p90/p100:",
          " / ".join(f"{v:.1f}" for v in q))
    print(f"dependency-resolution spread us (median over launches): {np.median(dep.max(axis=1)):.2f}")
    m = ex.mean(axis=0)
    half = a.steps // 2
    c = np.corrcoef(ex[:half].mean(axis=0), ex[half:].mean(axis=0))[0, 1]
    print(f"per-CTA mean exit: min {m.min():.1f} median {np.median(m):.1f} max {m.max():.1f}; "
          f"first-half vs second-half correlation {c:.2f}")
    order = np.argsort(m)
    print("slowest CTAs (blockIdx, mean exit us):", [(int(i), round(float(m[i]), 1)) for i in order[-10:]])
    print("fastest CTAs:", [(int(i), round(float(m[i]), 1)) for i in order[:6]])
    # how many CTAs are still running in the tail (median over launches)
    for back in (1, 2, 3, 4, 6, 8):
        alive = (ex > (k2[:, None] - back)).sum(axis=1)
        print(f"  CTAs still running {back} us before the last exit: {np.median(alive):.0f}")
    np.save("gpurun_out/tail_exit_%s%d_s%d_r%d.npy" % ("fp8_" if a.fp8 else "", a.heads, a.seed, a.rotate), ex)


if __name__ == "__main__":
    main()
