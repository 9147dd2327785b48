# SPDX-License-Identifier: Apache-2.0
"""The CTA-pair decode (128-head work units): parity against the oracle on small cases, then the
B=16 x 64K x 128-head step time (CUDA events, stream launches). Run with ETAP_PAIR=0 for the
single-CTA head-group-64 kernel on the same cases (A/B). Exits 1 on a parity miss."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_2506_01969_b200 import inputs, mla


def bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def check(seqlens, heads, q_tokens=1, causal=True, seed=5, num_parts=None, flags=0, idx=None):
    inp = inputs.make_mla_inputs(seqlens, heads=heads, q_tokens=q_tokens, seed=seed, pad_value=float("nan"))
    plan = mla.MlaDecodePlan.create(len(seqlens), heads, "cuda", num_parts, q_tokens=q_tokens)
    o, l = plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=flags, causal=causal)
    torch.cuda.synchronize()
    idx = list(range(len(seqlens))) if idx is None else idx
    q = bits(inp.q)[idx]
    bt = inp.block_table.cpu().numpy()[idx]
    sl = inp.seqlens.cpu().numpy()[idx]
    if q_tokens == 1:
        o_ref, l_ref = oracle.mla_decode_bf16(q[:, 0], bits(inp.kv_pool), bt, sl, inp.scale)
        o_ref, l_ref = o_ref[:, None], l_ref[:, None]
    else:
        o_ref, l_ref = oracle.mla_decode_bf16_tokens(q, bits(inp.kv_pool), bt, sl, inp.scale, causal)
    o = o.double().cpu().numpy()[idx]
    l = l.double().cpu().numpy()[idx]
    ne = np.array([s > 0 for s in sl])
    err = float(np.sqrt(np.mean((o[ne] - o_ref[ne]) ** 2))) if ne.any() else 0.0
    lerr = float(np.abs(l[ne] - l_ref[ne]).max()) if ne.any() else 0.0
    ok = np.isfinite(o).all() and err <= 2e-5 and lerr <= 1e-4
    if (~ne).any():
        ok = ok and (o[~ne] == 0).all() and np.isneginf(l[~ne]).all()
    print(f"heads={heads} T={q_tokens} seqlens={seqlens[:6]}{'...' if len(seqlens) > 6 else ''} parts={num_parts} "
          f"rmse={err:.2e} lse={lerr:.1e} {'ok' if ok else 'FAIL'}", flush=True)
    return ok


def main():
    bad = 0
    cases = [
        dict(seqlens=[64], heads=128),
        dict(seqlens=[1], heads=128),
        dict(seqlens=[300, 1500], heads=128),
        dict(seqlens=[3000, 64, 1, 777], heads=128),
        dict(seqlens=[0, 100, 0, 64], heads=128),
        dict(seqlens=[2048] * 4, heads=256),
        dict(seqlens=[4097, 65, 1000], heads=64, q_tokens=2),
        dict(seqlens=[4097, 65, 1000], heads=32, q_tokens=4, causal=True),
        dict(seqlens=[5000, 3000], heads=128, num_parts=2),
        dict(seqlens=[5000, 3000], heads=128, num_parts=7),
        dict(seqlens=[(131 * i) % 300 + 1 for i in range(65)], heads=128, idx=[0, 1, 40, 64]),
        dict(seqlens=[65536, 1000], heads=128, idx=[1]),
    ]
    for c in cases:
        bad += not check(**c)
    for flags, name in ((mla.FLAG_EAGER_RESCALE, "eager"),):
        bad += not check([3000, 700], 128, flags=flags)
    if "--no-time" in sys.argv:
        sys.exit(1 if bad else 0)
    for heads in (128,):
        seqlens = [65536] * 16
        inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=1)
        plan = mla.MlaDecodePlan.create(16, heads, "cuda")
        out = torch.empty((16, 1, heads, 512), dtype=torch.float32, device="cuda")
        lse = torch.empty((16, 1, heads), dtype=torch.float32, device="cuda")
        for _ in range(5):
            plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse)
        torch.cuda.synchronize()
        times = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1000 / 20)
        print(f"TIME heads={heads} B=16 ctx=64K pair={os.environ.get('ETAP_PAIR', '1')} us/step={min(times):.1f} "
              f"all={[round(t, 1) for t in times]}", flush=True)
        # a long-context sample against the oracle (one sequence, two heads' worth of rows checked)
        o = out.double().cpu().numpy()
        q = bits(inp.q)[:1]
        o_ref, l_ref = oracle.mla_decode_bf16(q[:, 0], bits(inp.kv_pool), inp.block_table.cpu().numpy()[:1],
                                              inp.seqlens.cpu().numpy()[:1], inp.scale)
        err = float(np.sqrt(np.mean((o[0, 0] - o_ref[0]) ** 2)))
        print(f"64K seq0 rmse={err:.2e} {'ok' if err <= 2e-5 else 'FAIL'}", flush=True)
        bad += err > 2e-5
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
