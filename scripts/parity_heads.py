# SPDX-License-Identifier: Apache-2.0
"""Parity of the paged decode against the oracle for several head counts (run with
ETAP_HEAD_GROUP=16 to force 16-head work units). Prints one line per case; exits 1 on a miss."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_2506_01969_b200 import inputs, mla

bad = 0
for seqlens, heads in [([4096] * 4, 32), ([4096] * 16, 32), ([3000, 64, 1, 777], 64), ([2048] * 4, 128),
                       ([65536] * 2, 32)]:
    inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=5, pad_value=float("nan"))
    plan = mla.MlaDecodePlan.create(len(seqlens), heads, "cuda")
    o, l = plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    torch.cuda.synchronize()
    err = 0.0
    for b, s in enumerate(seqlens[:2]):
        q = inp.q[b, 0].double().cpu().numpy()
        pages = inp.block_table[b, :(s + 63) // 64].long()
        kv = inp.kv_pool[pages].reshape(-1, 576)[:s].double().cpu().numpy()
        o_ref, l_ref = oracle.attention_ref(q, kv, kv[:, :512], inp.scale)
        err = max(err, float(np.sqrt(np.mean((o[b, 0].double().cpu().numpy() - o_ref) ** 2))))
    ok = err <= 2e-5
    bad += not ok
    print(f"hg={mla.head_group(heads)} heads={heads} seqlens={seqlens[:4]} rmse={err:.2e} {'ok' if ok else 'FAIL'}",
          flush=True)
sys.exit(1 if bad else 0)
