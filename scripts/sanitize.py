# SPDX-License-Identifier: Apache-2.0
"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
bf16 with head groups of 16 and 32, MTP, the FP8 path, the combine and K1 paths, and the
serving step from page-locked host buffers (ingest kernel, O / LSE stored to host memory).
    compute-sanitizer --tool memcheck python scripts/sanitize.py"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2506_01969_b200 import inputs, mla


def run() -> None:
    cases = [([300, 1, 0, 129], 16, 1, 148), ([700, 65], 32, 1, 7), ([200, 90], 16, 2, 148), ([5000], 64, 1, 148),
             ([3000, 64, 1, 777], 128, 1, 9), ([900, 4100], 96, 1, 148), ([640, 70], 64, 2, 5),
             ([1000, 300], 256, 1, 148), ([2000, 65], 128, 1, 148),  # CTA-pair kernel (128-head units)
             ([70 * (i % 5 + 1) for i in range(20)], 16, 1, 3)]  # FP8: > 4 splits per CTA (warp-3 Q terms)
    for seqlens, heads, t, parts in cases:
        inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=3, pad_value=float("nan"), q_tokens=t)
        plan = mla.MlaDecodePlan.create(len(seqlens), heads, "cuda", parts, q_tokens=t)
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
        if heads == 16:
            kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
            plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125)
    for n in (140, 300):  # block-wide fused schedule (<= 256 work units), then K1 + K2 + K3
        seqlens = [64] * n
        inp = inputs.make_mla_inputs(seqlens, heads=16, seed=5, pad_value=0.0)
        plan = mla.MlaDecodePlan.create(len(seqlens), 16, "cuda")
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    torch.cuda.synchronize()
    # serving step from page-locked host buffers: ingest kernel + O / LSE stored to host memory
    import ctypes as C

    from paper_2506_01969_b200 import _lib
    L = _lib.lib()
    seqlens = [300, 1, 129]
    inp = inputs.make_mla_inputs(seqlens, heads=16, seed=7, pad_value=0.0)
    last = inp.seqlens.long() - 1
    pages = inp.block_table.gather(1, (last // 64).unsqueeze(1)).squeeze(1).long()
    rows = inp.kv_pool[pages, last % 64].contiguous().cpu().pin_memory()
    q_h, sl_h = inp.q.cpu().pin_memory(), inp.seqlens.cpu().pin_memory()
    o_h, l_h = torch.empty((3, 16, 512)).pin_memory(), torch.empty((3, 16)).pin_memory()
    kv_h, bt_h = inp.kv_pool.cpu(), inp.block_table.cpu()
    ctx = C.c_void_p()
    _lib.check(L.etap_mla_host_ctx_create(3, 16, inp.kv_pool.shape[0], inp.block_table.shape[1], C.byref(ctx)), "ctx")
    _lib.check(L.etap_mla_host_ctx_load(ctx, kv_h.data_ptr(), bt_h.data_ptr()), "load")
    _lib.check(L.etap_mla_host_decode_step(ctx, q_h.data_ptr(), rows.data_ptr(), sl_h.data_ptr(), inp.scale, 0,
                                           o_h.data_ptr(), l_h.data_ptr()), "step")
    L.etap_mla_host_ctx_destroy(ctx)
    print("sanitize cases done")


if __name__ == "__main__":
    run()
