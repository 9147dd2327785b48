# SPDX-License-Identifier: Apache-2.0
"""Wall time of etap_mla_host_decode_step (the C-ABI serving step, bench.py's e2e_serving) at
several contexts with page-locked and pageable host buffers, beside the device-only step."""
import ctypes as C
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import _lib, inputs, mla

L = _lib.lib()
for ctx_len in (1024, 4096, 65536):
    B, H = 16, 16
    inp = inputs.make_mla_inputs([ctx_len] * B, heads=H, pad_value=0.0)
    last = inp.seqlens.long() - 1
    pages = inp.block_table.gather(1, (last // 64).unsqueeze(1)).squeeze(1).long()
    rows = inp.kv_pool[pages, last % 64].contiguous().cpu()
    plan = mla.MlaDecodePlan.create(B, H, "cuda")
    out = torch.empty((B, 1, H, 512), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, 1, H), dtype=torch.float32, device="cuda")
    for _ in range(5):
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse)
    e1.record()
    torch.cuda.synchronize()
    dev_us = e0.elapsed_time(e1) * 1e3 / 50
    ctx = C.c_void_p()
    _lib.check(L.etap_mla_host_ctx_create(B, H, inp.kv_pool.shape[0], inp.block_table.shape[1], C.byref(ctx)), "ctx")
    kv_h, bt_h = inp.kv_pool.cpu(), inp.block_table.cpu()
    _lib.check(L.etap_mla_host_ctx_load(ctx, kv_h.data_ptr(), bt_h.data_ptr()), "load")
    res = {}
    for pinned in (True, False):
        p = (lambda t: t.pin_memory()) if pinned else (lambda t: t)
        q_h, r_h, s_h = p(inp.q.cpu()), p(rows), p(inp.seqlens.cpu())
        o_h, l_h = p(torch.empty((B, H, 512))), p(torch.empty((B, H)))
        call = lambda: _lib.check(L.etap_mla_host_decode_step(ctx, q_h.data_ptr(), r_h.data_ptr(), s_h.data_ptr(),
                                                               inp.scale, 0, o_h.data_ptr(), l_h.data_ptr()), "step")
        for _ in range(5):
            call()
        t0 = time.perf_counter()
        for _ in range(50):
            call()
        res["pinned" if pinned else "pageable"] = (time.perf_counter() - t0) / 50 * 1e6
    L.etap_mla_host_ctx_destroy(ctx)
    print(f"ctx {ctx_len}: device step {dev_us:.1f} us; host_decode_step wall pinned {res['pinned']:.1f} us, "
          f"pageable {res['pageable']:.1f} us", flush=True)
