# SPDX-License-Identifier: Apache-2.0
"""Attainable HBM read rate for the decode kernel's TMA pattern (no compute)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import _lib

pages = 16 * 1024
pool = torch.zeros((pages, 64, 576), dtype=torch.bfloat16, device="cuda")
L = _lib.lib()
for grid in (148, 296):
    for nslot in (18, 24):
        ppc = pages // grid
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            _lib.check(L.etap_mla_stream_bench(pool.data_ptr(), pages, ppc, grid, nslot, s), "stream")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 20
        for _ in range(n):
            L.etap_mla_stream_bench(pool.data_ptr(), pages, ppc, grid, nslot, s)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000 / n
        nbytes = ppc * grid * 64 * 576 * 2
        print(f"grid {grid} nslot {nslot}: {us:.1f} us, {nbytes / us / 1e3:.1f} GB/s")
# plain copy-engine / torch read reference
x = pool.view(-1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): x.sum()
e0.record()
for _ in range(10): x.float().sum() if False else x.sum()
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1000 / 10
print(f"torch sum over pool: {us:.1f} us, {x.numel() * 2 / us / 1e3:.1f} GB/s")
