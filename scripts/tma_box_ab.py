# SPDX-License-Identifier: Apache-2.0
"""Full-load A/B of the TMA box shape for the decode's page stream (148 CTAs, distinct pages,
HBM-bound, no compute): nine 2-D chunk boxes per page vs 3-D boxes of 1 / 3 / 9 chunks.
Interleaved repetitions; prints the median chip rate per variant.

    python scripts/tma_box_ab.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2506_01969_b200 import _lib

L = _lib.lib()
pages = 16 * 1024
pool = torch.zeros((pages, 64, 576), dtype=torch.bfloat16, device="cuda")
s = torch.cuda.current_stream().cuda_stream
PB = 64 * 576 * 2
variants = {"2d x9": lambda ns: L.etap_mla_stream_bench(pool.data_ptr(), pages, 110, 148, ns, s)}
for bc in (1, 3, 9):
    variants[f"3d box {bc}"] = (lambda bc_: lambda ns: L.etap_mla_stream_bench_page(pool.data_ptr(), pages, 110, 148, ns, bc_, s))(bc)
for nslot in (18, 24):
    res = {k: [] for k in variants}
    for rep in range(6):
        for k, f in variants.items():
            f(nslot)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                f(nslot)
            e1.record()
            torch.cuda.synchronize()
            res[k].append(e0.elapsed_time(e1) * 100)
    for k, v in res.items():
        us = float(np.median(v))
        print(f"nslot {nslot} {k:9s}: {us:7.1f} us  {148 * 110 * PB / us / 1e3:7.1f} GB/s  (min {min(v):.1f} max {max(v):.1f})")
