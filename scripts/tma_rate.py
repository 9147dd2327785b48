# SPDX-License-Identifier: Apache-2.0
"""Per-SM TMA ingest rate with the decode's box pattern (no compute): alone vs under load,
HBM vs L2-resident pages, unicast vs cluster multicast (two CTAs streaming the same pages).

    python scripts/tma_rate.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import _lib

L = _lib.lib()
pages = 16 * 1024
pool = torch.zeros((pages, 64, 576), dtype=torch.bfloat16, device="cuda")
s = torch.cuda.current_stream().cuda_stream
PB = 64 * 576 * 2


def run(fn, grid, ppc, nslot, n=10):
    for _ in range(2):
        _lib.check(fn(pool.data_ptr(), pages, ppc, grid, nslot, s), "stream")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn(pool.data_ptr(), pages, ppc, grid, nslot, s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / n


for nslot in (18, 24):
    for grid in (2, 16, 74, 148):
        ppc = min(110, pages // grid)
        us = run(L.etap_mla_stream_bench, grid, ppc, nslot)
        print(f"unicast   nslot {nslot} grid {grid:3d} ppc {ppc}: {us:7.1f} us  per-SM ingest {ppc * PB / us / 1e3:6.1f} GB/s  "
              f"chip HBM {grid * ppc * PB / us / 1e3:7.1f} GB/s")
        # multicast pairs: grid CTAs, grid/2 distinct page ranges -> each SM ingests ppc pages
        ppc2 = min(110, pages // (grid // 2))
        us = run(L.etap_mla_stream_bench_mc, grid, ppc2, nslot)
        print(f"multicast nslot {nslot} grid {grid:3d} ppc {ppc2}: {us:7.1f} us  per-SM ingest {ppc2 * PB / us / 1e3:6.1f} GB/s  "
              f"chip HBM {(grid // 2) * ppc2 * PB / us / 1e3:7.1f} GB/s")
    # L2-resident: few pages re-read (grid CTAs all stream the same 40 pages region)
