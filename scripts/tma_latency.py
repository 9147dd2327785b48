# SPDX-License-Identifier: Apache-2.0
"""Per-SM TMA round trip of the decode's page boxes: one CTA pair streaming with 9 / 18 / 24
slots in flight, pages L2-resident (re-read) vs from HBM (L2 flushed before each launch).
rate = bytes in flight / round trip, so the slope gives the latency.

    python scripts/tma_latency.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import _lib

L = _lib.lib()
pages = 4096
pool = torch.zeros((pages, 64, 576), dtype=torch.bfloat16, device="cuda")
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
PB = 64 * 576 * 2
for fn_name in ("etap_mla_stream_bench", "etap_mla_stream_bench_page"):
  fn = getattr(L, fn_name) if fn_name.endswith("bench") else (lambda *a: L.etap_mla_stream_bench_page(*a[:5], 9, a[5]))
  print("==", fn_name, "(nine 8 KB chunk boxes per page)" if fn_name.endswith("bench") else "(one 72 KB 3-D box per page)")
  for ppc in (16, 110):
    for nslot in (9, 18, 24):
        for where in ("L2", "HBM"):
            ts = []
            for rep in range(8):
                if where == "HBM":
                    flush.fill_(rep)
                elif rep == 0:
                    _lib.check(fn(pool.data_ptr(), pages, ppc, 2, nslot, s), "stream")
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _lib.check(fn(pool.data_ptr(), pages, ppc, 2, nslot, s), "stream")
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1000)
            us = sorted(ts)[len(ts) // 2]
            rate = ppc * PB / us / 1e3
            print(f"  ppc {ppc:3d} nslot {nslot:2d} {where:3s}: {us:7.1f} us per launch, per-SM {rate:6.1f} GB/s, "
                  f"in flight {nslot * 8} KB -> round trip {nslot * 8192 / (rate * 1e3):.2f} us")
# under full load (148 CTAs, distinct pages, HBM-bound)
for fn_name in ("etap_mla_stream_bench", "etap_mla_stream_bench_page"):
    fn = getattr(L, fn_name) if fn_name.endswith("bench") else (lambda *a: L.etap_mla_stream_bench_page(*a[:5], 9, a[5]))
    big = torch.zeros((16 * 1024, 64, 576), dtype=torch.bfloat16, device="cuda") if fn_name.endswith("bench") else big
    for nslot in (18, 24):
        for _ in range(2):
            fn(big.data_ptr(), 16384, 110, 148, nslot, s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn(big.data_ptr(), 16384, 110, 148, nslot, s)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 100
        print(f"{fn_name} grid 148 nslot {nslot}: {us:.1f} us, chip {148 * 110 * PB / us / 1e3:.1f} GB/s")
