# SPDX-License-Identifier: Apache-2.0
"""Tensor-pipe microbenchmark of the UMMA operand variants / issue styles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import _lib

names = {0: "M128 N16 A-Kmaj", 1: "M128 N16 A-MNmaj B-MN", 2: "M128 N32 A-MNmaj B-MN", 3: "M64 N16 A-Kmaj",
         4: "M128 N64 A-Kmaj", 5: "M128 N16 A-MNmaj B-Kmaj", 6: "M128 N256 A-Kmaj"}
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for mode in (0, 1):
    for v in range(7):
        n = 256
        _lib.check(_lib.lib().etap_mla_umma_bench(mode * 10 + v, n, out.data_ptr(), 1), "bench")
        torch.cuda.synchronize()
        iss, tot = out.tolist()
        print(f"{'divergent' if mode == 0 else 'warp-elect':10s} {names[v]:26s} n={n:4d}: issue {iss/n:6.1f} cyc/mma, complete {tot/n:6.1f} cyc/mma")
