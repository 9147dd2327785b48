# SPDX-License-Identifier: Apache-2.0
"""Run the adjacent-step kernels a few times (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import mla
B, H = 16, 16
o = torch.randn((B, 1, H, 512), device="cuda")
w_uv = (torch.randn((H, 512, 128), device="cuda") * 0.05).to(torch.bfloat16)
q_nope = torch.randn((B, 1, H, 128), device="cuda").to(torch.bfloat16)
q_pe = torch.randn((B, 1, H, 64), device="cuda").to(torch.bfloat16)
w_uk = (torch.randn((H, 128, 512), device="cuda") * 0.05).to(torch.bfloat16)
cos = torch.ones((B, 1, 32), device="cuda"); sin = torch.zeros((B, 1, 32), device="cuda")
for _ in range(5):
    mla.up_proj(o, w_uv)
    mla.absorb_q(q_nope, q_pe, cos, sin, w_uk)
torch.cuda.synchronize()
