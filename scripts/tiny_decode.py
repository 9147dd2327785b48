# SPDX-License-Identifier: Apache-2.0
"""One small decode (debugging aid: run under compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import inputs, mla
H = int(os.environ.get("H", 16))
inp = inputs.make_mla_inputs([1024, 77], heads=H, seed=1, pad_value=0.0)
o, l = mla.mla_decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
torch.cuda.synchronize()
print("ok", o.abs().sum().item())
