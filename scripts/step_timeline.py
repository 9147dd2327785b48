# SPDX-License-Identifier: Apache-2.0
"""Cross-kernel timeline of consecutive decode steps (K2 + K3) from %globaltimer stamps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2506_01969_b200 import _lib, inputs, mla

B, CTX, H = int(os.environ.get("B", 16)), int(os.environ.get("CTX", 1024)), int(os.environ.get("HEADS", 16))
inp = inputs.make_mla_inputs([CTX] * B, heads=H, pad_value=0.0)
plan = mla.MlaDecodePlan.create(B, H, "cuda")
n, TT, STEPS = plan.num_sm_parts, 256, 4
k2 = [torch.zeros(n * TT * 16, dtype=torch.int64, device="cuda") for _ in range(STEPS)]
k3 = [torch.zeros(B * H * 4, dtype=torch.int64, device="cuda") for _ in range(STEPS)]
L = _lib.lib()
# EARLY=1: the opt-in early schedule; INDEP=1: the bench's flags (independent inputs, implies early)
FL = (mla.FLAG_INDEPENDENT_INPUTS if os.environ.get("INDEP") else
      mla.FLAG_EARLY_METADATA if os.environ.get("EARLY") else 0)
f = lambda: plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=FL)
if os.environ.get("FP8"):  # FP8 (e4m3) latent cache
    kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
    f = lambda: plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125, flags=FL)
for _ in range(5): f()
torch.cuda.synchronize()
for i in range(STEPS):  # back to back, a different trace buffer per step
    L.etap_mla_debug_trace(k2[i].data_ptr())
    L.etap_mla_debug_trace_combine(k3[i].data_ptr())
    f()
L.etap_mla_debug_trace(None); L.etap_mla_debug_trace_combine(None)
torch.cuda.synchronize()
# re-base %globaltimer ns in int64 before float conversion (float64 ulp at 1.7e18 ns is 256 ns)
gbase = int(k2[0].view(n, TT, 16)[:, TT - 1, 0].min().item())
t0 = 0.0
for i in range(STEPS):
    g = k2[i].view(n, TT, 16).cpu().numpy()[:, TT - 1, :]
    a = (g[:, :3] - gbase).astype(np.float64)
    ex = (g[:, 7:12] - gbase).astype(np.float64)  # dep-wait done, seqlens in, first KV TMA, last epilogue, softmax done
    c = k3[i].view(-1, 4).cpu().numpy()[:, :3]
    c = (c[c[:, 2] > 0] - gbase).astype(np.float64)
    r = lambda x: (x - t0) / 1e3
    print(f"step {i}: K2 entry {r(a[:,0].min()):7.2f}..{r(a[:,0].max()):7.2f}  sched-done med {r(np.median(a[:,1])):7.2f}  "
          f"exit med {r(np.median(a[:,2])):7.2f} max {r(a[:,2].max()):7.2f} | K3 entry min {r(c[:,0].min()):7.2f} "
          f"wait-release min {r(c[:,1].min()):7.2f} exit max {r(c[:,2].max()):7.2f}")
    m = lambda j: r(np.median(ex[:, j]))
    print(f"        dep-wait done med {m(0):7.2f} (min {r(ex[:,0].min()):7.2f})  seqlens-in med {m(1):7.2f}  "
          f"first-KV-TMA med {m(2):7.2f}  last-epilogue med {m(3):7.2f}  softmax-done med {m(4):7.2f}")
    if os.environ.get("FP8"):
        print(f"        first Q terms published med {r(np.median((g[:, 4] - gbase).astype(np.float64))):7.2f}")
    ck = g[:, 12:16].astype(np.int64)
    d = np.median(ck[:, 1:] - ck[:, :1], axis=0)
    print(f"        clock64 after dep-wait: seqlens-in +{d[0]:.0f}  sched-done +{d[1]:.0f}  first-KV-TMA +{d[2]:.0f} cycles")
    m = lambda j: r(np.median(ex[:, j]))
    print(f"        dep-wait done med {m(0):7.2f} (min {r(ex[:,0].min()):7.2f})  seqlens-in med {m(1):7.2f}  "
          f"first-KV-TMA med {m(2):7.2f}  last-epilogue med {m(3):7.2f}  softmax-done med {m(4):7.2f}")
