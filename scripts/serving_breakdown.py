# SPDX-License-Identifier: Apache-2.0
"""Where a serving decode step's time goes beyond the device step, on the COPY path of
etap_mla_host_decode_step (pageable host buffers: H2D of Q / new rows / seqlens, append, decode,
D2H of O / LSE, synchronize), with CUDA events between the pieces, plus the wall time. This
breakdown is what motivated the page-locked path (one ingest kernel, O / LSE stored to host
memory); scripts/serving_step.py times both paths through the C-ABI."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_01969_b200 import _lib, inputs, mla

B, H, CTX = 16, 16, int(os.environ.get("CTX", 65536))
inp = inputs.make_mla_inputs([CTX] * B, heads=H, pad_value=0.0)
plan = mla.MlaDecodePlan.create(B, H, "cuda")
L = _lib.lib()
last = (inp.seqlens.long() - 1)
pages = inp.block_table.gather(1, (last // 64).unsqueeze(1)).squeeze(1).long()
rows_h = inp.kv_pool[pages, last % 64].contiguous().cpu().pin_memory()
q_h, sl_h = inp.q.cpu().pin_memory(), inp.seqlens.cpu().pin_memory()
q_d, rows_d, sl_d = torch.empty_like(inp.q), torch.empty_like(rows_h, device="cuda"), torch.empty_like(inp.seqlens)
out_d = torch.empty((B, 1, H, 512), dtype=torch.float32, device="cuda")
lse_d = torch.empty((B, 1, H), dtype=torch.float32, device="cuda")
out_h, lse_h = torch.empty_like(out_d, device="cpu").pin_memory(), torch.empty_like(lse_d, device="cpu").pin_memory()
st = torch.cuda.current_stream()
names = ["H2D q", "H2D rows", "H2D seqlens", "append", "decode K2+K3", "D2H O", "D2H LSE"]


def step(evs=None):
    def mark(i):
        if evs is not None:
            evs[i].record()
    mark(0)
    q_d.copy_(q_h, non_blocking=True); mark(1)
    rows_d.copy_(rows_h, non_blocking=True); mark(2)
    sl_d.copy_(sl_h, non_blocking=True); mark(3)
    _lib.check(L.etap_mla_append_kv(rows_d.data_ptr(), inp.kv_pool.data_ptr(), inp.kv_pool.shape[0],
                                    inp.block_table.data_ptr(), inp.block_table.shape[1], sl_d.data_ptr(), B, 1,
                                    st.cuda_stream), "append"); mark(4)
    plan.decode(q_d, inp.kv_pool, inp.block_table, sl_d, inp.scale, out=out_d, lse=lse_d); mark(5)
    out_h.copy_(out_d, non_blocking=True); mark(6)
    lse_h.copy_(lse_d, non_blocking=True); mark(7)
    torch.cuda.synchronize()


for _ in range(5):
    step()
t0 = time.perf_counter()
for _ in range(50):
    step()
wall = (time.perf_counter() - t0) / 50 * 1e6
evs = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
acc = [0.0] * 7
for _ in range(20):
    step(evs)
    for i in range(7):
        acc[i] += evs[i].elapsed_time(evs[i + 1]) * 1e3 / 20
print(f"ctx {CTX}: wall {wall:.1f} us/step; device pieces (events): " +
      ", ".join(f"{n} {a:.1f}" for n, a in zip(names, acc)) + f"; sum {sum(acc):.1f}")
