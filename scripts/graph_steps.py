# SPDX-License-Identifier: Apache-2.0
"""Device time per decode step with many steps in ONE CUDA graph (no host launch cost between
steps, programmatic dependent launch edges inside the graph), beside stream launches and the
host enqueue cost per step. Small contexts are where the host side can hide the kernel."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2506_01969_b200 import inputs, mla

NSTEPS = int(os.environ.get("NSTEPS", 20))


def run(seqlens, heads=16, fp8=False):
    L2 = 126 << 20
    kvb = sum(seqlens) * 576 * (1 if fp8 else 2)
    ncopies = max(1, min(NSTEPS, (2 * L2) // max(1, kvb) + 1))
    inps = [inputs.make_mla_inputs(seqlens, heads=heads, seed=42 + i, pad_value=0.0) for i in range(ncopies)]
    kv8 = [(i.kv_pool.float() / 0.125).to(torch.float8_e4m3fn) for i in inps] if fp8 else None
    B = len(seqlens)
    plan = mla.MlaDecodePlan.create(B, heads, "cuda")
    out = torch.empty((B, 1, heads, 512), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, 1, heads), dtype=torch.float32, device="cuda")

    def step(j):
        i = inps[j % ncopies]
        if fp8:
            plan.decode_fp8(i.q, kv8[j % ncopies], i.block_table, i.seqlens, i.scale, 0.125, out=out, lse=lse)
        else:
            plan.decode(i.q, i.kv_pool, i.block_table, i.seqlens, i.scale, out=out, lse=lse)

    for j in range(5):
        step(j)
    torch.cuda.synchronize()
    # host enqueue cost per step (no sync inside)
    t0 = time.perf_counter()
    for j in range(NSTEPS):
        step(j)
    host_us = (time.perf_counter() - t0) / NSTEPS * 1e6
    torch.cuda.synchronize()
    # stream launches, device time
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for j in range(NSTEPS):
        step(j)
    e1.record()
    torch.cuda.synchronize()
    stream_us = e0.elapsed_time(e1) * 1e3 / NSTEPS
    # NSTEPS steps in one graph
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for j in range(NSTEPS):
            step(j)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    res = []
    for _ in range(3):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1e3 / NSTEPS)
    graph_us = sorted(res)[1]
    print(json.dumps({"batch": B, "ctx": seqlens[0], "heads": heads, "fp8": fp8, "host_enqueue_us": round(host_us, 2),
                      "stream_us": round(stream_us, 2), f"graph_{NSTEPS}_steps_us": round(graph_us, 2)}), flush=True)


if __name__ == "__main__":
    run([1024])
    for ctx in (1024, 2048, 4096, 16384, 65536):
        run([ctx] * 16)
    run([1024] * 16, fp8=True)
    run([4096] * 16, fp8=True)
