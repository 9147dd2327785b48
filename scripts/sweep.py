# SPDX-License-Identifier: Apache-2.0
"""Measure the BASELINE.json configs besides the headline one (one JSON line each):
config 1 (B=1, 16 heads, 1K), config 3 (B=16, 16 heads, ctx 1K..64K), config 4 (B=32
varlen 4K..128K), and the 128-head single-GPU point of config 5. Device time per step with
CUDA events (median of repeated blocks), stream launches and CUDA-graph replay; L2 is flushed
between steps for working sets below 2x L2 (KV buffer rotation)."""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2506_01969_b200 import inputs, mla

L2_BYTES = 126 * 1024 * 1024
GRAPH_STEPS = 20


def graph_multi(step) -> float:
    """GRAPH_STEPS consecutive steps in ONE CUDA graph (programmatic edges between them): the
    device time per step without the host's per-call cost (~10-15 us through Python, ~7 us
    through the C-ABI), which is what a serving loop that graphs its decode step sees."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    gm = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s), torch.cuda.graph(gm, stream=s):
        for j in range(GRAPH_STEPS):
            step(j)
    torch.cuda.synchronize()
    res = []
    for _ in range(3):
        gm.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gm.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1000 / GRAPH_STEPS)
    del gm
    return sorted(res)[1]


def measure(seqlens, heads, label, iters=50, q_tokens=1):
    kv_bytes = sum(seqlens) * 576 * 2
    ncopies = max(1, min(8, (2 * L2_BYTES) // max(1, kv_bytes) + 1))  # rotate through > L2
    inps = [inputs.make_mla_inputs(seqlens, heads=heads, seed=42 + i, pad_value=0.0, q_tokens=q_tokens)
            for i in range(ncopies)]
    B = len(seqlens)
    plan = mla.MlaDecodePlan.create(B, heads, "cuda", q_tokens=q_tokens)
    out = torch.empty((B, q_tokens, heads, 512), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, q_tokens, heads), dtype=torch.float32, device="cuda")
    graphs = [plan.capture(i.q, i.kv_pool, i.block_table, i.seqlens, i.scale, out, lse, with_metadata=False)
              for i in inps]

    def timed(fn):
        for j in range(5):
            fn(j)
        torch.cuda.synchronize()
        res = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for j in range(iters):
                fn(j)
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) * 1000 / iters)
        return sorted(res)[1]

    def stream_step(j):
        i = inps[j % ncopies]
        plan.decode(i.q, i.kv_pool, i.block_table, i.seqlens, i.scale, out=out, lse=lse)

    us_stream = timed(stream_step)
    us_graph = timed(lambda j: graphs[j % ncopies].replay())
    us_graph_multi = graph_multi(stream_step)
    nbytes = inputs.algorithmic_bytes(seqlens, heads * q_tokens)
    best = min(us_stream, us_graph, us_graph_multi)
    line = {"config": label, "batch": B, "heads": heads, "ctx_total": sum(seqlens),
            "ctx_min": min(seqlens), "ctx_max": max(seqlens), "us_per_step_stream": us_stream,
            "us_per_step_graph": us_graph, f"us_per_step_graph{GRAPH_STEPS}": us_graph_multi, "hbm_gbs": nbytes / best / 1e3,
            "tflops": inputs.flops(seqlens, heads * q_tokens) / best / 1e6, "q_tokens": q_tokens, "algorithmic_bytes": nbytes,
            "l2_rotation_copies": ncopies}
    print(json.dumps(line), flush=True)
    del inps, graphs
    torch.cuda.empty_cache()


def measure_layer(B=16, H=16, ctx=65536, iters=50):
    """Absorbed-MLA attention step: absorb_q (q_nope . W_UK + RoPE) -> decode -> up_proj
    (O . W_UV), device time per piece and for the chained step (CUDA events, stream launches)."""
    import math
    inp = inputs.make_mla_inputs([ctx] * B, heads=H, seed=42, pad_value=0.0)
    g = torch.Generator(device="cuda").manual_seed(1)
    q_nope = torch.randn((B, 1, H, 128), generator=g, device="cuda").to(torch.bfloat16)
    q_pe = torch.randn((B, 1, H, 64), generator=g, device="cuda").to(torch.bfloat16)
    w_uk = (torch.randn((H, 128, 512), generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    w_uv = (torch.randn((H, 512, 128), generator=g, device="cuda") * 0.05).to(torch.bfloat16)
    cos = torch.ones((B, 1, 32), device="cuda"); sin = torch.zeros((B, 1, 32), device="cuda")
    plan = mla.MlaDecodePlan.create(B, H, "cuda")
    q = torch.empty((B, 1, H, 576), dtype=torch.bfloat16, device="cuda")
    o = torch.empty((B, 1, H, 512), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, 1, H), dtype=torch.float32, device="cuda")
    scale = 1 / math.sqrt(192)

    def t(fn):
        # device time: 20 calls captured in one CUDA graph (no host launch gaps), replayed
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s), torch.cuda.graph(gr, stream=s):
            for _ in range(20):
                fn()
        torch.cuda.synchronize()
        gr.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(max(1, iters // 20)):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1000 / (max(1, iters // 20) * 20)
    absorb = lambda: mla.absorb_q(q_nope, q_pe, cos, sin, w_uk, out=q)
    dec = lambda: plan.decode(q, inp.kv_pool, inp.block_table, inp.seqlens, scale, out=o, lse=lse)
    up = lambda: mla.up_proj(o, w_uv)
    line = {"config": f"absorbed MLA layer step B={B} H={H} ctx={ctx}", "absorb_q_us": t(absorb),
            "decode_us": t(dec), "up_proj_us": t(up),
            "step_us": t(lambda: (absorb(), dec(), up())),
            "weight_bytes": (w_uk.numel() + w_uv.numel()) * 2}
    print(json.dumps(line), flush=True)


def measure_fp8(seqlens, heads, label, iters=50, q_tokens=1):
    """FP8 (e4m3) latent cache: device time per step (stream launches), bytes of the fp8 pool."""
    kv_bytes = sum(seqlens) * 576
    ncopies = max(1, min(8, (2 * L2_BYTES) // max(1, kv_bytes) + 1))
    B = len(seqlens)
    sets = []
    for i in range(ncopies):
        inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=42 + i, pad_value=0.0, q_tokens=q_tokens)
        kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
        inp.kv_pool = None
        sets.append((inp, kv8))
        torch.cuda.empty_cache()
    plan = mla.MlaDecodePlan.create(B, heads, "cuda", q_tokens=q_tokens)
    out = torch.empty((B, q_tokens, heads, 512), dtype=torch.float32, device="cuda")
    lse = torch.empty((B, q_tokens, heads), dtype=torch.float32, device="cuda")

    def step(j):
        inp, kv8 = sets[j % ncopies]
        plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125, out=out, lse=lse)

    for j in range(5):
        step(j)
    torch.cuda.synchronize()
    res = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for j in range(iters):
            step(j)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1000 / iters)
    us_stream = sorted(res)[1]
    us_graph_multi = graph_multi(step)
    us = min(us_stream, us_graph_multi)
    H = heads * q_tokens
    nbytes = (kv_bytes + B * H * 576 * 2 + B * H * 512 * 4 + B * H * 4
              + sum((s + 63) // 64 for s in seqlens) * 4 + 4 * B)
    line = {"config": label, "kv": "fp8 e4m3", "batch": B, "heads": heads, "ctx_total": sum(seqlens),
            "us_per_step_stream": us_stream, f"us_per_step_graph{GRAPH_STEPS}": us_graph_multi, "us_per_step": us, "hbm_gbs": nbytes / us / 1e3,
            "tflops": inputs.flops(seqlens, H) / us / 1e6, "algorithmic_bytes": nbytes,
            "l2_rotation_copies": ncopies}
    print(json.dumps(line), flush=True)
    del sets
    torch.cuda.empty_cache()


if __name__ == "__main__":
    if "--fp8" in sys.argv:
        measure_fp8([1024], 16, "fp8 config1 B=1 H=16 ctx=1K")
        for ctx in (1024, 4096, 16384, 65536):
            measure_fp8([ctx] * 16, 16, f"fp8 config3 B=16 H=16 ctx={ctx}")
        measure_fp8(inputs.varlen_seqlens(32), 16, "fp8 config4 B=32 varlen 4K-128K")
        measure_fp8([65536] * 16, 16, "fp8 B=16 ctx=64K H=16 q_tokens=2", iters=20, q_tokens=2)
        if "--heads" in sys.argv:
            for h in (32, 64, 128):
                measure_fp8([65536] * 16, h, f"fp8 B=16 ctx=64K H={h}", iters=10)
        sys.exit(0)
    if "--serving" in sys.argv:  # serving-style batches: many sequences, short-to-medium contexts
        import random
        for B, lo, hi in ((64, 2048, 8192), (128, 1024, 4096), (256, 512, 4096), (128, 4096, 32768)):
            rnd = random.Random(B * 7 + lo)
            measure([rnd.randint(lo, hi) for _ in range(B)], 16, f"serving B={B} ctx {lo}-{hi}", iters=20)
        sys.exit(0)
    if "--layer" in sys.argv:
        measure_layer()
        measure_layer(ctx=4096)
        sys.exit(0)
    if "--mtp" in sys.argv:  # multi-token decode: T tokens per sequence against the same context
        for t in (1, 2, 4):
            measure([65536] * 16, 16, f"B=16 ctx=64K H=16 q_tokens={t}", iters=20, q_tokens=t)
        sys.exit(0)
    if "--heads" in sys.argv:  # head-count sweep at the headline context (head group per ETAP_HEAD_GROUP)
        hg = os.environ.get("ETAP_HEAD_GROUP", "auto")
        unit = lambda h: mla.schedule_unit(h, mla.num_sm_parts())[0] if hg == "auto" else hg  # 128: CTA pairs
        for h in (16, 32, 64, 128, 256):
            measure([65536] * 16, h, f"B=16 ctx=64K H={h} work_unit={unit(h)}", iters=20 if h <= 128 else 10)
        measure([4096] * 64, 128, f"B=64 ctx=4K H=128 work_unit={unit(128)}", iters=20)
        sys.exit(0)
    measure([1024], 16, "config1 B=1 H=16 ctx=1K")
    for ctx in (1024, 2048, 4096, 8192, 16384, 32768, 65536):
        measure([ctx] * 16, 16, f"config3 B=16 H=16 ctx={ctx}")
    measure(inputs.varlen_seqlens(32), 16, "config4 B=32 varlen 4K-128K")
    if "--no-config5" not in sys.argv:
        measure([65536] * 16, 128, "config5 single-GPU B=16 H=128 ctx=64K (128-head units on CTA pairs)", iters=10)
