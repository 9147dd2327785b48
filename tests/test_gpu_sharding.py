# SPDX-License-Identifier: Apache-2.0
"""GPU test of the collective (non-peer) head-sharded path that `bench.py` falls back to when
peer access is unavailable (`sharding.gather_heads`): every rank runs the real
decode kernels on its head block of the replicated latent KV, the per-rank O / LSE blocks are
all-gathered as CUDA tensors, and the gathered result matches the binary64 oracle over all heads
(RMSE ≤ 2e-5, the north_star bar) and, bitwise, each shard decoded alone. The ranks share the
one visible GPU, so the collective is gloo (NCCL refuses two ranks on one device); the code path
above the backend is the same one the NCCL run takes."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SEQLENS = [3000, 64, 1, 777, 9000]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, total_heads: int, q_tokens: int, out_q):
    from paper_2506_01969_b200 import inputs, mla, sharding

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        inp = inputs.make_mla_inputs(SEQLENS, heads=total_heads, seed=21, q_tokens=q_tokens)
        h0, hn = sharding.head_shard(total_heads, world, rank)
        q = inp.q[:, :, h0:h0 + hn].contiguous()
        plan = mla.MlaDecodePlan.create(len(SEQLENS), hn, "cuda", q_tokens=q_tokens)
        plan.metadata(inp.seqlens)
        o, l = plan.decode(q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
        torch.cuda.synchronize()
        og, lg = sharding.gather_heads(o), sharding.gather_heads(l)
        torch.cuda.synchronize()
        if rank == 0:
            out_q.put((og.cpu().numpy(), lg.cpu().numpy(), o.cpu().numpy(), l.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,total_heads,q_tokens", [(2, 32, 1), (4, 64, 1), (2, 64, 2), (8, 128, 1)])
def test_collective_head_sharding_matches_oracle(cuda_device, world, total_heads, q_tokens):
    import oracle
    from paper_2506_01969_b200 import inputs

    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total_heads, q_tokens, out_q))
             for r in range(world)]
    for p in procs:
        p.start()
    og, lg, o0, l0 = out_q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    hn = total_heads // world
    assert og.shape == (len(SEQLENS), q_tokens, total_heads, 512) and lg.shape == og.shape[:3]
    # rank 0's block of the gathered tensor is its own decode, bit for bit
    assert np.array_equal(og[:, :, :hn], o0) and np.array_equal(lg[:, :, :hn], l0)

    inp = inputs.make_mla_inputs(SEQLENS, heads=total_heads, seed=21, q_tokens=q_tokens)
    bits = lambda t: t.contiguous().view(torch.int16).numpy().view(np.uint16)  # noqa: E731
    sl = inp.seqlens.cpu().numpy()
    o_ref, l_ref = oracle.mla_decode_bf16_tokens(bits(inp.q.cpu()), bits(inp.kv_pool.cpu()),
                                                 inp.block_table.cpu().numpy(), sl, inp.scale)
    for t in range(q_tokens):
        # token t of a causal multi-token decode sees the first seqlen - (T - 1 - t) rows
        ne = (sl - (q_tokens - 1 - t)) > 0
        o_t, l_t = og[:, t].astype(np.float64), lg[:, t].astype(np.float64)
        assert np.isfinite(o_t).all()
        assert float(np.sqrt(np.mean((o_t[ne] - o_ref[ne, t]) ** 2))) <= 2e-5
        assert np.abs(l_t[ne] - l_ref[ne, t]).max() <= 1e-4
        assert (o_t[~ne] == 0).all() and np.isneginf(l_t[~ne]).all()
