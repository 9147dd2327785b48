# SPDX-License-Identifier: Apache-2.0
"""Multi-process (gloo, world_size 2, CPU) test of the head-sharded path: each rank decodes
its head block against the replicated latent KV (oracle standing in for the GPU kernel) and
the all-gather reassembles exactly the single-process result."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2506_01969_b200 import sharding


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(total_heads: int):
    rng = np.random.default_rng(0)
    seqlens = np.array([70, 129], np.int32)
    pages = [(s + 63) // 64 for s in seqlens]
    pool = oracle.bf16_bits(rng.normal(size=(sum(pages), 64, 576)))
    bt = np.zeros((2, max(pages)), np.int32)
    bt[0, :pages[0]] = np.arange(pages[0])
    bt[1, :pages[1]] = np.arange(pages[0], pages[0] + pages[1])
    q = oracle.bf16_bits(rng.normal(size=(2, total_heads, 576)))
    return q, pool, bt, seqlens


def _worker(rank: int, world: int, port: int, total_heads: int, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q, pool, bt, sl = _problem(total_heads)
        h0, hn = sharding.head_shard(total_heads, world, rank)
        o, l = oracle.mla_decode_bf16(q[:, h0:h0 + hn], pool, bt, sl, 1 / 24, nthreads=1)
        o_t = torch.from_numpy(o).unsqueeze(1)          # [B, 1, Hl, 512]
        l_t = torch.from_numpy(l).unsqueeze(1)          # [B, 1, Hl]
        og = sharding.gather_heads(o_t)
        lg = sharding.gather_heads(l_t)
        if rank == 0:
            out_q.put((og.numpy(), lg.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total_heads", [32, 64])
def test_head_sharded_allgather_matches_full(total_heads):
    world = 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total_heads, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    og, lg = out_q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    q, pool, bt, sl = _problem(total_heads)
    o_full, l_full = oracle.mla_decode_bf16(q, pool, bt, sl, 1 / 24, nthreads=1)
    assert og.shape == (2, 1, total_heads, 512)
    assert np.array_equal(og[:, 0], o_full) and np.array_equal(lg[:, 0], l_full)


def test_head_shard_rules():
    assert sharding.head_shard(128, 8, 3) == (48, 16)
    assert sharding.head_shard(128, 1, 0) == (0, 128)
    with pytest.raises(ValueError):
        sharding.head_shard(128, 3, 0)
    with pytest.raises(ValueError):
        sharding.head_shard(64, 8, 0)
