# SPDX-License-Identifier: Apache-2.0
"""Fused all-gather check: `world` ranks (torchrun; any backend — gloo lets several ranks share
one GPU) each decode their head shard through PeerGather (etap_mla_decode_peer) and must hold
the full-head output afterwards, bitwise equal to plain decodes of every shard.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/peer_check.py [--q-tokens 2]
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_2506_01969_b200 import inputs, mla, peer


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--q-tokens", type=int, default=1)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--calls", type=int, default=6)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    gpu = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    if world > 1:
        dist.init_process_group(os.environ.get("ETAP_DIST_BACKEND", "gloo"))
    T, Hl = a.q_tokens, a.heads
    seqlens = [5000, 64, 1, 777, 20000]
    B = len(seqlens)
    total = Hl * world
    shards = [inputs.make_mla_inputs(seqlens, heads=Hl, seed=3, head_offset=r * Hl, total_heads=total,
                                     q_tokens=T, pad_value=float("nan")) for r in range(world)]
    plan = mla.MlaDecodePlan.create(B, Hl, "cuda", q_tokens=T)
    pg = peer.PeerGather(B, Hl, world, rank, q_tokens=T)
    bad = 0
    for call in range(a.calls):
        mine = shards[rank]
        scale = mine.scale * (1.0 + 0.25 * call)  # a different result every call
        o, l = pg.decode(plan, mine.q, mine.kv_pool, mine.block_table, mine.seqlens, scale)
        o, l = o.clone(), l.clone()
        for r in range(world):
            ref_plan = mla.MlaDecodePlan.create(B, Hl, "cuda", q_tokens=T)
            ro, rl = ref_plan.decode(shards[r].q, shards[r].kv_pool, shards[r].block_table, shards[r].seqlens, scale)
            sl = slice(r * Hl, (r + 1) * Hl)
            ok = torch.equal(o[:, :, sl], ro) and torch.equal(l[:, :, sl], rl)
            bad += not ok
            if not ok:
                print(f"rank {rank} call {call}: shard {r} differs (max {(o[:, :, sl] - ro).abs().max().item():.3e})",
                      flush=True)
        if world > 1:
            dist.barrier()  # every rank consumed this call before buffers come round again
    torch.cuda.synchronize()
    pg.close()
    print(f"peer_check rank {rank}/{world} T={T}: {'ok' if bad == 0 else f'{bad} mismatches'}", flush=True)
    if world > 1:
        dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
