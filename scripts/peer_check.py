# SPDX-License-Identifier: Apache-2.0
"""Fused all-gather check: `world` ranks (torchrun; any backend — gloo lets several ranks share
one GPU) each decode their head shard through PeerGather (etap_mla_decode_peer) and must hold
the full-head output afterwards. The calls run FREE (no barrier between them: only the
epoch / arrival-word protocol and the double-buffered outputs order the ranks); each rank
copies every call's full-head result on its stream and checks them afterwards
  * bitwise against plain decodes of every shard (all calls), and
  * against the binary64 oracle over ALL heads (rank 0, the last call; --oracle).
With 8 ranks x 16 heads this is the 128-head DeepSeek-R1 shape of BASELINE.json configs[4].

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/peer_check.py --oracle
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_2506_01969_b200 import inputs, mla, peer


def bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--q-tokens", type=int, default=1)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--calls", type=int, default=6)
    ap.add_argument("--oracle", action="store_true", help="rank 0 checks the last call against the oracle")
    ap.add_argument("--seqlens", type=str, default="5000,64,1,777,20000")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    gpu = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    if world > 1:
        dist.init_process_group(os.environ.get("ETAP_DIST_BACKEND", "gloo"))
    T, Hl = a.q_tokens, a.heads
    seqlens = [int(x) for x in a.seqlens.split(",")]
    B = len(seqlens)
    total = Hl * world
    shards = [inputs.make_mla_inputs(seqlens, heads=Hl, seed=3, head_offset=r * Hl, total_heads=total,
                                     q_tokens=T, pad_value=float("nan")) for r in range(world)]
    plan = mla.MlaDecodePlan.create(B, Hl, "cuda", q_tokens=T)
    pg = peer.PeerGather(B, Hl, world, rank, q_tokens=T)
    mine = shards[rank]
    scales = [mine.scale * (1.0 + 0.25 * c) for c in range(a.calls)]  # a different result every call
    results = []
    if world > 1:
        dist.barrier()  # start together; no barrier between the calls below
    for call in range(a.calls):
        o, l = pg.decode(plan, mine.q, mine.kv_pool, mine.block_table, mine.seqlens, scales[call])
        results.append((o.clone(), l.clone()))  # stream-ordered before this rank's next decode
    torch.cuda.synchronize()
    bad = 0
    for call, (o, l) in enumerate(results):
        for r in range(world):
            ref_plan = mla.MlaDecodePlan.create(B, Hl, "cuda", q_tokens=T)
            ro, rl = ref_plan.decode(shards[r].q, shards[r].kv_pool, shards[r].block_table, shards[r].seqlens,
                                     scales[call])
            sl = slice(r * Hl, (r + 1) * Hl)
            ok = torch.equal(o[:, :, sl], ro) and torch.equal(l[:, :, sl], rl)
            bad += not ok
            if not ok:
                print(f"rank {rank} call {call}: shard {r} differs (max {(o[:, :, sl] - ro).abs().max().item():.3e})",
                      flush=True)
    oracle_msg = ""
    if a.oracle and rank == 0 and T == 1:
        import oracle

        o, l = results[-1]
        q_all = torch.cat([s.q for s in shards], dim=2)  # [B, 1, total, 576], head order
        o_ref, l_ref = oracle.mla_decode_bf16(bits(q_all)[:, 0], bits(mine.kv_pool), mine.block_table.cpu().numpy(),
                                              mine.seqlens.cpu().numpy(), scales[-1])
        og = o[:, 0].double().cpu().numpy()
        lg = l[:, 0].double().cpu().numpy()
        ne = np.array(seqlens) > 0
        rmse = float(np.sqrt(np.mean((og[ne] - o_ref[ne]) ** 2)))
        lerr = float(np.abs(lg[ne] - l_ref[ne]).max())
        ok = np.isfinite(og).all() and rmse <= 2e-5 and lerr <= 1e-4
        bad += not ok
        oracle_msg = f" oracle[{total} heads] rmse={rmse:.2e} lse_err={lerr:.2e} {'ok' if ok else 'FAIL'}"
    if world > 1:
        dist.barrier()  # nobody frees an exported buffer while a peer may still hold it mapped
    pg.close()
    print(f"peer_check rank {rank}/{world} heads {Hl}x{world}={total} T={T} calls={a.calls} free-running:{oracle_msg} "
          f"{'ok' if bad == 0 else f'{bad} mismatches'}", flush=True)
    if world > 1:
        dist.destroy_process_group()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
