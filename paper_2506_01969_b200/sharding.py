# SPDX-License-Identifier: Apache-2.0
"""Head sharding for the 128-head DeepSeek-R1 decode shape (BASELINE.json configs[4]).

Every rank owns a contiguous block of heads and the full (replicated) latent KV; the only
exchange is an all-gather of O (and LSE) after the decode step. The
reference has no multi-device path; this is the B200 plumbing around the per-GPU kernel.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_shard(total_heads: int, world: int, rank: int) -> tuple[int, int]:
    """(first head, head count) of `rank`; heads split evenly in multiples of 16."""
    if total_heads % world != 0 or (total_heads // world) % 16 != 0:
        raise ValueError(f"{total_heads} heads cannot be split into {world} shards of 16k heads")
    per = total_heads // world
    return rank * per, per


def gather_heads(local: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather a per-rank head block [B, S, H_local, ...] into [B, S, world*H_local, ...]
    in head order (rank r's block lands at heads [r*H_local, (r+1)*H_local))."""
    world = dist.get_world_size(group)
    if world == 1:
        return local
    local = local.contiguous()
    if dist.get_backend(group) == "nccl":
        buf = torch.empty((world, *local.shape), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(buf, local, group=group)
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local, group=group)
        buf = torch.stack(parts)
    # [world, B, S, Hl, ...] -> [B, S, world, Hl, ...] -> [B, S, world*Hl, ...]
    perm = [1, 2, 0] + list(range(3, buf.dim()))
    out = buf.permute(*perm)
    return out.reshape(*local.shape[:2], world * local.shape[2], *local.shape[3:])
