# SPDX-License-Identifier: Apache-2.0
"""Synthetic MLA decode inputs in the reference's conventions, generated on the device.

Data follow the reference bench harness: instance b uses seed s_b = seed + 7919*b
(cli.cpp:239); Q_b = matrix_from_seed(H, 576, 3*s_b+1), latent KV_b =
matrix_from_seed(ctx_b, 576, 3*s_b+2) (attention.cpp:38-39), normal(0,1) by splitmix64 +
Box-Muller (matrix.cpp:23-48,153-165), then rounded to bf16. V is KV[:, :512] (MLA aliasing;
the reference's separate V stream 3*s_b+3 is deliberately not used). The generator is
restated here with torch int64 ops so 1.2 GB of KV is produced on the GPU in seconds; it is
input plumbing, not the checker (tests compare it against the C oracle's generator).

Pages: 64-row pages, block table = a seeded permutation of the page pool; rows past seqlen
in the last page are filled with ``pad_value`` (NaN exercises the kernel's masking).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

D_QK = 576
PAGE_ROWS = 64

_GAMMA = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB


def _s64(x: int) -> int:
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= (1 << 63) else x


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def _mix(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _lsr(z, 30)) * _s64(_C1)
    z = (z ^ _lsr(z, 27)) * _s64(_C2)
    return z ^ _lsr(z, 31)


def splitmix_normal(n: int, seed: int, device: torch.device | str, start: int = 0,
                    chunk: int = 1 << 24) -> torch.Tensor:
    """Elements [start, start+n) of matrix_from_seed(..., seed, normal) as float64."""
    device = torch.device(device)
    out = torch.empty(n, dtype=torch.float64, device=device)
    two_pi = 6.283185307179586476925286766559
    for c0 in range(0, n, chunk):
        m = min(chunk, n - c0)
        e = torch.arange(start + c0, start + c0 + m, dtype=torch.int64, device=device)
        k1 = 2 * e + 1  # draw index (1-based) of u1; u2 is the next draw
        z1 = _mix(k1 * _s64(_GAMMA) + _s64(seed))
        z2 = _mix((k1 + 1) * _s64(_GAMMA) + _s64(seed))
        u1 = (_lsr(z1, 11) + 1).to(torch.float64) * 2.0 ** -53
        u2 = _lsr(z2, 11).to(torch.float64) * 2.0 ** -53
        out[c0:c0 + m] = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(two_pi * u2)
    return out


def splitmix_uniform01(n: int, seed: int) -> list[float]:
    """First n uniform01 draws of the splitmix64 stream (matrix.cpp:35), on the host."""
    s = seed & ((1 << 64) - 1)
    out = []
    for _ in range(n):
        s = (s + _GAMMA) & ((1 << 64) - 1)
        z = s
        z = ((z ^ (z >> 30)) * _C1) & ((1 << 64) - 1)
        z = ((z ^ (z >> 27)) * _C2) & ((1 << 64) - 1)
        z ^= z >> 31
        out.append((z >> 11) * 2.0 ** -53)
    return out


def bf16_rne(x: torch.Tensor) -> torch.Tensor:
    """binary64 -> bfloat16 with a single round-to-nearest-even (no float32 double rounding)."""
    m, e = torch.frexp(x)                       # x = m * 2^e, |m| in [0.5, 1)
    q = torch.clamp(e.to(torch.int64) - 8, min=-133)
    r = torch.round(torch.ldexp(x, -q.to(torch.float64)))   # torch.round = half to even
    y = torch.ldexp(r, q.to(torch.float64))
    y = torch.where(y.abs() > 3.3895313892515355e38, torch.copysign(torch.full_like(y, math.inf), y), y)
    y = torch.where(x == 0, x, y)
    return y.to(torch.float32).to(torch.bfloat16)     # exact: y has <= 8 significant bits


def varlen_seqlens(batch: int, lo: int = 4096, hi: int = 131072, seed: int = 2506) -> list[int]:
    """Config-4 context lengths: uniform integers in [lo, hi] from splitmix64(seed)."""
    return [lo + int(u * (hi - lo + 1)) for u in splitmix_uniform01(batch, seed)]


@dataclass
class MlaInputs:
    q: torch.Tensor            # [B, T, H, 576] bf16 (T query tokens per sequence, 1 for decode)
    kv_pool: torch.Tensor      # [pages, 64, 576] bf16
    block_table: torch.Tensor  # [B, max_pages] int32
    seqlens: torch.Tensor      # [B] int32
    scale: float
    seqlens_list: list[int]

    @property
    def batch(self) -> int:
        return self.q.shape[0]

    @property
    def heads(self) -> int:
        return self.q.shape[2]

    @property
    def q_tokens(self) -> int:
        return self.q.shape[1]

    def kv_bytes(self) -> int:
        return sum(self.seqlens_list) * D_QK * 2


def make_mla_inputs(seqlens: list[int], heads: int = 16, seed: int = 42,
                    device: torch.device | str = "cuda", pad_value: float = float("nan"),
                    head_offset: int = 0, total_heads: int | None = None,
                    scale: float | None = None, shuffle_pages: bool = True,
                    q_scale: float = 1.0, q_tokens: int = 1) -> MlaInputs:
    """Build paged inputs. With ``total_heads`` > heads, Q is drawn for all heads and the
    slice [head_offset, head_offset + heads) is kept (head sharding across ranks). With
    ``q_tokens`` > 1 the Q stream of a sequence holds q_tokens consecutive [total_heads, 576]
    blocks (multi-token decode)."""
    device = torch.device(device)
    B = len(seqlens)
    th = total_heads or heads
    pages = [(int(s) + PAGE_ROWS - 1) // PAGE_ROWS for s in seqlens]
    n_pages = max(1, sum(pages))
    max_pages = max(1, max(pages))
    g = torch.Generator().manual_seed(seed * 1000003 + 17)
    perm = torch.randperm(n_pages, generator=g) if shuffle_pages else torch.arange(n_pages)
    bt = torch.zeros((B, max_pages), dtype=torch.int32)
    off = 0
    for b, np_ in enumerate(pages):
        bt[b, :np_] = perm[off:off + np_].to(torch.int32)
        off += np_
    bt = bt.to(device)
    pool = torch.empty((n_pages, PAGE_ROWS, D_QK), dtype=torch.bfloat16, device=device)
    q = torch.empty((B, q_tokens, heads, D_QK), dtype=torch.bfloat16, device=device)
    for b, s in enumerate(seqlens):
        sb = seed + 7919 * b
        qb = splitmix_normal(q_tokens * th * D_QK, 3 * sb + 1, device).view(q_tokens, th, D_QK)
        q[b] = bf16_rne(qb[:, head_offset:head_offset + heads] * q_scale)
        if pages[b] == 0:
            continue
        rows = pages[b] * PAGE_ROWS
        kvb = torch.full((rows, D_QK), pad_value, dtype=torch.bfloat16, device=device)
        # generate in row blocks to bound the float64 temporaries
        blk = 8192
        for r0 in range(0, int(s), blk):
            r1 = min(int(s), r0 + blk)
            vals = splitmix_normal((r1 - r0) * D_QK, 3 * sb + 2, device, start=r0 * D_QK)
            kvb[r0:r1] = bf16_rne(vals).view(r1 - r0, D_QK)
        pool[bt[b, :pages[b]].long()] = kvb.view(pages[b], PAGE_ROWS, D_QK)
        del kvb
    sl = torch.tensor([int(s) for s in seqlens], dtype=torch.int32, device=device)
    sc = scale if scale is not None else 1.0 / math.sqrt(D_QK)
    return MlaInputs(q=q, kv_pool=pool, block_table=bt, seqlens=sl, scale=sc,
                     seqlens_list=[int(s) for s in seqlens])


def algorithmic_bytes(seqlens: list[int], heads: int) -> int:
    """KV + Q + O(fp32) + LSE + block table + seqlens, per step."""
    B = len(seqlens)
    kv = sum(seqlens) * D_QK * 2
    q = B * heads * D_QK * 2
    o = B * heads * 512 * 4
    lse = B * heads * 4
    bt = sum((s + PAGE_ROWS - 1) // PAGE_ROWS for s in seqlens) * 4
    return kv + q + o + lse + bt + 4 * B


def flops(seqlens: list[int], heads: int) -> int:
    return 2 * heads * sum(seqlens) * (576 + 512)
