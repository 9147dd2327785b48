# SPDX-License-Identifier: Apache-2.0
"""GPU tests of the steps on either side of the decode kernel:
q absorption + RoPE (etap_mla_absorb_q) and the per-head value up-projection
(etap_mla_up_proj), each against a plain PyTorch fp32/fp64 reference of the same op, and the
whole absorbed-MLA decode (absorb -> ETAP decode -> up-projection) against the textbook,
non-absorbed MLA attention on the same latent cache."""
from __future__ import annotations

import math

import pytest
import torch

from paper_2506_01969_b200 import _lib, inputs, mla

pytestmark = pytest.mark.gpu


def rope_ref(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    x0, x1 = x[..., :32], x[..., 32:]
    c, s = cos.unsqueeze(-2), sin.unsqueeze(-2)
    return torch.cat([x0 * c - x1 * s, x1 * c + x0 * s], dim=-1)


def rand(shape, scale=1.0, dtype=torch.bfloat16, g=None):
    return (torch.randn(shape, generator=g, device="cuda") * scale).to(dtype)


@pytest.mark.parametrize("B,T,H", [(16, 1, 16), (3, 2, 32), (1, 1, 128), (200, 1, 16)])
def test_absorb_q_matches_torch(cuda_device, B, T, H):
    g = torch.Generator(device="cuda").manual_seed(B * 100 + H)
    q_nope, q_pe = rand((B, T, H, 128), g=g), rand((B, T, H, 64), g=g)
    w_uk = rand((H, 128, 512), 0.1, g=g)
    ang = torch.rand((B, T, 32), generator=g, device="cuda") * 6.28
    cos, sin = torch.cos(ang), torch.sin(ang)
    q = mla.absorb_q(q_nope, q_pe, cos, sin, w_uk)
    torch.cuda.synchronize()
    lat = torch.einsum("bthi,hic->bthc", q_nope.double(), w_uk.double())
    rot = rope_ref(q_pe.double(), cos.double(), sin.double())
    # fp32 accumulation then one bf16 rounding: within one bf16 ulp of the exact value plus
    # the fp32 summation error (~2^-22 of the sum of |products|, matters only near zero)
    lat_abs = torch.einsum("bthi,hic->bthc", q_nope.double().abs(), w_uk.double().abs())
    rot_abs = rope_ref(q_pe.double().abs(), cos.double().abs(), sin.double().abs()).abs()
    for got, ref, mag in ((q[..., :512].double(), lat, lat_abs), (q[..., 512:].double(), rot, rot_abs)):
        ulp = torch.exp2(torch.floor(torch.log2(ref.abs().clamp_min(1e-30))) - 7)
        assert ((got - ref).abs() <= ulp + 2.0 ** -22 * mag).all()


@pytest.mark.parametrize("B,T,H,fp32", [(16, 1, 16, True), (5, 3, 32, False), (64, 1, 128, True)])
def test_up_proj_matches_torch(cuda_device, B, T, H, fp32):
    g = torch.Generator(device="cuda").manual_seed(7 * B + H)
    o = rand((B, T, H, 512), 0.05, torch.float32, g=g)
    w_uv = rand((H, 512, 128), 0.05, g=g)
    out = mla.up_proj(o, w_uv, torch.float32 if fp32 else torch.bfloat16)
    torch.cuda.synchronize()
    # the GEMM runs on bf16 operands (O rounded to bf16 on load), fp32 accumulation
    ref = torch.einsum("bthd,hdc->bthc", o.to(torch.bfloat16).double(), w_uv.double())
    err = (out.double() - ref).abs().max().item()
    tol = 1e-5 if fp32 else 2 ** -8 * ref.abs().max().item()
    assert err <= tol, err


def test_proj_shape_errors(cuda_device):
    L = _lib.lib()
    x = torch.zeros(16, 16, 100, device="cuda", dtype=torch.bfloat16)
    w = torch.zeros(16, 100, 512, device="cuda", dtype=torch.bfloat16)
    y = torch.zeros(16, 16, 512, device="cuda", dtype=torch.bfloat16)
    rc = L.etap_mla_head_proj(x.data_ptr(), 0, 1600, 100, w.data_ptr(), 16, 16, 100, 512, y.data_ptr(), 0,
                              16 * 512, 512, None)
    assert rc == _lib.ETAP_ERR_SHAPE  # k_dim not a multiple of 64
    rc = L.etap_mla_head_proj(x.data_ptr(), 0, 1600, 100, w.data_ptr(), 300, 16, 64, 512, y.data_ptr(), 0,
                              16 * 512, 512, None)
    assert rc == _lib.ETAP_ERR_SHAPE  # more than 256 token rows
    with pytest.raises(_lib.EtapShapeError):
        mla.up_proj(torch.zeros(2, 1, 16, 512, device="cuda"), torch.zeros(16, 512, 64, device="cuda",
                                                                             dtype=torch.bfloat16))


def test_absorbed_mla_decode_equals_textbook_mla(cuda_device):
    """absorb_q -> ETAP decode on the latent cache -> up_proj equals standard (non-absorbed) MLA
    attention: k_nope = W_UK c, v = W_UV^T c, scores q_nope.k_nope + rope(q_pe).k_pe."""
    B, H, T = 4, 16, 1
    seqlens = [700, 64, 1, 2049]
    inp = inputs.make_mla_inputs(seqlens, heads=H, seed=23, pad_value=0.0)
    g = torch.Generator(device="cuda").manual_seed(11)
    q_nope, q_pe = rand((B, T, H, 128), g=g), rand((B, T, H, 64), g=g)
    w_uk, w_uv = rand((H, 128, 512), 0.05, g=g), rand((H, 512, 128), 0.05, g=g)
    ang = torch.rand((B, T, 32), generator=g, device="cuda") * 6.28
    cos, sin = torch.cos(ang), torch.sin(ang)
    scale = 1.0 / math.sqrt(192)
    q = mla.absorb_q(q_nope, q_pe, cos, sin, w_uk)
    o, lse = mla.mla_decode(q, inp.kv_pool, inp.block_table, inp.seqlens, scale)
    out = mla.up_proj(o, w_uv, torch.float32)
    torch.cuda.synchronize()
    pool = inp.kv_pool.double()
    rot = rope_ref(q_pe.double(), cos.double(), sin.double())
    for b, L in enumerate(seqlens):
        pages = inp.block_table[b, : (L + 63) // 64].long()
        c = pool[pages].reshape(-1, 576)[:L]                      # latent rows [L, 576]
        k_nope = torch.einsum("hic,jc->hji", w_uk.double(), c[:, :512])   # [H, L, 128]
        v = torch.einsum("hdc,jd->hjc", w_uv.double(), c[:, :512])        # [H, L, 128]
        s = (torch.einsum("hi,hji->hj", q_nope[b, 0].double(), k_nope) +
             torch.einsum("hr,jr->hj", rot[b, 0], c[:, 512:])) * scale
        ref = torch.einsum("hj,hjc->hc", torch.softmax(s, dim=-1), v)
        err = (out[b, 0].double() - ref).abs().max().item() / ref.abs().max().item()
        # bf16 roundings of q_latent and of O before W_UV bound the agreement (~2^-8)
        assert err <= 2e-2, (b, err)
