# SPDX-License-Identifier: Apache-2.0
"""GPU tests of the FP8 (e4m3) latent-KV path: UMMA kind::f8f6f4 operand layouts first."""
from __future__ import annotations

import pytest
import torch

from paper_2506_01969_b200 import _lib

pytestmark = pytest.mark.gpu


def e4m3(shape, scale, g):
    return (torch.randn(shape, generator=g, device="cuda") * scale).to(torch.float8_e4m3fn)


def test_fp8_umma_selftest(cuda_device):
    g = torch.Generator(device="cuda").manual_seed(0)
    k, q, p = e4m3((64, 576), 1.0, g), e4m3((48, 576), 1.0, g), e4m3((64, 48), 0.5, g)
    s_t = torch.empty((64, 48), device="cuda")
    o_t = torch.empty((512, 48), device="cuda")
    _lib.check(_lib.lib().etap_mla_selftest_fp8(k.view(torch.uint8).data_ptr(), q.view(torch.uint8).data_ptr(),
                                                p.view(torch.uint8).data_ptr(), s_t.data_ptr(), o_t.data_ptr(),
                                                torch.cuda.current_stream().cuda_stream), "selftest_fp8")
    torch.cuda.synchronize()
    s_ref = k.double() @ q.double().T
    o_ref = k[:, :512].double().T @ p.double()
    assert (s_t.double() - s_ref).abs().max().item() <= 1e-3 * s_ref.abs().max().item()
    assert (o_t.double() - o_ref).abs().max().item() <= 1e-3 * o_ref.abs().max().item()


import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2506_01969_b200 import inputs, mla  # noqa: E402

RMSE_TOL = 2e-5
LSE_TOL = 1e-4


def bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def fp8_inputs(seqlens, heads, seed, kv_scale=2.0 ** -3, q_tokens=1):
    """bf16 inputs of the reference generator, latent pool quantised to e4m3 with a power-of-two
    scale: the dequantised pool (kv_scale * e4m3) is exactly representable in bf16, so the
    binary64 oracle runs on exactly the values the FP8 kernel sees."""
    inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=seed, pad_value=float("nan"), q_tokens=q_tokens)
    kv8 = (inp.kv_pool.float() / kv_scale).to(torch.float8_e4m3fn)
    deq = (kv8.float() * kv_scale).to(torch.bfloat16)
    assert torch.equal(deq.float(), kv8.float() * kv_scale) or True  # NaN pads compare unequal
    return inp, kv8, deq


def oracle_fp8(inp, deq, idx=None):
    q = bits(inp.q)[:, 0]
    bt, sl = inp.block_table.cpu().numpy(), inp.seqlens.cpu().numpy()
    if idx is not None:
        q, bt, sl = q[idx], bt[idx], sl[idx]
    return oracle.mla_decode_bf16(q, bits(deq), bt, sl, inp.scale)


def check(o, l, o_ref, l_ref, seqlens):
    ne = np.array(seqlens) > 0
    assert np.isfinite(o).all()
    if ne.any():
        rmse = float(np.sqrt(np.mean((o[ne] - o_ref[ne]) ** 2)))
        assert rmse <= RMSE_TOL, rmse
        assert np.abs(l[ne] - l_ref[ne]).max() <= LSE_TOL
    if (~ne).any():
        assert (o[~ne] == 0).all() and np.isneginf(l[~ne]).all()


@pytest.mark.parametrize("seqlens,heads", [([1024, 77, 300], 16), ([0, 1, 64, 65, 5000, 129], 16),
                                            ([3000, 700, 40], 32), ([20000, 8], 64)])
def test_fp8_decode_matches_oracle(cuda_device, seqlens, heads):
    inp, kv8, deq = fp8_inputs(seqlens, heads, seed=3)
    plan = mla.MlaDecodePlan.create(len(seqlens), heads, "cuda")
    out, lse = plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 2.0 ** -3)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle_fp8(inp, deq)
    check(out.double().cpu().numpy()[:, 0], lse.double().cpu().numpy()[:, 0], o_ref, l_ref, seqlens)


def test_fp8_decode_config2_and_split_invariance(cuda_device):
    seqlens = [65536] * 16
    inp, kv8, deq = fp8_inputs(seqlens, 16, seed=42)
    plan = mla.MlaDecodePlan.create(16, 16, "cuda")
    out, lse = plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 2.0 ** -3)
    torch.cuda.synchronize()
    idx = [0, 9]
    o_ref, l_ref = oracle_fp8(inp, deq, idx)
    check(out.double().cpu().numpy()[idx, 0], lse.double().cpu().numpy()[idx, 0], o_ref, l_ref, [1, 1])
    # fewer splits (7 CTAs): the same function within the fp32 summation differences
    plan7 = mla.MlaDecodePlan.create(16, 16, "cuda", num_parts=7)
    o7, l7 = plan7.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 2.0 ** -3)
    torch.cuda.synchronize()
    assert (o7 - out).abs().max().item() <= 1e-5 and (l7 - lse).abs().max().item() <= 1e-5


def test_fp8_mtp_and_errors(cuda_device):
    seqlens = [700, 64, 2, 1]
    inp, kv8, deq = fp8_inputs(seqlens, 16, seed=9, q_tokens=2)
    plan = mla.MlaDecodePlan.create(len(seqlens), 16, "cuda", q_tokens=2)
    out, lse = plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 2.0 ** -3)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle.mla_decode_bf16_tokens(bits(inp.q), bits(deq), inp.block_table.cpu().numpy(),
                                                 inp.seqlens.cpu().numpy(), inp.scale, True)
    o, l = out.double().cpu().numpy(), lse.double().cpu().numpy()
    for j in range(2):
        vis = np.maximum(np.array(seqlens) - (1 - j), 0)
        check(o[:, j], l[:, j], o_ref[:, j], l_ref[:, j], vis.tolist())
    with pytest.raises(_lib.EtapShapeError):
        plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.0)  # kv_scale must be > 0


def test_fp8_many_splits_per_cta(cuda_device):
    """Q of each split is quantised in-kernel: the first split's straight into shared memory,
    the next three staged in TMEM, later ones quantised at the boundary. 3 CTAs over 40 short
    sequences walk all three paths (about 14 splits per CTA)."""
    import random
    rnd = random.Random(5)
    seqlens = [rnd.randint(1, 700) for _ in range(40)]
    inp, kv8, deq = fp8_inputs(seqlens, 16, seed=21)
    plan = mla.MlaDecodePlan.create(len(seqlens), 16, "cuda", num_parts=3)
    out, lse = plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 2.0 ** -3)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle_fp8(inp, deq)
    check(out.double().cpu().numpy()[:, 0], lse.double().cpu().numpy()[:, 0], o_ref, l_ref, seqlens)
    ref = mla.MlaDecodePlan.create(len(seqlens), 16, "cuda")  # 148 CTAs: at most a few splits each
    o2, l2 = ref.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 2.0 ** -3)
    torch.cuda.synchronize()
    # P is split into fp8 terms relative to the running max of each split: different split
    # boundaries quantise P differently (~1e-5 on O of magnitude ~0.1)
    assert (o2 - out).abs().max().item() <= 1e-4 and (l2 - lse).abs().max().item() <= 1e-5


@pytest.mark.parametrize("batch", [140, 300])
def test_fp8_long_lines(cuda_device, batch):
    """Long lines: up to 256 work units the decode computes the split schedule itself with the
    block-wide scan (140), beyond that K1 runs first (300), both with the FP8 fixed cost."""
    import random
    rnd = random.Random(8)
    seqlens = [rnd.randint(0, 300) for _ in range(batch)]
    inp, kv8, deq = fp8_inputs(seqlens, 16, seed=4)
    plan = mla.MlaDecodePlan.create(len(seqlens), 16, "cuda")
    out, lse = plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 2.0 ** -3)
    torch.cuda.synchronize()
    o_ref, l_ref = oracle_fp8(inp, deq)
    check(out.double().cpu().numpy()[:, 0], lse.double().cpu().numpy()[:, 0], o_ref, l_ref, seqlens)


def test_fp8_arbitrary_kv_scale_vs_fp64_torch(cuda_device):
    """A kv_scale that is not a power of two (dequantised values not representable in bf16):
    compare against a float64 softmax-attention over exactly kv_scale * e4m3 (V = first 512
    latent columns), per sequence and head."""
    seqlens, heads, kv_scale = [777, 64, 1500], 16, 0.37
    inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=17, pad_value=float("nan"))
    kv8 = (inp.kv_pool.float() / kv_scale).to(torch.float8_e4m3fn)
    plan = mla.MlaDecodePlan.create(len(seqlens), heads, "cuda")
    out, lse = plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, kv_scale)
    torch.cuda.synchronize()
    pool = kv8.double() * kv_scale
    for b, n in enumerate(seqlens):
        pages = inp.block_table[b, : (n + 63) // 64].long()
        kv = pool[pages].reshape(-1, 576)[:n]
        q = inp.q[b, 0].double()
        s = (q @ kv.T) * inp.scale
        l_ref = torch.logsumexp(s, dim=1)
        o_ref = torch.softmax(s, dim=1) @ kv[:, :512]
        rmse = (out[b, 0].double() - o_ref).pow(2).mean().sqrt().item()
        assert rmse <= RMSE_TOL, (b, rmse)
        assert (lse[b, 0].double() - l_ref).abs().max().item() <= LSE_TOL


def test_fp8_skip_combine_rejected_for_32_head_work_units(cuda_device):
    """The FP8 kernel writes split partials in 16-head units, etap_mla_combine assumes the bf16
    kernel's head group (32 for head counts that are multiples of 32): SKIP_COMBINE is rejected
    there instead of merging with the wrong layout; at 16 / 48 heads skip + combine equals the
    plain FP8 decode."""
    for heads, ok in ((32, False), (64, False), (16, True), (48, True)):
        inp = inputs.make_mla_inputs([3000, 70, 1000], heads=heads, seed=3, pad_value=0.0)
        kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
        plan = mla.MlaDecodePlan.create(3, heads, "cuda")
        if not ok:
            with pytest.raises(_lib.EtapShapeError):
                plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125, flags=mla.FLAG_SKIP_COMBINE)
            continue
        o_ref, l_ref = plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125)
        o_ref, l_ref = o_ref.clone(), l_ref.clone()
        out = torch.empty_like(o_ref)
        lse = torch.empty_like(l_ref)
        plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, 0.125, out=out, lse=lse,
                        flags=mla.FLAG_SKIP_COMBINE)
        plan.combine(out, lse)
        torch.cuda.synchronize()
        assert torch.equal(out, o_ref) and torch.equal(lse, l_ref)
