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
