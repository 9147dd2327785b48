# SPDX-License-Identifier: Apache-2.0
"""Dump the GPU path's outputs for fixed inputs as ATNM golden files (cross-run / cross-box
reproducibility of the sm_100a kernels). Run on a B200:
    python tests/golden/make_gpu_golden.py
Writes tests/golden/gpu_<case>_{o,lse}.atnm and gpu_golden.json."""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2506_01969_b200 import _lib, atnm, inputs, mla  # noqa: E402

OUT = Path(__file__).resolve().parent
CASES = {"b1_h16_ctx1024": ([1024], 16, 42), "varlen_b4_h32": ([100, 257, 64, 3000], 32, 7)}


def run(seqlens, heads, seed):
    inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=seed, pad_value=float("nan"))
    out, lse = mla.mla_decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    torch.cuda.synchronize()
    B, H = len(seqlens), heads
    return out.reshape(B * H, 512).cpu().numpy(), lse.reshape(B, H).cpu().numpy()


if __name__ == "__main__":
    meta = {"device": torch.cuda.get_device_name(), "num_sm": torch.cuda.get_device_properties(0).multi_processor_count,
            "library": _lib.lib().etap_mla_version().decode(), "cases": {}}
    for name, (seqlens, heads, seed) in CASES.items():
        o, l = run(seqlens, heads, seed)
        atnm.save(OUT / f"gpu_{name}_o.atnm", o)
        atnm.save(OUT / f"gpu_{name}_lse.atnm", l)
        meta["cases"][name] = {"seqlens": seqlens, "heads": heads, "seed": seed}
    (OUT / "gpu_golden.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(json.dumps(meta))
