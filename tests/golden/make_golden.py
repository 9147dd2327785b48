# SPDX-License-Identifier: Apache-2.0
"""Generate the golden fixtures in tests/golden/ by running the REFERENCE ITSELF
(oracle/_ref/libetaplab_ref.so, compiled from /root/reference/proj/src by oracle/Makefile).

Run in the build container (the reference sources are not on the GPU box):
    python tests/golden/make_golden.py
Every fixture records how it was produced. Inputs are NOT stored when they are reproducible
from the reference generator (matrix_from_seed) — a checksum of the bf16 inputs is stored
instead so a generator drift is detected.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def mla_problem(seed: int, heads: int, ctx: int):
    """Reference bench instance (cli.cpp:236-241, attention.cpp:33-42) with MLA aliasing:
    Q = matrix_from_seed(H,576,3s+1), KV = matrix_from_seed(ctx,576,3s+2), both rounded to
    bf16 (the GPU's input precision), V = KV[:, :512] (Matrix::col_block)."""
    q = oracle.bf16_round(oracle.ref_matrix_from_seed(heads, 576, 3 * seed + 1))
    kv = oracle.bf16_round(oracle.ref_matrix_from_seed(ctx, 576, 3 * seed + 2))
    return q, kv


def main() -> None:
    assert oracle.ref_available(), "reference sources / oracle/_ref required"
    meta = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref/libetaplab_ref.so "
            "(etaplab src/{matrix,attention,tiled_standard,etap}.cpp, unmodified)", "fixtures": {}}

    # 1. reference test_etap.cpp:137-146 — seed 42, 16 x 257 x 576/512, exact64 (independent V)
    q, k, v, sc = oracle.ref_make_problem(42, 16, 257, 576, 512)
    o, l = oracle.ref_run("ref", q, k, v, sc)
    oe, le = oracle.ref_run("etap", q, k, v, sc, b_r=16, b_c=64)
    np.savez_compressed(OUT / "seed42_16x257.npz", o=o, l=l, o_etap=oe, l_etap=le, scale=sc,
                        q_sha=sha(q), k_sha=sha(k), v_sha=sha(v))
    meta["fixtures"]["seed42_16x257.npz"] = "make_problem(42,16,257,576,512) exact64; attention_ref and run_etap{16,64,2}"

    # 2. MLA decode cases on bf16-rounded inputs: attention_ref per sequence (binary64)
    cases = {
        "mla_b1_h16_ctx1024": (42, [1024], 16),              # config 1
        "mla_varlen_b4": (7, [100, 257, 64, 1], 16),          # ragged, partial pages
        "mla_b2_h32_ctx300": (11, [300, 129], 32),           # two head groups
    }
    for name, (seed0, ctxs, heads) in cases.items():
        os_, ls_, qs_, ks_ = [], [], [], []
        for b, ctx in enumerate(ctxs):
            s = seed0 + 7919 * b
            qb, kvb = mla_problem(s, heads, ctx)
            ob, lb = oracle.ref_run("ref", qb, kvb, kvb[:, :512].copy(), 1.0 / 24.0)
            os_.append(ob); ls_.append(lb); qs_.append(sha(qb)); ks_.append(sha(kvb))
        np.savez_compressed(OUT / f"{name}.npz", o=np.stack(os_), l=np.stack(ls_), seed=seed0,
                            seqlens=np.array(ctxs, dtype=np.int32), heads=heads, scale=1.0 / 24.0,
                            q_sha=np.array(qs_), kv_sha=np.array(ks_))
        meta["fixtures"][f"{name}.npz"] = (f"seed={seed0} (instance seeds seed+7919*b), ctx={ctxs}, H={heads}; "
                                           "Q/KV matrix_from_seed rounded to bf16 RNE, V=KV[:,:512]; attention_ref")

    # 3. reference test_etap.cpp:231-240 — fp16emu run_etap RMSE at 8 x 512 x 64/64
    q, k, v, sc = oracle.ref_make_problem(42, 8, 512, 64, 64, -1.0, 2)
    o_ref, _ = oracle.ref_run("ref", q, k, v, sc, precision=0)
    o_et, _ = oracle.ref_run("etap", q, k, v, sc, precision=2, b_r=8, b_c=64)
    o_st, _ = oracle.ref_run("standard", q, k, v, sc, precision=2, b_r=8, b_c=64)
    rm = lambda a, b: float(np.sqrt(np.mean((a - b) ** 2)))  # noqa: E731
    meta["fp16emu_8x512x64"] = {"rmse_etap": rm(o_et, o_ref), "rmse_standard": rm(o_st, o_ref)}

    (OUT / "golden.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
