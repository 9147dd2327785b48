# SPDX-License-Identifier: Apache-2.0
"""Per-tile pipeline trace of the decode kernel (debug %globaltimer stamps, see
etap_mla_debug_trace in include/etap_mla.h). Prints where each tile's time goes.

    python scripts/trace_pipeline.py [--batch 16 --ctx 65536]
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

from paper_2506_01969_b200 import _lib, inputs, mla

TRACE_TILES = 256


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--ctx", type=int, default=65536)
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--fp8", action="store_true", help="FP8 (e4m3) latent cache (decode_fp8)")
    a = ap.parse_args()
    inp = inputs.make_mla_inputs([a.ctx] * a.batch, heads=a.heads, pad_value=0.0)
    plan = mla.MlaDecodePlan.create(a.batch, a.heads, "cuda")
    if a.fp8:
        kv8 = (inp.kv_pool.float() / 0.125).to(torch.float8_e4m3fn)
        plan.decode = lambda q, kv, bt, sl, sc: mla.MlaDecodePlan.decode_fp8(plan, q, kv8, bt, sl, sc, 0.125)
    nparts = plan.num_sm_parts
    buf = torch.zeros(nparts * TRACE_TILES * 16, dtype=torch.int64, device="cuda")
    for _ in range(2):
        plan.metadata(inp.seqlens)
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    torch.cuda.synchronize()
    _lib.lib().etap_mla_debug_trace(buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.metadata(inp.seqlens)
    plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
    e1.record()
    torch.cuda.synchronize()
    _lib.lib().etap_mla_debug_trace(None)
    print(f"traced step: {e0.elapsed_time(e1) * 1000:.1f} us")
    raw = buf.view(nparts, TRACE_TILES, 16).cpu().numpy()
    # re-base in int64 first: %globaltimer ns since the epoch (~1.7e18) has a float64 ulp of 256
    gbase = raw[:, TRACE_TILES - 1, 0].min()
    ent = (raw[:, TRACE_TILES - 1, :3] - gbase).astype(np.float64)
    # tile rows are SM clock64 cycles: convert with each CTA's measured clock (row 255, 5/6)
    ghz = (raw[:, TRACE_TILES - 1, 6] - raw[:, TRACE_TILES - 1, 5]).astype(np.float64) / np.maximum(1.0, ent[:, 2] - ent[:, 0])
    print(f"SM clock during the step: {np.median(ghz):.3f} GHz (median over CTAs)")
    valid = (raw[:, :TRACE_TILES - 1, :8] > 0).all(axis=2)
    # cycles -> ns on each CTA's clock, re-based to the CTA's global entry time
    t = (raw[:, :TRACE_TILES - 1, :] - raw[:, TRACE_TILES - 1, 5][:, None, None]).astype(np.float64)
    t = t / ghz[:, None, None] + ent[:, 0][:, None, None]
    t0 = t[valid].min()
    rows = []
    for c in range(nparts):
        n = int(valid[c].sum())
        for g in range(2, n - 1):
            e = t[c, g]
            nxt = t[c, g + 1]
            rows.append([
                e[2] - e[1],            # latency of the last chunk (issue -> landed seen by MMA)
                e[1] - e[0],            # producer: span issuing the tile's 9 chunks
                e[3] - e[2],            # GEMM1 tail issue after last chunk
                e[4] - e[3],            # S commit -> softmax sees S (GEMM1 execution)
                e[8] - e[4],            # softmax: S -> exp done
                e[9] - e[8],            # softmax: wait for the P buffer (GEMM2 of tile g-2)
                e[5] - e[9],            # softmax: P write + fences
                e[6] - e[5],            # P written -> MMA sees it
                e[7] - e[6],            # GEMM2 issue
                nxt[3] - e[3],          # tile period
                nxt[0] - e[7],          # GEMM2(g) commit -> producer issues first chunk of g+1
                nxt[1] - e[7],          # GEMM2(g) commit -> producer issued last chunk of g+1
                nxt[4] - e[5],          # softmax idle: P(g) written -> sees S(g+1)
                e[12] - e[4],           # softmax: TMEM load of S (bf16 kernel)
                e[13] - e[12],          # softmax: lazy-rescale vote (bar.red.or) wait
                e[8] - e[13],           # softmax: max exchange (if any) + exp
            ])
    r = np.array(rows) if rows else np.zeros((0, 16))
    labels = ["lat_tile(last issue->seen)", "issue_span", "g1_issue", "s_ready_wait", "softmax_exp",
              "softmax_pbuf_wait", "softmax_pwrite", "p_to_mma", "g2_issue", "PERIOD", "g2->next_first_issue",
              "g2->next_last_issue", "softmax_idle", "  s_tmem_ld", "  vote_wait", "  exp"]
    print(f"{len(rows)} steady-state tiles over {nparts} CTAs (ns): median / p10 / p90")
    for i, lab in enumerate(labels):
        if not len(r):
            break
        col = r[:, i]
        print(f"  {lab:26s} {np.median(col):9.0f} {np.percentile(col, 10):9.0f} {np.percentile(col, 90):9.0f}")
    # first tile of every working CTA, relative to kernel entry (us)
    first = [(t[c, 0] - ent[c, 0]) / 1e3 for c in range(nparts) if valid[c, 0]]
    if first:
        f = np.array(first)
        names0 = ["producer: first 6 chunks issued", "last 3 chunks issued", "G1 sees tile", "S committed",
                  "softmax sees S", "P written", "G2 sees P", "G2 committed"]
        print("first tile, us after kernel entry (median over CTAs):")
        for i, n in enumerate(names0):
            print(f"  {n:34s} {np.median(f[:, i]):7.2f}")
        print(f"  {'schedule done':34s} {np.median((ent[:, 1] - ent[:, 0]) / 1e3):7.2f}")
        print(f"  {'CTA exit':34s} {np.median((ent[:, 2] - ent[:, 0]) / 1e3):7.2f}")
    # CTA span
    span = [(t[c][valid[c]].max() - t[c][valid[c]].min()) for c in range(nparts) if valid[c].any()]
    starts = [t[c][valid[c]].min() - t0 for c in range(nparts) if valid[c].any()]
    print(f"CTA busy span us: median {np.median(span) / 1e3:.1f} max {np.max(span) / 1e3:.1f}; "
          f"start offsets us: max {np.max(starts) / 1e3:.1f}")
    print("tiles per CTA:", np.bincount(valid.sum(axis=1)).nonzero()[0].tolist())
    e0 = ent[:, 0].min()
    first_issue = np.array([t[c][valid[c]][:, 0].min() if valid[c].any() else np.nan for c in range(nparts)])
    last_g2 = np.array([t[c][valid[c]][:, 7].max() if valid[c].any() else np.nan for c in range(nparts)])
    print(f"kernel entry spread us: {(ent[:, 0].max() - e0) / 1e3:.2f}; prologue+dep-wait us (median): "
          f"{np.median(ent[:, 1] - ent[:, 0]) / 1e3:.2f}; dep-wait done -> first TMA issue us (median): "
          f"{np.nanmedian(first_issue - ent[:, 1]) / 1e3:.2f}")
    sched = plan.sched.view(nparts, 8).cpu().numpy()
    spans = ent[:, 2] - ent[:, 0]
    ntiles = valid.sum(axis=1)
    nsplit = np.array([sum(1 for vb in range(s[0], s[2] + 1)
                           if (s[1] if vb == s[0] else 0) < (s[3] if vb == s[2] else 10**9)) for s in sched])
    for ns_ in sorted(set(nsplit.tolist())):
        for nt in sorted(set(ntiles[nsplit == ns_].tolist())):
            sel = (nsplit == ns_) & (ntiles == nt)
            print(f"  splits={ns_} tiles={nt}: CTAs {sel.sum():3d}, span us median {np.median(spans[sel]) / 1e3:.1f} "
                  f"max {spans[sel].max() / 1e3:.1f}")
    print(f"last G2 commit -> CTA exit us (median/max): {np.nanmedian(ent[:, 2] - last_g2) / 1e3:.2f} / "
          f"{np.nanmax(ent[:, 2] - last_g2) / 1e3:.2f}; entry -> last exit us: {(ent[:, 2].max() - e0) / 1e3:.1f}")


if __name__ == "__main__":
    main()
