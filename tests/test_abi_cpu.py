# SPDX-License-Identifier: Apache-2.0
"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every symbol that
include/etap_mla.h declares, validates arguments like the reference (std::invalid_argument ->
ETAP_ERR_SHAPE) and refuses to compute without a GPU (no CPU fallback)."""
from __future__ import annotations

import ctypes as C
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2506_01969_b200 import _lib, etap, inputs, mla

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols() -> list[str]:
    text = (ROOT / "include" / "etap_mla.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(etap_mla_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (etap_mla_\w+)", out))
    assert set(syms) <= exported


def test_python_constants_match_the_header():
    text = (ROOT / "include" / "etap_mla.h").read_text()
    consts = {k: int(v) for k, v in re.findall(r"#define (ETAP_(?:FLAG|ERR|OK)\w*)\s+(\d+)u?", text)}
    assert consts["ETAP_OK"] == _lib.ETAP_OK
    assert consts["ETAP_ERR_SHAPE"] == _lib.ETAP_ERR_SHAPE and consts["ETAP_ERR_CUDA"] == _lib.ETAP_ERR_CUDA
    flags = {k[len("ETAP_FLAG_"):]: v for k, v in consts.items() if k.startswith("ETAP_FLAG_")}
    assert len(flags) >= 5
    for name, v in flags.items():
        assert getattr(_lib, "FLAG_" + name) == v, name
    assert len(set(flags.values())) == len(flags)


def test_library_targets_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05 + TMA, not HMMA
    assert " HMMA" not in sass


def test_sizes_and_shape_validation():
    L = _lib.lib()
    a, b = C.c_size_t(), C.c_size_t()
    assert L.etap_mla_sched_ints(16, 16, 148, C.byref(a), C.byref(b)) == _lib.ETAP_OK
    assert a.value == 148 * 8 and b.value == 17
    assert L.etap_mla_sched_ints(16, 24, 148, C.byref(a), C.byref(b)) == _lib.ETAP_ERR_SHAPE
    ws = C.c_size_t()
    assert L.etap_mla_workspace_bytes(16, 16, 148, C.byref(ws)) == _lib.ETAP_OK
    al = lambda x: (x + 1023) // 1024 * 1024  # noqa: E731
    # partial O + LSE (16 heads per unit), then the FP8 path's per-CTA Q-term scratch (3 slots)
    assert ws.value == al((148 + 16) * 16 * (512 + 1) * 4) + 148 * 3 * 48 * 576
    # head groups: 32 heads per work unit when heads % 32 == 0, else 16
    assert [mla.head_group(h) for h in (16, 32, 48, 64, 96, 128)] == [16, 32, 16, 64, 32, 64]
    # the schedule unit: 128-head units over CTA pairs for multiples of 128 (num_sm_parts >= 2)
    assert [mla.schedule_unit(h, 148) for h in (16, 64, 128, 256)] == [(16, 148), (64, 148), (128, 74), (128, 74)]
    assert mla.schedule_unit(128, 1) == (64, 1) and mla.schedule_unit(128, 7) == (128, 3)
    assert L.etap_mla_sched_ints(4, 128, 148, C.byref(a), C.byref(b)) == _lib.ETAP_OK and b.value == 4 * 8 + 1
    assert L.etap_mla_workspace_bytes(4, 128, 148, C.byref(ws)) == _lib.ETAP_OK
    assert ws.value == al((148 + 4 * 2) * 64 * (512 + 1) * 4) + 148 * 3 * 48 * 576
    hg = C.c_int()
    assert L.etap_mla_head_group(24, C.byref(hg)) == _lib.ETAP_ERR_SHAPE
    # decode rejects q_tokens outside [1, 8], q_tokens * heads not a multiple of 16 and a bad
    # scale before touching the device
    rc = L.etap_mla_decode(1, 1, 1, 1, 1, 1, 1, 9, 16, 1.0, 1, 1, 1, 148, 16, 16, 16, 0, None)
    assert rc == _lib.ETAP_ERR_SHAPE and "q_tokens" in _lib.last_error()
    rc = L.etap_mla_decode(1, 1, 1, 1, 1, 1, 1, 0, 16, 1.0, 1, 1, 1, 148, 16, 16, 16, 0, None)
    assert rc == _lib.ETAP_ERR_SHAPE and "q_tokens" in _lib.last_error()
    rc = L.etap_mla_decode(1, 1, 1, 1, 1, 1, 1, 3, 8, 1.0, 1, 1, 1, 148, 16, 16, 16, 0, None)
    assert rc == _lib.ETAP_ERR_SHAPE and "multiple of 16" in _lib.last_error()
    rc = L.etap_mla_decode(1, 1, 1, 1, 1, 1, 1, 1, 16, float("nan"), 1, 1, 1, 148, 16, 16, 16, 0, None)
    assert rc == _lib.ETAP_ERR_SHAPE and "scale" in _lib.last_error()
    # O rows are stored and split partials loaded as float4: out / workspace must be 16-byte aligned
    rc = L.etap_mla_decode(16, 16, 1, 16, 1, 16, 1, 1, 16, 1.0, 1, 16, 16, 148, 16, 20, 16, 0, None)
    assert rc == _lib.ETAP_ERR_SHAPE and "aligned" in _lib.last_error()
    rc = L.etap_mla_decode_fp8(16, 16, 1.0, 1, 16, 1, 16, 1, 1, 16, 1.0, 1, 16, 16, 148, 24, 16, 16, 0, None)
    assert rc == _lib.ETAP_ERR_SHAPE and "aligned" in _lib.last_error()


def test_reference_error_behaviour_mirrored():
    p = etap.make_mla_problem(42, 16, 100)
    with pytest.raises(_lib.EtapShapeError, match="tile config"):
        etap.run_etap(p, etap.TileConfig(1, 0, 2))
    with pytest.raises(_lib.EtapShapeError, match="K head dimension"):
        etap.make_problem(np.ones((2, 4)), np.ones((3, 5)), np.ones((3, 2)), 1.0)
    with pytest.raises(_lib.EtapShapeError, match="scale"):
        etap.make_problem(np.ones((2, 4)), np.ones((3, 4)), np.ones((3, 2)), -1.0)
    with pytest.raises(_lib.EtapShapeError, match="MLA"):
        etap.run_etap(etap.make_problem(np.ones((2, 4)), np.ones((3, 4)), np.ones((3, 2)), 1.0, "exact64"))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    p = etap.make_mla_problem(42, 16, 100)
    with pytest.raises(_lib.EtapError):
        etap.run_etap(p)
    L = _lib.lib()
    n = C.c_int()
    assert L.etap_mla_num_sm_parts(0, C.byref(n)) == _lib.ETAP_ERR_CUDA


def test_host_metadata_partition_invariants():
    """The split-KV schedule (host restatement of K1) covers every (sequence, head group,
    page) exactly once, numbers partials contiguously per sequence and balances the load.
    Virtual sequences are head-group major (vb = g * batch + b); with several head groups the
    CTAs form one lane per group and every lane cuts the same line (same page ranges)."""
    L = _lib.lib()
    cases = [([65536] * 16, 16, 148), (inputs.varlen_seqlens(32), 16, 148), ([0, 1, 64, 65, 0], 32, 148),
             ([100], 16, 3), ([1024], 16, 148), ([10**6], 128, 148), ([7] * 300, 16, 148),
             ([65536] * 16, 128, 148), ([4096] * 64, 128, 148), ([100, 3000], 64, 3), ([5000], 128, 2),
             ([0, 0, 900], 96, 148)]
    for seqlens, heads, nparts in cases:
        unit, parts = mla.schedule_unit(heads, nparts)  # 128-head units over CTA pairs when they run it
        B, G = len(seqlens), heads // unit
        sched = np.zeros(nparts * 8, np.int32)
        so = np.zeros(B * G + 1, np.int32)
        sl = np.array(seqlens, np.int32)
        assert L.etap_mla_metadata_host(sl.ctypes.data_as(C.c_void_p), B, heads, nparts,
                                        sched.ctypes.data_as(C.c_void_p), so.ctypes.data_as(C.c_void_p)) == 0
        lanes = G if (G > 1 and parts >= G) else 1
        p_line = parts // lanes
        tiles = [(seqlens[vb % B] + 63) // 64 for vb in range(B * G)]
        cover = [np.zeros(t, np.int32) for t in tiles]
        count = np.zeros(B * G, np.int32)
        idx_seen = {}
        work = []
        for k in range(parts):
            p0, t0, p1, t1, first, off = sched[k * 8:k * 8 + 6]
            if lanes > 1 and k < lanes * p_line:  # lanes share the cut of line CTA k % p_line
                assert off == (k // p_line) * B
                assert np.array_equal(sched[k * 8:k * 8 + 4], sched[(k % p_line) * 8:(k % p_line) * 8 + 4])
            w = 0
            for pos in range(p0, p1 + 1):
                vb = off + pos
                a = t0 if pos == p0 else 0
                e = t1 if pos == p1 else tiles[vb]
                if a < e:
                    cover[vb][a:e] += 1
                    idx = first if pos == p0 else so[vb]
                    assert so[vb] <= idx < so[vb + 1]
                    assert idx not in idx_seen
                    idx_seen[idx] = (k, vb)
                    count[vb] += 1
                    w += e - a
            work.append(w)
        for c in cover:
            assert (c == 1).all()
        assert np.array_equal(np.diff(so), count)
        total = sum(tiles)
        active = lanes * p_line
        if total >= active * 4:
            assert max(work) <= total / active + 4  # balanced to within the per-split overhead


def test_peer_gather_descriptor_and_validation():
    """etap_mla_peer_gather (include/etap_mla.h) as seen from Python, and the fused-all-gather
    entry point rejecting bad descriptors before touching the device."""
    from paper_2506_01969_b200 import peer

    assert C.sizeof(peer.PeerGatherDesc) == 4 * 4 + 3 * 8 * 8
    L = _lib.lib()
    d = peer.PeerGatherDesc()
    d.world, d.rank, d.heads_total, d.head_offset = 9, 0, 128, 0
    args = (1, 1, 1, 1, 1, 1, 1, 1, 16, 1.0, 1, 1, 1, 148, 1)
    assert L.etap_mla_decode_peer(*args, C.byref(d), 1, 0, None) == _lib.ETAP_ERR_SHAPE
    assert "world" in _lib.last_error()
    d.world, d.rank, d.head_offset = 2, 1, 120
    assert L.etap_mla_decode_peer(*args, C.byref(d), 1, 0, None) == _lib.ETAP_ERR_SHAPE
    assert "head_offset" in _lib.last_error()
    d.head_offset = 16
    assert L.etap_mla_decode_peer(*args, C.byref(d), 0, 0, None) == _lib.ETAP_ERR_SHAPE
    assert "epoch" in _lib.last_error()
    assert L.etap_mla_decode_peer(*args, None, 1, 0, None) == _lib.ETAP_ERR_SHAPE


def test_bf16_rounding_of_binary64_operands_is_bit_exact():
    """etap_mla_run_etap_f64 rounds the reference's binary64 AttentionProblem storage to bf16
    (ties to even, single rounding) with a bit-level fast path; it must equal the frexp /
    nearbyint reference form on random values, ties, carries into the exponent, the bf16
    subnormal range, overflow and non-finite values."""
    rng = np.random.default_rng(7)
    parts = [
        rng.standard_normal(200000) * 10.0 ** rng.integers(-45, 40, 200000),
        rng.standard_normal(20000),
        # exact ties and near-ties at bf16 resolution: 1 + k/256 (+- 1 ulp of binary64)
        (1 + np.arange(512) / 256.0) * 2.0 ** rng.integers(-130, 128, 512),
        np.nextafter(1 + np.arange(512) / 256.0, 2), np.nextafter(1 + np.arange(512) / 256.0, 0),
        (2 - 2.0 ** -9) * 2.0 ** np.arange(-130, 128),  # rounds up into the next binade
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 3.3895313892515355e38, 3.3961e38, 3.4e38, 1e300,
                  -1e300, 2.0 ** -126, 2.0 ** -127, 2.0 ** -133, 2.0 ** -134, 1.5 * 2.0 ** -134, 5e-324,
                  np.nextafter(2.0 ** -126, 0)]),
    ]
    x = np.ascontiguousarray(np.concatenate(parts), dtype=np.float64)
    fast = np.empty(x.size, dtype=np.uint16)
    ref = np.empty(x.size, dtype=np.uint16)
    L = _lib.lib()
    assert L.etap_mla_debug_bf16_rne(x.ctypes.data, x.size, fast.ctypes.data, 0) == 0
    assert L.etap_mla_debug_bf16_rne(x.ctypes.data, x.size, ref.ctypes.data, 1) == 0
    bad = np.nonzero(fast != ref)[0]
    assert bad.size == 0, [(x[i], hex(fast[i]), hex(ref[i])) for i in bad[:5]]
    # and both agree with torch's own RNE on everything that is not a float32 double-rounding case
    with np.errstate(over="ignore", invalid="ignore"):
        x32 = x.astype(np.float32)
        same32 = x32.astype(np.float64) == x
    t = torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert (fast[same32] == t[same32]).all()
