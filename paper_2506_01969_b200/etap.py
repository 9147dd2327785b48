# SPDX-License-Identifier: Apache-2.0
"""Mirror of the reference's operator interface for the hot path, backed by the GPU.

Names, argument meaning and error behaviour follow etaplab (paths relative to
/root/reference/proj):
  * ``AttentionProblem`` / ``AttentionOutput``  include/etaplab/attention.hpp:15-30
  * ``TileConfig``                              include/etaplab/tiled_standard.hpp:11-15
  * ``EtapFaults``                              include/etaplab/etap.hpp:39-41
  * ``make_problem``                            src/attention.cpp:10-42
  * ``run_etap``                                include/etaplab/etap.hpp:47-48, src/etap.cpp:102-148
std::invalid_argument maps to ``EtapShapeError`` (a ValueError).

Scope: the GPU path is MLA decode — d_qk = 576, d_v = 512 and V = K[:, :512] (the latent KV
aliasing). ``make_mla_problem`` builds such a problem from the reference's seeded generator;
a problem with an independent V is rejected (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import EtapShapeError, check

PRECISIONS = ("exact64", "fp32", "fp16emu", "bf16")


@dataclass
class TileConfig:
    b_r: int = 64    # query block size (GPU: 16 heads per CTA work unit)
    b_c: int = 64    # KV block size (GPU: one 64-row page per tile)
    stages: int = 2  # circular buffer depth (GPU: 24 chunk slots), no numeric effect


@dataclass
class EtapFaults:
    negate_rescale: bool = False


@dataclass
class AttentionProblem:
    n_q: int
    n_kv: int
    d_qk: int
    d_v: int
    scale: float
    precision: str
    q: np.ndarray  # n_q x d_qk, float64
    k: np.ndarray  # n_kv x d_qk
    v: np.ndarray  # n_kv x d_v


@dataclass
class SoftmaxState:  # tiled_standard.hpp:23-26
    m: np.ndarray
    l: np.ndarray


@dataclass
class BlockStepInfo:  # tiled_standard.hpp:32-38
    query_block: int
    kv_block: int
    m_old: np.ndarray
    state: SoftmaxState
    rescale: np.ndarray


@dataclass
class AttentionOutput:
    o: np.ndarray              # n_q x d_v
    l: np.ndarray = field(default_factory=lambda: np.zeros(0))  # per-query logsumexp


def _bf16_round(x: np.ndarray) -> np.ndarray:
    """binary64 -> bfloat16 round-to-nearest-even (single rounding), widened back."""
    import torch

    from .inputs import bf16_rne

    return bf16_rne(torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))).double().numpy()


def make_problem(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float,
                 precision: str = "bf16") -> AttentionProblem:
    """Validating constructor (attention.cpp:10-31): shape consistency, finite scale >= 0,
    operands rounded to ``precision`` (the GPU consumes bf16; exact64 keeps them)."""
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    k = np.atleast_2d(np.asarray(k, dtype=np.float64))
    v = np.atleast_2d(np.asarray(v, dtype=np.float64))
    if k.shape[1] != q.shape[1]:
        raise EtapShapeError("K head dimension does not match Q")
    if v.shape[0] != k.shape[0]:
        raise EtapShapeError("V context length does not match K")
    if not (scale >= 0.0) or not math.isfinite(scale):
        raise EtapShapeError("scale must be finite and >= 0")
    if precision not in PRECISIONS:
        raise EtapShapeError(f"unknown precision {precision!r}")
    if precision == "bf16":
        q, k = _bf16_round(q), _bf16_round(k)
        # keep the MLA aliasing exact after rounding when V is the K prefix
        v = k[:, :v.shape[1]].copy() if _is_prefix(v, k) else _bf16_round(v)
    return AttentionProblem(q.shape[0], k.shape[0], q.shape[1], v.shape[1], float(scale), precision,
                            np.ascontiguousarray(q), np.ascontiguousarray(k), np.ascontiguousarray(v))


def _is_prefix(v: np.ndarray, k: np.ndarray) -> bool:
    return v.shape[0] == k.shape[0] and v.shape[1] <= k.shape[1] and np.array_equal(v, k[:, :v.shape[1]])


def make_mla_problem(seed: int, n_q: int, n_kv: int, scale: float = -1.0) -> AttentionProblem:
    """Seeded MLA instance in the reference's conventions (attention.cpp:33-42): Q from
    sub-seed 3s+1, latent KV from 3s+2, both normal(0,1), rounded to bf16; V = KV[:, :512]
    (the reference's independent V stream 3s+3 is replaced by the MLA aliasing)."""
    import torch

    from .inputs import splitmix_normal

    if scale < 0:
        scale = 1.0 / math.sqrt(576.0)
    q = splitmix_normal(n_q * 576, 3 * seed + 1, "cpu").view(n_q, 576).numpy()
    kv = splitmix_normal(n_kv * 576, 3 * seed + 2, "cpu").view(n_kv, 576).numpy()
    del torch
    return make_problem(q, kv, kv[:, :512], scale, "bf16")


def run_etap(problem: AttentionProblem, tiles: TileConfig = TileConfig(),
             hook: Optional[Callable[[BlockStepInfo], None]] = None,
             faults: EtapFaults = EtapFaults(), eager: Optional[bool] = None) -> AttentionOutput:
    """GPU run_etap (etap.hpp:47-48) through the C-ABI entry ``etap_mla_run_etap_f64``.

    Raises EtapShapeError where the reference throws std::invalid_argument (tile fields < 1,
    etap.cpp:104-106) and for problems outside the GPU path's scope (d_qk != 576, d_v != 512,
    V not the first 512 columns of K).

    ``hook`` (BlockHook, tiled_standard.hpp:32-40): the device cannot call back per KV block,
    so the kernel records its softmax state (one split, the reference's serial block order)
    and the hook is replayed after the run exactly as run_etap calls it (etap.cpp:115-129):
    query blocks of ``tiles.b_r`` rows (outer), KV blocks of ``tiles.b_c`` rows (inner), each
    with BlockStepInfo(query_block, kv_block, m_old, SoftmaxState(m, l), rescale) over the
    block's query rows. Block boundaries off the 64-row tile grid are observed through prefix
    sequences (etap_mla_run_etap_f64_state). With a hook the rescale order defaults to the
    reference's eager one (``eager=True``); the default lazy mode gives the same invariants.

    ``problem.precision``: "exact64" and "bf16" (this mirror's name for exact64 storage rounded
    to bf16) map to the GPU's bf16 x bf16 -> fp32; the reference's fp32 / fp16emu emulation
    modes raise EtapShapeError instead of being computed differently.
    """
    if tiles.b_r < 1 or tiles.b_c < 1 or tiles.stages < 1:
        raise EtapShapeError("tile config fields must be >= 1")
    p = problem
    if p.precision not in ("exact64", "bf16"):
        raise EtapShapeError(f"precision {p.precision!r} is not mapped to the GPU path (exact64 / bf16 only)")
    if p.d_qk != 576 or p.d_v != 512:
        raise EtapShapeError("GPU ETAP path is MLA decode: d_qk=576, d_v=512")
    if not _is_prefix(p.v, p.k):
        raise EtapShapeError("GPU ETAP path requires V = K[:, :512] (MLA latent aliasing)")
    q = np.ascontiguousarray(p.q, dtype=np.float64)
    k = np.ascontiguousarray(p.k, dtype=np.float64)
    v = np.ascontiguousarray(p.v, dtype=np.float64)
    o = np.empty((p.n_q, p.d_v))
    l = np.empty(p.n_q)
    flags = _lib.FLAG_NEGATE_RESCALE if faults.negate_rescale else 0
    if eager if eager is not None else hook is not None:
        flags |= _lib.FLAG_EAGER_RESCALE
    vp = C.c_void_p
    if hook is None:
        check(_lib.lib().etap_mla_run_etap_f64(
            q.ctypes.data_as(vp), p.n_q, k.ctypes.data_as(vp), p.n_kv, p.d_qk, v.ctypes.data_as(vp), p.d_v,
            float(p.scale), _lib.PRECISION_EXACT64, tiles.b_r, tiles.b_c, tiles.stages, flags,
            o.ctypes.data_as(vp), l.ctypes.data_as(vp)), "etap_mla_run_etap_f64")
        return AttentionOutput(o, l)
    t_c = (p.n_kv + tiles.b_c - 1) // tiles.b_c
    state = np.empty((t_c, 4, p.n_q))
    check(_lib.lib().etap_mla_run_etap_f64_state(
        q.ctypes.data_as(vp), p.n_q, k.ctypes.data_as(vp), p.n_kv, p.d_qk, v.ctypes.data_as(vp), p.d_v,
        float(p.scale), _lib.PRECISION_EXACT64, tiles.b_c, flags, o.ctypes.data_as(vp), l.ctypes.data_as(vp),
        state.ctypes.data_as(vp)), "etap_mla_run_etap_f64_state")
    for qb, h0 in enumerate(range(0, p.n_q, tiles.b_r)):
        h1 = min(p.n_q, h0 + tiles.b_r)
        for j in range(t_c):
            st = state[j, :, h0:h1]
            hook(BlockStepInfo(qb, j, st[0].copy(), SoftmaxState(st[1].copy(), st[3].copy()), st[2].copy()))
    return AttentionOutput(o, l)


def rmse(a: np.ndarray, b: np.ndarray) -> float:
    """sqrt(mean((a - b)^2)) (matrix.cpp:235-245)."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        raise EtapShapeError("rmse shape mismatch")
    return float(np.sqrt(np.mean((a - b) ** 2)))
