# SPDX-License-Identifier: Apache-2.0
"""Device-side API over the C-ABI: paged MLA decode on torch CUDA tensors.

PyTorch is used only for device memory and streams; all compute runs in the sm_100a kernels
of libetap_mla.so (K1 scheduler, K2 transposed tcgen05 pipeline, K3 combine).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (FLAG_DEP_METADATA, FLAG_EAGER_RESCALE, FLAG_EARLY_METADATA,  # noqa: F401
                   FLAG_EXTERNAL_SCHEDULE, FLAG_INDEPENDENT_INPUTS, FLAG_NEGATE_RESCALE, FLAG_SKIP_COMBINE, check)

D_QK = 576
D_V = 512
PAGE_ROWS = 64
TILE_ROWS = 64
HEAD_GROUP = 16  # minimum heads per CTA work unit; see head_group()
SCHED_INTS = 8


def head_group(heads: int) -> int:
    """Heads per CTA work unit of the single-CTA kernels (64 / 32 / 16 as the head count allows),
    the unit the buffer sizes follow; see schedule_unit() for the CTA-pair kernel's 128."""
    out = C.c_int(0)
    check(_lib.lib().etap_mla_head_group(heads, C.byref(out)), "etap_mla_head_group")
    return out.value


def schedule_unit(heads: int, num_parts: int) -> tuple[int, int]:
    """(heads per schedule unit, schedule parts): 128-head units over num_parts / 2 CTA pairs when
    the pair kernel runs the head count, else (head_group(heads), num_parts)."""
    unit, parts = C.c_int(0), C.c_int(0)
    check(_lib.lib().etap_mla_schedule_unit(heads, num_parts, C.byref(unit), C.byref(parts)),
          "etap_mla_schedule_unit")
    return unit.value, parts.value


def _dev_index(device: torch.device | str | int | None) -> int:
    if device is None:
        return torch.cuda.current_device()
    if isinstance(device, int):
        return device
    device = torch.device(device)
    return device.index if device.index is not None else torch.cuda.current_device()


def num_sm_parts(device: torch.device | str | int | None = None) -> int:
    out = C.c_int(0)
    check(_lib.lib().etap_mla_num_sm_parts(_dev_index(device), C.byref(out)), "etap_mla_num_sm_parts")
    return out.value


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream_ptr(stream: torch.cuda.Stream | None) -> int:
    if stream is not None:
        return stream.cuda_stream
    # the current device's current stream without building a Stream object (~0.3 us instead
    # of ~3 us per call: at 1K contexts the host-side cost of a decode call is the step)
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


@dataclass
class MlaDecodePlan:
    """Scratch buffers (schedule, split offsets, split-KV workspace) for one shape.

    Mirrors the FlashMLA-style two-call protocol: ``metadata(seqlens)`` once per decode step
    (reusable across layers), then ``decode(...)`` per layer.
    """

    batch: int
    heads: int
    device: torch.device
    num_sm_parts: int
    sched: torch.Tensor
    split_off: torch.Tensor
    workspace: torch.Tensor
    q_tokens: int = 1  # query tokens per sequence (multi-token / MTP decode)

    @property
    def rows(self) -> int:
        """Query rows per sequence (tokens folded into heads): the C-ABI's sizing `heads`."""
        return self.q_tokens * self.heads

    @classmethod
    def create(cls, batch: int, heads: int, device: torch.device | str = "cuda",
               num_parts: int | None = None, q_tokens: int = 1) -> "MlaDecodePlan":
        device = torch.device(device)
        if device.type != "cuda":
            raise _lib.EtapShapeError("MlaDecodePlan needs a CUDA device (no CPU fallback)")
        L = _lib.lib()
        nparts = num_parts if num_parts is not None else num_sm_parts(device)
        n_sched, n_so, ws = C.c_size_t(0), C.c_size_t(0), C.c_size_t(0)
        rows = q_tokens * heads
        check(L.etap_mla_sched_ints(batch, rows, nparts, C.byref(n_sched), C.byref(n_so)),
              "etap_mla_sched_ints")
        check(L.etap_mla_workspace_bytes(batch, rows, nparts, C.byref(ws)), "etap_mla_workspace_bytes")
        return cls(
            batch=batch, heads=heads, device=device, num_sm_parts=nparts, q_tokens=q_tokens,
            # zero-filled once: the decode reads its previous-call range from it as an L2
            # prefetch hint before the schedule of this call is known
            sched=torch.zeros(n_sched.value, dtype=torch.int32, device=device),
            split_off=torch.zeros(n_so.value, dtype=torch.int32, device=device),
            # zero-filled once: the tail holds the combine's ready flags / counters, which every
            # decode call leaves at zero again
            workspace=torch.zeros(ws.value, dtype=torch.uint8, device=device),
        )

    def metadata(self, seqlens: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
        """K1: split-KV schedule for the current step's context lengths."""
        _check_tensor(seqlens, torch.int32, (self.batch,), "seqlens")
        check(_lib.lib().etap_mla_metadata(seqlens.data_ptr(), self.batch, self.rows, self.num_sm_parts,
                                           self.sched.data_ptr(), self.split_off.data_ptr(),
                                           _stream_ptr(stream)), "etap_mla_metadata")

    def decode(self, q: torch.Tensor, kv_pool: torch.Tensor, block_table: torch.Tensor,
               seqlens: torch.Tensor, scale: float, out: torch.Tensor | None = None,
               lse: torch.Tensor | None = None, flags: int = 0, causal: bool = True,
               stream: torch.cuda.Stream | None = None) -> tuple[torch.Tensor, torch.Tensor]:
        """K2 + K3. q [B,T,H,576] bf16 (T = q_tokens), kv_pool [pages,64,576] bf16, block_table
        [B,max_pages] int32, seqlens [B] int32 -> (out [B,T,H,512] fp32, lse [B,T,H] fp32, natural
        log). With T > 1 and ``causal`` token j sees KV rows [0, seqlen - T + j]."""
        q, out, lse = self._check_io(q, kv_pool, block_table, seqlens, out, lse, (torch.bfloat16,), "kv_pool")
        check(_lib.lib().etap_mla_decode(
            q.data_ptr(), kv_pool.data_ptr(), kv_pool.shape[0], block_table.data_ptr(),
            block_table.shape[1], seqlens.data_ptr(), self.batch, self.q_tokens, self.heads, float(scale), int(causal),
            self.sched.data_ptr(), self.split_off.data_ptr(), self.num_sm_parts,
            self.workspace.data_ptr(), out.data_ptr(), lse.data_ptr(), int(flags),
            _stream_ptr(stream)), "etap_mla_decode")
        return out, lse

    def decode_fp8(self, q: torch.Tensor, kv_pool8: torch.Tensor, block_table: torch.Tensor,
                   seqlens: torch.Tensor, scale: float, kv_scale: float, out: torch.Tensor | None = None,
                   lse: torch.Tensor | None = None, flags: int = 0, causal: bool = True,
                   stream: torch.cuda.Stream | None = None) -> tuple[torch.Tensor, torch.Tensor]:
        """K2-FP8 + K3 on an FP8 (e4m3) latent cache: kv_pool8 [pages,64,576] float8_e4m3fn (or
        its uint8 bytes), dequantised value = kv_scale * e4m3. Same q / block_table / seqlens /
        outputs as decode()."""
        q, out, lse = self._check_io(q, kv_pool8, block_table, seqlens, out, lse,
                                     (torch.float8_e4m3fn, torch.uint8), "kv_pool8")
        check(_lib.lib().etap_mla_decode_fp8(
            q.data_ptr(), kv_pool8.data_ptr(), float(kv_scale), kv_pool8.shape[0], block_table.data_ptr(),
            block_table.shape[1], seqlens.data_ptr(), self.batch, self.q_tokens, self.heads, float(scale),
            int(causal),
            self.sched.data_ptr(), self.split_off.data_ptr(), self.num_sm_parts,
            self.workspace.data_ptr(), out.data_ptr(), lse.data_ptr(), int(flags),
            _stream_ptr(stream)), "etap_mla_decode_fp8")
        return out, lse

    def _check_io(self, q, pool, block_table, seqlens, out, lse, pool_dtypes, pool_name, outputs=True):
        """Shape / dtype / device checks of one decode call (EtapShapeError, never a device fault);
        allocates out / lse when they are not given."""
        B, H, T = self.batch, self.heads, self.q_tokens
        if isinstance(q, torch.Tensor) and q.dim() == 3 and T == 1:
            q = q.unsqueeze(1)
        _check_tensor(q, torch.bfloat16, (B, T, H, D_QK), "q")
        if not isinstance(pool, torch.Tensor) or not pool.is_cuda:
            raise _lib.EtapShapeError(f"{pool_name} must be a CUDA tensor")
        if pool.dim() != 3 or pool.shape[1:] != (PAGE_ROWS, D_QK) or pool.dtype not in pool_dtypes \
                or not pool.is_contiguous():
            raise _lib.EtapShapeError(f"{pool_name} must be contiguous [pages,64,576] {pool_dtypes[0]}, got "
                                      f"{tuple(pool.shape)} {pool.dtype}")
        if not isinstance(block_table, torch.Tensor) or not block_table.is_cuda:
            raise _lib.EtapShapeError("block_table must be a CUDA tensor")
        if block_table.dim() != 2 or block_table.shape[0] != B or block_table.dtype != torch.int32 \
                or not block_table.is_contiguous():
            raise _lib.EtapShapeError("block_table must be contiguous [B, max_pages] int32")
        _check_tensor(seqlens, torch.int32, (B,), "seqlens")
        if not outputs:  # the caller owns the output buffers (peer gather)
            out, lse = q, seqlens  # device checks only
        if out is None:
            out = torch.empty((B, T, H, D_V), dtype=torch.float32, device=q.device)
        if lse is None:
            lse = torch.empty((B, T, H), dtype=torch.float32, device=q.device)
        if outputs:
            _check_tensor(out, torch.float32, (B, T, H, D_V), "out")
            _check_tensor(lse, torch.float32, (B, T, H), "lse")
        dev = self.device.index if self.device.index is not None else torch.cuda.current_device()
        for name, t in (("q", q), (pool_name, pool), ("block_table", block_table), ("seqlens", seqlens),
                        ("out", out), ("lse", lse)):
            if t.device.index != dev:
                raise _lib.EtapShapeError(f"{name} is on {t.device}, the plan on cuda:{dev}")
        return q, out, lse

    def capture(self, q: torch.Tensor, kv_pool: torch.Tensor, block_table: torch.Tensor,
                seqlens: torch.Tensor, scale: float, out: torch.Tensor, lse: torch.Tensor,
                flags: int = 0, with_metadata: bool = True) -> torch.cuda.CUDAGraph:
        """Capture one decode step (K1 -> K2 -> K3, programmatic dependent launches) into a
        CUDA graph; replay() re-runs it on the same buffers with one host call."""
        for _ in range(2):  # one-time host init (smem attributes) happens outside the capture
            if with_metadata:
                self.metadata(seqlens)
            self.decode(q, kv_pool, block_table, seqlens, scale, out=out, lse=lse, flags=flags)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            if with_metadata:
                self.metadata(seqlens)
            self.decode(q, kv_pool, block_table, seqlens, scale, out=out, lse=lse, flags=flags)
        return g

    def combine(self, out: torch.Tensor, lse: torch.Tensor, stream: torch.cuda.Stream | None = None) -> None:
        """K3 alone, after a decode(..., flags=FLAG_SKIP_COMBINE)."""
        check(_lib.lib().etap_mla_combine(self.split_off.data_ptr(), self.batch, self.rows, self.num_sm_parts,
                                          self.workspace.data_ptr(), out.data_ptr(), lse.data_ptr(),
                                          _stream_ptr(stream)), "etap_mla_combine")


def _check_tensor(t: torch.Tensor, dtype: torch.dtype, shape: tuple, name: str) -> None:
    if isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.shape == shape and t.is_contiguous():
        return
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise _lib.EtapShapeError(f"{name} must be a CUDA tensor")
    raise _lib.EtapShapeError(f"{name} must be contiguous {tuple(shape)} {dtype}, got {tuple(t.shape)} {t.dtype}")


def mla_decode(q: torch.Tensor, kv_pool: torch.Tensor, block_table: torch.Tensor,
               seqlens: torch.Tensor, scale: float, flags: int = 0,
               plan: MlaDecodePlan | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """One-shot convenience: K1 + K2 + K3 on the current stream. q [B,H,576] or
    [B,T,H,576] (T query tokens per sequence, causal)."""
    B, H = q.shape[0], q.shape[-2]
    T = q.shape[1] if q.dim() == 4 else 1
    plan = plan or MlaDecodePlan.create(B, H, q.device, q_tokens=T)
    plan.metadata(seqlens)
    return plan.decode(q, kv_pool, block_table, seqlens, scale, flags=flags)


def selftest_umma(k: torch.Tensor, q: torch.Tensor, p: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """Single-tile UMMA layout check. k [64,576] bf16, q [16,576] bf16, p [64,16] fp32 ->
    (S^T [64,16], O^T [512,32]) read back from TMEM; O^T columns 0-15 = V^T P_hi,
    16-31 = V^T P_lo (P = P_hi + P_lo in bf16)."""
    s_t = torch.empty((TILE_ROWS, HEAD_GROUP), dtype=torch.float32, device=k.device)
    o_t = torch.empty((D_V, 2 * HEAD_GROUP), dtype=torch.float32, device=k.device)
    check(_lib.lib().etap_mla_selftest_umma(k.data_ptr(), q.data_ptr(), p.data_ptr(), s_t.data_ptr(),
                                            o_t.data_ptr(), _stream_ptr(None)), "etap_mla_selftest_umma")
    return s_t, o_t


# ------------------------------------------------------------------ adjacent decode steps
def absorb_q(q_nope: torch.Tensor, q_pe: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor, w_uk: torch.Tensor,
             out: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Absorbed-MLA query: Q[b,t,h] = [q_nope[b,t,h] . W_UK[h] | RoPE(q_pe[b,t,h])] as the decode's
    bf16 [B, T, H, 576] input (etap_mla_absorb_q). q_nope [B,T,H,128], q_pe [B,T,H,64] bf16,
    cos/sin [B,T,32] fp32, w_uk [H,128,512] bf16."""
    B, T, H = q_nope.shape[:3]
    _check_tensor(q_nope, torch.bfloat16, (B, T, H, 128), "q_nope")
    _check_tensor(q_pe, torch.bfloat16, (B, T, H, 64), "q_pe")
    _check_tensor(cos, torch.float32, (B, T, 32), "cos")
    _check_tensor(sin, torch.float32, (B, T, 32), "sin")
    _check_tensor(w_uk, torch.bfloat16, (H, 128, D_V), "w_uk")
    if out is None:
        out = torch.empty((B, T, H, D_QK), dtype=torch.bfloat16, device=q_nope.device)
    _check_tensor(out, torch.bfloat16, (B, T, H, D_QK), "out")
    check(_lib.lib().etap_mla_absorb_q(q_nope.data_ptr(), q_pe.data_ptr(), cos.data_ptr(), sin.data_ptr(),
                                       w_uk.data_ptr(), B, T, H, out.data_ptr(), _stream_ptr(stream)),
          "etap_mla_absorb_q")
    return out


def up_proj(o: torch.Tensor, w_uv: torch.Tensor, out_dtype: torch.dtype = torch.bfloat16,
            stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Per-head value up-projection of the decode output: out[b,t,h] = O[b,t,h] . W_UV[h]
    (etap_mla_up_proj). o [B,T,H,512] fp32, w_uv [H,512,128] bf16 -> [B,T,H,128]."""
    B, T, H = o.shape[:3]
    _check_tensor(o, torch.float32, (B, T, H, D_V), "o")
    _check_tensor(w_uv, torch.bfloat16, (H, D_V, 128), "w_uv")
    if out_dtype not in (torch.bfloat16, torch.float32):
        raise _lib.EtapShapeError("out_dtype must be bfloat16 or float32")
    out = torch.empty((B, T, H, 128), dtype=out_dtype, device=o.device)
    check(_lib.lib().etap_mla_up_proj(o.data_ptr(), w_uv.data_ptr(), B, T, H, out.data_ptr(),
                                      int(out_dtype == torch.float32), _stream_ptr(stream)), "etap_mla_up_proj")
    return out
