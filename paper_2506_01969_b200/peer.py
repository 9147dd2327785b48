# SPDX-License-Identifier: Apache-2.0
"""Head-sharded decode with the all-gather of O fused into the kernels (NVLink peer memory).

SURVEY.md §8e: every rank owns a contiguous head block against the replicated latent KV and
the only exchange is the all-gather of O / LSE. ``sharding.gather_heads`` is the NCCL
baseline (decode, then ncclAllGather + permute). ``PeerGather`` removes the collective: each
rank's K2 epilogue / K3 store finished rows straight into every rank's full-head output
(buffers exported with CUDA IPC and mapped by every peer), and a one-warp arrival kernel
publishes an epoch so each rank knows all rows landed (etap_mla_decode_peer,
include/etap_mla.h). Host plumbing only: handles are exchanged with torch.distributed
(any backend), the data path never touches NCCL.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check
from .mla import D_V, MlaDecodePlan, _stream_ptr

MAX_PEERS = 8
HANDLE_BYTES = 64


class PeerGatherDesc(C.Structure):
    _fields_ = [("world", C.c_int), ("rank", C.c_int), ("heads_total", C.c_int), ("head_offset", C.c_int),
                ("out", C.c_void_p * MAX_PEERS), ("lse", C.c_void_p * MAX_PEERS),
                ("flags", C.c_void_p * MAX_PEERS)]


class _DevPtr:
    """__cuda_array_interface__ view of a raw device pointer (torch.as_tensor wraps it)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": shape, "typestr": typestr,
                                         "version": 3, "strides": None}


def _alloc(nbytes: int) -> tuple[int, bytes]:
    p = C.c_void_p()
    h = C.create_string_buffer(HANDLE_BYTES)
    check(_lib.lib().etap_mla_ipc_alloc(nbytes, C.byref(p), h), "etap_mla_ipc_alloc")
    return p.value, h.raw


def _open(handle: bytes) -> int:
    p = C.c_void_p()
    check(_lib.lib().etap_mla_ipc_open(C.create_string_buffer(handle, HANDLE_BYTES), C.byref(p)),
          "etap_mla_ipc_open")
    return p.value


class PeerAccessUnavailable(RuntimeError):
    """Some rank pair cannot map each other's memory (no CUDA peer access between their GPUs,
    or a peer GPU that is not visible to this process): the caller falls back to NCCL."""


def _device_uuid(index: int) -> str:
    return str(torch.cuda.get_device_properties(index).uuid)


def check_peer_access(my_index: int, uuids: list[str]) -> None:
    """Raise PeerAccessUnavailable unless this process can access every rank's GPU: the same
    device (CUDA IPC within one GPU) or a peer that cudaDeviceCanAccessPeer allows."""
    local = {_device_uuid(i): i for i in range(torch.cuda.device_count())}
    for r, u in enumerate(uuids):
        idx = local.get(u)
        if idx is None:
            raise PeerAccessUnavailable(f"rank {r}'s GPU {u} is not visible to this process")
        if idx != my_index and not torch.cuda.can_device_access_peer(my_index, idx):
            raise PeerAccessUnavailable(f"no CUDA peer access from GPU {my_index} to GPU {idx} (rank {r})")


class PeerGather:
    """Full-head output buffers shared by ``world`` ranks (``nbuf`` sets used round robin by
    epoch, so a rank one call ahead never overwrites rows a slower rank still reads)."""

    def __init__(self, batch: int, heads_local: int, world: int = 1, rank: int = 0, q_tokens: int = 1,
                 group=None, nbuf: int = 2, device: torch.device | str | None = None):
        if not 1 <= world <= MAX_PEERS:
            raise _lib.EtapShapeError(f"world must be in [1, {MAX_PEERS}]")
        self.batch, self.heads_local, self.world, self.rank, self.q_tokens = batch, heads_local, world, rank, q_tokens
        self.heads_total = heads_local * world
        self.head_offset = heads_local * rank
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.epoch = 0
        self.nbuf = nbuf
        rows = batch * q_tokens * self.heads_total
        self._sizes = [rows * D_V * 4, rows * 4]
        own, handles = [], []
        for _ in range(nbuf):
            for nb in self._sizes:
                p, h = _alloc(nb)
                own.append(p)
                handles.append(h)
        pf, hf = _alloc(MAX_PEERS * 4)
        own.append(pf)
        handles.append(hf)
        self._own = own
        my_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        mine = (_device_uuid(my_index), handles)
        if world > 1:
            import torch.distributed as dist

            alli = [None] * world
            dist.all_gather_object(alli, mine, group=group)
        else:
            alli = [mine]
        allh = [h for _, h in alli]
        # every peer pair is checked BEFORE any handle is mapped (cudaIpcOpenMemHandle with lazy
        # peer enable would otherwise fail late, or fault in the kernel)
        try:
            check_peer_access(my_index, [u for u, _ in alli])
        except PeerAccessUnavailable:
            for p in own:
                _lib.lib().etap_mla_ipc_free(C.c_void_p(p))
            raise
        self._opened = []
        ptrs = []  # ptrs[r] = rank r's pointers mapped in this process
        for r in range(world):
            if r == rank:
                ptrs.append(own)
            else:
                mapped = [_open(h) for h in allh[r]]
                self._opened += mapped
                ptrs.append(mapped)
        self._descs = []
        for s in range(nbuf):
            d = PeerGatherDesc()
            d.world, d.rank, d.heads_total, d.head_offset = world, rank, self.heads_total, self.head_offset
            for r in range(world):
                d.out[r] = ptrs[r][2 * s]
                d.lse[r] = ptrs[r][2 * s + 1]
                d.flags[r] = ptrs[r][-1]
            self._descs.append(d)
        shape_o = (batch, q_tokens, self.heads_total, D_V)
        shape_l = (batch, q_tokens, self.heads_total)
        self.outs = [torch.as_tensor(_DevPtr(own[2 * s], shape_o, "<f4"), device=self.device) for s in range(nbuf)]
        self.lses = [torch.as_tensor(_DevPtr(own[2 * s + 1], shape_l, "<f4"), device=self.device) for s in range(nbuf)]

    def decode(self, plan: MlaDecodePlan, q: torch.Tensor, kv_pool: torch.Tensor, block_table: torch.Tensor,
               seqlens: torch.Tensor, scale: float, flags: int = 0, causal: bool = True,
               stream: torch.cuda.Stream | None = None) -> tuple[torch.Tensor, torch.Tensor]:
        """This rank's heads through K2 + K3 with the all-gather fused in; returns this rank's
        full-head (out [B,T,H_total,512], lse [B,T,H_total]) for the call's epoch."""
        B, H, T = plan.batch, plan.heads, plan.q_tokens
        if (B, H, T) != (self.batch, self.heads_local, self.q_tokens):
            raise _lib.EtapShapeError("plan shape does not match the PeerGather buffers")
        # same checks as MlaDecodePlan.decode (out / lse are this object's own buffers)
        q, _, _ = plan._check_io(q, kv_pool, block_table, seqlens, None, None, (torch.bfloat16,), "kv_pool",
                                 outputs=False)
        self.epoch += 1
        s = self.epoch % self.nbuf
        check(_lib.lib().etap_mla_decode_peer(
            q.data_ptr(), kv_pool.data_ptr(), kv_pool.shape[0], block_table.data_ptr(), block_table.shape[1],
            seqlens.data_ptr(), B, T, H, float(scale), int(causal), plan.sched.data_ptr(),
            plan.split_off.data_ptr(), plan.num_sm_parts, plan.workspace.data_ptr(), C.byref(self._descs[s]),
            self.epoch & 0xFFFFFFFF, int(flags), _stream_ptr(stream)), "etap_mla_decode_peer")
        return self.outs[s], self.lses[s]

    def close(self) -> None:
        torch.cuda.synchronize(self.device)
        L = _lib.lib()
        for p in self._opened:
            L.etap_mla_ipc_close(C.c_void_p(p))
        for p in self._own:
            L.etap_mla_ipc_free(C.c_void_p(p))
        self._opened, self._own = [], []
