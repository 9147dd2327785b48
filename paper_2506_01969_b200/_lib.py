# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the C-ABI in include/etap_mla.h (libetap_mla.so, built in-tree).

There is no fallback: if the library cannot be loaded, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "lib" / "libetap_mla.so"
# experiments only (scripts/variant.sh builds A/B variants under lib/variants/)
if os.environ.get("ETAP_LIB_VARIANT"):
    LIB_PATH = _PKG / "lib" / "variants" / f"libetap_mla_{os.environ['ETAP_LIB_VARIANT']}.so"

ETAP_OK = 0
ETAP_ERR_SHAPE = 1
ETAP_ERR_CUDA = 2
FLAG_NEGATE_RESCALE = 1
FLAG_EAGER_RESCALE = 2
FLAG_SKIP_COMBINE = 4
FLAG_EXTERNAL_SCHEDULE = 8
FLAG_DEP_METADATA = 16  # no-op since round 2: seqlens / block_table are read after the grid dependency by default
PRECISION_EXACT64 = 0  # etaplab::Precision (matrix.hpp:22); fp32 = 1 / fp16emu = 2 are rejected
FLAG_EARLY_METADATA = 32  # opt-in: read seqlens / block_table before the grid dependency (etap_mla.h)
FLAG_INDEPENDENT_INPUTS = 64  # opt-in: the preceding kernel writes none of the inputs; wait only before writes

_lib = None


class EtapError(RuntimeError):
    """A CUDA-side failure of the ETAP MLA library."""


class EtapShapeError(ValueError):
    """Shape / argument rejected (the reference raises std::invalid_argument there)."""


def _declare(lib: C.CDLL, variant: bool = False) -> None:
    vp, i32, i64, u32, f32, f64, sz = C.c_void_p, C.c_int, C.c_int64, C.c_uint, C.c_float, C.c_double, C.c_size_t
    P = C.POINTER
    sig = {
        "etap_mla_last_error": (C.c_char_p, []),
        "etap_mla_version": (C.c_char_p, []),
        "etap_mla_num_sm_parts": (i32, [i32, P(i32)]),
        "etap_mla_head_group": (i32, [i32, P(i32)]),
        "etap_mla_schedule_unit": (i32, [i32, i32, P(i32), P(i32)]),
        "etap_mla_sched_ints": (i32, [i32, i32, i32, P(sz), P(sz)]),
        "etap_mla_workspace_bytes": (i32, [i32, i32, i32, P(sz)]),
        "etap_mla_metadata": (i32, [vp, i32, i32, i32, vp, vp, vp]),
        "etap_mla_metadata_host": (i32, [vp, i32, i32, i32, vp, vp]),
        "etap_mla_decode": (i32, [vp, vp, i64, vp, i32, vp, i32, i32, i32, f32, i32, vp, vp, i32,
                                  vp, vp, vp, u32, vp]),
        "etap_mla_combine": (i32, [vp, i32, i32, i32, vp, vp, vp, vp]),
        "etap_mla_decode_peer": (i32, [vp, vp, i64, vp, i32, vp, i32, i32, i32, f32, i32, vp, vp, i32,
                                       vp, vp, u32, u32, vp]),
        "etap_mla_ipc_alloc": (i32, [sz, P(vp), vp]),
        "etap_mla_ipc_open": (i32, [vp, P(vp)]),
        "etap_mla_ipc_close": (i32, [vp]),
        "etap_mla_ipc_free": (i32, [vp]),
        "etap_mla_host_ctx_create": (i32, [i32, i32, i64, i32, P(vp)]),
        "etap_mla_host_decode": (i32, [vp, vp, vp, vp, vp, f32, u32, vp, vp]),
        "etap_mla_host_ctx_load": (i32, [vp, vp, vp]),
        "etap_mla_host_decode_step": (i32, [vp, vp, vp, vp, f32, u32, vp, vp]),
        "etap_mla_append_kv": (i32, [vp, vp, i64, vp, i32, vp, i32, i32, vp]),
        "etap_mla_head_proj": (i32, [vp, i32, i64, i64, vp, i32, i32, i32, i32, vp, i32, i64, i64, vp]),
        "etap_mla_absorb_q": (i32, [vp, vp, vp, vp, vp, i32, i32, i32, vp, vp]),
        "etap_mla_up_proj": (i32, [vp, vp, i32, i32, i32, vp, i32, vp]),
        "etap_mla_selftest_fp8": (i32, [vp, vp, vp, vp, vp, vp]),
        "etap_mla_decode_fp8": (i32, [vp, vp, f32, i64, vp, i32, vp, i32, i32, i32, f32, i32, vp, vp, i32, vp, vp, vp,
                                      u32, vp]),
        "etap_mla_host_ctx_destroy": (None, [vp]),
        "etap_mla_run_etap_f64": (i32, [vp, i64, vp, i64, i64, vp, i64, f64, i32, i64, i64, i64, u32,
                                        vp, vp]),
        "etap_mla_selftest_umma": (i32, [vp, vp, vp, vp, vp, vp]),
        "etap_mla_debug_state": (i32, [vp, i32]),
        "etap_mla_run_etap_f64_state": (i32, [vp, i64, vp, i64, i64, vp, i64, f64, i32, i64, u32, vp, vp, vp]),
        "etap_mla_debug_trace": (i32, [vp]),
        "etap_mla_debug_span": (i32, [vp]),
        "etap_mla_debug_trace_combine": (i32, [vp]),
        "etap_mla_umma_bench": (i32, [i32, i32, vp, i32]),
        "etap_mla_stream_bench": (i32, [vp, i64, i32, i32, i32, vp]),
        "etap_mla_stream_bench_mc": (i32, [vp, i64, i32, i32, i32, vp]),
        "etap_mla_stream_bench_page": (i32, [vp, i64, i32, i32, i32, i32, vp]),
        "etap_mla_debug_pdl_write": (i32, [vp, vp, i32, i32, vp]),
        "etap_mla_debug_bf16_rne": (i32, [vp, i64, vp, i32]),
    }
    for name, (res, args) in sig.items():
        if "_bench" in name and variant and not hasattr(lib, name):
            continue  # an older A/B variant build without a later debug microbenchmark
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> C.CDLL:
    """Load libetap_mla.so (building it first if it is missing and nvcc is available)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        from . import build as _build

        _build.build()
    if not LIB_PATH.exists():
        raise EtapError(f"{LIB_PATH} is missing and could not be built")
    handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    _declare(handle, variant=bool(os.environ.get("ETAP_LIB_VARIANT")))
    _lib = handle
    return _lib


def last_error() -> str:
    return lib().etap_mla_last_error().decode()


def check(rc: int, what: str) -> None:
    if rc == ETAP_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == ETAP_ERR_SHAPE:
        raise EtapShapeError(msg)
    raise EtapError(msg)
