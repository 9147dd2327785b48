# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE — the CPU checker for the ETAP MLA decode path.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may use
this package, and only as the checker or the timed CPU baseline. The product path
(paper_2506_01969_b200) never imports it.

Two libraries:
  * ``_build/libetap_oracle.so`` — plain-C restatement (etap_oracle.c), citing the reference
    file:line it follows;
  * ``_ref/libetaplab_ref.so``   — the UNMODIFIED reference compiled from
    /root/reference/proj/src by oracle/Makefile (+ ref_shim.cpp marshalling only).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libetap_oracle.so"
REF_SO = HERE / "_ref" / "libetaplab_ref.so"
REF_SRC = Path("/root/reference/proj/src")

_oracle = None
_ref = None


def build(quiet: bool = True) -> None:
    """Build the C restatement and, when the reference sources are present, oracle/_ref."""
    out = subprocess.run(["make", "-C", str(HERE), "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _dp(a: np.ndarray) -> C.c_void_p:
    return a.ctypes.data_as(C.c_void_p)


def lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            build()
        L = C.CDLL(str(ORACLE_SO))
        vp, i64, u64, f64, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
        L.oracle_matrix_from_seed.argtypes = [i64, i64, u64, i32, vp]
        L.oracle_bf16_round.restype = f64
        L.oracle_bf16_round.argtypes = [f64]
        L.oracle_bf16_round_array.argtypes = [vp, vp, i64]
        L.oracle_bf16_bits.argtypes = [vp, vp, i64]
        L.oracle_bf16_widen.argtypes = [vp, vp, i64]
        L.oracle_round_half.restype = f64
        L.oracle_round_half.argtypes = [f64]
        L.oracle_attention_ref.argtypes = [vp, i64, vp, i64, i64, vp, i64, i64, f64, vp, vp]
        L.oracle_run_etap.restype = i32
        L.oracle_run_etap.argtypes = [vp, i64, vp, i64, i64, vp, i64, i64, f64, i64, i64, i32, vp, vp]
        L.oracle_mla_decode_bf16.restype = i32
        L.oracle_mla_decode_bf16.argtypes = [vp, vp, i64, vp, i64, vp, i64, i64, f64, i32, vp, vp]
        _oracle = L
    return _oracle


def ref_available() -> bool:
    if REF_SO.exists():
        return True
    if REF_SRC.exists():
        try:
            build()
        except RuntimeError:
            return False
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError("oracle/_ref/libetaplab_ref.so is not built (reference sources absent)")
        L = C.CDLL(str(REF_SO))
        vp, i64, u64, f64, i32 = C.c_void_p, C.c_int64, C.c_uint64, C.c_double, C.c_int
        L.ref_matrix_from_seed.argtypes = [i64, i64, u64, i32, vp]
        L.ref_round_half.restype = f64
        L.ref_round_half.argtypes = [f64]
        L.ref_make_problem_seeded.restype = i32
        L.ref_make_problem_seeded.argtypes = [u64, i64, i64, i64, i64, f64, i32, vp, vp, vp, vp]
        L.ref_run.restype = i32
        L.ref_run.argtypes = [i32, vp, i64, vp, i64, i64, vp, i64, f64, i32, i64, i64, i64, i32, vp, vp]
        L.ref_transpose_count.restype = u64
        L.ref_run_etap_state.restype = C.c_long
        L.ref_run_etap_state.argtypes = [vp, i64, vp, i64, i64, vp, i64, f64, i64, i64, vp, vp, vp]
        L.ref_save_matrix.restype = i32
        L.ref_save_matrix.argtypes = [C.c_char_p, vp, i64, i64]
        L.ref_load_matrix.restype = i32
        L.ref_load_matrix.argtypes = [C.c_char_p, vp, i64, C.POINTER(i64), C.POINTER(i64)]
        L.ref_mla_run_etap_batch.restype = f64
        L.ref_mla_run_etap_batch.argtypes = [vp, vp, i64, i64, i64, f64, i32, vp, vp]
        L.ref_mla_bench_create.restype = vp
        L.ref_mla_bench_create.argtypes = [i64, i64, i64, C.c_uint64, f64, i32]
        L.ref_mla_bench_step.restype = f64
        L.ref_mla_bench_step.argtypes = [vp, i32, vp, vp]
        L.ref_mla_bench_destroy.restype = None
        L.ref_mla_bench_destroy.argtypes = [vp]
        _ref = L
    return _ref


# ------------------------------------------------------------------ restatement wrappers
def matrix_from_seed(rows: int, cols: int, seed: int, dist: str = "normal") -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64)
    lib().oracle_matrix_from_seed(rows, cols, seed & (2**64 - 1), 1 if dist == "uniform" else 0, _dp(out))
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    lib().oracle_bf16_round_array(_dp(x), _dp(out), x.size)
    return out


def bf16_bits(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(x.shape, dtype=np.uint16)
    lib().oracle_bf16_bits(_dp(x), _dp(out), x.size)
    return out


def bf16_widen(bits: np.ndarray) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint16)
    out = np.empty(bits.shape, dtype=np.float64)
    lib().oracle_bf16_widen(_dp(bits), _dp(out), bits.size)
    return out


def attention_ref(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float) -> tuple[np.ndarray, np.ndarray]:
    """attention_ref (attention.cpp:44-77). v may be a column view of k (MLA aliasing)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    n_q, d_qk = q.shape
    n_kv, d_v = v.shape
    if v.base is k and v.strides[0] == k.strides[0] and v.__array_interface__["data"][0] == k.__array_interface__["data"][0]:
        vp, ldv = k, d_qk
    else:
        vp = np.ascontiguousarray(v, dtype=np.float64)
        ldv = d_v
    o = np.empty((n_q, d_v))
    l = np.empty(n_q)
    lib().oracle_attention_ref(_dp(q), n_q, _dp(k), n_kv, d_qk, _dp(vp), ldv, d_v, float(scale), _dp(o), _dp(l))
    return o, l


def run_etap(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float, b_r: int = 64, b_c: int = 64,
             negate_rescale: bool = False) -> tuple[np.ndarray, np.ndarray]:
    """exact64 run_etap (etap.cpp:102-148)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    n_q, d_qk = q.shape
    n_kv, d_v = v.shape
    o = np.empty((n_q, d_v))
    l = np.empty(n_q)
    rc = lib().oracle_run_etap(_dp(q), n_q, _dp(k), n_kv, d_qk, _dp(v), d_v, d_v, float(scale), b_r, b_c,
                               int(negate_rescale), _dp(o), _dp(l))
    if rc:
        raise ValueError("tile config fields must be >= 1")
    return o, l


def mla_decode_bf16(q_bits: np.ndarray, kv_pool_bits: np.ndarray, block_table: np.ndarray,
                    seqlens: np.ndarray, scale: float, nthreads: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Batched paged MLA decode oracle on bf16 bit patterns. q [B,(1,)H,576] uint16,
    kv_pool [pages,64,576] uint16 -> o [B,H,512], l [B,H] (binary64)."""
    q_bits = np.ascontiguousarray(q_bits, dtype=np.uint16)
    B = q_bits.shape[0]
    H = q_bits.shape[-2]
    kv_pool_bits = np.ascontiguousarray(kv_pool_bits, dtype=np.uint16)
    bt = np.ascontiguousarray(block_table, dtype=np.int32)
    sl = np.ascontiguousarray(seqlens, dtype=np.int32)
    o = np.empty((B, H, 512))
    l = np.empty((B, H))
    nt = nthreads or min(B, os.cpu_count() or 1)
    lib().oracle_mla_decode_bf16(_dp(q_bits), _dp(kv_pool_bits), kv_pool_bits.shape[0], _dp(bt), bt.shape[1],
                                 _dp(sl), B, H, float(scale), nt, _dp(o), _dp(l))
    return o, l


def mla_decode_bf16_tokens(q_bits: np.ndarray, kv_pool_bits: np.ndarray, block_table: np.ndarray,
                           seqlens: np.ndarray, scale: float, causal: bool = True,
                           nthreads: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Multi-token (MTP) decode oracle: q [B,T,H,576] uint16 -> o [B,T,H,512], l [B,T,H].
    No reference analog (SPEC.md:12,146,249 put multi-token decode out of scope); the causal
    rule is that token j of T sees KV rows [0, seqlen - T + j], i.e. each token is the
    single-token oracle above on a shortened context (attention_ref per row,
    attention.cpp:44-77). A token that sees no row gets O = 0, L = -inf."""
    q_bits = np.ascontiguousarray(q_bits, dtype=np.uint16)
    B, T, H = q_bits.shape[0], q_bits.shape[1], q_bits.shape[2]
    sl = np.asarray(seqlens, dtype=np.int64)
    o = np.empty((B, T, H, 512))
    l = np.empty((B, T, H))
    for j in range(T):
        slj = np.maximum(sl - (T - 1 - j), 0) if causal else sl
        o[:, j], l[:, j] = mla_decode_bf16(q_bits[:, j], kv_pool_bits, block_table, slj.astype(np.int32),
                                           scale, nthreads)
    return o, l


# ------------------------------------------------------------------ reference (oracle/_ref)
def ref_matrix_from_seed(rows: int, cols: int, seed: int, dist: str = "normal") -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64)
    ref().ref_matrix_from_seed(rows, cols, seed & (2**64 - 1), 1 if dist == "uniform" else 0, _dp(out))
    return out


def ref_make_problem(seed: int, n_q: int, n_kv: int, d_qk: int, d_v: int, scale: float = -1.0,
                     precision: int = 0):
    q = np.empty((n_q, d_qk)); k = np.empty((n_kv, d_qk)); v = np.empty((n_kv, d_v))
    sc = C.c_double(0.0)
    rc = ref().ref_make_problem_seeded(seed, n_q, n_kv, d_qk, d_v, scale, precision, _dp(q), _dp(k), _dp(v),
                                       C.byref(sc))
    if rc:
        raise ValueError("reference make_problem rejected the arguments")
    return q, k, v, sc.value


def ref_run(mode: str, q, k, v, scale: float, precision: int = 0, b_r: int = 64, b_c: int = 64,
            stages: int = 2, negate_rescale: bool = False):
    """mode: 'ref' (attention_ref), 'etap' (run_etap), 'standard' (run_standard)."""
    m = {"ref": 0, "etap": 1, "standard": 2}[mode]
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    o = np.empty((q.shape[0], v.shape[1]))
    l = np.empty(q.shape[0])
    rc = ref().ref_run(m, _dp(q), q.shape[0], _dp(k), k.shape[0], k.shape[1], _dp(v), v.shape[1], float(scale),
                       precision, b_r, b_c, stages, int(negate_rescale), _dp(o), _dp(l))
    if rc:
        raise ValueError("reference rejected the problem (std::invalid_argument)")
    return o, l


def ref_run_etap_state(q, k, v, scale: float, b_r: int = 16, b_c: int = 64):
    """The reference's run_etap (exact64) with its BlockHook recorded: returns
    (o, l, state[n_qblocks, t_c, 4, b_r]) with state fields m_old, m, rescale, l."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    n_q, n_kv = q.shape[0], k.shape[0]
    nqb, t_c = (n_q + b_r - 1) // b_r, (n_kv + b_c - 1) // b_c
    o = np.empty((n_q, v.shape[1]))
    l = np.empty(n_q)
    st = np.full((nqb, t_c, 4, b_r), np.nan)
    calls = ref().ref_run_etap_state(_dp(q), n_q, _dp(k), n_kv, k.shape[1], _dp(v), v.shape[1], float(scale),
                                     b_r, b_c, _dp(o), _dp(l), _dp(st))
    if calls != nqb * t_c:
        raise RuntimeError(f"reference hook called {calls} times, expected {nqb * t_c}")
    return o, l, st


def ref_save_matrix(path: str, m: np.ndarray) -> None:
    m = np.ascontiguousarray(m, dtype=np.float64)
    if ref().ref_save_matrix(str(path).encode(), _dp(m), m.shape[0], m.shape[1]):
        raise RuntimeError("reference save_matrix failed")


def ref_load_matrix(path: str, cap: int = 1 << 24) -> np.ndarray:
    out = np.empty(cap)
    r, c = C.c_int64(), C.c_int64()
    rc = ref().ref_load_matrix(str(path).encode(), _dp(out), cap, C.byref(r), C.byref(c))
    if rc:
        raise RuntimeError("reference load_matrix failed")
    return out[: r.value * c.value].reshape(r.value, c.value).copy()


def ref_mla_run_etap_batch(q: np.ndarray, kv: np.ndarray, scale: float, nthreads: int):
    """Time the reference's run_etap (exact64) over B MLA problems; returns (seconds, o, l)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    kv = np.ascontiguousarray(kv, dtype=np.float64)
    B, H, _ = q.shape
    ctx = kv.shape[1]
    o = np.empty((B, H, 512))
    l = np.empty((B, H))
    t = ref().ref_mla_run_etap_batch(_dp(q), _dp(kv), B, H, ctx, float(scale), int(nthreads), _dp(o), _dp(l))
    if t < 0:
        raise RuntimeError("reference run_etap failed")
    return t, o, l


class RefMlaBench:
    """The bench's full-size CPU workload on the reference (oracle/_ref): B MLA problems of
    ctx rows x H heads generated once with the reference generator (seeds seed0 + 7919 b,
    bf16-rounded, V = KV[:, :512]); step() times run_etap (exact64) over all of them."""

    def __init__(self, batch: int, heads: int, ctx: int, seed0: int, scale: float, nthreads: int):
        self.batch, self.heads, self.nthreads = batch, heads, nthreads
        self.h = ref().ref_mla_bench_create(batch, heads, ctx, seed0, float(scale), int(nthreads))
        if not self.h:
            raise RuntimeError("reference workload creation failed")

    def step(self, outputs: bool = False):
        o = np.empty((self.batch, self.heads, 512)) if outputs else None
        l = np.empty((self.batch, self.heads)) if outputs else None
        t = ref().ref_mla_bench_step(self.h, self.nthreads, _dp(o) if outputs else None, _dp(l) if outputs else None)
        if t < 0:
            raise RuntimeError("reference run_etap failed")
        return (t, o, l) if outputs else t

    def close(self) -> None:
        if self.h:
            ref().ref_mla_bench_destroy(self.h)
            self.h = None
