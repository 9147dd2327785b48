# SPDX-License-Identifier: Apache-2.0
"""ATNM golden-matrix files, the reference's exchange format (include/etaplab/matrix_io.hpp,
src/matrix_io.cpp:13-77): 4 magic bytes "ATNM", u32 little-endian rows and cols, then
rows*cols binary32 little-endian values, row-major. The GPU path's O / LSE are binary32
already, so a dump is bit-exact. Errors mirror the reference: RuntimeError on bad magic,
truncated header or payload, and zero dimensions.
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

MAGIC = b"ATNM"


def save(path: str | Path, m: np.ndarray) -> None:
    """save_matrix (matrix_io.cpp:34-46): values narrowed to binary32."""
    a = np.asarray(m)
    if a.ndim == 1:
        a = a[None, :]
    if a.ndim != 2 or a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError("matrix must be 2-D with dimensions >= 1")
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<II", a.shape[0], a.shape[1]))
        f.write(np.ascontiguousarray(a, dtype="<f4").tobytes())


def load(path: str | Path) -> np.ndarray:
    """load_matrix (matrix_io.cpp:54-77), returned as float32 [rows, cols]."""
    data = Path(path).read_bytes()
    if len(data) < 4 or data[:4] != MAGIC:
        raise RuntimeError("not a matrix file: bad magic")
    if len(data) < 12:
        raise RuntimeError("matrix file truncated in header")
    rows, cols = struct.unpack("<II", data[4:12])
    if rows < 1 or cols < 1:
        raise RuntimeError("matrix file has zero dimension")
    n = rows * cols
    if len(data) < 12 + 4 * n:
        raise RuntimeError("matrix file truncated in payload")
    return np.frombuffer(data, dtype="<f4", count=n, offset=12).reshape(rows, cols).astype(np.float32)
