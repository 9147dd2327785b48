# SPDX-License-Identifier: Apache-2.0
"""Build the sm_100a CUDA library (libetap_mla.so) in-tree with nvcc.

The library is a plain C-ABI shared object (include/etap_mla.h); Python reaches it with
ctypes, C++ callers link it directly. Built for sm_100a only:
``-gencode arch=compute_100a,code=sm_100a`` (tcgen05 is rejected in a generic compute_100
pass).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libetap_mla.so"
BENCH = LIBDIR / "etap_bench"
MODEL = LIBDIR / "etap_model"

SOURCES = [CSRC / "etap_mla.cu", CSRC / "etap_peer.cu", CSRC / "etap_proj.cu", CSRC / "etap_fp8.cu",
           CSRC / "etap_mla_host.cpp"]
DEPS = SOURCES + [CSRC / "etap_bench.cpp", CSRC / "sm100_ptx.cuh", CSRC / "etap_mla_kernels.cuh", CSRC / "etap_mla_pair.cuh", CSRC / "etap_fp8.cuh", ROOT / "include" / "etap_mla.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    cand = os.environ.get("NVCC") or shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found")
    return cand


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and up_to_date():
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, "-shared", *map(str, SOURCES), "-o", str(tmp),
           "-Xlinker", "--export-dynamic"]
    # C-ABI symbols are exported through an explicit visibility attribute-free version script
    vs = LIBDIR / "exports.map"
    vs.write_text("{ global: etap_mla_*; local: *; };\n")
    cmd += ["-Xlinker", f"--version-script={vs}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = LIBDIR / "build.log"
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, LIB)
    # native benchmark driver (C-ABI, no Python in the launch path)
    res = subprocess.run([nvcc(), "-O3", "-std=c++17", str(CSRC / "etap_bench.cpp"), "-o", str(BENCH),
                          "-L", str(LIBDIR), "-letap_mla", "-Xlinker", "-rpath=$ORIGIN"],
                         capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("etap_bench build failed")
    build_model()
    return LIB


def build_variant(name: str, defines: list[str]) -> Path:
    """An A/B variant of the library (lib/variants/libetap_mla_<name>.so, loaded with
    ETAP_LIB_VARIANT=<name>): same sources, extra -D defines. Experiments only."""
    out = LIBDIR / "variants" / f"libetap_mla_{name}.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    vs = LIBDIR / "exports.map"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-shared", *map(str, SOURCES), "-o", str(out),
           "-Xlinker", "--export-dynamic", "-Xlinker", f"--version-script={vs}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("variant build failed")
    return out


def build_model() -> Path:
    """Host-only tool: the reference's `etaplab model` report for tcgen05 (no CUDA)."""
    src = CSRC / "etap_model.cpp"
    hdr = ROOT / "include" / "etaplab_b200_umma.hpp"
    if MODEL.exists() and MODEL.stat().st_mtime >= max(src.stat().st_mtime, hdr.stat().st_mtime):
        return MODEL
    LIBDIR.mkdir(exist_ok=True)
    cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
    res = subprocess.run([cxx, "-O2", "-std=c++17", "-Wall", str(src), "-o", str(MODEL)], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("etap_model build failed")
    return MODEL


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
