"""Build libatom.so in-tree with nvcc for sm_100a (the only target)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libatom.so"
SOURCES = ["atom_api.cu", "quantize.cu", "gemm.cu", "mxfp.cu", "kvcache.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    f"-I{ROOT / 'include'}", f"-I{CSRC}",
]


# Debug library: identical kernels whose wait loops trap (with a message naming the CTA and the
# barrier) after 2 s instead of hanging -- ptx.cuh ATOM_WAIT_LOOP; tests/test_debug_lib.py
LIB_DEBUG = PKG / "libatom_debug.so"
DEBUG_FLAGS = ["-DATOM_MBAR_TIMEOUT_NS=2000000000"]


def _extra() -> list:
    return os.environ.get("ATOM_NVCC_EXTRA", "").split()   # development variants (A/B runs)


def _stale(lib: Path, flags: list) -> bool:
    stamp = lib.with_name(lib.name + ".flags")
    if not lib.exists() or not stamp.exists():
        return True
    if stamp.read_text() != " ".join(flags):               # built with other flags
        return True
    mt = lib.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + \
        [ROOT / "include" / "atom.h"]
    return any(d.stat().st_mtime > mt for d in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> Path:
    lib = LIB_DEBUG if debug else LIB
    flags = FLAGS + (DEBUG_FLAGS if debug else []) + _extra()
    if not force and not _stale(lib, flags):
        return lib
    tmp = lib.with_name(f"{lib.name}.tmp{os.getpid()}")
    cmd = [NVCC, *flags, "-o", str(tmp), *[str(CSRC / s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG / ("build_debug.log" if debug else "build.log")
    log.write_text(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, lib)
    lib.with_name(lib.name + ".flags").write_text(" ".join(flags))
    return lib
