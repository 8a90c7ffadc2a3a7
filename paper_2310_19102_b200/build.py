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


STAMP = LIB.with_name("libatom.so.flags")


def _extra() -> list:
    return os.environ.get("ATOM_NVCC_EXTRA", "").split()   # development variants (A/B runs)


def _stale() -> bool:
    if not LIB.exists() or not STAMP.exists():
        return True
    if STAMP.read_text() != " ".join(FLAGS + _extra()):     # built with other flags
        return True
    mt = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + \
        [ROOT / "include" / "atom.h"]
    return any(d.stat().st_mtime > mt for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    tmp = LIB.with_name(f"libatom.so.tmp{os.getpid()}")
    extra = _extra()
    cmd = [NVCC, *FLAGS, *extra, "-o", str(tmp), *[str(CSRC / s) for s in SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG / "build.log"
    log.write_text(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, LIB)
    STAMP.write_text(" ".join(FLAGS + extra))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
