"""The debug library (libatom_debug.so: every mbarrier / stream-K counter wait traps after a
bounded number of polls instead of hanging, csrc/ptx.cuh ATOM_WAIT_LOOP) runs the INT, MX and KV
kernels to completion and produces exactly the release library's outputs; the CPU test checks
that it exports the same ABI."""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
PKG = ROOT / "paper_2310_19102_b200"


def _debug_lib() -> Path:
    from paper_2310_19102_b200 import build as b
    return b.build(debug=True)


def test_debug_lib_exports_the_abi():
    import ctypes

    import paper_2310_19102_b200 as atom
    lib = ctypes.CDLL(str(_debug_lib()))
    for s in atom.ABI_SYMBOLS:
        assert hasattr(lib, s), s


@pytest.mark.gpu
def test_debug_lib_matches_release(tmp_path):
    dbg = _debug_lib()
    outs = {}
    for name, lib in (("release", PKG / "libatom.so"), ("debug", dbg)):
        out = tmp_path / f"{name}.npz"
        r = subprocess.run([sys.executable, str(ROOT / "tests" / "debug_lib_run.py"), str(lib),
                            str(out)], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        outs[name] = np.load(out)
    assert set(outs["release"].files) == set(outs["debug"].files)
    for k in outs["release"].files:
        np.testing.assert_array_equal(outs["debug"][k], outs["release"][k], err_msg=k)
