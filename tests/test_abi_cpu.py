"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, exports every symbol that
include/atom.h declares, and its host-side validation rejects bad arguments before touching a
device (no compute call is made here)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    from paper_2310_19102_b200 import build
    build.build()
    import paper_2310_19102_b200 as atom
    return atom.load()


def declared_symbols():
    h = (ROOT / "include" / "atom.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:atom_status_t|size_t|const char\*|int)\s+(atom_\w+)\(",
                                 h, re.M)))


def test_header_declares_the_three_calls():
    syms = declared_symbols()
    for s in ("atom_reorder_quantize", "atom_quantize_weights", "atom_w4a4_gemm",
              "atom_w4a4_gemm_f8"):
        assert s in syms


def test_every_declared_symbol_exported(lib):
    import paper_2310_19102_b200 as atom
    syms = declared_symbols()
    assert set(syms) == set(atom.ABI_SYMBOLS)
    for s in syms:
        assert hasattr(lib, s), s


def test_sm100a_only_cubin():
    import subprocess
    so = ROOT / "paper_2310_19102_b200" / "libatom.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out
    sass = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass       # tcgen05.mma kind::i8 (INT8 outlier group)
    assert "UTCQMMA" in sass       # tcgen05.mma kind::f8f6f4 (INT4 groups as E4M3)
    assert "UTMALDG" in sass       # TMA tile loads
    assert "LDTM" in sass          # tcgen05.ld


def test_version_and_status_strings(lib):
    assert lib.atom_abi_version() == 6
    for s in range(8):
        assert lib.atom_status_string(s).startswith(b"ATOM_")


def test_host_validation_without_device(lib):
    f = ctypes.c_float
    # shape / argument errors are detected before any device query
    z5 = (None,) * 5
    assert lib.atom_reorder_quantize(None, -1, 256, None, 256, 128, f(0.9), f(1.0), *z5,
                                     None) == 2
    assert lib.atom_reorder_quantize(None, 4, 256, None, 200, 128, f(0.9), f(1.0), *z5,
                                     None) == 2
    assert lib.atom_reorder_quantize(None, 4, 256, None, 256, 64, f(0.9), f(1.0), *z5,
                                     None) == 4
    assert lib.atom_reorder_quantize(None, 4, 256, None, 256, 128, f(1.5), f(1.0), *z5,
                                     None) == 4
    assert lib.atom_reorder_quantize(None, 4, 256, None, 256, 128, f(0.9), f(1.0), *z5,
                                     None) == 1
    assert lib.atom_quantize_weights(None, 4, 250, None, 256, 128, f(0.85), f(1.0), None, None,
                                     None, None, None) == 2
    z6 = (None,) * 6
    for gemm, zp, fl in ((lib.atom_w4a4_gemm, z6, ()), (lib.atom_w4a4_gemm_f8, z6[:5], (0,))):
        assert gemm(*zp, 4, 100, 256, 128, None, 128, 0, None, *fl, None, 0, None) == 2
        assert gemm(*zp, 4, 128, 256, 128, None, 128, 3, None, *fl, None, 0, None) == 4
        assert gemm(*zp, 4, 128, 256, 128, None, 128, 0, None, *fl, None, 0, None) == 1
        assert gemm(*zp, 4, 128, 256, 128, None, 100, 0, None, *fl, None, 0, None) == 2   # ldc < N
        # M == 0 is a no-op that succeeds without a device
        assert gemm(*zp, 0, 128, 256, 128, None, 128, 0, None, *fl, None, 0, None) == 0
    assert lib.atom_w4a4_gemm_workspace_size(1024, 28672, 8192, 128) == 0
    assert lib.atom_w4a4_gemm_f8_workspace_size(1024, 28672, 8192, 128) == 0
    assert lib.atom_last_launch_count() == 0
    # fused RMSNorm variant: eps < 0 is an argument error, M == 0 a no-op
    assert lib.atom_rmsnorm_reorder_quantize(None, 4, 256, None, f(-1.0), None, 256, 128, f(0.9),
                                             f(1.0), *z6) == 4
    assert lib.atom_rmsnorm_reorder_quantize(None, 0, 256, None, f(1e-6), None, 256, 128, f(0.9),
                                             f(1.0), *z6) == 0


def test_silu_mul_quantize_host_validation(lib):
    f = ctypes.c_float
    # missing up projection: a NULL error; M == 0: a no-op; both decided on the host
    z6 = (None,) * 6
    assert lib.atom_silu_mul_reorder_quantize(None, None, 4, 256, None, 256, 128, f(0.9), f(1.0),
                                              *z6) == 1
    assert lib.atom_silu_mul_reorder_quantize(None, None, 0, 256, None, 256, 128, f(0.9), f(1.0),
                                              *z6) == 0
    assert lib.atom_last_launch_count() == 0


def test_mx_and_kv_host_validation(lib):
    """NEXT-2 / NEXT-3 entry points: shape, argument and NULL errors are decided on the host
    before any device query; empty batches are no-ops."""
    # atom_mx_reorder_quantize(x, rows, ldx, perm, K, k_o, fp4, fp8, sf, ldsf, stream)
    q = lib.atom_mx_reorder_quantize
    assert q(None, 4, 256, None, 200, 128, None, None, None, 16, None) == 2      # K % 128
    assert q(None, 4, 256, None, 256, 64, None, None, None, 16, None) == 4       # k_outlier
    assert q(None, 4, 256, None, 256, 128, None, None, None, 4, None) == 2       # ldsf < K/32
    assert q(None, 4, 256, None, 256, 128, None, None, None, 16, None) == 1      # NULLs
    assert q(None, 0, 256, None, 256, 128, None, None, None, 16, None) == 0
    # atom_mx_gemm(a4, a8, asf, lda_sf, w4, w8, wsf, ldw_sf, M, N, K, k_o, c, ldc, ws, wsb, st)
    g = lib.atom_mx_gemm
    assert g(None, None, None, 16, None, None, None, 16, 4, 100, 256, 128, None, 128, None, 0,
             None) == 2                                                          # N % 128
    assert g(None, None, None, 16, None, None, None, 16, 4, 128, 256, 128, None, 100, None, 0,
             None) == 2                                                          # ldc < N
    assert g(None, None, None, 16, None, None, None, 16, 4, 128, 256, 128, None, 128, None, 0,
             None) == 1
    assert g(None, None, None, 16, None, None, None, 16, 0, 128, 256, 128, None, 128, None, 0,
             None) == 0
    assert lib.atom_mx_gemm_workspace_size(8, 4096, 11008, 128) == 0            # no device here
    # atom_kv_quantize(x, T, ldx, H, d, slots, codes, params, stream)
    k = lib.atom_kv_quantize
    assert k(None, 4, 256, 2, 64, None, None, None, None) == 2                  # head_dim 128 only
    assert k(None, 4, 200, 2, 128, None, None, None, None) == 2                 # ldx < 128 H
    assert k(None, 4, 256, 2, 128, None, None, None, None) == 1
    assert k(None, 0, 256, 2, 128, None, None, None, None) == 0
    # atom_decode_attention(q, B, H, d, kc, kp, vc, vp, bt, max_pages, lens, max_len, out, ws,
    # wsb, stream)
    a = lib.atom_decode_attention
    assert a(None, 2, 4, 128, None, None, None, None, None, 2, None, 40, None, None, 0,
             None) == 2                                                          # 40 > 16 * 2
    assert a(None, 2, 4, 128, None, None, None, None, None, 4, None, 40, None, None, 0,
             None) == 1
    assert a(None, 0, 4, 128, None, None, None, None, None, 4, None, 40, None, None, 0,
             None) == 0
    assert lib.atom_last_launch_count() == 0


def test_bench_gpus_2_spawns_two_ranks_dry_run():
    """`python bench.py --gpus 2` (the driver's launch form) starts two ranks itself (torchrun on
    127.0.0.1); --dry-run exercises that rank plumbing with gloo on CPU: both ranks report their
    N-shard and K-shard ranges, which tile the full problem."""
    import json
    import subprocess
    import sys
    for shard, total in (("n", 28672), ("k", 8192)):
        out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run",
                              "--shard", shard], capture_output=True, text=True, timeout=240,
                             cwd=str(ROOT))
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
        d = json.loads(line)
        assert d["n_gpus"] == 2 and [r[0] for r in d["ranks"]] == [0, 1]
        assert d["ranks"][0][1] == 0 and d["ranks"][0][2] == d["ranks"][1][1]
        assert d["ranks"][1][2] == total


def test_product_package_does_not_import_oracle():
    pkg = ROOT / "paper_2310_19102_b200"
    for f in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")) + \
            list(pkg.rglob("*.h")):
        txt = f.read_text()
        assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f
