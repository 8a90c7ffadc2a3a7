"""CPU oracle for the Atom W4A4 hot path (arXiv 2310.19102) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package ``paper_2310_19102_b200``
never imports it and shares no code with it.

The arithmetic lives in ``atom_oracle.c`` (plain C, fp32 steps pinned, int64 partials, double
output); this module only marshals numpy arrays through ctypes.  Paper citations are in the C file.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

GROUP = 128
_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "atom_oracle.c"
_SRCS = [_SRC, _HERE / "mx_oracle.c",   # mx_oracle.c: Atom (FP) on the MX format (NEXT-2)
         _HERE / "kv_oracle.c"]           # kv_oracle.c: quantized KV cache + decode attention (NEXT-3)
_LIB = _HERE / "liboracle.so"

ORC_OK, ORC_ERR_NULL, ORC_ERR_SHAPE, ORC_ERR_ARG, ORC_ERR_OVERFLOW = 0, 1, 2, 4, 8


def build(force: bool = False) -> Path:
    """Compile the oracle with pinned IEEE semantics (no contraction, no fast-math)."""
    if force or not _LIB.exists() or any(_LIB.stat().st_mtime < s.stat().st_mtime for s in _SRCS):
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.run(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
             "-fPIC", "-shared", "-o", str(tmp), *[str(s) for s in _SRCS], "-lm"],
            check=True)
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(build()))
        P = ctypes.c_void_p
        i64, i32, f32 = ctypes.c_int64, ctypes.c_int32, ctypes.c_float
        L.oracle_quantize_rows.argtypes = [P, i64, i64, P, i64, i32, f32, f32, P, P, P]
        L.oracle_group_partials.argtypes = [P, P, P, P, i64, i64, i64, i32, P]
        L.oracle_gemm_output.argtypes = [P, P, P, i64, i64, i64, P]
        L.oracle_output_rows.argtypes = [P, P, P, P, P, P, i64, i64, i64, i32, P, i64, P]
        L.oracle_rmsnorm_rows.argtypes = [P, i64, i64, i64, P, f32, P]
        L.oracle_rmsnorm_rows.restype = ctypes.c_int
        L.oracle_silu_mul_rows.argtypes = [P, P, i64, i64, P]
        L.oracle_silu_mul_rows.restype = ctypes.c_int
        L.oracle_expf_pinned.argtypes = [ctypes.c_float]
        L.oracle_expf_pinned.restype = ctypes.c_float
        u8p = P
        L.oracle_mx_quantize_rows.argtypes = [P, i64, i64, P, i64, i32, u8p, u8p, u8p]
        L.oracle_mx_quantize_rows.restype = ctypes.c_int
        L.oracle_mx_output_rows.argtypes = [P, P, P, P, P, P, i64, i64, i64, i32, P, i64, P]
        L.oracle_mx_output_rows.restype = ctypes.c_int
        for f in (L.oracle_e2m1_value, L.oracle_e4m3_value):
            f.argtypes = [ctypes.c_int]
            f.restype = ctypes.c_double
        for f in (L.oracle_e2m1_code, L.oracle_e4m3_code):
            f.argtypes = [ctypes.c_float]
            f.restype = ctypes.c_int
        L.oracle_mx_scale_byte.argtypes = [ctypes.c_float, ctypes.c_int]
        L.oracle_mx_scale_byte.restype = ctypes.c_int
        L.oracle_kv_quantize.argtypes = [P, i64, i32, i32, P, P, P]
        L.oracle_kv_quantize.restype = ctypes.c_int
        L.oracle_decode_attention.argtypes = [P, i64, i32, i32, P, P, P, P, P, i64, P, P]
        L.oracle_decode_attention.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_max_threads.restype = ctypes.c_int
        for f in (L.oracle_quantize_rows, L.oracle_group_partials, L.oracle_gemm_output,
                  L.oracle_output_rows):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st != ORC_OK:
        raise OracleError(f"{what} failed with oracle status {st}")


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def quantize_rows(x, perm, K: int, k_outlier: int = 128, clip_int4: float = 0.9,
                  clip_int8: float = 1.0):
    """O2-O6 (reorder, group amax, scale, code, pack) for every row of ``x``.

    ``x`` is an fp16 or fp32 [rows][ldx] array (fp16 is widened exactly to fp32 first).
    Returns (q4 uint8 [rows][(K-k_o)/2], q8 int8 [rows][k_o] or None, scales fp32 [K/128][rows]).
    Activations use clip_int4 = 0.9, weights 0.85; outliers clip_int8 = 1.0.
    """
    x32 = np.ascontiguousarray(np.asarray(x).astype(np.float32))
    rows, ldx = x32.shape
    perm = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    assert perm.shape == (K,)
    q4 = np.zeros((rows, (K - k_outlier) // 2), dtype=np.uint8)
    q8 = np.zeros((rows, k_outlier), dtype=np.int8) if k_outlier else None
    sc = np.zeros((K // GROUP, rows), dtype=np.float32)
    st = lib().oracle_quantize_rows(_ptr(x32), rows, ldx, _ptr(perm), K, k_outlier,
                                    ctypes.c_float(clip_int4), ctypes.c_float(clip_int8),
                                    _ptr(q4), _ptr(q8), _ptr(sc))
    _check(st, "oracle_quantize_rows")
    return q4, q8, sc


def rmsnorm_rows(x, gamma, eps: float = 1e-6, C: int = None):
    """N1: fp16 RMSNorm of every row of x over its first C channels (default: all), pinned as
    documented in atom_oracle.c; returns fp16 [rows][C] (the fp32 result rounded to nearest-even
    by numpy's float32 -> float16 conversion)."""
    x32 = np.ascontiguousarray(np.asarray(x).astype(np.float32))
    rows, ldx = x32.shape
    C = ldx if C is None else int(C)
    g32 = np.ascontiguousarray(np.asarray(gamma).astype(np.float32))
    assert g32.shape == (C,)
    y32 = np.zeros((rows, C), dtype=np.float32)
    st = lib().oracle_rmsnorm_rows(_ptr(x32), rows, ldx, C, _ptr(g32), ctypes.c_float(eps),
                                   _ptr(y32))
    _check(st, "oracle_rmsnorm_rows")
    return y32.astype(np.float16)


def rmsnorm_quantize_rows(x, gamma, perm, K: int, k_outlier: int = 128, eps: float = 1e-6,
                          clip_int4: float = 0.9, clip_int8: float = 1.0):
    """N1 followed by O2-O6: what the fused RMSNorm + reorder + quantize kernel must produce."""
    y = rmsnorm_rows(x, gamma, eps)
    return quantize_rows(y, perm, K, k_outlier, clip_int4, clip_int8)


def expf_pinned(x: float) -> float:
    """The binary32 exponential of the SwiGLU reading G20 (oracle_expf_pinned)."""
    return float(lib().oracle_expf_pinned(ctypes.c_float(x)))


def silu_mul_rows(g, u):
    """N4: h = fp16(RN32(RN32(silu(g)) * u)) for fp16 gate / up rows, silu in double (atom_oracle.c,
    reading G20); returns fp16 [rows][C]."""
    g32 = np.ascontiguousarray(np.asarray(g).astype(np.float32))
    u32 = np.ascontiguousarray(np.asarray(u).astype(np.float32))
    assert g32.shape == u32.shape and g32.ndim == 2
    rows, ldx = g32.shape
    h32 = np.zeros((rows, ldx), dtype=np.float32)
    st = lib().oracle_silu_mul_rows(_ptr(g32), _ptr(u32), rows, ldx, _ptr(h32))
    _check(st, "oracle_silu_mul_rows")
    return h32.astype(np.float16)


def silu_mul_quantize_rows(g, u, perm, K: int, k_outlier: int = 128, clip_int4: float = 0.9,
                           clip_int8: float = 1.0):
    """N4 followed by O2-O6: what the fused SwiGLU + reorder + quantize kernel must produce."""
    return quantize_rows(silu_mul_rows(g, u), perm, K, k_outlier, clip_int4, clip_int8)


def group_partials(a_q4, a_q8, w_q4, w_q8, M: int, N: int, K: int, k_outlier: int = 128):
    """O7: exact int32 partials [G][M][N] (int64 accumulation, overflow-checked)."""
    out = np.zeros((K // GROUP, M, N), dtype=np.int32)
    st = lib().oracle_group_partials(_ptr(_c(a_q4)), _ptr(_c(a_q8)), _ptr(_c(w_q4)),
                                     _ptr(_c(w_q8)), M, N, K, k_outlier, _ptr(out))
    _check(st, "oracle_group_partials")
    return out


def gemm_output(partials, a_scales, w_scales):
    """O8: C = sum_t s_a[t][m] s_w[t][n] P_t[m][n] in float64, t ascending."""
    G, M, N = partials.shape
    c = np.zeros((M, N), dtype=np.float64)
    st = lib().oracle_gemm_output(_ptr(_c(partials)), _ptr(_c(a_scales)), _ptr(_c(w_scales)),
                                  M, N, G, _ptr(c))
    _check(st, "oracle_gemm_output")
    return c


def output_rows(a_q4, a_q8, a_scales, w_q4, w_q8, w_scales, M: int, N: int, K: int,
                k_outlier: int, rows):
    """O7+O8 for selected token rows only (sampled parity at full size, CPU baseline timing)."""
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    c = np.zeros((rows.size, N), dtype=np.float64)
    st = lib().oracle_output_rows(_ptr(_c(a_q4)), _ptr(_c(a_q8)), _ptr(_c(a_scales)),
                                  _ptr(_c(w_q4)), _ptr(_c(w_q8)), _ptr(_c(w_scales)),
                                  M, N, K, k_outlier, _ptr(rows), rows.size, _ptr(c))
    _check(st, "oracle_output_rows")
    return c


def _c(a):
    return None if a is None else np.ascontiguousarray(a)


def quantized_linear(x, perm, w, K: int, k_outlier: int = 128, clip_a: float = 0.9,
                     clip_w: float = 0.85, clip_int8: float = 1.0):
    """Whole path on the CPU: quantize W (offline, a0) and X (a1), partials (a2) and output (a3-a5
    before the fp16 rounding).  Returns a dict of every intermediate."""
    M, N = x.shape[0], w.shape[0]
    a_q4, a_q8, a_s = quantize_rows(x, perm, K, k_outlier, clip_a, clip_int8)
    w_q4, w_q8, w_s = quantize_rows(w, perm, K, k_outlier, clip_w, clip_int8)
    P = group_partials(a_q4, a_q8, w_q4, w_q8, M, N, K, k_outlier)
    C = gemm_output(P, a_s, w_s)
    return dict(a_q4=a_q4, a_q8=a_q8, a_scales=a_s, w_q4=w_q4, w_q8=w_q8, w_scales=w_s,
                partials=P, c=C)


# ---------------------------------------------------------------------------------------------
# Atom (FP) on the MX format (NEXT-2, mx_oracle.c): readings G21-G24 of DESIGN.md
# ---------------------------------------------------------------------------------------------
MX_BLOCK = 32


def e2m1_value(code: int) -> float:
    return float(lib().oracle_e2m1_value(int(code)))


def e4m3_value(code: int) -> float:
    return float(lib().oracle_e4m3_value(int(code)))


def e2m1_code(x: float) -> int:
    return int(lib().oracle_e2m1_code(ctypes.c_float(x)))


def e4m3_code(x: float) -> int:
    return int(lib().oracle_e4m3_code(ctypes.c_float(x)))


def mx_scale_byte(amax: float, emax_elem: int) -> int:
    return int(lib().oracle_mx_scale_byte(ctypes.c_float(amax), int(emax_elem)))


def mx_quantize_rows(x, perm, K: int, k_outlier: int = 128):
    """Reorder + MX quantization of every row (mx_oracle.c).  Returns (fp4 uint8
    [rows][(K-k_o)/2] packed E2M1, fp8 uint8 [rows][k_o] E4M3 or None, sexp uint8 [rows][K/32]
    UE8M0 block-scale bytes)."""
    x32 = np.ascontiguousarray(np.asarray(x).astype(np.float32))
    rows, ldx = x32.shape
    perm = np.ascontiguousarray(np.asarray(perm, dtype=np.int32))
    assert perm.shape == (K,)
    f4 = np.zeros((rows, (K - k_outlier) // 2), dtype=np.uint8)
    f8 = np.zeros((rows, k_outlier), dtype=np.uint8) if k_outlier else None
    se = np.zeros((rows, K // MX_BLOCK), dtype=np.uint8)
    st = lib().oracle_mx_quantize_rows(_ptr(x32), rows, ldx, _ptr(perm), K, k_outlier, _ptr(f4),
                                       _ptr(f8), _ptr(se))
    _check(st, "oracle_mx_quantize_rows")
    return f4, f8, se


def mx_output_rows(a, w, M: int, N: int, K: int, k_outlier: int, rows=None):
    """G24 for the selected token rows (default: all): sum_j deq(a[m][j]) deq(w[n][j]) in
    float64.  ``a`` / ``w`` are mx_quantize_rows results."""
    rows = np.arange(M) if rows is None else rows
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    c = np.zeros((rows.size, N), dtype=np.float64)
    st = lib().oracle_mx_output_rows(_ptr(_c(a[0])), _ptr(_c(a[1])), _ptr(_c(a[2])),
                                     _ptr(_c(w[0])), _ptr(_c(w[1])), _ptr(_c(w[2])), M, N, K,
                                     k_outlier, _ptr(rows), rows.size, _ptr(c))
    _check(st, "oracle_mx_output_rows")
    return c


def mx_quantized_linear(x, perm, w, K: int, k_outlier: int = 128):
    """Atom (FP) on the CPU: MX-quantize W (offline) and X, then the double output."""
    a = mx_quantize_rows(x, perm, K, k_outlier)
    wq = mx_quantize_rows(w, perm, K, k_outlier)
    return dict(a=a, w=wq, c=mx_output_rows(a, wq, x.shape[0], w.shape[0], K, k_outlier))


# ---------------------------------------------------------------------------------------------
# NEXT-3: quantized paged KV cache + decode attention (kv_oracle.c): readings G25-G28
# ---------------------------------------------------------------------------------------------
KV_PAGE = 16


def kv_quantize(x, slots, num_pages: int, codes=None, params=None):
    """G25/G26: quantize token vectors x [T][H][d] (fp16 or fp32) into a paged cache at the
    given slots (page * 16 + offset).  Returns (codes uint8 [P][H][16][d/2], params fp32
    [P][H][16][2]); pass existing arrays to append."""
    x32 = np.ascontiguousarray(np.asarray(x).astype(np.float32))
    T, H, d = x32.shape
    slots = np.ascontiguousarray(np.asarray(slots, dtype=np.int64))
    assert slots.shape == (T,) and slots.max(initial=0) < num_pages * KV_PAGE
    if codes is None:
        codes = np.zeros((num_pages, H, KV_PAGE, d // 2), dtype=np.uint8)
        params = np.zeros((num_pages, H, KV_PAGE, 2), dtype=np.float32)
    st = lib().oracle_kv_quantize(_ptr(x32), T, H, d, _ptr(slots), _ptr(codes), _ptr(params))
    _check(st, "oracle_kv_quantize")
    return codes, params


def decode_attention(q, k_cache, v_cache, block_table, seq_lens):
    """G27: out [B][H][d] (float64) of one decode step over the dequantized paged cache;
    q [B][H][d] (fp16 values), caches as returned by kv_quantize."""
    q32 = np.ascontiguousarray(np.asarray(q).astype(np.float32))
    B, H, d = q32.shape
    bt = np.ascontiguousarray(np.asarray(block_table, dtype=np.int32))
    sl = np.ascontiguousarray(np.asarray(seq_lens, dtype=np.int32))
    out = np.zeros((B, H, d), dtype=np.float64)
    st = lib().oracle_decode_attention(_ptr(q32), B, H, d, _ptr(_c(k_cache[0])),
                                       _ptr(_c(k_cache[1])), _ptr(_c(v_cache[0])),
                                       _ptr(_c(v_cache[1])), _ptr(bt), bt.shape[1], _ptr(sl),
                                       _ptr(out))
    _check(st, "oracle_decode_attention")
    return out
