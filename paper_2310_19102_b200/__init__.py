"""B200-native Atom W4A4 hot path (arXiv 2310.19102) -- thin Python binding over libatom.so.

Argument marshalling only: every step of the path runs in the CUDA kernels behind the C ABI
(include/atom.h).  PyTorch supplies device memory and streams.  There is no CPU fallback: if the
in-tree ``libatom.so`` is missing or a call fails, an exception is raised.

Names follow the ABI and the paper:
  reorder_quantize(x, perm)        a1  online activation reorder + dynamic quantize
  quantize_weights(w, perm)        a0  offline weight reorder + quantize
  w4a4_gemm(a, w)                  a2-a5 fused group GEMM with INT8 outliers
  mx_quantize(x, perm) / mx_gemm(a, w)   NEXT-2 Atom (FP) on the MX format
  kv_quantize / decode_attention         NEXT-3 INT4 KV cache + decode attention
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libatom.so"
GROUP = 128

ATOM_OK = 0
STATUS_NAMES = {0: "ATOM_OK", 1: "ATOM_ERR_NULL", 2: "ATOM_ERR_SHAPE", 3: "ATOM_ERR_ALIGN",
                4: "ATOM_ERR_ARG", 5: "ATOM_ERR_WORKSPACE", 6: "ATOM_ERR_UNSUPPORTED",
                7: "ATOM_ERR_CUDA"}
ATOM_F16, ATOM_F32 = 0, 1

# every symbol include/atom.h declares
ABI_SYMBOLS = ("atom_reorder_quantize", "atom_rmsnorm_reorder_quantize",
               "atom_silu_mul_reorder_quantize", "atom_quantize_weights",
               "atom_w4a4_gemm", "atom_w4a4_gemm_f8",
               "atom_w4a4_gemm_workspace_size", "atom_w4a4_gemm_f8_workspace_size",
               "atom_w4a4_gemm_counter_bytes",
               "atom_mx_reorder_quantize", "atom_mx_gemm", "atom_mx_gemm_workspace_size",
               "atom_kv_quantize", "atom_decode_attention", "atom_decode_attention_workspace_size",
               "atom_validate_perm", "atom_status_string",
               "atom_abi_version", "atom_last_launch_count")


class AtomError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {STATUS_NAMES.get(status, status)} "
                         f"({_lib().atom_status_string(status).decode()})")


_L = None


def _lib():
    """Load the in-tree libatom.so (fail loudly if it was never built)."""
    global _L
    if _L is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                              f"g.build()'` (no CPU fallback exists)")
        L = ctypes.CDLL(str(LIB_PATH))
        P, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
        q_args = [P, i64, i64, P, i64, i32, f32, f32, P, P, P, P]
        L.atom_reorder_quantize.argtypes = q_args[:10] + [P, P] + q_args[10:]
        L.atom_quantize_weights.argtypes = q_args[:11] + [P] + q_args[11:]
        L.atom_rmsnorm_reorder_quantize.argtypes = [P, i64, i64, P, f32] + q_args[3:10] + \
            [P, P] + q_args[10:]
        L.atom_rmsnorm_reorder_quantize.restype = ctypes.c_int
        L.atom_silu_mul_reorder_quantize.argtypes = [P, P, i64, i64] + q_args[3:10] + \
            [P, P] + q_args[10:]
        L.atom_silu_mul_reorder_quantize.restype = ctypes.c_int
        g_tail = [i64, i64, i64, i32, P, i64, ctypes.c_int, P, P, ctypes.c_size_t, P]
        L.atom_w4a4_gemm.argtypes = [P] * 6 + g_tail
        L.atom_w4a4_gemm_f8.argtypes = [P] * 5 + g_tail[:8] + [i32] + g_tail[8:]
        L.atom_w4a4_gemm_f8.restype = ctypes.c_int
        for f in (L.atom_w4a4_gemm_workspace_size, L.atom_w4a4_gemm_f8_workspace_size):
            f.argtypes = [i64, i64, i64, i32]
            f.restype = ctypes.c_size_t
        L.atom_w4a4_gemm_counter_bytes.restype = ctypes.c_size_t
        L.atom_mx_reorder_quantize.argtypes = [P, i64, i64, P, i64, i32, P, P, P, i64, P]
        L.atom_mx_reorder_quantize.restype = ctypes.c_int
        L.atom_mx_gemm.argtypes = [P, P, P, i64, P, P, P, i64, i64, i64, i64, i32, P, i64, P,
                                   ctypes.c_size_t, P]
        L.atom_mx_gemm.restype = ctypes.c_int
        L.atom_mx_gemm_workspace_size.argtypes = [i64, i64, i64, i32]
        L.atom_mx_gemm_workspace_size.restype = ctypes.c_size_t
        L.atom_kv_quantize.argtypes = [P, i64, i64, i32, i32, P, P, P, P]
        L.atom_kv_quantize.restype = ctypes.c_int
        L.atom_decode_attention.argtypes = [P, i64, i32, i32, P, P, P, P, P, i64, P, i32, P, P,
                                            ctypes.c_size_t, P]
        L.atom_decode_attention.restype = ctypes.c_int
        L.atom_decode_attention_workspace_size.argtypes = [i64, i32, i32]
        L.atom_decode_attention_workspace_size.restype = ctypes.c_size_t
        L.atom_validate_perm.argtypes = [P, i64, i64, P, P, P]
        L.atom_status_string.argtypes = [ctypes.c_int]
        L.atom_status_string.restype = ctypes.c_char_p
        L.atom_abi_version.restype = ctypes.c_int
        L.atom_last_launch_count.restype = ctypes.c_int
        for f in (L.atom_reorder_quantize, L.atom_quantize_weights, L.atom_w4a4_gemm,
                  L.atom_validate_perm):
            f.restype = ctypes.c_int
        _L = L
    return _L


def load():
    """Return the ctypes handle of libatom.so (raises if it is missing)."""
    return _lib()


def abi_version() -> int:
    return int(_lib().atom_abi_version())


def last_launch_count() -> int:
    return int(_lib().atom_last_launch_count())


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _check(st: int, what: str):
    if st != ATOM_OK:
        raise AtomError(st, what)


@dataclass
class Quantized:
    """Quantized operand: q4 uint8 [rows][(K-k_o)/2] packed INT4, q8 int8 [rows][k_o] (or None),
    scales fp32 [K/128][rows] (group-major), with the reordered K and k_outlier.  Activations
    may also carry the GEMM operand form (include/atom.h): f8 uint8 [rows][K] (E4M3 codes) and
    ab fp32 [K/128][Mp][2] (per-row dequant constants, Mp = rows rounded up to 128), which
    atom_w4a4_gemm_f8 reads."""
    q4: object
    q8: object
    scales: object
    K: int
    k_outlier: int
    f8: object = None
    ab: object = None
    sp: object = None          # weights: scales in the GEMM channel order (include/atom.h "w_sp")

    @property
    def rows(self) -> int:
        return int(self.scales.shape[1])


def ab_rows(rows: int) -> int:
    """Rows of the a_ab operand per group: rows rounded up to the GEMM's 128-token tile."""
    return (rows + 127) // 128 * 128


def _check_quantized(out, rows, K, k_outlier, dev, operand):
    """Shapes / dtypes of a caller-supplied Quantized (the C ABI sees bare pointers)."""
    import torch
    G = K // GROUP

    def want(t, shape, dtype, name):
        if t is None:
            return
        if tuple(t.shape) != shape or t.dtype != dtype or not t.is_contiguous() \
                or t.device != dev:
            raise ValueError(f"out.{name}: expected contiguous {dtype} {shape} on {dev}")
    if out.K != K or out.k_outlier != k_outlier:
        raise ValueError("out was allocated for another K / k_outlier")
    want(out.q4, (rows, (K - k_outlier) // 2), torch.uint8, "q4")
    want(out.q8, (rows, k_outlier), torch.int8, "q8")
    want(out.scales, (G, rows), torch.float32, "scales")
    want(out.sp, (G, rows), torch.float32, "sp")
    if operand:
        want(out.f8, (rows, K), torch.uint8, "f8")
        want(out.ab, (G, ab_rows(rows), 2), torch.float32, "ab")
    if out.scales is None:
        raise ValueError("out.scales is required")


def _quantize(fn_name, x, perm, K, k_outlier, clip_int4, clip_int8, out, stream, operand=False,
              packed=True, norm=None, up=None):
    import torch
    if x.dtype != torch.float16 or x.dim() != 2 or not x.is_cuda:
        raise TypeError("expected a 2-D CUDA fp16 tensor")
    if x.stride(1) != 1:
        raise ValueError("rows must be contiguous")
    if perm.dtype != torch.int32 or not perm.is_cuda or not perm.is_contiguous():
        raise TypeError("perm must be a contiguous CUDA int32 tensor")
    rows, ld = x.shape[0], x.stride(0)
    K = int(perm.numel()) if K is None else int(K)
    if K > perm.numel():
        raise ValueError(f"K = {K} exceeds perm.numel() = {perm.numel()}")
    prepared = fn_name == "atom_quantize_weights" and rows % GROUP == 0
    if out is None:
        dev = x.device
        q4 = torch.empty((rows, (K - k_outlier) // 2), dtype=torch.uint8, device=dev) \
            if K > k_outlier and packed else None
        q8 = torch.empty((rows, k_outlier), dtype=torch.int8, device=dev) \
            if k_outlier and packed else None
        sc = torch.empty((K // GROUP, rows), dtype=torch.float32, device=dev)
        f8 = torch.empty((rows, K), dtype=torch.uint8, device=dev) if operand else None
        ab = torch.empty((K // GROUP, ab_rows(rows), 2), dtype=torch.float32, device=dev) \
            if operand else None
        sp = torch.empty((K // GROUP, rows), dtype=torch.float32, device=dev) if prepared else None
        out = Quantized(q4, q8, sc, K, k_outlier, f8, ab, sp)
    else:
        _check_quantized(out, rows, K, k_outlier, x.device, operand)
    codes = (_ptr(out.q4), _ptr(out.q8))
    if fn_name != "atom_quantize_weights":
        codes = codes + (_ptr(out.f8), _ptr(out.ab))
    tail = (_ptr(out.sp),) if fn_name == "atom_quantize_weights" else ()
    head = (_ptr(x), rows, ld)
    if up is not None:                        # the up projection of the fused SwiGLU
        if up.dtype != torch.float16 or not up.is_cuda or up.shape != x.shape \
                or up.stride() != x.stride():
            raise TypeError("up must be a CUDA fp16 tensor with the gate's shape and strides")
        head = (_ptr(x), _ptr(up), rows, ld)
    if norm is not None:                      # (gamma, eps) of the fused RMSNorm
        gamma, eps = norm
        if gamma.dtype != torch.float16 or not gamma.is_cuda or gamma.numel() != ld \
                or not gamma.is_contiguous():
            raise TypeError("gamma must be a contiguous CUDA fp16 tensor of the row length")
        if x.stride(0) != x.shape[1]:
            raise ValueError("the fused RMSNorm needs dense rows (ldx == hidden size)")
        head = head + (_ptr(gamma), ctypes.c_float(eps))
    st = getattr(_lib(), fn_name)(*head, _ptr(perm), K, k_outlier,
                                  ctypes.c_float(clip_int4), ctypes.c_float(clip_int8),
                                  *codes, _ptr(out.scales), *tail, _stream(stream))
    _check(st, fn_name)
    return out


def reorder_quantize(x, perm, K: Optional[int] = None, k_outlier: int = 128,
                     clip_int4: float = 0.9, clip_int8: float = 1.0, out: Quantized = None,
                     stream=None, packed: bool = True, operand: bool = True) -> Quantized:
    """a1: reorder + dynamically quantize activations x fp16 [M][ldx] (clip 0.9).

    Writes the canonical packed q4/q8 unless ``packed=False`` and the GEMM operand form
    (f8, ab) unless ``operand=False``."""
    return _quantize("atom_reorder_quantize", x, perm, K, k_outlier, clip_int4, clip_int8, out,
                     stream, operand=operand, packed=packed)


def rmsnorm_reorder_quantize(x, gamma, perm, eps: float = 1e-6, K: Optional[int] = None,
                             k_outlier: int = 128, clip_int4: float = 0.9, clip_int8: float = 1.0,
                             out: Quantized = None, stream=None, packed: bool = True,
                             operand: bool = True) -> Quantized:
    """NEXT-1: fp16 RMSNorm of x [M][hidden] (weight gamma fp16 [hidden]) fused with the reorder
    + dynamic quantize of a1 -- the paper's fusion into the prior operator."""
    return _quantize("atom_rmsnorm_reorder_quantize", x, perm, K, k_outlier, clip_int4,
                     clip_int8, out, stream, operand=operand, packed=packed, norm=(gamma, eps))


def silu_mul_reorder_quantize(gate, up, perm, K: Optional[int] = None, k_outlier: int = 128,
                              clip_int4: float = 0.9, clip_int8: float = 1.0,
                              out: Quantized = None, stream=None, packed: bool = True,
                              operand: bool = True) -> Quantized:
    """NEXT-4 piece: SwiGLU h = silu(gate) * up of a Llama MLP (fp16 [M][I] gate / up projection
    outputs) fused with the reorder + dynamic quantize of the down projection's input."""
    return _quantize("atom_silu_mul_reorder_quantize", gate, perm, K, k_outlier, clip_int4,
                     clip_int8, out, stream, operand=operand, packed=packed, up=up)


def quantize_weights(w, perm, K: Optional[int] = None, k_outlier: int = 128,
                     clip_int4: float = 0.85, clip_int8: float = 1.0, out: Quantized = None,
                     stream=None) -> Quantized:
    """a0: offline reorder + quantize of W fp16 [N][K] (nn.Linear layout, clip 0.85)."""
    return _quantize("atom_quantize_weights", w, perm, K, k_outlier, clip_int4, clip_int8, out,
                     stream)


def workspace_size(M: int, N: int, K: int, k_outlier: int = 128) -> int:
    """Workspace bytes of atom_w4a4_gemm (canonical inputs); also serves atom_w4a4_gemm_f8."""
    return int(_lib().atom_w4a4_gemm_workspace_size(M, N, K, k_outlier))


def counter_bytes() -> int:
    """Leading bytes of every GEMM workspace that must be zero between calls (include/atom.h)."""
    return int(_lib().atom_w4a4_gemm_counter_bytes())


_WORKSPACES = {}


def gemm_workspace(M: int, N: int, K: int, k_outlier: int = 128, stream=None):
    """A zero-filled GEMM workspace for this shape, cached per (device, stream): the GEMM leaves
    its counter region zero after every completed call (include/atom.h), so it is cleared only
    when first allocated."""
    import torch
    n = workspace_size(M, N, K, k_outlier)
    if n == 0:
        return None
    s = torch.cuda.current_stream() if stream is None else stream
    key = (s.device.index, s.cuda_stream)
    ws = _WORKSPACES.get(key)
    if ws is None or ws.numel() < n:
        with torch.cuda.stream(s):
            ws = torch.zeros(n, dtype=torch.uint8, device=s.device)
        _WORKSPACES[key] = ws
    return ws


GEMM_SPLIT_FREE = 1


def w4a4_gemm(a: Quantized, w: Quantized, out=None, out_dtype=None, debug_partials=None,
              workspace=None, stream=None, canonical: bool = False, split_free: bool = False):
    """a2-a5: C[m][n] = sum_t s_a[t][m] s_w[t][n] P_t[m][n] (fp32 accumulate), fp16 or fp32 out.

    Reads the activation operand form (a.f8, a.ab) through atom_w4a4_gemm_f8 when present,
    else (or with ``canonical=True``) the packed a.q4 / a.q8 through atom_w4a4_gemm.
    ``out`` may be a wider [M][ldc] view (ldc >= N) to write an N-shard in place.
    ``debug_partials``: optional int32 [K/128][M][N] CUDA tensor receiving every exact partial.
    ``split_free``: no K-split of output tiles (include/atom.h ATOM_GEMM_SPLIT_FREE): column
    shards then reproduce the unsharded output bit for bit (operand-form path only).
    """
    import torch
    if a.K != w.K or a.k_outlier != w.k_outlier:
        raise ValueError("activation and weight quantization disagree on K / k_outlier")
    M, N = a.rows, w.rows
    dev = a.scales.device
    if out is None:
        dt = torch.float16 if out_dtype is None else out_dtype
        out = torch.empty((M, N), dtype=dt, device=dev)
    if out.dtype not in (torch.float16, torch.float32) or out.dim() != 2 or out.stride(1) != 1:
        raise TypeError("out must be a 2-D fp16/fp32 tensor with contiguous rows")
    if out.shape[0] < M or out.shape[1] < N or out.device != dev:
        raise ValueError(f"out must be at least [{M}][{N}] on {dev}, got {tuple(out.shape)} "
                         f"on {out.device}")
    if debug_partials is not None and (
            tuple(debug_partials.shape) != (a.K // GROUP, M, N) or
            debug_partials.dtype != torch.int32 or not debug_partials.is_contiguous() or
            debug_partials.device != dev):
        raise ValueError("debug_partials must be a contiguous int32 [K/128][M][N] tensor")
    c_dtype = ATOM_F16 if out.dtype == torch.float16 else ATOM_F32
    use_f8 = a.f8 is not None and w.sp is not None and not canonical
    if split_free and not use_f8:
        raise ValueError("split_free needs the operand forms (a.f8 / a.ab and w.sp)")
    if not use_f8 and (a.q4 is None) != (a.K == a.k_outlier):
        raise ValueError("activations lack the packed codes (quantize with packed=True)")
    if workspace is None:
        workspace = gemm_workspace(M, N, a.K, a.k_outlier, stream)
    wsz = 0 if workspace is None else workspace.numel()
    if use_f8:
        st = _lib().atom_w4a4_gemm_f8(_ptr(a.f8), _ptr(a.ab), _ptr(w.q4),
                                      _ptr(w.q8), _ptr(w.sp), M, N, a.K, a.k_outlier,
                                      _ptr(out), out.stride(0), c_dtype, _ptr(debug_partials),
                                      GEMM_SPLIT_FREE if split_free else 0,
                                      _ptr(workspace), wsz, _stream(stream))
        _check(st, "atom_w4a4_gemm_f8")
    else:
        st = _lib().atom_w4a4_gemm(_ptr(a.q4), _ptr(a.q8), _ptr(a.scales), _ptr(w.q4),
                                   _ptr(w.q8), _ptr(w.scales), M, N, a.K, a.k_outlier,
                                   _ptr(out), out.stride(0), c_dtype, _ptr(debug_partials),
                                   _ptr(workspace), wsz, _stream(stream))
        _check(st, "atom_w4a4_gemm")
    return out


def validate_perm(perm, ldx: Optional[int] = None, stream=None) -> bool:
    """Device check that perm is a bijection of [0,K) (ldx == K) or an injection into [0,ldx)."""
    import torch
    K = perm.numel()
    ldx = K if ldx is None else ldx
    scratch = torch.empty(ldx, dtype=torch.int32, device=perm.device)
    ok = torch.empty(1, dtype=torch.int32, device=perm.device)
    _check(_lib().atom_validate_perm(_ptr(perm), K, ldx, _ptr(scratch), _ptr(ok),
                                     _stream(stream)), "atom_validate_perm")
    return bool(ok.item())


class QuantizedLinear:
    """Convenience wrapper: one Atom W4A4 linear layer (weights quantized once, offline)."""

    def __init__(self, weight_f16, perm, k_outlier: int = 128, clip_w: float = 0.85,
                 clip_a: float = 0.9, clip_int8: float = 1.0):
        self.perm = perm
        self.k_outlier = k_outlier
        self.clip_a, self.clip_int8 = clip_a, clip_int8
        self.w = quantize_weights(weight_f16, perm, k_outlier=k_outlier, clip_int4=clip_w,
                                  clip_int8=clip_int8)

    def __call__(self, x, out=None, stream=None):
        a = reorder_quantize(x, self.perm, k_outlier=self.k_outlier, clip_int4=self.clip_a,
                             clip_int8=self.clip_int8, stream=stream)
        return w4a4_gemm(a, self.w, out=out, stream=stream)


# ---------------------------------------------------------------------------------------------
# NEXT-2: Atom (FP) on the MX format (include/atom.h "Atom (FP)")
# ---------------------------------------------------------------------------------------------
MX_BLOCK = 32


@dataclass
class MxQuantized:
    """MX-quantized operand: fp4 uint8 [rows][(K-k_o)/2] (E2M1 nibbles), fp8 uint8 [rows][k_o]
    (E4M3, or None), sf uint8 [rows][ldsf] (UE8M0 block scales, bytes [0, K/32) used)."""
    fp4: Optional[object]
    fp8: Optional[object]
    sf: object
    K: int
    k_outlier: int

    @property
    def rows(self) -> int:
        return self.sf.shape[0]


def mx_quantize(x, perm, K: Optional[int] = None, k_outlier: int = 128, out=None,
                stream=None) -> MxQuantized:
    """Reorder + MX-quantize fp16 rows (activations online, weights offline)."""
    import torch
    if x.dtype != torch.float16 or x.dim() != 2 or x.stride(1) != 1:
        raise TypeError("x must be a 2-D fp16 tensor with contiguous rows")
    rows, ldx = x.shape[0], x.stride(0)
    K = perm.numel() if K is None else int(K)
    if perm.dtype != torch.int32 or K > perm.numel():
        raise ValueError("perm must be int32 with at least K entries")
    ldsf = ((K // MX_BLOCK + 15) // 16) * 16
    if out is None:
        dev = x.device
        fp4 = torch.empty((rows, (K - k_outlier) // 2), dtype=torch.uint8, device=dev) \
            if K > k_outlier else None
        fp8 = torch.empty((rows, k_outlier), dtype=torch.uint8, device=dev) if k_outlier else None
        sf = torch.zeros((rows, ldsf), dtype=torch.uint8, device=dev)
        out = MxQuantized(fp4, fp8, sf, K, k_outlier)
    else:   # a caller-supplied operand must have this call's shapes (the ABI checks only ldsf)
        want = [(out.fp4, (rows, (K - k_outlier) // 2) if K > k_outlier else None),
                (out.fp8, (rows, k_outlier) if k_outlier else None)]
        for t, shape in want:
            if (t is None) != (shape is None) or (t is not None and (
                    tuple(t.shape) != shape or t.dtype != torch.uint8 or not t.is_contiguous()
                    or t.device != x.device)):
                raise ValueError("out does not match this call's rows / K / k_outlier")
        if out.K != K or out.k_outlier != k_outlier or out.sf.shape[0] != rows or \
                out.sf.stride(0) < K // MX_BLOCK or out.sf.device != x.device:
            raise ValueError("out.sf does not match this call's rows / K")
    st = _lib().atom_mx_reorder_quantize(_ptr(x), rows, ldx, _ptr(perm), K, k_outlier,
                                         _ptr(out.fp4), _ptr(out.fp8), _ptr(out.sf),
                                         out.sf.stride(0), _stream(stream))
    _check(st, "atom_mx_reorder_quantize")
    return out


def mx_gemm(a: MxQuantized, w: MxQuantized, out=None, stream=None):
    """C[m][n] = fp16(sum_j deq(a[m][j]) deq(w[n][j])) on tcgen05 block-scaled MMAs."""
    import torch
    if a.K != w.K or a.k_outlier != w.k_outlier:
        raise ValueError("activation and weight quantization disagree on K / k_outlier")
    M, N = a.rows, w.rows
    if out is None:
        out = torch.empty((M, N), dtype=torch.float16, device=a.sf.device)
    if out.dtype != torch.float16 or out.dim() != 2 or out.stride(1) != 1 or \
            out.shape[0] < M or out.shape[1] < N:
        raise ValueError("out must be an fp16 [M][>=N] tensor with contiguous rows")
    n = _lib().atom_mx_gemm_workspace_size(M, N, a.K, a.k_outlier)
    ws = None
    if n:   # split-K partials; one buffer per (device, stream), grown on demand
        s = torch.cuda.current_stream() if stream is None else stream
        key = ("mx", s.device.index, s.cuda_stream)
        ws = _WORKSPACES.get(key)
        if ws is None or ws.numel() < n:
            with torch.cuda.stream(s):
                ws = _WORKSPACES[key] = torch.empty(n, dtype=torch.uint8, device=s.device)
    st = _lib().atom_mx_gemm(_ptr(a.fp4), _ptr(a.fp8), _ptr(a.sf), a.sf.stride(0), _ptr(w.fp4),
                             _ptr(w.fp8), _ptr(w.sf), w.sf.stride(0), M, N, a.K, a.k_outlier,
                             _ptr(out), out.stride(0), _ptr(ws), n, _stream(stream))
    _check(st, "atom_mx_gemm")
    return out


# ---------------------------------------------------------------------------------------------
# NEXT-3: quantized paged KV cache + decode attention (include/atom.h "KV cache")
# ---------------------------------------------------------------------------------------------
KV_PAGE = 16
HEAD_DIM = 128


@dataclass
class KvCache:
    """One of K or V: codes uint8 [num_pages][H][16][64], params fp32 [num_pages][H][16][2]."""
    codes: object
    params: object

    @staticmethod
    def empty(num_pages: int, H: int, device="cuda"):
        import torch
        return KvCache(torch.zeros((num_pages, H, KV_PAGE, HEAD_DIM // 2), dtype=torch.uint8,
                                   device=device),
                       torch.zeros((num_pages, H, KV_PAGE, 2), dtype=torch.float32,
                                   device=device))


def kv_quantize(x, slots, cache: KvCache, stream=None) -> KvCache:
    """Quantize T tokens' vectors x fp16 [T][H*128] into `cache` at int32 `slots`."""
    import torch
    if x.dtype != torch.float16 or x.dim() != 2 or x.stride(1) != 1:
        raise TypeError("x must be a 2-D fp16 tensor with contiguous rows")
    H = cache.codes.shape[1]
    if slots.dtype != torch.int32 or slots.numel() != x.shape[0] or x.shape[1] < H * HEAD_DIM:
        raise ValueError("slots must be int32 [T] and x [T][>= H*128]")
    st = _lib().atom_kv_quantize(_ptr(x), x.shape[0], x.stride(0), H, HEAD_DIM, _ptr(slots),
                                 _ptr(cache.codes), _ptr(cache.params), _stream(stream))
    _check(st, "atom_kv_quantize")
    return cache


_KV_WS = {}


def decode_attention(q, k: KvCache, v: KvCache, block_table, seq_lens, max_seq_len: int,
                     out=None, stream=None):
    """One decode step over the quantized cache: out fp32 [B][H][128]."""
    import torch
    B, H = q.shape[0], q.shape[1]
    if q.dtype != torch.float16 or tuple(q.shape[1:]) != (H, HEAD_DIM) or not q.is_contiguous():
        raise TypeError("q must be a contiguous fp16 [B][H][128] tensor")
    if block_table.dtype != torch.int32 or seq_lens.dtype != torch.int32:
        raise TypeError("block_table and seq_lens must be int32")
    if out is None:
        out = torch.empty((B, H, HEAD_DIM), dtype=torch.float32, device=q.device)
    n = _lib().atom_decode_attention_workspace_size(B, H, int(max_seq_len))
    ws = None
    if n:
        key = (q.device.index, n)
        ws = _KV_WS.get(key)
        if ws is None:
            ws = _KV_WS[key] = torch.empty(n, dtype=torch.uint8, device=q.device)
    st = _lib().atom_decode_attention(_ptr(q), B, H, HEAD_DIM, _ptr(k.codes), _ptr(k.params),
                                      _ptr(v.codes), _ptr(v.params), _ptr(block_table),
                                      block_table.shape[1], _ptr(seq_lens), int(max_seq_len),
                                      _ptr(out), _ptr(ws), n, _stream(stream))
    _check(st, "atom_decode_attention")
    return out
