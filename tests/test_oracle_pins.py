"""Pins of the CPU oracle against what the paper and mathematics fix.

None of these re-types the oracle's formulas: each compares the oracle with an independent fact
(a printed example, a closed form, a library routine on integers, a brute force, an invariant).
"""
import json
from fractions import Fraction
from pathlib import Path

import math

import numpy as np
import pytest

import oracle
import synth

G = 128
GOLDEN = Path(__file__).resolve().parent / "golden"
FLT_MIN = np.float32(np.finfo(np.float32).tiny)


# ----------------------------------------------------------------------------------------------
# independent helpers (no oracle code)
# ----------------------------------------------------------------------------------------------
def decode_q4(q4):
    """Two's-complement nibbles -> int codes, low nibble = even channel."""
    q4 = np.asarray(q4, dtype=np.int64)
    lo = q4 % 16
    hi = q4 // 16
    out = np.empty(q4.shape[:-1] + (2 * q4.shape[-1],), dtype=np.int64)
    out[..., 0::2] = np.where(lo >= 8, lo - 16, lo)
    out[..., 1::2] = np.where(hi >= 8, hi - 16, hi)
    return out


def codes_of(q4, q8):
    c = decode_q4(q4)
    if q8 is not None and q8.shape[-1]:
        c = np.concatenate([c, np.asarray(q8, dtype=np.int64)], axis=-1)
    return c


def pack_q4(codes):
    codes = np.asarray(codes, dtype=np.int64)
    lo = codes[..., 0::2] & 0xF
    hi = codes[..., 1::2] & 0xF
    return (lo | (hi << 4)).astype(np.uint8)


def f32_nearest(fr: Fraction) -> np.float32:
    """Round an exact rational to the nearest binary32 (ties to even) by exact comparison."""
    f = np.float32(float(fr))  # float() of a Fraction is correctly rounded to binary64
    # step to the correct binary32 neighbour using exact rational distances
    cands = [np.nextafter(f, np.float32(-np.inf)), f, np.nextafter(f, np.float32(np.inf))]
    best = min(cands, key=lambda c: (abs(Fraction(float(c)) - fr),
                                     int(np.float32(c).view(np.uint32)) & 1))
    return np.float32(best)


def unit_scale_block(rng, rows, K, k_o, gain_exp=None):
    """Integer-valued rows whose every group contains one +-7.5 (INT4) / +-127.5 (INT8) element,
    so that with clip = 1 the scale is exactly 2^e (P3).  Returns (values in REORDERED order,
    expected codes in reordered order)."""
    vals = np.zeros((rows, K), dtype=np.float64)
    codes = np.zeros((rows, K), dtype=np.int64)
    for t in range(K // G):
        int8 = k_o and t == K // G - 1
        lim, half = (127, 127.5) if int8 else (7, 7.5)
        blk = rng.integers(-lim, lim + 1, size=(rows, G))
        pos = rng.integers(0, G, size=rows)
        sign = rng.choice([-1.0, 1.0], size=rows)
        v = blk.astype(np.float64)
        c = blk.copy()
        v[np.arange(rows), pos] = sign * half
        # +7.5 -> rint 8 -> clamp 7 ; -7.5 -> rint -8 (ties-even) ; +127.5 -> 128 -> 127 ; -127.5 -> -128
        c[np.arange(rows), pos] = np.where(sign > 0, lim, -lim - 1)
        if gain_exp is not None:
            v *= 2.0 ** gain_exp[t][:, None]
        vals[:, t * G:(t + 1) * G] = v
        codes[:, t * G:(t + 1) * G] = c
    return vals, codes


def scatter(vals_reordered, perm):
    """Inverse of the gather x'[j] = x[perm[j]]: returns x with x[perm[j]] = x'[j]."""
    x = np.zeros_like(vals_reordered)
    x[:, perm] = vals_reordered
    return x


# ----------------------------------------------------------------------------------------------
# P1  effective bits (P:256 footnote)
# ----------------------------------------------------------------------------------------------
def test_p1_effective_bits_from_buffers():
    K, k_o, rows = 4096, 128, 3
    x = synth.activations(rows, K, 0)
    perm = synth.perm_for(K, 0)
    q4, q8, sc = oracle.quantize_rows(x, perm, K, k_o)
    code_bits = 8 * (q4.nbytes + q8.nbytes) / (rows * K)
    paper = code_bits + 16 / G          # 16-bit scales as in the footnote
    assert paper == 4.25                # P:256 "((4096-128)*4+128*8)/4096+16/128=4.25"
    build = code_bits + 8 * sc.nbytes / (rows * K)
    assert build == 4.375               # fp32 scales
    assert sc.shape == (K // G, rows)


def test_golden_spec_examples_file():
    ex = json.loads((GOLDEN / "spec_examples.json").read_text())
    assert ex["effective_bits"]["value"] == 4.25
    assert ex["pack"]["byte"] == 0x78


# ----------------------------------------------------------------------------------------------
# P2  SPEC / paper worked examples
# ----------------------------------------------------------------------------------------------
def _one_group_row(vals, k_o=0, K=128):
    x = np.zeros((1, K), dtype=np.float32)
    x[0, :len(vals)] = vals
    return x


def test_p2_pack_example_S55():
    # codes [-8, 7] -> one byte 0x78, low nibble first.  Scale 1 by the unit-scale construction.
    x = _one_group_row([-7.5, 7.0])
    q4, q8, sc = oracle.quantize_rows(x, np.arange(128), 128, 0, clip_int4=1.0)
    assert sc[0, 0] == np.float32(1.0)
    assert q4[0, 0] == 0x78


def test_p2_scale_example_S118_and_code_example_S136():
    x = _one_group_row([-1.0, 0.5, 1.0])
    q4, _, sc = oracle.quantize_rows(x, np.arange(128), 128, 0, clip_int4=1.0)
    # s = 2 * max|x| * c / (2^n - 1) = 2/15; binary32 rounding of alpha then of amax*alpha
    alpha = f32_nearest(Fraction(2, 15))
    assert alpha.view(np.uint32) == 0x3E088889
    s_expected = f32_nearest(Fraction(float(alpha)) * 1)
    assert sc[0, 0] == s_expected and sc[0, 0].view(np.uint32) == 0x3E088889
    # exact arithmetic gives [-8, 4, 7]: -7.5 ties to -8, 3.75 -> 4, 7.5 -> 8 -> 7
    exact = []
    for v in (Fraction(-1), Fraction(1, 2), Fraction(1)):
        r = v / Fraction(2, 15)
        fl = r.numerator // r.denominator
        rem = r - fl
        q = fl + 1 if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2) else fl
        exact.append(max(-8, min(7, q)))
    assert exact == [-8, 4, 7]
    # pinned binary32 pipeline: 1/s rounds down, -1*inv = -7.4999995 -> -7
    codes = decode_q4(q4)[0, :3]
    assert list(codes) == [-7, 4, 7]


def test_p2_int8_scale_example_S120():
    # x = [-3, 3], n = 8, c = 0.5 -> s = 2*3*0.5/255 = 3/255
    x = np.zeros((1, 128), dtype=np.float32)
    x[0, :2] = [-3.0, 3.0]
    _, _, sc = oracle.quantize_rows(x, np.arange(128), 128, 128, clip_int8=0.5)
    exact = Fraction(3, 255)
    # two roundings (alpha, then 3*alpha): error <= 3*(ulp(alpha)/2) + ulp(s)/2 < 2 ulp(s)
    assert abs(Fraction(float(sc[0, 0])) - exact) <= 2 * Fraction(float(np.spacing(np.float32(exact))))


def test_p2_dequant_example_S145():
    s = np.float64(np.float32(Fraction(2, 15).__float__()))
    deq = np.array([-8, 4, 7]) * s
    np.testing.assert_allclose(deq, [-1.0667, 0.5333, 0.9333], atol=1e-4)


def test_p2_group_counts_S154():
    x = synth.activations(1, 256, 1)
    _, _, sc = oracle.quantize_rows(x, np.arange(256), 256, 0)
    assert sc.shape == (2, 1)          # 1x256 row, g = 128 -> 2 groups
    _, q8, sc = oracle.quantize_rows(x, np.arange(256), 256, 128)
    assert sc.shape == (2, 1) and q8.shape == (1, 128)   # 1 normal + 1 outlier group


def test_p2_reorder_example_S227():
    # 1x3 [a, b, c] with permutation [0, 2, 1] -> [a, c, b]; the remaining channels are identity
    perm = np.arange(128)
    perm[1], perm[2] = 2, 1
    x = _one_group_row([1.0, 2.0, 3.0])
    x[0, 3] = 7.5                      # unit scale
    q4, _, _ = oracle.quantize_rows(x, perm, 128, 0, clip_int4=1.0)
    assert list(decode_q4(q4)[0, :3]) == [1, 3, 2]


def test_p2_all_ones_group_gemm_S285():
    a = np.ones((1, 128), dtype=np.int64)
    q4 = pack_q4(a)
    P = oracle.group_partials(q4, None, q4, None, 1, 1, 128, 0)
    assert P[0, 0, 0] == 128
    C = oracle.gemm_output(P, np.ones((1, 1), np.float32), np.ones((1, 1), np.float32))
    assert C[0, 0] == 128.0


# ----------------------------------------------------------------------------------------------
# P3  unit-scale closed form: whole pipeline == exact integer GEMM (numpy int64 matmul)
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("M,N,K,k_o", [(5, 7, 512, 128), (3, 4, 256, 0), (2, 3, 128, 128)])
def test_p3_unit_scale_closed_form(M, N, K, k_o):
    rng = np.random.default_rng(11)
    perm = rng.permutation(K).astype(np.int32)
    av, ac = unit_scale_block(rng, M, K, k_o)
    wv, wc = unit_scale_block(rng, N, K, k_o)
    X, W = scatter(av, perm).astype(np.float16), scatter(wv, perm).astype(np.float16)
    r = oracle.quantized_linear(X, perm, W, K, k_o, clip_a=1.0, clip_w=1.0)
    assert np.all(r["a_scales"] == 1.0) and np.all(r["w_scales"] == 1.0)
    # codes: gather direction and packing
    np.testing.assert_array_equal(codes_of(r["a_q4"], r["a_q8"]), ac)
    np.testing.assert_array_equal(codes_of(r["w_q4"], r["w_q8"]), wc)
    # output: library integer matmul
    np.testing.assert_array_equal(r["c"], (ac @ wc.T).astype(np.float64))
    # per-group partials: library integer matmul per group
    for t in range(K // G):
        sl = slice(t * G, (t + 1) * G)
        np.testing.assert_array_equal(r["partials"][t], ac[:, sl] @ wc[:, sl].T)


def test_p3_groupwise_pow2_scales_pin_scale_indexing():
    """Each (row, group) gets its own power-of-two scale 2^e: s must equal 2^e exactly and C must
    equal sum_t 2^(ea[t][m]+ew[t][n]) P_t exactly -- pins group/row indexing of both scale arrays."""
    rng = np.random.default_rng(5)
    M, N, K, k_o = 4, 6, 512, 128
    Gn = K // G
    ea = rng.integers(-3, 4, size=(Gn, M))
    ew = rng.integers(-3, 4, size=(Gn, N))
    perm = rng.permutation(K).astype(np.int32)
    av, ac = unit_scale_block(rng, M, K, k_o, ea)
    wv, wc = unit_scale_block(rng, N, K, k_o, ew)
    r = oracle.quantized_linear(scatter(av, perm).astype(np.float16), perm,
                                scatter(wv, perm).astype(np.float16), K, k_o, 1.0, 1.0)
    np.testing.assert_array_equal(r["a_scales"], 2.0 ** ea)
    np.testing.assert_array_equal(r["w_scales"], 2.0 ** ew)
    exp = np.zeros((M, N))
    for t in range(Gn):
        sl = slice(t * G, (t + 1) * G)
        exp += (2.0 ** (ea[t][:, None] + ew[t][None, :])) * (ac[:, sl] @ wc[:, sl].T)
    np.testing.assert_array_equal(r["c"], exp)


# ----------------------------------------------------------------------------------------------
# P4  round-trip and code-range invariants
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("clip4,clip8", [(0.9, 1.0), (0.85, 1.0), (1.0, 1.0), (0.7, 0.9)])
def test_p4_round_trip(clip4, clip8):
    K = 1024
    x = synth.activations(64, K, 3).astype(np.float32)
    perm = synth.perm_for(K, 3)
    q4, q8, sc = oracle.quantize_rows(x, perm, K, 128, clip4, clip8)
    codes = codes_of(q4, q8)
    xr = x[:, perm].astype(np.float64)
    s = np.repeat(sc.T.astype(np.float64), G, axis=1)
    nb = np.array([4] * (K - 128) + [8] * 128)
    lo = np.broadcast_to(-(2.0 ** (nb - 1)), codes.shape)
    hi = np.broadcast_to(2.0 ** (nb - 1) - 1, codes.shape)
    assert np.all(codes >= lo) and np.all(codes <= hi)
    err = np.abs(xr - codes * s)
    bound = s / 2 + 2 * np.spacing(np.abs(xr).astype(np.float32)).astype(np.float64)
    inside = (codes > lo) & (codes < hi)
    assert np.all(err[inside] <= bound[inside])
    # saturated codes only where |x|/s is beyond the last level
    sat_hi = codes == hi
    # (slack: two binary32 roundings in x * fl(1/s), relative 2^-22)
    assert np.all(xr[sat_hi] / s[sat_hi] >= (hi[sat_hi] - 0.5) * (1 - 2.0 ** -22))
    sat_lo = codes == lo
    assert np.all(xr[sat_lo] / s[sat_lo] <= (lo[sat_lo] + 0.5) * (1 - 2.0 ** -22))
    # group max element lands on the clipped top level: |x|/s = (2^n-1)/(2c)
    amax = np.abs(xr).reshape(64, K // G, G).max(axis=2)
    np.testing.assert_allclose(amax / sc.T, [[15 / (2 * clip4)] * (K // G - 1) + [255 / (2 * clip8)]] * 64,
                               rtol=1e-6)


def test_p4_degenerate_zero_group():
    x = np.zeros((2, 256), dtype=np.float32)
    x[1, 128:] = 3.0
    q4, q8, sc = oracle.quantize_rows(x, np.arange(256), 256, 128)
    assert sc[0, 0] == FLT_MIN and sc[0, 1] == FLT_MIN and sc[1, 0] == FLT_MIN
    assert np.all(q4 == 0) and np.all(q8[0] == 0)
    assert np.all(q8[1] == 127)     # constant group with clip 1: 3/(3*2/255) = 127.5 -> 127


def test_p4_adversarial_values():
    K = 256
    x = np.zeros((4, K), dtype=np.float16)
    x[0, :] = np.float16(65504)
    x[0, 1::2] = -np.float16(65504)
    x[1, :] = np.float16(2.0 ** -24)              # fp16 subnormal
    x[2, 5] = -3.0                                # group whose max is negative
    x[3, :] = np.float16(1e-3)
    q4, q8, sc = oracle.quantize_rows(x, np.arange(K), K, 128)
    assert np.all(np.isfinite(sc)) and np.all(sc > 0)
    c = codes_of(q4, q8)
    assert c[0, 0] == 7 and c[0, 1] == -8          # +-max saturate (clip 0.9: |v| = 8.33)
    assert c[2, 5] == -8 and np.all(np.delete(c[2, :128], 5) == 0)
    assert np.all(c[1, :128] == 7)                 # constant positive group -> top level
    assert np.all(c[1, 128:] == 127)


# ----------------------------------------------------------------------------------------------
# P5  reorder index invariants
# ----------------------------------------------------------------------------------------------
def test_p5_calibration_example_S217():
    np.testing.assert_array_equal(synth.calibration_perm(np.array([[1.0, 10.0, 1.0]]), 1), [0, 2, 1])
    # tie -> lower index
    np.testing.assert_array_equal(synth.calibration_perm(np.array([[2.0, 2.0, 1.0]]), 1), [1, 2, 0])


@pytest.mark.parametrize("K,seed", [(1024, 0), (4096, 1), (8192, 2)])
def test_p5_perm_invariants(K, seed):
    perm = synth.perm_for(K, seed)
    assert np.array_equal(np.sort(perm), np.arange(K))                   # bijection
    np.testing.assert_array_equal(perm[-128:], synth.outlier_channels(K, seed))   # tail = injected
    assert np.all(np.diff(perm[:-128]) > 0) and np.all(np.diff(perm[-128:]) > 0)


# ----------------------------------------------------------------------------------------------
# P6  brute-force partials on tiny inputs (independent decode + python loops)
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("M,N,K,k_o", [(3, 4, 256, 128), (2, 5, 384, 0), (4, 3, 128, 128)])
def test_p6_brute_force_partials(M, N, K, k_o):
    rng = np.random.default_rng(M * 100 + N)
    aq4 = rng.integers(0, 256, size=(M, (K - k_o) // 2), dtype=np.uint8)
    wq4 = rng.integers(0, 256, size=(N, (K - k_o) // 2), dtype=np.uint8)
    aq8 = rng.integers(-128, 128, size=(M, k_o), dtype=np.int8) if k_o else None
    wq8 = rng.integers(-128, 128, size=(N, k_o), dtype=np.int8) if k_o else None
    P = oracle.group_partials(aq4, aq8, wq4, wq8, M, N, K, k_o)

    def code(q4row, q8row, j):
        if j < K - k_o:
            b = int(q4row[j >> 1])
            v = (b >> 4) if (j & 1) else (b & 15)
            return v - 16 if v & 8 else v
        return int(q8row[j - (K - k_o)])

    for m in range(M):
        for n in range(N):
            for t in range(K // G):
                s = 0
                for j in range(t * G, (t + 1) * G):
                    s += code(aq4[m], None if aq8 is None else aq8[m], j) * \
                         code(wq4[n], None if wq8 is None else wq8[n], j)
                assert P[t, m, n] == s


def test_p6_extreme_partials_fit_int32():
    # worst case |P|: INT8 group all -128 * -128 = 2^21
    q8 = np.full((1, 128), -128, dtype=np.int8)
    q4 = np.full((1, 0), 0, dtype=np.uint8)
    P = oracle.group_partials(q4, q8, q4, q8, 1, 1, 128, 128)
    assert P[0, 0, 0] == 128 * 128 * 128
    q4 = np.full((1, 64), 0x88, dtype=np.uint8)     # all -8
    P = oracle.group_partials(q4, None, q4, None, 1, 1, 128, 0)
    assert P[0, 0, 0] == 128 * 64


# ----------------------------------------------------------------------------------------------
# P7  INT8 outlier closed form: normal block zero -> C = sum over outliers of x*w exactly
# ----------------------------------------------------------------------------------------------
def test_p7_outlier_closed_form():
    rng = np.random.default_rng(7)
    M, N, K = 3, 5, 512
    perm = rng.permutation(K).astype(np.int32)
    av, ac = unit_scale_block(rng, M, K, 128)
    wv, wc = unit_scale_block(rng, N, K, 128)
    av[:, :K - 128] = 0
    wv[:, :K - 128] = 0
    r = oracle.quantized_linear(scatter(av, perm).astype(np.float16), perm,
                                scatter(wv, perm).astype(np.float16), K, 128, 1.0, 1.0)
    np.testing.assert_array_equal(r["c"], (ac[:, -128:] @ wc[:, -128:].T).astype(np.float64))
    assert np.all(r["partials"][:-1] == 0)


# ----------------------------------------------------------------------------------------------
# P8  power-of-two bilinearity: exact in floating point
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("ka,kw", [(1, 0), (0, -3), (2, 2)])
def test_p8_pow2_bilinearity(ka, kw):
    M, N, K = 6, 8, 512
    X, W, perm = synth.problem(M, N, K, seed=4)
    base = oracle.quantized_linear(X, perm, W, K)
    X2 = (X.astype(np.float32) * 2.0 ** ka).astype(np.float16)
    W2 = (W.astype(np.float32) * 2.0 ** kw).astype(np.float16)
    assert np.array_equal(X2.astype(np.float32), X.astype(np.float32) * 2.0 ** ka)
    r = oracle.quantized_linear(X2, perm, W2, K)
    for k in ("a_q4", "a_q8", "w_q4", "w_q8", "partials"):
        np.testing.assert_array_equal(r[k], base[k])
    np.testing.assert_array_equal(r["a_scales"], base["a_scales"] * np.float32(2.0 ** ka))
    np.testing.assert_array_equal(r["w_scales"], base["w_scales"] * np.float32(2.0 ** kw))
    np.testing.assert_array_equal(r["c"], base["c"] * 2.0 ** (ka + kw))


# ----------------------------------------------------------------------------------------------
# P9  equivariance: permuting W rows / tokens permutes outputs bit-exactly
# ----------------------------------------------------------------------------------------------
def test_p9_equivariance():
    M, N, K = 5, 9, 384
    X, W, perm = synth.problem(M, N, K, seed=9)
    base = oracle.quantized_linear(X, perm, W, K)
    rng = np.random.default_rng(3)
    pn, pm = rng.permutation(N), rng.permutation(M)
    r = oracle.quantized_linear(X[pm], perm, W[pn], K)
    np.testing.assert_array_equal(r["c"], base["c"][pm][:, pn])
    np.testing.assert_array_equal(r["w_q4"], base["w_q4"][pn])
    np.testing.assert_array_equal(r["a_scales"], base["a_scales"][:, pm])
    np.testing.assert_array_equal(r["partials"], base["partials"][:, pm][:, :, pn])


# ----------------------------------------------------------------------------------------------
# P10 special cases of the mixed split
# ----------------------------------------------------------------------------------------------
def test_p10_zero_outlier_block_equals_int4_only():
    M, N, K = 4, 6, 512
    X, W, perm = synth.problem(M, N, K, seed=12)
    X = X.copy()
    X[:, perm[-128:]] = 0
    full = oracle.quantized_linear(X, perm, W, K, 128)
    assert np.all(full["partials"][-1] == 0)
    int4 = oracle.quantized_linear(X, perm[:-128], W, K - 128, 0)
    np.testing.assert_array_equal(full["c"], int4["c"])
    np.testing.assert_array_equal(full["a_q4"], int4["a_q4"])


def test_p10_single_group_is_textbook_w8a8():
    M, N = 5, 7
    X, W, perm = synth.problem(M, N, 128, seed=13)
    r = oracle.quantized_linear(X, perm, W, 128, 128)
    assert r["a_q4"].shape == (M, 0)
    # per-token x per-channel W8A8: C = diag(s_a) (A8 W8^T) diag(s_w)
    textbook = (r["a_scales"][0].astype(np.float64)[:, None] * r["w_scales"][0].astype(np.float64)[None, :]) \
        * (r["a_q8"].astype(np.int64) @ r["w_q8"].astype(np.int64).T)
    np.testing.assert_array_equal(r["c"], textbook)


def test_p10_output_rows_matches_full():
    M, N, K = 6, 5, 640
    X, W, perm = synth.problem(M, N, K, seed=2)
    r = oracle.quantized_linear(X, perm, W, K)
    rows = [5, 0, 3]
    c = oracle.output_rows(r["a_q4"], r["a_q8"], r["a_scales"], r["w_q4"], r["w_q8"],
                           r["w_scales"], M, N, K, 128, rows)
    np.testing.assert_array_equal(c, r["c"][rows])


def test_oracle_thread_count_invariance():
    M, N, K = 16, 64, 1024
    X, W, perm = synth.problem(M, N, K, seed=21)
    oracle.set_threads(1)
    a = oracle.quantized_linear(X, perm, W, K)
    oracle.set_threads(4)
    b = oracle.quantized_linear(X, perm, W, K)
    oracle.set_threads(oracle.max_threads())
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])


def test_quantization_error_info_O9():
    """O9 (info, not parity): relative Frobenius error vs the unquantized product ~1.2%."""
    M, N, K = 64, 256, 4096
    X, W, perm = synth.problem(M, N, K, seed=0)
    r = oracle.quantized_linear(X, perm, W, K)
    ref = X.astype(np.float64) @ W.astype(np.float64).T
    rel = np.linalg.norm(r["c"] - ref) / np.linalg.norm(ref)
    assert 0.002 < rel < 0.05


def test_oracle_rejects_bad_shapes():
    x = np.zeros((1, 256), np.float32)
    with pytest.raises(oracle.OracleError):
        oracle.quantize_rows(x, np.arange(200), 200, 0)          # K % 128
    with pytest.raises(oracle.OracleError):
        oracle.quantize_rows(x, np.arange(256), 256, 64)         # k_o not in {0,128}
    with pytest.raises(oracle.OracleError):
        oracle.quantize_rows(x, np.arange(256), 256, 128, clip_int4=1.5)


# ----------------------------------------------------------------------------------------------
# N1 (NEXT-1): RMSNorm, the prior operator the paper fuses reorder + quantize into
# ----------------------------------------------------------------------------------------------
def test_n1_single_nonzero_closed_form():
    """x = [v, 0, ..., 0], gamma = 1, eps = 0 over C = 1024 channels: mean(x^2) = v^2/1024, so
    y_0 = v / (|v|/32) = 32*sign(v) exactly (powers of two) and every other y_c = 0.  Catches a
    sum instead of a mean (y_0 = 1), a missing square root (y_0 = 1024/v) and dropped channels."""
    C = 1024
    for v in (4.0, -0.25, 1024.0):
        x = np.zeros((1, C), np.float16)
        x[0, 5] = v
        y = oracle.rmsnorm_rows(x, np.ones(C, np.float16), eps=0.0)
        want = np.zeros((1, C), np.float16)
        want[0, 5] = 32.0 * np.sign(v)
        np.testing.assert_array_equal(y, want)


def test_n1_constant_row_and_gamma():
    """A constant row normalizes to +-1 times gamma; gamma is applied per channel (a
    power-of-two gamma gives an exact power-of-two output)."""
    C = 256
    g = (2.0 ** (np.arange(C) % 7 - 3)).astype(np.float16)
    for a in (3.0, -0.5):
        x = np.full((2, C), a, np.float16)
        y = oracle.rmsnorm_rows(x, g, eps=0.0)
        np.testing.assert_array_equal(y, np.tile(np.sign(a) * g, (2, 1)).astype(np.float16))


def test_n1_pow2_scale_invariance():
    """RMSNorm(2^k x) == RMSNorm(x) bit for bit when eps = 0 (every pinned operation commutes
    with exact power-of-two scaling)."""
    rng = np.random.default_rng(3)
    # magnitudes in [0.5, 4): inputs and outputs stay fp16-normal under the 2^k scalings
    x = (np.sign(rng.standard_normal((8, 512))) * rng.uniform(0.5, 4, (8, 512))).astype(np.float16)
    g = (1 + 0.1 * rng.standard_normal(512)).astype(np.float16)
    y = oracle.rmsnorm_rows(x, g, eps=0.0)
    for k in (-3, 2):
        np.testing.assert_array_equal(oracle.rmsnorm_rows(x * np.float16(2.0 ** k), g, 0.0), y)


def test_n1_eps_and_float64_reference():
    """Against a float64 textbook RMSNorm: within fp16 rounding (plus the fp32 steps); eps counts
    (tiny inputs with eps = 1 are left almost unscaled)."""
    rng = np.random.default_rng(4)
    x = (rng.standard_normal((16, 768)) * np.exp(rng.standard_normal((16, 1)))).astype(np.float16)
    g = (1 + 0.2 * rng.standard_normal(768)).astype(np.float16)
    eps = 1e-6
    x64, g64 = x.astype(np.float64), g.astype(np.float64)
    ref = x64 / np.sqrt((x64 ** 2).mean(1, keepdims=True) + eps) * g64
    y = oracle.rmsnorm_rows(x, g, eps).astype(np.float64)
    assert np.all(np.abs(y - ref) <= 2.0 ** -10 * np.abs(ref) + 2.0 ** -24)
    tiny = np.full((1, 128), 1e-3, np.float16)
    yt = oracle.rmsnorm_rows(tiny, np.ones(128, np.float16), eps=1.0).astype(np.float64)
    assert np.allclose(yt, 1e-3 / np.sqrt(1.0 + 1e-6), rtol=2e-3)


def test_n1_exact_sum_of_squares_fractions_and_order():
    """Reading G19 pins the sum of squares as the EXACT sum rounded once to double.  Pinned
    against Python's exact rational arithmetic (fractions.Fraction, then one rounding to float64)
    on rows built so that a running double sum depends on the order (one huge square absorbs the
    tiny ones unless they are added first), and by order independence: reversing the channels
    (with gamma) reverses the output bit for bit."""
    from fractions import Fraction
    C = 1024
    x = np.full((2, C), np.float16(2.0 ** -12), np.float16)
    x[0, 0] = np.float16(60000.0)            # huge first: a running sum drops the tiny squares
    x[1, -1] = np.float16(60000.0)           # huge last: a running sum keeps them
    x[1, :8] = np.float16(-3.0)
    g = (1 + 0.05 * np.random.default_rng(9).standard_normal(C)).astype(np.float16)
    eps = 1e-6
    y = oracle.rmsnorm_rows(x, g, eps)
    for r in range(2):
        ss = float(sum(Fraction(float(v)) ** 2 for v in x[r].astype(np.float64)))   # exact, RN64
        rinv = np.float32(1.0 / math.sqrt(ss / C + float(np.float64(np.float32(eps)))))
        want = ((x[r].astype(np.float32) * rinv) * g.astype(np.float32)).astype(np.float16)
        np.testing.assert_array_equal(y[r], want)
    yr = oracle.rmsnorm_rows(x[:, ::-1].copy(), g[::-1].copy(), eps)
    np.testing.assert_array_equal(yr[:, ::-1], y)


def test_n1_fused_oracle_is_norm_then_quantize():
    rng = np.random.default_rng(5)
    K = 1024
    x = rng.standard_normal((6, K)).astype(np.float16)
    g = (1 + 0.1 * rng.standard_normal(K)).astype(np.float16)
    perm = synth.perm_for(K, seed=5)
    a = oracle.rmsnorm_quantize_rows(x, g, perm, K)
    b = oracle.quantize_rows(oracle.rmsnorm_rows(x, g), perm, K)
    for u, v in zip(a, b):
        np.testing.assert_array_equal(u, v)


# ----------------------------------------------------------------------------------------------
# N4 (NEXT-4 piece): SwiGLU h = silu(gate) * up, the down projection's prior operator (P:270,
# reading G20)
# ----------------------------------------------------------------------------------------------
def test_n4_special_values():
    """silu(0) = 0; for g >= 17, exp(-g) < 2^-24 so RN32(silu(g)) = g exactly and h = fp16(g*u);
    for g = -30, |silu(g)| < 1e-11 so h is a signed zero for any fp16 u; u = 0 gives 0."""
    C = 256
    rng = np.random.default_rng(11)
    u = rng.uniform(-4, 4, (3, C)).astype(np.float16)
    g = np.zeros((3, C), np.float16)
    g[1] = 17.0
    g[2] = -30.0
    h = oracle.silu_mul_rows(g, u)
    np.testing.assert_array_equal(h[0], np.zeros(C, np.float16))
    np.testing.assert_array_equal(h[1], (np.float32(17.0) * u[1].astype(np.float32)).astype(np.float16))
    assert np.all(h[2] == 0)
    np.testing.assert_array_equal(oracle.silu_mul_rows(rng.standard_normal((2, C)).astype(np.float16),
                                                       np.zeros((2, C), np.float16)) == 0, True)


def test_n4_expf_pinned_accuracy_and_special_values():
    """The binary32 exponential of reading G20 against libm's double exp on a dense grid of the
    domain it serves (x = -g for fp16 g): within 4 binary32 ulps (relative 2^-21) on
    [-87, 88]; exp(0) = 1 exactly; +inf above 88 and 0 below -87.  Catches a wrong constant,
    a dropped polynomial term or a mis-scaled 2^n."""
    xs = np.concatenate([np.linspace(-87, 88, 20001), np.float16(np.linspace(-30, 30, 4001))])
    for x in xs.astype(np.float32):
        got = oracle.expf_pinned(float(x))
        want = math.exp(float(x))
        assert abs(got / want - 1.0) <= 2.0 ** -21, (float(x), got, want)
    assert oracle.expf_pinned(0.0) == 1.0
    assert oracle.expf_pinned(88.5) == math.inf and oracle.expf_pinned(1e4) == math.inf
    assert oracle.expf_pinned(-87.5) == 0.0


def test_n4_tanh_form_and_sign():
    """Against the independent form silu(g) = g/2 * (1 + tanh(g/2)) in float64, rounded by the
    same pinned steps: identical except where the two double results straddle a binary32
    rounding boundary (never more than one fp16 ulp).  Catches exp(+g), a missing factor g, and
    swapped gate / up."""
    rng = np.random.default_rng(12)
    g = (rng.standard_normal((64, 512)) * 3).astype(np.float16)
    u = rng.standard_normal((64, 512)).astype(np.float16)
    g64 = g.astype(np.float64)
    s = (g64 / 2 * (1 + np.tanh(g64 / 2))).astype(np.float32)
    want = (s * u.astype(np.float32)).astype(np.float16)
    h = oracle.silu_mul_rows(g, u)
    same = (h == want) | ((h == 0) & (want == 0))
    assert same.mean() > 0.999
    ulp = np.abs(h.astype(np.float64) - want.astype(np.float64))
    assert np.all(ulp <= np.spacing(np.abs(want).astype(np.float16)).astype(np.float64) + 1e-30)
    assert not np.array_equal(oracle.silu_mul_rows(u, g), h)   # not symmetric in (gate, up)


def test_n4_fused_oracle_is_swiglu_then_quantize():
    K = 1024
    rng = np.random.default_rng(13)
    g = (rng.standard_normal((5, K)) * 2).astype(np.float16)
    u = rng.standard_normal((5, K)).astype(np.float16)
    perm = synth.perm_for(K, 13)
    a = oracle.silu_mul_quantize_rows(g, u, perm, K)
    b = oracle.quantize_rows(oracle.silu_mul_rows(g, u), perm, K)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
