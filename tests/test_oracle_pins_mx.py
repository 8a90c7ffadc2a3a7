"""Pins of the Atom (FP) MX oracle (oracle/mx_oracle.c, NEXT-2) to things other than itself:
the OCP element tables, torch's float8_e4m3fn conversion (a library routine), the defining
properties of round-to-nearest-even, power-of-two closed forms of the shared exponent, and a
lossless end-to-end case whose output is numpy's float64 matmul.

Paper: Atom (FP), "quantizing both weights and activations into FP4" with "group quantization
with the MX format" (Section 6; Table 5).  Readings G21-G24
(DESIGN.md): MXFP4 E2M1 blocks of 32 with UE8M0 scales for the normal channels, MXFP8 E4M3 for
the 128 outlier channels, the OCP MX v1.0 Section 6.3 conversion.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

# OCP Microscaling Formats (MX) v1.0, FP4 E2M1 element values (Section 5.3.3): the magnitudes of
# the 8 codes 0b000 .. 0b111
E2M1_SPEC = [0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0]


def test_e2m1_decode_is_the_spec_table():
    for c in range(8):
        assert oracle.e2m1_value(c) == E2M1_SPEC[c]
        assert oracle.e2m1_value(c | 8) == -E2M1_SPEC[c]


def test_e4m3_decode_matches_torch():
    codes = np.array([c for c in range(256) if (c & 0x7F) != 0x7F], dtype=np.uint8)
    t = torch.from_numpy(codes).view(torch.float8_e4m3fn).float().numpy()
    got = np.array([oracle.e4m3_value(int(c)) for c in codes])
    np.testing.assert_array_equal(got, t.astype(np.float64))


def test_e4m3_encode_matches_torch_rne():
    rng = np.random.default_rng(0)
    grid = np.array([oracle.e4m3_value(c) for c in range(0x7F)])
    mids = (grid[1:] + grid[:-1]) / 2          # exact ties (representable in fp32)
    v = np.concatenate([rng.uniform(-448, 448, 4000), rng.normal(0, 0.05, 2000), mids, -mids,
                        grid, -grid]).astype(np.float32)
    ref = torch.from_numpy(v).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    got = np.array([oracle.e4m3_code(float(x)) for x in v], dtype=np.uint8)
    # torch keeps the sign of a zero result only for negative inputs, as the oracle does
    np.testing.assert_array_equal(got, ref)


def test_e4m3_saturates():
    assert oracle.e4m3_code(1000.0) == 0x7E and oracle.e4m3_code(-460.0) == 0xFE
    assert oracle.e4m3_code(448.0) == 0x7E


def _grid_neighbours(a):
    g = np.array(E2M1_SPEC)
    lo = g[g <= a].max()
    hi = g[g >= a].min() if a <= 6.0 else 6.0
    return lo, hi


def test_e2m1_encode_is_round_to_nearest_even():
    """Uniquely characterises RNE with saturation: the result is a neighbour on the grid, no
    grid point is nearer, ties take the code with mantissa bit 0, beyond 6 saturates, the sign
    follows x, and the map is idempotent and monotone."""
    rng = np.random.default_rng(1)
    g = np.array(E2M1_SPEC)
    mids = (g[1:] + g[:-1]) / 2
    vals = np.concatenate([rng.uniform(0, 8, 3000), mids, g, [6.5, 7.0, 7.99, 1e6]])
    prev = -1.0
    for a in np.sort(vals.astype(np.float32)):
        c = oracle.e2m1_code(float(a))
        q = oracle.e2m1_value(c)
        assert c < 8
        if a >= 6.0:
            assert q == 6.0
            continue
        lo, hi = _grid_neighbours(float(a))
        assert q in (lo, hi)
        assert abs(a - q) <= min(abs(a - lo), abs(a - hi))
        if abs(a - lo) == abs(hi - a) and lo != hi:
            assert (c & 1) == 0, (a, c)
        assert q >= prev
        prev = q
        assert oracle.e2m1_code(-float(a)) == c | 8
    for c in range(8):
        assert oracle.e2m1_code(E2M1_SPEC[c]) == c


@pytest.mark.parametrize("emax", [2, 8])
def test_scale_byte_closed_form(emax):
    """shared_exp = floor(log2 amax) - emax_elem (OCP MX v1.0 6.3): on amax = f 2^k, f in [1,2)."""
    for k in range(-24, 16):
        for f in (1.0, 1.25, 1.999):
            amax = np.float32(f * 2.0 ** k)
            assert oracle.mx_scale_byte(float(amax), emax) == k - emax + 127
    assert oracle.mx_scale_byte(0.0, emax) == 0
    # the block max lands in [2^emax, 2^(emax+1)) before saturation
    rng = np.random.default_rng(emax)
    for amax in rng.uniform(1e-3, 6e4, 200).astype(np.float32):
        X = 2.0 ** (oracle.mx_scale_byte(float(amax), emax) - 127)
        assert 2 ** emax <= amax / X < 2 ** (emax + 1)


def _lossless_rows(rng, rows, K, k_o):
    """Rows whose 32-blocks are exactly representable: block b has exponent s_b in [-3, 3] and
    elements s * grid value, with one element of magnitude 4 (E2M1 blocks) or 256..448 (E4M3), so
    the OCP shared exponent is s_b exactly and the codes are lossless."""
    K4 = K - k_o
    x = np.zeros((rows, K), dtype=np.float64)
    for r in range(rows):
        for b in range(K // 32):
            s = rng.integers(-3, 4)
            if 32 * b < K4:
                vals = rng.choice(E2M1_SPEC, 32) * rng.choice([-1, 1], 32)
                vals[rng.integers(32)] = 4.0 * rng.choice([-1, 1])
            else:
                e4 = np.array([oracle.e4m3_value(c) for c in range(0x7F)])
                vals = rng.choice(e4[e4 <= 240], 32) * rng.choice([-1, 1], 32)
                vals[rng.integers(32)] = rng.choice([256.0, 320.0, 448.0]) * rng.choice([-1, 1])
            x[r, 32 * b:32 * b + 32] = vals * 2.0 ** s
    return x


@pytest.mark.parametrize("k_o", [128, 0])
def test_lossless_case_equals_numpy_matmul(k_o):
    """Whole Atom (FP) path on representable inputs: the reorder, shared exponents, E2M1 / E4M3
    codes and nibble packing are lossless, so decoding the oracle's codes with the spec table
    recovers X' exactly, and the oracle's output equals numpy's float64 matmul of the reordered
    operands (every product and partial sum is exact at these magnitudes)."""
    rng = np.random.default_rng(7 + k_o)
    M, N, K = 5, 12, 512
    xr, wr = _lossless_rows(rng, M, K, k_o), _lossless_rows(rng, N, K, k_o)
    perm = rng.permutation(K).astype(np.int32)
    X = np.zeros_like(xr)
    W = np.zeros_like(wr)
    X[:, perm], W[:, perm] = xr, wr                      # x'[j] = x[perm[j]]
    X16, W16 = X.astype(np.float16), W.astype(np.float16)
    assert np.array_equal(X16.astype(np.float64), X)
    a = oracle.mx_quantize_rows(X16, perm, K, k_o)
    w = oracle.mx_quantize_rows(W16, perm, K, k_o)
    # independent decode of the packed bytes (low nibble = even channel) with the spec table
    def decode(q, r):
        f4, f8, se = q
        K4 = K - k_o
        out = np.zeros(K)
        for j in range(K):
            X_ = 2.0 ** (int(se[r, j // 32]) - 127)
            if j < K4:
                nib = (f4[r, j // 2] >> (4 * (j & 1))) & 15
                out[j] = X_ * (-1 if nib & 8 else 1) * E2M1_SPEC[nib & 7]
            else:
                t = torch.tensor([f8[r, j - K4]], dtype=torch.uint8).view(torch.float8_e4m3fn)
                out[j] = X_ * float(t.float())
        return out
    for r in range(M):
        np.testing.assert_array_equal(decode(a, r), xr[r])
    c = oracle.mx_output_rows(a, w, M, N, K, k_o)
    np.testing.assert_array_equal(c, xr @ wr.T)


def test_quantization_error_bound_and_outlier_precision():
    """Round trip: every unsaturated element is within half a grid step of x / 2^s (RNE), and the
    E4M3 outlier blocks keep the injected outlier channels far more precisely than FP4 would."""
    M, K = 8, 1024
    X, _, perm = synth.problem(M, 128, K, seed=3)
    f4, f8, se = oracle.mx_quantize_rows(X, perm, K, 128)
    xr = X.astype(np.float64)[:, perm]
    g = np.array(E2M1_SPEC)
    K4 = K - 128
    for r in range(M):
        for j in range(0, K4, 7):
            s = 2.0 ** (int(se[r, j // 32]) - 127)
            v = abs(xr[r, j]) / s
            nib = (f4[r, j // 2] >> (4 * (j & 1))) & 15
            q = g[nib & 7]
            if v <= 6.0:
                step = np.diff(g)[min(np.searchsorted(g, v, side="right") - 1, 6)]
                assert abs(v - q) <= step / 2
            else:
                assert q == 6.0
    deq8 = np.array([[oracle.e4m3_value(int(c)) * 2.0 ** (int(se[r, (K4 + i) // 32]) - 127)
                      for i, c in enumerate(f8[r])] for r in range(M)])
    rel = np.abs(deq8 - xr[:, K4:]) / np.maximum(np.abs(xr[:, K4:]), 1e-3)
    assert np.median(rel) < 2 ** -4
