"""Pins of the KV-cache oracle (oracle/kv_oracle.c, NEXT-3) to things other than itself: the
round-trip bound of asymmetric rounding, the degenerate (constant) vector, the exact extremes,
the singleton softmax, torch's scaled_dot_product_attention (a library routine) on the
dequantized cache in float64, paging invariance and power-of-two linearity in V.

Paper: P:284-288 (Section 4.4) -- asymmetric low-bit KV quantization "with the granularity of
attention head", dequantized on load before the attention; PageAttention.  Readings
G25-G28."""
import numpy as np
import pytest
import torch

import oracle

P16 = oracle.KV_PAGE


def dequant(codes, params, page, h, off):
    c = codes[page, h, off]
    q = np.empty(c.size * 2)
    q[0::2], q[1::2] = c & 15, c >> 4
    s, mn = params[page, h, off]
    return q * np.float64(s) + np.float64(mn), q


def test_quantize_round_trip_and_extremes():
    rng = np.random.default_rng(0)
    T, H, d = 37, 3, 128
    x = (rng.normal(0, 1, (T, H, d)) * rng.uniform(0.01, 50, (T, H, 1))).astype(np.float16)
    codes, params = oracle.kv_quantize(x, np.arange(T), 3)
    for t in range(T):
        for h in range(H):
            deq, q = dequant(codes, params, t // P16, h, t % P16)
            v = x[t, h].astype(np.float64)
            s = np.float64(params[t // P16, h, t % P16, 0])
            assert q.min() >= 0 and q.max() <= 15
            assert q[np.argmin(v)] == 0 and q[np.argmax(v)] == 15   # range maps onto [0, 15]
            assert params[t // P16, h, t % P16, 1] == v.min()        # min stored exactly
            # asymmetric RNE: |x - deq| <= s/2 plus binary32 rounding of (x - mn) * (1/s)
            assert np.all(np.abs(v - deq) <= s * (0.5 + 2.0 ** -18) + 1e-7 * np.abs(v))


def test_constant_vector_dequantizes_exactly():
    x = np.full((2, 1, 128), -3.25, dtype=np.float16)
    x[1] = 0
    codes, params = oracle.kv_quantize(x, np.array([0, 5]), 1)
    for off in (0, 5):
        deq, q = dequant(codes, params, 0, 0, off)
        assert params[0, 0, off, 0] == 0.0 and np.all(q == 0)
        np.testing.assert_array_equal(deq, x[0 if off == 0 else 1, 0].astype(np.float64))


def _cache(rng, B, H, d, lens, perm_pages=False):
    max_pages = max((L + P16 - 1) // P16 for L in lens)
    npages = B * max_pages
    k = rng.normal(0, 1, (B, max_pages * P16, H, d)).astype(np.float16)
    v = rng.normal(0, 1, (B, max_pages * P16, H, d)).astype(np.float16)
    order = rng.permutation(npages) if perm_pages else np.arange(npages)
    bt = order.reshape(B, max_pages).astype(np.int32)
    kc = vc = None
    for b in range(B):
        slots = bt[b][np.arange(lens[b]) // P16] * P16 + np.arange(lens[b]) % P16
        kc = oracle.kv_quantize(k[b, :lens[b]], slots, npages, *(kc or (None, None)))
        vc = oracle.kv_quantize(v[b, :lens[b]], slots, npages, *(vc or (None, None)))
    return kc, vc, bt, np.array(lens, dtype=np.int32)


def test_singleton_softmax_returns_value():
    rng = np.random.default_rng(1)
    kc, vc, bt, sl = _cache(rng, 1, 2, 128, [1])
    q = rng.normal(0, 1, (1, 2, 128)).astype(np.float16)
    out = oracle.decode_attention(q, kc, vc, bt, sl)
    for h in range(2):
        np.testing.assert_array_equal(out[0, h], dequant(*vc, bt[0, 0], h, 0)[0])


@pytest.mark.parametrize("lens", [[1, 16, 17, 63], [200, 5]])
def test_equals_torch_sdpa_on_dequantized_cache(lens):
    rng = np.random.default_rng(len(lens))
    B, H, d = len(lens), 3, 128
    kc, vc, bt, sl = _cache(rng, B, H, d, lens, perm_pages=True)
    q = rng.normal(0, 1, (B, H, d)).astype(np.float16)
    out = oracle.decode_attention(q, kc, vc, bt, sl)
    for b, L in enumerate(lens):
        K = np.stack([[dequant(*kc, bt[b, t // P16], h, t % P16)[0] for t in range(L)]
                      for h in range(H)])
        V = np.stack([[dequant(*vc, bt[b, t // P16], h, t % P16)[0] for t in range(L)]
                      for h in range(H)])
        ref = torch.nn.functional.scaled_dot_product_attention(
            torch.from_numpy(q[b].astype(np.float64))[:, None, :], torch.from_numpy(K),
            torch.from_numpy(V))[:, 0, :].numpy()
        np.testing.assert_allclose(out[b], ref, rtol=1e-12, atol=1e-12)


def test_paging_invariance_and_value_linearity():
    rng = np.random.default_rng(3)
    lens = [40, 33]
    q = rng.normal(0, 1, (2, 2, 128)).astype(np.float16)
    r1 = _cache(np.random.default_rng(9), 2, 2, 128, lens, perm_pages=False)
    r2 = _cache(np.random.default_rng(9), 2, 2, 128, lens, perm_pages=True)
    o1 = oracle.decode_attention(q, *r1)
    o2 = oracle.decode_attention(q, *r2)
    np.testing.assert_array_equal(o1, o2)
    # V -> 4 V: scales and mins exactly x4, codes identical, output exactly x4
    kc, vc, bt, sl = r1
    vc4 = (vc[0], vc[1] * 4)
    np.testing.assert_array_equal(oracle.decode_attention(q, kc, vc4, bt, sl), 4 * o1)
