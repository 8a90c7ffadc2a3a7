"""GPU parity of the quantized KV cache + decode attention (NEXT-3, include/atom.h "KV cache")
against oracle/kv_oracle.c: bit-exact INT4 codes and (scale, min) parameters, and the attention
output within a tolerance derived from fp32 arithmetic.  Paper: P:284-291 (Section 4.4)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
P16 = 16


@pytest.fixture(scope="module")
def atom():
    import paper_2310_19102_b200 as a
    a.load()
    return a


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def build_cache(atom, rng, lens, H, perm_pages=True, scale=1.0):
    """Random K/V for every sequence, appended in random-size batches of tokens through the
    GPU quantizer, mirrored by the oracle; pages assigned through a (permuted) block table."""
    B = len(lens)
    max_pages = max((L + P16 - 1) // P16 for L in lens)
    npages = B * max_pages
    order = rng.permutation(npages) if perm_pages else np.arange(npages)
    bt = order.reshape(B, max_pages).astype(np.int32)
    kg, vg = atom.KvCache.empty(npages, H), atom.KvCache.empty(npages, H)
    ko = vo = None
    for b, L in enumerate(lens):
        k = (rng.normal(0, 1, (L, H * 128)) * scale).astype(np.float16)
        v = (rng.normal(0, 1, (L, H * 128)) * rng.uniform(0.1, 3, (L, 1))).astype(np.float16)
        slots = (bt[b][np.arange(L) // P16] * P16 + np.arange(L) % P16).astype(np.int32)
        t0 = 0
        while t0 < L:                                   # ragged appends (prefill + decode)
            t1 = min(L, t0 + int(rng.integers(1, 40)))
            atom.kv_quantize(dev(k[t0:t1]), dev(slots[t0:t1]), kg)
            atom.kv_quantize(dev(v[t0:t1]), dev(slots[t0:t1]), vg)
            t0 = t1
        ko = oracle.kv_quantize(k.reshape(L, H, 128), slots, npages, *(ko or (None, None)))
        vo = oracle.kv_quantize(v.reshape(L, H, 128), slots, npages, *(vo or (None, None)))
    return kg, vg, ko, vo, bt


@pytest.mark.parametrize("lens,H", [([1], 1), ([5, 16, 17], 2), ([300, 64, 1, 129], 4)])
def test_kv_quantize_bitexact(atom, lens, H):
    import torch
    rng = np.random.default_rng(len(lens) * 10 + H)
    kg, vg, ko, vo, bt = build_cache(atom, rng, lens, H)
    torch.cuda.synchronize()
    # only slots that were written are compared (untouched slots are zero on both sides)
    np.testing.assert_array_equal(kg.codes.cpu().numpy(), ko[0])
    np.testing.assert_array_equal(kg.params.cpu().numpy(), ko[1])
    np.testing.assert_array_equal(vg.codes.cpu().numpy(), vo[0])
    np.testing.assert_array_equal(vg.params.cpu().numpy(), vo[1])


def test_kv_quantize_adversarial(atom):
    """Constant vectors (s = 0), +-65504, fp16 subnormals, exact .5 ties of (x - min) / s."""
    import torch
    H = 2
    x = np.zeros((6, H * 128), dtype=np.float16)
    x[0] = 3.5
    x[1, ::2], x[1, 1::2] = 65504, -65504
    x[2] = (np.arange(H * 128) % 7 - 3) * 2.0 ** -24
    x[3] = np.arange(H * 128) % 16          # range 15: s = 1, integer codes
    x[4] = (np.arange(H * 128) % 31) * 0.5  # s = 1 with exact .5 ties
    x[5, :128] = -0.0
    slots = np.array([0, 3, 7, 8, 15, 16], dtype=np.int32)
    g = atom.KvCache.empty(2, H)
    atom.kv_quantize(dev(x), dev(slots), g)
    torch.cuda.synchronize()
    o = oracle.kv_quantize(x.reshape(6, H, 128), slots, 2)
    np.testing.assert_array_equal(g.codes.cpu().numpy(), o[0])
    np.testing.assert_array_equal(g.params.cpu().numpy(), o[1])


def assert_attention_close(got, ref, vmax, what):
    # fp32 arithmetic: dot products of 128 terms, softmax over L <= 4096, weighted sums; the
    # error stays below ~1e-5 of the value scale; 1e-4 leaves a 10x margin
    tol = 1e-4 * vmax + 1e-4 * np.abs(ref)
    err = np.abs(got - ref)
    assert np.all(err <= tol), f"{what}: max err/tol {(err / tol).max()}"


@pytest.mark.parametrize("lens,H", [([1], 2), ([16, 17, 5], 4), ([700, 64, 1, 129], 4),
                                    ([2048, 33], 2)])
def test_decode_attention_vs_oracle(atom, lens, H):
    import torch
    rng = np.random.default_rng(sum(lens) + H)
    kg, vg, ko, vo, bt = build_cache(atom, rng, lens, H)
    q = rng.normal(0, 1, (len(lens), H, 128)).astype(np.float16)
    out = atom.decode_attention(dev(q), kg, vg, dev(bt), dev(np.array(lens, np.int32)),
                                max(lens))
    torch.cuda.synchronize()
    ref = oracle.decode_attention(q, ko, vo, bt, np.array(lens, np.int32))
    vmax = np.abs(vo[1]).max() + 15 * np.abs(vo[1][..., 0]).max()
    assert_attention_close(out.cpu().numpy(), ref, vmax, f"lens={lens}")


def test_decode_attention_singleton_and_peaked(atom):
    """A single cached token returns its dequantized value; large-scale keys (a peaked softmax)
    stay within tolerance."""
    import torch
    rng = np.random.default_rng(5)
    lens = [1, 300]
    kg, vg, ko, vo, bt = build_cache(atom, rng, lens, 2, scale=8.0)
    q = (rng.normal(0, 1, (2, 2, 128)) * 4).astype(np.float16)
    out = atom.decode_attention(dev(q), kg, vg, dev(bt), dev(np.array(lens, np.int32)), 300)
    torch.cuda.synchronize()
    ref = oracle.decode_attention(q, ko, vo, bt, np.array(lens, np.int32))
    vmax = np.abs(vo[1]).max() + 15 * np.abs(vo[1][..., 0]).max()
    assert_attention_close(out.cpu().numpy(), ref, vmax, "peaked")
