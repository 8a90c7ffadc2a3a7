"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bars (BASELINE north_star): packed INT4/INT8 codes, scales and per-group int32 partials
bit-exact; fp16 output within 2^-10 absolute + 1e-3 relative of the oracle's double result.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

ATOL, RTOL = 2.0 ** -10, 1e-3


@pytest.fixture(scope="module")
def atom():
    import torch
    import paper_2310_19102_b200 as atom
    from paper_2310_19102_b200 import build
    build.build()
    atom.load()
    torch.cuda.init()
    return atom


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return None if t is None else t.cpu().numpy()


def assert_close_tol(c_gpu, c_ref, what=""):
    c = c_gpu.astype(np.float64)
    err = np.abs(c - c_ref)
    tol = ATOL + RTOL * np.abs(c_ref)
    bad = err > tol
    assert not bad.any(), (f"{what}: {bad.sum()} outputs out of tolerance, max err/tol "
                           f"{np.max(err / tol):.3f}")
    return float(np.max(err / tol))


def quant_both(atom, x, perm, K, k_o, clip4, weights=False):
    fn = atom.quantize_weights if weights else atom.reorder_quantize
    q = fn(dev(x), dev(perm), K=K, k_outlier=k_o, clip_int4=clip4)
    o4, o8, osc = oracle.quantize_rows(x, perm, K, k_o, clip4, 1.0)
    return q, (o4, o8, osc)


def codes_from_packed(o4):
    """Signed INT4 codes [rows][K - k_o] from packed two's-complement nibbles (low = even)."""
    lo = (o4 & 0xF).astype(np.int16)
    hi = (o4 >> 4).astype(np.int16)
    codes = np.empty((o4.shape[0], o4.shape[1] * 2), dtype=np.int16)
    codes[:, 0::2], codes[:, 1::2] = lo, hi
    return np.where(codes >= 8, codes - 16, codes)


def f8_from_packed(o4, o8, osc):
    """The GEMM operand form (include/atom.h "a_f8", "a_ab") rebuilt from the oracle's packed
    codes and scales with plain index arithmetic, independent of the kernels: INT4 code q as the
    E4M3 byte of q * 2^-9 (q, or 0x80 | -q when negative); within each 32-channel chunk byte
    16h + 4i + b holds channel 8i + 2b + h; the INT8 outlier group copied as is.  a_ab: per
    token and group (s * 2^18, fl32(fl32(-8 ca) * s)) for INT4 groups (ca = the group's code
    sum), (s, 0) for the outlier group, token 32b + r at position 32b + 4 (r % 8) + r / 8."""
    rows = o4.shape[0] if o4.size else o8.shape[0]
    parts, sums = [], []
    if o4.size:
        codes = codes_from_packed(o4)
        p = np.arange(codes.shape[1])
        c, r = (p % 128) // 32, p % 32
        h, i, b = r // 16, (r % 16) // 4, r % 4
        src = (p // 128) * 128 + 32 * c + 8 * i + 2 * b + h
        q = codes[:, src]
        parts.append(np.where(q < 0, 0x80 | (-q), q).astype(np.uint8))
        sums.append(codes.reshape(rows, -1, 128).sum(axis=2).T)
    G = osc.shape[0]
    G4 = len(sums[0]) if sums else 0
    if o8 is not None:
        parts.append(o8.view(np.uint8))
    ab = np.zeros((G, rows, 2), np.float32)
    for t in range(G):
        s = osc[t].astype(np.float32)
        if t < G4:
            ab[t, :, 0] = s * np.float32(262144.0)
            ab[t, :, 1] = (-8 * sums[0][t]).astype(np.float32) * s   # float(-8 ca): +0 for ca = 0
        else:
            ab[t, :, 0] = s
    pos = np.arange(rows)
    pos = (pos - pos % 32) + 4 * (pos % 8) + (pos % 32) // 8
    return np.concatenate(parts, axis=1), ab, pos


def assert_quant_equal(q, ref):
    o4, o8, osc = ref
    if o4.size and q.q4 is not None:
        np.testing.assert_array_equal(host(q.q4), o4)
    if o8 is not None and q.q8 is not None:
        np.testing.assert_array_equal(host(q.q8), o8)
    if q.f8 is not None:
        f8, ab, pos = f8_from_packed(o4, o8, osc)
        np.testing.assert_array_equal(host(q.f8), f8)
        got_ab = host(q.ab)[:, pos, :]
        np.testing.assert_array_equal(got_ab.view(np.uint32), ab.view(np.uint32))
    got = host(q.scales)
    np.testing.assert_array_equal(got.view(np.uint32), osc.view(np.uint32))
    if q.sp is not None:   # weight scales in the GEMM channel order (include/atom.h "w_sp")
        n = np.arange(osc.shape[1])
        nl = n % 128
        k = nl // 8
        pos = (n - nl) + 32 * (k // 4) + 8 * ((nl % 8) // 2) + 2 * (k % 4) + nl % 2
        want = np.empty_like(osc)
        want[:, pos] = osc
        np.testing.assert_array_equal(host(q.sp).view(np.uint32), want.view(np.uint32))


# ----------------------------------------------------------------------------------------------
# a1 / a0: reorder + quantize, bit-exact
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("K", [1024, 4096, 5120, 8192, 11008])
@pytest.mark.parametrize("M", [1, 7, 8, 127, 128, 129, 256])
def test_reorder_quantize_bitexact(atom, M, K):
    x = synth.activations(M, K, seed=M + K)
    perm = synth.perm_for(K, seed=M + K)
    q, ref = quant_both(atom, x, perm, K, 128, 0.9)
    assert_quant_equal(q, ref)


@pytest.mark.parametrize("k_o", [0, 128])
@pytest.mark.parametrize("clip4", [0.9, 0.85, 1.0, 0.5])
def test_quantize_weights_bitexact(atom, k_o, clip4):
    N, K = 384, 1024
    w = synth.weights(N, K, seed=3)
    perm = synth.perm_for(K, seed=3, n_outliers=k_o)
    q, ref = quant_both(atom, w, perm, K, k_o, clip4, weights=True)
    assert_quant_equal(q, ref)


def test_quantize_11008_down_proj(atom):
    M, K = 64, 11008
    K = 11008                     # 86 groups
    x = synth.activations(M, K, seed=5)
    perm = synth.perm_for(K, seed=5)
    q, ref = quant_both(atom, x, perm, K, 128, 0.9)
    assert_quant_equal(q, ref)


def adversarial_rows(K):
    rows = []
    z = np.zeros(K, np.float16)
    rows.append(z.copy())                                     # all-zero row
    r = z.copy(); r[::128] = 3.0; rows.append(r)              # single nonzero per group
    r = np.full(K, 65504, np.float16); r[1::2] = -65504; rows.append(r)   # fp16 extremes
    rows.append(np.full(K, np.float16(2.0 ** -24)))           # fp16 subnormal
    r = z.copy(); r[7] = -5.0; rows.append(r)                 # negative group max
    # exact .5 ties with clip = 1: x = 7.5 s and 127.5 s  (s = 1)
    r = z.copy(); r[:K - 128] = np.tile(np.array([7.5, -7.5, 6.5, -6.5, 0.5, -0.5, 1.5, -2.5],
                                                 np.float16), (K - 128) // 8)
    r[K - 128:] = np.tile(np.array([127.5, -127.5, 0.5, -1.5], np.float16), 32)
    rows.append(r)
    rng = np.random.default_rng(0)
    rows.append((rng.standard_normal(K) * 1e-4).astype(np.float16))   # tiny values
    rows.append((rng.standard_normal(K) * 3e3).astype(np.float16))    # large values
    return np.stack(rows)


@pytest.mark.parametrize("clip4,clip8", [(0.9, 1.0), (1.0, 1.0)])
@pytest.mark.parametrize("perm_kind", ["identity", "reversal", "calibrated"])
def test_quantize_adversarial(atom, clip4, clip8, perm_kind):
    K = 1024
    x = adversarial_rows(K)
    perm = {"identity": np.arange(K), "reversal": np.arange(K)[::-1],
            "calibrated": synth.perm_for(K, 1)}[perm_kind].astype(np.int32)
    q = atom.reorder_quantize(dev(x), dev(perm), K=K, k_outlier=128, clip_int4=clip4,
                              clip_int8=clip8)
    ref = oracle.quantize_rows(x, perm, K, 128, clip4, clip8)
    assert_quant_equal(q, ref)


def test_quantize_shard_slice(atom):
    """K-shard: perm + k0, own K, k_outlier only on the tail shard; ldx > K."""
    M, K = 33, 2048
    x = synth.activations(M, K, seed=8)
    perm = synth.perm_for(K, seed=8)
    for k0, Ks, ko in [(0, 1024, 0), (1024, 1024, 128)]:
        sl = np.ascontiguousarray(perm[k0:k0 + Ks])
        q = atom.reorder_quantize(dev(x), dev(sl), K=Ks, k_outlier=ko)
        assert_quant_equal(q, oracle.quantize_rows(x, sl, Ks, ko, 0.9, 1.0))


def test_quantize_strided_rows(atom):
    """ldx > K with a row-strided view."""
    import torch
    M, K, ld = 20, 1024, 1536
    big = synth.activations(M, ld, seed=2)
    perm = synth.perm_for(K, seed=2)
    xt = dev(big)
    q = atom.reorder_quantize(xt, dev(perm), K=K)
    assert_quant_equal(q, oracle.quantize_rows(big, perm, K, 128, 0.9, 1.0))


# ----------------------------------------------------------------------------------------------
# NEXT-1: RMSNorm fused into reorder + quantize, bit-exact against oracle N1 + O2-O6
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("M,K,eps", [(1, 1024, 1e-6), (7, 4096, 1e-5), (130, 4096, 1e-6),
                                     (33, 8192, 0.0), (16, 11008, 1e-6)])
def test_rmsnorm_reorder_quantize_bitexact(atom, M, K, eps):
    rng = np.random.default_rng(M + K)
    x = synth.activations(M, K, seed=M + K)
    g = (1 + 0.1 * rng.standard_normal(K)).astype(np.float16)
    perm = synth.perm_for(K, seed=M + K)
    q = atom.rmsnorm_reorder_quantize(dev(x), dev(g), dev(perm), eps=eps)
    assert_quant_equal(q, oracle.rmsnorm_quantize_rows(x, g, perm, K, 128, eps))


def test_rmsnorm_fused_layer_output(atom):
    """Fused norm + quantize feeding the GEMM equals the oracle's norm -> quantized linear."""
    M, N, K = 64, 512, 2048
    X, W, perm = synth.problem(M, N, K, seed=11)
    g = (1 + 0.1 * np.random.default_rng(11).standard_normal(K)).astype(np.float16)
    pd = dev(perm)
    aq = atom.rmsnorm_reorder_quantize(dev(X), dev(g), pd)
    c = atom.w4a4_gemm(aq, atom.quantize_weights(dev(W), pd))
    ref = oracle.quantized_linear(oracle.rmsnorm_rows(X, g), perm, W, K)
    assert_close_tol(host(c.float()), ref["c"], "norm+W4A4")


@pytest.mark.parametrize("M,I", [(1, 1024), (7, 4096), (130, 11008), (33, 5120), (16, 28672)])
def test_silu_mul_reorder_quantize_bitexact(atom, M, I):
    """NEXT-4 piece: fused SwiGLU + reorder + quantize equals oracle N4 then O2-O6, bit for bit."""
    rng = np.random.default_rng(M + I)
    gate = synth.activations(M, I, seed=M + I)           # outlier channels included
    up = rng.standard_normal((M, I)).astype(np.float16)
    perm = synth.perm_for(I, seed=M + I)
    q = atom.silu_mul_reorder_quantize(dev(gate), dev(up), dev(perm))
    assert_quant_equal(q, oracle.silu_mul_quantize_rows(gate, up, perm, I))


def test_llama_mlp_w4a4_chain(atom):
    """A whole Llama MLP on the W4A4 path: gate / up GEMMs -> fused SwiGLU + quantize -> down
    GEMM.  The down projection's codes are bit-exact against the oracle fed with the GPU's fp16
    gate / up outputs, and its output is within the GEMM tolerance of the oracle's."""
    import torch
    M, H, I = 64, 1024, 2816
    X, Wg, perm_h = synth.problem(M, I, H, seed=41)
    Wu = synth.weights(I, H, 42)
    Wd = synth.weights(H, I, 43)
    perm_i = synth.perm_for(I, 44)
    ph, pi = dev(perm_h), dev(perm_i)
    xq = atom.reorder_quantize(dev(X), ph)
    g = atom.w4a4_gemm(xq, atom.quantize_weights(dev(Wg), ph))
    u = atom.w4a4_gemm(xq, atom.quantize_weights(dev(Wu), ph))
    hq = atom.silu_mul_reorder_quantize(g, u, pi)
    wdq = atom.quantize_weights(dev(Wd), pi)
    y = atom.w4a4_gemm(hq, wdq)
    torch.cuda.synchronize()
    gh, uh = host(g), host(u)
    ref_q = oracle.silu_mul_quantize_rows(gh, uh, perm_i, I)
    assert_quant_equal(hq, ref_q)
    w4, w8, wsc = oracle.quantize_rows(Wd, perm_i, I, 128, 0.85, 1.0)
    ref = oracle.output_rows(*ref_q, w4, w8, wsc, M, H, I, 128, np.arange(M))
    assert_close_tol(host(y.float()), ref, "MLP down")


# ----------------------------------------------------------------------------------------------
# a2-a5: GEMM -- exact partials (debug mode) and tolerance outputs
# ----------------------------------------------------------------------------------------------
def run_gemm(atom, X, W, perm, K, k_o, debug=False, out_dtype=None, canonical=False):
    import torch
    pd = dev(perm)
    wq = atom.quantize_weights(dev(W), pd, K=K, k_outlier=k_o)
    aq = atom.reorder_quantize(dev(X), pd, K=K, k_outlier=k_o)
    dbg = torch.full((K // 128, X.shape[0], W.shape[0]), -7, dtype=torch.int32,
                     device="cuda") if debug else None
    c = atom.w4a4_gemm(aq, wq, debug_partials=dbg, out_dtype=out_dtype, canonical=canonical)
    torch.cuda.synchronize()
    return aq, wq, c, dbg


@pytest.mark.parametrize("M,N,K,k_o", [
    (1, 128, 128, 128),      # single INT8 group (textbook W8A8)
    (7, 128, 256, 128),
    (16, 256, 1024, 128),    # config 1 geometry (N reduced)
    (33, 128, 512, 0),       # pure INT4 (k_o = 0)
    (100, 256, 384, 128),
    (129, 128, 1024, 128),   # ragged token tail across two tiles
    (256, 256, 1024, 128),
    (300, 384, 640, 128),
    (512, 1536, 2048, 128),  # BT = 256, all tiles stream-K split (24 tiles, 148 CTAs)
    (1024, 3200, 1152, 128), # data-parallel waves + stream-K tail, ragged K split points
    (40, 11008, 640, 0),     # BT = 64, many n-tiles, pure INT4, tail segments
])
@pytest.mark.parametrize("canonical", [False, True])
def test_gemm_partials_bitexact(atom, M, N, K, k_o, canonical):
    X, W, perm = synth.problem(M, N, K, seed=M * 7 + N, k_outlier=k_o)
    aq, wq, c, dbg = run_gemm(atom, X, W, perm, K, k_o, debug=True, canonical=canonical)
    ref = oracle.quantized_linear(X, perm, W, K, k_o)
    np.testing.assert_array_equal(host(dbg), ref["partials"])
    assert_close_tol(host(c.float()), ref["c"], "C")
    # the production kernel (no debug stores) gives the same output bits
    c2 = atom.w4a4_gemm(aq, wq, canonical=canonical)
    assert __import__("torch").equal(c, c2)


@pytest.mark.parametrize("M,N,K,k_o", [
    (1, 384, 1024, 128),     # swap-AB kBT = 16
    (16, 256, 640, 128),
    (17, 640, 1152, 0),      # kBT = 32, pure INT4
    (32, 11008, 512, 128),   # kBT = 32, many channel tiles, stream-K segments
    (33, 384, 4096, 128),    # kBT = 64
    (64, 4096, 1408, 128),   # kBT = 64, ragged stream-K split points
])
def test_gemm_small_m_swap_partials_bitexact(atom, M, N, K, k_o):
    """The small-M swap-AB tiles (weights on the MMA M side, kBT = 16/32/64 tokens): every exact
    group partial, the output within tolerance, and the production kernel's bits equal to the
    debug kernel's."""
    X, W, perm = synth.problem(M, N, K, seed=M * 11 + K, k_outlier=k_o)
    aq, wq, c, dbg = run_gemm(atom, X, W, perm, K, k_o, debug=True)
    ref = oracle.quantized_linear(X, perm, W, K, k_o)
    np.testing.assert_array_equal(host(dbg), ref["partials"])
    assert_close_tol(host(c.float()), ref["c"], "C")
    assert __import__("torch").equal(c, atom.w4a4_gemm(aq, wq))


def test_gemm_split_free_same_chain_every_tile(atom):
    """Split-free outputs are one fp32 chain per output (groups ascending, h = fma(P', alpha,
    beta), acc = fma(s_w, h, acc)) in both epilogues: the same token rows computed inside a
    16-, 32-, 64-token swap-AB tile and a 128-token tile give identical bits."""
    import torch
    N, K = 1024, 2048
    X, W, perm = synth.problem(200, N, K, seed=5)
    pd = dev(perm)
    wq = atom.quantize_weights(dev(W), pd)
    full = atom.w4a4_gemm(atom.reorder_quantize(dev(X), pd), wq, split_free=True)
    for m in (5, 16, 30, 64):
        sub = atom.w4a4_gemm(atom.reorder_quantize(dev(X[:m]), pd), wq, split_free=True)
        torch.cuda.synchronize()
        assert torch.equal(sub, full[:m]), m


def test_gemm_canonical_equals_operand_form(atom):
    """atom_w4a4_gemm on the packed codes (expanded on the device) and atom_w4a4_gemm_f8 on the
    quantizer's operand form give identical bits; so does the oracle's packed activation bytes
    fed straight into the canonical entry."""
    import torch
    M, N, K = 200, 1024, 2048
    X, W, perm = synth.problem(M, N, K, seed=17)
    pd = dev(perm)
    wq = atom.quantize_weights(dev(W), pd)
    aq = atom.reorder_quantize(dev(X), pd)
    c_f8 = atom.w4a4_gemm(aq, wq)
    c_can = atom.w4a4_gemm(aq, wq, canonical=True)
    a4, a8, asc = oracle.quantize_rows(X, perm, K, 128, 0.9, 1.0)
    ora = atom.Quantized(dev(a4), dev(a8), dev(asc), K, 128)
    c_ora = atom.w4a4_gemm(ora, wq)
    w4, w8, wsc = oracle.quantize_rows(W, perm, K, 128, 0.85, 1.0)
    c_ora2 = atom.w4a4_gemm(ora, atom.Quantized(dev(w4), dev(w8), dev(wsc), K, 128))
    assert torch.equal(c_ora, c_ora2)
    torch.cuda.synchronize()
    assert torch.equal(c_f8, c_can) and torch.equal(c_f8, c_ora)
    assert_close_tol(host(c_f8.float()), oracle.quantized_linear(X, perm, W, K)["c"], "C")


@pytest.mark.parametrize("M", [1, 8, 16, 31, 64, 127, 128, 129, 256, 513])
def test_gemm_output_config1_family(atom, M):
    N, K = 1024, 1024
    X, W, perm = synth.problem(M, N, K, seed=M)
    _, _, c, _ = run_gemm(atom, X, W, perm, K, 128)
    ref = oracle.quantized_linear(X, perm, W, K)
    assert_close_tol(host(c.float()), ref["c"], f"M={M}")


@pytest.mark.parametrize("M", [1, 16, 33, 40, 64, 100, 300, 1024])
def test_gemm_unit_scale_exact_integer(atom, M):
    """P3 on the GPU, production kernel (no debug stores), fp32 output: clip 1 and integer-valued
    groups -> C is the exact integer GEMM (every split / tile path must be exact)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).parent))
    from test_oracle_pins import scatter, unit_scale_block
    rng = np.random.default_rng(M)
    N, K = 768, 1024
    perm = rng.permutation(K).astype(np.int32)
    av, ac = unit_scale_block(rng, M, K, 128)
    wv, wc = unit_scale_block(rng, N, K, 128)
    X, W = scatter(av, perm).astype(np.float16), scatter(wv, perm).astype(np.float16)
    pd = dev(perm)
    wq = atom.quantize_weights(dev(W), pd, clip_int4=1.0)
    aq = atom.reorder_quantize(dev(X), pd, clip_int4=1.0)
    c = atom.w4a4_gemm(aq, wq, out_dtype=__import__("torch").float32)
    exact = (ac @ wc.T).astype(np.float64)
    assert np.abs(exact).max() < 2 ** 24
    np.testing.assert_array_equal(host(c).astype(np.float64), exact)


def test_gemm_fp32_output(atom):
    import torch
    M, N, K = 64, 256, 1024
    X, W, perm = synth.problem(M, N, K, seed=4)
    _, _, c, _ = run_gemm(atom, X, W, perm, K, 128, out_dtype=torch.float32)
    ref = oracle.quantized_linear(X, perm, W, K)
    # fp32 output: only accumulation-order error
    np.testing.assert_allclose(host(c), ref["c"], rtol=1e-5, atol=1e-5)


CONFIGS = {
    "cfg2_7b_qkvo": (256, 4096, 4096),
    "cfg3_up_m8": (8, 11008, 4096),
    "cfg3_up_m64": (64, 11008, 4096),
    "cfg3_up_m256": (256, 11008, 4096),
    "cfg3_down_m256": (256, 4096, 11008),
    "cfg3_up_m1024": (1024, 11008, 4096),
    "cfg4_13b": (512, 13824, 5120),
    "cfg5_70b_mlp": (1024, 28672, 8192),
}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_gemm_baseline_configs_sampled(atom, name):
    """Full BASELINE sizes in the launch configuration bench.py times: codes and scales in full,
    C in full for configs 1-4 and on 64 rows (first and last included) for the
    70B MLP, against the oracle."""
    M, N, K = CONFIGS[name]
    X, W, perm = synth.problem(M, N, K, seed=0)
    pd = dev(perm)
    wq = atom.quantize_weights(dev(W), pd)
    aq = atom.reorder_quantize(dev(X), pd)
    c = atom.w4a4_gemm(aq, wq)
    w4, w8, ws = oracle.quantize_rows(W, perm, K, 128, 0.85, 1.0)
    a4, a8, as_ = oracle.quantize_rows(X, perm, K, 128, 0.9, 1.0)
    assert_quant_equal(wq, (w4, w8, ws))
    assert_quant_equal(aq, (a4, a8, as_))
    rng = np.random.default_rng(123)
    if M * N * K <= 5e10:
        rows = np.arange(M)
    else:
        rows = np.unique(np.concatenate([[0, M - 1], rng.choice(np.arange(1, M - 1), 62,
                                                                  replace=False)]))
    ref = oracle.output_rows(a4, a8, as_, w4, w8, ws, M, N, K, 128, rows)
    assert_close_tol(host(c.float())[rows], ref, name)


def test_workspace_shared_across_shapes_and_self_cleaning(atom):
    """One workspace serves every shape: after each call its counter region is zero again, and
    alternating shapes (different tiles, different split points) reproduces fresh results."""
    import torch
    shapes = [(256, 4096, 4096), (8, 11008, 4096), (64, 1024, 2048), (256, 4096, 4096)]
    nbytes = max(atom.workspace_size(M, N, K) for M, N, K in shapes)
    assert nbytes > 0
    ws = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    cb = atom.counter_bytes()
    for M, N, K in shapes:
        X, W, perm = synth.problem(M, N, K, seed=M + N)
        pd = dev(perm)
        wq = atom.quantize_weights(dev(W), pd)
        aq = atom.reorder_quantize(dev(X), pd)
        got = atom.w4a4_gemm(aq, wq, workspace=ws)
        fresh = atom.w4a4_gemm(aq, wq, workspace=torch.zeros_like(ws))
        torch.cuda.synchronize()
        assert torch.equal(got, fresh), (M, N, K)
        assert int(ws[:cb].count_nonzero()) == 0, (M, N, K)


# ----------------------------------------------------------------------------------------------
# tensor-parallel shard algebra on one device (the "fake backend" of SURVEY §4 T3)
# ----------------------------------------------------------------------------------------------
def test_n_shard_columns(atom):
    """Column shards written in place (ldc > N) assemble the unsharded output.  Each shard is its
    own GEMM with its own schedule, so the fp32 accumulation may be split at other K points than
    in the full GEMM: equal within the BASELINE tolerance, bit-identical to the same shard run
    alone (deterministic)."""
    import torch
    M, N, K, P = 96, 1024, 2048, 4
    X, W, perm = synth.problem(M, N, K, seed=6)
    pd = dev(perm)
    aq = atom.reorder_quantize(dev(X), pd)
    out = torch.empty((M, N), dtype=torch.float16, device="cuda")
    alone = []
    for r in range(P):
        sl = slice(r * N // P, (r + 1) * N // P)
        wq = atom.quantize_weights(dev(W[sl]), pd)
        atom.w4a4_gemm(aq, wq, out=out[:, sl])
        alone.append(atom.w4a4_gemm(aq, wq))
    torch.cuda.synchronize()
    for r in range(P):
        sl = slice(r * N // P, (r + 1) * N // P)
        assert torch.equal(out[:, sl], alone[r])
    ref = oracle.quantized_linear(X, perm, W, K)
    assert_close_tol(host(out.float()), ref["c"], "N-shard")


@pytest.mark.parametrize("M,N,K,P", [(96, 1024, 2048, 2), (200, 1536, 1024, 3),
                                     (1024, 28672, 8192, 4), (512, 13824, 5120, 2)])
def test_n_shard_bit_identical_split_free(atom, M, N, K, P):
    """with ATOM_GEMM_SPLIT_FREE every output is the same fp32 chain (groups
    ascending) whatever the tile schedule, so column shards written into place reproduce the
    unsharded GEMM on one GPU bit for bit (the default stream-K schedule splits tiles at
    shape-dependent K points: equal there only within the tolerance, test_n_shard_columns)."""
    import torch
    X, W, perm = synth.problem(M, N, K, seed=P)
    pd = dev(perm)
    aq = atom.reorder_quantize(dev(X), pd)
    full = atom.w4a4_gemm(aq, atom.quantize_weights(dev(W), pd), split_free=True)
    out = torch.empty_like(full)
    nb = N // 128
    for r in range(P):
        sl = slice(128 * (r * nb // P), 128 * ((r + 1) * nb // P))
        wq = atom.quantize_weights(dev(W[sl]), pd)
        atom.w4a4_gemm(aq, wq, out=out[:, sl], split_free=True)
    torch.cuda.synchronize()
    assert torch.equal(out, full)
    dflt = atom.w4a4_gemm(aq, atom.quantize_weights(dev(W), pd))
    rows = np.unique(np.concatenate([[0, M - 1], np.random.default_rng(P).integers(0, M, 6)]))
    a4, a8, asc = oracle.quantize_rows(X, perm, K, 128, 0.9, 1.0)
    w4, w8, wsc = oracle.quantize_rows(W, perm, K, 128, 0.85, 1.0)
    ref = oracle.output_rows(a4, a8, asc, w4, w8, wsc, M, N, K, 128, rows)
    assert_close_tol(host(full.float())[rows], ref, "split-free")
    assert_close_tol(host(dflt.float())[rows], ref, "stream-K")


def test_gemm_cuda_graph_replay(atom):
    """The GEMM (and the quantize kernel) captured in a CUDA graph and replayed: identical to
    eager launches (the split-tile counters are self-cleaning, so replays need no memset)."""
    import torch
    M, N, K = 320, 2048, 2048
    X, W, perm = synth.problem(M, N, K, seed=23)
    pd = dev(perm)
    xd = dev(X)
    wq = atom.quantize_weights(dev(W), pd)
    aq = atom.reorder_quantize(xd, pd)
    eager = atom.w4a4_gemm(aq, wq).clone()
    out = torch.empty_like(eager)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        atom.w4a4_gemm(aq, wq, out=out, stream=s)       # workspace for this stream
        with torch.cuda.graph(g, stream=s):
            atom.reorder_quantize(xd, pd, out=aq, stream=s)
            atom.w4a4_gemm(aq, wq, out=out, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, eager)


def test_pdl_back_to_back_reuse(atom):
    """Kernels are launched with programmatic dependent launch: a chain of weight quantize ->
    GEMM -> activation quantize (overwriting the GEMM's operand buffer) -> GEMM on one stream with
    no host synchronisation must equal the same calls synchronised one by one."""
    import torch
    M, N, K = 96, 1536, 2048
    X1, W, perm = synth.problem(M, N, K, seed=31)
    X2 = synth.activations(M, K, 32)
    pd = dev(perm)
    x1, x2, wd = dev(X1), dev(X2), dev(W)
    # reference: every call synchronised
    wq_ref = atom.quantize_weights(wd, pd)
    torch.cuda.synchronize()
    ref = []
    for x in (x1, x2):
        aq = atom.reorder_quantize(x, pd)
        torch.cuda.synchronize()
        ref.append(atom.w4a4_gemm(aq, wq_ref).clone())
        torch.cuda.synchronize()
    # chained: the weights are written by the kernel right before the first GEMM, and the second
    # quantize rewrites the operand buffer the first GEMM reads
    for _ in range(3):
        wq = atom.quantize_weights(wd, pd)
        aq = atom.reorder_quantize(x1, pd)
        c1 = atom.w4a4_gemm(aq, wq)
        atom.reorder_quantize(x2, pd, out=aq)
        c2 = atom.w4a4_gemm(aq, wq)
        torch.cuda.synchronize()
        assert torch.equal(c1, ref[0]) and torch.equal(c2, ref[1])


def test_gemm_fp32_split_into_wide_buffer(atom):
    """fp32 partial output of a split-tile shape written as a column block of a wider buffer."""
    import torch
    M, N, K = 200, 1024, 3072
    X, W, perm = synth.problem(M, N, K, seed=29)
    pd = dev(perm)
    aq = atom.reorder_quantize(dev(X), pd)
    wq = atom.quantize_weights(dev(W), pd)
    big = torch.full((M, N + 256), 7.0, dtype=torch.float32, device="cuda")
    atom.w4a4_gemm(aq, wq, out=big[:, 128:128 + N])
    torch.cuda.synchronize()
    ref = oracle.quantized_linear(X, perm, W, K)
    np.testing.assert_allclose(host(big[:, 128:128 + N]), ref["c"], rtol=1e-5, atol=1e-5)
    assert torch.all(big[:, :128] == 7.0) and torch.all(big[:, 128 + N:] == 7.0)


def test_gemm_deterministic(atom):
    """Split-K reductions sum the partials in split order: repeated calls are bit-identical."""
    import torch
    for M, N, K in [(16, 1024, 1024), (256, 4096, 4096), (40, 512, 2048)]:
        X, W, perm = synth.problem(M, N, K, seed=M)
        pd = dev(perm)
        aq = atom.reorder_quantize(dev(X), pd)
        wq = atom.quantize_weights(dev(W), pd)
        outs = [atom.w4a4_gemm(aq, wq) for _ in range(4)]
        torch.cuda.synchronize()
        for o in outs[1:]:
            assert torch.equal(o, outs[0]), (M, N, K)


def test_k_shard_partials_and_sum(atom):
    import torch
    M, N, K, P = 64, 512, 2048, 2
    X, W, perm = synth.problem(M, N, K, seed=7)
    ref = oracle.quantized_linear(X, perm, W, K)
    G = K // 128
    acc = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    for r in range(P):
        g0, g1 = r * G // P, (r + 1) * G // P
        sl = np.ascontiguousarray(perm[g0 * 128:g1 * 128])
        ko = 128 if r == P - 1 else 0
        Ks = (g1 - g0) * 128
        pd = dev(sl)
        aq = atom.reorder_quantize(dev(X), pd, K=Ks, k_outlier=ko)
        wq = atom.quantize_weights(dev(W), pd, K=Ks, k_outlier=ko)
        dbg = torch.empty((g1 - g0, M, N), dtype=torch.int32, device="cuda")
        part = atom.w4a4_gemm(aq, wq, out_dtype=torch.float32, debug_partials=dbg)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(host(dbg), ref["partials"][g0:g1])
        acc += part
    assert_close_tol(host(acc.half().float()), ref["c"], "K-shard sum")


# ----------------------------------------------------------------------------------------------
# ABI behaviour on the device
# ----------------------------------------------------------------------------------------------
def test_validate_perm(atom):
    import torch
    K = 1024
    assert atom.validate_perm(dev(synth.perm_for(K, 0)))
    bad = synth.perm_for(K, 0).copy()
    bad[3] = bad[4]
    assert not atom.validate_perm(dev(bad))
    assert atom.validate_perm(dev(np.arange(0, 2 * K, 2, dtype=np.int32)), ldx=2 * K)


def test_non_default_stream(atom):
    import torch
    M, N, K = 64, 256, 1024
    X, W, perm = synth.problem(M, N, K, seed=10)
    ref = oracle.quantized_linear(X, perm, W, K)
    s = torch.cuda.Stream()
    xd, wd, pd = dev(X), dev(W), dev(perm)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        wq = atom.quantize_weights(wd, pd, stream=s)
        aq = atom.reorder_quantize(xd, pd, stream=s)
        c = atom.w4a4_gemm(aq, wq, stream=s)
    s.synchronize()
    assert_close_tol(host(c.float()), ref["c"], "stream")


def test_error_codes_launch_nothing(atom):
    import ctypes
    import torch
    L = atom.load()
    x = torch.zeros((4, 256), dtype=torch.float16, device="cuda")
    perm = torch.arange(256, dtype=torch.int32, device="cuda")
    q4 = torch.full((4, 64), 0xAB, dtype=torch.uint8, device="cuda")
    q8 = torch.full((4, 128), 5, dtype=torch.int8, device="cuda")
    sc = torch.full((2, 4), 3.0, dtype=torch.float32, device="cuda")
    f = ctypes.c_float
    cases = [
        (2, (x.data_ptr(), 4, 256, perm.data_ptr(), 200, 128, f(0.9), f(1.0))),   # K % 128
        (4, (x.data_ptr(), 4, 256, perm.data_ptr(), 256, 64, f(0.9), f(1.0))),    # k_o
        (4, (x.data_ptr(), 4, 256, perm.data_ptr(), 256, 128, f(0.0), f(1.0))),   # clip
        (1, (None, 4, 256, perm.data_ptr(), 256, 128, f(0.9), f(1.0))),           # null x
        (3, (x.data_ptr() + 2, 4, 256, perm.data_ptr(), 256, 128, f(0.9), f(1.0))),  # misaligned
    ]
    for want, args in cases:
        st = L.atom_reorder_quantize(*args, q4.data_ptr(), q8.data_ptr(), None, None,
                                     sc.data_ptr(), None)
        assert st == want, (want, st)
        assert atom.last_launch_count() == 0
    torch.cuda.synchronize()
    assert torch.all(q4 == 0xAB) and torch.all(q8 == 5) and torch.all(sc == 3.0)
    # GEMM: N % 128, ldc < N, bad dtype
    args = [q4.data_ptr(), q8.data_ptr(), sc.data_ptr(), q4.data_ptr(), q8.data_ptr(),
            sc.data_ptr()]   # canonical entry: a_q4, a_q8, a_scales, w_q4, w_q8, w_scales
    out = torch.zeros((4, 256), dtype=torch.float16, device="cuda")
    assert L.atom_w4a4_gemm(*args, 4, 200, 256, 128, out.data_ptr(), 256, 0, None, None, 0,
                            None) == 2
    assert L.atom_w4a4_gemm(*args, 4, 256, 256, 128, out.data_ptr(), 128, 0, None, None, 0,
                            None) == 2
    assert L.atom_w4a4_gemm(*args, 4, 128, 256, 128, out.data_ptr(), 256, 5, None, None, 0,
                            None) == 4
    assert L.atom_w4a4_gemm(*args, 4, 128, 256, 0, out.data_ptr(), 256, 0, None, None, 0,
                            None) == 1     # k_o = 0 but q8 pointers given
    torch.cuda.synchronize()
    assert torch.all(out == 0)


def test_empty_m_is_noop(atom):
    import torch
    L = atom.load()
    f = __import__("ctypes").c_float
    assert L.atom_reorder_quantize(None, 0, 256, None, 256, 128, f(0.9), f(1.0), None, None,
                                   None, None, None, None) == 0
    assert L.atom_w4a4_gemm(None, None, None, None, None, None, 0, 128, 256, 128, None, 128, 0,
                            None, None, 0, None) == 0
    assert L.atom_w4a4_gemm_f8(None, None, None, None, None, 0, 128, 256, 128, None, 128, 0,
                               None, 0, None, 0, None) == 0
