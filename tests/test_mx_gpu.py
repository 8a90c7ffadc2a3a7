"""GPU parity of Atom (FP) on the MX format (NEXT-2, include/atom.h "Atom (FP)") against the CPU
oracle oracle/mx_oracle.c: bit-exact E2M1 / E4M3 codes and UE8M0 scale bytes, the block-scaled
GEMM within the BASELINE tolerance, and an exact closed form.  Paper: P:540 (Section 6)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def atom():
    import paper_2310_19102_b200 as a
    a.load()
    return a


def dev(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    return t.cpu().numpy()


def assert_close_tol(got, ref, what):
    tol = 2.0 ** -10 + 1e-3 * np.abs(ref)
    err = np.abs(got.astype(np.float64) - ref)
    bad = err > tol
    assert not bad.any(), f"{what}: {bad.sum()} outside tolerance, max err/tol {(err / tol).max()}"


def check_quant(atom, X, perm, K, k_o):
    import torch
    q = atom.mx_quantize(dev(X), dev(perm), K=K, k_outlier=k_o)
    torch.cuda.synchronize()
    f4, f8, se = oracle.mx_quantize_rows(X, perm, K, k_o)
    if K > k_o:
        np.testing.assert_array_equal(host(q.fp4), f4)
    if k_o:
        np.testing.assert_array_equal(host(q.fp8), f8)
    np.testing.assert_array_equal(host(q.sf)[:, :K // 32], se)
    return q, (f4, f8, se)


@pytest.mark.parametrize("M,K,k_o", [(1, 128, 128), (7, 512, 128), (33, 1024, 0),
                                     (130, 4096, 128), (64, 11008, 128), (16, 8192, 128)])
def test_mx_quantize_bitexact(atom, M, K, k_o):
    X, _, perm = synth.problem(M, 128, K, seed=M + K, k_outlier=k_o)
    check_quant(atom, X, perm, K, k_o)


def test_mx_quantize_adversarial(atom):
    """Zero blocks (byte 0), +-65504, fp16 subnormals, exact E2M1 ties after scaling, negative
    zeros, and single-nonzero blocks."""
    rng = np.random.default_rng(0)
    K = 1024
    X = rng.normal(0, 1, (12, K)).astype(np.float16)
    X[0] = 0
    X[1, ::3] = 65504
    X[1, 1::3] = -65504
    X[2] = (rng.integers(-1023, 1024, K) * 2.0 ** -24).astype(np.float16)   # subnormals
    X[3] = np.tile(np.array([4, 5, 2.5, 0.25, 0.75, 1.25, 1.75, 3.5, 7, -5, -2.5, -0.25],
                            np.float16), K // 12 + 1)[:K]
    X[4] = -0.0
    X[5] = 0
    X[5, ::32] = -3.0
    X[6] = np.float16(2.0 ** -14)
    perm = rng.permutation(K).astype(np.int32)
    check_quant(atom, X, perm, K, 128)
    check_quant(atom, X, np.arange(K, dtype=np.int32), K, 128)


@pytest.mark.parametrize("M,N,K,k_o", [
    (1, 128, 128, 128),      # only the outlier (MXFP8) stage
    (16, 1024, 1024, 128),   # config 1 geometry
    (7, 640, 512, 128),      # odd FP4 chunk count (3), partial 224-channel tile
    (200, 896, 2048, 0),     # pure MXFP4, two token tiles
    (129, 1152, 1152, 128),  # ragged token tail
    (300, 4096, 4096, 128),  # config 2 shape family
    (512, 13824, 5120, 128), # config 4: 256-token tiles (two MMA halves), ragged channel tile
    (1000, 28672, 1024, 128),  # 256-token tiles, ragged token tail
    (8, 4096, 11008, 128),   # split-K over 7 CTAs per tile (19 tiles), fp32 reduction
    (64, 11008, 4096, 0),    # split-K 2, pure MXFP4
    (1024, 28672, 256, 128),   # wave tail: 256-token tiles over 111 column tiles, then 128-token
    (4096, 4096, 512, 0),      # tiles over the rest (second launch); 18 + 1 column tiles
])
def test_mx_gemm_vs_oracle(atom, M, N, K, k_o):
    import torch
    X, W, perm = synth.problem(M, N, K, seed=M * 3 + N, k_outlier=k_o)
    a, ra = check_quant(atom, X, perm, K, k_o)
    w, rw = check_quant(atom, W, perm, K, k_o)
    c = atom.mx_gemm(a, w)
    torch.cuda.synchronize()
    rows = np.arange(M) if M * N * K <= 2 ** 31 else \
        np.unique(np.concatenate([[0, M - 1], np.random.default_rng(M).integers(0, M, 30)]))
    ref = oracle.mx_output_rows(ra, rw, M, N, K, k_o, rows)
    assert_close_tol(host(c.float())[rows], ref, "C")


def test_mx_gemm_full_size_sampled(atom):
    """BASELINE config 5 (Llama-70B MLP) through the same launch configuration bench.py times:
    64 sampled token rows (first and last included) against the oracle."""
    import torch
    M, N, K = 1024, 28672, 8192
    X = synth.activations(M, K, 0)
    perm = synth.perm_for(K, 0)
    W = synth.weights(N, K, 0)
    a = atom.mx_quantize(dev(X), dev(perm))
    w = atom.mx_quantize(dev(W), dev(perm))
    c = atom.mx_gemm(a, w)
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([[0, M - 1], np.random.default_rng(5).integers(0, M, 62)]))
    ra = (host(a.fp4)[rows], host(a.fp8)[rows], host(a.sf)[rows, :K // 32])
    fa = oracle.mx_quantize_rows(X[rows], perm, K, 128)
    for g, r in zip(ra, fa):
        np.testing.assert_array_equal(g, r)
    rw = (host(w.fp4), host(w.fp8), np.ascontiguousarray(host(w.sf)[:, :K // 32]))
    ref = oracle.mx_output_rows(fa, rw, rows.size, N, K, 128)
    assert_close_tol(host(c.float())[rows], ref, "C cfg5")


def _exact_rows(rng, rows, K, k_o):
    """Rows the MX conversion represents losslessly and whose GEMM is exact in fp32: E2M1 blocks
    = grid values * 2^s (s in [-1, 1]) with a +-4 * 2^s element (shared exponent s), E4M3 blocks
    = integers in [-15, 15] with a +-16 element (shared exponent -4: every k * 16 has <= 4
    significant bits).  Products are multiples of 2^-4 and every partial sum stays below 2^20."""
    grid = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    x = np.zeros((rows, K))
    for r in range(rows):
        for b in range(K // 32):
            if 32 * b < K - k_o:
                s = 2.0 ** rng.integers(-1, 2)
                v = rng.choice(grid, 32) * rng.choice([-1, 1], 32)
                v[rng.integers(32)] = 4.0 * rng.choice([-1, 1])
                x[r, 32 * b:32 * b + 32] = v * s
            else:
                v = rng.integers(-15, 16, 32).astype(np.float64)
                v[rng.integers(32)] = 16.0 * rng.choice([-1, 1])
                x[r, 32 * b:32 * b + 32] = v
    return x


def test_mx_gemm_lossless_exact(atom):
    """Representable inputs: the codes decode to the inputs exactly (checked by the oracle pins'
    lossless case) and every product and partial sum is exact in fp32, so the GPU's fp16 output
    equals fp16 of numpy's exact float64 matmul of the reordered operands."""
    import torch
    rng = np.random.default_rng(11)
    M, N, K = 40, 384, 640
    xr, wr = _exact_rows(rng, M, K, 128), _exact_rows(rng, N, K, 128)
    perm = rng.permutation(K).astype(np.int32)
    X = np.zeros_like(xr)
    W = np.zeros_like(wr)
    X[:, perm], W[:, perm] = xr, wr
    a, _ = check_quant(atom, X.astype(np.float16), perm, K, 128)
    w, _ = check_quant(atom, W.astype(np.float16), perm, K, 128)
    c = atom.mx_gemm(a, w)
    torch.cuda.synchronize()
    exact = xr @ wr.T
    assert np.abs(exact).max() < 2 ** 15
    np.testing.assert_array_equal(host(c), exact.astype(np.float16))


def test_mx_gemm_graph_and_wide_out(atom):
    """CUDA-graph replay equals eager; an N-shard written into a column block of a wider C."""
    import torch
    M, N, K = 96, 1024, 2048
    X, W, perm = synth.problem(M, N, K, seed=9)
    a = atom.mx_quantize(dev(X), dev(perm))
    w = atom.mx_quantize(dev(W), dev(perm))
    ref = atom.mx_gemm(a, w)
    big = torch.zeros((M, 2 * N), dtype=torch.float16, device="cuda")
    atom.mx_gemm(a, w, out=big[:, N:])
    g = torch.cuda.CUDAGraph()
    out = torch.empty_like(ref)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        atom.mx_gemm(a, w, out=out)
        with torch.cuda.graph(g, stream=s):
            atom.mx_gemm(a, w, out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref) and torch.equal(big[:, N:], ref)
    assert torch.all(big[:, :N] == 0)
