"""Multi-process (world_size 2, gloo, CPU) tests of the tensor-parallel host logic.

Each rank plays one GPU of an N-sharded or K-sharded layer; the per-rank GEMM output is the
ORACLE's output for that rank's shard (the GPU kernels are parity-tested separately), and the real
torch.distributed collective combines them.  Rank 0 checks the result against the unsharded
oracle: N-shard bit-identical, K-shard partials identical and the fp32 sum within tolerance.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2310_19102_b200 import tp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shard, M, N, K, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, perm = synth.activations(M, K, 3), synth.perm_for(K, 3)
        if shard == "n":
            n0, n1 = tp.n_shard_rows(N, world, rank)
            W = synth.weights(N, K, 3, rows=(n0, n1))     # the rank generates only its rows
            r = oracle.quantized_linear(X, perm, W, K)
            local = torch.from_numpy(r["c"].astype(np.float16))
            gathered = torch.empty((world, M, n1 - n0), dtype=torch.float16)
            dist.all_gather_into_tensor(gathered, local) if hasattr(dist, "all_gather_into_tensor") \
                and dist.get_backend() != "gloo" else dist.all_gather(list(gathered.unbind(0)), local)
            out = tp.blocks_to_matrix(gathered)
            parts = None
        else:
            W = synth.weights(N, K, 3)
            ps, Kr, ko = tp.k_shard(perm, K, world, rank)
            r = oracle.quantized_linear(X, np.ascontiguousarray(ps), W, Kr, ko)
            local = torch.from_numpy(r["c"].astype(np.float32))
            dist.all_reduce(local)
            out = local.half()
            parts = r["partials"]
        if rank == 0:
            full = oracle.quantized_linear(X, perm, synth.weights(N, K, 3), K)
            q.put(("out", out.numpy(), full))
        if shard == "k":
            q.put(("parts", rank, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shard", ["n", "k"])
def test_tp_world2_gloo(shard):
    M, N, K, world = 8, 512, 1024, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shard, M, N, K, q))
             for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=300) for _ in range(1 if shard == "n" else 3)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    out, full = next((m[1], m[2]) for m in msgs if m[0] == "out")
    ref16 = full["c"].astype(np.float16)
    if shard == "n":
        np.testing.assert_array_equal(out, ref16)         # bit-identical to one device
    else:
        parts = sorted([m for m in msgs if m[0] == "parts"], key=lambda m: m[1])
        np.testing.assert_array_equal(np.concatenate([p[2] for p in parts]), full["partials"])
        err = np.abs(out.astype(np.float64) - full["c"])
        assert np.all(err <= 2.0 ** -10 + 1e-3 * np.abs(full["c"]))


def test_shard_algebra():
    assert tp.n_shard_rows(28672, 8, 7) == (25088, 28672)
    with pytest.raises(ValueError):
        tp.n_shard_rows(4096, 3, 0)
    perm = np.arange(8192)
    spans = [tp.k_shard(perm, 8192, 8, r) for r in range(8)]
    assert sum(s[1] for s in spans) == 8192
    assert [s[2] for s in spans] == [0] * 7 + [128]
    assert np.array_equal(np.concatenate([s[0] for s in spans]), perm)
    b = np.arange(2 * 3 * 4).reshape(2, 3, 4)
    m = tp.blocks_to_matrix(b)
    assert m.shape == (3, 8) and np.array_equal(m[:, 4:], b[1])


def _mlp_worker(rank, world, port, M, H, I, q):
    """One rank of the paired MLP with the oracle standing in for the kernels (tp.mlp_shard is
    the host logic under test)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, perm_h = synth.activations(M, H, 9), synth.perm_for(H, 9)
        Wg, Wu, Wd = synth.weights(I, H, 91), synth.weights(I, H, 92), synth.weights(H, I, 93)
        perm_i = synth.perm_for(I, 94)
        rows, Ir, ko = tp.mlp_shard(perm_i, I, world, rank)
        g = oracle.quantized_linear(X, perm_h, Wg[rows], H)["c"].astype(np.float16)
        u = oracle.quantized_linear(X, perm_h, Wu[rows], H)["c"].astype(np.float16)
        ident = np.arange(Ir, dtype=np.int32)
        a = oracle.silu_mul_quantize_rows(g, u, ident, Ir, ko)
        w = oracle.quantize_rows(np.ascontiguousarray(Wd[:, rows]), ident, Ir, ko, 0.85, 1.0)
        part = torch.from_numpy(oracle.output_rows(*a, *w, M, H, Ir, ko, np.arange(M)))
        dist.all_reduce(part)
        q.put((rank, a))
        if rank == 0:
            q.put(("y", part.numpy()))
    finally:
        dist.destroy_process_group()


def test_tp_paired_mlp_world2_gloo():
    """Megatron-paired MLP shard algebra: the ranks' down-projection codes, concatenated, are the
    unsharded MLP's codes bit for bit, and the all-reduced output equals the unsharded one."""
    M, H, I, world = 6, 512, 1024, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mlp_worker, args=(r, world, port, M, H, I, q))
             for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=300) for _ in range(world + 1)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    y = next(m[1] for m in msgs if m[0] == "y")
    shards = [m[1] for m in sorted((m for m in msgs if m[0] != "y"), key=lambda m: m[0])]
    # unsharded reference: full gate / up, SwiGLU, down projection with perm_i
    X, perm_h = synth.activations(M, H, 9), synth.perm_for(H, 9)
    Wg, Wu, Wd = synth.weights(I, H, 91), synth.weights(I, H, 92), synth.weights(H, I, 93)
    perm_i = synth.perm_for(I, 94)
    g = oracle.quantized_linear(X, perm_h, Wg, H)["c"].astype(np.float16)
    u = oracle.quantized_linear(X, perm_h, Wu, H)["c"].astype(np.float16)
    a4, a8, asc = oracle.silu_mul_quantize_rows(g, u, perm_i, I)
    np.testing.assert_array_equal(np.concatenate([s[0] for s in shards], axis=1), a4)
    np.testing.assert_array_equal(shards[-1][1], a8)
    np.testing.assert_array_equal(np.concatenate([s[2] for s in shards], axis=0), asc)
    w4, w8, wsc = oracle.quantize_rows(Wd, perm_i, I, 128, 0.85, 1.0)
    ref = oracle.output_rows(a4, a8, asc, w4, w8, wsc, M, H, I, 128, np.arange(M))
    assert np.allclose(y, ref, rtol=1e-12, atol=1e-12)


def test_mlp_shard_algebra():
    perm = np.random.default_rng(0).permutation(2048).astype(np.int32)
    spans = [tp.mlp_shard(perm, 2048, 4, r) for r in range(4)]
    assert np.array_equal(np.concatenate([s[0] for s in spans]), perm)
    assert [s[1] for s in spans] == [512] * 4 and [s[2] for s in spans] == [0, 0, 0, 128]
