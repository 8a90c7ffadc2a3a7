"""Tensor-parallel layer through the real CUDA kernels: 2 ranks share cuda:0 (gloo backend, the
only way to run several ranks on one GPU); both within the output tolerance of the oracle (an
N-shard is its own GEMM schedule, so its fp32 sums may be split at other K points).  (Production runs use NCCL, one rank per GPU: bench.py.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, shard, M, N, K, q, split_free=False):
    import torch.distributed as dist
    import paper_2310_19102_b200 as atom
    from paper_2310_19102_b200 import tp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        X, perm = synth.activations(M, K, 5), synth.perm_for(K, 5)
        if shard == "n":
            n0, n1 = tp.n_shard_rows(N, world, rank)
            W = synth.weights(N, K, 5, rows=(n0, n1))
        else:
            W = synth.weights(N, K, 5)
        pd = torch.from_numpy(perm).cuda()
        layer = tp.TensorParallelLinear(torch.from_numpy(W).cuda(), pd, K, shard,
                                        split_free=split_free)
        out = layer(torch.from_numpy(X).cuda())
        if shard == "n":
            out = tp.blocks_to_matrix(out)
        torch.cuda.synchronize()
        if rank == 0:
            q.put(out.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shard", ["n", "k"])
def test_tp_two_ranks_one_gpu(shard):
    import paper_2310_19102_b200 as atom
    M, N, K = 64, 512, 2048
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, shard, M, N, K, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = q.get(timeout=600)
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    X, W, perm = synth.activations(M, K, 5), synth.weights(N, K, 5), synth.perm_for(K, 5)
    pd = torch.from_numpy(perm).cuda()
    ref_gpu = atom.QuantizedLinear(torch.from_numpy(W).cuda(), pd)(torch.from_numpy(X).cuda())
    assert out.shape == tuple(ref_gpu.shape)
    ref = oracle.quantized_linear(X, perm, W, K)["c"]
    err = np.abs(out.astype(np.float64) - ref)
    assert np.all(err <= 2.0 ** -10 + 1e-3 * np.abs(ref))


def _mlp_worker(rank, world, port, M, H, I, q):
    import torch.distributed as dist
    from paper_2310_19102_b200 import tp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        X, perm_h = synth.activations(M, H, 7), synth.perm_for(H, 7)
        Wg, Wu, Wd = synth.weights(I, H, 71), synth.weights(I, H, 72), synth.weights(H, I, 73)
        perm_i = synth.perm_for(I, 74)
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        mlp = tp.TensorParallelMLP(cu(Wg), cu(Wu), cu(Wd), cu(perm_h), cu(perm_i))
        x = cu(X)
        _, (g, u, hq) = mlp.local(x)
        y = mlp(x)
        torch.cuda.synchronize()
        # this rank's down-projection input: bit-exact against the oracle fed with the GPU's
        # fp16 gate / up shard (which must be the perm_i-reordered channels of this rank)
        Ir, ko = mlp.Ir, mlp.ko
        g0, _ = tp.k_shard_groups(I, world, rank)
        rows = perm_i[g0 * 128:g0 * 128 + Ir]
        ident = np.arange(Ir, dtype=np.int32)
        a4, a8, asc = oracle.silu_mul_quantize_rows(g.cpu().numpy(), u.cpu().numpy(), ident, Ir, ko)
        if a4.size:
            np.testing.assert_array_equal(hq.q4.cpu().numpy(), a4)
        if ko:
            np.testing.assert_array_equal(hq.q8.cpu().numpy(), a8)
        np.testing.assert_array_equal(hq.scales.cpu().numpy().view(np.uint32), asc.view(np.uint32))
        # the gate shard is the reordered channels of the unsharded gate projection
        full_g = oracle.quantized_linear(X, perm_h, Wg[rows], H)["c"]
        assert np.all(np.abs(g.float().cpu().numpy() - full_g) <= 2.0 ** -10 + 1e-3 * np.abs(full_g))
        # oracle partial of this rank's down projection, summed over ranks like the GPU partials
        w4, w8, wsc = oracle.quantize_rows(np.ascontiguousarray(Wd[:, rows]), ident, Ir, ko, 0.85, 1.0)
        part = torch.from_numpy(oracle.output_rows(a4, a8, asc, w4, w8, wsc, M, H, Ir, ko,
                                                   np.arange(M)))
        dist.all_reduce(part)
        if rank == 0:
            q.put((y.cpu().numpy(), part.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_tp_paired_mlp(world):
    """NEXT-4: Megatron-paired Llama MLP (gate/up column parallel without a gather, SwiGLU fused
    into the down projection's quantizer, down row parallel, one all-reduce) on the real kernels,
    world ranks sharing cuda:0."""
    M, H, I = 48, 1024, 2048
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_mlp_worker, args=(r, world, port, M, H, I, q)) for r in range(world)]
    for p in ps:
        p.start()
    y, ref = q.get(timeout=600)
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    err = np.abs(y.astype(np.float64) - ref)
    assert np.all(err <= 2.0 ** -10 + 1e-3 * np.abs(ref)), np.max(err)


def test_tp_n_shard_split_free_bit_identical_to_one_gpu():
    """Two N-shard ranks (gloo, one GPU) with the split-free GEMM: the gathered output equals the
    single-GPU split-free GEMM of the whole layer bit for bit."""
    import paper_2310_19102_b200 as atom
    from paper_2310_19102_b200 import tp
    M, N, K = 64, 1024, 2048
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, "n", M, N, K, q, True)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=600)
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    X, perm = synth.activations(M, K, 5), synth.perm_for(K, 5)
    W = synth.weights(N, K, 5)
    pd = torch.from_numpy(perm).cuda()
    one = tp.TensorParallelLinear(torch.from_numpy(W).cuda(), pd, K, "n", split_free=True)
    full = one(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.view(np.uint16), full.cpu().numpy().view(np.uint16))


def _nccl_worker(rank, world, port, M, N, K, q):
    import torch.distributed as dist
    from paper_2310_19102_b200 import tp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        X, perm = synth.activations(M, K, 6), synth.perm_for(K, 6)
        n0, n1 = tp.n_shard_rows(N, world, rank)
        W = synth.weights(N, K, 6, rows=(n0, n1))
        layer = tp.TensorParallelLinear(torch.from_numpy(W).cuda(), torch.from_numpy(perm).cuda(),
                                        K, "n", split_free=True)
        out = tp.blocks_to_matrix(layer(torch.from_numpy(X).cuda()))
        torch.cuda.synchronize()
        if rank == 0:
            q.put(out.cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs (NCCL world 2)")
def test_tp_nccl_world2_n_shard():
    """NCCL, one rank per GPU (the production collective): the all-gathered N-shard output of a
    split-free layer equals the single-GPU split-free GEMM bit for bit."""
    from paper_2310_19102_b200 import tp
    M, N, K = 128, 2048, 4096
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_nccl_worker, args=(r, 2, port, M, N, K, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=600)
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    X, perm = synth.activations(M, K, 6), synth.perm_for(K, 6)
    W = synth.weights(N, K, 6)
    one = tp.TensorParallelLinear(torch.from_numpy(W).cuda(), torch.from_numpy(perm).cuda(), K,
                                  "n", split_free=True)
    full = one(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.view(np.uint16), full.cpu().numpy().view(np.uint16))
