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


def _worker(rank, world, port, shard, M, N, K, q):
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
        layer = tp.TensorParallelLinear(torch.from_numpy(W).cuda(), pd, K, shard)
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
