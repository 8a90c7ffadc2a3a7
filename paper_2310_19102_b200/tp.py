"""Tensor-parallel sharding of one Atom W4A4 linear layer.

Host-side shard algebra (pure Python, unit-tested with gloo on CPU) plus the NCCL forward used by
bench.py.  Nothing here computes the method: quantization and the GEMM run in libatom.so.

N-shard (column parallel): rank r owns output channels [n0, n1) (multiples of 128); X is
replicated; each rank writes an fp16 [M][N/P] block; all-gather -> [P][M][N/P] -> [M][N].
Each shard's output equals one GPU's within the fp32-reordering tolerance (each shard GEMM has
its own work schedule, which may split a tile's K accumulation at other points).

K-shard (row parallel): rank r owns a contiguous range of 128-channel groups [g0, g1) of the
REORDERED channels; its perm slice is perm[g0*128 : g1*128]; the INT8 outlier group (the last
one) lives on the last rank only (k_outlier = 128 there, 0 elsewhere).  Each rank writes fp32
partial sums; all-reduce(SUM) in fp32, then fp16.  Partials are bit-identical to one GPU; the
output is within the fp32-reordering tolerance.
"""
from __future__ import annotations

GROUP = 128


def n_shard_rows(N: int, P: int, r: int) -> tuple[int, int]:
    if N % (GROUP * P):
        raise ValueError(f"N={N} must split into {P} shards of whole 128-channel tiles")
    return r * N // P, (r + 1) * N // P


def k_shard_groups(K: int, P: int, r: int) -> tuple[int, int]:
    G = K // GROUP
    if K % GROUP or G < P:
        raise ValueError(f"K={K} must have at least {P} groups of 128")
    return r * G // P, (r + 1) * G // P


def k_shard(perm, K: int, P: int, r: int, k_outlier: int = 128):
    """(perm slice, K_r, k_outlier_r) for rank r of a K-sharded layer."""
    g0, g1 = k_shard_groups(K, P, r)
    ko = k_outlier if r == P - 1 else 0
    return perm[g0 * GROUP:g1 * GROUP], (g1 - g0) * GROUP, ko


def blocks_to_matrix(blocks):
    """[P][M][N/P] all-gather result -> [M][N] (torch or numpy)."""
    P, M, Nb = blocks.shape
    if hasattr(blocks, "permute"):
        return blocks.permute(1, 0, 2).reshape(M, P * Nb)
    return blocks.transpose(1, 0, 2).reshape(M, P * Nb)


class TensorParallelLinear:
    """One Atom linear layer sharded over the default process group (CUDA + NCCL)."""

    def __init__(self, w_shard_f16, perm, K: int, shard: str, k_outlier: int = 128,
                 clip_w: float = 0.85, clip_a: float = 0.9, clip_int8: float = 1.0):
        import torch
        import torch.distributed as dist

        import paper_2310_19102_b200 as atom
        self.atom, self.dist = atom, dist
        init = dist.is_available() and dist.is_initialized()
        self.P, self.r = (dist.get_world_size(), dist.get_rank()) if init else (1, 0)
        self.shard = shard
        self.clip_a, self.clip_int8 = clip_a, clip_int8
        if shard == "n":
            self.perm, self.K, self.ko = perm, K, k_outlier
        elif shard == "k":
            self.perm, self.K, self.ko = k_shard(perm, K, self.P, self.r, k_outlier)
            self.perm = self.perm.contiguous()
        else:
            raise ValueError(shard)
        self.w = atom.quantize_weights(w_shard_f16, self.perm, K=self.K, k_outlier=self.ko,
                                       clip_int4=clip_w, clip_int8=clip_int8)
        self.torch = torch

    def quantize(self, x, out=None):
        return self.atom.reorder_quantize(x, self.perm, K=self.K, k_outlier=self.ko,
                                          clip_int4=self.clip_a, clip_int8=self.clip_int8,
                                          out=out)

    def gemm(self, a, out=None):
        dt = self.torch.float16 if self.shard == "n" else self.torch.float32
        return self.atom.w4a4_gemm(a, self.w, out=out, out_dtype=dt)

    def combine(self, local, gathered=None):
        """The collective step (a6).  NCCL in production; the gloo branch (CPU staging) exists
        only so the sharded path can be exercised with several ranks on one GPU in tests."""
        if self.P == 1:
            return local if local.dtype == self.torch.float16 else local.half()
        gloo = self.dist.get_backend() == "gloo"
        if self.shard == "n":
            if gathered is None:
                gathered = local.new_empty((self.P,) + tuple(local.shape))
            if gloo:
                parts = [self.torch.empty_like(local, device="cpu") for _ in range(self.P)]
                self.dist.all_gather(parts, local.cpu())
                gathered.copy_(self.torch.stack(parts))
            else:
                self.dist.all_gather_into_tensor(gathered, local)
            return gathered
        if gloo:
            h = local.cpu()
            self.dist.all_reduce(h)
            local.copy_(h)
        else:
            self.dist.all_reduce(local)
        return local.half() if gathered is None else gathered.copy_(local)

    def __call__(self, x):
        return self.combine(self.gemm(self.quantize(x)))
