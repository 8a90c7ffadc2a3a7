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
                 clip_w: float = 0.85, clip_a: float = 0.9, clip_int8: float = 1.0,
                 split_free: bool = False):
        import torch
        import torch.distributed as dist

        import paper_2310_19102_b200 as atom
        self.atom, self.dist = atom, dist
        init = dist.is_available() and dist.is_initialized()
        self.P, self.r = (dist.get_world_size(), dist.get_rank()) if init else (1, 0)
        self.shard = shard
        # N-shard with split_free: every output is the unsharded GEMM's fp32 chain (bit-identical
        # to one GPU running the same split-free GEMM, include/atom.h ATOM_GEMM_SPLIT_FREE)
        self.split_free = split_free
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
        """a1 on the hot path: writes only what the GEMM reads (the operand form + scales)."""
        return self.atom.reorder_quantize(x, self.perm, K=self.K, k_outlier=self.ko,
                                          clip_int4=self.clip_a, clip_int8=self.clip_int8,
                                          out=out, packed=False)

    def gemm(self, a, out=None):
        dt = self.torch.float16 if self.shard == "n" else self.torch.float32
        return self.atom.w4a4_gemm(a, self.w, out=out, out_dtype=dt,
                                   split_free=self.split_free and self.shard == "n")

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


def mlp_shard(perm_i, I: int, P: int, r: int, k_outlier: int = 128):
    """(rows, I_r, k_outlier_r) of rank r in the paired MLP: the original intermediate channels
    perm_i[i0:i1] whose gate / up rows the rank owns (in reordered order), which are also its
    down-projection K-shard (identity perm inside the shard, INT8 group on the last rank)."""
    g0, g1 = k_shard_groups(I, P, r)
    return perm_i[g0 * GROUP:g1 * GROUP], (g1 - g0) * GROUP, (k_outlier if r == P - 1 else 0)


class TensorParallelMLP:
    """NEXT-4: a Llama MLP  y = down(silu(gate(x)) * up(x))  on the W4A4 path, Megatron-paired
    over the default process group: gate / up are column parallel WITHOUT a gather, the SwiGLU is
    fused into the down projection's quantizer (atom_silu_mul_reorder_quantize), and down is row
    parallel, so the only collective is one fp32 all-reduce of [M][H] partials per MLP (the
    reduce-scatter of a sequence-parallel layer moves the same bytes).

    The down projection's reorder is folded into the ROW order of W_gate / W_up offline (the
    paper's static weight reorder): their outputs come out already in the reordered
    channel order, so rank r's gate / up shard [i0, i1) is exactly the down projection's K-shard
    of reordered groups k_shard_groups(I, P, r) -- contiguous, with an identity perm inside the
    shard and the INT8 outlier group on the last rank.  Every rank holds the same perm_h (input
    reorder of gate / up) and perm_i (reorder of the intermediate channels)."""

    def __init__(self, w_gate, w_up, w_down, perm_h, perm_i, k_outlier: int = 128,
                 clip_w: float = 0.85, clip_a: float = 0.9, clip_int8: float = 1.0):
        import torch
        import torch.distributed as dist

        import paper_2310_19102_b200 as atom
        self.atom, self.dist, self.torch = atom, dist, torch
        init = dist.is_available() and dist.is_initialized()
        self.P, self.r = (dist.get_world_size(), dist.get_rank()) if init else (1, 0)
        I, H = w_gate.shape
        if w_up.shape != (I, H) or w_down.shape != (H, I):
            raise ValueError("expected W_gate, W_up [I][H] and W_down [H][I]")
        rows, self.Ir, self.ko = mlp_shard(perm_i, I, self.P, self.r, k_outlier)
        rows = rows.long()                                # reordered channels of this rank
        self.H = H
        self.perm_h = perm_h
        self.ident = torch.arange(self.Ir, dtype=torch.int32, device=perm_i.device)
        self.clip_a, self.clip_int8 = clip_a, clip_int8
        q = dict(clip_int4=clip_w, clip_int8=clip_int8)
        self.wg = atom.quantize_weights(w_gate[rows].contiguous(), perm_h, k_outlier=k_outlier, **q)
        self.wu = atom.quantize_weights(w_up[rows].contiguous(), perm_h, k_outlier=k_outlier, **q)
        self.wd = atom.quantize_weights(w_down[:, rows].contiguous(), self.ident, K=self.Ir,
                                        k_outlier=self.ko, **q)
        self.k_outlier = k_outlier

    def local(self, x):
        """This rank's fp32 partial of y [M][H] (and the quantized down-projection input)."""
        atom = self.atom
        xq = atom.reorder_quantize(x, self.perm_h, k_outlier=self.k_outlier,
                                   clip_int4=self.clip_a, clip_int8=self.clip_int8)
        g = atom.w4a4_gemm(xq, self.wg)
        u = atom.w4a4_gemm(xq, self.wu)
        hq = atom.silu_mul_reorder_quantize(g, u, self.ident, K=self.Ir, k_outlier=self.ko,
                                            clip_int4=self.clip_a, clip_int8=self.clip_int8)
        return atom.w4a4_gemm(hq, self.wd, out_dtype=self.torch.float32), (g, u, hq)

    def __call__(self, x):
        y, _ = self.local(x)
        if self.P > 1:
            if self.dist.get_backend() == "gloo":     # tests: several ranks on one GPU
                h = y.cpu()
                self.dist.all_reduce(h)
                y.copy_(h)
            else:
                self.dist.all_reduce(y)
        return y.half()
