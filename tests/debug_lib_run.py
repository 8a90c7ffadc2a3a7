"""Runs the hot path's kernels on a few shapes through a given libatom build and saves every
output to an .npz (used by tests/test_debug_lib.py to compare the timeout-trap debug library with
the release library bit for bit).  Usage: python tests/debug_lib_run.py LIB OUT.npz"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2310_19102_b200 as atom  # noqa: E402
import synth  # noqa: E402

# INT path: swap-AB small M, stream-K / even-split mid M, split-free; MX path: split-K small M,
# 256-token tiles with the wave-tail launch; KV: ragged sequences over permuted pages
INT_SHAPES = [(16, 1024, 1024), (256, 4096, 4096), (300, 2048, 1152)]
MX_SHAPES = [(8, 4096, 2048), (1000, 28672, 256)]


def run(lib: str, out: str) -> None:
    atom.LIB_PATH = Path(lib)
    atom.load()
    dev = torch.device("cuda:0")
    res = {}
    for M, N, K in INT_SHAPES:
        X, W, perm = synth.problem(M, N, K, seed=M + N)
        p = torch.from_numpy(perm).to(dev)
        a = atom.reorder_quantize(torch.from_numpy(X).to(dev), p)
        w = atom.quantize_weights(torch.from_numpy(W).to(dev), p)
        res[f"int_{M}_{N}_{K}"] = atom.w4a4_gemm(a, w).cpu().numpy()
        res[f"int_sf_{M}_{N}_{K}"] = atom.w4a4_gemm(a, w, split_free=True).cpu().numpy()
    for M, N, K in MX_SHAPES:
        X, W, perm = synth.problem(M, N, K, seed=M + 7)
        p = torch.from_numpy(perm).to(dev)
        a = atom.mx_quantize(torch.from_numpy(X).to(dev), p)
        w = atom.mx_quantize(torch.from_numpy(W).to(dev), p)
        res[f"mx_{M}_{N}_{K}"] = atom.mx_gemm(a, w).cpu().numpy()
    rng = np.random.default_rng(3)
    lens, H = [700, 64, 1, 129], 4
    max_pages = max((L + 15) // 16 for L in lens)
    bt = rng.permutation(len(lens) * max_pages).reshape(len(lens), max_pages).astype(np.int32)
    kg = atom.KvCache.empty(len(lens) * max_pages, H)
    vg = atom.KvCache.empty(len(lens) * max_pages, H)
    for b, L in enumerate(lens):
        slots = (bt[b][np.arange(L) // 16] * 16 + np.arange(L) % 16).astype(np.int32)
        s = torch.from_numpy(slots).to(dev)
        atom.kv_quantize(torch.from_numpy(rng.normal(0, 1, (L, H * 128)).astype(np.float16)).to(dev),
                         s, kg)
        atom.kv_quantize(torch.from_numpy(rng.normal(0, 1, (L, H * 128)).astype(np.float16)).to(dev),
                         s, vg)
    q = torch.from_numpy(rng.normal(0, 1, (len(lens), H, 128)).astype(np.float16)).to(dev)
    res["kv_codes"] = vg.codes.cpu().numpy()
    res["kv_attn"] = atom.decode_attention(q, kg, vg, torch.from_numpy(bt).to(dev),
                                           torch.tensor(lens, dtype=torch.int32, device=dev),
                                           max(lens)).cpu().numpy()
    torch.cuda.synchronize()
    np.savez(out, **res)


if __name__ == "__main__":
    run(sys.argv[1], sys.argv[2])
