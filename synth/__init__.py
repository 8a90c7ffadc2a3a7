"""Seeded synthetic inputs shared by the oracle and the CUDA path (tests, smoke, bench).

Holds none of the method's arithmetic: it only draws random numbers and picks the reorder index
(an INPUT of the hot path) with the calibration rule of the paper.  Recipe (DESIGN.md "Inputs",
SURVEY §8(d)):

* X  fp16 [M][K]: x = r_m * z, z ~ N(0,1), per-token gain r_m = exp(0.5 N(0,1)); 128 outlier
  channels drawn without replacement and multiplied by 100 ("several orders greater", P:228;
  SPEC S:249 x100 injection).
* perm int32 [K]: top-128 channels by square sum over a separate 128-token calibration batch
  ("128 channels with the highest square sum values"), outliers moved to the tail in
  ascending original index, the rest ascending (SPEC S:214 tie rule: lower index first).
* W  fp16 [N][K]: N(0, 0.02^2) (random-init Llama-like weights; BASELINE "random-init weights").

All generators use numpy PCG64(seed).
"""
from __future__ import annotations

import numpy as np

N_OUTLIERS = 128


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def outlier_channels(K: int, seed: int, n_outliers: int = N_OUTLIERS) -> np.ndarray:
    """The injected outlier channel set (sorted), a pure function of (K, seed)."""
    if n_outliers == 0:
        return np.zeros(0, dtype=np.int64)
    return np.sort(_rng(seed + 7919).choice(K, size=n_outliers, replace=False))


def activations(M: int, K: int, seed: int, n_outliers: int = N_OUTLIERS,
                outlier_gain: float = 100.0) -> np.ndarray:
    """fp16 [M][K] Llama-like activations with injected outlier channels."""
    g = _rng(seed)
    z = g.standard_normal((M, K), dtype=np.float64)
    r = np.exp(0.5 * g.standard_normal((M, 1)))
    x = r * z
    ch = outlier_channels(K, seed, n_outliers)
    x[:, ch] *= outlier_gain
    return x.astype(np.float16)


W_BLOCK = 1024   # weight rows per independently seeded block


def weights(N: int, K: int, seed: int, std: float = 0.02, rows: tuple | None = None) -> np.ndarray:
    """fp16 [N][K] random-init weights, N(0, std^2).  Rows come in blocks of W_BLOCK, each from
    its own PCG64 stream (SeedSequence([seed, block])), so a tensor-parallel rank can generate
    exactly its row range ``rows = (r0, r1)`` of the same matrix without the rest."""
    r0, r1 = (0, N) if rows is None else rows
    out = np.empty((r1 - r0, K), dtype=np.float16)
    for b in range(r0 // W_BLOCK, (r1 + W_BLOCK - 1) // W_BLOCK):
        b0, b1 = b * W_BLOCK, min(N, (b + 1) * W_BLOCK)
        g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 104729, b])))
        blk = (np.float32(std) * g.standard_normal((b1 - b0, K), dtype=np.float32))
        lo, hi = max(b0, r0), min(b1, r1)
        out[lo - r0:hi - r0] = blk[lo - b0:hi - b0].astype(np.float16)
    return out


def calibration_perm(calib: np.ndarray, n_outliers: int = N_OUTLIERS) -> np.ndarray:
    """Reorder index from a calibration batch [T][K]: top-n_outliers channels by square sum go to
    the tail (ascending original index), the rest keep ascending order.  Ties -> lower index."""
    calib = np.asarray(calib, dtype=np.float64)
    K = calib.shape[1]
    if n_outliers == 0:
        return np.arange(K, dtype=np.int32)
    score = (calib * calib).sum(axis=0)
    # stable sort by descending score: lower index wins ties
    order = np.lexsort((np.arange(K), -score))
    outl = np.sort(order[:n_outliers])
    mask = np.ones(K, dtype=bool)
    mask[outl] = False
    return np.concatenate([np.nonzero(mask)[0], outl]).astype(np.int32)


def perm_for(K: int, seed: int, n_outliers: int = N_OUTLIERS) -> np.ndarray:
    """Synthetic reorder index: calibrated on 128 tokens drawn with seed+1000 but the SAME outlier
    channels as ``activations(.., seed)`` (mirrors 128 calibration sentences)."""
    g = _rng(seed + 1000)
    z = g.standard_normal((128, K))
    r = np.exp(0.5 * g.standard_normal((128, 1)))
    x = r * z
    x[:, outlier_channels(K, seed, n_outliers)] *= 100.0
    return calibration_perm(x.astype(np.float16), n_outliers)


def problem(M: int, N: int, K: int, seed: int = 0, k_outlier: int = N_OUTLIERS):
    """(X fp16 [M][K], W fp16 [N][K], perm int32 [K]) for one linear layer."""
    return (activations(M, K, seed, k_outlier), weights(N, K, seed),
            perm_for(K, seed, k_outlier))
