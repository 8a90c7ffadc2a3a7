"""Run the GEMM once for one shape (argv: M N K [seed]) and compare a few rows with the oracle.
Development tool: each shape runs in its own process under `timeout` (tools/_run.sh)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2310_19102_b200 as atom  # noqa: E402
import synth  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4])
X, W, perm = synth.problem(M, N, K, seed=0)
pd = torch.from_numpy(perm).cuda()
wq = atom.quantize_weights(torch.from_numpy(W).cuda(), pd)
aq = atom.reorder_quantize(torch.from_numpy(X).cuda(), pd)
c = atom.w4a4_gemm(aq, wq)
torch.cuda.synchronize()
w4, w8, ws = oracle.quantize_rows(W, perm, K, 128, 0.85, 1.0)
a4, a8, as_ = oracle.quantize_rows(X, perm, K, 128, 0.9, 1.0)
rows = np.unique(np.array([0, M - 1, M // 2]))
ref = oracle.output_rows(a4, a8, as_, w4, w8, ws, M, N, K, 128, rows)
got = c.float().cpu().numpy()[rows].astype(np.float64)
err = np.max(np.abs(got - ref) / (2.0 ** -10 + 1e-3 * np.abs(ref)))
print(f"M={M} N={N} K={K} ws={atom.workspace_size(M, N, K)} max err/tol {err:.3f}", flush=True)
