"""Development: run one MX GEMM with a given library build, report max error vs the oracle."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import oracle  # noqa: E402
import paper_2310_19102_b200 as atom  # noqa: E402
import synth  # noqa: E402

atom.LIB_PATH = Path(sys.argv[1])
M, N, K = (int(v) for v in sys.argv[2].split(","))
X, W, perm = synth.problem(M, N, K, seed=1)
a = atom.mx_quantize(torch.from_numpy(X).cuda(), torch.from_numpy(perm).cuda())
w = atom.mx_quantize(torch.from_numpy(W).cuda(), torch.from_numpy(perm).cuda())
c = atom.mx_gemm(a, w)
torch.cuda.synchronize()
ra = oracle.mx_quantize_rows(X, perm, K)
rw = oracle.mx_quantize_rows(W, perm, K)
ref = oracle.mx_output_rows(ra, rw, M, N, K, 128)
err = np.abs(c.float().cpu().numpy() - ref)
tol = 2.0 ** -10 + 1e-3 * np.abs(ref)
print(sys.argv[1], "max err", err.max(), "max err/tol", (err / tol).max(), "ref max", np.abs(ref).max())
