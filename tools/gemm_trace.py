"""Development: run one GEMM of a BASELINE config through a probe build of the library
(ab/libatom_probe.so, built with -DATOM_DEV_PROBES) with ATOM_GEMM_TRACE=1, which prints the
per-group timeline of CTA 0 (clock64) to stderr."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ["ATOM_GEMM_TRACE"] = "1"
import torch  # noqa: E402
import paper_2310_19102_b200 as atom  # noqa: E402
import synth  # noqa: E402

atom.LIB_PATH = ROOT / "ab" / "libatom_probe.so"
cfgs = {"cfg5": (1024, 28672, 8192), "cfg2": (256, 4096, 4096), "cfg4": (512, 13824, 5120),
        "cfg3u": (1024, 11008, 4096)}
arg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
M, N, K = cfgs[arg] if arg in cfgs else tuple(int(v) for v in arg.split(","))
X = torch.from_numpy(synth.activations(M, K, 0)).cuda()
perm = torch.from_numpy(synth.perm_for(K, 0)).cuda()
W = torch.from_numpy(synth.weights(N, K, 0)).cuda()
wq = atom.quantize_weights(W, perm)
aq = atom.reorder_quantize(X, perm, packed=False)
for _ in range(3):
    atom.w4a4_gemm(aq, wq)
torch.cuda.synchronize()
