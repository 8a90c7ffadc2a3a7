"""Development: time small-M GEMMs several ways (warm back-to-back, graph of launches, split-free)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_2310_19102_b200 as atom  # noqa: E402
import synth  # noqa: E402

if len(sys.argv) > 2:
    atom.LIB_PATH = Path(sys.argv[2])
for arg in sys.argv[1].split(";"):
    M, N, K = (int(v) for v in arg.split(","))
    X = torch.from_numpy(synth.activations(M, K, 0)).cuda()
    perm = torch.from_numpy(synth.perm_for(K, 0)).cuda()
    W = torch.from_numpy(synth.weights(N, K, 0)).cuda()
    wq = atom.quantize_weights(W, perm)
    aq = atom.reorder_quantize(X, perm, packed=False)
    out = torch.empty((M, N), dtype=torch.float16, device="cuda")
    for sf in (False, True):
        ws = atom.gemm_workspace(M, N, K, 128) if not sf else None
        f = lambda: atom.w4a4_gemm(aq, wq, out=out, workspace=ws, split_free=sf)
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            f()
        e1.record()
        torch.cuda.synchronize()
        eager = e0.elapsed_time(e1) / 50 * 1e3
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            f()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    f()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        gr = e0.elapsed_time(e1) / 100 * 1e3
        print(f"M={M} N={N} K={K} split_free={sf}: eager {eager:.1f} us, graph {gr:.1f} us/launch")
