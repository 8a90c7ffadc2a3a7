"""Development: time the Atom (FP) MX GEMM and quantizer (warm graph of back-to-back launches and
single L2-cold launches)."""
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
    a = atom.mx_quantize(X, perm)
    w = atom.mx_quantize(W, perm)
    out = torch.empty((M, N), dtype=torch.float16, device="cuda")
    flush = torch.empty(int(400e6), dtype=torch.uint8, device="cuda")
    for name, f in (("gemm", lambda: atom.mx_gemm(a, w, out=out)),
                    ("quant", lambda: atom.mx_quantize(X, perm, out=a))):
        for _ in range(3):
            f()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            f()
            with torch.cuda.graph(g, stream=s):
                for _ in range(20):
                    f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.replay()
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        warm = e0.elapsed_time(e1) / 100 * 1e3
        cold = []
        for _ in range(10):
            flush.fill_(1)
            e0.record()
            f()
            e1.record()
            torch.cuda.synchronize()
            cold.append(e0.elapsed_time(e1) * 1e3)
        cold.sort()
        ops = 2 * M * N * K
        print(f"M={M} N={N} K={K} {name}: warm {warm:.1f} us ({ops / warm / 1e6:.0f} TOPS), "
              f"cold median {cold[5]:.1f} us")
