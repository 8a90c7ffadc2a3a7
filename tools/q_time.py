"""Development: time the INT reorder+quantize (operand form, as the bench step) for a shape."""
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
    M, K = (int(v) for v in arg.split(","))
    X = torch.from_numpy(synth.activations(M, K, 0)).cuda()
    perm = torch.from_numpy(synth.perm_for(K, 0)).cuda()
    aq = atom.reorder_quantize(X, perm, packed=False)
    f = lambda: atom.reorder_quantize(X, perm, packed=False, out=aq)
    flush = torch.empty(int(400e6), dtype=torch.uint8, device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        f()
        with torch.cuda.graph(g, stream=s):
            f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    warm, cold = [], []
    for i in range(20):
        if i % 2:
            flush.fill_(1)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        (cold if i % 2 else warm).append(e0.elapsed_time(e1) * 1e3)
    warm.sort()
    cold.sort()
    print(f"{sys.argv[2] if len(sys.argv) > 2 else 'lib'} M={M} K={K}: warm {warm[5]:.1f} us, cold {cold[5]:.1f} us")
