"""Development A/B: time the GEMM of one BASELINE config with a given libatom build.
usage: python tools/ab_gemm.py LIB.so CONFIG [reps]  -> prints 'LIB CONFIG us'  (CUDA events over a
graph of `reps` back-to-back GEMMs, L2 flushed before each graph replay, median of 7)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_2310_19102_b200 as atom  # noqa: E402
import synth  # noqa: E402

lib, cfg = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
what = sys.argv[4] if len(sys.argv) > 4 else "gemm"     # gemm | quant
atom.LIB_PATH = Path(lib).resolve()
cfgs = {"cfg5": (1024, 28672, 8192), "cfg2": (256, 4096, 4096), "cfg4": (512, 13824, 5120),
        "cfg3u": (1024, 11008, 4096), "cfg3d": (1024, 4096, 11008), "m64": (64, 11008, 4096),
        "m16": (16, 11008, 4096)}
M, N, K = cfgs[cfg]
X = torch.from_numpy(synth.activations(M, K, 0)).cuda()
perm = torch.from_numpy(synth.perm_for(K, 0)).cuda()
W = torch.from_numpy(synth.weights(N, K, 0)).cuda()
wq = atom.quantize_weights(W, perm)
aq = atom.reorder_quantize(X, perm, packed=False)
out = atom.w4a4_gemm(aq, wq)
ref = out.clone()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
def call():
    if what == "quant":
        atom.reorder_quantize(X, perm, out=aq, packed=False, stream=s)
    else:
        atom.w4a4_gemm(aq, wq, out=out, stream=s)


with torch.cuda.stream(s):
    call()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            call()
torch.cuda.current_stream().wait_stream(s)
flush = torch.empty(2 * torch.cuda.get_device_properties(0).L2_cache_size, dtype=torch.uint8,
                    device="cuda")
ts = []
for _ in range(9):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3 / reps)
ts.sort()
ok = torch.equal(out, ref)
print(f"{Path(lib).name} {cfg} {what} {ts[len(ts) // 2]:.1f} us  (min {ts[0]:.1f}) "
      f"{'ok' if ok else 'MISMATCH'}")
