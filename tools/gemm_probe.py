"""Time the GEMM kernel alone (CUDA events, L2 flushed) for a config, optionally in a probe mode
(ATOM_GEMM_PROBE_MODE: 1 = no epilogue math, 2 = no TMEM loads, ...; only honoured by a library
built with ATOM_NVCC_EXTRA=-DATOM_DEV_PROBES).  Development tool."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2310_19102_b200 as atom  # noqa: E402
import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
if "," in cfg:                       # an explicit shape "M,N,K"
    M, N, K = (int(v) for v in cfg.split(","))
else:
    M, N, K, _ = CONFIGS[cfg]
X, perm = synth.activations(M, K, 0), synth.perm_for(K, 0)
W = synth.weights(N, K, 0)
pd = torch.from_numpy(perm).cuda()
wq = atom.quantize_weights(torch.from_numpy(W).cuda(), pd)
aq = atom.reorder_quantize(torch.from_numpy(X).cuda(), pd)
c = torch.empty((M, N), dtype=torch.float16, device="cuda")
flush = torch.empty(300 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(300 << 20, dtype=torch.uint8, device="cuda")
FLUSH = os.environ.get("PROBE_FLUSH", "write")      # write | write+read | none


def flush_l2():
    if FLUSH != "none":
        flush.zero_()
    if FLUSH == "write+read":          # evict the flush's dirty lines (write-backs) before timing
        clean.sum(dtype=torch.int32)
for _ in range(3):
    atom.w4a4_gemm(aq, wq, out=c)
if os.environ.get("ATOM_GEMM_TRACE"):
    sys.exit(0)
# PROBE_REPS > 1: one CUDA graph of REPS back-to-back launches (warm L2 after the first) per
# sample, for shapes below the event timer's resolution and the host launch rate
REPS = int(os.environ.get("PROBE_REPS", "1"))
graph = None
if REPS > 1:
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        atom.w4a4_gemm(aq, wq, out=c, stream=side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            for _ in range(REPS):
                atom.w4a4_gemm(aq, wq, out=c, stream=side)
    torch.cuda.current_stream().wait_stream(side)
    graph.replay()
    torch.cuda.synchronize()
ts = []
for _ in range(10):
    flush_l2()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if graph is not None:
        graph.replay()
    else:
        atom.w4a4_gemm(aq, wq, out=c)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / REPS)
ts.sort()
us = ts[len(ts) // 2] * 1e3
print(f"{cfg} mode={os.environ.get('ATOM_GEMM_PROBE_MODE', '0')} gemm {us:.1f} us  "
      f"{2 * M * N * K / us / 1e6:.0f} TOPS")
xd = torch.from_numpy(X).cuda()
qt = []
for _ in range(10):
    flush_l2()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    atom.reorder_quantize(xd, pd, out=aq)
    e1.record()
    torch.cuda.synchronize()
    qt.append(e0.elapsed_time(e1))
qt.sort()
print(f"{cfg} quantize {qt[len(qt) // 2] * 1e3:.1f} us")
