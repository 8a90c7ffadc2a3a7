"""Development: time the NEXT-3 decode attention over the INT4 paged KV cache (graph replay,
warm and after an L2 flush) and report the achieved HBM bandwidth on the cache bytes."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2310_19102_b200 as atom  # noqa: E402

if len(sys.argv) > 2:
    atom.LIB_PATH = Path(sys.argv[2])
for arg in sys.argv[1].split(";"):
    B, L, H = (int(v) for v in arg.split(","))
    rng = np.random.default_rng(0)
    pages = (L + 15) // 16
    bt = torch.from_numpy(rng.permutation(B * pages).reshape(B, pages).astype(np.int32)).cuda()
    k, v = atom.KvCache.empty(B * pages, H), atom.KvCache.empty(B * pages, H)
    slots = (bt[:, :, None] * 16 + torch.arange(16, device="cuda")).reshape(B, -1)[:, :L]
    for b in range(B):
        x = torch.randn((L, H * 128), device="cuda").half()
        atom.kv_quantize(x, slots[b].contiguous().int(), k)
        atom.kv_quantize(x * 0.5, slots[b].contiguous().int(), v)
    q = torch.randn((B, H, 128), device="cuda").half()
    sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
    out = atom.decode_attention(q, k, v, bt, sl, L)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        atom.decode_attention(q, k, v, bt, sl, L, out=out, stream=s)
        with torch.cuda.graph(g, stream=s):
            atom.decode_attention(q, k, v, bt, sl, L, out=out, stream=s)
    torch.cuda.synchronize()
    flush = torch.empty(int(400e6), dtype=torch.uint8, device="cuda")
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
    nbytes = 2 * B * L * H * (64 + 8)
    print(f"B={B} L={L} H={H}: warm {warm[5]:.1f} us ({nbytes / warm[5] / 1e3:.0f} GB/s), cold "
          f"{cold[5]:.1f} us ({nbytes / cold[5] / 1e3:.0f} GB/s), cache {nbytes / 1e6:.1f} MB")
