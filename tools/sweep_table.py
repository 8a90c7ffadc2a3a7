"""Print a sweep JSONL (bench.py lines) as a table; optional second file for before/after."""
import json
import sys


def load(p):
    out = {}
    for line in open(p):
        line = line.strip()
        if line.startswith("{"):
            d = json.loads(line)
            out[d["config"]["workload"]] = d
    return out


new = load(sys.argv[1])
old = load(sys.argv[2]) if len(sys.argv) > 2 else {}
print(f"{'config':16s} {'M':>5s} {'N':>6s} {'K':>6s} {'step us':>8s} {'gemm us':>8s} {'quant us':>8s} "
      f"{'spec frac':>9s} {'old gemm':>8s}")
for k, d in new.items():
    c = d["config"]
    g = d["kernels"]["w4a4_gemm"]["us"]
    o = old.get(k, {}).get("kernels", {}).get("w4a4_gemm", {}).get("us", float("nan"))
    print(f"{k:16s} {c['M']:5d} {c['N']:6d} {c['K']:6d} {d['ms_per_step'] * 1e3:8.1f} {g:8.1f} "
          f"{d['kernels']['reorder_quantize']['us']:8.1f} {d['roofline_spec']['frac']:9.3f} {o:8.1f}")
