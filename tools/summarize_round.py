"""Summarise a gpu_round.sh output directory into profiles/<tag>/ (ncu summaries, launch-list
shares, bench lines) and profiles/traffic.json (DRAM bytes per launch of the GEMM, read by
bench.py for the roofline 'traffic' field)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
src = ROOT / "gpurun_out" / sys.argv[1]
dst = ROOT / "profiles" / sys.argv[2]
dst.mkdir(parents=True, exist_ok=True)


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return {r[0][i]: (r[2][i], r[1][i]) for i in range(len(r[0]))}


traffic_file = ROOT / "profiles" / "traffic.json"
traffic = json.loads(traffic_file.read_text()) if traffic_file.exists() else {}
for rep in sorted(src.glob("prof_*.ncu-rep")):
    s = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep), "30"],
                       capture_output=True, text=True).stdout
    (dst / (rep.stem + ".txt")).write_text(s)
    if rep.stem.startswith("prof_gemm_"):
        d = raw_metrics(rep)
        def mb(k):
            v, u = d[k]
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
        cfg = rep.stem[len("prof_gemm_"):]
        traffic[f"{cfg}:gemm:P1n"] = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
traffic_file.write_text(json.dumps(traffic, indent=1) + "\n")

for lc in sorted(src.glob("launches_*.csv")):
    rows = [r for r in csv.reader(open(lc)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r[4].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[14].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = ["kernel, launches, mean_us, share_of_listed_time"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k}, {n}, {t / n / 1e3:.2f}, {t / tot:.3f}")
    (dst / (lc.stem + "_shares.csv")).write_text("\n".join(lines) + "\n")
    (dst / lc.name).write_text(lc.read_text())
for b in sorted(src.glob("bench_*.json")):
    (dst / b.name).write_text(b.read_text())
print("wrote", dst)
