"""Summarise an ncu report: key metrics, stall reasons, hottest SASS lines, per-role samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
d = {h[i]: (v[i], u[i]) for i in range(len(h))}
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "launch__registers_per_thread", "launch__grid_size"]
for k in keys:
    if k in d:
        print(f"{k:80s} {d[k][0]} {d[k][1]}")
st = sorted([(float(d[k][0].replace(",", "") or 0), k) for k in d
             if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")], reverse=True)
print("stalls:", ", ".join(f"{k.split('stalled_')[1]}={int(a)}" for a, k in st[:8]))
src = [r for r in csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source=sass")))
       if len(r) > 2 and r[2].strip().isdigit()]
tot = sum(int(r[2]) for r in src)
print("samples", tot)
for r in sorted(src, key=lambda r: -int(r[2]))[:top]:
    print(r[0][-5:], r[2].rjust(6), r[1][:90])
