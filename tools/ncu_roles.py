"""Per-role breakdown of an ncu source page for the W4A4 GEMM (development tool): samples, issued
instructions per warp per group, and the hottest lines of each role.  Roles are delimited by the
setmaxnreg (USETMAXREG) at the top of each warpgroup's branch."""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

rep, groups_per_sm = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 10
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))[2:]
names = {0: "prologue", 1: "WG0 producer/MMA/A", 2: "WG1 unpack", 3: "WG2-3 epilogue"}
seen, out = 0, []
for r in rows:
    src = r[1].strip()
    if "USETMAXREG" in src:
        seen += 1
    out.append((int(r[0], 16) & 0xfffff, src, int(r[2]), int(r[5] or 0), names.get(seen, "?")))
warps = {"WG0 producer/MMA/A": 4, "WG1 unpack": 4, "WG2-3 epilogue": 8, "prologue": 16}
samp, ex, ops = defaultdict(int), defaultdict(int), defaultdict(Counter)
for a, s, n, e, c in out:
    samp[c] += n
    ex[c] += e
    op = s.split()[1] if s.startswith("@") else (s.split() or ["?"])[0]
    ops[c][op] += e
for c in samp:
    per = ex[c] / (148 * warps.get(c, 1) * groups_per_sm)
    print(f"== {c}: samples {samp[c]}, {per:.0f} warp-instr per warp per group")
    print("   ops:", ", ".join(f"{k} {v / (148 * warps.get(c, 1) * groups_per_sm):.0f}"
                             for k, v in ops[c].most_common(12)))
    for a, s, n, e, cc in sorted([o for o in out if o[4] == c], key=lambda o: -o[2])[:top]:
        print(f"   {a:05x} {n:6d} {s[:90]}")
