"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report:
python scripts/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, k = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = [x for x in r if x and x[0] == "Address"][0]
rows = [x for x in r if len(x) == len(h) and x[0].startswith("0x")]
i = h.index("Warp Stall Sampling (All Samples)")
e = h.index("Instructions Executed")
f = lambda v: float(v) if v not in ("", "-") else 0.0
n = len(rows)
# ncu may print one listing per launch: keep the first
seen = set()
uniq = []
for x in rows:
    if x[0] in seen:
        break
    seen.add(x[0])
    uniq.append(x)
rows = uniq
tot = sum(f(x[i]) for x in rows)
print(f"samples {tot:.0f} instructions {sum(f(x[e]) for x in rows):.0f} sass lines {len(rows)}")
for k2, x in sorted(enumerate(rows), key=lambda kx: -f(kx[1][i]))[:top]:
    print(f"{k2:5d} {f(x[i]):6.0f} {f(x[e]):10.0f}  {x[1].strip()[:90]}")
