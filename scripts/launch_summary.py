"""Summarize an ncu launch-list CSV (gpu__time_duration.sum [+ inst]) for the
last complete step (steps split at k_prep)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
by = collections.OrderedDict()
for d in data:
    v = d["Metric Value"].replace(",", "")
    by.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = (float(v) if v not in ("", "n/a") else 0.0,
                                                                            d["Metric Unit"])
steps, cur = [], []
for d in by.values():
    if "k_prep" in d["name"] and cur:
        steps.append(cur)
        cur = []
    cur.append(d)
steps.append(cur)
s = steps[-1]


def us(v):
    val, u = v
    return val / 1e3 if u == "ns" else (val * 1e3 if u == "ms" else val)


tot = 0.0
agg = collections.OrderedDict()
for d in s:
    t = us(d["gpu__time_duration.sum"])
    tot += t
    a = agg.setdefault(d["name"][:60], [0.0, 0, 0.0])
    a[0] += t
    a[1] += 1
    a[2] += d.get("smsp__inst_executed.sum", (0.0, ""))[0]
print("launches", len(s), "kernel time us", round(tot, 1))
for k, (v, c, ins) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v:8.1f} {c:3d} {ins / 1e6:8.1f}M {k}")
