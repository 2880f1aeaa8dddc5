"""Print the launches of the last run from an ncu CSV launch list
(gpu__time_duration.sum, dram bytes, SM throughput); argv[2] = runs in the
capture (default 4)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
hdr = None
data = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        data.setdefault(d["ID"], {"name": d["Kernel Name"][:70]})[d["Metric Name"]] = d["Metric Value"].replace(",", "")
items = list(data.values())
tot = 0.0
for it in items[-(len(items) // runs):]:
    t = float(it.get("gpu__time_duration.sum", 0)) / 1000
    tot += t
    rd = float(it.get("dram__bytes_read.sum", 0)) / 1e6
    wr = float(it.get("dram__bytes_write.sum", 0)) / 1e6
    print(f"{t:8.1f}us R {rd:8.1f}MB W {wr:7.1f}MB {(rd + wr) / 1e3 / max(t, 1e-9) * 1e3:7.0f}GB/s "
          f"sm {it.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', ''):>6} {it['name']}")
print(f"total {tot:.1f} us over {len(items) // runs} launches")
