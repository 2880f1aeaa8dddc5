"""Summarize ncu reports + launch lists into profiles/<round>/ (tracked).

    python scripts/ncu_summarize.py r01 gpurun_out/prof_c2.ncu-rep:c2 gpurun_out/prof_c4m.ncu-rep:c4 \
        --launches gpurun_out/launches_c2.csv:c2
"""
import argparse
import collections
import csv
import json
import os
import subprocess

METRICS = {
    "gpu__time_duration.sum": "duration",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_ghz",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return float(v) * mult.get(unit, 1)


def summarize_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        e = {"kernel": r[hdr.index("Kernel Name")]}
        for m, k in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                val = r[i].replace(",", "")
                try:
                    if k.startswith("dram_read") or k.startswith("dram_write"):
                        e[k + "_bytes"] = to_bytes(val, units[i])
                    elif k == "duration":
                        e["duration_ms"] = float(val) * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                                                         "second": 1e3}.get(units[i], 1.0)
                    else:
                        e[k] = float(val)
                except ValueError:
                    e[k] = val
        e["dram_traffic_bytes"] = e.get("dram_read_bytes", 0) + e.get("dram_write_bytes", 0)
        res.append(e)
    return res


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        if r[ki].startswith("void at::"):  # bench.py's L2 flush (torch), not an engine kernel
            continue
        if "k_issue_peak" in r[ki]:  # bench.py's issue-peak microbenchmark, outside the timed steps
            continue
        v = float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    top = sorted(agg.items(), key=lambda x: -x[1][1])
    return {"total_us": tot, "launches": sum(c for c, _ in agg.values()),
            "kernels": [{"kernel": k, "launches": c, "us": v, "share": v / tot} for k, (c, v) in top[:25]]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("round")
    ap.add_argument("reports", nargs="*")
    ap.add_argument("--launches", nargs="*", default=[])
    a = ap.parse_args()
    outdir = os.path.join("profiles", a.round)
    os.makedirs(outdir, exist_ok=True)
    summary = {}
    for spec in a.reports:
        # path:tag (dominance kernels) or path:tag:stream (HBM streaming passes)
        parts = spec.split(":")
        path, tag = parts[0], parts[1]
        if len(parts) > 2 and parts[2] == "stream":
            summary.setdefault("stream", {})[tag] = summarize_report(path)
        else:
            summary[tag] = summarize_report(path)
    for spec in a.launches:
        path, tag = spec.split(":")
        summary[f"{tag}_launch_list"] = summarize_launches(path)
    with open(os.path.join(outdir, "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: (v if isinstance(v, dict) else [{kk: e.get(kk) for kk in ("kernel", "duration_ms",
                      "dram_traffic_bytes", "alu_pipe_pct", "fma_pipe_pct", "warps_active_pct")} for e in v])
                      for k, v in summary.items()}, indent=1)[:3000])


if __name__ == "__main__":
    main()
