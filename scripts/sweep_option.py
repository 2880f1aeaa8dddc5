"""Time one BASELINE config under values of one engine option (device-resident
input, CUDA events around sky_run, median of K runs after W warm-ups), with
the result checked against the first value's. Usage:
    python scripts/sweep_option.py CONFIG OPTION v1 v2 ... [--steps K]"""
import argparse
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2411_14968_b200 import Engine, generate  # noqa: E402
from paper_2411_14968_b200.configs import make_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("option")
ap.add_argument("values", type=int, nargs="+")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--warmup", type=int, default=2)
a = ap.parse_args()
w = make_config(a.config)
x = generate(w.kind, w.n, w.d, 42)
xd = torch.from_numpy(x).cuda()
e = Engine(0)
st = torch.cuda.current_stream()
e.set_stream(st.cuda_stream)
ref = None
e.set_option("kernel_events", 1)  # dom_kernel_ms in the output (25-55 us per step of event records)
for v in a.values:
    e.set_option(a.option, v)
    run = lambda: e.run(None, w.config, w.normalized, device_ptr=xd.data_ptr(), n=w.n, d=w.d)
    for _ in range(a.warmup):
        r = run()
    ms, dom, loc = [], [], []
    for _ in range(a.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        r = run()
        e1.record(st)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
        dom.append(r.metrics.dom_kernel_ms)
        loc.append(r.metrics.local_ms)
    if ref is None:
        ref = r.skyline
    print(json.dumps({"config": a.config, a.option: v, "ms": statistics.median(ms), "local_ms": statistics.median(loc),
                      "merge_ms": r.metrics.merge_ms, "dom_ms": statistics.median(dom),
                      "tests_local": r.metrics.tests_local, "same": bool(np.array_equal(ref, r.skyline)),
                      "lss0": r.metrics.local_skyline_sizes[:3]}), flush=True)
