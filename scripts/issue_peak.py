"""The dominance core's issue peak (sky_issue_peak) for every kernel shape:
K candidates per thread x CTAs per SM, at d = 6, 8, 10; one JSON line each."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2411_14968_b200 import Engine  # noqa: E402

e = Engine(0)
for d in (6, 10):
    for k in (1, 2, 4, 8):
        for cps in (1, 2, 4, 8):
            for iters in (2000,):
                t0 = time.perf_counter()
                v = e.issue_peak(d, k, cps, iters)
                print(json.dumps({"d": d, "k": k, "ctas_per_sm": cps, "iters": iters, "gtests_s": v / 1e9,
                                  "wall_s": time.perf_counter() - t0}), flush=True)
    print(json.dumps({"d": d, "best_gtests_s": e.issue_peak(d) / 1e9}), flush=True)
