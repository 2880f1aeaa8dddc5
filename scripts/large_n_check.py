"""Large-N sanity: BASELINE families beyond their sizes, one GPU and two
sharded ranks; checks ids sorted/unique, equal across both runs, no sampled
output row dominated by any input row (GPU relative skyline), every sampled
non-output row dominated."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2411_14968_b200 import (Engine, EngineConfig, FilterKind, LocalAlgo, MergeKind, PartitionConfig,
                                   Strategy)

e1 = Engine(0)
e2 = Engine.group([0, 0], loopback=True)
rng = np.random.default_rng(1)
cases = [
    (3, 40_000_000, 8, EngineConfig(partition=PartitionConfig(Strategy.Grid, p=256), filter=FilterKind.Representative,
                                    rep_q=5, merge=MergeKind.NoSeq)),
    (2, 8_000_000, 6, EngineConfig(partition=PartitionConfig(Strategy.Angular, p=64), filter=FilterKind.Representative,
                                   rep_q=8, merge=MergeKind.NoSeq)),
    (4, 6_000_000, 10, EngineConfig(partition=PartitionConfig(Strategy.Sliced, p=128), filter=FilterKind.Representative,
                                    rep_q=5, merge=MergeKind.NoSeq, local_algo=LocalAlgo.BNL)),
    (5, 20_000_000, 5, EngineConfig(partition=PartitionConfig(Strategy.Random, p=32, seed=3),
                                    filter=FilterKind.Representative, rep_q=5, merge=MergeKind.NoSeq)),
]
for kind, n, d, cfg in cases:
    x = torch.empty((n, d), dtype=torch.float32, device="cuda:0")
    e1.generate_device(kind, n, d, 42, x.data_ptr())
    torch.cuda.synchronize()
    xh = x.cpu().numpy()
    # one untimed run first: buffers grow to this size and the random
    # partitioner builds its jump polynomials once per process (~0.8 s of
    # host time at 20M rows)
    e1.run(None, cfg, kind != 5, device_ptr=x.data_ptr(), n=n, d=d)
    e2.run(xh, cfg, kind != 5)
    t0 = time.perf_counter()
    r1 = e1.run(None, cfg, kind != 5, device_ptr=x.data_ptr(), n=n, d=d)
    t1 = time.perf_counter()
    r2 = e2.run(xh, cfg, kind != 5)
    t2 = time.perf_counter()
    ids = r1.skyline
    ok = bool(np.all(np.diff(ids) > 0)) and np.array_equal(ids, r2.skyline) and \
        r1.metrics.local_skyline_sizes == r2.metrics.local_skyline_sizes and \
        r1.metrics.filtered_count == r2.metrics.filtered_count
    out = rng.choice(ids, min(200, ids.size), replace=False)
    keep = e1.relative_skyline(xh[out], xh)  # no input row dominates an output row
    non = np.setdiff1d(rng.integers(0, n, 400), ids)[:200]
    dom = ~e1.relative_skyline(xh[non], xh[ids])  # each non-output row has a dominator in the skyline
    print(f"kind {kind} n={n} d={d}: |Sky|={ids.size} union={r1.metrics.union_size} gpu {r1.metrics.total_ms:.2f} ms "
          f"(wall {1e3*(t1-t0):.1f} ms, 2 ranks {1e3*(t2-t1):.1f} ms) consistent={ok} "
          f"outputs undominated={bool(keep.all())} non-outputs dominated={bool(dom.all())}", flush=True)
    del x
    torch.cuda.empty_cache()
