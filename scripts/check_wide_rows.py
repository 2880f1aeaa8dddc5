"""d > 16 (the exact-compare core): every strategy x filter x merge x local
algorithm against the oracle on small inputs. Prints the failing cases."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2411_14968_b200 import Engine, EngineConfig, FilterKind, LocalAlgo, MergeKind, PartitionConfig, RepSelection, Strategy
from paper_2411_14968_b200.abi import SkyConfig
eng = Engine(0)
rng = np.random.default_rng(5)
bad = 0
for d in (17, 20, 24, 32):
    for n in (1, 700, 6000):
        x = rng.random((n, d), dtype=np.float32)
        x[:, : d - 3] = np.round(x[:, : d - 3] * 2) / 2  # few distinct values: a skyline smaller than the input
        for strat in range(4):
            for filt in ((0, 1, 2) if strat == 1 else (0, 2)):
                for merge in (0, 1):
                    for algo in (0, 1):
                        for sel in ((0, 1, 2) if filt == 2 else (0,)):
                            p = 2 ** 17 if (strat == 1 and d == 17) else (2 ** d if strat == 1 and d <= 20 else 9)
                            cfg = SkyConfig.make(strategy=strat, p=p, seed=3, slice_dim=d - 1, filter=filt, rep_q=4,
                                                 merge=merge, workers=1, rep_selection=sel)
                            ecfg = EngineConfig(partition=PartitionConfig(Strategy(strat), p, 0, 3, d - 1),
                                                filter=FilterKind(filt), rep_q=4, merge=MergeKind(merge),
                                                rep_selection=RepSelection(sel), seed=3, local_algo=LocalAlgo(algo),
                                                bnl_window_cap=64)
                            tag = (d, n, strat, filt, merge, algo, sel)
                            try:
                                exp = O.oracle_run(x, cfg, True)
                            except O.CpuError as e:
                                continue
                            try:
                                r = eng.run(x, ecfg, True)
                            except Exception as e:
                                bad += 1
                                print("FAIL", tag, type(e).__name__, e, flush=True)
                                continue
                            ok = (np.array_equal(r.skyline, exp["ids"]) and r.metrics.union_size == exp["union_size"]
                                  and r.metrics.filtered_count == exp["filtered_count"]
                                  and r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist())
                            if not ok:
                                bad += 1
                                print("MISMATCH", tag, r.skyline.size, len(exp["ids"]), flush=True)
print("bad", bad)
