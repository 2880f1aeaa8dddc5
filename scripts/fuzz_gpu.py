"""Randomised parity sweep on the GPU against the oracle: wider ranges than
the test suite (d 1..32, up to 60k rows, thousands of partitions, large q,
FP64 rows, duplicate-heavy and unnormalised data, forced stream path and
merge options). Usage: python scripts/fuzz_gpu.py [cases] [seed]. Prints
every failing case; exit code 1 if any."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2411_14968_b200 import (Engine, EngineConfig, FilterKind, LocalAlgo, MergeKind, PartitionConfig,
                                   RepSelection, Strategy, generate)
from paper_2411_14968_b200.abi import SkyConfig

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 600
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
budget_s = float(sys.argv[3]) if len(sys.argv) > 3 else 1e9
rng = np.random.default_rng(seed)
world = int(os.environ.get("FUZZ_WORLD", "1"))  # > 1: a loopback group of ranks on GPU 0 (the multi-rank engine)
eng = Engine(0) if world == 1 else Engine.group([0] * world, loopback=True)
bad = 0
only = {int(v) for v in os.environ.get("FUZZ_ONLY", "").split(",") if v}  # rerun these iterations only
t_start = time.time()
done = 0
for it in range(cases):
    if time.time() - t_start > budget_s:
        break
    d = int(rng.choice([1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 15, 16, 17, 20, 32]))
    n = int(rng.choice([0, 1, 2, 33, 257, 1000, 5000, 20000, 60000], p=[.03, .03, .04, .1, .15, .25, .2, .15, .05]))
    if d > 12 and n > 5000:
        n = 5000
    kind = int(rng.integers(0, 6))
    f64 = False
    if kind == 0:
        x = rng.random((n, d), dtype=np.float32)
    elif kind == 1:
        x = (rng.integers(0, 4, (n, d)) / 3).astype(np.float32)       # lattice, many duplicates and ties
    elif kind == 2:
        x = rng.integers(0, 9, (n, d)).astype(np.float32)             # unnormalised integers
    elif kind == 3:
        x = generate(2, max(n, 1), d, it)[:n] if d > 1 else rng.random((n, d), dtype=np.float32)
    elif kind == 4:
        x = generate(3, max(n, 1), d, it)[:n] if d > 1 else rng.random((n, d), dtype=np.float32)
    else:
        f64 = True
        base = rng.integers(0, 1 << 12, (n, d)) / float(1 << 12)
        x = np.clip(base + rng.integers(-2, 3, (n, d)) * 2.0 ** -40, 0.0, 1.0)
    norm = kind != 2
    strat = int(rng.integers(0, 4))
    filt = int(rng.choice([0, 2, 2] + ([1] if strat == 1 else [])))
    if strat == 1:
        m = int(rng.choice([1, 2, 3, 4, 7]))
        while m ** d > 300000 and m > 1:
            m -= 1
        p = m ** d
    else:
        p = int(rng.choice([1, 2, 7, 32, 100, 1000, 5000]))
    q = int(rng.choice([1, 2, 5, 8, 30, 100]))
    sel = int(rng.integers(0, 3)) if filt == 2 else 0
    merge = int(rng.integers(0, 2))
    cfg = SkyConfig.make(strategy=strat, p=p, seed=int(rng.integers(0, 1000)), slice_dim=int(rng.integers(0, d)),
                         filter=filt, rep_q=q, merge=merge, workers=1, rep_selection=sel)
    ecfg = EngineConfig(partition=PartitionConfig(Strategy(strat), p, 0, cfg.seed, cfg.slice_dim),
                        filter=FilterKind(filt), rep_q=q, merge=MergeKind(merge), rep_selection=RepSelection(sel),
                        seed=cfg.rep_seed, local_algo=LocalAlgo(it % 2),
                        bnl_window_cap=int(rng.choice([16, 64, 512, 4096])))
    opts = {"stream": int(rng.choice([-1, 0, 1])), "host_merge": int(rng.integers(0, 2)),
            "cap_sync": int(rng.choice([-1, 0, 1])), "small_tail": int(rng.integers(0, 2)),
            "merge_index": int(rng.integers(0, 2))}
    if world == 1:
        eng.reset_options()
        for k, v in opts.items():
            eng.set_option(k, v)
    tag = dict(it=it, n=n, d=d, kind=kind, strat=strat, p=p, filt=filt, q=q, sel=sel, merge=merge, algo=it % 2,
               win=ecfg.bnl_window_cap, **opts)
    if only and it not in only:
        continue
    if os.environ.get("FUZZ_TRACE"):
        print("CASE", tag, flush=True)
    try:
        exp = O.oracle_run(x, cfg, norm)
    except O.CpuError as e:
        try:
            eng.run(x, ecfg, norm)
            bad += 1
            print("NOERROR", tag, "oracle raised", e.code, flush=True)
        except Exception as ge:
            if getattr(ge, "code", None) != e.code:
                bad += 1
                print("ERRCODE", tag, e.code, getattr(ge, "code", None), ge, flush=True)
        done += 1
        continue
    try:
        r = eng.run(x, ecfg, norm)
    except Exception as ge:
        bad += 1
        print("FAIL", tag, type(ge).__name__, ge, flush=True)
        done += 1
        continue
    ok = (np.array_equal(r.skyline, exp["ids"]) and r.metrics.union_size == exp["union_size"]
          and r.metrics.filtered_count == exp["filtered_count"] and r.effective_p == exp["effective_p"]
          and r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist())
    if not ok:
        bad += 1
        print("MISMATCH", tag, r.skyline.size, len(exp["ids"]), r.metrics.union_size, exp["union_size"],
              r.metrics.filtered_count, exp["filtered_count"], flush=True)
    done += 1
print(f"cases {done} bad {bad} in {time.time() - t_start:.0f} s")
sys.exit(1 if bad else 0)
