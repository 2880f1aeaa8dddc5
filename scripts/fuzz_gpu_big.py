"""Randomised parity at BASELINE-like sizes (100k - 1.5M rows, d <= 8): the
GPU engine with its default options (stream path above 32 MB, device-planned
merges, indexed merge) against the reference itself (oracle/_ref, all host
threads). Usage: python scripts/fuzz_gpu_big.py [cases] [seed] [budget_s]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2411_14968_b200 import (Engine, EngineConfig, FilterKind, LocalAlgo, MergeKind, PartitionConfig,
                                   RepSelection, Strategy, generate)
from paper_2411_14968_b200.abi import SkyConfig

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
budget_s = float(sys.argv[3]) if len(sys.argv) > 3 else 1e9
assert O.ref_available(), "oracle/_ref/libskyref.so was not built"
rng = np.random.default_rng(seed)
world = int(os.environ.get("FUZZ_WORLD", "1"))
eng = Engine(0) if world == 1 else Engine.group([0] * world, loopback=True)
workers = os.cpu_count() or 8
bad = done = 0
t_start = time.time()
for it in range(cases):
    if time.time() - t_start > budget_s:
        break
    d = int(rng.choice([3, 4, 5, 6, 8]))
    n = int(rng.choice([100_000, 300_000, 1_000_000, 1_500_000]))
    kind = int(rng.choice([1, 3, 3, 5, 2]))          # BASELINE generators; anti-correlated only when small
    if kind == 2 and n > 300_000:
        kind = 3
    x = generate(kind, n, d, int(rng.integers(1 << 30)))
    norm = kind != 5
    strat = int(rng.integers(0, 4))
    filt = int(rng.choice([0, 2, 2] + ([1] if strat == 1 else [])))
    if strat == 1:
        m = int(rng.choice([2, 3, 4]))
        while m ** d > 5000 and m > 1:
            m -= 1
        p = m ** d
    else:
        p = int(rng.choice([8, 32, 128, 500]))
    if kind == 5 and strat == 1:
        strat = 0                                    # integers are not in [0,1]: grid raises (covered elsewhere)
        p = 32
        if filt == 1:
            filt = 2
    q = int(rng.choice([1, 5, 8, 20]))
    sel = int(rng.choice([0, 0, 1, 2])) if filt == 2 else 0
    if sel == 1 and not norm:
        sel = 0
    merge = int(rng.integers(0, 2))
    cfg = SkyConfig.make(strategy=strat, p=p, seed=int(rng.integers(0, 1000)), slice_dim=int(rng.integers(0, d)),
                         filter=filt, rep_q=q, merge=merge, workers=workers, rep_selection=sel)
    ecfg = EngineConfig(partition=PartitionConfig(Strategy(strat), p, 0, cfg.seed, cfg.slice_dim),
                        filter=FilterKind(filt), rep_q=q, merge=MergeKind(merge), rep_selection=RepSelection(sel),
                        seed=cfg.rep_seed, local_algo=LocalAlgo(it % 2), bnl_window_cap=4096)
    tag = dict(it=it, n=n, d=d, kind=kind, strat=strat, p=p, filt=filt, q=q, sel=sel, merge=merge, algo=it % 2)
    print("CASE", tag, flush=True)
    t0 = time.time()
    exp = O.ref_run(x, cfg, norm)
    t1 = time.time()
    try:
        r = eng.run(x, ecfg, norm)
    except Exception as ge:
        bad += 1
        print("FAIL", tag, type(ge).__name__, ge, flush=True)
        done += 1
        continue
    t2 = time.time()
    ok = (np.array_equal(r.skyline, exp["ids"]) and r.metrics.union_size == exp["union_size"]
          and r.metrics.filtered_count == exp["filtered_count"] and r.effective_p == exp["effective_p"]
          and r.metrics.local_skyline_sizes == exp["local_skyline_sizes"].astype(int).tolist())
    print(f"  {'ok' if ok else 'MISMATCH'} |Sky|={r.skyline.size} union={r.metrics.union_size} "
          f"filtered={r.metrics.filtered_count} ref {t1 - t0:.2f} s gpu {1e3 * (t2 - t1):.1f} ms", flush=True)
    bad += 0 if ok else 1
    done += 1
print(f"cases {done} bad {bad} in {time.time() - t_start:.0f} s")
sys.exit(1 if bad else 0)
