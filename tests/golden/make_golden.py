"""Generate the golden fixtures from the REFERENCE ITSELF.

Runs the unmodified reference engine (oracle/_ref/libskyref.so, compiled in
place from /root/reference by `make -C oracle ref`) on:
  * the known-answer literals of the reference's own unit tests
    (proj/tests/test_core.cpp, test_partition.cpp, test_filter.cpp,
    test_sequential.cpp, test_engine.cpp), and
  * the five BASELINE configs at reduced N on sky_generate inputs
    (SHA-256 of the float32 input recorded),
and writes tests/golden/golden.json + tests/golden/configs.npz.

Usage (in the build container, where /root/reference exists):
    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2411_14968_b200.abi import SkyConfig  # noqa: E402
from paper_2411_14968_b200.configs import make_config  # noqa: E402
from paper_2411_14968_b200.skyline import generate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# reduced sizes: the single-threaded oracle must finish each in seconds
REDUCED_N = {1: 100_000, 2: 100_000, 3: 1_000_000, 4: 40_000, 5: 500_000}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


def known_answers():
    L = []

    def sky(rows, src):
        x = np.array(rows, np.float32)
        L.append({"kind": "skyline", "src": src, "points": x.tolist(),
                  "expect": O.bruteforce(x, ref=True).tolist()})

    sky([[1, 2], [2, 1], [2, 2]], "test_core.cpp:65-67")
    sky([[3, 3]], "test_core.cpp:72-74")
    sky([[1, 1], [1, 1], [2, 2]], "test_core.cpp:75-78")
    sky([[0.5, 0.5], [0.5, 0.5]], "test_sequential.cpp:54-56")

    def rel(r, c, src):
        r = np.array(r, np.float32)
        c = np.array(c, np.float32)
        L.append({"kind": "relative", "src": src, "r": r.tolist(), "c": c.tolist(),
                  "expect": O.relative_skyline(r, c, ref=True).astype(int).tolist()})

    rel([[2, 2], [3, 1]], [[1, 1]], "test_core.cpp:83-86")
    rel([[1, 2], [2, 1]], [[1, 2], [2, 1]], "test_core.cpp:91-94")
    rel([[2, 2], [0.5, 3]], [[1, 1]], "test_filter.cpp:136-141")
    rel([[2, 2], [1, 3]], [[2, 2], [1, 3]], "test_filter.cpp:147-153")

    ref = O.ref_lib()
    for pt, m, src in [([0.3, 0.7], 2, "test_partition.cpp:53"), ([0.0, 0.0], 2, "test_partition.cpp:54"),
                       ([0.0, 0.0], 5, "test_partition.cpp:55"), ([1.0, 1.0], 2, "test_partition.cpp:56")]:
        x = np.array(pt, np.float32)
        L.append({"kind": "grid_index", "src": src, "x": x.tolist(), "m": m,
                  "expect": int(ref.skyref_grid_index(x.ctypes.data_as(O._f32p), len(x), m))})
    for pt, m, src in [([1, 1], 4, "test_partition.cpp:137"), ([1, 0], 4, "test_partition.cpp:138"),
                       ([0, 1], 4, "test_partition.cpp:139")]:
        x = np.array(pt, np.float32)
        L.append({"kind": "angular_index", "src": src, "x": x.tolist(), "m": m,
                  "expect": int(ref.skyref_angular_index(x.ctypes.data_as(O._f32p), len(x), m))})
    for tp, k in [(16, 4), (120, 4), (120, 3), (120, 2), (120, 1), (1, 3), (64, 5), (256, 8)]:
        L.append({"kind": "snap", "src": "test_partition.cpp:228-234", "p": tp, "k": k,
                  "expect": int(ref.skyref_snap_slices(tp, k))})
    # sliced rank formula on rows (i/100, 0.5)
    x = np.array([[i / 100.0, 0.5] for i in range(100)], np.float32)
    po, cnt = O.oracle_assign(x, SkyConfig.make(strategy=3, p=4), True, ref=True)
    L.append({"kind": "assign", "src": "test_partition.cpp:153-162", "points": x.tolist(),
              "cfg": {"strategy": 3, "p": 4}, "normalized": True, "expect": po.astype(int).tolist(),
              "count": cnt})
    # grid engine example (test_engine.cpp:140-149)
    x = np.array([[0.1, 0.1], [0.6, 0.6], [0.7, 0.2], [0.2, 0.8]], np.float32)
    for strat, p in [(1, 4), (0, 2), (2, 4), (3, 3)]:
        for merge in (0, 1):
            cfg = SkyConfig.make(strategy=strat, p=p, seed=3, merge=merge)
            r = O.ref_run(x, cfg, True)
            L.append({"kind": "run", "src": "test_engine.cpp:140-149", "points": x.tolist(), "normalized": True,
                      "cfg": cfg.as_dict(), "expect": r["ids"].tolist(),
                      "local_skyline_sizes": r["local_skyline_sizes"].astype(int).tolist()})
    # reps (test_filter.cpp:68-85)
    x = np.array([[1, 2], [2, 1], [3, 3]], np.float32)
    L.append({"kind": "reps", "src": "test_filter.cpp:70-73", "points": x.tolist(), "partition_of": [0, 0, 0],
              "p": 1, "q": 2, "expect": O.representatives(x, [0, 0, 0], 1, 2, ref=True).tolist()})
    x = np.array([[1, 1], [2, 2]], np.float32)
    L.append({"kind": "reps", "src": "test_filter.cpp:79-82", "points": x.tolist(), "partition_of": [0, 1],
              "p": 2, "q": 1, "expect": O.representatives(x, [0, 1], 2, 1, ref=True).tolist()})
    return L


def lattice(n, d, levels, seed):
    """test_support.hpp:46-60 style lattice data (ties and duplicates)."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, levels + 1, (n, d)) / levels).astype(np.float32)


def plane():
    """A slice of the reference's configuration plane (test_engine.cpp:16-46,
    acceptance.cpp:54-114) on smooth and lattice data."""
    out = []
    arrays = {}
    k = 0
    for dist in ("uniform", "lattice", "ints"):
        for d in (2, 3, 5, 8):
            for n in (60, 700):
                rng = np.random.default_rng(1000 + 10 * d + n)
                if dist == "uniform":
                    x = rng.random((n, d), dtype=np.float32)
                elif dist == "lattice":
                    x = lattice(n, d, 4, 2000 + d + n)
                else:
                    x = rng.integers(0, 6, (n, d)).astype(np.float32)
                norm = dist != "ints"
                for strat in (0, 1, 2, 3):
                    if strat == 1 and not norm:
                        continue
                    filters = (0, 2, 1) if strat == 1 else (0, 2)
                    for filt in filters:
                        for merge in (0, 1):
                            # representative selection: Sorted, Region (normalized only), Random
                            sels = ((0, 1, 2) if norm else (0, 2)) if filt == 2 else (0,)
                            for q, sel in [(3 if filt == 2 else 5, sel) for sel in sels]:
                                cfg = SkyConfig.make(strategy=strat, p=7, seed=11, slice_dim=d - 1, filter=filt,
                                                     rep_q=q, merge=merge, workers=4, rep_selection=sel)
                                r = O.ref_run(x, cfg, norm)
                                key = f"plane{k}"
                                arrays[key + "_x"] = x
                                arrays[key + "_ids"] = r["ids"]
                                arrays[key + "_lss"] = r["local_skyline_sizes"].astype(np.int64)
                                out.append({"key": key, "dist": dist, "n": n, "d": d, "normalized": norm,
                                            "cfg": cfg.as_dict(), "effective_p": r["effective_p"],
                                            "union_size": r["union_size"], "filtered_count": r["filtered_count"],
                                            "final_size": r["final_size"]})
                                k += 1
    return out, arrays


def plane64():
    """FP64 inputs (the reference's own coordinate type): the reference's
    generators (datagen.cpp:16-57) and a k/7 lattice (ties, not float32)."""
    out = []
    arrays = {}
    k = 0
    for dist in ("uniform", "correlated", "anticorrelated", "lattice7"):
        for d in (2, 4, 7):
            n = 500
            if dist == "lattice7":
                x = np.random.default_rng(77 + d).integers(0, 8, (n, d)) / 7.0
            else:
                x = O.ref_generate({"uniform": 0, "correlated": 1, "anticorrelated": 2}[dist], n, d, 40 + d)
            xkey = f"p64_{dist}_{d}_x"
            arrays[xkey] = x
            for strat in (0, 1, 2, 3):
                for filt in ((0, 2, 1) if strat == 1 else (0, 2)):
                    for sel in ((0, 1, 2) if filt == 2 else (0,)):
                        for merge in (0, 1):
                            cfg = SkyConfig.make(strategy=strat, p=7, seed=13, slice_dim=d - 1, filter=filt,
                                                 rep_q=3, merge=merge, workers=4, rep_selection=sel)
                            r = O.ref_run(x, cfg, True)
                            key = f"p64c{k}"
                            arrays[key + "_ids"] = r["ids"]
                            arrays[key + "_lss"] = r["local_skyline_sizes"].astype(np.int64)
                            out.append({"key": key, "x": xkey, "dist": dist, "n": n, "d": d, "normalized": True,
                                        "cfg": cfg.as_dict(), "effective_p": r["effective_p"],
                                        "union_size": r["union_size"], "filtered_count": r["filtered_count"],
                                        "final_size": r["final_size"]})
                            k += 1
    return out, arrays


INGEST_CASES = [
    # (name, csv text, columns, maximize)
    ("plain", "a,b,c\n1,2,3\n4,5,6\n7,8,9\n", None, None),
    ("trim_cr_blank", " a , b \r\n1.5, 2\r\n\r\n  \n3 ,4.25\r\n-1,0\r\n", None, None),
    ("bad_rows", "x,y\n1,2\nfoo,3\n4,\n5\n6,7,8\n1e3,nan\ninf,1\n9,10\n", None, None),
    ("select_max", "p,q,r\n1,10,100\n2,30,50\n3,20,75\n", ["r", "p"], ["r"]),
    ("constant_col", "u,v\n5,1\n5,2\n5,3\n", None, None),
    ("precision", "a,b\n0.1,0.7\n0.2,0.30000000000000004\n1e-300,2.5e10\n", None, None),
    ("unknown_col", "a,b\n1,2\n", ["zz"], None),
    ("empty", "", None, None),
    ("no_rows", "a,b\nq,r\n", None, None),
]


def dataio():
    """The steps either side of the path: the reference's
    generators, CSV ingest and CSV output."""
    import tempfile
    gens = []
    for dist in (0, 1, 2):
        for n, d, seed in ((1000, 1, 0), (2000, 3, 7), (500, 8, 123456789), (3000, 5, 2 ** 63 + 5)):
            x = O.ref_generate(dist, n, d, seed)
            gens.append({"dist": dist, "n": n, "d": d, "seed": seed,
                         "sha256": hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
                         "head": x[:3].tolist()})
    ingest = []
    with tempfile.TemporaryDirectory() as td:
        for name, text, cols, mx in INGEST_CASES:
            path = os.path.join(td, name + ".csv")
            with open(path, "w", newline="") as f:
                f.write(text)
            case = {"name": name, "text": text, "columns": cols, "maximize": mx}
            try:
                r = O.ref_ingest_csv(path, cols, mx)
                case["rows_hex"] = [[v.hex() for v in row] for row in r.tolist()]
                case["shape"] = list(r.shape)
            except O.CpuError as e:
                case["error"] = e.code
            ingest.append(case)
        rows = O.ref_generate(2, 50, 4, 99)
        rows[0, 0] = 1e-7
        rows[1, 1] = 123456.0
        rows[2, 2] = 0.0
        path = os.path.join(td, "w.csv")
        O.ref_write_csv(path, rows)
        wcsv = {"rows_hex": [[v.hex() for v in r] for r in rows.tolist()], "text": open(path).read()}
        # skyline-cli generate: the reference's generate() + write_csv() bytes
        gen_csv = []
        for dist, n, d, seed in ((2, 200, 3, 5), (0, 100, 6, 0), (1, 150, 2, 77)):
            path = os.path.join(td, f"g{dist}.csv")
            O.ref_write_csv(path, O.ref_generate(dist, n, d, seed))
            gen_csv.append({"dist": dist, "n": n, "d": d, "seed": seed,
                            "sha256": hashlib.sha256(open(path, "rb").read()).hexdigest()})
    # skyline-cli run: the reference's run() on its own generated data
    cli = []
    for gen, flags in ((("anticorrelated", 20000, 4, 3), dict(strategy=2, filter=2, merge=1, p=16)),
                       (("uniform", 5000, 3, 9), dict(strategy=0, filter=0, merge=0, p=8)),
                       (("correlated", 8000, 5, 1), dict(strategy=3, filter=2, merge=1, p=12, rep_selection=2)),
                       (("anticorrelated", 6000, 2, 4), dict(strategy=1, filter=1, merge=1, p=9))):
        dist = {"uniform": 0, "correlated": 1, "anticorrelated": 2}[gen[0]]
        x = O.ref_generate(dist, gen[1], gen[2], gen[3])
        cfg = SkyConfig.make(seed=gen[3], rep_q=5, workers=1, **flags)
        r = O.ref_run(x, cfg, True)
        cli.append({"gen": list(gen), "cfg": cfg.as_dict(), "ids": r["ids"].tolist(),
                    "effective_p": r["effective_p"], "union_size": r["union_size"],
                    "filtered_count": r["filtered_count"], "final_size": r["final_size"]})
    return {"generate": gens, "ingest": ingest, "write_csv": wcsv, "generate_csv": gen_csv, "cli_run": cli}


def acceptance():
    """The reference's acceptance criteria 3-7 (tests/acceptance/acceptance.cpp:
    200-378) measured by the reference itself on its own generated data: the
    GPU suite must reproduce every count, so it passes or fails exactly where
    the reference does."""
    import time
    out = {"c3": [], "c4": [], "c5": {}, "c6": {}, "c7": []}
    for dist in (0, 1, 2):
        for m in (4, 8):
            for seed in (1, 2, 3):
                x = O.ref_generate(dist, 100000, 4, seed)
                r = O.ref_run(x, SkyConfig.make(strategy=1, m=m, p=1, filter=1, workers=2), True)
                out["c3"].append({"dist": dist, "m": m, "seed": seed, "filtered": r["filtered_count"]})
        for seed in (1, 2, 3):
            x = O.ref_generate(dist, 100000, 4, seed)
            for sel in (0, 1):
                r = O.ref_run(x, SkyConfig.make(strategy=0, p=8, seed=seed, filter=2, rep_selection=sel, rep_q=3,
                                                workers=2), True)
                out["c4"].append({"dist": dist, "seed": seed, "sel": sel, "filtered": r["filtered_count"]})
    x = O.ref_generate(2, 1000000, 4, 1)
    for strat in (0, 1, 2, 3):
        r = O.ref_run(x, SkyConfig.make(strategy=strat, p=120, seed=1, workers=2), True)
        out["c5"][str(strat)] = r["union_size"]
    for name, kw, w in (("sliced+_1", dict(filter=2, merge=0), 1), ("sliced+_8", dict(filter=2, merge=0), 8),
                        ("noseq_8", dict(filter=0, merge=1), 8)):
        r = O.ref_run(x, SkyConfig.make(strategy=3, p=120, rep_q=5, workers=w, **kw), True)
        out["c6"][name] = {"local_merge_ms": r["local_ms"] + r["merge_ms"], "final_size": r["final_size"],
                           "union_size": r["union_size"], "filtered": r["filtered_count"]}
    x = O.ref_generate(2, 100000, 4, 1)
    for p in (8, 64, 512):
        r = O.ref_run(x, SkyConfig.make(strategy=3, p=p, workers=2), True)
        out["c7"].append({"p": p, "union_size": r["union_size"]})
    out["host_threads"] = O.ref_lib().skyref_hardware_concurrency()
    return out


def configs():
    out = []
    arrays = {}
    for i in range(1, 6):
        w = make_config(i, REDUCED_N[i])
        x = generate(w.kind, w.n, w.d, 42)
        cfg = w.config.to_c()
        cfg.workers = 8
        r = O.ref_run(x, cfg, w.normalized)
        arrays[f"c{i}_ids"] = r["ids"]
        arrays[f"c{i}_lss"] = r["local_skyline_sizes"].astype(np.int64)
        out.append({"config": i, "name": w.name, "n": w.n, "d": w.d, "kind": w.kind, "seed": 42,
                    "normalized": w.normalized, "sha256": sha(x), "cfg": cfg.as_dict(),
                    "effective_p": r["effective_p"], "union_size": r["union_size"],
                    "filtered_count": r["filtered_count"], "final_size": r["final_size"],
                    "ref_run_ms": r["run_ms"]})
        print(w.name, r["final_size"], r["union_size"], r["filtered_count"], f"{r['run_ms']:.0f} ms", flush=True)
    return out, arrays


def main():
    O.build(ref=True)
    ka = known_answers()
    pl, pl_arr = plane()
    p64, p64_arr = plane64()
    dio = dataio()
    acc = acceptance()
    if "--keep-configs" in sys.argv:
        # reuse the (slow) BASELINE-config fixtures already committed
        with open(os.path.join(HERE, "golden.json")) as f:
            cf = json.load(f)["configs"]
        cf_arr = dict(np.load(os.path.join(HERE, "configs.npz")))
    else:
        cf, cf_arr = configs()
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "source": "oracle/_ref/libskyref.so "
                   "(unmodified /root/reference/proj/src)", "known_answers": ka, "plane": pl, "plane64": p64, "dataio": dio, "acceptance": acc, "configs": cf}, f)
    np.savez_compressed(os.path.join(HERE, "plane64.npz"), **p64_arr)
    np.savez_compressed(os.path.join(HERE, "plane.npz"), **pl_arr)
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **cf_arr)
    print(len(ka), "known answers;", len(pl), "plane cases;", len(cf), "configs")


if __name__ == "__main__":
    main()
