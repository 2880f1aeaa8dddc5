"""Full-size goldens for the five BASELINE configs, from the REFERENCE ITSELF.

Runs the unmodified reference engine (oracle/_ref/libskyref.so, compiled in
place from /root/reference by `make -C oracle ref`) at BASELINE.json's full
sizes on the exact float32 inputs the GPU path consumes
(`skyref_generate_baseline`, include/skyline_baseline_gen.h, seed 42), with
workers = the host's hardware threads, and writes

  tests/golden/full/c{i}.json   effective_p, union_size, filtered_count,
                                final_size, local_skyline_sizes, input and
                                ids SHA-256, reference run time and threads
  tests/golden/full/c{i}.npz    the skyline as a packed membership bitmap
                                over row ids (np.packbits, compressed)

C4 (4M x 10, sliced NoSeq) takes ~25 minutes on 8 cores; the others seconds.
The reference has no BNL, so C4's golden comes from its SFS local phase: the
local skylines (and so every metric) are the same sets.

Usage (in the build container, where /root/reference exists):
    python tests/golden/make_full_golden.py [1 2 3 4 5]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2411_14968_b200.configs import make_config  # noqa: E402  (pure Python; loads no library)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "full")


def main(which):
    O.build(ref=True)
    os.makedirs(OUT, exist_ok=True)
    threads = O.ref_lib().skyref_hardware_concurrency()
    for i in which:
        w = make_config(i)
        x = O.ref_generate_baseline(w.kind, w.n, w.d, 42)
        cfg = w.config.to_c()
        cfg.workers = threads
        t0 = time.time()
        r = O.ref_run(x, cfg, w.normalized)
        wall = time.time() - t0
        ids = np.ascontiguousarray(r["ids"], np.int64)
        mask = np.zeros(w.n, bool)
        mask[ids] = True
        np.savez_compressed(os.path.join(OUT, f"c{i}.npz"), bitmap=np.packbits(mask))
        meta = {"config": i, "name": w.name, "n": w.n, "d": w.d, "kind": w.kind, "seed": 42,
                "normalized": w.normalized, "cfg": cfg.as_dict(),
                "input_sha256": hashlib.sha256(x.tobytes()).hexdigest(),
                "ids_sha256": hashlib.sha256(ids.tobytes()).hexdigest(),
                "effective_p": r["effective_p"], "union_size": r["union_size"],
                "filtered_count": r["filtered_count"], "final_size": r["final_size"],
                "local_skyline_sizes": r["local_skyline_sizes"].astype(int).tolist(),
                "ref_run_ms": r["run_ms"], "ref_phase_ms": {"partition": r["partition_ms"], "local": r["local_ms"],
                                                            "merge": r["merge_ms"]},
                "ref_threads": threads, "wall_s": wall,
                "source": "oracle/_ref/libskyref.so (unmodified /root/reference/proj/src), "
                          "tests/golden/make_full_golden.py"}
        with open(os.path.join(OUT, f"c{i}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        print(w.name, "final", r["final_size"], "union", r["union_size"], "filtered", r["filtered_count"],
              f"{r['run_ms'] / 1e3:.1f} s", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 5, 4])
