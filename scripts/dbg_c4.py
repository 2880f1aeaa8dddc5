import dataclasses, json, sys
import numpy as np
sys.path.insert(0, '.')
from paper_2411_14968_b200 import Engine, generate, LocalAlgo
from paper_2411_14968_b200.configs import make_config
w = make_config(4)
x = generate(w.kind, w.n, w.d, 42)
g = json.load(open('tests/golden/full/c4.json'))
gl = g["local_skyline_sizes"]
def rep(tag, r):
    d = [(i, a, b) for i, (a, b) in enumerate(zip(r.metrics.local_skyline_sizes, gl)) if a != b]
    print(tag, "final", r.metrics.final_size, "union", r.metrics.union_size, "filtered", r.metrics.filtered_count,
          "nreps", r.metrics.n_reps, "diff", d, flush=True)
single = Engine(0)
rep("single", single.run(x, w.config, w.normalized))
single.set_sharded(True)
for algo in (LocalAlgo.BNL, LocalAlgo.SFS):
    cfg = dataclasses.replace(w.config, local_algo=algo)
    rep(f"W1-sharded {algo.name}", single.run(x, cfg, w.normalized))
for W in (2, 3, 4):
    e = Engine.group([0] * W, loopback=True)
    for algo in (LocalAlgo.BNL, LocalAlgo.SFS):
        cfg = dataclasses.replace(w.config, local_algo=algo)
        for rep_i in range(2):
            rep(f"W{W} {algo.name} #{rep_i}", e.run(x, cfg, w.normalized))
    e.close()
