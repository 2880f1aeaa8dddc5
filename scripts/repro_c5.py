import sys, dataclasses, json
sys.path.insert(0, '.')
import numpy as np
from paper_2411_14968_b200 import Engine, generate, LocalAlgo
from paper_2411_14968_b200.configs import make_config
g = json.load(open('tests/golden/golden.json'))
c = [c for c in g["configs"] if c["config"] == 5][0]
x = generate(c["kind"], c["n"], c["d"], c["seed"])
w = make_config(5)
e = Engine(0)
cfg = dataclasses.replace(w.config, local_algo=LocalAlgo.BNL)
r = e.run(x, cfg, c["normalized"])
print("ok", r.metrics.union_size, c["union_size"])
